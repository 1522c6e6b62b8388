"""Build register-budget variants of the CUDA library into build/variants/
(select one at run time with LFP_LIB_PATH=...)."""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import __graft_entry__ as g  # noqa: E402

out = os.path.join(REPO, "build", "variants")
os.makedirs(out, exist_ok=True)
srcs = [os.path.join(g.CSRC, "lfp_capi.cu"), os.path.join(g.CSRC, "lfp_bake.cu")]
# arguments: nested budgets ("4") or persistent budgets ("p3")
for mb in sys.argv[1:] or ["1", "2", "3", "4", "5"]:
    if "=" in mb:   # explicit macro list: NAME=VAL[,NAME=VAL...]
        defs = [f"-D{kv}" for kv in mb.split(",")]
        lib = os.path.join(out, "liblfprobe_b200_" +
                           mb.replace("=", "").replace(",", "_") + ".so")
        subprocess.run([g._nvcc(), *g.NVCC_FLAGS, *defs, "-Xptxas", "-v",
                        "-o", lib, *srcs], check=True,
                       stderr=open(lib + ".ptxas.txt", "w"))
        print(lib)
        continue
    macro = {"p": "LFP_PERSIST_MIN_BLOCKS", "s": "LFP_MERGED_SEGMENT",
             "c": "LFP_CF_SMEM", "h": "LFP_MIN_BLOCKS_HI_RES",
             "b": "LFP_BAKE_FAST"}.get(mb[0], "LFP_MIN_BLOCKS")
    val = mb.lstrip("pschb")
    lib = os.path.join(out, f"liblfprobe_b200_mb{mb}.so")
    subprocess.run([g._nvcc(), *g.NVCC_FLAGS, f"-D{macro}={val}",
                    "-Xptxas", "-v", "-o", lib, *srcs], check=True,
                   stderr=open(lib + ".ptxas.txt", "w"))
    print(lib)
