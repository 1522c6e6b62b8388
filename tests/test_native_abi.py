"""CPU-side checks of the drop-in boundary: the CUDA library is built for
sm_100a, loads without a GPU and exports every symbol the header declares;
the package never imports the oracle."""

import ctypes
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "lfprobe_b200.h")


@pytest.fixture(scope="module")
def lib_path():
    import __graft_entry__
    __graft_entry__.build()
    return __graft_entry__.LIB


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(lfp_\w+)\(",
                                 src, re.M)))


def test_header_declares_expected_api():
    names = header_functions()
    for n in ("lfp_probeset_create", "lfp_probeset_destroy",
              "lfp_render_cameras", "lfp_render_grid", "lfp_trace_rays",
              "lfp_last_error", "lfp_untile"):
        assert n in names


def test_library_exports_every_header_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in header_functions():
        assert hasattr(lib, name), f"{name} missing from {lib_path}"
    from paper_2507_14624_b200 import native
    assert sorted(native.exported_symbols()) == header_functions()


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_without_gpu(lib_path):
    lib = ctypes.CDLL(lib_path)
    assert lib.lfp_version() >= 100
    lib.lfp_last_error.restype = ctypes.c_char_p
    lib.lfp_probeset_destroy.argtypes = [ctypes.c_void_p]
    assert lib.lfp_probeset_destroy(None) == 0
    # invalid arguments fail loudly with a message, never crash
    lib.lfp_probeset_create.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 5 + [
        ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32,
        ctypes.c_void_p, ctypes.c_void_p]
    out = ctypes.c_void_p()
    rc = lib.lfp_probeset_create(0, None, None, None, None, None, 1, 32, 8, 0,
                                 None, ctypes.byref(out))
    assert rc == -1
    assert b"null" in lib.lfp_last_error()
    lib.lfp_num_tiles.restype = ctypes.c_int64
    assert lib.lfp_num_tiles(2, 100, 77) == 2 * 13 * 5


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2507_14624_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(root, f)).read()
                assert not re.search(
                    r"^\s*(from\s+oracle|import\s+oracle)|liblfp_oracle|lfpo_",
                    src, re.M), f


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2507_14624_b200 import configs, render_frame
    from paper_2507_14624_b200.native import LfpError
    cfg = configs.c1()
    with pytest.raises(LfpError):
        render_frame(cfg.grid, cfg.cameras[0])
