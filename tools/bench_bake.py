"""Point-cloud bake benchmark (bake.py:140-207,
grid.py:96-109): bake the C3 probe lattice (8x4x8 probes, cell 1 m,
256^2 / 64^2 maps) from a seeded surface cloud of the C3 room.

Prints one JSON line: value = point-probe projections per second with the
cloud resident in HBM (lfp_bake_points, LFP_SRC_DEVICE), e2e = the same
through pointbake.bake_points_device from HOST arrays (cloud H2D inside the
timed region), cpu_baseline = the numpy restatement of the reference bake
(oracle/bake_oracle.py, one thread) on a bounded sample.

    python tools/bench_bake.py [--density 16000] [--steps 3] [--warmup 1]
"""

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--density", type=float, default=16000.0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--r-hi", type=int, default=256)
    ap.add_argument("--r-lo", type=int, default=64)
    ap.add_argument("--cpu-points", type=int, default=1 << 21)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--lib", default=None, help="alternative library build")
    a = ap.parse_args()

    import torch

    if a.lib:
        os.environ["LFP_LIB_PATH"] = os.path.abspath(a.lib)
    else:
        import __graft_entry__
        __graft_entry__.build()
    from paper_2507_14624_b200 import configs, native, pointbake, scenes
    from paper_2507_14624_b200.bake import lattice_origins

    cloud = scenes.sample_point_cloud(configs.c3_scene(303), a.density, seed=1)
    org = np.ascontiguousarray(lattice_origins((0.0, 0.0, 0.0), 1.0, (8, 4, 8)))
    N, P, R, r = len(cloud), len(org), a.r_hi, a.r_lo
    dv = torch.device("cuda", 0)
    pos = torch.from_numpy(np.array(cloud.positions)).to(dv)
    col = torch.from_numpy(np.array(cloud.colors)).to(dv)
    maps = [torch.empty(s, dtype=torch.float32, device=dv) for s in
            ((P, R, R), (P, R, R, 3), (P, R, R, 3), (P, r, r))]
    st = torch.cuda.current_stream(dv)
    vp = ctypes.c_void_p
    L = native.lib()
    skipped = np.zeros(P, np.int64)

    def step():
        native.check(L.lfp_bake_points(
            0, vp(pos.data_ptr()), vp(col.data_ptr()), N,
            org.ctypes.data_as(vp), P, R, r, native.LFP_SRC_DEVICE,
            *[vp(m.data_ptr()) for m in maps], skipped.ctypes.data_as(vp),
            vp(st.cuda_stream)))

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(
        enable_timing=True)
    e0.record(st)
    for _ in range(a.steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    value = N * P / (ms * 1e-3) / 1e9

    # e2e: host cloud -> device maps through the public API
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        pointbake.bake_points_device(cloud, org, R, r)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / a.steps

    cpu = None
    if not a.no_cpu:
        from oracle import bake_oracle
        n = min(N, a.cpu_points)
        sel = np.random.default_rng(0).choice(N, n, replace=False)
        t0 = time.perf_counter()
        bake_oracle.bake_maps(cloud.positions[sel], cloud.colors[sel], org[0],
                              R, r)
        dt = time.perf_counter() - t0
        cpu = {"value": n / dt / 1e9, "unit": "Gpoint-probes/s", "cores": 1,
               "kind": "port",
               "sample": f"{n} of {N} points x 1 probe (numpy restatement "
                         "of bake_probe, one thread)"}
    out = {"metric": "point-cloud bake throughput", "value": value,
           "unit": "Gpoint-probes/s", "ms_per_step": ms,
           "config": {"workload": "C3 lattice 8x4x8 (256 probes) "
                                  f"{R}^2/{r}^2 from a C3-room surface cloud",
                      "points": N, "probes": P, "density": a.density},
           "e2e": {"value": N * P / (e2e_ms * 1e-3) / 1e9,
                   "unit": "Gpoint-probes/s", "ms_per_step": e2e_ms,
                   "h2d_bytes_per_step": N * 36,
                   "d2h_bytes_per_step": P * 8},
           "cpu_baseline": cpu, "gpu_launches_per_step": 3 * ((P + 63) // 64) + 1}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
