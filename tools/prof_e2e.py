"""cProfile of render_frame on a config (host-side overhead of the public
API): python tools/prof_e2e.py c1|c2 [calls]"""
import cProfile
import os
import pstats
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2507_14624_b200 import configs, render_frame  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 500
cfg = {"c1": configs.c1, "c2": configs.c2}.get(name, lambda: configs.c3(n_views=1))()
cam = cfg.cameras[0]
for _ in range(20):
    render_frame(cfg.grid, cam)
t0 = time.perf_counter()
for _ in range(calls):
    f = render_frame(cfg.grid, cam)
dt = (time.perf_counter() - t0) / calls
print(f"{name}: {dt * 1e3:.3f} ms per call, traceMs {f.stats['traceMs']:.3f}")
pr = cProfile.Profile()
pr.enable()
for _ in range(calls):
    render_frame(cfg.grid, cam)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
