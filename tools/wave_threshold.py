"""Device time of explicit-ray batches of 2^k rays under the persistent
(binned) and wavefront schedules: where the default switch-over
(LFP_WAVE_MIN_RAYS) should sit. python tools/wave_threshold.py [k ...]"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2507_14624_b200 import configs  # noqa: E402
from paper_2507_14624_b200 import device as dev  # noqa: E402
from paper_2507_14624_b200.render import device_probe_set  # noqa: E402
from paper_2507_14624_b200.trace import DEFAULT_CONFIG  # noqa: E402

ks = [int(a) for a in sys.argv[1:]] or [16, 17, 18, 19, 20, 21]
scene, grid = configs.c3_grid()
dps = device_probe_set(grid)


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


for k in ks:
    o, d = configs.c5_rays(scene, 1 << k, seed=505)
    to, td = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
    out = dev.RayOutputs(len(o), dps.device)
    row = [f"2^{k}"]
    for sched in ("persistent", "wave"):
        g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                            DEFAULT_CONFIG, schedule=sched)
        if sched == "persistent":
            def fn():
                order = dev.ray_order(dev.bin_rays(g, to, td))
                dev.trace_rays_ordered(dps, g, to, td, order, out)
        else:
            def fn():
                dev.trace_rays(dps, g, to, td, out)
        ms = timed(fn)
        row.append(f"{sched} {ms:8.2f} ms {len(o) / ms / 1e3:7.1f} Mrays/s")
    print("  ".join(row))
