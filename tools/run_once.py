"""Run one render / trace launch pattern for profiling:
    python tools/run_once.py c2|c5 nested|persistent [min_active]
Three launches (two warm-up + one measured); prints the CUDA-event time of
the last one."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2507_14624_b200 import configs  # noqa: E402
from paper_2507_14624_b200 import device as dev  # noqa: E402
from paper_2507_14624_b200.render import device_probe_set  # noqa: E402
from paper_2507_14624_b200.trace import DEFAULT_CONFIG  # noqa: E402

cfg_name, sched = sys.argv[1], sys.argv[2]
ma = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if cfg_name in ("c2", "c3"):
    cfg = configs.c2() if cfg_name == "c2" else configs.c3(n_views=1)
    grid = cfg.grid
    cam = cfg.cameras[0]
    n = cam.width * cam.height
else:
    scene, grid = configs.c3_grid()
    o, d = configs.c5_rays(scene, 1 << int(os.environ.get("LFP_C5_LOG2", "20")),
                           seed=505)
    to, td = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
    n = len(o)
dps = device_probe_set(grid)
g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims, DEFAULT_CONFIG,
                    schedule=sched, min_active=ma)
out = dev.RayOutputs(n, dps.device, fetch=True)
if cfg_name == "c5":
    order = dev.ray_order(dev.bin_rays(g, to, td))
for _ in range(3):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    if cfg_name in ("c2", "c3"):
        dev.render_cameras(dps, g, [cam], cam.width, cam.height, out)
    else:
        dev.trace_rays_ordered(dps, g, to, td, order, out)
    e1.record()
    torch.cuda.synchronize()
print(cfg_name, sched, ma, "ms", e0.elapsed_time(e1), "fetch",
      float(out.fetch.float().mean()))
