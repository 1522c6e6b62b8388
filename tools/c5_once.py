"""One C5 wavefront trace (2^k rays, default 26) for launch-list / traffic
captures: python tools/c5_once.py [log2_rays]"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2507_14624_b200 import configs  # noqa: E402
from paper_2507_14624_b200 import device as dev  # noqa: E402
from paper_2507_14624_b200.render import device_probe_set  # noqa: E402
from paper_2507_14624_b200.trace import DEFAULT_CONFIG  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 26
scene, grid = configs.c3_grid()
o, d = configs.c5_rays(scene, 1 << k, seed=505)
to, td = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
dps = device_probe_set(grid)
g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims, DEFAULT_CONFIG)
out = dev.RayOutputs(len(o), dps.device)
torch.cuda.synchronize()
dev.trace_rays(dps, g, to, td, out)
torch.cuda.synchronize()
print("ok", len(o), "rays, launches", dev.last_launches() if hasattr(dev, "last_launches") else "?")
