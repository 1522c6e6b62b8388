"""Per-step device time of the C5 wavefront trace (2^k rays), several steps
in one process: python tools/c5_steps.py [log2_rays] [steps]"""
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
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
scene, grid = configs.c3_grid()
o, d = configs.c5_rays(scene, 1 << k, seed=505)
to, td = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
dps = device_probe_set(grid)
g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims, DEFAULT_CONFIG)
out = dev.RayOutputs(len(o), dps.device)
ts = []
for s in range(steps + 1):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    dev.trace_rays(dps, g, to, td, out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
lib = os.path.basename(os.environ.get("LFP_LIB_PATH", "default"))
print(lib, "ms per step:", " ".join(f"{t:.1f}" for t in ts[1:]),
      f"-> {len(o) / (sum(ts[1:]) / steps) / 1e3:.1f} Mrays/s")
