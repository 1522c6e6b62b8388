"""Phase timing of the C5 public path (render.trace_rays): H2D, binning,
trace, D2H -- at 2^22 and 2^26 rays."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2507_14624_b200 as pkg  # noqa: E402
from paper_2507_14624_b200 import configs, device as dev  # noqa: E402
from paper_2507_14624_b200.render import device_probe_set  # noqa: E402
from paper_2507_14624_b200.trace import DEFAULT_CONFIG  # noqa: E402

cfg = configs.c3(n_views=1)
o_all, d_all = configs.c5_rays(cfg.scene, 1 << 26, seed=505)
grid = cfg.grid
dps = device_probe_set(grid)
g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims, DEFAULT_CONFIG)


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for n in (1 << 22, 1 << 26):
    o, d = o_all[:n], d_all[:n]
    pkg.trace_rays(grid, o, d)
    t0 = t()
    pkg.trace_rays(grid, o, d)
    t1 = t()
    to = torch.from_numpy(o).to("cuda")
    td = torch.from_numpy(d).to("cuda")
    t2 = t()
    keys = dev.bin_rays(g, to, td)
    t3 = t()
    order = dev.ray_order(keys)
    t4 = t()
    out = dev.RayOutputs(n, dps.device, probe=True, texel=True, fetch=True,
                         hit_t=True)
    out.rgb.zero_()
    t5 = t()
    dev.trace_rays_ordered(dps, g, to, td, order, out, rgb_mode=1)
    t6 = t()
    for a in (out.status, out.probe, out.texel, out.fetch, out.rgb, out.hit_t):
        a.cpu()
    t7 = t()
    dev.trace_rays(dps, g, to, td, out, rgb_mode=1)
    t8 = t()
    print(f"n={n}: api {1e3*(t1-t0):.1f} ms ({n/(t1-t0)/1e6:.1f} Mrays/s) | "
          f"h2d {1e3*(t2-t1):.1f} bin {1e3*(t3-t2):.1f} argsort "
          f"{1e3*(t4-t3):.1f} alloc {1e3*(t5-t4):.1f} trace "
          f"{1e3*(t6-t5):.1f} d2h {1e3*(t7-t6):.1f} | unbinned trace "
          f"{1e3*(t8-t7):.1f}", flush=True)
