"""Camera rays through the wavefront schedule vs the nested camera kernel
(same view, same outputs): python tools/wave_cam.py [c2|c3] [views]"""
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

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = configs.c2() if name == "c2" else configs.c3(n_views=nv)
grid = cfg.grid
dps = device_probe_set(grid)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
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


tot_n, t_nest, t_wave, same = 0, 0.0, 0.0, True
for cam in cfg.cameras[:nv]:
    n = cam.width * cam.height
    g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims, DEFAULT_CONFIG)
    a = dev.RayOutputs(n, dps.device, probe=True, texel=True, fetch=True)
    t_nest += timed(lambda: dev.render_cameras(dps, g, [cam], cam.width, cam.height, a))
    dirs = torch.from_numpy(np.ascontiguousarray(cam.ray_directions().reshape(-1, 3))).cuda()
    gw = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims, DEFAULT_CONFIG,
                         schedule="wave")
    b = dev.RayOutputs(n, dps.device, probe=True, texel=True, fetch=True)
    t_wave += timed(lambda: dev.render_grid_dirs(dps, gw, np.asarray(cam.eye, np.float64), dirs, b))
    for k in ("status", "probe", "texel", "fetch"):
        same &= bool(torch.equal(getattr(a, k), getattr(b, k)))
    tot_n += n
print(f"{name} {nv} view(s): nested {t_nest:.2f} ms ({tot_n / t_nest / 1e3:.1f} Mrays/s), "
      f"wave {t_wave:.2f} ms ({tot_n / t_wave / 1e3:.1f} Mrays/s), identical={same}")
