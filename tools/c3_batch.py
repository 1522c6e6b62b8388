"""C3: one 64-view launch vs per-view launches vs per-view 2-stream bands
(device time, CUDA events)."""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2507_14624_b200 import configs  # noqa: E402
from paper_2507_14624_b200 import device as dev  # noqa: E402
from paper_2507_14624_b200.render import device_probe_set  # noqa: E402
from paper_2507_14624_b200.trace import DEFAULT_CONFIG  # noqa: E402

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = configs.c3(n_views=nv)
cams = cfg.cameras
W, H = cams[0].width, cams[0].height
dps = device_probe_set(cfg.grid)
g = dev.grid_params(cfg.grid.grid_origin, cfg.grid.cell_size, cfg.grid.dims,
                    DEFAULT_CONFIG)
out = dev.RayOutputs(len(cams) * W * H, dps.device)


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def batch():
    dev.render_cameras(dps, g, cams, W, H, out)


def per_view():
    for i, c in enumerate(cams):
        dev.render_cameras(dps, g, [c], W, H, out)


def host_path():
    for c in cams:
        dev.render_frame_host(dps, g, c)


n = len(cams) * W * H
for name, fn in (("batch", batch), ("per_view", per_view), ("frame_host", host_path)):
    ms = timed(fn)
    print(f"{name:10s} {ms:9.2f} ms  {n / ms / 1e3:7.1f} Mrays/s")
