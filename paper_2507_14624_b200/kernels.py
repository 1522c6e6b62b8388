"""Drop-in replacements for the reference's numba entry points
(`pkg/src/lfprobe/kernels.py`), same signatures and in-place semantics,
executed by the CUDA library.

    import lfprobe.kernels, paper_2507_14624_b200.kernels as gpu
    lfprobe.kernels.render_grid = gpu.render_grid

routes the reference's own `render_frame` (which resolves
`kernels.render_grid` at call time, `render.py:13, 132`) to the GPU.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as dev
from .trace import (DEFAULT_EPS_ALIGN, DEFAULT_EPS_START, DEFAULT_SLACK, HIT,
                    MISS, UNKNOWN, TraceConfig)

__all__ = ["render_grid", "trace_grid_ray", "HIT", "MISS", "UNKNOWN",
           "DEFAULT_SLACK", "DEFAULT_EPS_START", "DEFAULT_EPS_ALIGN"]


def render_grid(dist_hi_all, dir_hi_all, irr_all, dist_lo_all, origins,
                grid_origin, cell, nx, ny, nz, eye, dirs, eps_start,
                eps_align, slack, out_status, out_rgb, out_fetch, device=0):
    """`kernels.py:825-843`: trace every ray of `dirs` (N, 3) from `eye`;
    writes out_status / out_fetch for every ray and out_rgb only on HIT
    rows (the caller pre-zeroes it, as with the reference)."""
    dps = dev.cached_probe_set(dist_hi_all, dir_hi_all, irr_all, dist_lo_all,
                               origins, device=device)
    cfg = TraceConfig(eps_start=eps_start, eps_align=eps_align, slack=slack)
    g = dev.grid_params(grid_origin, cell, (nx, ny, nz), cfg)
    n = len(dirs)
    d_dirs = torch.from_numpy(np.ascontiguousarray(dirs, np.float64)).to(
        dps.device, non_blocking=False)
    out = dev.RayOutputs(n, dps.device, fetch=True, stats=False)
    dev.render_grid_dirs(dps, g, np.asarray(eye, np.float64), d_dirs, out,
                         rgb_mode=1)
    status = out.status.cpu().numpy()
    out_status[:] = status
    out_fetch[:] = out.fetch.cpu().numpy()
    hit = status == HIT
    rgb = out.rgb.cpu().numpy()
    out_rgb[hit] = rgb[hit]


def trace_grid_ray(dist_hi_all, dir_hi_all, irr_all, dist_lo_all, origins,
                   grid_origin, cell, nx, ny, nz, ex, ey, ez, dx, dy, dz,
                   eps_start, eps_align, slack, rgb_out, device=0):
    """`kernels.py:653-822` for one ray: returns (status, probe, tx, ty,
    fetches) and writes rgb_out on HIT. One launch per call -- use
    `device.trace_rays` for batches."""
    dps = dev.cached_probe_set(dist_hi_all, dir_hi_all, irr_all, dist_lo_all,
                               origins, device=device)
    cfg = TraceConfig(eps_start=eps_start, eps_align=eps_align, slack=slack)
    g = dev.grid_params(grid_origin, cell, (nx, ny, nz), cfg)
    o = torch.tensor([[ex, ey, ez]], dtype=torch.float64, device=dps.device)
    d = torch.tensor([[dx, dy, dz]], dtype=torch.float64, device=dps.device)
    out = dev.RayOutputs(1, dps.device, probe=True, texel=True, fetch=True,
                         stats=False)
    dev.trace_rays(dps, g, o, d, out, rgb_mode=1)
    st = int(out.status.cpu()[0])
    p = int(out.probe.cpu()[0])
    tex = int(out.texel.cpu()[0])
    tx, ty = (-1, -1) if tex < 0 else (tex & 0xFFFF, tex >> 16)
    if st == HIT:
        rgb_out[:] = out.rgb.cpu().numpy()[0]
    return st, p, tx, ty, int(out.fetch.cpu()[0])
