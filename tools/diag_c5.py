"""C5 diagnostics: 2^20 incoherent rays against the C3 probe set, traced
unbinned / binned, with decision-filter counters and per-ray cost
statistics. Also used as the ncu target for the C5 kernel."""
import json
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
scene, grid = configs.c3_grid()
o, d = configs.c5_rays(scene, n, seed=505)
dps = device_probe_set(grid)
to, td = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
res = {"rays": n}
variants = [("nested", 0, False), ("nested", 0, True)] + [
    ("persistent", ma, b) for ma in (8, 16, 24) for b in (False, True)]
for sched, ma, binned in variants:
    g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                        DEFAULT_CONFIG, schedule=sched, min_active=ma)
    out = dev.RayOutputs(n, dps.device, fetch=True, diag=True)
    for it in range(2):
        out.diag.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if binned:
            order = dev.ray_order(dev.bin_rays(g, to, td))
            e1.record()
            dev.trace_rays_ordered(dps, g, to, td, order, out)
        else:
            e1.record()
            dev.trace_rays(dps, g, to, td, out)
        e2.record()
        torch.cuda.synchronize()
    f = out.fetch.cpu().numpy()
    dg = [int(v) for v in out.diag.cpu()]
    res[f"{sched}_ma{ma}_{'binned' if binned else 'unbinned'}"] = {
        "sort_ms": e0.elapsed_time(e1), "trace_ms": e1.elapsed_time(e2),
        "lo": dg[0] + dg[1], "lo_rseg": dg[5], "hi": dg[2] + dg[3],
        "hi_sq": dg[6], "segs": dg[7], "lo_slow": dg[1], "hi_slow": dg[3],
        "fetch_mean": float(f.mean()), "fetch_p50": float(np.percentile(f, 50)),
        "fetch_p99": float(np.percentile(f, 99)), "fetch_max": int(f.max())}
print(json.dumps(res, indent=1))
