"""Print decision-filter statistics (trace_mode 'check') for a config."""
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

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = configs.c2() if name == "c2" else configs.c3(n_views=1)
cam = cfg.cameras[0]
dps = device_probe_set(cfg.grid)
res = {}
for mode in ("check", "filtered", "exact"):
    g = dev.grid_params(cfg.grid.grid_origin, cfg.grid.cell_size, cfg.grid.dims,
                        DEFAULT_CONFIG, mode=mode)
    out = dev.RayOutputs(cam.width * cam.height, dps.device, fetch=True, diag=True)
    dev.render_cameras(dps, g, [cam], cam.width, cam.height, out)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    out.diag.zero_()
    e0.record()
    dev.render_cameras(dps, g, [cam], cam.width, cam.height, out)
    e1.record()
    torch.cuda.synchronize()
    d = [int(v) for v in out.diag.cpu()]
    f = out.fetch.cpu().numpy()
    res[mode] = {"ms": e0.elapsed_time(e1), "lo_fast": d[0], "lo_slow": d[1],
                 "hi_fast": d[2], "hi_slow": d[3], "mismatch": d[4],
                 "lo_rseg": d[5], "hi_sq": d[6], "segs": d[7],
                 "hi_f_cont": d[8], "hi_f_occ": d[9], "hi_f_cand": d[10],
                 "fetch_mean": float(f.mean()),
                 "fetch_p50": float(np.percentile(f, 50)),
                 "fetch_p99": float(np.percentile(f, 99)),
                 "fetch_max": int(f.max())}
print(json.dumps({"config": name, **res}, indent=1))
