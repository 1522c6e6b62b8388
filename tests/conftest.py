import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (B200, sm_100a) and the built "
        "liblfprobe_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"),
                        allow_pickle=False))


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]
    return get


class GoldenProbeSet:
    def __init__(self, z):
        self.dist_hi = np.ascontiguousarray(z["dist_hi"], np.float32)
        self.dir_hi = np.ascontiguousarray(z["dir_hi"], np.float32)
        self.irr_hi = np.ascontiguousarray(z["irr_hi"], np.float32)
        self.dist_lo = np.ascontiguousarray(z["dist_lo"], np.float32)
        self.origins = np.ascontiguousarray(z["origins"], np.float64)


def golden_grid(z):
    from paper_2507_14624_b200.grid import ProbeGrid, ProbeSet
    ps = ProbeSet(arrays=(z["dist_hi"], z["dir_hi"], z["irr_hi"],
                          z["dist_lo"], z["origins"]))
    return ProbeGrid(z["grid_origin"], float(z["cell"]),
                     tuple(int(v) for v in z["dims"]), probe_set=ps)


def golden_camera(z, prefix="cam_"):
    from paper_2507_14624_b200.render import Camera
    w, h = (int(v) for v in z[prefix + "wh"])
    return Camera(eye=tuple(z[prefix + "eye"]),
                  forward=tuple(z[prefix + "forward"]),
                  up=tuple(z[prefix + "up"]), vfov_deg=float(z[prefix + "vfov"]),
                  width=w, height=h)
