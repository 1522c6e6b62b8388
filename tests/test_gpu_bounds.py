"""Bounds and write-once evidence for every kernel family (the GPU pool does
not allow compute-sanitizer): tools/sanitize_run.py runs against the
LFP_CHECK_BOUNDS=1 build, which checks every texel / direction-table /
payload / origin / ray-order index against its array extent and counts the
writes of every per-ray output record; it asserts zero violations and
exactly one write per ray (the reference's row-ownership guarantee,
kernels.py:831-843), including the wavefront schedule's queue."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_check_build_all_kernels():
    import __graft_entry__
    __graft_entry__.build()
    env = dict(os.environ, LFP_LIB_PATH=__graft_entry__.LIB_CHECK)
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools",
                                                     "sanitize_run.py")],
                       capture_output=True, text=True, timeout=1200, env=env,
                       cwd=REPO)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "0 index violations, every output record written exactly once" in out
