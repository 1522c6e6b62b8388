"""Multi-rank paths on one GPU (gloo process group, 2 ranks both on
cuda:0): the public dist.render_frames / dist.trace_rays_sharded entry
points (tile-sharded trace, gather to rank 0, CUDA untile, D2H) reproduce
the single-rank results exactly, and bench.py's own launcher starts the
requested number of ranks."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    from paper_2507_14624_b200 import Camera, configs
    cfg = configs.c1()
    cams = cfg.cameras + configs.random_cameras(cfg.scene, 2, 128, 128, 9)
    cams = [Camera(eye=c.eye, forward=c.forward, width=100, height=77)
            for c in cams]
    o, d = configs.c5_rays(cfg.scene, 5000, seed=77)
    return cfg, cams, o, d


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_14624_b200 import dist as pdist
        cfg, cams, o, d = _inputs()
        frames = pdist.render_frames(cfg.grid, cams)
        res = pdist.trace_rays_sharded(cfg.grid, o, d)
        if rank == 0:
            q.put({"frames": [(f.pixels, f.status, f.stats) for f in frames],
                   "rays": {k: getattr(res, k) for k in
                            ("status", "probe", "tx", "ty", "fetch", "rgb",
                             "hit_t", "stats")}})
        else:
            assert frames is None and res is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_entry_points_match_single_rank(world):
    import torch.multiprocessing as mp
    import __graft_entry__
    __graft_entry__.build()
    from paper_2507_14624_b200 import render_frame, trace_rays
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    cfg, cams, o, d = _inputs()
    for (pix, st, stats), cam in zip(got["frames"], cams):
        ref = render_frame(cfg.grid, cam)
        np.testing.assert_array_equal(st, ref.status)
        np.testing.assert_array_equal(pix, ref.pixels)
        for k in ("perPixelTexelFetches", "missFraction", "unknownFraction"):
            assert stats[k] == ref.stats[k], k
    ref = trace_rays(cfg.grid, o, d)
    for k, v in got["rays"].items():
        np.testing.assert_array_equal(v, getattr(ref, k), err_msg=k)


def test_render_frames_single_rank_and_hierarchy():
    """World 1 (no process group): render_frames == render_frame per
    camera, for a grid and for a probe hierarchy."""
    from paper_2507_14624_b200 import ProbeHierarchy, configs, render_frame
    from paper_2507_14624_b200 import dist as pdist
    cfg, cams, _, _ = _inputs()
    for src in (cfg.grid, ProbeHierarchy([configs.c2().grid, cfg.grid])):
        frames = pdist.render_frames(src, cams)
        for f, cam in zip(frames, cams):
            ref = render_frame(src, cam)
            np.testing.assert_array_equal(f.status, ref.status)
            np.testing.assert_array_equal(f.pixels, ref.pixels)
            assert f.stats["perPixelTexelFetches"] == \
                ref.stats["perPixelTexelFetches"]


def _bench(args, timeout=900):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args],
                       capture_output=True, text=True, timeout=timeout,
                       cwd=REPO, env=env)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-4000:]
    return json.loads(lines[0])


def test_bench_default_is_c3():
    line = _bench(["--gpus", "1", "--steps", "1", "--warmup", "3",
                   "--no-e2e", "--no-cpu-baseline"])
    assert line["n_gpus"] == 1
    assert line["config"]["workload"].startswith("C3")
    assert line["config"]["rays_per_step"] == 64 * 1920 * 1080
    assert line["roofline"]["frac"] > 0


def test_bench_gpus_2_self_launches():
    line = _bench(["--gpus", "2", "--dist-backend", "gloo", "--config", "c2",
                   "--steps", "2", "--warmup", "3", "--no-cpu-baseline"])
    assert line["n_gpus"] == 2
    assert line["config"]["rays_per_step"] == 2 * 512 * 512
    assert "render_frames" in line["e2e"]["api"]
