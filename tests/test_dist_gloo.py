"""Multi-GPU host logic on CPU: the interleaved tile shard plan, the
gather of padded compact shards to rank 0 (gloo, world_size 2 and 3) and the
untile scatter reproduce the full frames."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_14624_b200.dist import (TILE_PIX, TILE_W, TILE_H, ShardPlan,
                                        gather_shards, num_tiles, untile_numpy)


def test_plan_partitions_tiles():
    for C, W, H in ((1, 512, 512), (3, 100, 77), (2, 1, 1), (64, 1920, 1080)):
        T = num_tiles(C, W, H)
        for world in (1, 2, 3, 4, 8):
            seen = np.zeros(T, np.int64)
            for k in range(world):
                p = ShardPlan(C, W, H, world, k)
                g = p.global_tiles()
                assert len(g) == p.n_tiles <= p.max_tiles
                seen[g] += 1
            assert (seen == 1).all()


def _pixel_value(cam, x, y, W, H):
    v = (cam * H + y) * W + x
    return (v % 251).astype(np.uint8), np.stack(
        [v * 1.0, v * 0.5, -v * 1.0], -1).astype(np.float32)


def _render_shard(plan):
    """Test-side emulation of lfp_render_cameras' compact layout."""
    m = plan.max_tiles * TILE_PIX
    st = np.zeros(m, np.uint8)
    rgb = np.zeros((m, 3), np.float32)
    tx_n = -(-plan.width // TILE_W)
    per_cam = tx_n * (-(-plan.height // TILE_H))
    lane = np.arange(TILE_PIX)
    for j, g in enumerate(plan.global_tiles()):
        cam, t = divmod(int(g), per_cam)
        x = (t % tx_n) * TILE_W + (lane & 7)
        y = (t // tx_n) * TILE_H + (lane >> 3)
        ok = (x < plan.width) & (y < plan.height)
        s, c = _pixel_value(cam, x[ok], y[ok], plan.width, plan.height)
        st[j * TILE_PIX + lane[ok]] = s
        rgb[j * TILE_PIX + lane[ok]] = c
    return st, rgb


def _worker(rank, world, port, C, W, H, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = ShardPlan(C, W, H, world, rank)
        st, rgb = _render_shard(plan)
        g = gather_shards(plan, torch.from_numpy(st), torch.from_numpy(rgb))
        if rank == 0:
            st_all, rgb_all = g
            m = plan.max_tiles * TILE_PIX
            shards_s = [st_all[k * m:(k + 1) * m].numpy() for k in range(world)]
            shards_c = [rgb_all[k * m:(k + 1) * m].numpy() for k in range(world)]
            fs, fc = untile_numpy(plan, shards_s, shards_c)
            yy, xx = np.mgrid[0:H, 0:W]
            ok = True
            for cam in range(C):
                es, ec = _pixel_value(cam, xx.ravel(), yy.ravel(), W, H)
                ok &= np.array_equal(fs[cam * H * W:(cam + 1) * H * W], es)
                ok &= np.array_equal(fc[cam * H * W:(cam + 1) * H * W], ec)
            q.put(bool(ok))
        else:
            assert g is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,C,W,H", [(2, 2, 100, 77), (3, 1, 64, 48)])
def test_gather_untile_gloo(world, C, W, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, C, W, H, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


def _rows_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_14624_b200.dist import gather_rows, ray_share
        n = 1001
        lo, hi = ray_share(n, world, rank)
        idx = torch.arange(lo, hi)
        m = (n + world - 1) // world
        parts = gather_rows([idx.to(torch.int32),
                             torch.stack([idx * 1.0, -idx * 1.0], 1)], m)
        if rank == 0:
            keep = torch.cat([torch.arange(k * m, k * m + ray_share(n, world, k)[1]
                                           - ray_share(n, world, k)[0])
                              for k in range(world)])
            a = parts[0][keep]
            b = parts[1][keep]
            q.put(bool(torch.equal(a, torch.arange(n, dtype=torch.int32)) and
                       torch.equal(b[:, 0], torch.arange(n) * 1.0)))
        else:
            assert parts is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_rows_ray_shares_gloo(world):
    """Ray-batch sharding (C5): contiguous shares padded to ceil(n/world)
    rows, gathered to rank 0 and trimmed back to input order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
