"""Multi-GPU image sharding.

One process per GPU. A batch of frames is cut into 8x16-pixel tiles; rank k
of N traces tiles k, k + N, k + 2N, ... (interleaved round robin, because the
per-ray cost is heavy-tailed) against its own replica of the probe set and
writes them in compact shard order. The only collective is the framebuffer
gather to rank 0 over NCCL (NVLink / NVSwitch); rank 0 scatters the shards
back into frame order with `lfp_untile`.

The plan / gather logic is backend-agnostic (tested with gloo on CPU);
tracing and untiling are CUDA kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

TILE_W, TILE_H = 8, 16
TILE_PIX = TILE_W * TILE_H


def num_tiles(n_cams, width, height):
    return n_cams * (-(-width // TILE_W)) * (-(-height // TILE_H))


@dataclass(frozen=True)
class ShardPlan:
    """Which tiles of a (n_cams, width, height) batch rank `rank` traces."""

    n_cams: int
    width: int
    height: int
    world: int
    rank: int

    @property
    def total_tiles(self):
        return num_tiles(self.n_cams, self.width, self.height)

    def tiles_of(self, k):
        t = self.total_tiles
        return t // self.world + (1 if k < t % self.world else 0)

    @property
    def n_tiles(self):
        return self.tiles_of(self.rank)

    @property
    def max_tiles(self):
        return self.tiles_of(0)

    @property
    def tile_begin(self):
        return self.rank

    @property
    def tile_step(self):
        return self.world

    def global_tiles(self, k=None):
        k = self.rank if k is None else k
        return np.arange(k, self.total_tiles, self.world)


def untile_numpy(plan: ShardPlan, shards_status, shards_rgb):
    """Host mirror of lfp_untile for CPU tests: shards[k] hold rank k's
    compact tiles (padded to max_tiles)."""
    W, H, C = plan.width, plan.height, plan.n_cams
    st = np.zeros((C * H * W,), np.uint8)
    rgb = np.zeros((C * H * W, 3), np.float32)
    tx_n = -(-W // TILE_W)
    per_cam = tx_n * (-(-H // TILE_H))
    lane = np.arange(TILE_PIX)
    for k in range(plan.world):
        for j, g in enumerate(plan.global_tiles(k)):
            cam, t = divmod(int(g), per_cam)
            x = (t % tx_n) * TILE_W + (lane & 7)
            y = (t // tx_n) * TILE_H + (lane >> 3)
            ok = (x < W) & (y < H)
            dst = (cam * H + y[ok]) * W + x[ok]
            src = j * TILE_PIX + lane[ok]
            st[dst] = shards_status[k][src]
            rgb[dst] = shards_rgb[k][src]
    return st, rgb


def gather_shards(plan: ShardPlan, status, rgb, dst=0, group=None):
    """Gather every rank's padded compact shard (max_tiles * 128 pixels) to
    rank `dst`. Returns (status[world * M], rgb[world * M, 3]) on dst, None
    elsewhere. One NCCL gather per buffer (grouped send/recv under the
    hood); on gloo the same call runs on CPU tensors."""
    m = plan.max_tiles * TILE_PIX
    assert status.shape[0] == m and rgb.shape[0] == m, "shards must be padded"
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if rank == dst:
        st_all = torch.empty((world * m,), dtype=status.dtype,
                             device=status.device)
        rgb_all = torch.empty((world * m, 3), dtype=rgb.dtype, device=rgb.device)
        st_list = list(st_all.chunk(world))
        rgb_list = list(rgb_all.chunk(world))
    else:
        st_list = rgb_list = None
    dist.gather(status, st_list, dst=dst, group=group)
    dist.gather(rgb, rgb_list, dst=dst, group=group)
    if rank == dst:
        return st_all, rgb_all
    return None


def _is_gloo(group=None):
    return dist.get_backend(group) == "gloo"


def _comm(t, group=None):
    """Tensor as the backend can move it (gloo: host memory)."""
    return t.cpu() if _is_gloo(group) else t


def gather_rows(tensors, m, dst=0, group=None):
    """Gather per-rank row buffers, each padded to `m` rows, to rank `dst`.
    Returns a list of (world * m, ...) tensors on dst (rank k's rows at
    [k*m, k*m + n_k)), None elsewhere. One gather per buffer."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    outs = []
    for t in tensors:
        t = _comm(t, group)
        if t.shape[0] < m:
            pad = torch.zeros((m - t.shape[0],) + tuple(t.shape[1:]),
                              dtype=t.dtype, device=t.device)
            t = torch.cat([t, pad])
        if rank == dst:
            full = torch.empty((world * m,) + tuple(t.shape[1:]),
                               dtype=t.dtype, device=t.device)
            dist.gather(t, list(full.chunk(world)), dst=dst, group=group)
            outs.append(full)
        else:
            dist.gather(t, None, dst=dst, group=group)
    return outs if rank == dst else None


def render_batch_sharded(dps, gparams, cams, width, height, plan: ShardPlan,
                         out, frame_status=None, frame_rgb=None, stream=None):
    """Trace this rank's tiles into `out` (compact, padded to max_tiles),
    gather to rank 0 and untile into frame_status / frame_rgb there.

    Everything runs on `stream` (default: the current stream), made current
    for the body so that the collective (which orders itself against the
    current stream) waits for the trace and the untile for the gather."""
    from . import device as dev

    st = stream if stream is not None else torch.cuda.current_stream(dps.device)
    with torch.cuda.stream(st):
        dev.render_cameras(dps, gparams, cams, width, height, out,
                           tile_begin=plan.tile_begin, tile_step=plan.tile_step,
                           n_tiles=plan.n_tiles, compact=True, stream=st)
        if plan.world == 1:
            st_all, rgb_all = out.status, out.rgb
        else:
            g = gather_shards(plan, _comm(out.status), _comm(out.rgb))
            if g is None:
                return False
            st_all, rgb_all = (t.to(dps.device) for t in g)
        if frame_status is not None:
            dev.untile(len(cams), width, height, plan.world, st_all, rgb_all,
                       frame_status, frame_rgb, shard_stride=plan.max_tiles,
                       stream=st)
    return True


def _world(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _cam_stats(plan, status, fetch, n_cams, tiles_per_cam):
    """Per-camera {fetch sum, #MISS, #UNKNOWN, #HIT} of this rank's compact
    shard (padding pixels hold status 255 and fetch 0)."""
    dvc = status.device
    n = plan.n_tiles * TILE_PIX
    stats = torch.zeros(n_cams * 4, dtype=torch.int64, device=dvc)
    if n == 0:
        return stats
    cam = torch.as_tensor(plan.global_tiles() // tiles_per_cam, device=dvc)
    cam = cam.repeat_interleave(TILE_PIX) * 4
    st = status[:n]
    stats.index_add_(0, cam, fetch[:n].to(torch.int64))
    for k, code in ((1, 0), (2, 2), (3, 1)):
        stats.index_add_(0, cam + k, (st == code).to(torch.int64))
    return stats


def render_frames(source, cams, config=None, background=(0.0, 0.0, 0.0),
                  unknown_color=(1.0, 0.0, 1.0), device=None, group=None):
    """`render_frame` for a batch of cameras over every rank of the process
    group (one process per GPU; world 1 without a group).

    The batch is cut into 8x16 tiles dealt round robin to the ranks (the
    per-ray cost is heavy-tailed); each rank traces its tiles against its
    own replica of the probe set (`source`: a ProbeGrid or ProbeHierarchy,
    uploaded once per device and cached), the compact shards are gathered to
    rank 0 over the group's backend (NCCL over NVLink; gloo through host
    memory), untiled on rank 0's GPU and copied to host. Returns the list of
    Frames on rank 0 (pixels f32 (H, W, 3), status u8 (H, W), the reference
    stats keys per frame; traceMs = this rank's device time of the batch),
    None on the other ranks. All cameras must share one resolution."""
    from . import device as dev
    from .render import Frame, _stats_dict, device_probe_set
    from .trace import DEFAULT_CONFIG

    config = config or DEFAULT_CONFIG
    cams = list(cams)
    if not cams:
        raise ValueError("render_frames needs at least one camera")
    W, H = cams[0].width, cams[0].height
    if any((c.width, c.height) != (W, H) for c in cams):
        raise ValueError("render_frames: cameras must share one resolution")
    world, rank = _world(group)
    dvc = torch.device("cuda", torch.cuda.current_device() if device is None
                       else int(device))
    plan = ShardPlan(len(cams), W, H, world, rank)
    m = plan.max_tiles * TILE_PIX
    out = dev.RayOutputs(m, dvc, fetch=True, stats=False)
    stream = torch.cuda.current_stream(dvc)
    with torch.cuda.device(dvc), torch.cuda.stream(stream):
        out.status.fill_(255)
        out.fetch.zero_()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        kw = dict(tile_begin=plan.tile_begin, tile_step=plan.tile_step,
                  n_tiles=plan.n_tiles, compact=True, background=background,
                  unknown_color=unknown_color, stream=stream)
        if hasattr(source, "levels"):
            levels = [(device_probe_set(g, dvc.index),
                       dev.grid_params(g.grid_origin, g.cell_size, g.dims,
                                       config)) for g in source.levels]
            dev.render_hierarchy(levels, cams, W, H, out, **kw)
        else:
            dps = device_probe_set(source, dvc.index)
            g = dev.grid_params(source.grid_origin, source.cell_size,
                                source.dims, config)
            dev.render_cameras(dps, g, cams, W, H, out, **kw)
        t1.record(stream)
        tiles_per_cam = num_tiles(1, W, H)
        stats = _cam_stats(plan, out.status, out.fetch, len(cams),
                           tiles_per_cam)
        if world > 1:
            g_all = gather_shards(plan, _comm(out.status, group),
                                  _comm(out.rgb, group), group=group)
            stats = _comm(stats, group)
            dist.reduce(stats, dst=0, group=group)
            if rank != 0:
                return None
            st_all, rgb_all = (t.to(dvc) for t in g_all)
            stats = stats.to(dvc)
        else:
            st_all, rgb_all = out.status, out.rgb
        n = len(cams) * H * W
        frame_st = torch.empty(n, dtype=torch.uint8, device=dvc)
        frame_rgb = torch.empty((n, 3), dtype=torch.float32, device=dvc)
        dev.untile(len(cams), W, H, world, st_all, rgb_all, frame_st,
                   frame_rgb, shard_stride=plan.max_tiles, stream=stream)
        st_h, rgb_h, stats_h = dev.to_host(frame_st, frame_rgb, stats)
        trace_ms = t0.elapsed_time(t1)
    stats_h = stats_h.reshape(len(cams), 4)
    st_h = st_h.reshape(len(cams), H, W)
    rgb_h = rgb_h.reshape(len(cams), H, W, 3)
    return [Frame(pixels=rgb_h[c], status=st_h[c],
                  stats=_stats_dict(stats_h[c], H * W, trace_ms))
            for c in range(len(cams))]


def ray_share(n, world, rank):
    """Contiguous [lo, hi) share of n rays for `rank` (ray-batch sharding)."""
    return rank * n // world, (rank + 1) * n // world


def trace_rays_sharded(grid, origins, dirs, config=None, device=None,
                       group=None, binned=True):
    """`trace_rays` for one ray batch over every rank of the process group:
    every rank holds the same host arrays (N, 3), traces its contiguous
    share on its own GPU against its probe-set replica, and all per-ray
    outputs (status, probe, texel, fetch, rgb, hit_t) are gathered to rank
    0 and copied to host in input order. Returns a RayBatchResult on rank 0
    (stats summed over ranks), None elsewhere."""
    from . import device as dev
    from .render import (RayBatchResult, device_probe_set, ray_result_host,
                         trace_rays_device)
    from .trace import DEFAULT_CONFIG

    config = config or DEFAULT_CONFIG
    o = np.ascontiguousarray(origins)
    d = np.ascontiguousarray(dirs)
    if o.shape != d.shape or o.ndim != 2 or o.shape[1] != 3:
        raise ValueError("origins and dirs must both be (N, 3)")
    dt = torch.float32 if (o.dtype == np.float32 and d.dtype == np.float32) \
        else torch.float64
    world, rank = _world(group)
    dvc = torch.device("cuda", torch.cuda.current_device() if device is None
                       else int(device))
    n = len(d)
    lo, hi = ray_share(n, world, rank)
    dps = device_probe_set(grid, dvc.index)
    g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims, config)
    with torch.cuda.device(dvc), torch.cuda.stream(
            torch.cuda.current_stream(dvc)):
        to = torch.from_numpy(o[lo:hi]).to(device=dvc, dtype=dt)
        td = torch.from_numpy(d[lo:hi]).to(device=dvc, dtype=dt)
        out = trace_rays_device(dps, g, to, td, binned=binned)
        if world == 1:
            return ray_result_host(out)
        m = (n + world - 1) // world
        parts = gather_rows([out.status, out.probe, out.texel, out.fetch,
                             out.rgb, out.hit_t], m, group=group)
        stats = _comm(out.stats, group)
        dist.reduce(stats, dst=0, group=group)
        if rank != 0:
            return None
        keep = torch.cat([torch.arange(k * m, k * m + (ray_share(n, world, k)[1]
                                                       - ray_share(n, world, k)[0]))
                          for k in range(world)]).to(parts[0].device)
        full = dev.RayOutputs.__new__(dev.RayOutputs)
        full.n = n
        (full.status, full.probe, full.texel, full.fetch, full.rgb,
         full.hit_t) = (p.index_select(0, keep).to(dvc) for p in parts)
        full.stats = stats.to(dvc)
        res = ray_result_host(full)
    return res
