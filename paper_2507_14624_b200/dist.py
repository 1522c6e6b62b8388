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


def render_batch_sharded(dps, gparams, cams, width, height, plan: ShardPlan,
                         out, frame_status=None, frame_rgb=None, stream=None):
    """Trace this rank's tiles into `out` (compact, padded to max_tiles),
    gather to rank 0 and untile into frame_status / frame_rgb there."""
    from . import device as dev

    dev.render_cameras(dps, gparams, cams, width, height, out,
                       tile_begin=plan.tile_begin, tile_step=plan.tile_step,
                       n_tiles=plan.n_tiles, compact=True, stream=stream)
    if plan.world == 1:
        st_all, rgb_all = out.status, out.rgb
    else:
        g = gather_shards(plan, out.status, out.rgb)
        if g is None:
            return False
        st_all, rgb_all = g
    if frame_status is not None:
        dev.untile(len(cams), width, height, plan.world, st_all, rgb_all,
                   frame_status, frame_rgb, shard_stride=plan.max_tiles,
                   stream=stream)
    return True
