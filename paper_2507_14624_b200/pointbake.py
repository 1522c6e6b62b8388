"""The reference's point-cloud bake on the GPU (`lfp_bake_points`).

`bake_probe`, `simulate_probe` (`pkg/src/lfprobe/bake.py:140-222`) and
`bake_grid` (`grid.py:96-109`) keep the reference's signatures, errors and
stderr warnings; the maps are bit-identical to the numpy bake (nearest point
per texel, deterministic ties, RGB565 / float16 / 8-bit sub-texel values in
memory). `bake_grid` bakes every lattice probe in one call and leaves the
probe set resident on the device, registered as the grid's cached
`DeviceProbeSet`, so `render_frame(grid, cam)` starts without an upload.
"""

from __future__ import annotations

import ctypes
import sys
import time

import numpy as np

from . import native
from .grid import MapChain, ProbeData, ProbeGrid, ProbeSet
from .octmap import texel_center_directions


def _cloud_arrays(cloud):
    pos = np.ascontiguousarray(np.asarray(cloud.positions, np.float64))
    col = np.ascontiguousarray(np.asarray(cloud.colors, np.float32))
    if pos.ndim != 2 or pos.shape[1] != 3 or col.shape != pos.shape:
        raise ValueError("cloud positions / colors must be (N, 3)")
    return pos, col


def bake_points_device(cloud, origins, r_hi, r_lo, device=0, stream=None):
    """Bake probes at `origins` (P, 3) from `cloud` on the GPU. Returns the
    device tensors (dist_hi, dir_hi, irr_hi, dist_lo) in the ProbeSet layout
    and the per-probe count of points skipped at the origin."""
    import torch

    if r_hi % r_lo != 0:
        raise ValueError("r_hi must be a multiple of r_lo")
    pos, col = _cloud_arrays(cloud)
    if len(pos) == 0:
        raise ValueError("no usable points for bake")
    if not torch.cuda.is_available():
        raise native.LfpError("the point bake needs a CUDA device (no CPU "
                              "fallback)")
    origins = np.ascontiguousarray(np.asarray(origins, np.float64).reshape(-1, 3))
    P = len(origins)
    dv = torch.device("cuda", device)
    f32 = torch.float32
    t_dist = torch.empty((P, r_hi, r_hi), dtype=f32, device=dv)
    t_dir = torch.empty((P, r_hi, r_hi, 3), dtype=f32, device=dv)
    t_irr = torch.empty((P, r_hi, r_hi, 3), dtype=f32, device=dv)
    t_lo = torch.empty((P, r_lo, r_lo), dtype=f32, device=dv)
    skipped = np.zeros(P, np.int64)
    st = stream if stream is not None else torch.cuda.current_stream(dv)
    vp = ctypes.c_void_p
    native.check(native.lib().lfp_bake_points(
        device, pos.ctypes.data_as(vp), col.ctypes.data_as(vp), len(pos),
        origins.ctypes.data_as(vp), P, r_hi, r_lo, 0, vp(t_dist.data_ptr()),
        vp(t_dir.data_ptr()), vp(t_irr.data_ptr()), vp(t_lo.data_ptr()),
        skipped.ctypes.data_as(vp), vp(st.cuda_stream)))
    return (t_dist, t_dir, t_irr, t_lo), skipped


def _check_skipped(skipped, n):
    for s in np.atleast_1d(skipped):
        if s:
            print(f"bake_probe: skipped {int(s)} points coincident with the "
                  f"probe origin", file=sys.stderr)
        if s >= n:
            raise ValueError("no usable points for bake")


def bake_probe(cloud, origin, r_hi=2048, r_lo=128, source="") -> ProbeData:
    """`bake.py:140-207` on the GPU: one probe, host maps."""
    if r_hi % r_lo != 0:
        raise ValueError("r_hi must be a multiple of r_lo")
    origin = np.asarray(origin, dtype=np.float64)
    (d, dr, ir, lo), skipped = bake_points_device(cloud, origin[None], r_hi,
                                                  r_lo)
    _check_skipped(skipped, len(cloud.positions))
    chain = MapChain(irradiance_hi=ir[0].cpu().numpy(),
                     distance_hi=d[0].cpu().numpy(),
                     direction_hi=dr[0].cpu().numpy(),
                     distance_lo=lo[0].cpu().numpy(),
                     direction_lo=texel_center_directions(r_lo).astype(
                         np.float32))
    b_lo, b_hi = cloud.bounds
    return ProbeData(origin=origin, chain=chain, bounds_lo=b_lo,
                     bounds_hi=b_hi, source=source,
                     point_count=len(cloud.positions), timestamp=time.time())


def simulate_probe(cloud, origin, r_hi=2048, r_lo=128, source="") -> ProbeData:
    """`bake.py:210-222`: bake anywhere; warns outside the cloud bounds."""
    origin = np.asarray(origin, dtype=np.float64)
    lo, hi = cloud.bounds
    if np.any(origin < lo) or np.any(origin > hi):
        print(f"simulate_probe: origin {origin.tolist()} is outside the "
              f"cloud bounds", file=sys.stderr)
    return bake_probe(cloud, origin, r_hi=r_hi, r_lo=r_lo, source=source)


def bake_grid(cloud, grid_origin, cell_size, dims, r_hi=512, r_lo=64,
              source="", device=0, host_maps=True) -> ProbeGrid:
    """`grid.py:96-109`: a probe at every lattice vertex, all probes in one
    bake. The device maps become the grid's resident probe set; with
    host_maps the host ProbeSet arrays are filled too (the reference
    layout, for save_grid / inspection)."""
    from . import device as dev
    from .bake import lattice_origins

    if r_hi % r_lo != 0:
        raise ValueError("r_hi must be a multiple of r_lo")
    nx, ny, nz = (int(x) for x in dims)
    origins = lattice_origins(grid_origin, cell_size, (nx, ny, nz))
    tensors, skipped = bake_points_device(cloud, origins, r_hi, r_lo, device)
    _check_skipped(skipped, len(cloud.positions))
    t_dist, t_dir, t_irr, t_lo = tensors
    dps = dev.DeviceProbeSet.from_device_tensors(t_dist, t_dir, t_irr, t_lo,
                                                 origins, device=device)
    if host_maps:
        ps = ProbeSet(arrays=(t_dist.cpu().numpy(), t_dir.cpu().numpy(),
                              t_irr.cpu().numpy(), t_lo.cpu().numpy(),
                              origins))
    else:
        ps = _LazyProbeSet(tensors, origins)
    grid = ProbeGrid(grid_origin, cell_size, (nx, ny, nz), probe_set=ps)
    if host_maps:
        dev.register(dps, (ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo,
                           ps.origins), device)
    grid._device_probe_set = dps
    return grid


class _LazyProbeSet(ProbeSet):
    """Device-only probe set: shapes and origins on the host, maps copied
    back on first attribute access."""

    def __init__(self, tensors, origins):
        self._t = tensors
        self.probes = None
        self.origins = origins
        self._host = None

    def _load(self):
        if self._host is None:
            self._host = [t.cpu().numpy() for t in self._t]
        return self._host

    dist_hi = property(lambda self: self._load()[0])
    dir_hi = property(lambda self: self._load()[1])
    irr_hi = property(lambda self: self._load()[2])
    dist_lo = property(lambda self: self._load()[3])

    @property
    def n_probes(self):
        return self._t[0].shape[0]

    @property
    def res_hi(self):
        return self._t[0].shape[1]

    @property
    def res_lo(self):
        return self._t[3].shape[1]
