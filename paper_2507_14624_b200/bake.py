"""Ray-cast probe bake (host, numpy): the input production for the tracer.

The reference bakes probes from point clouds (`pkg/src/lfprobe/bake.py:
140-207`); the BASELINE configurations bake by ray-casting analytic
primitives, which the reference has no code for. Per probe
and texel: direction = texel-centre direction (`octmap.py:46, 75`),
distance = nearest hit t (f32, EMPTY = +inf), direction map = that
direction (the reference's probe->surface "incoming direction",
`kernels.py:247-252`), radiance = Lambertian shading of the hit. The low-res
map is the blockwise MIN (`bake.py:94-102`).

`quant="f16"` pre-quantises radiance and direction through float16 and back,
so the f32 arrays the oracle reads equal the half-precision texels the
device stores.
"""

from __future__ import annotations

import numpy as np

from .grid import ProbeGrid, ProbeSet
from .octmap import texel_center_directions
from .scenes import intersect, shade


def derive_low_res(distance_hi, factor):
    """Blockwise MIN over factor x factor blocks; EMPTY (+inf) is ignored
    and an all-EMPTY block stays EMPTY (`bake.py:94-102`). Accepts
    (R, R) or (P, R, R)."""
    d = np.asarray(distance_hi)
    r_hi = d.shape[-1]
    if r_hi % factor != 0:
        raise ValueError("factor must divide the high resolution")
    r_lo = r_hi // factor
    lead = d.shape[:-2]
    blocks = d.reshape(*lead, r_lo, factor, r_lo, factor)
    return blocks.min(axis=(-3, -1))


def _quantize(a, quant):
    a = np.asarray(a, np.float64)
    if quant == "f16":
        return a.astype(np.float16).astype(np.float32)
    if quant == "f32":
        return a.astype(np.float32)
    raise ValueError(f"unknown quantisation {quant!r}")


def bake_probes(scene, origins, r_hi, r_lo, quant="f32", shadows=True,
                chunk_rays=1 << 20):
    """Bake probes at `origins` (P, 3); returns a ProbeSet."""
    if r_hi % r_lo != 0:
        raise ValueError("r_hi must be a multiple of r_lo")
    origins = np.asarray(origins, np.float64).reshape(-1, 3)
    n_p = len(origins)
    dirs = texel_center_directions(r_hi).reshape(-1, 3)
    n_t = len(dirs)
    dist_hi = np.full((n_p, n_t), np.inf, np.float32)
    dir_hi = np.zeros((n_p, n_t, 3), np.float32)
    irr_hi = np.zeros((n_p, n_t, 3), np.float32)
    per = max(1, chunk_rays // n_t)
    for p0 in range(0, n_p, per):
        p1 = min(n_p, p0 + per)
        o = np.repeat(origins[p0:p1], n_t, axis=0)
        d = np.tile(dirs, (p1 - p0, 1))
        t, prim = intersect(scene, o, d)
        rgb = shade(scene, o, d, t, prim, shadows=shadows)
        hit = (prim >= 0).reshape(p1 - p0, n_t)
        dist_hi[p0:p1] = np.where(hit, t.reshape(p1 - p0, n_t), np.inf
                                  ).astype(np.float32)
        dq = _quantize(d.reshape(p1 - p0, n_t, 3), quant)
        dir_hi[p0:p1] = np.where(hit[..., None], dq, 0.0)
        irr_hi[p0:p1] = np.where(hit[..., None],
                                 _quantize(rgb.reshape(p1 - p0, n_t, 3), quant),
                                 0.0)
    dist_hi = dist_hi.reshape(n_p, r_hi, r_hi)
    dist_lo = derive_low_res(dist_hi, r_hi // r_lo).astype(np.float32)
    return ProbeSet(arrays=(dist_hi, dir_hi.reshape(n_p, r_hi, r_hi, 3),
                            irr_hi.reshape(n_p, r_hi, r_hi, 3), dist_lo,
                            origins))


def lattice_origins(grid_origin, cell, dims):
    nx, ny, nz = dims
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz),
                             indexing="ij")
    idx = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], -1).astype(np.float64)
    return np.asarray(grid_origin, np.float64) + float(cell) * idx


def bake_grid(scene, grid_origin, cell, dims, r_hi, r_lo, quant="f32",
              shadows=True):
    """Ray-cast bake of a probe at every lattice vertex -> ProbeGrid."""
    ps = bake_probes(scene, lattice_origins(grid_origin, cell, dims),
                     r_hi, r_lo, quant=quant, shadows=shadows)
    return ProbeGrid(grid_origin, cell, dims, probe_set=ps)
