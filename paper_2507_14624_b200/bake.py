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


def scene_prims(scene):
    """Scene primitives / light as the C structs of lfp_bake_probes."""
    from . import native
    from .scenes import Box
    prims = (native.PrimC * len(scene.primitives))()
    for i, p in enumerate(scene.primitives):
        if isinstance(p, Box):
            prims[i].kind = 0
            a, b = p.lo, p.hi
        else:
            prims[i].kind = 1
            a, b = p.center, (p.radius, 0.0, 0.0)
        for k in range(3):
            prims[i].a[k] = float(a[k])
            prims[i].b[k] = float(b[k])
            prims[i].albedo[k] = float(p.albedo[k])
    light = native.LightC()
    for k in range(3):
        light.position[k] = float(scene.light.position[k])
    light.power = float(scene.light.power)
    light.ambient = float(scene.light.ambient)
    return prims, light


def bake_probes_gpu(scene, origins, r_hi, r_lo, quant="f32", shadows=True,
                    device=0, keep_device=False):
    """GPU ray-cast bake (`lfp_bake_probes`); returns a host ProbeSet (and
    the device tensors when keep_device)."""
    import ctypes

    import torch

    from . import native
    if r_hi % r_lo != 0:
        raise ValueError("r_hi must be a multiple of r_lo")
    if not torch.cuda.is_available():
        raise native.LfpError("GPU bake needs a CUDA device")
    origins = np.ascontiguousarray(np.asarray(origins, np.float64).reshape(-1, 3))
    P = len(origins)
    dv = torch.device("cuda", device)
    t_dist = torch.empty((P, r_hi, r_hi), dtype=torch.float32, device=dv)
    t_dir = torch.empty((P, r_hi, r_hi, 3), dtype=torch.float32, device=dv)
    t_irr = torch.empty((P, r_hi, r_hi, 3), dtype=torch.float32, device=dv)
    t_lo = torch.empty((P, r_lo, r_lo), dtype=torch.float32, device=dv)
    prims, light = scene_prims(scene)
    st = torch.cuda.current_stream(dv)
    vp = ctypes.c_void_p
    native.check(native.lib().lfp_bake_probes(
        device, prims, len(scene.primitives), ctypes.byref(light),
        origins.ctypes.data_as(vp), P, r_hi, r_lo, int(quant == "f16"),
        int(bool(shadows)), vp(t_dist.data_ptr()), vp(t_dir.data_ptr()),
        vp(t_irr.data_ptr()), vp(t_lo.data_ptr()), vp(st.cuda_stream)))
    ps = ProbeSet(arrays=(t_dist.cpu().numpy(), t_dir.cpu().numpy(),
                          t_irr.cpu().numpy(), t_lo.cpu().numpy(), origins))
    if keep_device:
        return ps, (t_dist, t_dir, t_irr, t_lo)
    return ps


def bake_grid_gpu(scene, grid_origin, cell, dims, r_hi, r_lo, quant="f32",
                  shadows=True, device=0):
    ps = bake_probes_gpu(scene, lattice_origins(grid_origin, cell, dims),
                         r_hi, r_lo, quant=quant, shadows=shadows,
                         device=device)
    return ProbeGrid(grid_origin, cell, dims, probe_set=ps)


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
