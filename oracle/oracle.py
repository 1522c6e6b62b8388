"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads oracle/liblfp_oracle.so (built by `make -C oracle`, or by
__graft_entry__.build()). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` leg may import this module; the
product package never does.

Every function mirrors a reference entry point (see lfp_oracle.c for the
file:line of each restated routine) and takes the reference's array layout.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblfp_oracle.so")
_lib = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64
_dbl = ctypes.c_double


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.lfpo_num_threads.restype = ctypes.c_int
        L.lfpo_set_num_threads.argtypes = [ctypes.c_int]
        L.lfpo_camera_dirs.argtypes = [_f64p, _dbl, _dbl, _i64, _i64, _f64p]
        L.lfpo_trace_rays.argtypes = [
            _f32p, _f32p, _f32p, _f32p, _f64p, _i64, _i64, _i64,
            _f64p, _dbl, _i64, _i64, _i64, _f64p, _i64, _f64p, _i64,
            _dbl, _dbl, _dbl, _u8p, _i32p, _i32p, _i32p, _i64p, _f64p]
        L.lfpo_render_single_probe.argtypes = [
            _f32p, _f32p, _f32p, _f32p, _i64, _i64, _f64p, _f64p, _f64p, _i64,
            _f64p, _f64p, _dbl, _dbl, _u8p, _f64p, _i64p]
        L.lfpo_render_few_probes.argtypes = [
            _f32p, _f32p, _f32p, _f32p, _f64p, _i64, _i64, _i64, _f64p, _f64p,
            _f64p, _f64p, _i64, _dbl, _dbl, _dbl, _u8p, _f64p, _i64p]
        L.lfpo_oct_encode.argtypes = [_dbl, _dbl, _dbl, _f64p]
        L.lfpo_oct_decode.argtypes = [_dbl, _dbl, _f64p]
        L.lfpo_distance_to_intersection.argtypes = [_f64p, _f64p, _f64p]
        L.lfpo_distance_to_intersection.restype = _dbl
        L.lfpo_fold_boundaries.argtypes = [_f64p, _f64p, _dbl, _dbl, _f64p]
        L.lfpo_fold_boundaries.restype = ctypes.c_int
        L.lfpo_trace_probe_range.argtypes = [
            _f32p, _f32p, _f32p, _i64, _i64, _f64p, _f64p, _dbl, _dbl, _dbl,
            ctypes.c_int, _i64p]
        _lib = L
    return _lib


def num_threads():
    return lib().lfpo_num_threads()


def set_num_threads(n):
    lib().lfpo_set_num_threads(int(n))


def _c64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def camera_dirs(basis_ruf, tan_v, tan_h, width, height):
    """render.py:50-62 restated: (H*W, 3) f64 pixel directions."""
    out = np.empty((height * width, 3), np.float64)
    lib().lfpo_camera_dirs(_c64(basis_ruf, (9,)), float(tan_v), float(tan_h),
                           int(width), int(height), out)
    return out


def camera_params(cam):
    """Host-side basis/tan values exactly as Camera.basis/ray_directions
    compute them (render.py:33-55)."""
    r, u, f = cam.basis()
    tan_v = np.tan(np.radians(cam.vfov_deg) / 2.0)
    tan_h = tan_v * cam.width / cam.height
    return np.concatenate([r, u, f]).astype(np.float64), float(tan_v), float(tan_h)


class Result:
    def __init__(self, n):
        self.status = np.zeros(n, np.uint8)
        self.probe = np.zeros(n, np.int32)
        self.tx = np.zeros(n, np.int32)
        self.ty = np.zeros(n, np.int32)
        self.fetch = np.zeros(n, np.int64)
        self.rgb = np.zeros((n, 3), np.float64)


def trace_rays(ps, grid_origin, cell, dims, origins, dirs,
               eps_start=1e-4, eps_align=1e-4, slack=1e-3):
    """kernels.trace_grid_ray (K:653) over a batch; `origins` is (3,) for a
    shared eye or (N, 3)."""
    dirs = _c64(dirs).reshape(-1, 3)
    n = len(dirs)
    o = _c64(origins)
    stride = 0 if o.ndim == 1 else 3
    o = o.reshape(-1)
    res = Result(n)
    nx, ny, nz = dims
    lib().lfpo_trace_rays(
        ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo, _c64(ps.origins),
        ps.dist_hi.shape[0], ps.dist_hi.shape[1], ps.dist_lo.shape[1],
        _c64(grid_origin, (3,)), float(cell), nx, ny, nz, o, stride, dirs, n,
        eps_start, eps_align, slack, res.status, res.probe, res.tx, res.ty,
        res.fetch, res.rgb)
    return res


def render_grid(dist_hi_all, dir_hi_all, irr_all, dist_lo_all, origins,
                grid_origin, cell, nx, ny, nz, eye, dirs, eps_start,
                eps_align, slack, out_status, out_rgb, out_fetch):
    """Same signature and in-place semantics as kernels.render_grid
    (K:825-843)."""
    n = len(dirs)
    tx = np.empty(n, np.int32)
    lib().lfpo_trace_rays(
        dist_hi_all, dir_hi_all, irr_all, dist_lo_all, _c64(origins),
        dist_hi_all.shape[0], dist_hi_all.shape[1], dist_lo_all.shape[1],
        _c64(grid_origin, (3,)), float(cell), int(nx), int(ny), int(nz),
        _c64(eye, (3,)), 0, _c64(dirs), n, eps_start, eps_align, slack,
        out_status, np.empty(n, np.int32), tx, np.empty(n, np.int32),
        out_fetch, out_rgb)


def render_camera(ps, grid_origin, cell, dims, cam, config=None):
    """render_frame(ProbeGrid, cam) restated: returns (Result, dirs)."""
    basis, tan_v, tan_h = camera_params(cam)
    dirs = camera_dirs(basis, tan_v, tan_h, cam.width, cam.height)
    kw = {}
    if config is not None:
        kw = dict(eps_start=config.eps_start, eps_align=config.eps_align,
                  slack=config.slack)
    return trace_rays(ps, grid_origin, cell, dims, np.asarray(cam.eye,
                                                              np.float64),
                      dirs, **kw), dirs


def frame_pixels(res, height, width, background=(0.0, 0.0, 0.0),
                 unknown_color=(1.0, 0.0, 1.0)):
    """render.py:147-150 post-processing."""
    rgb = res.rgb.astype(np.float32)
    rgb[res.status == 0] = np.asarray(background, np.float32)
    rgb[res.status == 2] = np.asarray(unknown_color, np.float32)
    return rgb.reshape(height, width, 3), res.status.reshape(height, width)


def trace_hierarchy(levels, eye, dirs):
    """Coarse-to-fine composition of per-level oracle traces (the reference
    has no hierarchy): MISS rays re-trace on the next
    level, fetches add up, first HIT wins."""
    n = len(dirs)
    out = Result(n)
    out.probe[:] = -1
    out.tx[:] = -1
    out.ty[:] = -1
    todo = np.arange(n)
    for lvl, g in enumerate(levels):
        if len(todo) == 0:
            break
        o = eye if np.ndim(eye) == 1 else eye[todo]
        r = trace_rays(g.probe_set, g.grid_origin, g.cell_size, g.dims,
                              o, dirs[todo])
        out.fetch[todo] += r.fetch
        hit = r.status == 1
        diag = (~hit) & (r.probe >= 0)
        for m in (hit, diag):
            idx = todo[m]
            out.probe[idx] = (lvl << 24) | r.probe[m]
            out.tx[idx] = r.tx[m]
            out.ty[idx] = r.ty[m]
        out.status[todo[hit]] = 1
        out.rgb[todo[hit]] = r.rgb[hit]
        todo = todo[~hit]
    return out



def oct_encode(d):
    out = np.empty(2)
    lib().lfpo_oct_encode(float(d[0]), float(d[1]), float(d[2]), out)
    return out


def oct_decode(uv):
    out = np.empty(3)
    lib().lfpo_oct_decode(float(uv[0]), float(uv[1]), out)
    return out


def distance_to_intersection(w, d, v):
    return lib().lfpo_distance_to_intersection(_c64(w), _c64(d), _c64(v))


def fold_boundaries(w, d, t0, t1):
    out = np.empty(5)
    n = lib().lfpo_fold_boundaries(_c64(w), _c64(d), t0, t1, out)
    return out[:n].copy()


def trace_probe_range(dist_hi, dir_hi, dist_lo, w, d, t0, t1, slack=1e-3,
                      brute=False):
    out = np.empty(4, np.int64)
    lib().lfpo_trace_probe_range(
        np.ascontiguousarray(dist_hi, np.float32),
        np.ascontiguousarray(dir_hi, np.float32),
        np.ascontiguousarray(dist_lo, np.float32),
        dist_hi.shape[0], dist_lo.shape[0], _c64(w), _c64(d), t0, t1, slack,
        int(bool(brute)), out)
    return tuple(int(x) for x in out)


def render_single_probe(dist_hi, dir_hi, irr_hi, dist_lo, origin, eye, dirs,
                        blo, bhi, eps_start, slack):
    n = len(dirs)
    st = np.zeros(n, np.uint8)
    rgb = np.zeros((n, 3))
    fe = np.zeros(n, np.int64)
    lib().lfpo_render_single_probe(
        np.ascontiguousarray(dist_hi, np.float32),
        np.ascontiguousarray(dir_hi, np.float32),
        np.ascontiguousarray(irr_hi, np.float32),
        np.ascontiguousarray(dist_lo, np.float32),
        dist_hi.shape[0], dist_lo.shape[0], _c64(origin), _c64(eye),
        _c64(dirs), n, _c64(blo), _c64(bhi), eps_start, slack, st, rgb, fe)
    return st, rgb, fe


def render_few_probes(ps, blo, bhi, eye, dirs, eps_start, eps_align, slack):
    n = len(dirs)
    st = np.zeros(n, np.uint8)
    rgb = np.zeros((n, 3))
    fe = np.zeros(n, np.int64)
    lib().lfpo_render_few_probes(
        ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo, _c64(ps.origins),
        ps.dist_hi.shape[0], ps.dist_hi.shape[1], ps.dist_lo.shape[1],
        _c64(blo), _c64(bhi), _c64(eye), _c64(dirs), n, eps_start, eps_align,
        slack, st, rgb, fe)
    return st, rgb, fe
