"""ctypes binding of the C ABI in include/lfprobe_b200.h.

The shared library `liblfprobe_b200.so` is built in-tree by
`__graft_entry__.build()` (nvcc, sm_100a). There is no fallback: if the
library or a GPU is missing every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LFP_LIB_PATH selects an alternative build (tools/build_variants.py)
LIB_PATH = os.environ.get("LFP_LIB_PATH") or os.path.join(_HERE,
                                                          "liblfprobe_b200.so")

LFP_SRC_DEVICE = 0x1
LFP_FMT_AUTO_HALF = 0x2
LFP_FMT_FORCE_F32 = 0x4

LFP_SOURCE_SINGLE = 1
LFP_SOURCE_FEW = 2
LFP_SOURCE_LOOKUP = 3


class LfpError(RuntimeError):
    pass


class GridParams(ctypes.Structure):
    _fields_ = [("grid_origin", ctypes.c_double * 3),
                ("cell", ctypes.c_double),
                ("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("nz", ctypes.c_int32),
                ("eps_start", ctypes.c_double),
                ("eps_align", ctypes.c_double),
                ("slack", ctypes.c_double),
                ("trace_mode", ctypes.c_int32),
                ("schedule", ctypes.c_int32),
                ("min_active", ctypes.c_int32)]


class CameraC(ctypes.Structure):
    _fields_ = [("eye", ctypes.c_double * 3),
                ("basis", ctypes.c_double * 9),
                ("tan_v", ctypes.c_double), ("tan_h", ctypes.c_double)]


class PrimC(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("a", ctypes.c_double * 3),
                ("b", ctypes.c_double * 3), ("albedo", ctypes.c_float * 3)]


class LightC(ctypes.Structure):
    _fields_ = [("position", ctypes.c_double * 3), ("power", ctypes.c_double),
                ("ambient", ctypes.c_double)]


class Outputs(ctypes.Structure):
    _fields_ = [("status", ctypes.c_void_p), ("rgb", ctypes.c_void_p),
                ("probe", ctypes.c_void_p), ("texel", ctypes.c_void_p),
                ("fetch", ctypes.c_void_p), ("hit_t", ctypes.c_void_p),
                ("stats", ctypes.c_void_p),
                ("diag", ctypes.c_void_p),
                ("rgb_mode", ctypes.c_int32),
                ("background", ctypes.c_float * 3),
                ("unknown_color", ctypes.c_float * 3),
                ("rgb8", ctypes.c_void_p)]


_lib = None


def lib():
    """Load the CUDA library; raises LfpError if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LfpError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, "
                "sm_100a). There is no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u32 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                             ctypes.c_uint32)
        L.lfp_version.restype = ctypes.c_int
        L.lfp_last_error.restype = ctypes.c_char_p
        L.lfp_last_launches.restype = ctypes.c_int64
        L.lfp_probeset_create.argtypes = [
            ctypes.c_int, vp, vp, vp, vp, vp, i64, i32, i32, u32, vp,
            ctypes.POINTER(vp)]
        L.lfp_probeset_create_packed.argtypes = [
            ctypes.c_int, vp, vp, vp, vp, vp, i64, i32, i32, u32, vp, vp, vp,
            vp, vp, ctypes.POINTER(vp)]
        L.lfp_probeset_destroy.argtypes = [vp]
        L.lfp_probeset_info.argtypes = [vp, ctypes.POINTER(i64),
                                        ctypes.POINTER(i32),
                                        ctypes.POINTER(i32)]
        L.lfp_render_cameras.argtypes = [
            vp, ctypes.POINTER(GridParams), ctypes.POINTER(CameraC), i32, i32,
            i32, i64, i64, i64, i32, ctypes.POINTER(Outputs), vp]
        L.lfp_render_frame_host.argtypes = [
            vp, ctypes.POINTER(GridParams), ctypes.POINTER(CameraC), i32, i32,
            ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float), vp,
            vp, vp, vp, ctypes.POINTER(ctypes.c_float), vp]
        L.lfp_render_probes.argtypes = [
            vp, i32, ctypes.POINTER(i32), i32, ctypes.POINTER(ctypes.c_double),
            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(GridParams),
            ctypes.POINTER(CameraC), i32, i32, i32, ctypes.POINTER(Outputs), vp]
        L.lfp_render_hierarchy.argtypes = [
            ctypes.POINTER(vp), ctypes.POINTER(GridParams), i32,
            ctypes.POINTER(CameraC), i32, i32, i32, i64, i64, i64, i32,
            ctypes.POINTER(Outputs), vp]
        L.lfp_num_tiles.argtypes = [i32, i32, i32]
        L.lfp_num_tiles.restype = i64
        L.lfp_render_grid.argtypes = [
            vp, ctypes.POINTER(GridParams), ctypes.POINTER(ctypes.c_double),
            vp, i32, i64, ctypes.POINTER(Outputs), vp]
        L.lfp_trace_rays.argtypes = [
            vp, ctypes.POINTER(GridParams), vp, vp, i32, i64,
            ctypes.POINTER(Outputs), vp]
        L.lfp_bin_rays.argtypes = [ctypes.POINTER(GridParams), vp, vp, i32,
                                    i64, vp, vp]
        L.lfp_trace_rays_ordered.argtypes = [
            vp, ctypes.POINTER(GridParams), vp, vp, i32, i64, vp,
            ctypes.POINTER(Outputs), vp]
        L.lfp_selftest_division.argtypes = [vp, vp, i64, vp, vp, vp, vp]
        L.lfp_selftest_division_recip.argtypes = [vp, vp, i64, vp, vp, vp, vp]
        L.lfp_debug_bounds.argtypes = [ctypes.c_int, vp, i64]
        L.lfp_debug_report.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                                       ctypes.POINTER(i32)]
        L.lfp_untile.argtypes = [i32, i32, i32, i32, i64, vp, vp, vp, vp, vp]
        L.lfp_bake_probes.argtypes = [
            ctypes.c_int, ctypes.POINTER(PrimC), i32, ctypes.POINTER(LightC),
            vp, i64, i32, i32, i32, i32, vp, vp, vp, vp, vp]
        L.lfp_bake_points.argtypes = [
            ctypes.c_int, vp, vp, i64, vp, i64, i32, i32, u32, vp, vp, vp, vp,
            vp, vp]
        for name in ("lfp_selftest_division", "lfp_selftest_division_recip",
                     "lfp_debug_bounds",
                     "lfp_debug_report", "lfp_bake_points", "lfp_render_hierarchy", "lfp_probeset_create_packed",
                     "lfp_render_frame_host",
                     "lfp_bin_rays", "lfp_trace_rays_ordered",
                     "lfp_bake_probes", "lfp_render_probes",
                     "lfp_probeset_create", "lfp_probeset_destroy",
                     "lfp_probeset_info", "lfp_render_cameras",
                     "lfp_render_grid", "lfp_trace_rays", "lfp_untile"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def check(rc):
    if rc != 0:
        msg = lib().lfp_last_error().decode(errors="replace")
        raise LfpError(f"lfprobe_b200 error {rc}: {msg}")


def exported_symbols():
    """Names declared in include/lfprobe_b200.h (for the ABI load test)."""
    return ["lfp_version", "lfp_last_error", "lfp_probeset_create",
            "lfp_probeset_destroy", "lfp_probeset_info", "lfp_render_cameras",
            "lfp_num_tiles", "lfp_render_grid", "lfp_trace_rays",
            "lfp_untile", "lfp_bake_probes", "lfp_render_probes",
            "lfp_bin_rays", "lfp_trace_rays_ordered",
            "lfp_probeset_create_packed", "lfp_render_hierarchy",
            "lfp_bake_points", "lfp_last_launches", "lfp_render_frame_host",
            "lfp_selftest_division", "lfp_selftest_division_recip",
            "lfp_debug_bounds", "lfp_debug_report"]
