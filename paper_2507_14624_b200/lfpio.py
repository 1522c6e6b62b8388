""".lfp probe files and grid manifests loaded straight to the device
(SURVEY.md §8(f) row 3).

File format (reference `pkg/src/lfprobe/bake.py:27-34, 228-341`): magic
`LFPROBE1`, header `<3dII3H2x6dQd64s` (origin, r_hi, r_lo, format codes,
bounds, point count, timestamp, source), then irradiance RGB565, distance
f16, 2 x u8 sub-texel direction for the hi-res maps and f16 distance + 2 x u8
direction for the low-res maps. The manifest is the reference's JSON
(`grid.py:243-274`).

The host only parses headers and slices the payload bytes; the packed
payloads (6 B per texel instead of 28 B of f32 maps) go to the GPU, which
decodes them exactly as `load_probe` does (`lfp_probeset_create_packed`).
The decoded arrays are copied back into the ProbeSet mirror so host-side
users (and the oracle) see the reference's arrays.
"""

from __future__ import annotations

import ctypes
import json
import os
import struct

import numpy as np

from . import device as dev
from . import native
from .grid import MapChain, ProbeData, ProbeGrid, ProbeSet

MAGIC = b"LFPROBE1"
FMT_IRR_RGB565 = 1
FMT_DIST_F16 = 2
FMT_DIR_SUBTEXEL8 = 3
_HEADER = struct.Struct("<3dII3H2x6dQd64s")


class ProbeFormatError(Exception):
    """Malformed probe file (`bake.py:37-38`)."""


def computed_file_size(r_hi, r_lo):
    """Bytes of a probe file under the documented layout (`bake.py:272-276`)."""
    return len(MAGIC) + _HEADER.size + r_hi * r_hi * 6 + r_lo * r_lo * 4


def read_probe_file(path):
    """Parse and validate one .lfp file (errors as `bake.py:301-320`);
    returns the header fields and zero-copy payload views."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:len(MAGIC)] != MAGIC:
        raise ProbeFormatError(f"{path}: bad magic, not a probe file")
    off = len(MAGIC)
    try:
        fields = _HEADER.unpack_from(data, off)
    except struct.error:
        raise ProbeFormatError(f"{path}: truncated header") from None
    off += _HEADER.size
    ox, oy, oz, r_hi, r_lo, f_irr, f_dist, f_dir = fields[:8]
    if (f_irr, f_dist, f_dir) != (FMT_IRR_RGB565, FMT_DIST_F16,
                                  FMT_DIR_SUBTEXEL8):
        raise ProbeFormatError(f"{path}: unsupported payload format codes "
                               f"{(f_irr, f_dist, f_dir)}")
    expected = computed_file_size(r_hi, r_lo)
    if len(data) != expected:
        raise ProbeFormatError(
            f"{path}: expected {expected} bytes, got {len(data)}")
    n_hi, n_lo = r_hi * r_hi, r_lo * r_lo
    buf = np.frombuffer(data, dtype=np.uint8)
    irr = buf[off:off + 2 * n_hi].view("<u2"); off += 2 * n_hi
    dist = buf[off:off + 2 * n_hi].view("<u2"); off += 2 * n_hi
    dirq = buf[off:off + 2 * n_hi]; off += 2 * n_hi
    dist_lo = buf[off:off + 2 * n_lo].view("<u2")
    return {"origin": np.array([ox, oy, oz]), "r_hi": r_hi, "r_lo": r_lo,
            "bounds_lo": np.array(fields[8:11]),
            "bounds_hi": np.array(fields[11:14]),
            "point_count": fields[14], "timestamp": fields[15],
            "source": fields[16].rstrip(b"\x00").decode("utf-8"),
            "irr": irr, "dist": dist, "dir": dirq, "dist_lo": dist_lo}


def _upload_packed(recs, device=0):
    """Decode a list of parsed probe files on the device; returns the
    DeviceProbeSet and the decoded host arrays."""
    import torch
    res = {(r["r_hi"], r["r_lo"]) for r in recs}
    if len(res) != 1:
        raise ValueError("all probes must share the same resolutions")
    (R, r), = res
    P = len(recs)
    irr = np.ascontiguousarray(np.concatenate([x["irr"] for x in recs]))
    dist = np.ascontiguousarray(np.concatenate([x["dist"] for x in recs]))
    dirq = np.ascontiguousarray(np.concatenate([x["dir"] for x in recs]))
    lo = np.ascontiguousarray(np.concatenate([x["dist_lo"] for x in recs]))
    origins = np.ascontiguousarray(np.stack([x["origin"] for x in recs]),
                                   dtype=np.float64)
    h_dist = np.empty((P, R, R), np.float32)
    h_dir = np.empty((P, R, R, 3), np.float32)
    h_irr = np.empty((P, R, R, 3), np.float32)
    h_lo = np.empty((P, r, r), np.float32)
    d = dev._require_cuda(device)
    handle = ctypes.c_void_p()
    vp = ctypes.c_void_p
    with torch.cuda.device(d):
        st = torch.cuda.current_stream(d)
        native.check(native.lib().lfp_probeset_create_packed(
            d.index, irr.ctypes.data_as(vp), dist.ctypes.data_as(vp),
            dirq.ctypes.data_as(vp), lo.ctypes.data_as(vp),
            origins.ctypes.data_as(vp), P, R, r, native.LFP_FMT_AUTO_HALF,
            h_dist.ctypes.data_as(vp), h_dir.ctypes.data_as(vp),
            h_irr.ctypes.data_as(vp), h_lo.ctypes.data_as(vp),
            vp(st.cuda_stream), ctypes.byref(handle)))
    dps = dev.DeviceProbeSet.from_handle(handle, d, P, R, r)
    return dps, (h_dist, h_dir, h_irr, h_lo, origins)


def _probe_data(rec, arrays, p):
    h_dist, h_dir, h_irr, h_lo, origins = arrays
    r = rec["r_lo"]
    chain = MapChain(irradiance_hi=h_irr[p], distance_hi=h_dist[p],
                     direction_hi=h_dir[p], distance_lo=h_lo[p],
                     direction_lo=np.zeros((r, r, 3), np.float32))
    return ProbeData(origin=origins[p], chain=chain,
                     bounds_lo=rec["bounds_lo"], bounds_hi=rec["bounds_hi"],
                     source=rec["source"])


def load_probe(path, device=0) -> ProbeData:
    """`bake.load_probe` (bake.py:301-341) with the decode on the GPU."""
    rec = read_probe_file(path)
    dps, arrays = _upload_packed([rec], device)
    probe = _probe_data(rec, arrays, 0)
    c = probe.chain
    dev.register(dps, (c.distance_hi, c.direction_hi, c.irradiance_hi,
                       c.distance_lo), device)
    return probe


def load_grid(manifest_path, device=0) -> ProbeGrid:
    """`grid.load_grid` (grid.py:268-274): manifest + per-probe files, one
    packed upload, decoded on the device; the returned grid's device probe
    set is already resident for render_frame."""
    with open(manifest_path) as fh:
        manifest = json.load(fh)
    base = os.path.dirname(os.path.abspath(manifest_path))
    recs = [read_probe_file(os.path.join(base, p)) for p in manifest["probes"]]
    dps, arrays = _upload_packed(recs, device)
    probes = [_probe_data(rec, arrays, p) for p, rec in enumerate(recs)]
    ps = ProbeSet(arrays=arrays)
    ps.probes = probes
    grid = ProbeGrid(manifest["gridOrigin"], manifest["cellSize"],
                     manifest["dims"], probes, probe_set=ps)
    dev.register(dps, (ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo,
                       ps.origins), device)
    return grid
