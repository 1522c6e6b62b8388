"""B200-native light-field-probe grid tracer (arXiv 2507.14624 hot path).

Public names mirror the reference package `lfprobe`
(`pkg/src/lfprobe/__init__.py:15-26`) for the traced path: grids and probe
sets, cameras, frames, `render_frame`, `psnr`, `bench_views`, the trace
status codes and `TraceConfig`. Tracing runs in the CUDA library
`liblfprobe_b200.so` (sm_100a) behind the C ABI in include/lfprobe_b200.h.
"""

from .grid import MapChain, ProbeData, ProbeGrid, ProbeHierarchy, ProbeSet
from .octmap import EMPTY_DISTANCE, oct_decode, oct_encode
from .render import (Camera, Frame, bench_views, psnr, render_frame,
                     trace_rays, write_image)
from .trace import HIT, MISS, UNKNOWN, TraceConfig

__all__ = [
    "ProbeData", "MapChain", "ProbeGrid", "ProbeSet", "ProbeHierarchy",
    "HIT", "MISS", "UNKNOWN", "TraceConfig",
    "EMPTY_DISTANCE", "oct_encode", "oct_decode",
    "Camera", "Frame", "render_frame", "psnr", "bench_views", "write_image",
    "trace_rays",
]

__version__ = "0.1.0"
