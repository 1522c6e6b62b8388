"""Trace constants and configuration (`pkg/src/lfprobe/trace.py:32-40`,
`kernels.py:18-27`)."""

from __future__ import annotations

from dataclasses import dataclass

MISS = 0
HIT = 1
UNKNOWN = 2

STATUS_NAMES = {MISS: "MISS", HIT: "HIT", UNKNOWN: "UNKNOWN"}

DEFAULT_SLACK = 1e-3       # distance comparison slack (kernels.py:23)
DEFAULT_EPS_START = 1e-4   # ray start offset (kernels.py:25)
DEFAULT_EPS_ALIGN = 1e-4   # eye-at-probe threshold (kernels.py:27)


@dataclass(frozen=True)
class TraceConfig:
    eps_start: float = DEFAULT_EPS_START
    eps_align: float = DEFAULT_EPS_ALIGN
    slack: float = DEFAULT_SLACK
    bounds_pad: float = 0.5


DEFAULT_CONFIG = TraceConfig()
