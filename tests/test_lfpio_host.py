"""Host-side .lfp parsing (no GPU): header fields and validation errors
match the reference's loader (bake.py:301-320)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2507_14624_b200 import lfpio


def test_header_and_sizes():
    rec = lfpio.read_probe_file(os.path.join(GOLDEN, "lfp_grid",
                                             "probe_0_1_1.lfp"))
    assert (rec["r_hi"], rec["r_lo"]) == (64, 16)
    np.testing.assert_allclose(rec["origin"], [0.5, 2.25, 2.5])
    assert rec["source"] == "golden"
    assert lfpio.computed_file_size(64, 16) == os.path.getsize(
        os.path.join(GOLDEN, "lfp_grid", "probe_0_1_1.lfp"))
    # the reference's documented 2048^2/128^2 budget (C5 acceptance)
    assert lfpio.computed_file_size(2048, 128) == 25231536


def test_format_errors(tmp_path):
    data = open(os.path.join(GOLDEN, "lfp_grid", "probe_0_0_0.lfp"), "rb").read()
    p = tmp_path / "x.lfp"
    p.write_bytes(data[:40])
    with pytest.raises(lfpio.ProbeFormatError, match="truncated header"):
        lfpio.read_probe_file(str(p))
    hdr = bytearray(data)
    off = 8 + 3 * 8 + 2 * 4
    hdr[off:off + 2] = (9).to_bytes(2, "little")
    p.write_bytes(bytes(hdr))
    with pytest.raises(lfpio.ProbeFormatError, match="format codes"):
        lfpio.read_probe_file(str(p))
