"""Point-cloud bake (bake.py:140-207, grid.py:96-109): oracle pinned to the
reference's outputs (CPU), then the CUDA bake (lfp_bake_points) bit-exact
against both (GPU). Bar: integer / byte work -> identical maps."""

import hashlib
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

from oracle import bake_oracle  # noqa: E402  (test infrastructure)

MAPS = ("irradiance_hi", "distance_hi", "direction_hi", "distance_lo",
        "direction_lo")
KEYS = {"irradiance_hi": "irr", "distance_hi": "dist", "direction_hi": "dir",
        "distance_lo": "lo", "direction_lo": "dirlo"}
CASES = (("room_a_", "room", (2.0, 1.5, 2.0), 64, 16),
         ("room_b_", "room", (0.7, 0.4, 3.1), 32, 8),
         ("tie_a_", "tie", (0.0, 0.0, 0.0), 4, 2),
         ("tie_b_", "tie", (0.0, 0.0, 0.0), 16, 4),
         ("tie_c_", "tie", (10.0, -3.0, 2.0), 8, 2),
         ("tie_d_", "tie", (10.0, -3.0, 2.0), 64, 16),
         ("rand_", "rand", (0.0, 0.0, 0.0), 16, 4))


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(
        a.view(np.uint32) if a.dtype == np.float32 else a,
        b.view(np.uint32) if b.dtype == np.float32 else b)


def _diff(a, b):
    """Where two maps differ (assertion message)."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return f"shape/dtype {a.shape} {a.dtype} vs {b.shape} {b.dtype}"
    av = a.view(np.uint32) if a.dtype == np.float32 else a
    bv = b.view(np.uint32) if b.dtype == np.float32 else b
    bad = np.argwhere(av != bv)
    if len(bad) == 0:
        return "equal"
    i = tuple(bad[0])
    return f"{len(bad)} differ; first {i}: {a[i]!r} vs {b[i]!r}"


@pytest.fixture(scope="module")
def pb(golden):
    return golden("pointbake")


@pytest.fixture(scope="module")
def clouds(pb):
    from paper_2507_14624_b200 import scenes
    from paper_2507_14624_b200.pointcloud import PointCloud
    room = scenes.sample_point_cloud(scenes.room_scene(11), 100.0, seed=5)
    h = hashlib.sha256(room.positions.tobytes() + room.colors.tobytes())
    assert h.hexdigest() == str(pb["room_digest"]), "room cloud generator drifted"
    return {"room": room,
            "tie": PointCloud(pb["tie_pos"], pb["tie_col"]),
            "rand": PointCloud(pb["rand_pos"], pb["rand_col"])}


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference(pb, clouds, case):
    prefix, cloud, origin, rh, rl = case
    c = clouds[cloud]
    out = bake_oracle.bake_maps(c.positions, c.colors, origin, rh, rl)
    for m in MAPS:
        assert _same(out[m], pb[prefix + KEYS[m]]), (prefix, m)


def test_oracle_grid_matches_reference(pb, clouds):
    from paper_2507_14624_b200.bake import lattice_origins
    c = clouds["room"]
    org = lattice_origins(pb["grid_origin"], float(pb["cell"]),
                          tuple(pb["dims"]))
    assert np.array_equal(org, pb["origins"])
    d, dr, ir, lo, sk = bake_oracle.bake_grid_maps(c.positions, c.colors, org,
                                                   32, 8)
    for a, k in ((d, "dist_hi"), (dr, "dir_hi"), (ir, "irr_hi"),
                 (lo, "dist_lo")):
        assert _same(a, pb[k]), k
    assert (sk == 0).all()


def test_tie_cloud_exercises_edges(pb):
    """The crafted cloud really contains the edge cases it claims."""
    d = pb["tie_d_dist"]
    assert np.isinf(d).any() and np.isfinite(d).any()
    occupied = (pb["tie_d_irr"] != 0).any(-1) | (pb["tie_d_dir"] != 0).any(-1)
    assert (occupied & np.isinf(d)).any(), "f16 overflow texel expected"
    for k in ("tie_d_dist",):
        vals = set(np.unique(pb[k][np.isfinite(pb[k])]).tolist())
        assert 2048.0 in vals and 2052.0 in vals, k   # halfway 2049 / 2051
        assert min(vals) < 6.1e-5                       # float16 subnormal


def test_pointcloud_contract(tmp_path):
    from paper_2507_14624_b200.pointcloud import (PointCloud, PointCloudError,
                                                  load_xyz, save_xyz)
    with pytest.raises(PointCloudError):
        PointCloud(np.zeros((0, 3)), np.zeros((0, 3)))
    with pytest.raises(PointCloudError):
        PointCloud(np.array([[np.nan, 0, 0]]), np.zeros((1, 3)))
    c = PointCloud(np.array([[1.0, 2.0, 3.0], [0.5, -1, 2]]),
                   np.array([[1.0, 0.5, 0.0], [0.2, 0.4, 0.6]]))
    assert not c.positions.flags.writeable
    p = tmp_path / "c.xyz"
    save_xyz(c, p)
    r = load_xyz(p)
    assert np.allclose(r.positions, c.positions, atol=1e-6)
    assert np.allclose(r.colors, c.colors, atol=1 / 255)
    p.write_text("1 2 3 4 5 6\n" + "bad line\n" + "1 2 3 0 0 0\n" * 20)
    with pytest.raises(PointCloudError, match="malformed"):
        load_xyz(p)


def test_bake_argument_errors():
    from paper_2507_14624_b200 import pointbake
    from paper_2507_14624_b200.pointcloud import PointCloud
    c = PointCloud(np.array([[0.0, 2.0, 0.0]]), np.ones((1, 3)))
    with pytest.raises(ValueError, match="multiple"):
        pointbake.bake_probe(c, (0, 0, 0), r_hi=10, r_lo=4)
    with pytest.raises(ValueError, match="multiple"):
        pointbake.bake_grid(c, (0, 0, 0), 1.0, (2, 2, 2), r_hi=10, r_lo=4)


# ------------------------------------------------------------------ GPU ----

def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    import __graft_entry__
    __graft_entry__.build()
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_gpu_bake_matches_reference(pb, clouds, case):
    _gpu()
    from paper_2507_14624_b200 import pointbake
    prefix, cloud, origin, rh, rl = case
    pr = pointbake.bake_probe(clouds[cloud], origin, r_hi=rh, r_lo=rl)
    for m in MAPS:
        g = getattr(pr.chain, m)
        assert _same(g, pb[prefix + KEYS[m]]), (prefix, m,
                                                  _diff(g, pb[prefix + KEYS[m]]))
    assert pr.point_count == len(clouds[cloud])


@pytest.mark.gpu
def test_gpu_bake_grid_matches_reference(pb, clouds):
    _gpu()
    from paper_2507_14624_b200 import pointbake
    g = pointbake.bake_grid(clouds["room"], pb["grid_origin"],
                            float(pb["cell"]), tuple(pb["dims"]), r_hi=32,
                            r_lo=8)
    ps = g.probe_set
    for k in ("dist_hi", "dir_hi", "irr_hi", "dist_lo", "origins"):
        assert _same(getattr(ps, k), pb[k]), k


@pytest.mark.gpu
def test_gpu_bake_skip_warning(capsys):
    _gpu()
    from paper_2507_14624_b200 import pointbake
    from paper_2507_14624_b200.pointcloud import PointCloud
    c = PointCloud(np.array([[0.0, 0.0, 0.0], [0.0, 2.0, 0.0]]),
                   np.zeros((2, 3)))
    pr = pointbake.bake_probe(c, (0, 0, 0), r_hi=4, r_lo=2)
    assert "skipped 1 points" in capsys.readouterr().err
    assert np.isfinite(pr.chain.distance_hi).sum() == 1
    assert pr.chain.distance_hi[2, 2] == 2.0     # test_bake.py:21-29 example
    only = PointCloud(np.zeros((1, 3)), np.zeros((1, 3)))
    with pytest.raises(ValueError, match="no usable points"):
        pointbake.bake_probe(only, (0, 0, 0), r_hi=4, r_lo=2)


@pytest.mark.gpu
def test_gpu_bake_order_independent_and_oracle_at_scale():
    """200k points, 512^2 maps, 3 probes in one launch: identical to the
    oracle, and to the bake of a shuffled cloud (bake.py:116-118)."""
    torch = _gpu()
    from paper_2507_14624_b200 import pointbake, scenes
    from paper_2507_14624_b200.pointcloud import PointCloud
    c = scenes.sample_point_cloud(scenes.room_scene(3), 1000.0, seed=1)
    perm = np.random.default_rng(0).permutation(len(c))
    cs = PointCloud(c.positions[perm], c.colors[perm])
    org = np.array([[2.0, 1.5, 2.0], [0.5, 0.5, 0.5], [3.7, 2.9, 0.2]])
    (a, _, _, _), _ = pointbake.bake_points_device(c, org, 512, 64)
    tb, _ = pointbake.bake_points_device(cs, org, 512, 64)
    names = ("distance_hi", "direction_hi", "irradiance_hi", "distance_lo")
    for i, o in enumerate(org):
        ref = bake_oracle.bake_maps(c.positions, c.colors, o, 512, 64)
        for t, m in zip(tb, names):
            g = t[i].cpu().numpy()
            assert _same(g, ref[m]), (i, m, _diff(g, ref[m]))
        assert _same(a[i].cpu().numpy(), ref["distance_hi"])
    assert len(c) > 200_000
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_gpu_baked_grid_renders_like_oracle():
    """bake_grid leaves the probe set resident; render_frame on it equals
    the C oracle traced over the same (GPU-baked) maps."""
    _gpu()
    from oracle import oracle
    from paper_2507_14624_b200 import pointbake, scenes
    from paper_2507_14624_b200.render import Camera, render_frame
    c = scenes.sample_point_cloud(scenes.room_scene(11), 400.0, seed=2)
    g = pointbake.bake_grid(c, (0.0, 0.0, 0.0), 4.0 / 3.0, (4, 3, 4),
                            r_hi=64, r_lo=16)
    assert g._device_probe_set is not None
    cam = Camera(eye=(1.9, 1.4, 2.2), forward=(0.3, -0.1, 1.0), width=96,
                 height=64)
    fr = render_frame(g, cam)
    res, _ = oracle.render_camera(g.probe_set, g.grid_origin, g.cell_size,
                                  g.dims, cam)
    px, st = oracle.frame_pixels(res, cam.height, cam.width)
    assert np.array_equal(fr.status, st)
    assert np.array_equal(fr.pixels, px)
    assert (st == 1).mean() > 0.3
