"""Pin the C oracle (oracle/lfp_oracle.c) to the reference's own outputs.

The fixtures under tests/golden/ were produced by running the reference
numba kernels (tests/golden/make_golden.py). Everything here is bit-exact:
status, probe, texel, fetch count and radiance must be identical.
"""

import numpy as np
import pytest

from conftest import GoldenProbeSet, golden_camera
from oracle import oracle


def _check_outputs(res, z, prefix):
    np.testing.assert_array_equal(res.status, z[prefix + "status"])
    np.testing.assert_array_equal(res.probe, z[prefix + "probe"])
    np.testing.assert_array_equal(res.tx, z[prefix + "tx"])
    np.testing.assert_array_equal(res.ty, z[prefix + "ty"])
    np.testing.assert_array_equal(res.fetch, z[prefix + "fetch"])
    if prefix + "rgb" in z:
        np.testing.assert_array_equal(res.rgb, z[prefix + "rgb"])


class TestScalarKAT:
    def test_oct_encode(self, golden):
        z = golden("scalars")
        got = np.array([oracle.oct_encode(d) for d in z["enc_in"]])
        np.testing.assert_array_equal(got, z["enc_out"])
        # reference test constants (pkg/tests/test_octmap.py:14-27)
        assert tuple(oracle.oct_encode([0.0, 1.0, 0.0])) == (0.5, 0.5)
        assert tuple(oracle.oct_encode([1.0, 0.0, 0.0])) == (1.0, 0.5)
        assert tuple(oracle.oct_encode([0.0, -1.0, 0.0])) == (1.0, 1.0)

    def test_oct_decode(self, golden):
        z = golden("scalars")
        got = np.array([oracle.oct_decode(uv) for uv in z["dec_in"]])
        np.testing.assert_array_equal(got, z["dec_out"])
        for uv in ([0, 0], [0, 1], [1, 0], [1, 1]):   # test_octmap.py:29-31
            np.testing.assert_allclose(oracle.oct_decode(uv), [0, -1, 0],
                                       atol=1e-15)

    def test_distance_to_intersection(self, golden):
        z = golden("scalars")
        got = np.array([oracle.distance_to_intersection(w, d, v) for w, d, v in
                        zip(z["d2i_w"], z["d2i_d"], z["d2i_v"])])
        np.testing.assert_array_equal(got, z["d2i_out"])
        # worked examples, pkg/tests/test_trace.py:87-95
        v = np.array([1.0, 0.0, 1.0]) / np.sqrt(2.0)
        assert oracle.distance_to_intersection([1, 0, 0], [0, 0, 1], v) == \
            pytest.approx(np.sqrt(2.0))
        assert oracle.distance_to_intersection(
            [2, 1, 2], [0, 1, 0], np.array([2, 1, 2]) / 3.0) == pytest.approx(3.0)

    def test_fold_boundaries(self, golden):
        z = golden("scalars")
        for i in range(len(z["fb_n"])):
            got = oracle.fold_boundaries(z["d2i_w"][i], z["enc_in"][i],
                                         z["fb_t0"][i], z["fb_t1"][i])
            assert len(got) == z["fb_n"][i]
            np.testing.assert_array_equal(got, z["fb_out"][i, :len(got)])

    @pytest.mark.parametrize("brute", [False, True])
    def test_trace_probe_range(self, golden, brute):
        z = golden("scalars")
        key = "pr_out_brute" if brute else "pr_out"
        got = np.array([oracle.trace_probe_range(
            z["pr_dist_hi"], z["pr_dir_hi"], z["pr_dist_lo"], w, d, 1e-4, 6.0,
            1e-3, brute=brute) for w, d in zip(z["pr_w"], z["pr_d"])])
        np.testing.assert_array_equal(got, z[key])
        assert (got[:, 0] == 1).sum() > 100   # the case exercises hits


class TestCameraRays:
    @pytest.mark.parametrize("name", ["c1", "pcgrid"])
    def test_camera_dirs_bit_exact(self, golden, name):
        z = golden(name)
        cam = golden_camera(z)
        basis, tan_v, tan_h = oracle.camera_params(cam)
        np.testing.assert_array_equal(basis, z["cam_basis"])
        got = oracle.camera_dirs(basis, tan_v, tan_h, cam.width, cam.height)
        np.testing.assert_array_equal(got, z["cam_dirs"])
        # and this package's host Camera reproduces the reference directions
        np.testing.assert_array_equal(cam.ray_directions(), z["cam_dirs"])


class TestGridTrace:
    @pytest.mark.parametrize("name,prefix", [("c1", "cam_"), ("c1", "inc_"),
                                             ("pcgrid", "cam_"),
                                             ("pcgrid", "inc_"),
                                             ("pcgrid", "al_")])
    def test_trace_rays(self, golden, name, prefix):
        z = golden(name)
        ps = GoldenProbeSet(z)
        dims = tuple(int(v) for v in z["dims"])
        if prefix == "inc_":
            o, d = z["inc_origins"], z["inc_dirs"]
        else:
            o, d = z[prefix + "eye"], z[prefix + "dirs"]
        res = oracle.trace_rays(ps, z["grid_origin"], float(z["cell"]), dims,
                                o, d)
        _check_outputs(res, z, prefix)

    @pytest.mark.parametrize("name,prefix", [("c1", "cam_"), ("pcgrid", "cam_"),
                                             ("pcgrid", "al_")])
    def test_render_frame(self, golden, name, prefix):
        z = golden(name)
        ps = GoldenProbeSet(z)
        dims = tuple(int(v) for v in z["dims"])
        cam = golden_camera(z, prefix)
        res, _ = oracle.render_camera(ps, z["grid_origin"], float(z["cell"]),
                                      dims, cam)
        pix, st = oracle.frame_pixels(res, cam.height, cam.width)
        np.testing.assert_array_equal(pix, z[prefix + "frame_pixels"])
        np.testing.assert_array_equal(st, z[prefix + "frame_status"])
        assert res.fetch.mean() == z[prefix + "frame_fetch_mean"]

    def test_render_grid_signature(self, golden):
        """oracle.render_grid keeps kernels.render_grid's in-place contract
        (K:825-843): rgb rows written on HIT only."""
        z = golden("c1")
        ps = GoldenProbeSet(z)
        n = len(z["cam_dirs"])
        st = np.zeros(n, np.uint8)
        rgb = np.full((n, 3), -7.0)
        fe = np.zeros(n, np.int64)
        oracle.render_grid(ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo,
                           ps.origins, z["grid_origin"], float(z["cell"]),
                           *(int(v) for v in z["dims"]), z["cam_eye"],
                           z["cam_dirs"], 1e-4, 1e-4, 1e-3, st, rgb, fe)
        np.testing.assert_array_equal(st, z["cam_status"])
        np.testing.assert_array_equal(fe, z["cam_fetch"])
        hit = st == 1
        np.testing.assert_array_equal(rgb[hit], z["cam_rgb"][hit])
        assert np.all(rgb[~hit] == -7.0)


@pytest.mark.slow
def test_c2_full_frame(golden):
    """C2 inputs regenerate bit-identically (sha256) and the oracle matches
    the reference on all 262,144 rays."""
    from paper_2507_14624_b200 import configs
    z = golden("c2")
    cfg = configs.c2()
    ps = cfg.grid.probe_set
    assert configs.probe_set_digest(ps) == str(z["digest"])
    cam = cfg.cameras[0]
    res, _ = oracle.render_camera(ps, cfg.grid.grid_origin, cfg.grid.cell_size,
                                  cfg.grid.dims, cam)
    _check_outputs(res, z, "cam_")
    pix, st = oracle.frame_pixels(res, cam.height, cam.width)
    np.testing.assert_array_equal(pix, z["cam_frame_pixels"])


class TestNonGridModes:
    """render_frame's single-probe / probe-list / eye-aligned sources
    (render.py:118-144) restated by the oracle vs the reference's frames."""

    def _probe(self, z, i):
        return {k: z[f"p{i}_{k}"] for k in ("dist_hi", "dir_hi", "irr_hi",
                                           "dist_lo", "origin", "blo", "bhi")}

    def _fill(self, st, rgb):
        px = rgb.astype(np.float32)
        px[st == 0] = 0.0
        px[st == 2] = np.array([1.0, 0.0, 1.0], np.float32)
        return px

    def test_single_probe(self, golden):
        z = golden("modes")
        p = self._probe(z, 0)
        cam = golden_camera(z, "single_")
        st, rgb, fe = oracle.render_single_probe(
            p["dist_hi"], p["dir_hi"], p["irr_hi"], p["dist_lo"], p["origin"],
            np.asarray(cam.eye, np.float64), z["single_dirs"], p["blo"] - 0.5,
            p["bhi"] + 0.5, 1e-4, 1e-3)
        np.testing.assert_array_equal(st.reshape(cam.height, cam.width),
                                      z["single_frame_status"])
        np.testing.assert_array_equal(
            self._fill(st, rgb).reshape(cam.height, cam.width, 3),
            z["single_frame_pixels"])
        assert fe.mean() == z["single_frame_fetch_mean"]
        assert (st == 2).mean() == z["single_frame_unknown"] > 0.1

    def test_probe_list(self, golden):
        from types import SimpleNamespace
        z = golden("modes")
        ps = [self._probe(z, i) for i in range(3)]
        cam = golden_camera(z, "few_")
        eye = np.asarray(cam.eye, np.float64)
        stack = SimpleNamespace(
            dist_hi=np.stack([p["dist_hi"] for p in ps]),
            dir_hi=np.stack([p["dir_hi"] for p in ps]),
            irr_hi=np.stack([p["irr_hi"] for p in ps]),
            dist_lo=np.stack([p["dist_lo"] for p in ps]),
            origins=np.stack([p["origin"] for p in ps]))
        blo = np.min([p["blo"] for p in ps], axis=0) - 0.5
        bhi = np.max([p["bhi"] for p in ps], axis=0) + 0.5
        st, rgb, fe = oracle.render_few_probes(stack, blo, bhi, eye,
                                               z["few_dirs"], 1e-4, 1e-4, 1e-3)
        np.testing.assert_array_equal(st.reshape(cam.height, cam.width),
                                      z["few_frame_status"])
        np.testing.assert_array_equal(
            self._fill(st, rgb).reshape(cam.height, cam.width, 3),
            z["few_frame_pixels"])
        assert fe.mean() == z["few_frame_fetch_mean"]
        assert (st == 2).any()
