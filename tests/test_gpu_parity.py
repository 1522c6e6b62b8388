"""CUDA path vs the reference (golden fixtures) and vs the C oracle.

Bars (BASELINE.json north_star): integer outputs identical on >= 99.99% of
rays -- this implementation reproduces the reference's fp64 decisions
exactly, so the tests require 100% (status, probe, texel, fetch); radiance
<= 1e-3 absolute (here: identical); hit distance <= 1e-4 relative; PSNR >=
60 dB (here: +inf).
"""

import numpy as np
import pytest

from conftest import GoldenProbeSet, golden_camera, golden_grid

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    import __graft_entry__
    __graft_entry__.build()


def _dev():
    from paper_2507_14624_b200 import device
    return device


def _trace(grid, origins, dirs, f32=False, config=None):
    dev = _dev()
    from paper_2507_14624_b200.render import device_probe_set
    from paper_2507_14624_b200.trace import DEFAULT_CONFIG
    dps = device_probe_set(grid)
    g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                        config or DEFAULT_CONFIG)
    dt = torch.float32 if f32 else torch.float64
    d = torch.as_tensor(np.ascontiguousarray(dirs), dtype=dt).cuda()
    o = np.asarray(origins)
    n = len(d)
    out = dev.RayOutputs(n, dps.device, probe=True, texel=True, fetch=True,
                         hit_t=True)
    if o.ndim == 1:
        o = np.broadcast_to(o, (n, 3))
    ot = torch.as_tensor(np.ascontiguousarray(o), dtype=dt).cuda()
    dev.trace_rays(dps, g, ot, d, out, rgb_mode=1)
    torch.cuda.synchronize()
    tex = out.texel.cpu().numpy()
    return dict(status=out.status.cpu().numpy(),
                probe=out.probe.cpu().numpy(),
                tx=np.where(tex < 0, -1, tex & 0xFFFF),
                ty=np.where(tex < 0, -1, tex >> 16),
                fetch=out.fetch.cpu().numpy(),
                rgb=out.rgb.cpu().numpy(),
                hit_t=out.hit_t.cpu().numpy(),
                stats=out.stats.cpu().numpy())


def _assert_same(got, exp, prefix="", rgb=True):
    for k in ("status", "probe", "tx", "ty", "fetch"):
        a = got[k]
        b = exp[prefix + k] if isinstance(exp, dict) else getattr(exp, k)
        bad = int((np.asarray(a) != np.asarray(b)).sum())
        assert bad == 0, f"{k}: {bad} of {len(a)} rays differ"
    if rgb:
        st = got["status"]
        b = exp[prefix + "rgb"] if isinstance(exp, dict) else exp.rgb
        hit = st == 1
        np.testing.assert_array_equal(got["rgb"][hit].astype(np.float64),
                                      np.asarray(b)[hit])


class TestGolden:
    """CUDA vs outputs of the reference itself (tests/golden)."""

    @pytest.mark.parametrize("name,prefix", [("c1", "cam_"), ("c1", "inc_"),
                                             ("pcgrid", "cam_"),
                                             ("pcgrid", "inc_"),
                                             ("pcgrid", "al_")])
    def test_trace_rays_vs_reference(self, golden, name, prefix):
        z = golden(name)
        grid = golden_grid(z)
        if prefix == "inc_":
            o, d = z["inc_origins"], z["inc_dirs"]
        else:
            o, d = z[prefix + "eye"], z[prefix + "dirs"]
        _assert_same(_trace(grid, o, d), z, prefix)

    @pytest.mark.parametrize("name,prefix", [("c1", "cam_"), ("pcgrid", "cam_"),
                                             ("pcgrid", "al_")])
    def test_render_frame_vs_reference(self, golden, name, prefix):
        from paper_2507_14624_b200 import psnr, render_frame
        z = golden(name)
        grid = golden_grid(z)
        cam = golden_camera(z, prefix)
        fr = render_frame(grid, cam)
        np.testing.assert_array_equal(fr.status, z[prefix + "frame_status"])
        np.testing.assert_array_equal(fr.pixels, z[prefix + "frame_pixels"])
        assert fr.stats["perPixelTexelFetches"] == pytest.approx(
            float(z[prefix + "frame_fetch_mean"]), abs=1e-12)
        assert fr.stats["missFraction"] == pytest.approx(
            float(z[prefix + "frame_miss"]), abs=1e-12)
        assert fr.stats["unknownFraction"] == 0.0   # grid mode: K:822
        assert fr.pixels.dtype == np.float32 and fr.status.dtype == np.uint8
        ref = z[prefix + "frame_pixels"]
        assert psnr(fr, np.clip(np.rint(ref * 255.0), 0, 255).astype(
            np.uint8)) == float("inf")

    def test_c2_full_frame_vs_reference(self, golden):
        from paper_2507_14624_b200 import configs, render_frame
        z = golden("c2")
        cfg = configs.c2()
        assert configs.probe_set_digest(cfg.grid.probe_set) == str(z["digest"])
        cam = cfg.cameras[0]
        fr = render_frame(cfg.grid, cam)
        np.testing.assert_array_equal(fr.status, z["cam_frame_status"])
        np.testing.assert_array_equal(fr.pixels, z["cam_frame_pixels"])
        dirs = cam.ray_directions()
        got = _trace(cfg.grid, np.asarray(cam.eye), dirs)
        _assert_same(got, z, "cam_", rgb=False)


class TestOracleParity:
    """CUDA vs the C oracle on freshly generated inputs."""

    def test_c3_subsample(self):
        from oracle import oracle
        from paper_2507_14624_b200 import configs
        cfg = configs.c3(n_views=4)
        rng = np.random.default_rng(7)
        for cam in cfg.cameras:
            basis, tv, th = oracle.camera_params(cam)
            dirs = oracle.camera_dirs(basis, tv, th, cam.width, cam.height)
            idx = np.sort(rng.choice(len(dirs), len(dirs) // 16, replace=False))
            d = dirs[idx]
            exp = oracle.trace_rays(cfg.grid.probe_set, cfg.grid.grid_origin,
                                    cfg.grid.cell_size, cfg.grid.dims,
                                    np.asarray(cam.eye, np.float64), d)
            got = _trace(cfg.grid, np.asarray(cam.eye), d)
            _assert_same(got, exp)

    def test_c3_camera_kernel_matches_ray_kernel(self):
        """In-kernel ray generation == host (oracle) directions, full pose."""
        from oracle import oracle
        from paper_2507_14624_b200 import configs
        from paper_2507_14624_b200 import device as dev
        from paper_2507_14624_b200.render import device_probe_set
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG
        cfg = configs.c3(n_views=2)
        dps = device_probe_set(cfg.grid)
        g = dev.grid_params(cfg.grid.grid_origin, cfg.grid.cell_size,
                            cfg.grid.dims, DEFAULT_CONFIG)
        cam = cfg.cameras[1]
        n = cam.width * cam.height
        out = dev.RayOutputs(n, dps.device, probe=True, texel=True, fetch=True)
        dev.render_cameras(dps, g, [cam], cam.width, cam.height, out)
        basis, tv, th = oracle.camera_params(cam)
        dirs = oracle.camera_dirs(basis, tv, th, cam.width, cam.height)
        got = _trace(cfg.grid, np.asarray(cam.eye), dirs)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.status.cpu().numpy(), got["status"])
        np.testing.assert_array_equal(out.fetch.cpu().numpy(), got["fetch"])
        tex = out.texel.cpu().numpy()
        np.testing.assert_array_equal(np.where(tex < 0, -1, tex & 0xFFFF),
                                      got["tx"])

    def test_c5_incoherent_f32_rays(self):
        from oracle import oracle
        from paper_2507_14624_b200 import configs
        scene, grid = configs.c3_grid()
        o32, d32 = configs.c5_rays(scene, 1 << 16, seed=505)
        exp = oracle.trace_rays(grid.probe_set, grid.grid_origin,
                                grid.cell_size, grid.dims,
                                o32.astype(np.float64), d32.astype(np.float64))
        got = _trace(grid, o32, d32, f32=True)
        _assert_same(got, exp)

    def test_hit_distance(self, golden):
        """hit_t = (origin_p + dist_hi[p,ty,tx] v_texel - eye) . d matches
        the oracle-derived value to 1e-4 relative."""
        from oracle import oracle
        z = golden("c1")
        grid = golden_grid(z)
        o, d = z["inc_origins"], z["inc_dirs"]
        got = _trace(grid, o, d)
        hit = got["status"] == 1
        assert hit.sum() > 1000
        R = grid.probe_set.dist_hi.shape[1]
        exp = np.full(len(d), np.inf)
        for i in np.flatnonzero(hit):
            p, tx, ty = z["inc_probe"][i], z["inc_tx"][i], z["inc_ty"][i]
            v = oracle.oct_decode(((tx + 0.5) / R, (ty + 0.5) / R))
            pt = grid.probe_set.origins[p] + float(
                grid.probe_set.dist_hi[p, ty, tx]) * v
            exp[i] = np.dot(pt - o[i], d[i])
        np.testing.assert_allclose(got["hit_t"][hit], exp[hit], rtol=1e-4,
                                   atol=1e-6)
        assert np.all(np.isinf(got["hit_t"][~hit]))


class TestBoundaryAndEdges:
    def test_render_grid_dropin_signature(self, golden):
        """kernels.render_grid keeps K:825-843's in-place contract."""
        from paper_2507_14624_b200 import kernels
        z = golden("pcgrid")
        ps = GoldenProbeSet(z)
        n = len(z["cam_dirs"])
        st = np.zeros(n, np.uint8)
        rgb = np.full((n, 3), -7.0)
        fe = np.zeros(n, np.int64)
        kernels.render_grid(ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo,
                            ps.origins, z["grid_origin"], float(z["cell"]),
                            *(int(v) for v in z["dims"]), z["cam_eye"],
                            z["cam_dirs"], 1e-4, 1e-4, 1e-3, st, rgb, fe)
        np.testing.assert_array_equal(st, z["cam_status"])
        np.testing.assert_array_equal(fe, z["cam_fetch"])
        hit = st == 1
        np.testing.assert_array_equal(rgb[hit], z["cam_rgb"][hit])
        assert np.all(rgb[~hit] == -7.0)

    def test_trace_grid_ray_twin(self, golden):
        from paper_2507_14624_b200 import kernels
        z = golden("pcgrid")
        ps = GoldenProbeSet(z)
        for i in range(0, 4096, 257):
            rgb = np.zeros(3)
            o, d = z["inc_origins"][i], z["inc_dirs"][i]
            out = kernels.trace_grid_ray(
                ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo, ps.origins,
                z["grid_origin"], float(z["cell"]),
                *(int(v) for v in z["dims"]), *o, *d, 1e-4, 1e-4, 1e-3, rgb)
            assert out == (z["inc_status"][i], z["inc_probe"][i],
                           z["inc_tx"][i], z["inc_ty"][i], z["inc_fetch"][i])
            if out[0] == 1:
                np.testing.assert_array_equal(rgb, z["inc_rgb"][i])

    def test_edge_rays(self, golden):
        """Axis-aligned directions (d_a == 0 branches), rays missing the
        lattice, eye on the lattice boundary and on a probe, vs the oracle."""
        from oracle import oracle
        z = golden("pcgrid")
        grid = golden_grid(z)
        o = []
        d = []
        axes = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0],
                         [0, 0, 1], [0, 0, -1]], np.float64)
        diag = np.array([[1, 1, 0], [0, 1, -1], [1, 0, 1], [-1, -1, -1]],
                        np.float64)
        diag /= np.linalg.norm(diag, axis=1, keepdims=True)
        eyes = [(1.3, 1.1, 1.7), (0.5, 0.25, 0.5), (2.5, 2.25, 2.5),
                (0.5, 1.0, 1.0), (10.0, 10.0, 10.0), (1.5, 1.25, 1.5),
                (2.5, 0.25, 0.5)]
        for e in eyes:
            for v in np.concatenate([axes, diag]):
                o.append(e)
                d.append(v)
        o = np.array(o)
        d = np.array(d)
        exp = oracle.trace_rays(grid.probe_set, grid.grid_origin,
                                grid.cell_size, grid.dims, o, d)
        got = _trace(grid, o, d)
        _assert_same(got, exp)
        # rays that never meet the lattice AABB cost nothing (K:668-691)
        far = np.all(o == 10.0, axis=1) & np.any(d > 0.0, axis=1)
        assert (got["fetch"][far] == 0).all() and (got["status"][far] == 0).all()

    def test_odd_frame_sizes_and_determinism(self, golden):
        from oracle import oracle
        from paper_2507_14624_b200 import Camera, render_frame
        z = golden("pcgrid")
        grid = golden_grid(z)
        for w, h in ((33, 17), (1, 1), (8, 16), (130, 3)):
            cam = Camera(eye=(1.3, 1.1, 1.7), forward=(0.4, -0.2, -1.0),
                         width=w, height=h)
            a = render_frame(grid, cam)
            b = render_frame(grid, cam)
            np.testing.assert_array_equal(a.pixels, b.pixels)
            np.testing.assert_array_equal(a.status, b.status)
            res, _ = oracle.render_camera(grid.probe_set, grid.grid_origin,
                                          grid.cell_size, grid.dims, cam)
            pix, st = oracle.frame_pixels(res, h, w)
            np.testing.assert_array_equal(a.pixels, pix)
            np.testing.assert_array_equal(a.status, st)

    def test_compact_shards_untile(self, golden):
        """Interleaved tile shards (the multi-GPU layout) reassemble into
        the single-launch frame."""
        from paper_2507_14624_b200 import configs
        from paper_2507_14624_b200 import device as dev
        from paper_2507_14624_b200.render import device_probe_set
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG
        cfg = configs.c1()
        cams = cfg.cameras + configs.random_cameras(cfg.scene, 2, 128, 128, 9)
        W, H = 100, 77
        cams = [type(c)(eye=c.eye, forward=c.forward, width=W, height=H)
                for c in cams]
        dps = device_probe_set(cfg.grid)
        g = dev.grid_params(cfg.grid.grid_origin, cfg.grid.cell_size,
                            cfg.grid.dims, DEFAULT_CONFIG)
        full = dev.RayOutputs(len(cams) * W * H, dps.device)
        dev.render_cameras(dps, g, cams, W, H, full)
        T = dev.num_tiles(len(cams), W, H)
        for n_ranks in (1, 2, 3, 8):
            parts_s, parts_c = [], []
            tot = 0
            for k in range(n_ranks):
                nk = (T - k + n_ranks - 1) // n_ranks
                o = dev.RayOutputs(max(nk, 1) * 128, dps.device)
                dev.render_cameras(dps, g, cams, W, H, o, tile_begin=k,
                                   tile_step=n_ranks, n_tiles=nk, compact=True)
                parts_s.append(o.status[:nk * 128])
                parts_c.append(o.rgb[:nk * 128])
                tot += int(o.stats[3])
            cat_s = torch.cat(parts_s)
            cat_c = torch.cat(parts_c)
            st = torch.empty(len(cams) * W * H, dtype=torch.uint8, device="cuda")
            rgb = torch.empty((len(cams) * W * H, 3), dtype=torch.float32,
                              device="cuda")
            dev.untile(len(cams), W, H, n_ranks, cat_s, cat_c, st, rgb)
            torch.cuda.synchronize()
            assert torch.equal(st, full.status)
            assert torch.equal(rgb, full.rgb)
            assert tot == int(full.stats[3])

    def test_degenerate_and_empty(self, golden):
        from paper_2507_14624_b200 import ProbeGrid, ProbeSet
        z = golden("pcgrid")
        grid = golden_grid(z)
        got = _trace(grid, np.zeros((0, 3)), np.zeros((0, 3)))
        assert len(got["status"]) == 0
        ps = grid.probe_set
        sel = [0, 4]   # probes (0,0,0) and (1,0,0): a (2, 1, 1) lattice
        sub = ProbeSet(arrays=(ps.dist_hi[sel], ps.dir_hi[sel], ps.irr_hi[sel],
                               ps.dist_lo[sel], ps.origins[sel]))
        flat = ProbeGrid((0.5, 0.25, 0.5), 2.0, (2, 1, 1), probe_set=sub)
        r = _trace(flat, np.array([1.0, 0.25, 0.5]),
                   np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]))
        assert (r["status"] == 0).all() and (r["fetch"] == 0).all()


class TestGpuBake:
    def test_gpu_bake_matches_host_bake(self):
        """lfp_bake_probes reproduces the numpy ray-cast bake (bake.py) up
        to last-ulp direction rounding: same EMPTY texels, distances to
        1e-6 relative, radiance to 1e-4, on the C1 scene."""
        from paper_2507_14624_b200 import configs
        from paper_2507_14624_b200.bake import bake_grid_gpu
        cfg = configs.c1()
        g = cfg.grid
        gg = bake_grid_gpu(cfg.scene, g.grid_origin, g.cell_size, g.dims, 32, 8)
        a, b = g.probe_set, gg.probe_set
        fa, fb = np.isfinite(a.dist_hi), np.isfinite(b.dist_hi)
        assert (fa != fb).mean() < 1e-3
        both = fa & fb
        rel = np.abs(a.dist_hi[both] - b.dist_hi[both]) / a.dist_hi[both]
        assert np.quantile(rel, 0.999) < 1e-6
        close = np.abs(a.irr_hi - b.irr_hi).max(axis=-1)[both] < 1e-4
        assert close.mean() > 0.999
        np.testing.assert_array_equal(
            np.isfinite(b.dist_lo),
            np.isfinite(b.dist_hi.reshape(8, 8, 4, 8, 4)).any(axis=(2, 4)))


class TestDecisionFilters:
    """The fp32 decision filters never change a decision: every filtered
    decision is re-checked against the exact fp64 path (trace_mode
    'check') and the filtered, exact and check modes produce identical
    outputs."""

    def _run(self, grid, o, d, mode):
        dev = _dev()
        from paper_2507_14624_b200.render import device_probe_set
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG
        dps = device_probe_set(grid)
        g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                            DEFAULT_CONFIG, mode=mode)
        dt = torch.float32 if d.dtype == np.float32 else torch.float64
        n = len(d)
        o = np.broadcast_to(np.asarray(o), (n, 3))
        out = dev.RayOutputs(n, dps.device, probe=True, texel=True, fetch=True,
                             diag=True)
        dev.trace_rays(dps, g, torch.as_tensor(np.ascontiguousarray(o), dtype=dt).cuda(),
                       torch.as_tensor(np.ascontiguousarray(d), dtype=dt).cuda(),
                       out, rgb_mode=1)
        torch.cuda.synchronize()
        return {k: getattr(out, k).cpu().numpy() for k in
                ("status", "probe", "texel", "fetch", "diag")}

    def _check(self, grid, o, d):
        a = self._run(grid, o, d, "exact")
        b = self._run(grid, o, d, "filtered")
        c = self._run(grid, o, d, "check")
        for k in ("status", "probe", "texel", "fetch"):
            np.testing.assert_array_equal(a[k], b[k])
            np.testing.assert_array_equal(a[k], c[k])
        lo_fast, lo_slow, hi_fast, hi_slow, mism = (int(v) for v in c["diag"][:5])
        assert mism == 0, f"{mism} filtered decisions disagree with exact fp64"
        assert lo_fast + lo_slow > 0 and hi_fast + hi_slow > 0
        # the filter must decide the bulk of the steps
        assert lo_fast / (lo_fast + lo_slow) > 0.9
        assert hi_fast / (hi_fast + hi_slow) > 0.8
        return c["diag"]

    def test_c2_frame(self):
        from paper_2507_14624_b200 import configs
        cfg = configs.c2()
        cam = cfg.cameras[0]
        self._check(cfg.grid, np.asarray(cam.eye), cam.ray_directions())

    def test_pcgrid_incoherent(self, golden):
        z = golden("pcgrid")
        self._check(golden_grid(z), z["inc_origins"], z["inc_dirs"])

    def test_c5_incoherent(self):
        from paper_2507_14624_b200 import configs
        scene, grid = configs.c3_grid()
        o32, d32 = configs.c5_rays(scene, 1 << 18, seed=515)
        self._check(grid, o32, d32)


class TestNonGridSources:
    """render_frame on a ProbeData (single-probe marching K:567-596 and the
    eye-aligned lookup R:86-99) and on a probe list (K:846-892) vs the
    reference's own frames (tests/golden/modes.npz)."""

    def _probe(self, z, i):
        from paper_2507_14624_b200 import MapChain, ProbeData
        ch = MapChain(irradiance_hi=z[f"p{i}_irr_hi"],
                      distance_hi=z[f"p{i}_dist_hi"],
                      direction_hi=z[f"p{i}_dir_hi"],
                      distance_lo=z[f"p{i}_dist_lo"])
        return ProbeData(origin=z[f"p{i}_origin"], chain=ch,
                         bounds_lo=z[f"p{i}_blo"], bounds_hi=z[f"p{i}_bhi"])

    @pytest.mark.parametrize("name", ["single", "few", "lookup"])
    def test_vs_reference(self, golden, name):
        from paper_2507_14624_b200 import render_frame
        z = golden("modes")
        probes = [self._probe(z, i) for i in range(3)]
        src = {"single": probes[0], "few": probes, "lookup": probes[1]}[name]
        cam = golden_camera(z, name + "_")
        fr = render_frame(src, cam)
        np.testing.assert_array_equal(fr.status, z[name + "_frame_status"])
        np.testing.assert_array_equal(fr.pixels, z[name + "_frame_pixels"])
        assert fr.stats["perPixelTexelFetches"] == pytest.approx(
            float(z[name + "_frame_fetch_mean"]), abs=1e-12)
        assert fr.stats["unknownFraction"] == pytest.approx(
            float(z[name + "_frame_unknown"]), abs=1e-12)
        if name == "lookup":
            assert fr.stats["perPixelTexelFetches"] == 1.0
        else:
            assert fr.stats["unknownFraction"] > 0.1   # UNKNOWN -> magenta


class TestLfpLoad:
    """.lfp files written by the reference, decoded on the GPU
    (lfp_probeset_create_packed) == the reference loader's arrays; the
    loaded grid renders the reference frame."""

    def test_load_grid_matches_reference_loader(self, golden):
        import os
        from conftest import GOLDEN
        from paper_2507_14624_b200 import lfpio, render_frame
        z = golden("lfp")
        grid = lfpio.load_grid(os.path.join(GOLDEN, "lfp_grid", "grid.json"))
        ps = grid.probe_set
        for k in ("dist_hi", "dir_hi", "irr_hi", "dist_lo", "origins"):
            np.testing.assert_array_equal(getattr(ps, k), z[k], err_msg=k)
        assert grid.dims == tuple(int(v) for v in z["dims"])
        fr = render_frame(grid, golden_camera(z))
        np.testing.assert_array_equal(fr.status, z["cam_frame_status"])
        np.testing.assert_array_equal(fr.pixels, z["cam_frame_pixels"])

    def test_load_probe_and_format_errors(self, golden, tmp_path):
        import os
        from conftest import GOLDEN
        from paper_2507_14624_b200 import lfpio
        z = golden("lfp")
        src = os.path.join(GOLDEN, "lfp_grid", "probe_1_0_1.lfp")
        p = lfpio.load_probe(src)
        idx = (1 * 2 + 0) * 2 + 1
        np.testing.assert_array_equal(p.chain.distance_hi, z["dist_hi"][idx])
        np.testing.assert_array_equal(p.chain.direction_hi, z["dir_hi"][idx])
        np.testing.assert_array_equal(p.chain.irradiance_hi, z["irr_hi"][idx])
        data = open(src, "rb").read()
        bad = tmp_path / "bad.lfp"
        bad.write_bytes(b"NOTPROBE" + data[8:])
        with pytest.raises(lfpio.ProbeFormatError, match="bad magic"):
            lfpio.load_probe(str(bad))
        bad.write_bytes(data[:-3])
        with pytest.raises(lfpio.ProbeFormatError, match="expected"):
            lfpio.load_probe(str(bad))


class TestHierarchy:
    """Config-4 coarse-to-fine hierarchy (lfp_render_hierarchy) vs the
    oracle's per-level composition, on the C4 block scene with the three
    C4 lattices at reduced map resolution (32^2 / 8^2)."""

    def test_hierarchy_vs_oracle(self):
        from oracle import oracle
        from paper_2507_14624_b200 import configs
        from paper_2507_14624_b200 import device as dev
        from paper_2507_14624_b200.render import device_probe_set
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG
        scene, grids = configs.c4_levels(r_hi=32, r_lo=8)
        cam = configs.street_cameras(scene, 1, 240, 136, 4404)[0]
        levels = [(device_probe_set(g), dev.grid_params(
            g.grid_origin, g.cell_size, g.dims, DEFAULT_CONFIG)) for g in grids]
        n = cam.width * cam.height
        out = dev.RayOutputs(n, levels[0][0].device, probe=True, texel=True,
                             fetch=True)
        dev.render_hierarchy(levels, [cam], cam.width, cam.height, out)
        torch.cuda.synchronize()
        basis, tv, th = oracle.camera_params(cam)
        dirs = oracle.camera_dirs(basis, tv, th, cam.width, cam.height)
        exp = oracle.trace_hierarchy(grids, np.asarray(cam.eye, np.float64), dirs)
        tex = out.texel.cpu().numpy()
        got = dict(status=out.status.cpu().numpy(), probe=out.probe.cpu().numpy(),
                   tx=np.where(tex < 0, -1, tex & 0xFFFF),
                   ty=np.where(tex < 0, -1, tex >> 16),
                   fetch=out.fetch.cpu().numpy())
        for k in ("status", "probe", "tx", "ty", "fetch"):
            np.testing.assert_array_equal(got[k], getattr(exp, k), err_msg=k)
        hit = got["status"] == 1
        np.testing.assert_array_equal(out.rgb.cpu().numpy()[hit],
                                      exp.rgb[hit].astype(np.float32))
        lv = got["probe"][hit] >> 24
        assert hit.mean() > 0.3 and len(np.unique(lv)) >= 2   # >1 level used


class TestPersistentSchedule:
    """The persistent flattened traversal (schedule 'persistent') produces
    exactly the nested traversal's outputs (and hence the reference's)."""

    def _run(self, grid, o, d, schedule, mode="filtered", min_active=0,
             ordered=False):
        dev = _dev()
        from paper_2507_14624_b200.render import device_probe_set
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG
        dps = device_probe_set(grid)
        g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                            DEFAULT_CONFIG, mode=mode, schedule=schedule,
                            min_active=min_active)
        dt = torch.float32 if d.dtype == np.float32 else torch.float64
        n = len(d)
        o = np.broadcast_to(np.asarray(o), (n, 3))
        to = torch.as_tensor(np.ascontiguousarray(o), dtype=dt).cuda()
        td = torch.as_tensor(np.ascontiguousarray(d), dtype=dt).cuda()
        out = dev.RayOutputs(n, dps.device, probe=True, texel=True, fetch=True,
                             hit_t=True, diag=True)
        out.rgb.zero_()
        if ordered:
            order = dev.ray_order(dev.bin_rays(g, to, td))
            dev.trace_rays_ordered(dps, g, to, td, order, out)
        else:
            dev.trace_rays(dps, g, to, td, out)
        torch.cuda.synchronize()
        return {k: getattr(out, k).cpu().numpy() for k in
                ("status", "probe", "texel", "fetch", "rgb", "hit_t", "stats",
                 "diag")}

    def _same(self, a, b):
        for k in ("status", "probe", "texel", "fetch", "rgb", "hit_t", "stats"):
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)

    @pytest.mark.parametrize("min_active", [1, 16, 32])
    def test_pcgrid_incoherent(self, golden, min_active):
        z = golden("pcgrid")
        grid = golden_grid(z)
        a = self._run(grid, z["inc_origins"], z["inc_dirs"], "nested")
        b = self._run(grid, z["inc_origins"], z["inc_dirs"], "persistent",
                      min_active=min_active)
        self._same(a, b)
        np.testing.assert_array_equal(b["status"], z["inc_status"])
        np.testing.assert_array_equal(b["fetch"], z["inc_fetch"])

    def test_c5_binned_and_check(self):
        from paper_2507_14624_b200 import configs
        scene, grid = configs.c3_grid()
        o32, d32 = configs.c5_rays(scene, 1 << 17, seed=525)
        a = self._run(grid, o32, d32, "nested")
        b = self._run(grid, o32, d32, "persistent", ordered=True)
        c = self._run(grid, o32, d32, "persistent", mode="check")
        self._same(a, b)
        self._same(a, c)
        assert int(c["diag"][4]) == 0

    def test_pcgrid_incoherent_wave(self, golden):
        """Wavefront schedule: golden reference outputs, shared-eye
        render_grid path included."""
        z = golden("pcgrid")
        grid = golden_grid(z)
        a = self._run(grid, z["inc_origins"], z["inc_dirs"], "nested")
        b = self._run(grid, z["inc_origins"], z["inc_dirs"], "wave")
        c = self._run(grid, z["inc_origins"], z["inc_dirs"], "wave",
                      ordered=True)
        self._same(a, b)
        self._same(a, c)
        np.testing.assert_array_equal(b["status"], z["inc_status"])
        np.testing.assert_array_equal(b["fetch"], z["inc_fetch"])

    def test_c5_wave_and_check(self):
        from paper_2507_14624_b200 import configs
        scene, grid = configs.c3_grid()
        o32, d32 = configs.c5_rays(scene, 1 << 17, seed=526)
        a = self._run(grid, o32, d32, "nested")
        b = self._run(grid, o32, d32, "wave", ordered=True)
        c = self._run(grid, o32, d32, "wave", mode="check")
        e = self._run(grid, o32, d32, "wave", mode="exact")
        self._same(a, b)
        self._same(a, c)
        self._same(a, e)
        assert int(c["diag"][4]) == 0

    def test_camera_persistent(self):
        from paper_2507_14624_b200 import configs
        from paper_2507_14624_b200 import device as dev
        from paper_2507_14624_b200.render import device_probe_set
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG
        cfg = configs.c2()
        cams = cfg.cameras + configs.random_cameras(cfg.scene, 1, 512, 512, 77)
        W, H = 500, 333
        cams = [type(c)(eye=c.eye, forward=c.forward, width=W, height=H)
                for c in cams]
        dps = device_probe_set(cfg.grid)
        res = []
        for sched in ("nested", "persistent"):
            g = dev.grid_params(cfg.grid.grid_origin, cfg.grid.cell_size,
                                cfg.grid.dims, DEFAULT_CONFIG, schedule=sched)
            out = dev.RayOutputs(len(cams) * W * H, dps.device, probe=True,
                                 texel=True, fetch=True)
            dev.render_cameras(dps, g, cams, W, H, out)
            torch.cuda.synchronize()
            res.append({k: getattr(out, k).cpu().numpy() for k in
                        ("status", "rgb", "probe", "texel", "fetch", "stats")})
            # compact shards too
            T = dev.num_tiles(len(cams), W, H)
            o2 = dev.RayOutputs(((T + 2) // 3) * 128, dps.device, fetch=True)
            o2.status.fill_(255)
            dev.render_cameras(dps, g, cams, W, H, o2, tile_begin=1,
                               tile_step=3, compact=True)
            torch.cuda.synchronize()
            res[-1]["compact"] = o2.status.cpu().numpy()
        for k in res[0]:
            np.testing.assert_array_equal(res[0][k], res[1][k], err_msg=k)


@pytest.mark.gpu
@pytest.mark.parametrize("entry", ["lfp_selftest_division",
                                   "lfp_selftest_division_recip"])
def test_branch_free_division_is_ieee(entry):
    """The tracer's branch-free division (rcp_nv / div_nv, LFP_FAST_DIV)
    equals nvcc's IEEE `a / b` bit for bit whenever its fast-path test
    passes (and falls back to `a / b` otherwise): random operands over the
    magnitudes the tracer sees, wide exponents, signs, zeros, infinities,
    NaN, subnormals; the fast path must be the common case."""
    import ctypes
    from paper_2507_14624_b200 import native
    rng = np.random.default_rng(11)
    n = 1 << 21
    a = rng.normal(size=n) * 10.0 ** rng.uniform(-6, 6, n)
    b = rng.normal(size=n) * 10.0 ** rng.uniform(-6, 6, n)
    a[: n // 4] = rng.uniform(-4, 4, n // 4)
    b[: n // 4] = rng.uniform(0.01, 3, n // 4)
    ex = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 5e-324, 1e-310,
                   1e308, 1.7976931348623157e308, 2.2250738585072014e-308,
                   3.0, 7.0, 1e-200, 1e200])
    aa, bb = np.meshgrid(ex, ex)
    a = np.concatenate([a, aa.ravel(), 2.0 ** rng.integers(-1070, 1023, 4096)])
    b = np.concatenate([b, bb.ravel(), 2.0 ** rng.integers(-1070, 1023, 4096)
                        * rng.uniform(1, 2, 4096)])
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    ref = torch.empty_like(ta)
    fast = torch.empty_like(ta)
    took = torch.empty(len(a), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    native.check(getattr(native.lib(), entry)(
        ctypes.c_void_p(ta.data_ptr()), ctypes.c_void_p(tb.data_ptr()), len(a),
        ctypes.c_void_p(ref.data_ptr()), ctypes.c_void_p(fast.data_ptr()),
        ctypes.c_void_p(took.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
    torch.cuda.synchronize()
    r, f = ref.cpu().numpy(), fast.cpu().numpy()
    bad = r.view(np.uint64) != f.view(np.uint64)
    assert int((bad & ~(np.isnan(r) & np.isnan(f))).sum()) == 0
    with np.errstate(all="ignore"):
        np.testing.assert_array_equal(r, a / b)
    assert took[:n].float().mean().item() > 0.99
