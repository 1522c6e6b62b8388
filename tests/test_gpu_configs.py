"""CUDA vs the C oracle at the configurations as benchmarked (BASELINE.json
configs[2..4], SURVEY.md §8(d) parity plan), the reference's acceptance
setups at 2048^2 probes (pkg/tests/test_acceptance.py C6 / C8), and the
reference's property tests re-run on the CUDA backend.

Bars: integer outputs (status, probe, texel, fetch) identical on 100% of
the compared rays (north star: >= 99.99%), radiance identical (bar 1e-3),
hit distance <= 1e-4 relative, PSNR +inf (bar 60 dB).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    import __graft_entry__
    __graft_entry__.build()
    from oracle import oracle
    import os
    oracle.set_num_threads(os.cpu_count() or 1)


def _grid_params(grid, **kw):
    from paper_2507_14624_b200 import device as dev
    from paper_2507_14624_b200.trace import DEFAULT_CONFIG
    return dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                           DEFAULT_CONFIG, **kw)


def _host(out, idx=None):
    """Device RayOutputs -> dict of host arrays (optionally rows idx)."""
    def h(t):
        if t is None:
            return None
        if idx is not None:
            t = t[torch.as_tensor(idx, device=t.device)]
        return t.cpu().numpy()
    tex = h(out.texel)
    return dict(status=h(out.status), probe=h(out.probe),
                tx=np.where(tex < 0, -1, tex & 0xFFFF),
                ty=np.where(tex < 0, -1, tex >> 16), fetch=h(out.fetch),
                rgb=h(out.rgb), hit_t=h(out.hit_t))


def _assert_same(got, exp, what=""):
    n = len(got["status"])
    for k in ("status", "probe", "tx", "ty", "fetch"):
        bad = int((np.asarray(got[k]) != np.asarray(getattr(exp, k))).sum())
        assert bad == 0, f"{what} {k}: {bad} of {n} rays differ"
    hit = got["status"] == 1
    np.testing.assert_array_equal(got["rgb"][hit].astype(np.float64),
                                  exp.rgb[hit], err_msg=what)


def _oct_decode(u, v):
    """K:48-59 vectorised (numpy fp64, the reference's op order)."""
    fx = u * 2.0 - 1.0
    fz = v * 2.0 - 1.0
    y = 1.0 - np.abs(fx) - np.abs(fz)
    neg = y < 0.0
    sx = np.where(fx >= 0.0, 1.0, -1.0)
    sz = np.where(fz >= 0.0, 1.0, -1.0)
    ux = np.where(neg, sx * (1.0 - np.abs(fz)), fx)
    uz = np.where(neg, sz * (1.0 - np.abs(fx)), fz)
    inv = 1.0 / np.sqrt(ux * ux + y * y + uz * uz)
    return np.stack([ux * inv, y * inv, uz * inv], -1)


def _hit_t_expected(ps, eye, dirs, exp):
    """hit_t = (origin_p + dist_hi[p,ty,tx] v - eye) . d,
    v = oct_decode(texel centre), from the oracle's integer outputs."""
    hit = np.flatnonzero(exp.status == 1)
    R = ps.dist_hi.shape[1]
    e = np.broadcast_to(np.asarray(eye, np.float64), dirs.shape)[hit]
    p, tx, ty = exp.probe[hit], exp.tx[hit], exp.ty[hit]
    v = _oct_decode((tx + 0.5) / R, (ty + 0.5) / R)
    st = ps.dist_hi[p, ty, tx].astype(np.float64)[:, None]
    pt = ps.origins[p] + st * v
    return hit, np.einsum("ij,ij->i", pt - e, dirs[hit])


@pytest.fixture(scope="module")
def c3cfg():
    from paper_2507_14624_b200 import configs
    return configs.c3(n_views=64)


class TestC3AsBenchmarked:
    """C3: 8x4x8 probes at 256^2/64^2 (f16 payloads), 64 poses at 1080p --
    the bench's own config object; 4 full poses + a seeded 1/16 pixel
    subsample of all 64 poses vs the oracle."""

    def _render(self, cfg, cams):
        from paper_2507_14624_b200 import device as dev
        from paper_2507_14624_b200.render import device_probe_set
        dps = device_probe_set(cfg.grid)
        W, H = cams[0].width, cams[0].height
        out = dev.RayOutputs(len(cams) * W * H, dps.device, probe=True,
                             texel=True, fetch=True, hit_t=True)
        dev.render_cameras(dps, _grid_params(cfg.grid), cams, W, H, out)
        torch.cuda.synchronize()
        return out

    def test_four_full_poses(self, c3cfg):
        from oracle import oracle
        from paper_2507_14624_b200 import psnr
        cfg = c3cfg
        cams = cfg.cameras[:4]
        out = self._render(cfg, cams)
        n = cams[0].width * cams[0].height
        g = cfg.grid
        for c, cam in enumerate(cams):
            got = _host(out, np.arange(c * n, (c + 1) * n))
            exp, dirs = oracle.render_camera(g.probe_set, g.grid_origin,
                                             g.cell_size, g.dims, cam)
            _assert_same(got, exp, f"pose {c}")
            pix, st = oracle.frame_pixels(exp, cam.height, cam.width)
            mine = np.where((got["status"] == 1)[:, None], got["rgb"],
                            0.0).astype(np.float32).reshape(pix.shape)
            assert psnr(np.clip(np.rint(mine * 255), 0, 255).astype(np.uint8),
                        np.clip(np.rint(pix * 255), 0, 255).astype(np.uint8)
                        ) == float("inf")
            hit, ht = _hit_t_expected(g.probe_set, cam.eye, dirs, exp)
            np.testing.assert_allclose(got["hit_t"][hit], ht, rtol=1e-4,
                                       atol=1e-6)
            assert np.isinf(got["hit_t"][exp.status != 1]).all()
            assert (exp.status == 1).mean() > 0.5

    def test_subsample_of_all_64_poses(self, c3cfg):
        from oracle import oracle
        cfg = c3cfg
        cams = cfg.cameras
        assert len(cams) == 64
        out = self._render(cfg, cams)
        n = cams[0].width * cams[0].height
        rng = np.random.default_rng(316)
        g = cfg.grid
        for c, cam in enumerate(cams):
            idx = np.sort(rng.choice(n, n // 16, replace=False))
            got = _host(out, c * n + idx)
            basis, tv, th = oracle.camera_params(cam)
            dirs = oracle.camera_dirs(basis, tv, th, cam.width, cam.height)[idx]
            exp = oracle.trace_rays(g.probe_set, g.grid_origin, g.cell_size,
                                    g.dims, np.asarray(cam.eye, np.float64),
                                    dirs)
            _assert_same(got, exp, f"pose {c}")


class TestC4AsBenchmarked:
    """C4: the 8x2x8 / 16x4x16 / 32x8x32 hierarchy at 128^2/32^2 (9,344
    probes) and a 3840x2160 view, as bench.py builds it; a seeded 1/64 pixel
    subsample vs the oracle's per-level composition."""

    def test_4k_hierarchy_subsample(self):
        from oracle import oracle
        from paper_2507_14624_b200 import configs
        from paper_2507_14624_b200 import device as dev
        from paper_2507_14624_b200.render import device_probe_set
        cfg = configs.c4(n_views=1)
        assert [g.probe_set.dist_hi.shape[1:] for g in cfg.levels] == \
            [(128, 128)] * 3
        assert sum(g.probe_set.n_probes for g in cfg.levels) == 9344
        cam = cfg.cameras[0]
        assert (cam.width, cam.height) == (3840, 2160)
        levels = [(device_probe_set(g), _grid_params(g)) for g in cfg.levels]
        n = cam.width * cam.height
        out = dev.RayOutputs(n, levels[0][0].device, probe=True, texel=True,
                             fetch=True)
        dev.render_hierarchy(levels, [cam], cam.width, cam.height, out)
        torch.cuda.synchronize()
        idx = np.sort(np.random.default_rng(404).choice(n, n // 64,
                                                        replace=False))
        got = _host(out, idx)
        basis, tv, th = oracle.camera_params(cam)
        dirs = oracle.camera_dirs(basis, tv, th, cam.width, cam.height)[idx]
        exp = oracle.trace_hierarchy(cfg.levels, np.asarray(cam.eye,
                                                            np.float64), dirs)
        _assert_same(got, exp, "C4")
        hit = got["status"] == 1
        assert hit.mean() > 0.3
        assert len(np.unique(got["probe"][hit] >> 24)) >= 2


class TestC5AsBenchmarked:
    """C5: the first 2^20 rays of the bench's 2^26-ray set (configs.c5_rays
    block structure) against the C3 probe set, through the schedule the
    bench uses at this size (wavefront) and trace_rays' public path."""

    def test_first_2e20_rays(self, c3cfg):
        from oracle import oracle
        from paper_2507_14624_b200 import configs, trace_rays
        g = c3cfg.grid
        o32, d32 = configs.c5_rays(c3cfg.scene, 1 << 20)
        o_full, d_full = configs.c5_rays(c3cfg.scene, (1 << 20) + 5)
        np.testing.assert_array_equal(o32, o_full[:1 << 20])
        # the schedule the bench's 2^26-ray batch takes (default from 2^21 rays)
        res = trace_rays(g, o32, d32, schedule="wave")
        res_p = trace_rays(g, o32, d32)   # default at this size: persistent
        for k in ("status", "probe", "tx", "ty", "fetch", "rgb"):
            np.testing.assert_array_equal(getattr(res_p, k), getattr(res, k), err_msg=k)
        got = dict(status=res.status, probe=res.probe, tx=res.tx, ty=res.ty,
                   fetch=res.fetch, rgb=res.rgb, hit_t=res.hit_t)
        o64, d64 = o32.astype(np.float64), d32.astype(np.float64)
        exp = oracle.trace_rays(g.probe_set, g.grid_origin, g.cell_size,
                                g.dims, o64, d64)
        _assert_same(got, exp, "C5")
        sel = np.flatnonzero(exp.status == 1)[:20000]
        sub = oracle.Result(len(sel))
        for k in ("status", "probe", "tx", "ty"):
            getattr(sub, k)[:] = getattr(exp, k)[sel]
        _, ht = _hit_t_expected(g.probe_set, o64[sel], d64[sel], sub)
        np.testing.assert_allclose(res.hit_t[sel], ht, rtol=1e-4, atol=1e-6)


    def test_page_locked_inputs_take_the_async_upload(self, c3cfg):
        """trace_rays uploads page-locked host arrays asynchronously ahead
        of the trace; results equal those from pageable arrays, f32 and f64,
        and across the two record strides of the wavefront state."""
        import torch
        from paper_2507_14624_b200 import configs, trace_rays
        g = c3cfg.grid
        n = (1 << 20) + 3
        o32, d32 = configs.c5_rays(c3cfg.scene, n)
        ref = trace_rays(g, o32, d32, schedule="wave")
        po = torch.from_numpy(o32).pin_memory()
        pd = torch.from_numpy(d32).pin_memory()
        assert torch.from_numpy(po.numpy()).is_pinned()
        got = trace_rays(g, po.numpy(), pd.numpy(), schedule="wave")
        got64 = trace_rays(g, o32.astype(np.float64), d32.astype(np.float64),
                           schedule="wave")
        for r in (got, got64):
            for k in ("status", "probe", "tx", "ty", "fetch", "rgb"):
                np.testing.assert_array_equal(getattr(r, k), getattr(ref, k), err_msg=k)


class TestMapRatios:
    """High-res / low-res map ratios other than the benchmarked 4: the
    high-res DDA set-up takes its increments from the low-res DDA by exact
    power-of-two scaling (ratios 2, 8) and falls back to one IEEE reciprocal
    per axis otherwise (ratio 3, 6); equal maps (ratio 1)."""

    @pytest.mark.parametrize("r_hi,r_lo", [(48, 16), (32, 16), (64, 8),
                                           (48, 8), (24, 24)])
    def test_frame_and_rays_vs_oracle(self, r_hi, r_lo):
        from oracle import oracle
        from paper_2507_14624_b200 import (Camera, render_frame, scenes,
                                           trace_rays)
        from paper_2507_14624_b200.bake import bake_grid_gpu
        scene = scenes.room_scene(77, size=(4.0, 3.0, 4.0), n_boxes=6,
                                  n_spheres=3)
        g = bake_grid_gpu(scene, (0.0, 0.0, 0.0), 2.0, (3, 2, 3), r_hi, r_lo)
        cam = Camera(eye=(1.3, 1.1, 0.9), forward=(0.5, 0.1, 0.85),
                     vfov_deg=60.0, width=96, height=64)
        frame = render_frame(g, cam)
        res, _ = oracle.render_camera(g.probe_set, g.grid_origin, g.cell_size,
                                      g.dims, cam)
        pix, st = oracle.frame_pixels(res, cam.height, cam.width)
        np.testing.assert_array_equal(frame.status, st)
        np.testing.assert_array_equal(frame.pixels, pix)
        assert abs(frame.stats["perPixelTexelFetches"] - res.fetch.mean()) < 1e-9
        rng = np.random.default_rng(5)
        n = 20000
        o = rng.uniform((0.2, 0.2, 0.2), (3.8, 2.8, 3.8), (n, 3))
        d = rng.normal(size=(n, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        got = trace_rays(g, o, d)
        exp = oracle.trace_rays(g.probe_set, g.grid_origin, g.cell_size, g.dims,
                                o, d)
        _assert_same(dict(status=got.status, probe=got.probe, tx=got.tx,
                          ty=got.ty, fetch=got.fetch, rgb=got.rgb), exp,
                     f"ratio {r_hi}/{r_lo}")


# ---------------------------------------------------------------------------
# The reference's acceptance setups (pkg/tests/test_acceptance.py) on the
# CUDA path: the fixed room (scenes.py:249-270), a dense point cloud, the
# point-cloud bake (lfp_bake_points, bit-identical to bake_probe) at 2048^2.
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def dense_cloud():
    from paper_2507_14624_b200 import scenes
    return scenes.sample_point_cloud(scenes.acceptance_room(), 3.0e5, seed=11)


def _single_probe_oracle(p, cam, config):
    from oracle import oracle
    basis, tv, th = oracle.camera_params(cam)
    dirs = oracle.camera_dirs(basis, tv, th, cam.width, cam.height)
    pad = config.bounds_pad
    st, rgb, fe = oracle.render_single_probe(
        p.chain.distance_hi, p.chain.direction_hi, p.chain.irradiance_hi,
        p.chain.distance_lo, p.origin, np.asarray(cam.eye, np.float64), dirs,
        np.asarray(p.bounds_lo, np.float64) - pad,
        np.asarray(p.bounds_hi, np.float64) + pad, config.eps_start,
        config.slack)
    return st, rgb, fe


def _frame_vs_oracle(frame, st, rgb, fe, cam):
    from oracle import oracle

    class R:
        pass
    r = R()
    r.status, r.rgb = st, rgb
    pix, status = oracle.frame_pixels(r, cam.height, cam.width)
    np.testing.assert_array_equal(frame.status, status)
    np.testing.assert_array_equal(frame.pixels, pix)
    assert frame.stats["perPixelTexelFetches"] == pytest.approx(fe.mean(),
                                                                abs=1e-12)


class TestAcceptance2048:
    def test_c8_low_res_invariance(self, dense_cloud):
        """test_acceptance.py:318-337: renders from 2048^2/128^2 and
        2048^2/64^2 probes of the same cloud are pixel-identical -- and each
        equals the oracle's frame."""
        from paper_2507_14624_b200 import Camera, render_frame, scenes
        from paper_2507_14624_b200.pointbake import bake_probe
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG
        c = scenes.acceptance_center()
        pa = bake_probe(dense_cloud, c, r_hi=2048, r_lo=128)
        pb = bake_probe(dense_cloud, c, r_hi=2048, r_lo=64)
        eye = c + np.array([0.5, 0.0, 0.0])
        cam = Camera(eye=tuple(eye), forward=(0.3, 0.0, 1.0), width=512,
                     height=512)
        fa = render_frame(pa, cam)
        fb = render_frame(pb, cam)
        np.testing.assert_array_equal(fa.pixels, fb.pixels)
        np.testing.assert_array_equal(fa.status, fb.status)
        for p, f in ((pa, fa), (pb, fb)):
            _frame_vs_oracle(f, *_single_probe_oracle(p, cam, DEFAULT_CONFIG),
                             cam)
        assert (fa.status == 1).mean() > 0.5

    def test_c1_eye_aligned_2048(self, dense_cloud):
        """test_acceptance.py:72-108: from the probe origin the frame is the
        direct octahedral lookup, exactly on every non-EMPTY texel."""
        from paper_2507_14624_b200 import Camera, oct_encode, render_frame, scenes
        from paper_2507_14624_b200.pointbake import bake_probe
        c = scenes.acceptance_center()
        p = bake_probe(dense_cloud, c, r_hi=2048, r_lo=128)
        cam = Camera(eye=tuple(c), forward=(0.0, 0.0, 1.0), width=512,
                     height=512)
        frame = render_frame(p, cam)
        uv = oct_encode(cam.ray_directions())
        tx = np.minimum((uv[:, 0] * 2048).astype(int), 2047)
        ty = np.minimum((uv[:, 1] * 2048).astype(int), 2047)
        direct = p.chain.irradiance_hi[ty, tx].reshape(512, 512, 3)
        filled = np.isfinite(p.chain.distance_hi[ty, tx]).reshape(512, 512)
        assert np.array_equal(frame.pixels[filled], direct[filled])
        close = (np.abs(frame.pixels - direct) <= 1.0 / 255.0).all(axis=2)
        assert close.mean() >= 0.99
        assert frame.stats["perPixelTexelFetches"] == 1.0

    def test_c6_multi_probe_fallback(self):
        """test_acceptance.py:218-274: a probe in front of a pillar cannot
        certify its back face (patch pixels UNKNOWN/MISS, no false hit); a
        second probe removes >= 90% of those pixels; an 8-probe grid walk
        leaves < 0.5%. Every frame equals the oracle's."""
        from oracle import oracle
        from paper_2507_14624_b200 import Camera, render_frame, scenes
        from paper_2507_14624_b200.pointbake import bake_grid, simulate_probe
        from paper_2507_14624_b200.grid import ProbeSet
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG as cfg
        pillar = scenes.Box((1.3, 0.0, 3.8), (1.7, 2.5, 4.2),
                            albedo=(0.0, 1.0, 1.0))
        occ = scenes.acceptance_room(with_boxes=False, extra=(pillar,))
        cloud = scenes.sample_point_cloud(occ, 3e4, seed=5)
        front = simulate_probe(cloud, (1.5, 1.25, 3.2), r_hi=512, r_lo=64)
        behind = simulate_probe(cloud, (2.3, 1.25, 4.8), r_hi=512, r_lo=64)
        eye = np.array([2.6, 1.25, 4.9])
        cam = Camera(eye=tuple(eye), forward=tuple((1.5, 1.25, 4.2) - eye),
                     width=256, height=256)
        dirs = cam.ray_directions()
        t, prim = scenes.intersect(occ, eye, dirs)
        pts = eye + t[:, None] * dirs
        patch = (np.isfinite(t) & (np.abs(pts[:, 2] - 4.2) < 1e-6)
                 & (pts[:, 0] >= 1.3) & (pts[:, 0] <= 1.7)
                 & (pts[:, 1] >= 0.3) & (pts[:, 1] <= 2.2))
        n_patch = int(patch.sum())
        assert n_patch > 1000
        colors = np.asarray([p.albedo for p in occ.primitives])[prim]

        f1 = render_frame(front, cam)
        _frame_vs_oracle(f1, *_single_probe_oracle(front, cam, cfg), cam)
        bad1 = int(((f1.status.reshape(-1) != 1) & patch).sum())
        hitp = (f1.status.reshape(-1) == 1) & patch
        false_hits = int((np.abs(f1.pixels.reshape(-1, 3)[hitp]
                                 - colors[hitp]).max(axis=1) > 0.02).sum())

        f2 = render_frame([front, behind], cam)
        ps = ProbeSet([front, behind])
        blo = np.minimum(front.bounds_lo, behind.bounds_lo) - cfg.bounds_pad
        bhi = np.maximum(front.bounds_hi, behind.bounds_hi) + cfg.bounds_pad
        st, rgb, fe = oracle.render_few_probes(     # sorts nearest-first
            ps, blo, bhi, eye, dirs, cfg.eps_start, cfg.eps_align, cfg.slack)
        _frame_vs_oracle(f2, st, rgb, fe, cam)
        bad2 = int(((f2.status.reshape(-1) != 1) & patch).sum())

        grid = bake_grid(cloud, (1.0, 0.25, 3.4), 1.8, (2, 2, 2), r_hi=512,
                         r_lo=64)
        fg = render_frame(grid, cam)
        g = grid
        res, _ = oracle.render_camera(g.probe_set, g.grid_origin, g.cell_size,
                                      g.dims, cam)
        _frame_vs_oracle(fg, res.status, res.rgb, res.fetch, cam)
        badg = int(((fg.status.reshape(-1) != 1) & patch).sum())

        assert bad1 >= 0.5 * n_patch
        assert false_hits == 0
        assert bad2 <= 0.1 * bad1
        assert badg < 0.005 * n_patch


# ---------------------------------------------------------------------------
# The reference's property tests, on the CUDA backend
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def room_grid():
    """pkg/tests/test_grid.py:14-17 recipe: the fixed room's cloud at 2000
    pts/m^2 baked on a (0.5, 0.25, 0.5) + 2 m 2x2x2 lattice at 128^2/32^2."""
    from paper_2507_14624_b200 import scenes
    from paper_2507_14624_b200.pointbake import bake_grid
    cloud = scenes.sample_point_cloud(scenes.acceptance_room(), 2000.0,
                                      seed=7)
    return bake_grid(cloud, (0.5, 0.25, 0.5), 2.0, (2, 2, 2), r_hi=128,
                     r_lo=32)


class TestReferencePropertiesOnGpu:
    def test_hits_satisfy_visibility_sign(self, room_grid, c3cfg):
        """test_trace.py:256-266: every HIT's stored direction agrees with
        the ray direction (dir_hi . d > 0), on incoherent rays."""
        from paper_2507_14624_b200 import configs, trace_rays
        for grid, scene in ((room_grid, None), (c3cfg.grid, c3cfg.scene)):
            rng = np.random.default_rng(1234)
            n = 1 << 16
            if scene is None:
                o = np.array([1.5, 1.25, 1.5]) + rng.uniform(-0.8, 0.8, (n, 3))
                d = rng.normal(size=(n, 3))
                d /= np.linalg.norm(d, axis=1, keepdims=True)
            else:
                o, d = configs.c5_rays(scene, n, seed=9)
                o, d = o.astype(np.float64), d.astype(np.float64)
            r = trace_rays(grid, o, d)
            hit = np.flatnonzero(r.status == 1)
            assert len(hit) > n // 10
            stored = grid.probe_set.dir_hi[r.probe[hit], r.ty[hit], r.tx[hit]]
            assert (np.einsum("ij,ij->i", stored.astype(np.float64),
                              d[hit]) > 0.0).all()

    def test_hit_stops_probe_loop(self, room_grid):
        """test_grid.py:99-107: straight down onto the cyan box top: HIT,
        and the trace stops at the hitting probe -- the CUDA fetch count
        equals the oracle's (which returns at the first HIT, K:639-643)
        and is below the cost of tracing every corner probe."""
        from oracle import oracle
        from paper_2507_14624_b200 import trace_rays
        g = room_grid
        o = np.array([[0.9, 1.25, 1.4]])
        d = np.array([[0.0, -1.0, 0.0]])
        r = trace_rays(g, o, d)
        exp = oracle.trace_rays(g.probe_set, g.grid_origin, g.cell_size,
                                g.dims, o, d)
        assert r.status[0] == 1 and exp.status[0] == 1
        assert r.fetch[0] == exp.fetch[0] and r.probe[0] == exp.probe[0]
        # the ray stays in cube (0,0,0) for t in [0, 1] (y 1.25 -> 0.25):
        # the corners in the kernel's order (stable by squared eye
        # distance, K:758-785) are traced until the first HIT, and the
        # fetch count is exactly the sum over those probes -- no probe
        # after the hitting one is touched
        ps = g.probe_set
        corners = [(i * 2 + j) * 2 + k for i in (0, 1) for j in (0, 1)
                   for k in (0, 1)]
        d2 = [float(np.sum((ps.origins[c] - o[0]) ** 2)) for c in corners]
        order = [corners[i] for i in np.argsort(d2, kind="stable")]
        total = 0
        for n_traced, p in enumerate(order, 1):
            st, tx, ty, fe = oracle.trace_probe_range(
                ps.dist_hi[p], ps.dir_hi[p], ps.dist_lo[p], o[0] - ps.origins[p],
                d[0], 0.0, 1.0)
            total += fe
            if st == 1:
                break
        assert st == 1 and p == r.probe[0] and n_traced < 8
        assert r.fetch[0] == total

    def test_coverage_monotone_in_probe_count(self, room_grid):
        """test_grid.py:175-190: the non-HIT fraction of few-probe renders
        is non-increasing over nested probe subsets [1, 2, 4, 7] (300
        seeded rays, each a 1x1 camera whose pixel ray is its forward)."""
        from paper_2507_14624_b200 import Camera, ProbeData, MapChain
        from paper_2507_14624_b200 import device as dev
        from paper_2507_14624_b200.render import (_probe_bounds,
                                                  few_probe_order)
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG as cfg
        g = room_grid
        ps = g.probe_set
        rng = np.random.default_rng(1234)
        rays = []
        for _ in range(300):
            o = np.array([rng.uniform(0.7, 2.3), rng.uniform(0.4, 2.0),
                          rng.uniform(0.7, 2.3)])
            v = rng.normal(size=3)
            rays.append((o, v / np.linalg.norm(v)))
        probes = [ProbeData(origin=ps.origins[i], chain=MapChain(
            irradiance_hi=ps.irr_hi[i], distance_hi=ps.dist_hi[i],
            direction_hi=ps.dir_hi[i], distance_lo=ps.dist_lo[i]),
            bounds_lo=np.zeros(3), bounds_hi=np.array([3.0, 2.5, 6.0]))
            for i in range(8)]
        fractions = []
        for k in (1, 2, 4, 7):
            sub = probes[:k]
            dps = dev.DeviceProbeSet(ps.dist_hi[:k], ps.dir_hi[:k],
                                     ps.irr_hi[:k], ps.dist_lo[:k],
                                     ps.origins[:k])
            bounds = _probe_bounds(sub, cfg.bounds_pad)
            miss = 0
            for o, d in rays:
                cam = Camera(eye=tuple(o), forward=tuple(d), width=1,
                             height=1)
                out = dev.RayOutputs(1, dps.device)
                dev.render_probes(dps, dev.native.LFP_SOURCE_FEW, [cam], 1, 1,
                                  out, dev.grid_params((0, 0, 0), 1.0,
                                                       (1, 1, 1), cfg),
                                  order=few_probe_order(ps.origins[:k], o),
                                  bounds=bounds)
                miss += int(out.status.cpu()[0]) != 1
            fractions.append(miss / len(rays))
        assert all(a >= b - 1e-9 for a, b in zip(fractions, fractions[1:]))
        assert fractions[-1] < fractions[0]

    def test_few_probe_list_beyond_256(self, golden):
        """render_frame on a probe list longer than 256 (the order travels
        in device memory) equals the oracle's render_few_probes (which sorts
        nearest-first itself, stable: repeated origins tie)."""
        from conftest import golden_grid
        from oracle import oracle
        from paper_2507_14624_b200 import (Camera, MapChain, ProbeData,
                                           render_frame)
        from paper_2507_14624_b200.grid import ProbeSet
        from paper_2507_14624_b200.trace import DEFAULT_CONFIG as cfg
        ps = golden_grid(golden("pcgrid")).probe_set
        P = ps.dist_hi.shape[0]
        lo, hi = ps.origins.min(0) - 0.5, ps.origins.max(0) + 0.5
        probes = [ProbeData(origin=ps.origins[i % P], chain=MapChain(
            irradiance_hi=ps.irr_hi[i % P], distance_hi=ps.dist_hi[i % P],
            direction_hi=ps.dir_hi[i % P], distance_lo=ps.dist_lo[i % P]),
            bounds_lo=lo, bounds_hi=hi) for i in range(300)]
        cam = Camera(eye=(1.3, 1.1, 1.7), forward=(0.4, -0.2, -1.0),
                     width=48, height=40)
        fr = render_frame(probes, cam)
        basis, tv, th = oracle.camera_params(cam)
        dirs = oracle.camera_dirs(basis, tv, th, cam.width, cam.height)
        st, rgb, fe = oracle.render_few_probes(
            ProbeSet(probes), lo - cfg.bounds_pad, hi + cfg.bounds_pad,
            np.asarray(cam.eye, np.float64), dirs, cfg.eps_start,
            cfg.eps_align, cfg.slack)
        _frame_vs_oracle(fr, st, rgb, fe, cam)
        assert (fr.status == 2).any() or (fr.status == 1).any()


class TestDropInSemantics:
    def test_bench_views_runs(self):
        """render.py:169-201 mirror on the GPU: report keys, per-view
        medians, stats equal to render_frame's."""
        from paper_2507_14624_b200 import bench_views, configs, render_frame
        cfg = configs.c1()
        cams = cfg.cameras + configs.random_cameras(cfg.scene, 2, 128, 128, 5)
        rep = bench_views(cfg.grid, cams, warmup=1, reps=4)
        assert set(rep) == {"views", "medianMsMean", "relativeStdOfMedians",
                            "warmup", "reps"}
        assert len(rep["views"]) == 3 and rep["reps"] == 4
        for i, v in enumerate(rep["views"]):
            assert v["view"] == i
            assert 0 < v["minMs"] <= v["medianMs"] <= v["maxMs"]
            fr = render_frame(cfg.grid, cams[i])
            for k in ("missFraction", "unknownFraction",
                      "perPixelTexelFetches"):
                assert v[k] == fr.stats[k]
        med = np.array([v["medianMs"] for v in rep["views"]])
        assert rep["medianMsMean"] == pytest.approx(med.mean())
        assert rep["relativeStdOfMedians"] == pytest.approx(
            med.std() / med.mean())
        with pytest.raises(ValueError):
            bench_views(cfg.grid, [])

    def test_render_grid_cache_sees_in_place_edits(self, golden):
        """kernels.render_grid caches the device copy per host array; an
        in-place edit is picked up after device.invalidate() or with
        VERIFY_CONTENT on, matching the numba kernel which reads the arrays
        on every call (K:825-843)."""
        from conftest import GoldenProbeSet
        from oracle import oracle
        from paper_2507_14624_b200 import device as dev
        from paper_2507_14624_b200 import kernels
        z = golden("pcgrid")
        ps = GoldenProbeSet(z)
        # private copies: the session-scoped golden arrays must stay intact
        for k in ("dist_hi", "dir_hi", "irr_hi", "dist_lo", "origins"):
            setattr(ps, k, getattr(ps, k).copy())
        args_tail = (z["grid_origin"], float(z["cell"]),
                     *(int(v) for v in z["dims"]), z["cam_eye"], z["cam_dirs"],
                     1e-4, 1e-4, 1e-3)
        n = len(z["cam_dirs"])

        def run():
            st = np.zeros(n, np.uint8)
            rgb = np.zeros((n, 3))
            fe = np.zeros(n, np.int64)
            kernels.render_grid(ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo,
                                ps.origins, *args_tail, st, rgb, fe)
            return st, fe

        def expect():
            st = np.zeros(n, np.uint8)
            rgb = np.zeros((n, 3))
            fe = np.zeros(n, np.int64)
            oracle.render_grid(ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo,
                               ps.origins, *args_tail, st, rgb, fe)
            return st, fe

        st0, fe0 = run()
        np.testing.assert_array_equal(st0, z["cam_status"])
        ps.dist_hi[:, ::2, :] = np.inf          # in-place edit
        ps.dist_lo[:] = np.inf
        dev.invalidate(ps.dist_hi)
        st1, fe1 = run()
        e_st, e_fe = expect()
        np.testing.assert_array_equal(st1, e_st)
        np.testing.assert_array_equal(fe1, e_fe)
        assert not np.array_equal(st1, st0)
        old = dev.VERIFY_CONTENT
        dev.VERIFY_CONTENT = True
        try:
            ps.dist_lo[:] = z["dist_lo"]        # another in-place edit
            st2, fe2 = run()
            e_st, e_fe = expect()
            np.testing.assert_array_equal(st2, e_st)
            np.testing.assert_array_equal(fe2, e_fe)
        finally:
            dev.VERIFY_CONTENT = old
