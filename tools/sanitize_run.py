"""Small workload that launches every kernel family of liblfprobe_b200.so once,
for compute-sanitizer (tools/sanitize.sh): camera frames (nested and
persistent schedules, frame-ordered and compact shards, the zero-copy host
frame path), untile, the probe hierarchy, explicit rays (nested, persistent,
wavefront, binned / ordered), the non-grid sources (single probe, probe
list, eye-aligned lookup), the ray-cast and point-cloud bakes, the packed
.lfp load and the division self-test. Checks a few outputs against the CPU
oracle so a sanitizer run that silently changes results is also caught."""

import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from conftest import GOLDEN, golden_camera, golden_grid, load_golden  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2507_14624_b200 import (Camera, MapChain, ProbeData,  # noqa: E402
                                   ProbeHierarchy, configs, lfpio,
                                   render_frame)
from paper_2507_14624_b200 import device as dev  # noqa: E402
from paper_2507_14624_b200 import scenes  # noqa: E402
from paper_2507_14624_b200.bake import bake_grid_gpu  # noqa: E402
from paper_2507_14624_b200.pointbake import bake_grid as pc_bake_grid  # noqa: E402
from paper_2507_14624_b200.render import device_probe_set  # noqa: E402
from paper_2507_14624_b200.trace import DEFAULT_CONFIG  # noqa: E402


def step(name):
    print(f"[sanitize] {name}", flush=True)


# With the bounds-check build (LFP_LIB_PATH=.../liblfprobe_b200_check.so)
# every call below runs with index checks on and, where the call writes n
# per-ray records, a write counter per record.
import ctypes  # noqa: E402

from paper_2507_14624_b200 import native  # noqa: E402

DEBUG = native.lib().lfp_debug_bounds(0, None, 0) == 0
CHECKED = 0


def checked(n, fn, expect=None):
    """Run fn(); in the check build assert no index violation and that the
    n output records were written exactly once each (or `expect(result)`
    times: an int array)."""
    global CHECKED
    if not DEBUG:
        return fn()
    L = native.lib()
    wc = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    native.check(L.lfp_debug_bounds(0, ctypes.c_void_p(wc.data_ptr()), n))
    r = fn()
    v, site = ctypes.c_uint64(), ctypes.c_int32()
    native.check(L.lfp_debug_report(0, ctypes.byref(v), ctypes.byref(site)))
    native.check(L.lfp_debug_bounds(0, None, 0))
    assert v.value == 0, f"{v.value} index violations, first at site {site.value}"
    w = wc.cpu().numpy()[:n]
    want = np.ones(n, np.int32) if expect is None else np.asarray(expect(r))
    assert np.array_equal(w, want), \
        f"write counts: {int((w != want).sum())} of {n} records wrong " \
        f"(max {int(w.max()) if n else 0})"
    CHECKED += 1
    return r


def main():
    z = load_golden("pcgrid")
    grid = golden_grid(z)
    dps = device_probe_set(grid)

    step("camera frame (render_frame: zero-copy host frame path)")
    cam = golden_camera(z, "cam_")
    cam = Camera(eye=cam.eye, forward=cam.forward, up=cam.up,
                 vfov_deg=cam.vfov_deg, width=64, height=48)
    fr = checked(64 * 48, lambda: render_frame(grid, cam))
    res, _ = oracle.render_camera(grid.probe_set, grid.grid_origin,
                                  grid.cell_size, grid.dims, cam)
    assert np.array_equal(fr.status.ravel(), res.status)

    for sched in ("nested", "persistent"):
        step(f"render_cameras {sched}: frame order + compact shards + untile")
        g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                            DEFAULT_CONFIG, schedule=sched)
        cams = [cam, Camera(eye=(1.1, 0.9, 1.2), forward=(-0.3, 0.1, 1.0),
                            width=64, height=48)]
        full = dev.RayOutputs(2 * 64 * 48, dps.device, probe=True, texel=True,
                              fetch=True, hit_t=True, rgb8=True)
        checked(2 * 64 * 48,
                lambda: dev.render_cameras(dps, g, cams, 64, 48, full))
        T = dev.num_tiles(2, 64, 48)
        parts_s, parts_c = [], []
        for k in range(3):
            nk = (T - k + 2) // 3
            o = dev.RayOutputs(((T + 2) // 3) * 128, dps.device)
            o.status.fill_(255)
            o.rgb.zero_()
            checked(o.n, lambda: dev.render_cameras(
                dps, g, cams, 64, 48, o, tile_begin=k, tile_step=3,
                n_tiles=nk, compact=True),
                expect=lambda _: (o.status != 255).int().cpu().numpy())
            o.status[o.status == 255] = 0
            parts_s.append(o.status)
            parts_c.append(o.rgb)
        st = torch.empty(2 * 64 * 48, dtype=torch.uint8, device="cuda")
        rgb = torch.empty((2 * 64 * 48, 3), dtype=torch.float32, device="cuda")
        dev.untile(2, 64, 48, 3, torch.cat(parts_s), torch.cat(parts_c), st, rgb,
                   shard_stride=(T + 2) // 3)
        torch.cuda.synchronize()
        assert torch.equal(st, full.status)

    step("check mode (decision re-check, diag counters)")
    g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                        DEFAULT_CONFIG, mode="check")
    o = dev.RayOutputs(64 * 48, dps.device, diag=True)
    checked(64 * 48, lambda: dev.render_cameras(dps, g, [cam], 64, 48, o))
    torch.cuda.synchronize()
    assert int(o.diag[4]) == 0

    step("hierarchy (two levels of different resolution)")
    c1 = configs.c1()
    h = ProbeHierarchy([c1.grid, grid])
    frh = checked(40 * 24, lambda: render_frame(
        h, Camera(eye=(1.3, 1.1, 1.7), forward=(0.4, -0.2, -1.0), width=40,
                  height=24)))
    assert frh.status.shape == (24, 40)

    o32 = z["inc_origins"][:1024].astype(np.float64)
    d32 = z["inc_dirs"][:1024].astype(np.float64)
    exp = oracle.trace_rays(grid.probe_set, grid.grid_origin, grid.cell_size,
                            grid.dims, o32, d32)
    to = torch.from_numpy(o32).cuda()
    td = torch.from_numpy(d32).cuda()
    for sched in ("nested", "persistent", "wave"):
        for binned in (False, True):
            step(f"trace_rays schedule={sched} binned={binned}")
            g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                                DEFAULT_CONFIG, schedule=sched)
            out = dev.RayOutputs(1024, dps.device, probe=True, texel=True,
                                 fetch=True, hit_t=True)
            out.rgb.zero_()
            if binned:
                order = dev.ray_order(dev.bin_rays(g, to, td))
                checked(1024, lambda: dev.trace_rays_ordered(
                    dps, g, to, td, order, out))
            else:
                checked(1024, lambda: dev.trace_rays(dps, g, to, td, out))
            torch.cuda.synchronize()
            assert np.array_equal(out.status.cpu().numpy(), exp.status)
            assert np.array_equal(out.fetch.cpu().numpy(), exp.fetch)

    step("render_grid (shared eye, f32 dirs)")
    g = dev.grid_params(grid.grid_origin, grid.cell_size, grid.dims,
                        DEFAULT_CONFIG)
    out = dev.RayOutputs(1024, dps.device, fetch=True)
    checked(1024, lambda: dev.render_grid_dirs(dps, g, o32[0], td.float(), out))
    torch.cuda.synchronize()

    step("non-grid sources: single probe, probe list, eye-aligned lookup")
    zm = load_golden("modes")
    probes = []
    for i in range(3):
        ch = MapChain(irradiance_hi=zm[f"p{i}_irr_hi"],
                      distance_hi=zm[f"p{i}_dist_hi"],
                      direction_hi=zm[f"p{i}_dir_hi"],
                      distance_lo=zm[f"p{i}_dist_lo"])
        probes.append(ProbeData(origin=zm[f"p{i}_origin"], chain=ch,
                                bounds_lo=zm[f"p{i}_blo"],
                                bounds_hi=zm[f"p{i}_bhi"]))
    for name, src in (("single", probes[0]), ("few", probes),
                      ("lookup", probes[1])):
        c = golden_camera(zm, name + "_")
        c = Camera(eye=c.eye, forward=c.forward, up=c.up, vfov_deg=c.vfov_deg,
                   width=48, height=32)
        checked(48 * 32, lambda: render_frame(src, c))

    step("ray-cast bake (lfp_bake_probes)")
    bake_grid_gpu(c1.scene, (0.0, 0.0, 0.0), 4.0, (2, 2, 2), 32, 8, quant="f16")

    step("point-cloud bake (lfp_bake_points)")
    cloud = scenes.sample_point_cloud(scenes.acceptance_room(), 200.0, seed=3)
    pc_bake_grid(cloud, (0.5, 0.25, 0.5), 2.0, (2, 2, 2), r_hi=32, r_lo=8)

    step("packed .lfp load (lfp_probeset_create_packed)")
    lfpio.load_grid(os.path.join(GOLDEN, "lfp_grid", "grid.json"))

    step("division self-test")
    import ctypes
    from paper_2507_14624_b200 import native
    a = torch.randn(4096, dtype=torch.float64, device="cuda")
    b = torch.randn(4096, dtype=torch.float64, device="cuda")
    r1, r2 = torch.empty_like(a), torch.empty_like(a)
    took = torch.empty(4096, dtype=torch.uint8, device="cuda")
    native.check(native.lib().lfp_selftest_division(
        ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), 4096,
        ctypes.c_void_p(r1.data_ptr()), ctypes.c_void_p(r2.data_ptr()),
        ctypes.c_void_p(took.data_ptr()),
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    if DEBUG:
        step("C5-like wavefront batch at 2^20 rays")
        o5, d5 = configs.c5_rays(c1.scene, 1 << 20, seed=3)
        t5o, t5d = torch.from_numpy(o5).cuda(), torch.from_numpy(d5).cuda()
        g = dev.grid_params(c1.grid.grid_origin, c1.grid.cell_size,
                            c1.grid.dims, DEFAULT_CONFIG, schedule="wave")
        out = dev.RayOutputs(1 << 20, dps.device, probe=True, texel=True,
                             fetch=True, hit_t=True)
        c1dps = device_probe_set(c1.grid)
        checked(1 << 20, lambda: dev.trace_rays(c1dps, g, t5o, t5d, out))
        print(f"[sanitize] bounds-check build: {CHECKED} checked calls, 0 "
              "index violations, every output record written exactly once",
              flush=True)
    print("[sanitize] all kernel families ran", flush=True)


if __name__ == "__main__":
    main()
