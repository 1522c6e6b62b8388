"""Seeded benchmark configurations C1..C5 (BASELINE.json `configs`,
SURVEY.md §8(d)). Every seed is fixed here; scenes, probes, cameras and
incoherent rays are synthetic stand-ins built from these seeds.

  C1  room 4x4 floor, 3 m high, 8 boxes + 4 spheres; 2x2x2 probes, cell 4,
      32^2 / 8^2 f32 maps; one 128x128 view, 60 deg
  C2  same generator, new seed; 4x4x4 probes, cell 4/3, 128^2 / 32^2 f32;
      one 512x512 view
  C3  room 7x7 floor, 3 m high, 64 boxes + 32 spheres; 8x4x8 probes, cell 1,
      256^2 / 64^2, f32 distance, fp16 radiance / direction; 64 poses at
      1920x1080
  C5  the C3 probe set; 2^26 rays, origins U(room interior), directions
      normalised Gaussian, stored f32 and up-cast exactly on both sides
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

from .bake import bake_grid, bake_grid_gpu
from .grid import ProbeGrid, ProbeHierarchy
from .render import Camera
from .scenes import city_scene, free_point, room_scene


@dataclass
class Config:
    name: str
    scene: object
    grid: ProbeGrid
    cameras: list
    description: str

    @property
    def rays_per_batch(self):
        return sum(c.width * c.height for c in self.cameras)


def random_cameras(scene, n, width, height, seed, vfov=60.0,
                   pitch_deg=30.0, margin=0.3):
    """Eye ~ U(interior, >= margin from walls, outside primitives); forward
    ~ U(yaw) with pitch U[-pitch, pitch]."""
    rng = np.random.default_rng(seed)
    cams = []
    for _ in range(n):
        eye = free_point(scene, rng, margin=margin)
        yaw = rng.uniform(0.0, 2.0 * np.pi)
        pitch = np.radians(rng.uniform(-pitch_deg, pitch_deg))
        fwd = (np.cos(pitch) * np.cos(yaw), np.sin(pitch),
               np.cos(pitch) * np.sin(yaw))
        cams.append(Camera(eye=tuple(float(v) for v in eye),
                           forward=tuple(float(v) for v in fwd),
                           vfov_deg=vfov, width=width, height=height))
    return cams


def c1(seed=101, cam_seed=1101, width=128, height=128):
    scene = room_scene(seed, size=(4.0, 3.0, 4.0), n_boxes=8, n_spheres=4)
    grid = bake_grid(scene, (0.0, 0.0, 0.0), 4.0, (2, 2, 2), 32, 8)
    cams = random_cameras(scene, 1, width, height, cam_seed)
    return Config("c1", scene, grid, cams,
                  "room 4x4x3 m, 8 boxes + 4 spheres; 2x2x2 probes cell 4; "
                  "32^2/8^2 f32; 128x128 view")


def c2(seed=202, cam_seed=2202, width=512, height=512, n_views=1):
    scene = room_scene(seed, size=(4.0, 3.0, 4.0), n_boxes=8, n_spheres=4)
    grid = bake_grid(scene, (0.0, 0.0, 0.0), 4.0 / 3.0, (4, 4, 4), 128, 32)
    cams = random_cameras(scene, n_views, width, height, cam_seed)
    return Config("c2", scene, grid, cams,
                  "room 4x4x3 m, 8 boxes + 4 spheres; 4x4x4 probes cell 4/3; "
                  "128^2/32^2 f32; 512x512 view")


def c3_scene(seed=303):
    return room_scene(seed, size=(7.0, 3.0, 7.0), n_boxes=64, n_spheres=32,
                      box_side=(0.2, 1.0), sphere_r=(0.1, 0.5))


def c3_grid(seed=303, device=0):
    """C3 probes, baked on the GPU (lfp_bake_probes): 256 probes x 256^2
    texels ray-cast against 102 primitives with shadow rays."""
    scene = c3_scene(seed)
    grid = bake_grid_gpu(scene, (0.0, 0.0, 0.0), 1.0, (8, 4, 8), 256, 64,
                         quant="f16", device=device)
    return scene, grid


def c3(seed=303, cam_seed=3303, n_views=64, width=1920, height=1080,
       device=0):
    scene, grid = c3_grid(seed, device)
    cams = random_cameras(scene, n_views, width, height, cam_seed)
    return Config("c3", scene, grid, cams,
                  "room 7x7x3 m, 64 boxes + 32 spheres; 8x4x8 probes cell 1; "
                  "256^2/64^2 f32 dist, f16 radiance/direction; "
                  f"{n_views} poses at {width}x{height}")


C4_LEVELS = (((8, 2, 8), 64.0 / 7.0), ((16, 4, 16), 64.0 / 15.0),
             ((32, 8, 32), 64.0 / 31.0))


def c4_levels(seed=404, device=0, levels=C4_LEVELS, r_hi=128, r_lo=32):
    """C4 probe hierarchy: three lattices over the 64 x 64 m block (8x2x8,
    16x4x16, 32x8x32 probes, cubic cells 64/7, 64/15, 64/31 m; y spans 9.1 /
    12.8 / 14.5 m), 128^2 / 32^2 maps, f16 radiance / direction, all baked
    on the GPU against the 2001 primitives. Returns (scene, [ProbeGrid])."""
    scene = city_scene(seed)
    grids = [bake_grid_gpu(scene, (0.0, 0.0, 0.0), cell, dims, r_hi, r_lo,
                           quant="f16", device=device)
             for dims, cell in levels]
    return scene, grids


def street_cameras(scene, n, width, height, seed, vfov=60.0):
    """Eyes 1.5-12 m above the ground at free points of the block, looking
    across it pitched 10-30 degrees down."""
    rng = np.random.default_rng(seed)
    cams = []
    for _ in range(n):
        for _ in range(1000):
            eye = free_point(scene, rng, margin=4.0)
            eye[1] = rng.uniform(1.5, 12.0)
            if free_point_ok(scene, eye):
                break
        yaw = rng.uniform(0.0, 2.0 * np.pi)
        pitch = np.radians(rng.uniform(-30.0, -10.0))
        fwd = (np.cos(pitch) * np.cos(yaw), np.sin(pitch),
               np.cos(pitch) * np.sin(yaw))
        cams.append(Camera(eye=tuple(float(v) for v in eye),
                           forward=tuple(float(v) for v in fwd),
                           vfov_deg=vfov, width=width, height=height))
    return cams


def free_point_ok(scene, p):
    from .scenes import Box, scene_skip
    for prim in scene.primitives[scene_skip(scene):]:
        if isinstance(prim, Box) and np.all(p > np.asarray(prim.lo) - 0.05) \
                and np.all(p < np.asarray(prim.hi) + 0.05):
            return False
    return True


def c4(seed=404, cam_seed=4404, n_views=1, width=3840, height=2160, device=0):
    scene, grids = c4_levels(seed, device)
    cams = street_cameras(scene, n_views, width, height, cam_seed)
    cfg = Config("c4", scene, grids[-1], cams,
                 "block 64x64x16 m, ground + 2000 boxes (lognormal heights); "
                 "3-level probe hierarchy 8x2x8 / 16x4x16 / 32x8x32 at "
                 f"128^2/32^2 (f16 payloads), coarse-to-fine; {n_views} view(s) "
                 f"at {width}x{height}")
    cfg.levels = grids
    cfg.hierarchy = ProbeHierarchy(grids)
    return cfg


C5_BLOCK = 1 << 20


def c5_rays(scene, n, seed=505, start=0):
    """Incoherent rays [start, start + n) of the seeded C5 ray sequence:
    origins U(interior), directions normalised Gaussian
    (`pkg/tests/conftest.py:29-31`), both stored as float32. The sequence
    is generated in blocks of 2^20 rays, block b from default_rng([seed, b]),
    so any slice (a rank's share, the first 2^20 rays of the bench set) is
    reproducible without generating the whole 2^26-ray set."""
    lo = np.asarray(scene.interior_lo, np.float64)
    hi = np.asarray(scene.interior_hi, np.float64)
    o = np.empty((n, 3), np.float32)
    d = np.empty((n, 3), np.float32)
    b0, b1 = start // C5_BLOCK, (start + n + C5_BLOCK - 1) // C5_BLOCK
    for b in range(b0, b1):
        rng = np.random.default_rng([seed, b])
        bo = rng.uniform(lo, hi, size=(C5_BLOCK, 3)).astype(np.float32)
        bd = rng.normal(size=(C5_BLOCK, 3))
        bd /= np.linalg.norm(bd, axis=-1, keepdims=True)
        s0 = max(start, b * C5_BLOCK)
        s1 = min(start + n, (b + 1) * C5_BLOCK)
        o[s0 - start:s1 - start] = bo[s0 - b * C5_BLOCK:s1 - b * C5_BLOCK]
        d[s0 - start:s1 - start] = bd[s0 - b * C5_BLOCK:s1 - b * C5_BLOCK]
    return o, d


def probe_set_digest(ps):
    h = hashlib.sha256()
    for a in (ps.dist_hi, ps.dir_hi, ps.irr_hi, ps.dist_lo, ps.origins):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


BUILDERS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4}
