"""Seeded analytic scenes (boxes, spheres, one point light) for the
benchmark configurations.

The reference ships flat-colour boxes/spheres and one fixed room
(`pkg/src/lfprobe/scenes.py:41-75, 254-265`); the BASELINE configurations
need seeded rooms with Lambertian albedo lit by a point light, which the
reference does not have. This module is input production
for the tracer, not part of the traced path: it only feeds the bake.

Intersection semantics follow `scenes.py:122-148` (smallest t > eps; a ray
starting inside a box hits the inside of the far face; ties go to the lower
primitive index).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_EPS = 1e-9


@dataclass(frozen=True)
class Box:
    lo: tuple
    hi: tuple
    albedo: tuple = (0.8, 0.8, 0.8)


@dataclass(frozen=True)
class Sphere:
    center: tuple
    radius: float
    albedo: tuple = (0.8, 0.8, 0.8)


@dataclass(frozen=True)
class PointLight:
    position: tuple
    power: float = 6.0
    ambient: float = 0.15


@dataclass(frozen=True)
class Scene:
    primitives: tuple = field(default_factory=tuple)
    light: PointLight = PointLight((0.0, 2.5, 0.0))
    # interior AABB the cameras / incoherent rays live in
    interior_lo: tuple = (0.0, 0.0, 0.0)
    interior_hi: tuple = (1.0, 1.0, 1.0)

    def describe(self):
        nb = sum(isinstance(p, Box) for p in self.primitives)
        ns = sum(isinstance(p, Sphere) for p in self.primitives)
        return {"boxes": nb, "spheres": ns,
                "light": list(self.light.position),
                "interior": [list(self.interior_lo), list(self.interior_hi)]}


def _intersect_box(lo, hi, o, d):
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        t1 = (lo - o) * inv
        t2 = (hi - o) * inv
    tmin = np.where(np.isnan(t1), -np.inf, np.minimum(t1, t2))
    tmax = np.where(np.isnan(t2), np.inf, np.maximum(t1, t2))
    par = d == 0.0
    outside = par & ((o < lo) | (o > hi))
    tmin = np.where(par, -np.inf, tmin)
    tmax = np.where(par, np.inf, tmax)
    t_near = tmin.max(axis=-1)
    t_far = tmax.min(axis=-1)
    t_far = np.where(outside.any(axis=-1), -np.inf, t_far)
    hit = t_near <= t_far
    t = np.where(t_near > _EPS, t_near, t_far)
    return np.where(hit & (t > _EPS), t, np.inf)


def _intersect_sphere(c, r, o, d):
    oc = o - c
    b = np.sum(oc * d, axis=-1)
    cc = np.sum(oc * oc, axis=-1) - r * r
    disc = b * b - cc
    sq = np.sqrt(np.maximum(disc, 0.0))
    t0 = -b - sq
    t1 = -b + sq
    t = np.where(t0 > _EPS, t0, t1)
    return np.where((disc >= 0.0) & (t > _EPS), t, np.inf)


def _prim_arrays(scene):
    return [(np.asarray(p.lo, np.float64), np.asarray(p.hi, np.float64))
            if isinstance(p, Box) else
            (np.asarray(p.center, np.float64), float(p.radius))
            for p in scene.primitives]


def intersect(scene, origins, dirs, t_max=None):
    """Nearest hit for N rays: (t, prim index); t = +inf / -1 on a miss."""
    o = np.atleast_2d(np.asarray(origins, np.float64))
    d = np.atleast_2d(np.asarray(dirs, np.float64))
    n = max(len(o), len(d))
    o = np.broadcast_to(o, (n, 3))
    d = np.broadcast_to(d, (n, 3))
    best_t = np.full(n, np.inf)
    best_p = np.full(n, -1, np.int64)
    for i, (p, arr) in enumerate(zip(scene.primitives, _prim_arrays(scene))):
        if isinstance(p, Box):
            t = _intersect_box(arr[0], arr[1], o, d)
        else:
            t = _intersect_sphere(arr[0], arr[1], o, d)
        closer = t < best_t
        best_t = np.where(closer, t, best_t)
        best_p = np.where(closer, i, best_p)
    if t_max is not None:
        far = best_t >= t_max
        best_t = np.where(far, np.inf, best_t)
        best_p = np.where(far, -1, best_p)
    return best_t, best_p


def _normals(scene, prim, points):
    nrm = np.zeros_like(points)
    for i, p in enumerate(scene.primitives):
        m = prim == i
        if not m.any():
            continue
        q = points[m]
        if isinstance(p, Sphere):
            v = q - np.asarray(p.center)
            nrm[m] = v / np.linalg.norm(v, axis=-1, keepdims=True)
        else:
            lo = np.asarray(p.lo)
            hi = np.asarray(p.hi)
            dist = np.stack([np.abs(q[:, 0] - lo[0]), np.abs(q[:, 0] - hi[0]),
                             np.abs(q[:, 1] - lo[1]), np.abs(q[:, 1] - hi[1]),
                             np.abs(q[:, 2] - lo[2]), np.abs(q[:, 2] - hi[2])],
                            axis=-1)
            face = np.argmin(dist, axis=-1)
            axis = face // 2
            sign = np.where(face % 2 == 0, -1.0, 1.0)
            v = np.zeros_like(q)
            v[np.arange(len(q)), axis] = sign
            nrm[m] = v
    return nrm


def shade(scene, origins, dirs, t, prim, shadows=True):
    """Lambertian radiance of the hit points, clamped to [0, 1]; black on a
    miss. The normal is flipped toward the viewer so thin walls shade from
    either side."""
    n = len(t)
    rgb = np.zeros((n, 3))
    hit = prim >= 0
    if not hit.any():
        return rgb
    o = np.broadcast_to(np.asarray(origins, np.float64), (n, 3))[hit]
    d = np.broadcast_to(np.asarray(dirs, np.float64), (n, 3))[hit]
    ph = prim[hit]
    pts = o + t[hit, None] * d
    nrm = _normals(scene, ph, pts)
    flip = np.sum(nrm * d, axis=-1) > 0.0
    nrm[flip] *= -1.0
    lp = np.asarray(scene.light.position, np.float64)
    to_l = lp - pts
    dist_l = np.linalg.norm(to_l, axis=-1)
    ldir = to_l / dist_l[:, None]
    ndl = np.maximum(np.sum(nrm * ldir, axis=-1), 0.0)
    if shadows:
        s_t, _ = intersect(scene, pts + 1e-6 * nrm, ldir)
        ndl = np.where(s_t < dist_l - 1e-6, 0.0, ndl)
    albedo = np.asarray([scene.primitives[i].albedo for i in range(
        len(scene.primitives))], np.float64)[ph]
    lum = scene.light.ambient + (1.0 - scene.light.ambient) * ndl * np.minimum(
        1.0, scene.light.power / (1.0 + dist_l * dist_l))
    rgb[hit] = np.clip(albedo * lum[:, None], 0.0, 1.0)
    return rgb


def _walls(size, thick, rng):
    w, h, l = size
    t = thick
    spans = [((-t, -t, -t), (0.0, h + t, l + t)),      # -x
             ((w, -t, -t), (w + t, h + t, l + t)),     # +x
             ((-t, -t, -t), (w + t, 0.0, l + t)),      # floor
             ((-t, h, -t), (w + t, h + t, l + t)),     # ceiling
             ((-t, -t, -t), (w + t, h + t, 0.0)),      # -z
             ((-t, -t, l), (w + t, h + t, l + t))]     # +z
    return [Box(lo, hi, tuple(rng.uniform(0.2, 0.9, 3))) for lo, hi in spans]


def room_scene(seed, size=(4.0, 3.0, 4.0), n_boxes=8, n_spheres=4,
               box_side=(0.2, 1.0), sphere_r=(0.1, 0.5), wall=0.1):
    """Seeded room: six wall slabs bounding the interior [0, size], boxes
    resting on the floor, free-floating spheres, one point light under the
    ceiling. `size` is (x width, y height, z length) as in the reference's
    ROOM_SIZE (`scenes.py:251`). Albedo RGB ~ U[0.2, 0.9]^3."""
    rng = np.random.default_rng(seed)
    w, h, l = size
    prims = _walls(size, wall, rng)
    for _ in range(n_boxes):
        s = rng.uniform(*box_side, 3)
        s[1] = min(s[1], h * 0.8)
        x = rng.uniform(0.0, w - s[0])
        z = rng.uniform(0.0, l - s[2])
        prims.append(Box((x, 0.0, z), (x + s[0], s[1], z + s[2]),
                         tuple(rng.uniform(0.2, 0.9, 3))))
    for _ in range(n_spheres):
        r = rng.uniform(*sphere_r)
        c = (rng.uniform(r, w - r), rng.uniform(r, h - r),
             rng.uniform(r, l - r))
        prims.append(Sphere(c, r, tuple(rng.uniform(0.2, 0.9, 3))))
    light = PointLight((rng.uniform(0.3 * w, 0.7 * w), h - 0.3,
                        rng.uniform(0.3 * l, 0.7 * l)),
                       power=1.5 * max(w, l), ambient=0.15)
    return Scene(tuple(prims), light, (0.0, 0.0, 0.0), (w, h, l))


def city_scene(seed, size=64.0, height=16.0, n_boxes=2000,
               footprint=(1.0, 4.0), height_mu=1.0, height_sigma=0.5):
    """Seeded block-scale scene (BASELINE config 4): a 64 x 64 m ground slab
    and `n_boxes` axis-aligned buildings with footprint sides U[1, 4] m
    (the footprint distribution is this builder's choice) and heights
    exp(N(mu = 1, sigma = 0.5)) m clipped to the 16 m scene height, placed
    uniformly (overlaps allowed), albedo U[0.2, 0.9]^3, one high point
    light. Open sky: rays that leave the scene hit nothing (EMPTY texels)."""
    rng = np.random.default_rng(seed)
    prims = [Box((0.0, -1.0, 0.0), (size, 0.0, size),
                 tuple(rng.uniform(0.2, 0.9, 3)))]
    for _ in range(n_boxes):
        sx, sz = rng.uniform(*footprint, 2)
        h = float(np.clip(np.exp(rng.normal(height_mu, height_sigma)), 0.2,
                          height - 0.5))
        x = rng.uniform(0.0, size - sx)
        z = rng.uniform(0.0, size - sz)
        prims.append(Box((x, 0.0, z), (x + sx, h, z + sz),
                         tuple(rng.uniform(0.2, 0.9, 3))))
    light = PointLight((0.45 * size, 3.0 * height, 0.35 * size),
                       power=4.0 * size * size, ambient=0.15)
    return Scene(tuple(prims), light, (0.0, 0.0, 0.0), (size, height, size))


def scene_skip(scene):
    """Leading primitives that bound the scene (room walls / ground slab)
    and may contain camera positions."""
    p0 = scene.primitives[0] if scene.primitives else None
    if isinstance(p0, Box) and p0.hi[1] <= 0.0:     # ground slab (city)
        return 1
    return 6                                          # six room walls


def free_point(scene, rng, margin=0.3, tries=1000):
    """A point in the interior at least `margin` from the walls and outside
    every box/sphere (camera placement)."""
    lo = np.asarray(scene.interior_lo) + margin
    hi = np.asarray(scene.interior_hi) - margin
    for _ in range(tries):
        p = rng.uniform(lo, hi)
        ok = True
        for prim in scene.primitives[scene_skip(scene):]:
            if isinstance(prim, Box):
                if np.all(p > np.asarray(prim.lo) - 0.05) and np.all(
                        p < np.asarray(prim.hi) + 0.05):
                    ok = False
                    break
            elif np.linalg.norm(p - np.asarray(prim.center)) < prim.radius + 0.05:
                ok = False
                break
        if ok:
            return p
    raise RuntimeError("no free camera position found")


def sample_point_cloud(scene, density, seed=0):
    """Seeded surface sampling at ~`density` points per m^2 (input
    production for the point-cloud bake, in the spirit of the reference's
    `scenes.py:200-251`): every box face gets round(density * area) uniform
    points, every sphere round(density * 4 pi r^2) Gaussian-normalised
    points; colour = the primitive's albedo. Each primitive draws from its
    own stream default_rng([seed, i]). Returns a PointCloud."""
    from .pointcloud import PointCloud

    if density <= 0:
        raise ValueError("density must be positive")
    pts, cols = [], []
    for i, prim in enumerate(scene.primitives):
        rng = np.random.default_rng([seed, i])
        if isinstance(prim, Box):
            lo = np.asarray(prim.lo, np.float64)
            hi = np.asarray(prim.hi, np.float64)
            ext = hi - lo
            for ax in range(3):
                a, b = (ax + 1) % 3, (ax + 2) % 3
                n = int(round(density * ext[a] * ext[b]))
                for side in (lo[ax], hi[ax]):
                    p = np.empty((n, 3))
                    p[:, ax] = side
                    p[:, a] = lo[a] + rng.random(n) * ext[a]
                    p[:, b] = lo[b] + rng.random(n) * ext[b]
                    pts.append(p)
                    cols.append(np.broadcast_to(prim.albedo, (n, 3)))
        else:
            n = int(round(density * 4.0 * np.pi * prim.radius ** 2))
            v = rng.normal(size=(n, 3))
            v /= np.linalg.norm(v, axis=-1, keepdims=True)
            pts.append(np.asarray(prim.center) + prim.radius * v)
            cols.append(np.broadcast_to(prim.albedo, (n, 3)))
    return PointCloud(np.concatenate(pts), np.concatenate(cols).astype(np.float32))


# The reference's fixed test room (`scenes.py:249-270`: a 3 m x 2.5 m x 6 m
# room, x width, y height, z length, with two interior boxes), used by the
# acceptance-style GPU tests (`pkg/tests/test_acceptance.py`) together with
# sample_point_cloud and the point-cloud bake. Geometry only; one albedo per
# primitive (the reference's per-face wall colours do not affect tracing).
ACCEPTANCE_ROOM = (3.0, 2.5, 6.0)


def acceptance_room(with_boxes=True, extra=()):
    w, h, l = ACCEPTANCE_ROOM
    prims = [Box((0.0, 0.0, 0.0), (w, h, l), albedo=(0.5, 0.5, 0.5))]
    if with_boxes:
        prims.append(Box((0.4, 0.0, 1.0), (1.1, 0.9, 1.8), albedo=(0.0, 1.0, 1.0)))
        prims.append(Box((2.0, 0.0, 4.2), (2.7, 1.2, 5.0), albedo=(1.0, 0.0, 1.0)))
    prims.extend(extra)
    return Scene(primitives=tuple(prims), light=PointLight((w / 2, h - 0.1, l / 2)),
                 interior_lo=(0.0, 0.0, 0.0), interior_hi=(w, h, l))


def acceptance_center():
    w, h, l = ACCEPTANCE_ROOM
    return np.array([w / 2, h / 2, l / 2])
