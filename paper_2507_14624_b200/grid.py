"""Probe containers with the reference's array layout.

`MapChain`, `ProbeData`, `ProbeSet` and `ProbeGrid` mirror
`pkg/src/lfprobe/octmap.py:93-129`, `bake.py:45-59` and `grid.py:19-93`:
the same constructor arguments, attribute names, dtypes, shapes and
validation errors. They are the host-side source of the device upload
(`lfp_probeset_create`, see `include/lfprobe_b200.h`).

Layout (reference, C-contiguous):
  dist_hi f32 (P, R, R) [ty, tx], EMPTY = +inf
  dir_hi  f32 (P, R, R, 3)        probe -> surface direction, 0 if EMPTY
  irr_hi  f32 (P, R, R, 3)        radiance, 0 if EMPTY
  dist_lo f32 (P, r, r)           block MIN of dist_hi
  origins f64 (P, 3)
Probe (i, j, k) of a grid sits at grid_origin + cell * (i, j, k); flat index
(i * ny + j) * nz + k (`grid.py:48-74`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class MapChain:
    """Five octahedral maps of one probe (`octmap.py:93-129`)."""

    irradiance_hi: np.ndarray
    distance_hi: np.ndarray
    direction_hi: np.ndarray
    distance_lo: np.ndarray
    direction_lo: np.ndarray | None = None

    def __post_init__(self):
        if self.res_hi % self.res_lo != 0:
            raise ValueError(
                "high resolution must be a multiple of low resolution")
        for arr in (self.irradiance_hi, self.distance_hi, self.direction_hi,
                    self.distance_lo):
            if arr.shape[0] != arr.shape[1]:
                raise ValueError("octahedral maps must be square")

    @property
    def res_hi(self) -> int:
        return self.distance_hi.shape[0]

    @property
    def res_lo(self) -> int:
        return self.distance_lo.shape[0]

    @property
    def factor(self) -> int:
        return self.res_hi // self.res_lo


@dataclass(frozen=True)
class ProbeData:
    """One probe: origin, map chain, bake metadata (`bake.py:45-59`)."""

    origin: np.ndarray
    chain: MapChain
    bounds_lo: np.ndarray = None
    bounds_hi: np.ndarray = None
    source: str = ""
    point_count: int = 0
    timestamp: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "origin",
                           np.asarray(self.origin, dtype=np.float64))


class ProbeSet:
    """Probes stacked into dense arrays (`grid.py:19-45`)."""

    def __init__(self, probes=None, *, arrays=None):
        if arrays is not None:
            dist_hi, dir_hi, irr_hi, dist_lo, origins = arrays
            self.probes = None
            self.dist_hi = np.ascontiguousarray(dist_hi, dtype=np.float32)
            self.dir_hi = np.ascontiguousarray(dir_hi, dtype=np.float32)
            self.irr_hi = np.ascontiguousarray(irr_hi, dtype=np.float32)
            self.dist_lo = np.ascontiguousarray(dist_lo, dtype=np.float32)
            self.origins = np.ascontiguousarray(origins, dtype=np.float64)
        else:
            chains = [p.chain for p in probes]
            res = {(c.res_hi, c.res_lo) for c in chains}
            if len(res) != 1:
                raise ValueError("all probes must share the same resolutions")
            self.probes = list(probes)
            self.dist_hi = np.stack([c.distance_hi for c in chains])
            self.dir_hi = np.stack([c.direction_hi for c in chains])
            self.irr_hi = np.stack([c.irradiance_hi for c in chains])
            self.dist_lo = np.stack([c.distance_lo for c in chains])
            self.origins = np.stack([p.origin for p in probes])
        self._check()

    def _check(self):
        p, r, r2 = self.dist_hi.shape
        if r != r2:
            raise ValueError("octahedral maps must be square")
        if self.dir_hi.shape != (p, r, r, 3) or self.irr_hi.shape != (p, r, r, 3):
            raise ValueError("direction/irradiance maps must be (P, R, R, 3)")
        pl, rl, rl2 = self.dist_lo.shape
        if pl != p or rl != rl2 or r % rl != 0:
            raise ValueError("low-res maps must be (P, r, r) with r | R")
        if self.origins.shape != (p, 3):
            raise ValueError("origins must be (P, 3)")

    @property
    def n_probes(self):
        return self.dist_hi.shape[0]

    @property
    def res_hi(self):
        return self.dist_hi.shape[1]

    @property
    def res_lo(self):
        return self.dist_lo.shape[1]

    @property
    def bounds(self):
        """Union of the probes' bake bounds (`grid.py:41-45`); probe sets
        built from bare arrays fall back to the origins' box."""
        probes = self.probes or []
        if probes and all(getattr(p, "bounds_lo", None) is not None
                          for p in probes):
            lo = np.min([p.bounds_lo for p in probes], axis=0)
            hi = np.max([p.bounds_hi for p in probes], axis=0)
            return lo, hi
        return self.origins.min(axis=0), self.origins.max(axis=0)

    @property
    def nbytes(self):
        return sum(a.nbytes for a in (self.dist_hi, self.dir_hi, self.irr_hi,
                                      self.dist_lo, self.origins))


class ProbeGrid:
    """Probes at the vertices of a uniform lattice of cubes
    (`grid.py:48-93`). `probes` is a list of ProbeData, or pass
    `probe_set=` with stacked arrays (large configurations)."""

    def __init__(self, grid_origin, cell_size, dims, probes=None, *,
                 probe_set: ProbeSet | None = None):
        self.grid_origin = np.asarray(grid_origin, dtype=np.float64)
        self.cell_size = float(cell_size)
        self.dims = tuple(int(d) for d in dims)
        nx, ny, nz = self.dims
        if nx < 1 or ny < 1 or nz < 1:
            raise ValueError("grid dims must be >= 1 per axis")
        count = probe_set.n_probes if probe_set is not None else len(probes)
        if count != nx * ny * nz:
            raise ValueError("probe count does not match grid dims")
        self.probes = list(probes) if probes is not None else None
        self._set = probe_set
        origins = (self.probe_set.origins if probes is None else
                   np.stack([p.origin for p in self.probes]))
        ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz),
                                 indexing="ij")
        expect = self.grid_origin + self.cell_size * np.stack(
            [ii.ravel(), jj.ravel(), kk.ravel()], axis=-1).astype(np.float64)
        bad = np.max(np.abs(origins - expect), axis=-1) > 1e-6
        if bad.any():
            f = int(np.flatnonzero(bad)[0])
            i, j, k = np.unravel_index(f, (nx, ny, nz))
            raise ValueError(f"probe ({i},{j},{k}) is off-lattice")

    def probe(self, i, j, k):
        nx, ny, nz = self.dims
        return self.probes[(i * ny + j) * nz + k]

    @property
    def probe_set(self) -> ProbeSet:
        if self._set is None:
            self._set = ProbeSet(self.probes)
        return self._set

    @property
    def n_cubes(self):
        nx, ny, nz = self.dims
        return (max(nx - 1, 1), max(ny - 1, 1), max(nz - 1, 1))

    def cube_bounds(self, cube):
        lo = self.grid_origin + self.cell_size * np.asarray(cube, dtype=float)
        return lo, lo + self.cell_size

    @property
    def bounds(self):
        return self.probe_set.bounds


class ProbeHierarchy:
    """Coarse-to-fine stack of probe grids (BASELINE config 4; no reference
    counterpart): a ray is traced through level 0 and falls through to the
    next level on MISS (`lfp_render_hierarchy`)."""

    def __init__(self, levels):
        self.levels = list(levels)
        if not 1 <= len(self.levels) <= 4:
            raise ValueError("a hierarchy has 1..4 levels")

    @property
    def n_probes(self):
        return sum(g.probe_set.n_probes for g in self.levels)
