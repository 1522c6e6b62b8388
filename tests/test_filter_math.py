"""The identities the CUDA decision filters rest on (DESIGN.md §5,
`csrc/lfp_trace.cuh` ChordF / radii_classify / dda_init_hi), checked on the
CPU against the oracle's restatement of the reference functions:

* every radius of a ray point is sqrt((t - t*)^2 + rperp^2);
* `distance_to_intersection` (kernels.py:62-81) is the radius at
  t_v = ((w.v)(d.v) + t*) / (1 - (d.v)^2) for unit d, v;
* the quotient a / b follows bit for bit from the correctly rounded
  reciprocal of b by q0 = a y, r = fma(-b, q0, a), q = fma(y, r, q0)
  (Markstein), including the exactly scaled reciprocal (1 / (b / 4)) / 4."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle


def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def test_radius_from_ray_parameter():
    rng = np.random.default_rng(3)
    n = 2000
    w = rng.normal(size=(n, 3)) * 10.0 ** rng.uniform(-2, 1, (n, 1))
    d = _unit(rng.normal(size=(n, 3)))
    t = rng.uniform(0.0, 20.0, n)
    tstar = -np.einsum("ij,ij->i", w, d)
    rp2 = np.einsum("ij,ij->i", w, w) - tstar ** 2
    r_ref = np.linalg.norm(w + t[:, None] * d, axis=1)
    r_t = np.sqrt((t - tstar) ** 2 + rp2)
    np.testing.assert_allclose(r_t, r_ref, rtol=1e-9, atol=1e-12)


def test_d2i_is_a_ray_radius_at_the_closest_approach_parameter():
    rng = np.random.default_rng(4)
    n = 500
    w = rng.normal(size=(n, 3)) * 3.0
    d = _unit(rng.normal(size=(n, 3)))
    v = _unit(rng.normal(size=(n, 3)))
    tstar = -np.einsum("ij,ij->i", w, d)
    rp2 = np.einsum("ij,ij->i", w, w) - tstar ** 2
    wv = np.einsum("ij,ij->i", w, v)
    dv = np.einsum("ij,ij->i", d, v)
    den = 1.0 - dv * dv
    ok = den > 1e-4
    tv = (wv * dv + tstar) / den
    r_t = np.sqrt((tv - tstar) ** 2 + rp2)
    ref = np.array([oracle.distance_to_intersection(w[i], d[i], v[i])
                    for i in range(n)])
    np.testing.assert_allclose(r_t[ok], ref[ok], rtol=1e-7, atol=1e-10)
    assert ok.mean() > 0.99


def _fma(a, b, c):
    """Correctly rounded a * b + c for finite doubles."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


@pytest.mark.parametrize("scaled", [False, True])
def test_markstein_quotient_from_rounded_reciprocal(scaled):
    rng = np.random.default_rng(5)
    n = 3000
    a = rng.uniform(-1.0, 1.0, n)          # n - q: distance to the next texel edge
    b = rng.normal(size=n) * 10.0 ** rng.uniform(-6, 3, n)   # sdu
    a[:50] = 0.0
    bad = 0
    for x, y in zip(a.tolist(), b.tolist()):
        rec = (1.0 / (y * 0.25)) * 0.25 if scaled else 1.0 / y
        q0 = x * rec
        r = _fma(-y, q0, x)
        q = _fma(rec, r, q0)
        # (the Fraction emulation of fma cannot produce -0; the sign of a
        # zero quotient is covered by the GPU self-test)
        if x == 0.0:
            bad += q != 0.0
        else:
            bad += np.float64(q).tobytes() != np.float64(x / y).tobytes()
    assert bad == 0
