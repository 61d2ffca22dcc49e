"""The fast strip kernel's RK4 algebra for heat3d, checked on the CPU.

heat_strip.cuh evaluates one RK4 step of the linear field L = kk (S - 6), S the
sum of the six ghost-substituted neighbours, as the polynomial
P(z(S - 6)) = q0 + q1 S + q2 S^2 + q3 S^3 + q4 S^4 (z = hk kk) in the form
w1 = S x + (q3/q4) x, w2 = S w1 + (q2/q4) x, w3 = S w2 + (q1/q4) x,
y = q4 S w3 + q0 x  (heat.cuh heat_sform_coeffs).  These tests restate that
evaluation in float64 numpy and compare it with the oracle's RK4
(rk4.cpp:30-76 on models.cpp:92-133) -- pinning the algebra, including the
ghost substitution at the Robin and insulated faces, independently of the GPU.
"""
import numpy as np
import pytest

import paper_2001_10635_b200 as pk
from oracle import oracle as O


def sform_coeffs(z):
    """heat.cuh heat_sform_coeffs (long double on the host)."""
    Z = np.longdouble(z)
    q4 = Z ** 4 / 24
    q3 = Z ** 3 * (1 - 6 * Z) / 6
    q2 = Z ** 2 * (1 - 6 * Z + 18 * Z ** 2) / 2
    q1 = Z * (1 - 6 * Z + 18 * Z ** 2 - 36 * Z ** 3)
    q0 = 1 - 6 * Z + 18 * Z ** 2 - 36 * Z ** 3 + 54 * Z ** 4
    return [np.float64(v) for v in (q3 / q4, q2 / q4, q1 / q4, q4, q0)]


def neighbour_sum(v, robin):
    """S with the kernel's ghost values: insulated faces mirror the centre,
    the x = 0 face has the Robin ghost x(1) - robin x(0) (models.cpp:113-119).
    v is indexed [z, y, x] (component i = x + g y + g^2 z)."""
    p = np.pad(v, 1, mode="edge")
    s = (p[:-2, 1:-1, 1:-1] + p[2:, 1:-1, 1:-1]) + (p[1:-1, :-2, 1:-1] + p[1:-1, 2:, 1:-1])
    xm = p[1:-1, 1:-1, :-2].copy()
    xp = p[1:-1, 1:-1, 2:]
    xm[:, :, 0] = xp[:, :, 0] - robin * v[:, :, 0]
    return s + (xm + xp)


def sform_step(x, z, robin):
    a1, a2, a3, q4, q0 = sform_coeffs(z)
    w = neighbour_sum(x, robin) + a1 * x
    w = neighbour_sum(w, robin) + a2 * x
    w = neighbour_sum(w, robin) + a3 * x
    return q4 * neighbour_sum(w, robin) + q0 * x


@pytest.mark.parametrize("g,z,steps", [(6, 0.2, 3), (9, 1.0 / 6.0, 2), (12, 0.0319, 5), (8, 2e-6, 2)])
def test_sform_matches_reference_rk4(g, z, steps):
    m = pk.make_heat3d(g)
    delta = 1.0 / (g - 1)
    kk = 1.0 / (delta * delta)
    robin = 2.0 * delta * 1.0
    h = z / kk
    n = g ** 3
    rng = np.random.default_rng(g)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    ref = O.mixed_monotonicity(m, lo, hi, None, None, 0.0, steps * h, h, 0)
    for x0, r in ((lo, ref.lower[-1]), (hi, ref.upper[-1])):
        x = x0.reshape(g, g, g)
        for k in range(steps):
            x = sform_step(x, h * kk, robin)
        got = x.reshape(-1)
        assert np.max(np.abs(got - r) / np.abs(r)) <= 1e-13


def test_sform_coefficients_reproduce_rk4_polynomial():
    """sum_k q_k s^k equals the RK4 polynomial 1 + u + u^2/2 + u^3/6 + u^4/24 at
    u = z (s - 6) for scalar s (the stencil's eigen-relation)."""
    for z in (1e-5, 0.01, 0.128, 1.0 / 6.0, 0.23):
        a1, a2, a3, q4, q0 = sform_coeffs(z)
        for s in (-6.0, 0.0, 3.0, 6.0):
            u = z * (s - 6.0)
            want = 1 + u + u * u / 2 + u ** 3 / 6 + u ** 4 / 24
            got = q4 * (s ** 4 + a1 * s ** 3 + a2 * s ** 2 + a3 * s) + q0
            assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
