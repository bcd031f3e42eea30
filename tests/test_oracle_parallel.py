"""Row f3 (parallel beam, Eq. 9-10 and Theorem 1): pins of the
oracle's parallel-beam mode (kind = 1) against values fixed independently:

* Theorem 1: with parallel rays the blurred footprint IS a 3-direction box
  spline, i.e. it equals the exact chord of the indicator pixel averaged over
  the bin -- checked against Liang-Barsky clipping of parallel lines and
  piecewise Gauss-Legendre (tests/_exact.py), not the oracle's box splines;
* the fan-beam weight tends to it as the source recedes (magnification 1);
* theta + pi flips the detector axis: W(theta + pi, s, k) = W(theta, -s, k);
* the projector pair is adjoint.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
from tests import _exact as X

PAR = dict(n=32, pixel=1.0, n_views=16, n_det=80, det_pitch=0.8, det_width=0.8, sid=0.0, sdd=0.0,
           kind=1)


def _parallel_exact(g, theta, s, k):
    u = np.array([math.cos(theta), math.sin(theta)])
    e = np.array([-u[1], u[0]])
    hh = 0.5 * g["pixel"]
    corners = [np.array([k[0] + a * hh, k[1] + b * hh]) for a in (-1, 1) for b in (-1, 1)]
    breaks = [float(c @ e) for c in corners]  # orthogonal projection onto the detector axis
    tau = g["det_width"]
    return X.bin_average(lambda t: X.chord_square(t * e, u, k, g["pixel"]), s - tau / 2, s + tau / 2,
                         breaks)


@pytest.mark.parametrize("width", [0.3, 0.8, 2.5])
def test_parallel_weight_is_exact_bin_average(width):
    g = dict(PAR, det_width=width)
    rng = np.random.default_rng(int(width * 10))
    for _ in range(200):
        theta = rng.uniform(0, 2 * math.pi)
        k = rng.uniform(-10, 10, size=2)
        s = float(k @ np.array([-math.sin(theta), math.cos(theta)])) + rng.uniform(-1.6, 1.6)
        want = _parallel_exact(g, theta, s, k)
        assert oracle.weight(g, theta, s, k) == pytest.approx(want, abs=1e-12)


def test_fan_tends_to_parallel():
    rng = np.random.default_rng(9)
    for R in (1e5, 1e7):
        fan = dict(PAR, kind=0, sid=R, sdd=2 * R, det_pitch=1.6, det_width=1.6)
        for _ in range(50):
            theta = rng.uniform(0, 2 * math.pi)
            k = rng.uniform(-10, 10, size=2)
            s = float(k @ np.array([-math.sin(theta), math.cos(theta)])) + rng.uniform(-1.2, 1.2)
            # detector coordinate and bin width scale with the magnification 2
            w_fan = oracle.weight(fan, theta, 2 * s, k)
            w_par = oracle.weight(PAR, theta, s, k)
            # the pixels sit up to 14 mm off the rotation centre: magnification 2 (1 +- 14/R)
            assert w_fan == pytest.approx(w_par, abs=500.0 / R)


def test_half_turn_flips_the_detector():
    rng = np.random.default_rng(4)
    for _ in range(100):
        theta = rng.uniform(0, math.pi)
        k = rng.uniform(-10, 10, size=2)
        s = rng.uniform(-12, 12)
        assert oracle.weight(PAR, theta + math.pi, s, k) == pytest.approx(oracle.weight(PAR, theta, -s, k),
                                                                          abs=1e-12)


def test_parallel_projector_pair_is_adjoint():
    rng = np.random.default_rng(1)
    c = rng.random((32, 32))
    y = rng.random((16, 80))
    a = float((oracle.forward(PAR, c) * y).sum())
    b = float((c * oracle.back(PAR, y)).sum())
    assert a == pytest.approx(b, rel=1e-13)


def test_parallel_forward_matches_ref_forward():
    # Theorem 1 at the projector level: CNSF == Ref for parallel rays
    rng = np.random.default_rng(2)
    c = rng.random((32, 32))
    np.testing.assert_allclose(oracle.forward(PAR, c), oracle.ref_forward(PAR, c), rtol=1e-11, atol=1e-11)
