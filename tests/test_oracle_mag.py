"""Pins of the oracle's magnified-footprint model (model = 1, row f3; the
reading of BASELINE.json's prose: "maps the pixel centre through the
fan-beam perspective ... forms the projected box-spline footprint convolved
with the detector-cell box"), against routes independent of its box-spline
code:

* its shape: the bin average of the LINEARISED projection of the pixel --
  the chord function of the square along lines perpendicular to grad P(k)
  (Liang-Barsky), mapped to the detector coordinate s = P(k) + |grad P| t --
  by piecewise Gauss-Legendre (tests/_exact.py);
* its mass: tau * sum_j W (tau = Delta_s, the bins tile the detector) equals
  the pixel's detector-integrated chord length, the 2-D integral of
  (ds/d angle)/|x - p| over the pixel, to the linearisation's O((h/delta)^2);
* parallel beam: the map is linear, so the variant equals the CNSF weight;
* the projector pair is adjoint; the CNSF model is the more accurate one.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import workloads as W
from tests import _exact as X

FAN = dict(W.FIG6, n=64, n_views=16, n_det=300, model=1)


def _grad_p(g, theta, k):
    """numerical gradient of the detector coordinate of x at k (central differences)"""
    eps = 1e-6
    gx = (oracle.perspective_project(g, theta, (k[0] + eps, k[1])) -
          oracle.perspective_project(g, theta, (k[0] - eps, k[1]))) / (2 * eps)
    gy = (oracle.perspective_project(g, theta, (k[0], k[1] + eps)) -
          oracle.perspective_project(g, theta, (k[0], k[1] - eps))) / (2 * eps)
    return np.array([gx, gy])


def _linearised_bin_average(g, theta, s, k, scale):
    h, tau = g["pixel"], g["det_width"]
    grad = _grad_p(g, theta, k)
    gn = float(np.linalg.norm(grad))
    nhat = grad / gn
    d = np.array([-nhat[1], nhat[0]])  # lines perpendicular to grad P
    sk = oracle.perspective_project(g, theta, k)
    k = np.asarray(k, dtype=float)

    def dens(sv):
        t = (sv - sk) / gn
        return scale * X.chord_square(k + t * nhat, d, k, h) / gn

    corners = [k + np.array([a * h / 2, b * h / 2]) for a in (-1, 1) for b in (-1, 1)]
    breaks = [sk + float(grad @ (c - k)) for c in corners]
    return X.bin_average(dens, s - tau / 2, s + tau / 2, breaks)


def _scale(g, theta, k):
    """(ds / d angle) / |k - p| at the pixel centre, from the geometry"""
    u = np.array([math.cos(theta), math.sin(theta)])
    p = g["sid"] * u
    r = float(np.linalg.norm(np.asarray(k) - p))
    sk = oracle.perspective_project(g, theta, k)
    if g.get("kind", 0) == 2:
        return g["sdd"] / r
    return (g["sdd"] ** 2 + sk ** 2) / (g["sdd"] * r)


@pytest.mark.parametrize("kind", [0, 2])
def test_mag_is_the_linearised_projection(kind):
    g = dict(FAN, kind=kind)
    rng = np.random.default_rng(kind)
    for _ in range(120):
        theta = rng.uniform(0, 2 * math.pi)
        k = rng.uniform(-30, 30, size=2)
        s = oracle.perspective_project(g, theta, k) + rng.uniform(-1.5, 1.5)
        want = _linearised_bin_average(g, theta, s, k, _scale(g, theta, k))
        assert oracle.weight(g, theta, s, k) == pytest.approx(want, abs=1e-7)


@pytest.mark.parametrize("kind", [0, 2])
def test_mag_mass_is_the_detector_integrated_chord(kind):
    # tau = Delta_s: the bins tile the detector
    g = dict(FAN, kind=kind, n_det=2001, det_pitch=0.5, det_width=0.5)
    c0 = 0.5 * (g["n_det"] - 1)
    xs, ws = np.polynomial.legendre.leggauss(16)
    for theta, k in ((0.4, (10.0, -20.0)), (2.0, (-25.0, 5.0)), (5.1, (0.0, 0.0))):
        sk = oracle.perspective_project(g, theta, k)
        j0, j1 = int(sk / 0.5 + c0) - 12, int(sk / 0.5 + c0) + 12
        mass = 0.5 * sum(oracle.weight(g, theta, (j - c0) * 0.5, k) for j in range(j0, j1 + 1))
        # 2-D integral of (ds/d angle)/|x - p| over the unit pixel
        u = np.array([math.cos(theta), math.sin(theta)])
        p = g["sid"] * u
        tot = 0.0
        for xi, wi in zip(xs, ws):
            for yj, wj in zip(xs, ws):
                x = np.array([k[0] + 0.5 * xi, k[1] + 0.5 * yj])
                tot += wi * wj * _scale(g, theta, x) * 0.25
        assert mass == pytest.approx(tot, rel=2e-5)  # O((h / delta)^2), delta ~ 200 mm


def test_mag_equals_cnsf_in_parallel_beam():
    g = dict(n=32, pixel=1.0, n_views=16, n_det=80, det_pitch=0.8, det_width=0.8, sid=0.0, sdd=0.0, kind=1)
    rng = np.random.default_rng(3)
    for _ in range(100):
        theta = rng.uniform(0, 2 * math.pi)
        k = rng.uniform(-10, 10, size=2)
        s = float(k @ np.array([-math.sin(theta), math.cos(theta)])) + rng.uniform(-1.5, 1.5)
        assert oracle.weight(dict(g, model=1), theta, s, k) == pytest.approx(oracle.weight(g, theta, s, k),
                                                                            abs=1e-13)


def test_mag_projector_pair_is_adjoint():
    rng = np.random.default_rng(4)
    c = rng.random((64, 64))
    y = rng.random((16, 300))
    a = float((oracle.forward(FAN, c) * y).sum())
    b = float((c * oracle.back(FAN, y)).sum())
    assert a == pytest.approx(b, rel=1e-13)


def test_cnsf_is_more_accurate_than_mag():
    # Fig. 6b setting: the paper's per-ray model tracks the exact
    # reference ~1e-4 of the peak; the pixel-linearised variant ~1e-3
    g = dict(W.FIG6, n=204)
    k = (100.5, 50.5)
    c0 = 0.5 * (g["n_det"] - 1)
    err = {0: 0.0, 1: 0.0}
    for v in range(0, 360, 15):
        th = 2 * math.pi * v / 360
        sk = oracle.perspective_project(g, th, k)
        for j in range(int(sk / 0.5 + c0) - 4, int(sk / 0.5 + c0) + 5):
            s = (j - c0) * 0.5
            ref = oracle.ref_weight(g, th, s, k)
            for model in (0, 1):
                err[model] = max(err[model], abs(oracle.weight(dict(g, model=model), th, s, k) - ref))
    assert err[0] < 1e-3 and err[0] < err[1] < 5e-2


def test_candidate_window_is_a_superset_close_source():
    """The model's support is |s - P(k)| < (h(|dP/dx| + |dP/dy|) + tau)/2, which
    for a source close to the field of view reaches past the perspective
    images of the pixel corners; widening the candidate window must not
    change the projection (any superset is exact).  This
    geometry (source 1.23 field radii away, narrow bins) found the gap."""
    g = dict(n=10, pixel=1.069340183528383, n_views=120, n_det=54, det_pitch=0.39025943122344087,
             det_width=0.0819854190161896, sid=9.339360648764503, sdd=13.032752470587264, kind=0, model=1)
    img = W.random_image(10, 1348).astype(np.float64)
    base = oracle.forward(g, img)
    y = W.random_sino(120, 54, 1349).astype(np.float64)
    base_b = oracle.back(g, y)
    try:
        oracle.set_candidate_margin_scale(25.0)
        wide = oracle.forward(g, img)
        wide_b = oracle.back(g, y)
    finally:
        oracle.set_candidate_margin_scale(1.0)
    np.testing.assert_array_equal(base, wide)
    np.testing.assert_array_equal(base_b, wide_b)
