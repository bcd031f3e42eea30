"""Pins of the oracle's reference projector "Ref" (row f2): the
exact fan-beam chord of the indicator pixel (Eq. 10) averaged over the
detector bin.  Each pin reaches the value by a route independent of
oracle/cnsf_oracle.c (ref_*):

* the chord against Liang-Barsky clipping in tests/_exact.py;
* the bin average against piecewise Gauss-Legendre-24 in tests/_exact.py
  (the oracle uses adaptive Simpson);
* the detector integral of the chord against the change of variables
  x = p + t (q(s) - p):  integral chord(s) ds = integral over the pixel of
  (D_ps^2 + s(x)^2) / (D_ps |x - p|) dA  (dA = t D_ps ds dt), by 2-D
  Gauss-Legendre over the square;
* the projector against a brute-force sum of per-bin weights.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import workloads as W
from tests import _exact as X

GEOMS = {
    "fig6": W.FIG6,
    "fig5": W.FIG5,
    "cfg1": W.geometry("1"),
    "fig7": W.FIG7,
}


def _rng_cases(g, count, seed):
    rng = np.random.default_rng(seed)
    half = 0.5 * g["n"] * g["pixel"]
    for _ in range(count):
        theta = rng.uniform(0, 2 * math.pi)
        k = rng.uniform(-half, half, size=2) * 0.9
        s_k = X.project_point(g, theta, k)
        s = s_k + rng.uniform(-1.5, 1.5) * (g["pixel"] * 2 + g["det_width"])
        yield theta, s, k


@pytest.mark.parametrize("name", list(GEOMS))
def test_ref_chord_is_liang_barsky(name):
    g = GEOMS[name]
    for theta, s, k in _rng_cases(g, 300, 11):
        want = X.ray_chord_square(g, theta, s, k, g["pixel"])
        assert oracle.ref_chord(g, theta, s, k) == pytest.approx(want, abs=1e-12 * g["pixel"])


@pytest.mark.parametrize("name", list(GEOMS))
def test_ref_weight_is_piecewise_gauss_legendre(name):
    g = GEOMS[name]
    for theta, s, k in _rng_cases(g, 150, 12):
        want = X.exact_pixel_bin(g, theta, s, k)
        got = oracle.ref_weight(g, theta, s, k)
        assert got == pytest.approx(want, abs=1e-11 * g["pixel"]), (theta, s, k)


def _pixel_mass_2d(g, theta, k, m=24):
    """integral of (D_ps^2 + s(x)^2) / (D_ps |x - p|) over the pixel (2-D GL)."""
    xs, ws = np.polynomial.legendre.leggauss(m)
    hh = 0.5 * g["pixel"]
    u = np.array([math.cos(theta), math.sin(theta)])
    p = g["sid"] * u
    tot = 0.0
    for xi, wi in zip(xs, ws):
        for yj, wj in zip(xs, ws):
            x = np.array([k[0] + hh * xi, k[1] + hh * yj])
            s = X.project_point(g, theta, x)
            r = float(np.linalg.norm(x - p))
            tot += wi * wj * (g["sdd"] ** 2 + s * s) / (g["sdd"] * r)
    return tot * hh * hh


@pytest.mark.parametrize("theta", [0.0, 0.37, 1.2, 2.9, 4.4])
@pytest.mark.parametrize("k", [(0.0, 0.0), (100.5, 50.5), (-37.0, 81.25)])
def test_ref_detector_integral_is_change_of_variables(theta, k):
    # tau = Delta_s: the bins tile the detector, so tau * sum_j W_ref(j) is the
    # integral of the chord over the whole shadow
    g = dict(W.FIG6, n=256, n_det=4001, det_pitch=0.5, det_width=0.5)
    c0 = 0.5 * (g["n_det"] - 1)
    corners = [(k[0] + a * 0.5, k[1] + b * 0.5) for a in (-1, 1) for b in (-1, 1)]
    ss = [X.project_point(g, theta, c) for c in corners]
    j0 = max(0, int(math.floor(min(ss) / g["det_pitch"] + c0)) - 2)
    j1 = min(g["n_det"] - 1, int(math.ceil(max(ss) / g["det_pitch"] + c0)) + 2)
    total = sum(oracle.ref_weight(g, theta, (j - c0) * g["det_pitch"], k) for j in range(j0, j1 + 1))
    total *= g["det_width"]
    assert total == pytest.approx(_pixel_mass_2d(g, theta, k), rel=1e-11)


def test_ref_forward_is_sum_of_weights():
    g = dict(W.geometry("1"), n=5, n_views=7, n_det=24, pixel=3.0, det_pitch=2.5, det_width=1.7)
    rng = np.random.default_rng(5)
    img = rng.random((5, 5))
    img[1, 3] = 0.0
    y = oracle.ref_forward(g, img)
    want = np.zeros_like(y)
    c0 = 0.5 * (g["n_det"] - 1)
    for v in range(g["n_views"]):
        th = 2 * math.pi * v / g["n_views"]
        for j in range(g["n_det"]):
            s = (j - c0) * g["det_pitch"]
            for r in range(5):
                for c in range(5):
                    k = oracle.pixel_center(g, r, c)
                    want[v, j] += img[r, c] * oracle.ref_weight(g, th, s, k)
    np.testing.assert_allclose(y, want, rtol=1e-13, atol=1e-13)


def test_ref_close_to_cnsf_in_the_papers_setting():
    # P:459-463 (Fig. 6 a): pixel at the origin, D_po = D_so = 200 mm, tau = 0.5:
    # the effective-blur model (Eq. 14) is a close approximation of Ref
    g = W.FIG6
    c0 = 0.5 * (g["n_det"] - 1)
    worst = 0.0
    for v in range(0, 90, 7):
        th = math.radians(v)
        for j in range(int(c0) - 4, int(c0) + 5):
            s = (j - c0) * g["det_pitch"]
            worst = max(worst, abs(oracle.weight(g, th, s, (0, 0)) - oracle.ref_weight(g, th, s, (0, 0))))
    assert worst < 1e-3  # of a peak ~1 mm
