"""Row f3 (arc detector, "the extension to the arc geometry is easily
obtained as a special case"): pins of the oracle's kind = 2 mode, where the
detector is the circle of radius D_ps about the source and s is arc length.

* the detector point of P(x) is collinear with the source and x, and lies
  at distance D_ps from the source;
* ray identity: the arc ray at angle gamma IS the flat-detector ray at
  s = D_ps tan(gamma), so the unblurred footprints (Eq. 12) agree exactly;
* Eq. 13 on the arc in closed form: the bin subtends tau / D_ps at the
  source symmetrically about its central ray, so tau'(k) = 2 d tan(tau / 2 D_ps)
  with d = (k - p).v the pixel depth along the ray;
* the reference chord against Liang-Barsky with an independently built ray;
* adjointness of the projector pair.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
from tests import _exact as X

ARC = dict(n=48, pixel=1.0, n_views=20, n_det=140, det_pitch=0.9, det_width=0.7, sid=60.0, sdd=120.0,
           kind=2)
FLAT = dict(ARC, kind=0)


def _frame(theta):
    u = np.array([math.cos(theta), math.sin(theta)])
    return u, np.array([-u[1], u[0]])


def _cases(count, seed):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        theta = rng.uniform(0, 2 * math.pi)
        k = rng.uniform(-16, 16, size=2)
        yield theta, k, rng


def test_projection_is_collinear_at_radius_dps():
    for theta, k, _ in _cases(100, 1):
        s = oracle.perspective_project(ARC, theta, k)
        q = oracle.detector_point(ARC, theta, s)
        u, e = _frame(theta)
        p = ARC["sid"] * u
        assert np.linalg.norm(q - p) == pytest.approx(ARC["sdd"], rel=1e-13)
        a, b = q - p, np.asarray(k) - p
        assert abs(a[0] * b[1] - a[1] * b[0]) <= 1e-10 * np.linalg.norm(a) * np.linalg.norm(b)
        assert a @ b > 0


def test_arc_ray_is_the_flat_ray_at_dps_tan_gamma():
    for theta, k, rng in _cases(200, 2):
        s = oracle.perspective_project(ARC, theta, k) + rng.uniform(-1.5, 1.5)
        s_flat = ARC["sdd"] * math.tan(s / ARC["sdd"])
        assert oracle.footprint(ARC, theta, s, k) == pytest.approx(oracle.footprint(FLAT, theta, s_flat, k),
                                                                  abs=1e-12)


def test_effective_blur_closed_form_on_the_arc():
    for theta, k, rng in _cases(200, 3):
        s = rng.uniform(-50, 50)
        u, e = _frame(theta)
        p = ARC["sid"] * u
        gam = s / ARC["sdd"]
        v = -math.cos(gam) * u + math.sin(gam) * e  # unit direction of the bin-centre ray
        d = float((np.asarray(k) - p) @ v)
        want = 2.0 * d * math.tan(ARC["det_width"] / (2.0 * ARC["sdd"]))
        assert oracle.effective_blur(ARC, theta, s, k) == pytest.approx(want, rel=1e-12)


def test_reference_chord_on_the_arc():
    for theta, k, rng in _cases(200, 4):
        s = oracle.perspective_project(ARC, theta, k) + rng.uniform(-1.0, 1.0)
        u, e = _frame(theta)
        p = ARC["sid"] * u
        gam = s / ARC["sdd"]
        d = -math.cos(gam) * u + math.sin(gam) * e
        want = X.chord_square(p, d, k, ARC["pixel"])
        assert oracle.ref_chord(ARC, theta, s, k) == pytest.approx(want, abs=1e-12)


def test_arc_projector_pair_is_adjoint():
    rng = np.random.default_rng(5)
    c = rng.random((48, 48))
    y = rng.random((20, 140))
    a = float((oracle.forward(ARC, c) * y).sum())
    b = float((c * oracle.back(ARC, y)).sum())
    assert a == pytest.approx(b, rel=1e-13)


def test_arc_cnsf_close_to_reference():
    # the effective-blur model on the arc is as close to the exact bin average
    # as on the flat detector (a special case of the same construction)
    rng = np.random.default_rng(6)
    c = rng.random((48, 48))
    ya, ra = oracle.forward(ARC, c, 0, 4), oracle.ref_forward(ARC, c, 0, 4)
    yf, rf = oracle.forward(FLAT, c, 0, 4), oracle.ref_forward(FLAT, c, 0, 4)
    ea = np.abs(ya - ra).max() / np.abs(ra).max()
    ef = np.abs(yf - rf).max() / np.abs(rf).max()
    assert ea < 5e-3 and ef < 5e-3
