"""Independent exact references used to PIN the oracle (never the oracle itself).

The scanner conventions are the DESIGN.md ledger readings restated (source
p = D_po u, detector line through -D_so u along e = (-sin, cos), bin centres
(j - (N_s-1)/2) Delta_s); the arithmetic is a different route from the
paper's box-spline formulas:

* ``chord_square``: Liang-Barsky clipping of a line against an axis-aligned
  square (the exact line integral of an indicator pixel, which Eq. 12 claims
  to reproduce);
* ``bin_average``: the paper's reference projector: the exact
  footprint averaged over the detector bin (unit-mass blur, ledger #3),
  integrated piecewise by Gauss-Legendre between the projected corners, where
  the integrand is smooth;
* ``chord_disk``: analytic chord of a line through a disk.
"""
from __future__ import annotations

import math

import numpy as np

_GL_X, _GL_W = np.polynomial.legendre.leggauss(24)


def frame(geom: dict, theta: float):
    u = np.array([math.cos(theta), math.sin(theta)])
    e = np.array([-u[1], u[0]])
    p = geom["sid"] * u
    dso = geom["sdd"] - geom["sid"]
    return u, e, p, dso


def det_point(geom, theta, s):
    u, e, p, dso = frame(geom, theta)
    return -dso * u + s * e


def chord_square(a: np.ndarray, d: np.ndarray, center, side: float) -> float:
    """length of {a + t d} inside the square of the given centre and side."""
    d = d / np.linalg.norm(d)
    t0, t1 = -np.inf, np.inf
    for ax in range(2):
        lo = center[ax] - side / 2.0
        hi = center[ax] + side / 2.0
        if abs(d[ax]) < 1e-300:
            if a[ax] < lo or a[ax] > hi:
                return 0.0
            continue
        ta = (lo - a[ax]) / d[ax]
        tb = (hi - a[ax]) / d[ax]
        if ta > tb:
            ta, tb = tb, ta
        t0, t1 = max(t0, ta), min(t1, tb)
    return max(0.0, t1 - t0)


def chord_disk(a: np.ndarray, d: np.ndarray, center, radius: float) -> float:
    d = d / np.linalg.norm(d)
    w = np.asarray(center, dtype=float) - a
    dist2 = float(w @ w - (w @ d) ** 2)
    return 2.0 * math.sqrt(radius * radius - dist2) if dist2 < radius * radius else 0.0


def ray_chord_square(geom, theta, s, center, side):
    u, e, p, dso = frame(geom, theta)
    q = det_point(geom, theta, s)
    return chord_square(p, q - p, center, side)


def project_point(geom, theta, x):
    """detector coordinate where the line from the source through x lands."""
    u, e, p, dso = frame(geom, theta)
    x = np.asarray(x, dtype=float)
    # intersect p + t (x - p) with the detector line {-dso u + s e}
    dvec = x - p
    t = (-(dso) - p @ u) / (dvec @ u)
    hit = p + t * dvec
    return float((hit + dso * u) @ e)


def bin_average(f_of_s, lo: float, hi: float, breaks) -> float:
    """(1/(hi-lo)) * integral_lo^hi f(s) ds, piecewise Gauss-Legendre-24."""
    pts = sorted([lo, hi] + [b for b in breaks if lo < b < hi])
    total = 0.0
    for a, b in zip(pts[:-1], pts[1:]):
        mid, half = 0.5 * (a + b), 0.5 * (b - a)
        total += half * sum(w * f_of_s(mid + half * x) for x, w in zip(_GL_X, _GL_W))
    return total / (hi - lo)


def exact_pixel_bin(geom, theta, s, center, side=None):
    """reference projector for one pixel and one bin."""
    side = geom["pixel"] if side is None else side
    tau = geom["det_width"]
    cx, cy = center
    corners = [(cx + sx * side / 2, cy + sy * side / 2) for sx in (-1, 1) for sy in (-1, 1)]
    breaks = [project_point(geom, theta, c) for c in corners]
    return bin_average(lambda t: ray_chord_square(geom, theta, t, center, side),
                       s - tau / 2, s + tau / 2, breaks)
