"""Two more pins of the oracle from BASELINE.json's north_star ("brute-force
fine ray-sampling integration on tiny images", "analytic line integrals of
... a disk phantom"), by routes that share nothing with its box-spline code:

* brute force: each bin's value is the average, over K equally spaced
  sub-rays across the bin (midpoint rule), of the exact line integral of
  the pixel image along the sub-ray -- the sum over pixels of the chord the
  ray cuts through each square (vectorised Liang-Barsky, restated here).
  That is the reference projector by plain sampling; where no
  ray runs parallel to a pixel edge the integrand is continuous and
  piecewise smooth and the sampling error falls as O(K^-2) (with rays along
  an edge, at 0 and 90 degrees, the chord jumps across the edge's thin
  perspective ramp and it falls as O(K^-1) until K resolves the ramp), and
  CNSF must sit within its effective-blur error of it (~1.7e-4
  of peak in the config-1 geometry);
* disk: a disk's area-weighted pixel image, projected by the oracle,
  approaches the disk's analytic bin-averaged chord as the grid refines;
  the discretisation error is O(h) (the pixelated boundary), so it must
  roughly halve each time n doubles at a fixed field of view.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle as O
import workloads as W
from tests import _exact as X


def _chords(p, dirs, centers, h):
    """[R, P] chord lengths of the rays p + t dirs[r] through the squares of
    side h centred at centers[k] (Liang-Barsky, vectorised)."""
    d = dirs / np.linalg.norm(dirs, axis=1, keepdims=True)
    t0 = np.full((len(d), len(centers)), -np.inf)
    t1 = np.full((len(d), len(centers)), np.inf)
    for ax in range(2):
        lo = centers[None, :, ax] - h / 2 - p[ax]
        hi = centers[None, :, ax] + h / 2 - p[ax]
        da = d[:, ax:ax + 1]
        with np.errstate(divide="ignore", invalid="ignore"):
            ta, tb = lo / da, hi / da
        tmin, tmax = np.minimum(ta, tb), np.maximum(ta, tb)
        par = np.abs(da) < 1e-300  # parallel to this axis: inside the slab or not
        inside = (lo <= 0) & (hi >= 0)
        tmin = np.where(par, np.where(inside, -np.inf, np.inf), tmin)
        tmax = np.where(par, np.where(inside, np.inf, -np.inf), tmax)
        t0, t1 = np.maximum(t0, tmin), np.minimum(t1, tmax)
    return np.maximum(0.0, t1 - t0)


def _brute_force(g, img, views, K):
    n, h = g["n"], g["pixel"]
    c = 0.5 * (n - 1)
    rows, cols = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    centers = np.stack([(cols - c) * h, (c - rows) * h], axis=-1).reshape(-1, 2)
    vals = img.reshape(-1).astype(np.float64)
    tau = g["det_width"]
    off = ((np.arange(K) + 0.5) / K - 0.5) * tau
    out = np.zeros((len(views), g["n_det"]))
    for iv, v in enumerate(views):
        th = O.view_angle(g, v)
        u, e, p, dso = X.frame(g, th)
        s = np.array([O.bin_center(g, j) for j in range(g["n_det"])])
        ss = (s[:, None] + off[None, :]).reshape(-1)
        q = -dso * u[None, :] + ss[:, None] * e[None, :]
        ch = _chords(p, q - p[None, :], centers, h)
        out[iv] = (ch @ vals).reshape(g["n_det"], K).mean(axis=1)
    return out


def _tiny(n):
    # the config-1 scanner (h = 1 mm, D_po/D_ps = 500/1000, tau = Delta_s = 1.5 mm)
    return dict(W.geometry("1"), n=n, n_views=16, n_det=2 * n + 8)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_brute_force_subrays_tiny_images(n):
    g = _tiny(n)
    img = W.random_image(n, 40 + n).astype(np.float64) + 0.1
    views = list(range(0, 16, 3))
    y = np.stack([O.forward(g, img, view_begin=v, view_count=1)[0] for v in views])
    ref = _brute_force(g, img, views, 1024)  # views 0, 3, ..., 15: 0 and 90 degrees included
    peak = np.abs(ref).max()
    # CNSF within the effective-blur error of the sampled exact projection
    # (measured: 2.5e-5 .. 7.5e-5 of peak for n = 1 .. 8)
    assert np.abs(y - ref).max() <= 3e-4 * peak, np.abs(y - ref).max() / peak
    # and the sampled projection is the reference projector: the oracle's
    # exact bin average (adaptive Simpson) matches it to the sampling error
    # (measured <= 6.6e-5 of peak, at n = 1 with rays along the pixel edges)
    exact = np.stack([O.ref_forward(g, img, view_begin=v, view_count=1)[0] for v in views])
    assert np.abs(ref - exact).max() <= 1.5e-4 * peak


def test_brute_force_converges_at_second_order():
    # midpoint sub-rays at views with no ray along a pixel edge (22.5 and
    # 112.5 degrees): the error against the exact bin average falls ~K^-2
    # (measured 1.3e-3, 7.7e-5, 8.1e-6 of peak at K = 8, 32, 128)
    g = _tiny(4)
    img = W.random_image(4, 7).astype(np.float64)
    views = [1, 5]
    exact = np.stack([O.ref_forward(g, img, view_begin=v, view_count=1)[0] for v in views])
    errs = [np.abs(_brute_force(g, img, views, K) - exact).max() for K in (8, 32, 128)]
    assert errs[1] < errs[0] / 6.0 and errs[2] < errs[1] / 6.0, errs  # 16x expected for K x 4


def _disk_error(n, views):
    fov = 64.0
    g = dict(W.geometry("1"), n=n, pixel=fov / n, det_pitch=96.0 / n, det_width=96.0 / n, n_det=2 * n,
             n_views=90)
    ctr, rad = (7.0, -4.0), 19.0
    img = W.disk(n, g["pixel"], ctr, rad, supersample=16).astype(np.float64)
    err2 = ref2 = 0.0
    for v in views:
        y = O.forward(g, img, view_begin=v, view_count=1)[0]
        th = O.view_angle(g, v)
        u, e, p, dso = X.frame(g, th)
        ref = np.array([X.bin_average(lambda t: X.chord_disk(p, X.det_point(g, th, t) - p, ctr, rad),
                                      s - g["det_width"] / 2, s + g["det_width"] / 2, [])
                        for s in (O.bin_center(g, j) for j in range(g["n_det"]))])
        err2 += float(((y - ref) ** 2).sum())
        ref2 += float((ref ** 2).sum())
    return math.sqrt(err2 / ref2)


def test_disk_phantom_converges_with_the_grid():
    views = [0, 11, 37, 68]
    errs = [_disk_error(n, views) for n in (32, 64, 128)]
    assert errs[0] < 3e-2, errs
    assert errs[1] < errs[0] / 1.5 and errs[2] < errs[1] / 1.5, errs
