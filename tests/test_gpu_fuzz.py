"""Randomised parity: seeded random scanners (every kind and weight model,
odd and even grids, ragged tiles, one view / one bin, close and far
sources, wide and narrow bins, tau != Delta_s), batches and view ranges,
FP and BP of the CUDA path against the oracle at the parity bar of
test_gpu_parity.py.  The draws are fixed by the seed, so a failure
reproduces; they cover the symmetric paths (full scans with n_views % 4,
% 8 == 0) as well as the direct and batched ones."""
import numpy as np
import pytest

import oracle as O
import paper_1907_10526_b200 as cbp
import workloads as W

from tests.test_gpu_parity import _assert_parity, _bp, _fp, torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu


def draw(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = int(rng.integers(0, 3))
    model = int(rng.random() < 0.3)
    n = int(rng.choice([1, 2, 5, 16, 31, 32, 33, 48, 64, 70, 97, 130]))
    h = float(rng.uniform(0.3, 2.0))
    n_views = int(rng.choice([1, 3, 8, 16, 24, 30, 40, 45, 64, 72]))
    pitch = float(rng.uniform(0.4, 2.5)) * h
    width = float(np.exp(rng.uniform(np.log(0.05), np.log(3.0)))) * pitch  # tau/Delta_s 0.05 .. 3
    R = n * h / np.sqrt(2.0)
    sid = float(R * rng.uniform(1.15, 6.0) + 1.0)
    sdd = float(sid * rng.uniform(1.0, 2.5))
    # enough bins to cover the field of view (plus a random margin or shortfall)
    if kind == 1:
        span = 2 * R
    else:
        span = 2 * sdd * np.tan(np.arcsin(min(R / sid, 0.999)))
    n_det = max(1, int(span / pitch * rng.uniform(0.6, 1.3)) + int(rng.integers(0, 4)))
    if kind == 2:  # arc: every bin within +-90 degrees (arc length / sdd)
        n_det = max(1, min(n_det, int(2.9 * sdd / pitch) - 2))
    g = dict(n=n, pixel=h, n_views=n_views, n_det=n_det, det_pitch=pitch, det_width=width,
             sid=sid if kind != 1 else 0.0, sdd=sdd if kind != 1 else 0.0, kind=kind, model=model)
    if cbp.validate(g) != cbp.CBP_OK:  # rare draws: a bin wider than 2 D_ps, or arc bins past 90 degrees
        g["det_width"] = min(width, 1.9 * sdd) if kind != 1 else width
        while kind == 2 and g["n_det"] > 1 and cbp.validate(g) != cbp.CBP_OK:
            g["n_det"] -= 1
    batch = int(rng.choice([1, 1, 1, 2, 3, 5]))
    full = rng.random() < 0.6
    v0 = 0 if full else int(rng.integers(0, n_views))
    nv = n_views - v0 if full else int(rng.integers(1, n_views - v0 + 1))
    return g, batch, v0, nv, rng


# 248 and 665 found a bug (fixed): with a source ~2 field radii away and bins
# wider than 2 pixels, the first FP candidate of a line can sit in the zero
# border behind the source with tau' < 0, and clamping it shifted tau' of
# every later candidate on the line (1 % errors in a few views)
@pytest.mark.parametrize("seed", list(range(160)) + [248, 665])
def test_random_scanner_parity(torch_cuda, seed):
    g, batch, v0, nv, rng = draw(seed)
    assert cbp.validate(g) == cbp.CBP_OK, g
    n = g["n"]
    imgs = W.random_image(n, 500 + seed, batch=batch) if batch > 1 else W.random_image(n, 500 + seed)
    what = f"seed {seed} {g} batch {batch} views {v0}+{nv}"
    want = O.forward(g, imgs, view_begin=v0, view_count=nv)
    got = _fp(torch_cuda, g, imgs, view_begin=v0, view_count=nv)
    if np.abs(want).max() == 0.0:  # the bins miss the image entirely: exact zeros
        assert not got.any(), what
    else:
        _assert_parity_or_tail(got, want, _mass(imgs, batch), g["pixel"], "FP " + what)
    y = W.random_sino(nv, g["n_det"], 600 + seed, batch=batch) if batch > 1 else \
        W.random_sino(nv, g["n_det"], 600 + seed)
    want_b = O.back(g, y, view_begin=v0)
    if np.abs(want_b).max() == 0.0:
        assert not _bp(torch_cuda, g, y, view_begin=v0).any(), what
    else:
        _assert_parity_or_tail(_bp(torch_cuda, g, y, view_begin=v0), want_b, _mass(y, batch), g["pixel"],
                               "BP " + what)


# Ledger #23: outputs that see only support-edge tails.  Each
# output is a sum of weights times inputs, |dy_j| <= max|dW| sum_k |c_k|, and
# the FP32 weight's absolute error is bounded relative to the LARGEST weight,
# not to the weight itself: |dW| <= DELTA_W W_max with W_max = h^2 max M <=
# h^2 / A <= sqrt(2) h (A = max|zeta| >= h / sqrt 2; the magnified model's
# h^2 m / A obeys the same bound since m / |grad P| = 1), DELTA_W = 1e-6 (twice
# the pinned 5e-7 of tests/test_weight_form.py).  So when max|y| < 1e4
# eps_abs, eps_abs = DELTA_W sqrt(2) h sum|inputs| per slice, the 1e-4
# max-normalised bar would demand more than FP32 weights can give, and the
# bar is the derived absolute bound itself.  Everywhere else the bar of
# test_gpu_parity.py applies unchanged.
DELTA_W = 1e-6


def _mass(x, batch):
    """sum of |inputs| per slice, the largest slice's"""
    x = np.abs(np.asarray(x, dtype=np.float64))
    return float(x.reshape(batch, -1).sum(axis=1).max()) if batch > 1 else float(x.sum())


def _assert_parity_or_tail(got, want, mass, h, what):
    eps_abs = DELTA_W * np.sqrt(2.0) * h * mass
    if np.abs(want).max() < 1e4 * eps_abs:
        err = np.abs(np.asarray(got, np.float64) - want).max()
        assert err <= eps_abs, f"{what}: tail case, max|dy| {err:.3e} > eps_abs {eps_abs:.3e}"
    else:
        _assert_parity(got, want, what)

