"""Pins of the row-f4 oracle (oracle/tv.py) against values fixed by the
definitions, not by re-running its own formulas:

* TV of a constant image is n^2 eps (flat field);
* a unit step edge of length n has TV ~ n (coarea), exactly n up to eps;
* tv_gradient equals central finite differences of tv_value (1e-6 relative,
  randomized 16 x 16 images);
* ASD-POCS: zero sinogram -> zero image; SART's fixed point on consistent
  data with n_tv = 0; the reference projector's own adjoint (ref_back is the
  transpose of ref_forward).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import tv
import workloads as W


def test_tv_flat_field():
    c = np.full((16, 16), 3.25)
    assert tv.tv_value(c) == pytest.approx(256 * tv.EPS_TV, rel=1e-12)
    assert np.abs(tv.tv_gradient(c)).max() == 0.0


def test_tv_step_edge_is_its_length():
    n = 32
    c = np.zeros((n, n))
    c[:, n // 2:] = 1.0
    assert tv.tv_value(c) == pytest.approx(n, rel=1e-6)
    c = np.zeros((n, n))
    c[n // 3:, :] = 1.0
    assert tv.tv_value(c) == pytest.approx(n, rel=1e-6)


@pytest.mark.parametrize("seed", range(4))
def test_tv_gradient_is_finite_difference_of_value(seed):
    rng = np.random.default_rng(seed)
    c = rng.random((16, 16))
    g = tv.tv_gradient(c)
    h = 1e-6
    for _ in range(40):
        r, k = rng.integers(0, 16, size=2)
        cp, cm = c.copy(), c.copy()
        cp[r, k] += h
        cm[r, k] -= h
        fd = (tv.tv_value(cp) - tv.tv_value(cm)) / (2 * h)
        assert g[r, k] == pytest.approx(fd, rel=1e-6, abs=1e-8)


def test_snr_definition():
    t = np.ones((4, 4))
    assert tv.snr_db(t, t) == 300.0
    assert tv.snr_db(t * 1.1, t) == pytest.approx(20.0, abs=1e-12)  # |t| / |0.1 t| = 10


def _small():
    return dict(W.FIG7, n=16, n_views=12, n_det=40)


def test_asd_pocs_zero_data_gives_zero():
    g = _small()
    y = np.zeros((12, 40))
    x = tv.asd_pocs(y, 16, lambda c, v0, m: oracle.ref_forward(g, c, v0, m),
                    lambda s, v0: oracle.ref_back(g, s, v0), tv.AsdPocsConfig(n_iterations=3, n_tv=5, subsets=4))
    assert np.abs(x).max() == 0.0


def test_ref_back_is_transpose_of_ref_forward():
    g = _small()
    rng = np.random.default_rng(2)
    c, y = rng.random((16, 16)), rng.random((12, 40))
    a = float((oracle.ref_forward(g, c) * y).sum())
    b = float((c * oracle.ref_back(g, y)).sum())
    assert a == pytest.approx(b, rel=1e-13)


def test_sart_fixed_point_without_tv():
    g = _small()
    rng = np.random.default_rng(3)
    c = rng.random((16, 16))
    fwd = lambda x: oracle.ref_forward(g, x)
    back = lambda s: oracle.ref_back(g, s)
    y = fwd(c)
    rows, cols = fwd(np.ones((16, 16))), back(np.ones_like(y))
    x = tv.sart_step(c, y, fwd, back, rows, cols, 1.0)
    np.testing.assert_allclose(x, c, atol=1e-12)


def test_ordered_subsets_is_a_permutation_with_jumps():
    for count in (1, 2, 3, 5, 8, 12, 16):
        o = tv._order(count)
        assert sorted(o) == list(range(count))
    assert tv._order(8) == [0, 4, 2, 6, 1, 5, 3, 7]


def test_one_subset_sweep_equals_sart_step():
    g = _small()
    rng = np.random.default_rng(6)
    c = rng.random((16, 16))
    y = oracle.ref_forward(g, c) * 1.1
    fwd = lambda x, v0, m: oracle.ref_forward(g, x, v0, m)
    back = lambda s, v0: oracle.ref_back(g, s, v0)
    cfg = tv.AsdPocsConfig(n_iterations=1, n_tv=0, nonneg=False, subsets=1)
    x = tv.asd_pocs(y, 16, fwd, back, cfg)
    rows, cols = fwd(np.ones((16, 16)), 0, 12), back(np.ones_like(y), 0)
    want = tv.sart_step(np.zeros((16, 16)), y, lambda z: fwd(z, 0, 12), lambda s: back(s, 0), rows, cols, 1.0)
    np.testing.assert_allclose(x, want, atol=1e-13)
