"""Row f2 on the GPU: the reference projector (``cbp_ref_forward``,
FP64 piecewise Gauss-Legendre) against the oracle's reference projector
(FP64 adaptive Simpson, pinned in test_oracle_ref.py), element by element.

Tolerance: both sides integrate the same exact chord to ~1e-13 of the pixel
size; 1e-9 of the sinogram's peak leaves room for FP64 rounding only.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
cbp = pytest.importorskip("paper_1907_10526_b200")

pytestmark = pytest.mark.gpu

TOL = 1e-9


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _check(g, img, view_begin=0, view_count=None):
    dev = _cuda()
    y = cbp.ref_forward(g, torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).to(dev),
                        view_begin=view_begin, view_count=view_count).cpu().numpy()
    want = oracle.ref_forward(g, img.astype(np.float32).astype(np.float64), view_begin=view_begin,
                              view_count=view_count)
    peak = max(np.abs(want).max(), 1e-300)
    err = np.abs(y - want).max() / peak
    assert err < TOL, err
    return y, want


def test_ref_config1_random():
    g = W.geometry("1")
    _check(g, W.random_image(g["n"], 3))


def test_ref_fig6a_single_pixel_all_views():
    _check(W.FIG6, np.ones((1, 1), dtype=np.float32))


def test_ref_fig6b_offset_pixel():
    # the 1 mm pixel centred at (100.5, 50.5) mm: pixel (row 51,
    # col 202) of a 204 x 204 grid (centres (col - 101.5, 101.5 - row))
    g = dict(W.FIG6, n=204)
    img = W.single_pixel(204, 51, 202)
    _check(g, img)


def test_ref_fig7_shepp_logan_views():
    g = W.FIG7
    img = W.shepp_logan(g["n"])
    _check(g, img, view_begin=37, view_count=6)


def test_ref_batch_and_ragged():
    g = dict(W.geometry("1"), n=37, n_views=11, n_det=61, pixel=1.9, det_pitch=2.3, det_width=3.1)
    img = W.random_image(37, 8, batch=2)
    dev = _cuda()
    y = cbp.ref_forward(g, torch.from_numpy(img).to(dev)).cpu().numpy()
    want = oracle.ref_forward(g, img.astype(np.float64))
    assert np.abs(y - want).max() / np.abs(want).max() < TOL


def test_ref_fig5_close_geometry():
    # P:414-416 (Fig. 5): D_po = D_so = 3 mm, a 1 mm pixel, 0.01 mm bins
    _check(W.FIG5, np.ones((1, 1), dtype=np.float32), view_begin=0, view_count=12)


def test_cnsf_against_ref_matches_oracle():
    # the accuracy gap |CNSF - Ref| measured on the GPU equals the oracle's
    g = W.FIG6
    dev = _cuda()
    img = torch.ones((1, 1), device=dev)
    y_c = cbp.forward(g, img).double().cpu().numpy()
    y_r = cbp.ref_forward(g, img).cpu().numpy()
    o_c = oracle.forward(g, np.ones((1, 1)))
    o_r = oracle.ref_forward(g, np.ones((1, 1)))
    gap_gpu = np.abs(y_c - y_r).max(axis=1)
    gap_orc = np.abs(o_c - o_r).max(axis=1)
    # FP32 CNSF: the gaps agree to the FP32 rounding of a ~1 mm peak
    np.testing.assert_allclose(gap_gpu, gap_orc, atol=2e-6)
