"""Row f3 on the GPU: the parallel-beam mode (kind = CBP_PARALLEL, Eq. 9-10)
of the same FP / BP kernels against the oracle's parallel-beam mode (pinned
in test_oracle_parallel.py), at the parity bar of test_gpu_parity.py, on the
direct, 4-fold and 8-fold symmetric and batched paths; plus Theorem 1 on the
GPU (CNSF equals the exact bin-averaged chord in parallel geometry)."""
import numpy as np
import pytest

import oracle as O
import paper_1907_10526_b200 as cbp
import workloads as W

from tests.test_gpu_parity import _assert_parity, _bp, _fp, torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu


def _par(**kw):
    g = dict(n=64, pixel=1.0, n_views=90, n_det=128, det_pitch=0.75, det_width=0.75, sid=0.0, sdd=0.0,
             kind=cbp.PARALLEL)
    g.update(kw)
    return g


@pytest.mark.parametrize("n_views", [90, 92, 88])  # direct / 4-fold / 8-fold symmetric paths
def test_parallel_forward_back(torch_cuda, n_views):
    g = _par(n_views=n_views)
    for img in (W.shepp_logan(64), W.random_image(64, 5)):
        _assert_parity(_fp(torch_cuda, g, img), O.forward(g, img), f"FP par {n_views}")
    y = W.random_sino(n_views, 128, 6)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), f"BP par {n_views}")
    assert cbp.adjoint_check(g, seed=3) <= 1e-5


def test_parallel_batch_and_ragged(torch_cuda):
    g = _par(n=37, n_views=30, n_det=77, det_pitch=1.1, det_width=0.6, pixel=1.3)
    imgs = W.random_image(37, 7, batch=5)
    got = _fp(torch_cuda, g, imgs)
    ref = O.forward(g, imgs)
    _assert_parity(got, ref, "FP par batch")
    y = W.random_sino(30, 77, 8, batch=5)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), "BP par batch")


def test_parallel_view_range(torch_cuda):
    g = _par()
    img = W.random_image(64, 9)
    _assert_parity(_fp(torch_cuda, g, img, view_begin=17, view_count=9),
                   O.forward(g, img, view_begin=17, view_count=9), "FP par range")


def test_parallel_is_exact_theorem1(torch_cuda):
    # in parallel geometry the CNSF weights are the exact bin
    # averages, so the FP32 projector matches the FP64 exact reference to FP32 rounding
    g = _par(n_views=88)
    img = W.shepp_logan(64)
    _assert_parity(_fp(torch_cuda, g, img), O.ref_forward(g, img), "FP par vs exact")


def _ref_parity(torch, g, img, what):
    got = cbp.ref_forward(g, torch.from_numpy(img).cuda()).cpu().numpy()
    want = O.ref_forward(g, img.astype(np.float64))
    assert np.abs(got - want).max() / np.abs(want).max() < 1e-9, what
    y = W.random_sino(g["n_views"], g["n_det"], 9).astype(np.float64)
    gb = cbp.ref_back(g, torch.from_numpy(y).cuda()).cpu().numpy()
    wb = O.ref_back(g, y)
    assert np.abs(gb - wb).max() / np.abs(wb).max() < 1e-9, what


def test_parallel_reference_projector(torch_cuda):
    # the GPU reference pair in parallel geometry against the oracle's, and
    # Theorem 1 once more: the FP32 CNSF projector equals it to FP32 rounding
    torch = torch_cuda
    g = _par(n=32, n_views=12, n_det=64)
    img = W.random_image(32, 13)
    _ref_parity(torch, g, img, "ref parallel")
    ref = cbp.ref_forward(g, torch.from_numpy(img).cuda()).cpu().numpy()
    _assert_parity(_fp(torch, g, img), ref, "CNSF parallel vs GPU ref")


# ------------------------------------------------------------ arc detector
def _arc(**kw):
    g = dict(n=64, pixel=1.0, n_views=90, n_det=160, det_pitch=1.2, det_width=1.0, sid=100.0, sdd=200.0,
             kind=cbp.FAN_ARC)
    g.update(kw)
    return g


@pytest.mark.parametrize("n_views", [90, 92, 88])  # direct / 4-fold / 8-fold symmetric paths
def test_arc_forward_back(torch_cuda, n_views):
    g = _arc(n_views=n_views)
    for img in (W.shepp_logan(64), W.random_image(64, 5)):
        _assert_parity(_fp(torch_cuda, g, img), O.forward(g, img), f"FP arc {n_views}")
    y = W.random_sino(n_views, 160, 6)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), f"BP arc {n_views}")
    assert cbp.adjoint_check(g, seed=3) <= 1e-5


def test_arc_batch_ragged_and_wide_fan(torch_cuda):
    # ragged tiles, a batch, and a wide fan (+-60 degrees, close source)
    g = _arc(n=37, n_views=30, n_det=101, pixel=1.3, det_pitch=1.35, det_width=1.1, sid=40.0, sdd=65.0)
    imgs = W.random_image(37, 7, batch=5)
    _assert_parity(_fp(torch_cuda, g, imgs), O.forward(g, imgs), "FP arc batch")
    y = W.random_sino(30, 101, 8, batch=5)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), "BP arc batch")


def test_arc_config2_scale_sampled(torch_cuda):
    # the bench scanner with an equiangular detector of the same pitch at the centre
    g = dict(W.geometry("2"), kind=cbp.FAN_ARC)
    img = W.shepp_logan(g["n"])
    y = _fp(torch_cuda, g, img)
    for v in (0, 101, 333, 719):
        _assert_parity(y[v], O.forward(g, img, view_begin=v, view_count=1)[0], f"FP arc cfg2 v{v}")
    s = W.random_sino(g["n_views"], g["n_det"], 12)
    c = _bp(torch_cuda, g, s)
    rows, cols = np.array([0, 511, 256, 37, 400]), np.array([0, 511, 256, 450, 3])
    _assert_parity(c[rows, cols], O.back_pixels(g, s, rows, cols), "BP arc cfg2 sampled")


def test_arc_reference_projector_and_validation(torch_cuda):
    torch = torch_cuda
    g = _arc(n=32, n_views=12, n_det=80, sid=60.0, sdd=120.0)
    _ref_parity(torch, g, W.random_image(32, 14), "ref arc")
    with pytest.raises(cbp.CbpError):  # bins beyond 90 degrees
        cbp.forward(_arc(n_det=600), torch.zeros((64, 64), device="cuda"))


@pytest.mark.parametrize("kind", [cbp.PARALLEL, cbp.FAN_ARC])
def test_variant_batch_full_scan(torch_cuda, kind):
    # a batch over a full scan (n_views % 8 == 0): batched FP, per-image
    # dihedral BP, for the parallel beam and the arc detector
    g = _par(n_views=88) if kind == cbp.PARALLEL else _arc(n_views=88)
    imgs = W.random_image(64, 41, batch=3)
    _assert_parity(_fp(torch_cuda, g, imgs), O.forward(g, imgs), f"FP batch kind {kind}")
    y = W.random_sino(88, g["n_det"], 42, batch=3)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), f"BP batch kind {kind}")


def test_arc_bp_close_source_bin_range(torch_cuda):
    # regression (tools/fuzz.py wide seed 2009): a source within a few pixels
    # of the field of view; the arc BP's per-tile bin range used the small-angle
    # bound 1.01 sigma/delta for asin(sigma/|k - p|) and dropped bins (2.4e-2)
    g = dict(n=1, pixel=1.4937332023018055, n_views=4, n_det=19, det_pitch=0.6050390134164245,
             det_width=0.13130810019606656, sid=1.2585, sdd=4.0084, kind=cbp.FAN_ARC)
    for view_begin in (0, 2):
        y = W.random_sino(2, 19, 2016)
        _assert_parity(_bp(torch_cuda, g, y, view_begin=view_begin), O.back(g, y, view_begin=view_begin),
                       f"arc BP close source from view {view_begin}")
    g5 = dict(g, n=5, pixel=0.5, sid=4.0, sdd=9.0, n_views=16, n_det=60, det_pitch=0.4)
    y = W.random_sino(16, 60, 2017)
    _assert_parity(_bp(torch_cuda, g5, y), O.back(g5, y), "arc BP close source, 5x5")
