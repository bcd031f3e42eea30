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


def test_parallel_rejected_by_reference_projector(torch_cuda):
    torch = torch_cuda
    with pytest.raises(cbp.CbpError):
        cbp.ref_forward(_par(), torch.zeros((64, 64), device="cuda"))
