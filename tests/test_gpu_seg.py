"""The persistent dihedral BP (opt-in, CBP_BP_SEG=1): one
wave of CTAs over cost-balanced segments of the (tile, base view) pairs, each
segment's 8 frames written as a compact block in output orientation, summed
by cbp_seg_reduce_kernel (n a multiple of 32: one CTA per output tile;
ragged n: one thread per pixel).  Checked against the FP64 oracle at the
parity bar of tests/test_gpu_parity.py: one image, a batch of images,
accumulate mode, dihedral shards (base views not starting at 0), CTA counts
that put several tiles in one CTA or leave CTAs without work, and bitwise
repeatability (segment boundaries are fixed, so is the summation order)."""
import numpy as np
import pytest

import oracle as O
import paper_1907_10526_b200 as cbp
import workloads as W

from tests.test_gpu_parity import _assert_parity, torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu


def _geom(n, n_views=48):
    h = 64.0 / n
    return dict(n=n, pixel=h, n_views=n_views, n_det=2 * n + 6, det_pitch=1.5 * h, det_width=1.5 * h,
                sid=500.0, sdd=1000.0)


@pytest.fixture(autouse=True)
def seg_on(monkeypatch):
    monkeypatch.setenv("CBP_BP_SEG", "1")


@pytest.mark.parametrize("n", [64, 96, 70])  # 70: ragged tiles, the per-pixel reduction
@pytest.mark.parametrize("ctas", [None, "5", "2000"])
def test_seg_bp_matches_oracle(torch_cuda, monkeypatch, n, ctas):
    torch = torch_cuda
    if ctas:
        monkeypatch.setenv("CBP_BP_SEG_CTAS", ctas)
    g = _geom(n)
    y_np = W.random_sino(g["n_views"], g["n_det"], 41)
    got = cbp.back(g, torch.from_numpy(y_np).cuda()).cpu().numpy()
    _assert_parity(got, O.back(g, y_np), f"seg BP n={n} ctas={ctas}")
    again = cbp.back(g, torch.from_numpy(y_np).cuda()).cpu().numpy()
    assert np.array_equal(got, again), "seg BP not bitwise repeatable"


def test_seg_bp_batch_and_accumulate(torch_cuda):
    torch = torch_cuda
    g = _geom(64)
    ys = W.random_sino(g["n_views"], g["n_det"], 42, batch=3)
    want = np.stack([O.back(g, ys[b]) for b in range(3)])
    got = cbp.back(g, torch.from_numpy(ys).cuda()).cpu().numpy()
    _assert_parity(got, want, "seg BP batch of 3 images")
    base = torch.ones((3, 64, 64), device="cuda")
    cbp.back(g, torch.from_numpy(ys).cuda(), image=base, accumulate=True)
    _assert_parity(base.cpu().numpy() - 1.0, want, "seg BP accumulate")


def test_seg_bp_dihedral_shards(torch_cuda):
    torch = torch_cuda
    from paper_1907_10526_b200 import sharded
    g = _geom(96)
    y_np = W.random_sino(g["n_views"], g["n_det"], 43)
    y = torch.from_numpy(y_np).cuda()
    total = torch.zeros((96, 96), device="cuda")
    for r in range(3):
        sh = sharded.make_shard(g["n_views"], r, 3, dihedral=True)
        total += cbp.back_dihedral(g, y, sh.begin, sh.count)
    _assert_parity(total.cpu().numpy(), O.back(g, y_np), "seg BP dihedral shards x3")
