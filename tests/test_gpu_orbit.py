"""The dihedral BP as clusters of 8 CTAs over tile orbits:
each output tile summed from its orbit's frame accumulators through
distributed shared memory (no frame planes).  Checked against the FP64
oracle at the parity bar and against the frame-plane path (the default;
the orbit path is opt-in, CBP_ORBIT=1, being slower)
on tile grids with every orbit size: T = 2, 4 (orbits of 8 and of 4 on the
diagonals) and T = 3, 5 (odd: the centre tile's orbit of 1, the middle
row's orbits of 4); one image, a batch (images as slice groups), accumulate
mode, dihedral shards (base views not starting at 0), several view groups."""
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
def orbit_on(monkeypatch):
    monkeypatch.setenv("CBP_ORBIT", "1")  # the opt-in orbit path


def _both(monkeypatch, fn):
    a = fn()
    monkeypatch.setenv("CBP_ORBIT", "0")
    b = fn()
    monkeypatch.setenv("CBP_ORBIT", "1")
    return a, b


@pytest.mark.parametrize("n", [64, 96, 128, 160])
def test_orbit_bp_matches_oracle_and_planes(torch_cuda, monkeypatch, n):
    torch = torch_cuda
    g = _geom(n)
    assert cbp.symmetry_fold(g) == 8
    y_np = W.random_sino(g["n_views"], g["n_det"], 70 + n)
    y = torch.from_numpy(y_np).cuda()
    orb, pl = _both(monkeypatch, lambda: cbp.back(g, y).cpu().numpy())
    want = O.back(g, y_np)
    _assert_parity(orb, want, f"orbit BP n={n}")
    _assert_parity(pl, want, f"plane BP n={n}")
    assert np.abs(orb - pl).max() <= 1e-6 * np.abs(want).max()


@pytest.mark.parametrize("groups", ["1", "3"])
def test_orbit_bp_batch_accumulate_groups(torch_cuda, monkeypatch, groups):
    torch = torch_cuda
    monkeypatch.setenv("CBP_BP_GROUPS", groups)  # (the orbit path reads it per call)
    g = _geom(128)
    ys = W.random_sino(g["n_views"], g["n_det"], 81, batch=3)
    want = O.back(g, ys)
    got = cbp.back(g, torch.from_numpy(ys).cuda()).cpu().numpy()
    _assert_parity(got, want, "orbit BP batch")
    base = torch.from_numpy(W.random_image(g["n"], 82, batch=3)).cuda()
    acc = base.clone()
    cbp.back(g, torch.from_numpy(ys).cuda(), image=acc, accumulate=True)
    _assert_parity(acc.cpu().numpy(), want + base.cpu().numpy(), "orbit BP accumulate")


def test_orbit_bp_dihedral_shards(torch_cuda):
    torch = torch_cuda
    g = _geom(128, n_views=64)
    y_np = W.random_sino(g["n_views"], g["n_det"], 83)
    y = torch.from_numpy(y_np).cuda()
    acc = None
    for b0, nb in ((0, 3), (3, 4), (7, 2)):  # base views [0, 8] = n_views/8 + 1
        acc = cbp.back_dihedral(g, y, b0, nb) if acc is None else \
            cbp.back_dihedral(g, y, b0, nb, image=acc, accumulate=True)
    _assert_parity(acc.cpu().numpy(), O.back(g, y_np), "orbit BP dihedral shards")
