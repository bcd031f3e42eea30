"""Row f3 on the GPU: the magnified-footprint weight model (model =
CBP_MODEL_MAG, csrc/cbp_mag.cuh) against the oracle's model 1 (pinned in
test_oracle_mag.py), at the parity bar of test_gpu_parity.py: flat and arc
detectors and parallel beam, batches, ragged sizes, view ranges, the orbit
and dihedral shard calls, sampled outputs at the bench scanner, adjointness."""
import numpy as np
import pytest

import oracle as O
import paper_1907_10526_b200 as cbp
import workloads as W

from tests.test_gpu_parity import _assert_parity, _bp, _fp, torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu


def _mag(kind=cbp.FAN_FLAT, **kw):
    if kind == cbp.PARALLEL:
        g = dict(n=64, pixel=1.0, n_views=90, n_det=128, det_pitch=0.75, det_width=0.75, sid=0.0, sdd=0.0)
    elif kind == cbp.FAN_ARC:
        g = dict(n=64, pixel=1.0, n_views=90, n_det=160, det_pitch=1.2, det_width=1.0, sid=100.0, sdd=200.0)
    else:
        g = dict(W.geometry("1"))
    g.update(kind=kind, model=cbp.MODEL_MAG)
    g.update(kw)
    return g


@pytest.mark.parametrize("kind", [cbp.FAN_FLAT, cbp.FAN_ARC, cbp.PARALLEL])
@pytest.mark.parametrize("n_views", [90, 88])  # 88: the 4-fold rotational path
def test_mag_forward_back(torch_cuda, kind, n_views):
    g = _mag(kind, n_views=n_views)
    # a full scan with n_views % 4 == 0 on an even grid: one footprint per 4 views
    assert cbp.symmetry_fold(g) == (4 if n_views % 4 == 0 else 1)  # the BP at n = 64: 4 frames
    for img in (W.shepp_logan(64), W.random_image(64, 5)):
        _assert_parity(_fp(torch_cuda, g, img), O.forward(g, img), f"FP mag kind {kind} {n_views}")
    y = W.random_sino(n_views, g["n_det"], 6)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), f"BP mag kind {kind} {n_views}")
    assert cbp.adjoint_check(g, seed=3) <= 1e-5


@pytest.mark.parametrize("kind", [cbp.FAN_FLAT, cbp.FAN_ARC])
def test_mag_batch_ragged_wide_fan(torch_cuda, kind):
    # ragged sizes, a batch, a wide fan with a close source (depth varies most)
    g = _mag(kind, n=37, n_views=30, n_det=101, pixel=1.3, det_pitch=1.35, det_width=1.1, sid=40.0, sdd=65.0)
    imgs = W.random_image(37, 7, batch=5)
    _assert_parity(_fp(torch_cuda, g, imgs), O.forward(g, imgs), "FP mag batch")
    y = W.random_sino(30, 101, 8, batch=5)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), "BP mag batch")


def test_mag_view_range_accumulate_and_empty_edges(torch_cuda):
    torch = torch_cuda
    g = _mag()
    img = W.random_image(64, 9)
    _assert_parity(_fp(torch, g, img, view_begin=17, view_count=9),
                   O.forward(g, img, view_begin=17, view_count=9), "FP mag range")
    y = W.random_sino(9, g["n_det"], 10)
    got = _bp(torch, g, y, view_begin=17)
    _assert_parity(got, O.back(g, y, view_begin=17), "BP mag range")
    # accumulate adds to the image; a zero image projects to exactly zero
    base = torch.ones((64, 64), device="cuda")
    cbp.back(g, torch.from_numpy(y).cuda(), image=base, view_begin=17, accumulate=True)
    np.testing.assert_allclose(base.cpu().numpy(), got + 1.0, rtol=1e-6, atol=1e-6)
    assert not _fp(torch, g, np.zeros((64, 64), np.float32)).any()


def test_mag_single_pixel_and_one_by_one(torch_cuda):
    # one lit pixel off centre, and a 1 x 1 image: the footprint and its support edges
    g = _mag()
    img = np.zeros((64, 64), np.float32)
    img[5, 50] = 1.0
    _assert_parity(_fp(torch_cuda, g, img), O.forward(g, img), "FP mag single pixel")
    g1 = _mag(n=1, pixel=3.0, n_det=16)
    one = np.ones((1, 1), np.float32)
    _assert_parity(_fp(torch_cuda, g1, one), O.forward(g1, one), "FP mag 1x1")


def test_mag_parallel_equals_cnsf(torch_cuda):
    # parallel beam: the perspective map is linear, so both models are the
    # exact bin-averaged chord (Theorem 1) and agree to FP32 rounding
    g = _mag(cbp.PARALLEL, n_views=88)
    img = W.random_image(64, 11)
    _assert_parity(_fp(torch_cuda, g, img), _fp(torch_cuda, dict(g, model=cbp.MODEL_CNSF), img), "par mag=cnsf")


def test_mag_config2_sampled(torch_cuda):
    # the bench scanner: sampled views (FP) and pixels (BP) against the oracle
    g = dict(W.geometry("2"), model=cbp.MODEL_MAG)
    img = W.shepp_logan(g["n"])
    y = _fp(torch_cuda, g, img)
    for v in (0, 101, 333, 719):
        _assert_parity(y[v], O.forward(g, img, view_begin=v, view_count=1)[0], f"FP mag cfg2 v{v}")
    s = W.random_sino(g["n_views"], g["n_det"], 12)
    c = _bp(torch_cuda, g, s)
    rows, cols = np.array([0, 511, 256, 37, 400]), np.array([0, 511, 256, 450, 3])
    _assert_parity(c[rows, cols], O.back_pixels(g, s, rows, cols), "BP mag cfg2 sampled")


def test_mag_orbit_and_dihedral_shards(torch_cuda):
    torch = torch_cuda
    from paper_1907_10526_b200 import sharded
    g = _mag(n_views=88)
    img = torch.from_numpy(W.random_image(64, 51)).cuda()
    full_y = cbp.forward(g, img)
    y_rand = torch.from_numpy(W.random_sino(88, g["n_det"], 52)).cuda()
    full_c = cbp.back(g, y_rand)
    for dihedral in (False, True):
        total = torch.zeros_like(full_c)
        seen = []
        for r in range(3):
            sh = sharded.make_shard(88, r, 3, dihedral=dihedral)
            rows = torch.as_tensor(sh.views(), device="cuda")
            if dihedral:
                y = cbp.forward_dihedral(g, img, sh.begin, sh.count)
                _assert_parity(y[rows].cpu().numpy(), full_y[rows].cpu().numpy(), f"FP mag dihedral {r}")
                total += cbp.back_dihedral(g, y_rand, sh.begin, sh.count)
            else:
                y = cbp.forward_orbit(g, img, sh.begin, sh.count)
                _assert_parity(y.reshape(-1, g["n_det"]).cpu().numpy(), full_y[rows].cpu().numpy(),
                               f"FP mag orbit {r}")
                cbp.back_orbit(g, y_rand[rows].reshape(4, sh.count, -1).contiguous(), sh.begin, image=total,
                               accumulate=True)
            seen += sh.views().tolist()
        assert sorted(seen) == list(range(88))
        torch.cuda.synchronize()
        _assert_parity(total.cpu().numpy(), full_c.cpu().numpy(), f"BP mag shards dihedral={dihedral}")


def test_mag_symmetric_equals_plain(torch_cuda):
    # the 4-fold path against the same projector run view by view (no symmetry)
    torch = torch_cuda
    g = _mag(cbp.FAN_ARC, n=48, n_views=40, n_det=120)
    img = torch.from_numpy(W.random_image(48, 21)).cuda()
    y_sym = cbp.forward(g, img)
    y_plain = torch.cat([cbp.forward(g, img, view_begin=v, view_count=1) for v in range(40)])
    _assert_parity(y_sym.cpu().numpy(), y_plain.cpu().numpy(), "mag FP sym vs plain")
    s = torch.from_numpy(W.random_sino(40, 120, 22)).cuda()
    c_sym = cbp.back(g, s)
    c_plain = sum(cbp.back(g, s[v:v + 1].contiguous(), view_begin=v) for v in range(40))
    _assert_parity(c_sym.cpu().numpy(), c_plain.cpu().numpy(), "mag BP sym vs plain")


def test_mag_dihedral_bp_large_grid(torch_cuda):
    # n = 1024: the BP takes the 8-frame dihedral triangle (diagonal pixels 4 frames);
    # sampled pixels on and off the diagonals against the oracle
    g = dict(W.geometry("3"), model=cbp.MODEL_MAG, n_views=48)
    assert cbp.symmetry_fold(g) == 8
    s = W.random_sino(48, g["n_det"], 77)
    c = _bp(torch_cuda, g, s)
    rows = np.array([0, 511, 512, 1023, 100, 923, 300, 5, 700])
    cols = np.array([0, 511, 512, 1023, 100, 100, 723, 900, 20])
    _assert_parity(c[rows, cols], O.back_pixels(g, s, rows, cols), "BP mag dihedral n=1024")
    # every pixel against the same projector view by view (no symmetry)
    torch = torch_cuda
    st = torch.from_numpy(s).cuda()
    plain = sum(cbp.back(g, st[v:v + 1].contiguous(), view_begin=v) for v in range(48))
    _assert_parity(c, plain.cpu().numpy(), "BP mag dihedral vs plain n=1024")
