"""Row a7 fused into the BP (CBP_ACC_MULTIMEM): the BP's last kernel adds the
rank's partial image into a multicast address with multimem.red.add.f32.
On one B200 a one-member multicast object (tests/_multicast.py) stands for
the ranks' symmetric buffer: shards issued one after another add into it as
separate ranks would, and the result must equal the full back-projection
(parity bar of test_gpu_parity.py; the sum order is the switch's)."""
import numpy as np
import pytest

import oracle as O
import paper_1907_10526_b200 as cbp
import workloads as W

from tests.test_gpu_parity import _assert_parity, _bp_sample_pixels, torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mc_factory(torch_cuda):
    torch_cuda.cuda.init()
    torch_cuda.zeros(1, device="cuda")  # the primary context is current
    made = []

    def make(nbytes):
        from tests._multicast import Multicast
        try:
            m = Multicast(nbytes)
        except Exception as e:  # noqa: BLE001
            pytest.skip(f"no multicast object on this GPU: {e}")
        made.append(m)
        return m
    yield make
    for m in made:
        m.close()


def _read(torch, m, n):
    out = torch.empty((n, n), device="cuda")
    m.read_into(out)
    return out.cpu().numpy()


@pytest.mark.parametrize("model", [cbp.MODEL_CNSF, cbp.MODEL_MAG])
@pytest.mark.parametrize("cfg,world", [("1", 3), ("2", 8)])
def test_multimem_dihedral_and_orbit_shards(torch_cuda, mc_factory, model, cfg, world):
    torch = torch_cuda
    from paper_1907_10526_b200 import sharded
    g = dict(W.geometry(cfg), n_views=88, model=model) if cfg == "1" else dict(W.geometry(cfg), model=model)
    n = g["n"]
    y_np = W.random_sino(g["n_views"], g["n_det"], 31)
    y = torch.from_numpy(y_np).cuda()
    if cfg == "1":
        rows, cols = np.divmod(np.arange(n * n), n)
        want = O.back(g, y_np).ravel()
    else:
        rows, cols = _bp_sample_pixels(n, 64)
        want = O.back_pixels(g, y_np, rows, cols)
    m = mc_factory(4 * n * n)
    for dihedral in (True, False):
        m.zero()
        for r in range(world):  # the ranks' calls, one after another
            sh = sharded.make_shard(g["n_views"], r, world, dihedral=dihedral)
            if sh.mode == "orbit":
                rows = torch.as_tensor(sh.views(), device="cuda")
                ys = y[rows].reshape(4, sh.count, -1).contiguous()
            else:
                ys = y
            cbp.back_multimem(g, ys, m.mc, shard=sh)
        torch.cuda.synchronize()
        _assert_parity(_read(torch, m, n)[rows, cols], want, f"multimem {sh.mode} shards x{world} model {model}")


def test_multimem_view_blocks_batch_path(torch_cuda, mc_factory):
    # plain view blocks (no symmetry), including the single-group BP that
    # otherwise writes the image directly
    torch = torch_cuda
    g = dict(W.geometry("1"), n_views=90)
    y_np = W.random_sino(90, g["n_det"], 32)
    y = torch.from_numpy(y_np).cuda()
    full = O.back(g, y_np)
    m = mc_factory(4 * 64 * 64)
    m.zero()
    for v0, nv in ((0, 7), (7, 50), (57, 33)):
        cbp.back_multimem(g, y[v0:v0 + nv].contiguous(), m.mc, view_begin=v0)
    torch.cuda.synchronize()
    _assert_parity(_read(torch, m, 64), full, "multimem view blocks")
    # a whole scan in one call (the library's own dihedral path) adds on top
    cbp.back_multimem(g, y, m.mc)
    torch.cuda.synchronize()
    _assert_parity(_read(torch, m, 64), 2 * full, "multimem second add")
    with pytest.raises(cbp.CbpError):  # a host sinogram is rejected
        cbp.back_multimem(g, y.cpu().numpy(), m.mc)
