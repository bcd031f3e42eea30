"""Row a7 / 8(e) host logic on CPU: view sharding (block and symmetric
orbit shards) and the partial-image sum, world_size 2 over gloo.  The
projector callables are the FP64 oracle here (test infrastructure), so the
check is exactly: the forward shards are the full sinogram's rows, and the
all-reduced partial back-projections equal the full back-projection."""
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads as W
from paper_1907_10526_b200 import sharded


def test_view_shard_partition():
    for n_views in (1, 7, 90, 720, 721):
        for world in (1, 2, 3, 4, 8):
            blocks = [sharded.view_shard(n_views, r, world) for r in range(world)]
            assert blocks[0][0] == 0
            for (a, na), (b, _) in zip(blocks, blocks[1:]):
                assert a + na == b
            assert sum(nv for _, nv in blocks) == n_views
            assert max(nv for _, nv in blocks) - min(nv for _, nv in blocks) <= 1
    with pytest.raises(ValueError):
        sharded.view_shard(10, 2, 2)


@pytest.mark.parametrize("n_views,world", [(720, 8), (720, 3), (90, 4), (12, 2), (8, 4)])
def test_shards_cover_every_view_once(n_views, world):
    views = np.concatenate([sharded.make_shard(n_views, r, world).views() for r in range(world)])
    assert sorted(views.tolist()) == list(range(n_views))
    modes = {sharded.make_shard(n_views, r, world).mode for r in range(world)}
    assert modes == ({"orbit"} if n_views % 4 == 0 and n_views // 4 >= world else {"block"})
    assert sharded.make_shard(n_views, 0, 1).views().tolist() == list(range(n_views))
    assert sharded.make_shard(n_views, 0, world, batch=3).mode == "block"


def _orc_forward(geom, image, sino=None, view_begin=0, view_count=None, stream=None):
    return torch.from_numpy(O.forward(geom, image.numpy(), view_begin, view_count, threads=2))


def _orc_back(geom, sino, image=None, view_begin=0, stream=None):
    c = torch.from_numpy(O.back(geom, sino.numpy(), view_begin, threads=2))
    if image is None:
        return c
    image.copy_(c)
    return image


def _orc_forward_orbit(geom, image, base_begin, base_count, sino=None, stream=None):
    m = geom["n_views"] // 4
    return torch.from_numpy(np.stack([
        O.forward(geom, image.numpy(), base_begin + q * m, base_count, threads=2)
        for q in range(4)]))


def _orc_back_orbit(geom, sino, base_begin, image=None, accumulate=False, stream=None):
    m = geom["n_views"] // 4
    c = sum(O.back(geom, sino[q].numpy(), base_begin + q * m, threads=2) for q in range(4))
    c = torch.from_numpy(c)
    if image is None:
        return c
    image.copy_(c)
    return image


FNS = dict(forward=_orc_forward, forward_orbit=_orc_forward_orbit)
BNS = dict(back=_orc_back, back_orbit=_orc_back_orbit)


def _worker(rank, world, port, geom, img, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        y, sh = sharded.forward_sharded(geom, torch.from_numpy(img), **FNS)
        c = sharded.back_sharded(geom, y, sh, **BNS)
        r = sharded.back_sharded(geom, y, sh, image=torch.zeros_like(c), dst=0, **BNS)
        yl = y.reshape(-1, geom["n_det"]).numpy()
        q.put((rank, sh.views(), yl, c.numpy(), r.numpy() if rank == 0 else None, sh.mode))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n_views", [9, 12])  # 9: block shards; 12: orbit shards
def test_sharded_forward_back_gloo(n_views):
    world = 2
    geom = dict(W._fan(16, n_views, 32))
    img = W.shepp_logan(16).astype(np.float64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, geom, img, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full_y = O.forward(geom, img)
    full_c = O.back(geom, full_y)
    seen = np.concatenate([r[1] for r in res])
    assert sorted(seen.tolist()) == list(range(n_views))
    for rank, views, yl, c, red, mode in res:
        assert mode == ("orbit" if n_views % 4 == 0 else "block")
        np.testing.assert_array_equal(yl, full_y[views])  # FP shards are exact rows
        np.testing.assert_allclose(c, full_c, rtol=1e-12, atol=1e-9)  # all_reduce
    np.testing.assert_allclose(res[0][4], full_c, rtol=1e-12, atol=1e-9)  # reduce to rank 0


# ------------------------------------------------------- dihedral shards
def _d4_orbit(n_views, v):
    """views of base view v under the 8 frames R^q M^m,
    written out independently of the package"""
    N = n_views
    return {((N - v if m else v) + q * (N // 4)) % N for m in (0, 1) for q in range(4)}


@pytest.mark.parametrize("n_views,world", [(720, 8), (720, 3), (88, 2), (16, 3), (8, 2)])
def test_dihedral_shards_cover_every_view_once(n_views, world):
    shards = [sharded.make_shard(n_views, r, world, dihedral=True) for r in range(world)]
    assert {s.mode for s in shards} == {"dihedral"}
    views = np.concatenate([s.views() for s in shards])
    assert sorted(views.tolist()) == list(range(n_views))  # a partition of the scan
    for s in shards:
        want = set()
        for v in range(s.begin, s.begin + s.count):
            want |= _d4_orbit(n_views, v)
        assert set(s.views().tolist()) == want
    # batches and non-multiples of 8 fall back to orbit / block shards
    assert sharded.make_shard(n_views, 0, world, batch=2, dihedral=True).mode == "block"
    assert sharded.make_shard(92, 0, 2, dihedral=True).mode == "orbit"


def _orc_forward_dihedral(geom, image, base_begin, base_count, sino=None, stream=None):
    N = geom["n_views"]
    y = np.zeros((N, geom["n_det"]))
    for v in sorted(set().union(*[_d4_orbit(N, b) for b in range(base_begin, base_begin + base_count)])):
        y[v] = O.forward(geom, image.numpy(), v, 1, threads=2)[0]
    return torch.from_numpy(y)


def _orc_back_dihedral(geom, sino, base_begin, base_count, image=None, accumulate=False, stream=None):
    N = geom["n_views"]
    views = sorted(set().union(*[_d4_orbit(N, b) for b in range(base_begin, base_begin + base_count)]))
    c = sum(O.back(geom, sino[v:v + 1].numpy(), v, threads=2) for v in views)
    c = torch.from_numpy(c)
    if image is None:
        return c
    image.copy_(c)
    return image


def _worker_dihedral(rank, world, port, geom, img, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        y, sh = sharded.forward_sharded(geom, torch.from_numpy(img), dihedral=True,
                                        forward_dihedral=_orc_forward_dihedral)
        c = sharded.back_sharded(geom, y, sh, back_dihedral=_orc_back_dihedral)
        q.put((rank, sh.views(), y.numpy()[sh.views()], c.numpy(), sh.mode))
    finally:
        dist.destroy_process_group()


def test_sharded_dihedral_gloo():
    world, n_views = 2, 16
    geom = dict(W._fan(16, n_views, 32))
    img = W.shepp_logan(16).astype(np.float64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_dihedral, args=(r, world, port, geom, img, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full_y = O.forward(geom, img)
    full_c = O.back(geom, full_y)
    assert sorted(np.concatenate([r[1] for r in res]).tolist()) == list(range(n_views))
    for rank, views, yl, c, mode in res:
        assert mode == "dihedral"
        np.testing.assert_array_equal(yl, full_y[views])
        np.testing.assert_allclose(c, full_c, rtol=1e-12, atol=1e-9)
