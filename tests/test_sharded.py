"""Row a7 / 8(e) host logic on CPU: view sharding and the partial-image sum,
world_size 2 over gloo.  The projector callables are the FP64 oracle here
(test infrastructure), so the check is exactly: concatenated forward shards
== the full forward, and the all-reduced partial back-projections == the
full back-projection."""
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


def _orc_forward(geom, image, sino=None, view_begin=0, view_count=None, stream=None):
    return torch.from_numpy(O.forward(geom, image.numpy(), view_begin, view_count, threads=2))


def _orc_back(geom, sino, image=None, view_begin=0, stream=None):
    c = torch.from_numpy(O.back(geom, sino.numpy(), view_begin, threads=2))
    if image is None:
        return c
    image.copy_(c)
    return image


def _worker(rank, world, port, geom, img, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        y, v0 = sharded.forward_sharded(geom, torch.from_numpy(img), forward=_orc_forward)
        c = sharded.back_sharded(geom, y, back=_orc_back)
        r = sharded.back_sharded(geom, y, image=torch.zeros_like(c), dst=0, back=_orc_back)
        q.put((rank, v0, y.numpy(), c.numpy(), r.numpy() if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_forward_back_gloo(world):
    geom = dict(W._fan(16, 9, 32))
    img = W.shepp_logan(16).astype(np.float64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, geom, img, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full_y = O.forward(geom, img)
    full_c = O.back(geom, full_y)
    ys = np.concatenate([r[2] for r in res], axis=0)
    np.testing.assert_array_equal(ys, full_y)  # FP shards are exact slices
    for r in res:
        v0, nv = sharded.view_shard(geom["n_views"], r[0], world)
        assert r[1] == v0 and r[2].shape[0] == nv
        np.testing.assert_allclose(r[3], full_c, rtol=1e-12, atol=1e-9)  # all_reduce
    np.testing.assert_allclose(res[0][4], full_c, rtol=1e-12, atol=1e-9)  # reduce to rank 0
