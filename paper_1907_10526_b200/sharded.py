"""Row a7 / 8(e): the projector sharded over GPUs by VIEWS (one process per
GPU, torch.distributed over NCCL).

Forward projection needs no communication: rank g owns the contiguous view
block [v0_g, v0_g + nv_g) and writes its own sinogram rows.  The
back-projection is a sum over views, so each rank back-projects its block
into a partial image and the partials are summed with one collective
(all_reduce, or reduce to one rank) -- the only exchange step of the path.

Argument marshalling and the collective only; the projections themselves run
in libcbp.so (``paper_1907_10526_b200.forward`` / ``back``).  The projector
functions are parameters so the host logic can be tested on CPU with gloo.
"""
from __future__ import annotations

from typing import Callable, Optional

import paper_1907_10526_b200 as _cbp


def view_shard(n_views: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous view block (view_begin, view_count) of `rank` out of `world`;
    the first n_views % world ranks get one extra view."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, rem = divmod(n_views, world)
    v0 = rank * base + min(rank, rem)
    return v0, base + (1 if rank < rem else 0)


def _rank_world(group):
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def forward_sharded(geom, image, sino=None, group=None,
                    forward: Callable = _cbp.forward, stream=None):
    """This rank's block of y = A c: returns (sino_shard, view_begin).
    No communication."""
    rank, world = _rank_world(group)
    n_views = geom["n_views"] if isinstance(geom, dict) else geom.n_views
    v0, nv = view_shard(n_views, rank, world)
    if nv == 0:
        return None, v0
    return forward(geom, image, sino, view_begin=v0, view_count=nv, stream=stream), v0


def back_sharded(geom, sino_shard, image=None, group=None, dst: Optional[int] = None,
                 back: Callable = _cbp.back, stream=None):
    """c = sum_g A_g^T y_g: back-projects this rank's views, then sums the
    partial images over the group (all_reduce, or reduce to `dst`).
    `sino_shard` holds views view_shard(n_views, rank, world)."""
    import torch
    import torch.distributed as dist
    rank, world = _rank_world(group)
    n_views = geom["n_views"] if isinstance(geom, dict) else geom.n_views
    v0, nv = view_shard(n_views, rank, world)
    if sino_shard is not None and sino_shard.shape[-2] != nv:
        raise ValueError(f"rank {rank} holds {sino_shard.shape[-2]} views, expected {nv}")
    if nv > 0:
        image = back(geom, sino_shard, image, view_begin=v0, stream=stream)
    elif image is not None:
        image[...] = 0
    else:
        raise ValueError("a rank without views needs an image buffer to receive the sum")
    if world > 1:
        t = image if isinstance(image, torch.Tensor) else torch.from_numpy(image)
        if dst is None:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        else:
            dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return image


def normal_sharded(geom, image, group=None, forward: Callable = _cbp.forward,
                   back: Callable = _cbp.back, stream=None):
    """A^T A c over the group (one FP+BP pair, the benchmark's step)."""
    y, _ = forward_sharded(geom, image, group=group, forward=forward, stream=stream)
    return back_sharded(geom, y, group=group, back=back, stream=stream)
