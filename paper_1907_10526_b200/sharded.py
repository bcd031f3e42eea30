"""Row a7 / 8(e): the projector sharded over GPUs by VIEWS (one process per
GPU, torch.distributed over NCCL).

Forward projection needs no communication: each rank owns a set of views and
writes its own sinogram rows.  The back-projection is a sum over views, so
each rank back-projects its views into a partial image and the partials are
summed with one collective (all_reduce, or reduce to one rank) -- the only
exchange step of the path.

Three shard shapes (``Shard.mode``):

* ``"orbit"`` (one image, n_views % 4 == 0): the n_views/4 base views are
  split in contiguous blocks and each rank takes the 4 rotated copies of its
  block, views {b + q n_views/4}; the library's 90-degree rotational symmetry
  then computes each weight once for 4 views (``forward_orbit`` /
  ``back_orbit``, local sinogram [4, nb, n_det]);
* ``"dihedral"`` (one image, n_views % 8 == 0, requested with
  ``dihedral=True``): the n_views/8 + 1 base views of the 8-fold symmetry
  are split in contiguous blocks and each rank takes their orbits under
  the rotations and the mirror (``forward_dihedral`` / ``back_dihedral``,
  local sinogram = the natural [n_views, n_det] with this rank's rows),
  so every rank's BP keeps one weight per 8 views;
* ``"block"`` (otherwise): a contiguous block of views (local sinogram
  [B?, nv, n_det]).

Argument marshalling and the collective only; the projections run in
libcbp.so.  The projector callables are parameters so the host logic is
testable on CPU with gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

import paper_1907_10526_b200 as _cbp


def view_shard(n_views: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block (begin, count) of `rank` out of `world` for n_views
    items; the first n_views % world ranks get one extra."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, rem = divmod(n_views, world)
    v0 = rank * base + min(rank, rem)
    return v0, base + (1 if rank < rem else 0)


@dataclass(frozen=True)
class Shard:
    mode: str    # "orbit", "dihedral" or "block"
    begin: int   # first base view (orbit) or first view (block)
    count: int   # base views (orbit) or views (block)
    n_views: int

    def views(self) -> np.ndarray:
        """global view index of each local sinogram row (dihedral: the rows of
        the natural sinogram this shard owns, sorted)"""
        if self.mode == "block":
            return np.arange(self.begin, self.begin + self.count)
        if self.mode == "dihedral":
            return np.asarray(_cbp.dihedral_views(self.n_views, self.begin, self.count))
        m = self.n_views // 4
        return np.concatenate([np.arange(self.begin, self.begin + self.count) + q * m
                               for q in range(4)])


def make_shard(n_views: int, rank: int, world: int, batch: int = 1, dihedral: bool = False) -> Shard:
    if world == 1:  # the whole scan: the library picks its widest symmetry itself
        return Shard("block", 0, n_views, n_views)
    if dihedral and batch == 1 and n_views % 8 == 0 and n_views // 8 + 1 >= world:
        b0, nb = view_shard(n_views // 8 + 1, rank, world)
        return Shard("dihedral", b0, nb, n_views)
    if batch == 1 and n_views % 4 == 0 and n_views // 4 >= world:
        b0, nb = view_shard(n_views // 4, rank, world)
        return Shard("orbit", b0, nb, n_views)
    v0, nv = view_shard(n_views, rank, world)
    return Shard("block", v0, nv, n_views)


def _rank_world(group):
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _n_views(geom):
    return geom["n_views"] if isinstance(geom, dict) else geom.n_views


def forward_sharded(geom, image, group=None, forward: Callable = _cbp.forward,
                    forward_orbit: Callable = _cbp.forward_orbit,
                    forward_dihedral: Callable = _cbp.forward_dihedral, dihedral: bool = False,
                    stream=None):
    """This rank's part of y = A c: returns (local sinogram, Shard).  No
    communication.  Row i of the local sinogram is view shard.views()[i]
    (dihedral: the natural sinogram, rows shard.views() filled)."""
    rank, world = _rank_world(group)
    batch = 1 if image.ndim == 2 else image.shape[0]
    sh = make_shard(_n_views(geom), rank, world, batch, dihedral)
    if sh.count == 0:
        return None, sh
    if sh.mode == "orbit":
        return forward_orbit(geom, image, sh.begin, sh.count, stream=stream), sh
    if sh.mode == "dihedral":
        return forward_dihedral(geom, image, sh.begin, sh.count, stream=stream), sh
    return forward(geom, image, view_begin=sh.begin, view_count=sh.count, stream=stream), sh


class MulticastImage:
    """The image buffer of the fused reduction (CBP_ACC_MULTIMEM): one n x n
    FP32 buffer per rank in torch symmetric memory, bound to an NVLink
    multicast object.  The BP adds every finished tile into all ranks' copies
    through ``multicast_ptr`` (the NVSwitch sums them), so no NCCL call follows
    the BP.  Raises RuntimeError where the system has no multicast support
    (e.g. a single GPU, or no NVSwitch)."""

    def __init__(self, n: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        device = device or torch.device("cuda", torch.cuda.current_device())
        group = group or dist.group.WORLD
        self.buf = symm_mem.empty((n, n), dtype=torch.float32, device=device)
        self.hdl = symm_mem.rendezvous(self.buf, group)
        # has_multicast_support is a static query (device type, index); the
        # handle's multicast_ptr is 0 when the group got no multicast object
        from torch._C._distributed_c10d import _SymmetricMemory
        dev_ok = _SymmetricMemory.has_multicast_support(symm_mem.DeviceType.CUDA, self.buf.device.index)
        self.mc = int(self.hdl.multicast_ptr) if dev_ok else 0
        if not self.mc:
            raise RuntimeError("no NVLink multicast support for this group")

    def barrier(self):
        self.hdl.barrier(channel=0)


def back_sharded(geom, sino_local, shard: Shard, image=None, group=None, dst: Optional[int] = None,
                 back: Callable = _cbp.back, back_orbit: Callable = _cbp.back_orbit,
                 back_dihedral: Callable = _cbp.back_dihedral, stream=None,
                 multimem: Optional[MulticastImage] = None):
    """c = sum_g A_g^T y_g: back-projects this rank's views, then sums the
    partial images over the group (all_reduce, or reduce to `dst`).  With
    `multimem` the sum is fused into the BP instead (CBP_ACC_MULTIMEM: every
    rank's BP adds its tiles into all ranks' ``multimem.buf`` through the
    multicast address; barriers before and after) and ``multimem.buf`` is
    returned."""
    import contextlib

    import torch
    import torch.distributed as dist
    rank, world = _rank_world(group)
    # the zero fill and the collective run on the BP's stream (NCCL enqueues on
    # torch's current stream: a different `stream` would let it read the
    # partial image before the BP has written it)
    on_bp_stream = contextlib.nullcontext()
    ref = image if image is not None else sino_local
    if stream is not None and isinstance(ref, torch.Tensor) and ref.is_cuda:
        s = stream if isinstance(stream, torch.cuda.Stream) else torch.cuda.ExternalStream(int(stream))
        on_bp_stream = torch.cuda.stream(s)
    if multimem is not None:
        with on_bp_stream:
            multimem.buf.zero_()
            multimem.barrier()  # every copy is zero before any rank adds
            if shard.count > 0:
                _cbp.back_multimem(geom, sino_local, multimem.mc, shard=shard, stream=stream)
            multimem.barrier()  # every rank's adds have landed
        return multimem.buf
    if shard.count > 0:
        if shard.mode == "orbit":
            image = back_orbit(geom, sino_local, shard.begin, image=image, stream=stream)
        elif shard.mode == "dihedral":
            image = back_dihedral(geom, sino_local, shard.begin, shard.count, image=image, stream=stream)
        else:
            image = back(geom, sino_local, image, view_begin=shard.begin, stream=stream)
    elif image is None:
        raise ValueError("a rank without views needs an image buffer to receive the sum")
    with on_bp_stream:
        if shard.count == 0:
            image[...] = 0
        if world > 1:
            t = image if isinstance(image, torch.Tensor) else torch.from_numpy(image)
            if dst is None:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            else:
                dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return image


def normal_sharded(geom, image, group=None, stream=None, dihedral: bool = False, **fns):
    """A^T A c over the group (one FP+BP pair, the benchmark's step)."""
    fwd = {k: v for k, v in fns.items() if k in ("forward", "forward_orbit", "forward_dihedral")}
    bwd = {k: v for k, v in fns.items() if k in ("back", "back_orbit", "back_dihedral")}
    y, sh = forward_sharded(geom, image, group=group, stream=stream, dihedral=dihedral, **fwd)
    return back_sharded(geom, y, sh, group=group, stream=stream, **bwd)
