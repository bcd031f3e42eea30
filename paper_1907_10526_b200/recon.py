"""Row f1: iterative reconstruction around the projector --
SART and CGLS, view-sharded over the GPUs of a process group exactly like
the projector (``sharded.py``): each rank forward-projects its views, forms
its residual rows locally, and the back-projected partial images (and the
CGLS scalars) are summed with NCCL all_reduce.

* SART (the data step of ASD-POCS):
      c <- max(c + beta A^T((y - A c) ./ A 1) ./ A^T 1, 0)
  (a zero-guard 1e-12 on the weight sums).
* CGLS (conjugate gradients on the normal equations A^T A c = A^T y), with
  the step lengths kept in device FP64 scalars (no host round trip).

Every vector operation runs in libcbp.so (``cbp_sart_*``, ``cbp_dot``,
``cbp_cgls_*``); torch provides buffers and the collectives.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

import paper_1907_10526_b200 as cbp
from paper_1907_10526_b200 import sharded


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


class ShardedOperator:
    """A (this rank's views) and A^T (summed over the group) for one image."""

    def __init__(self, geom, device=None, group=None):
        self.g = geom
        self.group = group
        self.rank, self.world = _world(group)
        self.shard = sharded.make_shard(geom["n_views"], self.rank, self.world)
        self.views = torch.as_tensor(self.shard.views(), dtype=torch.long, device=device)
        self.n = geom["n"]
        self.device = device

    def local_rows(self, y_full: torch.Tensor) -> torch.Tensor:
        """this rank's rows of a full [n_views, n_det] sinogram, in its layout"""
        y = y_full.index_select(0, self.views)
        if self.shard.mode == "orbit":
            y = y.view(4, self.shard.count, -1)
        return y.contiguous()

    def fwd(self, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        sh = self.shard
        if sh.mode == "orbit":
            return cbp.forward_orbit(self.g, x, sh.begin, sh.count, sino=out)
        return cbp.forward(self.g, x, out, view_begin=sh.begin, view_count=sh.count)

    def adj(self, y: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        sh = self.shard
        if sh.mode == "orbit":
            img = cbp.back_orbit(self.g, y, sh.begin, image=out)
        else:
            img = cbp.back(self.g, y, out, view_begin=sh.begin)
        if self.world > 1:
            dist.all_reduce(img, group=self.group)
        return img

    def allreduce_scalar(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t


def sart(geom, y_full: torch.Tensor, iters: int, beta: float = 1.0, nonneg: bool = True,
         x0: Optional[torch.Tensor] = None, group=None,
         callback: Optional[Callable[[int, torch.Tensor], None]] = None) -> torch.Tensor:
    """SART from x0 (zeros) on the full measured sinogram y_full [n_views, n_det]."""
    op = ShardedOperator(geom, y_full.device, group)
    n = geom["n"]
    y = op.local_rows(y_full)
    ones = cbp.fill(torch.empty((n, n), device=y.device), 1.0)
    rowsum = op.fwd(ones)                              # A 1 (local rows)
    colsum = op.adj(cbp.fill(torch.empty_like(y), 1.0))  # A^T 1 (global)
    x = torch.zeros((n, n), device=y.device) if x0 is None else x0.clone()
    ax = torch.empty_like(y)
    r = torch.empty_like(y)
    bp = torch.empty_like(x)
    for it in range(iters):
        op.fwd(x, ax)
        cbp.sart_residual(y, ax, rowsum, r)
        op.adj(r, bp)
        cbp.sart_update(x, bp, colsum, beta, nonneg)
        if callback:
            callback(it, x)
    return x


def cgls(geom, y_full: torch.Tensor, iters: int, group=None,
         callback: Optional[Callable[[int, torch.Tensor], None]] = None) -> torch.Tensor:
    """CGLS from x = 0: minimises |y - A x|_2 over growing Krylov spaces."""
    op = ShardedOperator(geom, y_full.device, group)
    n = geom["n"]
    r = op.local_rows(y_full)           # r = y - A 0
    x = torch.zeros((n, n), device=r.device)
    s = op.adj(r)                       # s = A^T r
    p = s.clone()
    gamma = torch.zeros(1, dtype=torch.float64, device=r.device)
    gnew = torch.zeros_like(gamma)
    qq = torch.zeros_like(gamma)
    cbp.dot(s, s, gamma)
    q = torch.empty_like(r)
    for it in range(iters):
        op.fwd(p, q)
        cbp.dot(q, q, qq)
        op.allreduce_scalar(qq)         # |A p|^2 over all views
        cbp.cgls_step(x, p, r, q, gamma, qq)  # alpha = gamma / |Ap|^2
        op.adj(r, s)
        cbp.dot(s, s, gnew)
        cbp.cgls_direction(p, s, gnew, gamma)  # beta = gamma_new / gamma
        gamma.copy_(gnew)
        if callback:
            callback(it, x)
    return x
