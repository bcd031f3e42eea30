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
* ASD-POCS (row f4; Sidky & Pan 2008; schedule DESIGN.md ledger
  #21): SART with positivity, then n_tv normalised TV-gradient steps of
  length alpha |data step|, alpha reduced when the TV steps outgrow r_max
  |data step|.  The TV steps act on the full image, identically on every
  rank (the image is replicated after the BP all-reduce).

Every vector operation runs in libcbp.so (``cbp_sart_*``, ``cbp_dot``,
``cbp_cgls_*``); torch provides buffers and the collectives.
"""
from __future__ import annotations

from dataclasses import dataclass
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


@dataclass
class AsdPocsConfig:
    n_iterations: int = 50
    beta0: float = 1.0
    beta_red: float = 0.995
    n_tv: int = 20
    alpha: float = 0.2
    alpha_red: float = 0.95
    r_max: float = 0.95
    nonneg: bool = True
    subsets: int = 1  # ordered subsets of contiguous views (> 1: one device)
    eps_tv: float = 1e-8  # TV smoothing (ledger #20)


def subset_order(count: int) -> list[int]:
    """Visiting order of `count` ordered subsets with large angular jumps:
    bit-reversed when count is a power of two, else golden-ratio stepping."""
    if count & (count - 1) == 0:
        bits = max(1, count.bit_length() - 1)
        return [int(format(i, f"0{bits}b")[::-1], 2) for i in range(count)] if count > 1 else [0]
    order, seen, k = [], set(), 0
    step = max(1, round(count * 0.6180339887))
    while len(order) < count:
        while k in seen:
            k = (k + 1) % count
        order.append(k)
        seen.add(k)
        k = (k + step) % count
    return order


def view_subsets(n_views: int, count: int) -> list[tuple[int, int]]:
    """contiguous view blocks (begin, size) of `count` near-equal subsets"""
    base, rem = divmod(n_views, count)
    out, v = [], 0
    for i in range(count):
        m = base + (1 if i < rem else 0)
        out.append((v, m))
        v += m
    return out


def cnsf_ops(geom):
    """(fwd, adj) over a view block with the CNSF library projector"""
    def fwd(x, out, v0, nv):
        return cbp.forward(geom, x, out, view_begin=v0, view_count=nv)

    def adj(r, out, v0):
        return cbp.back(geom, r, out, view_begin=v0)
    return fwd, adj


def asd_pocs(geom, y_full: torch.Tensor, cfg: AsdPocsConfig, group=None, ops=None,
             callback: Optional[Callable[[int, torch.Tensor], None]] = None) -> torch.Tensor:
    """ASD-POCS from zero on the measured sinogram y_full [n_views, n_det].

    ops = (fwd(x, out, v0, nv), adj(r, out, v0)) over view blocks; default:
    the CNSF projector, sharded over `group` when cfg.subsets == 1."""
    n, nviews = geom["n"], geom["n_views"]
    dev = y_full.device
    if ops is None and cfg.subsets == 1:
        op = ShardedOperator(geom, dev, group)
        y = op.local_rows(y_full)
        blocks = [(lambda x, out: op.fwd(x, out), lambda r, out: op.adj(r, out), y)]
    else:
        fwd, adj = ops if ops is not None else cnsf_ops(geom)
        blocks = []
        for v0, nv in view_subsets(nviews, cfg.subsets):
            blocks.append((lambda x, out, v0=v0, nv=nv: fwd(x, out, v0, nv),
                           lambda r, out, v0=v0: adj(r, out, v0), y_full[v0:v0 + nv].contiguous()))
    order = subset_order(len(blocks))
    ones = cbp.fill(torch.empty((n, n), device=dev), 1.0)
    rows = [f(ones, torch.empty_like(yb)) for f, _, yb in blocks]
    cols = [a(cbp.fill(torch.empty_like(yb), 1.0), torch.empty((n, n), device=dev)) for _, a, yb in blocks]
    x = torch.zeros((n, n), device=dev)
    xd = torch.empty_like(x)
    ax = [torch.empty_like(yb) for _, _, yb in blocks]
    r = [torch.empty_like(yb) for _, _, yb in blocks]
    bp, grad = torch.empty_like(x), torch.empty_like(x)
    d64 = dict(dtype=torch.float64, device=dev)
    alpha = torch.full((1,), cfg.alpha, **d64)
    dp2, dg2, gg = torch.zeros(1, **d64), torch.zeros(1, **d64), torch.zeros(1, **d64)
    beta = cfg.beta0
    for it in range(cfg.n_iterations):
        xd.copy_(x)
        for b in order:  # the data (POCS) step: SART over the ordered subsets
            f, a, yb = blocks[b]
            f(xd, ax[b])
            cbp.sart_residual(yb, ax[b], rows[b], r[b])
            a(r[b], bp)
            cbp.sart_update(xd, bp, cols[b], beta, cfg.nonneg)
        cbp.diff_norm2(xd, x, dp2)
        x.copy_(xd)
        for _ in range(cfg.n_tv):  # the TV steepest-descent steps
            cbp.tv_gradient(x, grad, cfg.eps_tv)
            cbp.dot(grad, grad, gg)
            cbp.tv_step(x, grad, gg, alpha, dp2)
        cbp.diff_norm2(x, xd, dg2)
        cbp.asd_adapt(alpha, dp2, dg2, cfg.r_max, cfg.alpha_red)
        beta *= cfg.beta_red
        if callback:
            callback(it, x)
    return x
