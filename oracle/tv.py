"""Row f4 oracle: isotropic total variation and ASD-POCS, plain numpy FP64.

TEST INFRASTRUCTURE ONLY (see cnsf_oracle.h): used by tests/ and the f4
study's CPU cross-check, never by the product path.

* TV (the regulariser of ASD-POCS):
      TV(c) = sum_{r,c} sqrt(dx^2 + dy^2 + eps^2),
  dx = c[r, c+1] - c[r, c], dy = c[r+1, c] - c[r, c] (forward differences),
  reflective boundary (the difference past the last row / column is 0),
  eps = 1e-8; tv_gradient is its exact analytic gradient.
* ASD-POCS (Sidky & Pan 2008, cited at P:547; schedule per S:368-375 and
  DESIGN.md ledger #21): per iteration
      x_d = SART sweep from x over the ordered view subsets (positivity after
            each subset);  dp = |x_d - x|
      step = alpha dp;  n_tv times: x <- x - step grad TV(x) / |grad TV(x)|
      dg = |x - x_d|;  if dg > r_max dp: alpha <- alpha alpha_red
      beta <- beta beta_red
  SART(x, beta) = x + beta A^T((y - A x) / A1) / A^T 1 (zero-guard 1e-12).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

EPS_TV = 1e-8


def _diffs(c: np.ndarray):
    dx = np.zeros_like(c)
    dy = np.zeros_like(c)
    dx[..., :, :-1] = c[..., :, 1:] - c[..., :, :-1]
    dy[..., :-1, :] = c[..., 1:, :] - c[..., :-1, :]
    return dx, dy


def tv_value(c: np.ndarray, eps: float = EPS_TV) -> float:
    dx, dy = _diffs(np.asarray(c, dtype=np.float64))
    return float(np.sqrt(dx * dx + dy * dy + eps * eps).sum())


def tv_gradient(c: np.ndarray, eps: float = EPS_TV) -> np.ndarray:
    """d TV / d c: pixel (r, c) enters its own term (as -dx - dy) and the
    terms of its left neighbour (as +dx) and upper neighbour (as +dy)."""
    c = np.asarray(c, dtype=np.float64)
    dx, dy = _diffs(c)
    mag = np.sqrt(dx * dx + dy * dy + eps * eps)
    gx, gy = dx / mag, dy / mag
    g = -(gx + gy)
    g[..., :, 1:] += gx[..., :, :-1]
    g[..., 1:, :] += gy[..., :-1, :]
    return g


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
    subsets: int = 1
    eps_tv: float = EPS_TV


def sart_step(x, y, fwd: Callable, back: Callable, rows, cols, beta: float):
    r = np.where(rows > 1e-12, (y - fwd(x)) / np.where(rows > 1e-12, rows, 1.0), 0.0)
    return x + beta * np.where(cols > 1e-12, back(r) / np.where(cols > 1e-12, cols, 1.0), 0.0)


def _order(count):
    """bit-reversed order for a power of two, else golden-ratio stepping"""
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


def asd_pocs(y: np.ndarray, n: int, fwd: Callable, back: Callable, cfg: AsdPocsConfig,
             log: list | None = None) -> np.ndarray:
    """fwd(c, v0, nv) -> rows v0..v0+nv-1; back(r, v0) -> image (view blocks);
    with cfg.subsets == 1 they are called with the whole view range."""
    nviews = y.shape[0]
    base, rem = divmod(nviews, cfg.subsets)
    blocks, v = [], 0
    for i in range(cfg.subsets):
        m = base + (1 if i < rem else 0)
        blocks.append((v, m))
        v += m
    rows = [fwd(np.ones((n, n)), v0, m) for v0, m in blocks]
    cols = [back(np.ones((m, y.shape[1])), v0) for v0, m in blocks]
    x = np.zeros((n, n))
    beta, alpha = cfg.beta0, cfg.alpha
    for it in range(cfg.n_iterations):
        xd = x.copy()
        for b in _order(len(blocks)):
            v0, m = blocks[b]
            xd = sart_step(xd, y[v0:v0 + m], lambda c: fwd(c, v0, m), lambda s: back(s, v0),
                           rows[b], cols[b], beta)
            if cfg.nonneg:
                xd = np.maximum(xd, 0.0)
        dp = float(np.linalg.norm(xd - x))
        step = alpha * dp
        x = xd.copy()
        for _ in range(cfg.n_tv):
            g = tv_gradient(x, cfg.eps_tv)
            gn = float(np.linalg.norm(g))
            if gn > 0.0:
                x = x - step * g / gn
        dg = float(np.linalg.norm(x - xd))
        if dg > cfg.r_max * dp:
            alpha *= cfg.alpha_red
        beta *= cfg.beta_red
        if log is not None:
            log.append(dict(it=it, dp=dp, dg=dg, alpha=alpha, beta=beta))
    return x


def snr_db(rec: np.ndarray, truth: np.ndarray) -> float:
    """20 log10(|truth| / |rec - truth|), capped at 300 dB."""
    err = float(np.linalg.norm(np.asarray(rec, np.float64) - truth))
    if err == 0.0:
        return 300.0
    return min(300.0, 20.0 * np.log10(float(np.linalg.norm(truth)) / err))
