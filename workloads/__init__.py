"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests,
``bench.py`` and ``__graft_entry__.smoke()``.

This module holds NONE of the projector's arithmetic: only the scanner
numbers of each configuration, phantom rasterisation and seeded random draws.
Recipe:

* one scale-similar fan geometry for configs 1-5: SID = D_po = 500 mm,
  SDD = D_ps = 1000 mm, a 64 mm square field of view, pixel h = 64/n mm,
  detector pitch = bin width = 1.5 h, n_det = 2 n bins, views over [0, 2 pi);
* the paper's own timing shapes and accuracy set-ups
  (Fig. 5: P:414-416; Fig. 6: P:459-463; Fig. 7: P:482-486) as extra cases;
* images: Shepp-Logan (original 10-ellipse table, point-sampled at pixel
  centres, field of view mapped to [-1, 1]^2), U[0,1) images (seeds 1-3),
  U[0,1) sinograms (seeds 101-103), all-ones, single pixels,
  a 64-slice jittered Shepp-Logan batch (seed 7), area-weighted disks.
"""
from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# scanner configurations (plain numbers; BASELINE.json "configs")


def _fan(n: int, n_views: int, n_det: int | None = None) -> dict:
    h = 64.0 / n
    return dict(n=n, pixel=h, n_views=n_views, n_det=2 * n if n_det is None else n_det,
                det_pitch=1.5 * h, det_width=1.5 * h, sid=500.0, sdd=1000.0)


CONFIGS: dict[str, dict] = {
    # BASELINE.json configs[0]: 64x64, 90 views, 128 cells, SID 500 / SDD 1000
    "1": _fan(64, 90, 128),
    # configs[1]: 512^2 Shepp-Logan, 720 views, 1024 cells (the bench workload)
    "2": _fan(512, 720, 1024),
    # configs[2]: 1024^2, 1440 views, 2048 cells
    "3": _fan(1024, 1440, 2048),
    # configs[3]: batch of 64 512^2 slices, 720 views (geometry of config 2)
    "4": _fan(512, 720, 1024),
    # configs[4]: 2048^2, 2880 views, 4096 cells (SART/CGLS loop)
    "5": _fan(2048, 2880, 4096),
}
BATCH = {"1": 1, "2": 1, "3": 1, "4": 64, "5": 1}

# all-ones images of side 64..2048 mm (h = 1 mm), 360 views,
# tau = Delta_s = 1 mm, N_s and (D_po, D_so) per size.
PAPER_TIMING = {
    n: dict(n=n, pixel=1.0, n_views=360, n_det=ns, det_pitch=1.0, det_width=1.0,
            sid=float(d), sdd=2.0 * d)
    for n, ns, d in [(64, 205, 100), (128, 409, 200), (256, 815, 400), (512, 1627, 800),
                     (1024, 3250, 1600), (2048, 6499, 3200)]
}

# P:414-416 (Fig. 5): 1 mm pixel at the origin, tau = 0.5, D_po = D_so = 3,
# Delta_s = 0.01, N_s = 601; angles 0/15/35/45 deg are views 0/3/7/9 of 72.
FIG5 = dict(n=1, pixel=1.0, n_views=72, n_det=601, det_pitch=0.01, det_width=0.5, sid=3.0,
            sdd=6.0)
FIG5_VIEWS = (0, 3, 7, 9)

# P:459-463 (Fig. 6): tau = Delta_s = 0.5, D_po = D_so = 200; (a) pixel at the
# origin, 90 angles over 90 deg; (b) pixel at (100.5, 50.5), 360 over 360 deg.
FIG6 = dict(n=1, pixel=1.0, n_views=360, n_det=1101, det_pitch=0.5, det_width=0.5, sid=200.0,
            sdd=400.0)
FIG6B_PIXEL = (100.5, 50.5)

# P:482-486 (Fig. 7, Shepp-Logan row): 128 mm, N_s = 409, Delta_s = 1,
# tau = 0.5, D = 200/200, 360 angles.
FIG7 = dict(n=128, pixel=1.0, n_views=360, n_det=409, det_pitch=1.0, det_width=0.5, sid=200.0,
            sdd=400.0)


# Extra bench workloads for the general (non-symmetric) path and the paper's
# own timing shapes: config 2's geometry with 721 views (no
# 4- or 8-fold view symmetry: the direct kernels), and P:512-515's all-ones
# shapes at 256, 512 and 1024 mm.
EXTRA: dict[str, dict] = {
    "2v721": _fan(512, 721, 1024),
    "p256": dict(PAPER_TIMING[256]),
    "p512": dict(PAPER_TIMING[512]),
    "p1024": dict(PAPER_TIMING[1024]),
}


def geometry(name: str) -> dict:
    return dict(CONFIGS[name] if name in CONFIGS else EXTRA[name])


# ---------------------------------------------------------------------------
# phantoms and seeded draws

# Original Shepp-Logan table (x0, y0, a, b, phi_deg, intensity) on [-1,1]^2.
SHEPP_LOGAN = [
    (0.0, 0.0, 0.69, 0.92, 0.0, 2.0),
    (0.0, -0.0184, 0.6624, 0.874, 0.0, -0.98),
    (0.22, 0.0, 0.11, 0.31, -18.0, -0.02),
    (-0.22, 0.0, 0.16, 0.41, 18.0, -0.02),
    (0.0, 0.35, 0.21, 0.25, 0.0, 0.01),
    (0.0, 0.1, 0.046, 0.046, 0.0, 0.01),
    (0.0, -0.1, 0.046, 0.046, 0.0, 0.01),
    (-0.08, -0.605, 0.046, 0.023, 0.0, 0.01),
    (0.0, -0.605, 0.023, 0.023, 0.0, 0.01),
    (0.06, -0.605, 0.023, 0.046, 0.0, 0.01),
]
MODIFIED_INTENSITY = [1.0, -0.8, -0.2, -0.2, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1]


def _grid_norm(n: int):
    """pixel-centre coordinates mapped to [-1, 1]^2 (row 0 at +y)."""
    c = 0.5 * (n - 1)
    x = (np.arange(n) - c) / (0.5 * n)
    y = (c - np.arange(n)) / (0.5 * n)
    return np.meshgrid(x, y)  # X[row, col], Y[row, col]


def shepp_logan(n: int, modified: bool = False) -> np.ndarray:
    X, Y = _grid_norm(n)
    img = np.zeros((n, n), dtype=np.float64)
    for i, (x0, y0, a, b, phi, val) in enumerate(SHEPP_LOGAN):
        if modified:
            val = MODIFIED_INTENSITY[i]
        t = math.radians(phi)
        xr = (X - x0) * math.cos(t) + (Y - y0) * math.sin(t)
        yr = -(X - x0) * math.sin(t) + (Y - y0) * math.cos(t)
        img[(xr / a) ** 2 + (yr / b) ** 2 <= 1.0] += val
    return img.astype(np.float32)


def random_image(n: int, seed: int, batch: int | None = None) -> np.ndarray:
    rng = np.random.default_rng(seed)
    shape = (n, n) if batch is None else (batch, n, n)
    return rng.random(shape, dtype=np.float32)


def random_sino(n_views: int, n_det: int, seed: int, batch: int | None = None) -> np.ndarray:
    rng = np.random.default_rng(seed)
    shape = (n_views, n_det) if batch is None else (batch, n_views, n_det)
    return rng.random(shape, dtype=np.float32)


def ones(n: int) -> np.ndarray:
    return np.ones((n, n), dtype=np.float32)


def single_pixel(n: int, row: int, col: int, value: float = 1.0) -> np.ndarray:
    if not (0 <= row < n and 0 <= col < n):
        raise IndexError("pixel outside the grid")
    img = np.zeros((n, n), dtype=np.float32)
    img[row, col] = value
    return img


def jittered_batch(n: int, batch: int = 64, seed: int = 7) -> np.ndarray:
    """config 4: Shepp-Logan x (1 + 0.1 U[-1,1]) per pixel, per slice."""
    rng = np.random.default_rng(seed)
    base = shepp_logan(n).astype(np.float64)
    jit = 1.0 + 0.1 * rng.uniform(-1.0, 1.0, size=(batch, n, n))
    return (base[None] * jit).astype(np.float32)


def disk(n: int, pixel: float, center: tuple[float, float], radius: float,
         supersample: int = 8) -> np.ndarray:
    """area-weighted indicator of a disk (mm units), supersample^2 points per pixel."""
    c = 0.5 * (n - 1)
    off = (np.arange(supersample) + 0.5) / supersample - 0.5
    xs = ((np.arange(n) - c)[:, None] + off[None, :]).reshape(-1) * pixel
    ys = ((c - np.arange(n))[:, None] - off[None, :]).reshape(-1) * pixel
    X, Y = np.meshgrid(xs, ys)
    inside = ((X - center[0]) ** 2 + (Y - center[1]) ** 2 < radius ** 2).astype(np.float64)
    return inside.reshape(n, supersample, n, supersample).mean(axis=(1, 3)).astype(np.float32)
