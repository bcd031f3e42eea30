"""A wider randomised sweep than tests/test_gpu_fuzz.py: harder scanners
(sources 1.05 field radii away, tau / Delta_s up to 6, pixels down to 0.1 mm,
batches up to 8), FP and BP of the CUDA path against the oracle.
usage: python tools/fuzz_wide.py LO HI"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import oracle as O  # noqa: E402
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402
from tests.test_gpu_parity import _metrics  # noqa: E402


def draw(seed):
    rng = np.random.default_rng(90000 + seed)
    kind = int(rng.integers(0, 3))
    model = int(rng.random() < 0.3)
    n = int(rng.integers(1, 161))
    h = float(np.exp(rng.uniform(np.log(0.1), np.log(3.0))))
    n_views = int(rng.choice([1, 2, 4, 7, 8, 12, 16, 36, 60, 64, 100, 120]))
    pitch = float(np.exp(rng.uniform(np.log(0.2), np.log(4.0)))) * h
    R = n * h / np.sqrt(2.0)
    sid = float(R * np.exp(rng.uniform(np.log(1.05), np.log(20.0))) + 0.01 * h)
    sdd = float(sid * rng.uniform(1.0, 4.0))
    width = float(np.exp(rng.uniform(np.log(0.02), np.log(6.0)))) * pitch
    if kind != 1:
        width = min(width, 1.9 * sdd)
    span = 2 * R if kind == 1 else 2 * sdd * np.tan(np.arcsin(min(R / sid, 0.999)))
    n_det = max(1, min(2000, int(span / pitch * rng.uniform(0.5, 1.4)) + int(rng.integers(0, 5))))
    g = dict(n=n, pixel=h, n_views=n_views, n_det=n_det, det_pitch=pitch, det_width=width,
             sid=sid if kind != 1 else 0.0, sdd=sdd if kind != 1 else 0.0, kind=kind, model=model)
    while kind == 2 and g["n_det"] > 1 and cbp.validate(g) != cbp.CBP_OK:
        g["n_det"] -= 1
    batch = int(rng.choice([1, 1, 1, 2, 3, 4, 5, 8]))
    full = rng.random() < 0.6
    v0 = 0 if full else int(rng.integers(0, n_views))
    nv = n_views - v0 if full else int(rng.integers(1, n_views - v0 + 1))
    return g, batch, v0, nv


lo, hi = int(sys.argv[1]), int(sys.argv[2])
bad = 0
for seed in range(lo, hi):
    g, batch, v0, nv = draw(seed)
    if cbp.validate(g) != cbp.CBP_OK:
        continue
    n = g["n"]
    imgs = W.random_image(n, seed, batch=batch) if batch > 1 else W.random_image(n, seed)
    y = W.random_sino(nv, g["n_det"], seed + 7, batch=batch) if batch > 1 else W.random_sino(nv, g["n_det"], seed + 7)
    want = O.forward(g, imgs, view_begin=v0, view_count=nv)
    got = cbp.forward(g, torch.from_numpy(np.ascontiguousarray(imgs, dtype=np.float32)).cuda(),
                      view_begin=v0, view_count=nv).cpu().numpy()
    wantb = O.back(g, y, view_begin=v0)
    gotb = cbp.back(g, torch.from_numpy(y).cuda(), view_begin=v0).cpu().numpy()
    for what, a, b, scale in (("FP", got, want, g["pixel"]), ("BP", gotb, wantb, g["pixel"])):
        if np.abs(b).max() == 0:
            ok, r = not a.any(), (0, 0)
        else:
            r = _metrics(a, b)
            ok = r[0] <= 1e-5 and r[1] <= 1e-4
            if not ok and np.abs(b).max() < 1e-2 * scale:  # support-edge tails only
                ok = np.abs(a - b).max() <= 1e-6 * scale
        if not ok:
            bad += 1
            print("FAIL", seed, what, r, g, batch, v0, nv, flush=True)
print("done", hi - lo, "draws, failures:", bad)
