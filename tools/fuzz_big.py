"""Randomised parity on larger grids (n 100..520, several BP tiles, ragged
edges) with few views (8..40, multiples of 8 included: the 4- and 8-fold
paths), every kind and model, batches 1..4; FP and BP against the oracle.
usage: python tools/fuzz_big.py LO HI"""
import sys

import numpy as np
import torch

lo, hi = int(sys.argv[1]), int(sys.argv[2])
sys.argv = ['x', '0', '0']
exec(open('tools/fuzz_wide.py').read().split('lo, hi =')[0])
from tests.test_gpu_parity import _metrics  # noqa: E402

bad = tried = 0
for seed in range(lo, hi):
    rng = np.random.default_rng(70000 + seed)
    g, _, _, _ = draw(seed)
    n = int(rng.integers(100, 521))
    h = g["pixel"]
    R = n * h / np.sqrt(2.0)
    kind = g["kind"]
    sid = float(R * np.exp(rng.uniform(np.log(1.15), np.log(15.0))))
    sdd = float(sid * rng.uniform(1.0, 3.0))
    pitch = float(np.exp(rng.uniform(np.log(0.3), np.log(3.0)))) * h
    width = float(np.exp(rng.uniform(np.log(0.2), np.log(4.0)))) * pitch
    span = 2 * R if kind == 1 else 2 * sdd * np.tan(np.arcsin(min(R / sid, 0.999)))
    n_det = max(1, min(3000, int(span / pitch * rng.uniform(0.7, 1.2))))
    g = dict(g, n=n, sid=sid if kind != 1 else 0.0, sdd=sdd if kind != 1 else 0.0, det_pitch=pitch,
             det_width=min(width, 1.9 * sdd) if kind != 1 else width, n_det=n_det,
             n_views=int(rng.choice([8, 12, 16, 24, 40])))
    while kind == 2 and g["n_det"] > 1 and cbp.validate(g) != cbp.CBP_OK:
        g["n_det"] -= 1
    if cbp.validate(g) != cbp.CBP_OK:
        continue
    batch = int(rng.choice([1, 1, 2, 4]))
    tried += 1
    imgs = W.random_image(n, seed, batch=batch) if batch > 1 else W.random_image(n, seed)
    y = W.random_sino(g["n_views"], g["n_det"], seed + 7, batch=batch) if batch > 1 else \
        W.random_sino(g["n_views"], g["n_det"], seed + 7)
    want = O.forward(g, imgs)
    got = cbp.forward(g, torch.from_numpy(np.ascontiguousarray(imgs, dtype=np.float32)).cuda()).cpu().numpy()
    wantb = O.back(g, y)
    gotb = cbp.back(g, torch.from_numpy(y).cuda()).cpu().numpy()
    for what, a, b in (("FP", got, want), ("BP", gotb, wantb)):
        if np.abs(b).max() == 0:
            continue
        r = _metrics(a, b)
        if not (r[0] <= 1e-5 and r[1] <= 1e-4):
            bad += 1
            print("FAIL", seed, what, r, g, batch, flush=True)
print("done", tried, "scanners, failures:", bad)
