"""Randomised check of the FP64 reference projector pair (row f2) against the
oracle's on small random scanners of tools/fuzz_wide.py (relative 1e-9).
usage: python tools/fuzz_ref.py LO HI"""
import sys

import numpy as np
import torch

lo, hi = int(sys.argv[1]), int(sys.argv[2])
sys.argv = ['x', '0', '0']
exec(open('tools/fuzz_wide.py').read().split('lo, hi =')[0])

bad = tried = 0
for seed in range(lo, hi):
    g, batch, v0, nv = draw(seed)
    if g["n"] > 24 or cbp.validate(g) != cbp.CBP_OK:
        continue
    g = dict(g, n_views=min(g["n_views"], 12), n_det=min(g["n_det"], 200))
    if cbp.validate(g) != cbp.CBP_OK:
        continue
    tried += 1
    img = W.random_image(g["n"], seed)
    want = O.ref_forward(g, img.astype(np.float64))
    got = cbp.ref_forward(g, torch.from_numpy(img).cuda()).cpu().numpy()
    y = W.random_sino(g["n_views"], g["n_det"], seed + 3).astype(np.float64)
    wb = O.ref_back(g, y)
    gb = cbp.ref_back(g, torch.from_numpy(y).cuda()).cpu().numpy()
    for what, a, b in (("FP", got, want), ("BP", gb, wb)):
        m = np.abs(b).max()
        err = np.abs(a - b).max() / m if m > 0 else np.abs(a).max()
        if not err <= 1e-9:
            bad += 1
            print("FAIL", what, seed, err, g, flush=True)
print("done", tried, "scanners, failures:", bad)
