"""Randomised FP / BP parity against the oracle over a range of fuzz seeds
(tests/test_gpu_fuzz.draw); prints the failures.  usage: python tools/fuzz_more.py LO HI"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, paper_1907_10526_b200 as cbp, workloads as W
from tests.test_gpu_fuzz import draw
from tests.test_gpu_parity import _metrics
bad = 0
lo, hi = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (160, 700)
for seed in range(lo, hi):
    g, batch, v0, nv, rng = draw(seed)
    n = g["n"]
    imgs = W.random_image(n, 500 + seed, batch=batch) if batch > 1 else W.random_image(n, 500 + seed)
    want = O.forward(g, imgs, view_begin=v0, view_count=nv)
    got = cbp.forward(g, torch.from_numpy(np.ascontiguousarray(imgs, dtype=np.float32)).cuda(), view_begin=v0, view_count=nv).cpu().numpy()
    y = W.random_sino(nv, g["n_det"], 600 + seed, batch=batch) if batch > 1 else W.random_sino(nv, g["n_det"], 600 + seed)
    wantb = O.back(g, y, view_begin=v0)
    gotb = cbp.back(g, torch.from_numpy(y).cuda(), view_begin=v0).cpu().numpy()
    for what, a, b in (("FP", got, want), ("BP", gotb, wantb)):
        if np.abs(b).max() == 0:
            ok = not a.any()
            r = (0, 0)
        else:
            r = _metrics(a, b); ok = r[0] <= 1e-5 and r[1] <= 1e-4
            # a projection holding only support-edge tails (max|y| far below a pixel's
            # chord, h): the max-normalised metric is meaningless there; FP32's
            # absolute accuracy (~1e-7 of a full weight) is the bar
            scale = g["pixel"] * max(float(np.abs(imgs).max()), 1.0) if what == "FP" else g["pixel"] * float(np.abs(y).max())
            if not ok and np.abs(b).max() < 1e-2 * scale:
                ok = np.abs(a - b).max() <= 1e-6 * scale
        if not ok:
            bad += 1
            print("FAIL", seed, what, r, g, batch, v0, nv, flush=True)
print("done, failures:", bad)
