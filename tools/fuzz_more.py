import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, paper_1907_10526_b200 as cbp, workloads as W
from tests.test_gpu_fuzz import draw
from tests.test_gpu_parity import _metrics
bad = 0
for seed in range(160, 700):
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
        if not ok:
            bad += 1
            print("FAIL", seed, what, r, g, batch, v0, nv, flush=True)
print("done, failures:", bad)
