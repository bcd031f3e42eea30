import sys
sys.argv = ['x', '0', '0']
src = open('tools/fuzz_wide.py').read().split('lo, hi =')[0]
exec(src)
import numpy as np, torch
from tests.test_gpu_parity import _metrics
for seed in (109, 1329, 1348, 2646, 2916, 2009, 997):
    g, batch, v0, nv = draw(seed)
    n = g["n"]
    imgs = W.random_image(n, seed, batch=batch) if batch > 1 else W.random_image(n, seed)
    y = W.random_sino(nv, g["n_det"], seed + 7, batch=batch) if batch > 1 else W.random_sino(nv, g["n_det"], seed + 7)
    want = O.forward(g, imgs, view_begin=v0, view_count=nv)
    got = cbp.forward(g, torch.from_numpy(np.ascontiguousarray(imgs, dtype=np.float32)).cuda(), view_begin=v0, view_count=nv).cpu().numpy()
    wantb = O.back(g, y, view_begin=v0)
    gotb = cbp.back(g, torch.from_numpy(y).cuda(), view_begin=v0).cpu().numpy()
    print(seed, "model", g["model"], "tau/h", round(g["det_width"] / g["pixel"], 4), "FP", _metrics(got, want), "BP", _metrics(gotb, wantb), flush=True)
