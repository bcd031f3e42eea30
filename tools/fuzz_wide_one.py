"""Debug probe for a tools/fuzz_wide.py seed: per-view FP errors against the
oracle (batch 1), the worst bins, and the BP error."""
import sys

import numpy as np
import torch

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1348
sys.argv = ['x', '0', '0']
exec(open('tools/fuzz_wide.py').read().split('lo, hi =')[0])
from tests.test_gpu_parity import _metrics  # noqa: E402

g, batch, v0, nv = draw(seed)
print(g, batch, v0, nv)
img = W.random_image(g["n"], seed)
want = O.forward(g, img, view_begin=v0, view_count=nv)
got = cbp.forward(g, torch.from_numpy(img).cuda(), view_begin=v0, view_count=nv).cpu().numpy()
print("FP batch 1", _metrics(got, want))
d = np.abs(got - want)
peak = np.abs(want).max()
for v in np.argsort(-d.max(axis=1))[:4]:
    j = int(d[v].argmax())
    print(f"  view {v0 + v}: worst bin {j} got {got[v, j]:.6g} want {want[v, j]:.6g} (err/peak {d[v, j] / peak:.2e})")
for nmod in (dict(), dict(n_views=g["n_views"] + 1)):
    gg = dict(g, **nmod)
    y = W.random_sino(gg["n_views"], gg["n_det"], 7)
    print("BP", nmod, _metrics(cbp.back(gg, torch.from_numpy(y).cuda()).cpu().numpy(), O.back(gg, y)))
