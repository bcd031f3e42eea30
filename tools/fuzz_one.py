"""Debug probe for a fuzz seed: FP and BP of the CUDA path against the oracle,
per view (FP) and overall (BP), for batch 1 and the seed's batch."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import oracle as O  # noqa: E402
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402
from tests.test_gpu_fuzz import draw  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1670
g, batch, v0, nv, rng = draw(seed)
print(g, batch, v0, nv)
n = g["n"]
imgs = W.random_image(n, 500 + seed, batch=batch) if batch > 1 else W.random_image(n, 500 + seed)[None]
for bb in sorted({1, batch}):
    x = np.ascontiguousarray(imgs[:bb], dtype=np.float32)
    want = O.forward(g, x, view_begin=v0, view_count=nv)
    got = cbp.forward(g, torch.from_numpy(x).cuda(), view_begin=v0, view_count=nv).cpu().numpy()
    d = np.abs(got - want).max(axis=(0, 2)) / np.abs(want).max()
    print("FP batch", bb, "bad views", [(int(v), float(d[v])) for v in np.where(d > 1e-4)[0]][:12])
    for v in np.where(d > 1e-4)[0][:3]:
        print("   view", int(v), "got", got[0, v], "want", want[0, v])
