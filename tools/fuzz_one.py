"""Debug probe for fuzz seeds: the GPU FP of a single view against the oracle,
with the bin width varied across the K = 6 / 7 boundary of the FP's
candidates per line (K > 6 takes the generic walk)."""
import sys
import numpy as np
import torch

sys.path.insert(0, '.')
import oracle as O  # noqa: E402
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402
from tests.test_gpu_fuzz import draw  # noqa: E402

g, batch, v0, nv, rng = draw(int(sys.argv[1]) if len(sys.argv) > 1 else 665)
n = g["n"]
img = W.random_image(n, 1) + 0.5
for tw in (2.0, 3.0, 3.5, g["det_width"] / g["det_pitch"] * g["det_pitch"] / g["det_pitch"], 2.4, 2.2):
    gg = dict(g, det_width=tw * g["det_pitch"])
    for v in (4, 5, 10):
        want = O.forward(gg, img, view_begin=v, view_count=1)[0]
        got = cbp.forward(gg, torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).cuda(),
                          view_begin=v, view_count=1).cpu().numpy()[0]
        print(f"tau/pitch {tw:.3f} view {v} rel {np.abs(got - want).max() / np.abs(want).max():.2e}", got, want)
