"""Small driver for ncu on the magnified-footprint model (row f3): W warm-up
FP+BP pairs then one pair of the given config with model = 1.
usage: python tools/prof_mag.py [config] [warmup]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = dict(W.geometry(cfg), model=1)
img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
for _ in range(warm + 1):
    y = cbp.forward(g, img)
    c = cbp.back(g, y)
torch.cuda.synchronize()
print("ok", float(y.sum()), float(c.sum()))
