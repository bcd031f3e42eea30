"""Small driver for ncu: W warm-up FP+BP pairs then ONE pair of the given
config (default 2), all through the C ABI on cuda:0.  Usage:
  python tools/prof_step.py [config] [warmup] [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g = W.geometry(cfg)
img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
if batch > 1:
    img = img.expand(batch, -1, -1).contiguous()
for _ in range(warm + 1):
    y = cbp.forward(g, img)
    c = cbp.back(g, y)
torch.cuda.synchronize()
print("ok", float(y.sum()), float(c.sum()), "launches", cbp.launch_count())
