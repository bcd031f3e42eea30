"""ncu driver for one dihedral view shard (the W = 8 launch
list): warm-up plus a few FP+BP pairs of rank 1's shard of a W-rank split.
usage: python tools/shard_once.py [config] [world]"""
import sys
sys.path.insert(0, '.')
import torch
import paper_1907_10526_b200 as cbp
from paper_1907_10526_b200 import sharded
import workloads as W
g = W.geometry(sys.argv[1] if len(sys.argv) > 1 else "2")
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
y = torch.zeros((g["n_views"], g["n_det"]), device="cuda")
out = torch.empty_like(img)
sh = sharded.make_shard(g["n_views"], 1, world, dihedral=True)
for _ in range(4):
    cbp.forward_dihedral(g, img, sh.begin, sh.count, sino=y)
    cbp.back_dihedral(g, y, sh.begin, sh.count, image=out)
torch.cuda.synchronize()
print("ok", sh)
