"""Randomised check of the view-shard calls (orbit, dihedral) on the harder
scanners of tools/fuzz_wide.py: each shard's FP rows equal the full FP's
rows and the shards' BPs sum to the full BP (GPU against GPU, the parity
bar), for 2..8 emulated ranks.  usage: python tools/fuzz_shards.py LO HI"""
import sys

import numpy as np
import torch

lo, hi = int(sys.argv[1]), int(sys.argv[2])
sys.argv = ['x', '0', '0']
exec(open('tools/fuzz_wide.py').read().split('lo, hi =')[0])
from paper_1907_10526_b200 import sharded  # noqa: E402
from tests.test_gpu_parity import _metrics  # noqa: E402

bad = tried = 0
for seed in range(lo, hi):
    g, batch, v0, nv = draw(seed)
    N = g["n_views"]
    if N % 4 or cbp.validate(g) != cbp.CBP_OK:
        continue
    tried += 1
    img = torch.from_numpy(W.random_image(g["n"], seed)).cuda()
    y = torch.from_numpy(W.random_sino(N, g["n_det"], seed + 1)).cuda()
    full_y = cbp.forward(g, img)
    full_c = cbp.back(g, y)
    for world in (2, 3, 8):
        for dihedral in (False, True):
            if dihedral and N % 8:
                continue
            total = torch.zeros_like(full_c)
            for r in range(world):
                sh = sharded.make_shard(N, r, world, dihedral=dihedral)
                if sh.count == 0:  # more ranks than views: nothing to do (sharded.py returns None)
                    continue
                rows = torch.as_tensor(sh.views(), device="cuda")
                if sh.mode == "dihedral":
                    ys = cbp.forward_dihedral(g, img, sh.begin, sh.count)[rows]
                    total += cbp.back_dihedral(g, y, sh.begin, sh.count)
                elif sh.mode == "orbit":
                    ys = cbp.forward_orbit(g, img, sh.begin, sh.count).reshape(-1, g["n_det"])
                    cbp.back_orbit(g, y[rows].reshape(4, sh.count, -1).contiguous(), sh.begin, image=total,
                                   accumulate=True)
                else:
                    ys = cbp.forward(g, img, view_begin=sh.begin, view_count=sh.count)
                    cbp.back(g, y[rows].contiguous(), image=total, view_begin=sh.begin, accumulate=True)
                want = full_y[rows]
                if want.abs().max() > 0:
                    r_fp = _metrics(ys.cpu().numpy(), want.cpu().numpy())
                    if not (r_fp[0] <= 1e-5 and r_fp[1] <= 1e-4):
                        bad += 1
                        print("FAIL FP", seed, world, dihedral, r, r_fp, g, flush=True)
            torch.cuda.synchronize()
            if full_c.abs().max() > 0:
                r_bp = _metrics(total.cpu().numpy(), full_c.cpu().numpy())
                if not (r_bp[0] <= 1e-5 and r_bp[1] <= 1e-4):
                    bad += 1
                    print("FAIL BP", seed, world, dihedral, r_bp, g, flush=True)
print("done", tried, "scanners, failures:", bad)
