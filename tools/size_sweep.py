"""FP+BP pair time vs problem size on one B200 (the scale-similar geometry of
configs 1-5, plus 4096^2): device-resident, CUDA events, warm L2."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402

res = []
for n in (256, 512, 1024, 2048, 4096):
    g = W._fan(n, int(720 * n / 512), 2 * n)
    img = torch.from_numpy(W.shepp_logan(n)).cuda()
    y = cbp.forward(g, img)
    c = cbp.back(g, y)
    torch.cuda.synchronize()
    reps = max(3, int(200 * (512 / n) ** 3))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(reps):
        cbp.forward(g, img, y)
    ev[1].record()
    for _ in range(reps):
        cbp.back(g, y, c)
    ev[2].record()
    ev[2].synchronize()
    fp, bp = ev[0].elapsed_time(ev[1]) / reps, ev[1].elapsed_time(ev[2]) / reps
    nw = 2.7011 * n * n * g["n_views"]  # nonzero weights per projection (2.701 per view-pixel)
    r = dict(n=n, n_views=g["n_views"], n_det=g["n_det"], fp_ms=fp, bp_ms=bp, pairs_per_s=1e3 / (fp + bp),
             gweights_per_s=2 * nw / ((fp + bp) * 1e-3) / 1e9, adjoint=cbp.adjoint_check(g, 3) if n <= 2048 else None)
    res.append(r)
    print(json.dumps(r), flush=True)
