"""Narrow-bin accuracy of the two weight paths: FP and BP
relL2 / max-normalised error against the oracle as tau/h shrinks, with the
precise mode forced off (CBP_PRECISE=0) and on (=1), every kind and model,
plus the time of both modes at config 2 (FP, BP ms).  Picks the library's
switch-over (CBP_NARROW_RATIO): the standard path must stay well inside the
bar above it.  usage: python tools/narrow_sweep.py [out.jsonl]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402
from tests.test_gpu_narrow import _narrow  # noqa: E402
from tests.test_gpu_parity import _metrics  # noqa: E402

out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout
for kind in (0, 1, 2):
    for model in (0, 1):
        for tau_h in (0.005, 0.01, 0.02, 0.05, 0.1, 0.2, 0.35, 0.5, 0.75, 1.0, 1.5):
            g = _narrow(kind, model, tau_h, n=40, n_views=16)
            img = W.random_image(g["n"], 51)
            y = W.random_sino(g["n_views"], g["n_det"], 52)
            want_f, want_b = O.forward(g, img), O.back(g, y)
            rec = dict(kind=kind, model=model, tau_h=tau_h, narrow_ratio=cbp.narrow_ratio(g))
            for mode in ("0", "1"):
                os.environ["CBP_PRECISE"] = mode
                f = cbp.forward(g, torch.from_numpy(img).cuda()).cpu().numpy()
                b = cbp.back(g, torch.from_numpy(y).cuda()).cpu().numpy()
                rec["precise" if mode == "1" else "standard"] = dict(fp=_metrics(f, want_f), bp=_metrics(b, want_b))
            os.environ.pop("CBP_PRECISE")
            print(json.dumps(rec), file=out, flush=True)

# time of the two modes at config 2 (one image, all views; warm)
g = W.geometry("2")
img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
for mode in ("0", "1"):
    os.environ["CBP_PRECISE"] = mode
    for _ in range(3):
        y = cbp.forward(g, img)
        c = cbp.back(g, y)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf = tb = 0.0
    for _ in range(10):
        e[0].record()
        y = cbp.forward(g, img, sino=y)
        e[1].record()
        cbp.back(g, y, image=c)
        e[2].record()
        torch.cuda.synchronize()
        tf += e[0].elapsed_time(e[1]) / 10
        tb += e[1].elapsed_time(e[2]) / 10
    print(json.dumps(dict(config="2", precise=int(mode), fp_ms=tf, bp_ms=tb)), file=out, flush=True)
os.environ.pop("CBP_PRECISE")
