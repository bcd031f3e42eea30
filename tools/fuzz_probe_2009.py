"""Probe of wide-sweep seed 2009 (arc detector, source 1.08 field radii away,
tau/h 0.009): BP and FP error against the oracle as tau and the source
distance vary, to separate a narrow-bin precision limit from a range bug."""
import sys

import numpy as np
import torch

sys.argv = ['x', '0', '0']
exec(open('tools/fuzz_wide.py').read().split('lo, hi =')[0])
from tests.test_gpu_parity import _metrics  # noqa: E402

g0, batch, v0, nv = draw(2009)
print(g0, batch, v0, nv)
for tau_scale in (1.0, 10.0, 50.0):
    for sid_scale in (1.0, 1.1, 1.3):
        g = dict(g0, det_width=g0["det_width"] * tau_scale, sid=g0["sid"] * sid_scale, sdd=g0["sdd"] * sid_scale)
        if cbp.validate(g) != cbp.CBP_OK:
            print("invalid", tau_scale, sid_scale)
            continue
        n = g["n"]
        y = W.random_sino(nv, g["n_det"], 2016)
        wantb = O.back(g, y, view_begin=v0)
        gotb = cbp.back(g, torch.from_numpy(y).cuda(), view_begin=v0).cpu().numpy()
        img = W.random_image(n, 2009)
        want = O.forward(g, img, view_begin=v0, view_count=nv)
        got = cbp.forward(g, torch.from_numpy(img).cuda(), view_begin=v0, view_count=nv).cpu().numpy()
        print(f"tau x{tau_scale} sid x{sid_scale}: FP {_metrics(got, want)} BP {_metrics(gotb, wantb)}", flush=True)
