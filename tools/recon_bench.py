"""Row f1 measurement: 20-iteration SART and CGLS at BASELINE config 5
(2048^2 Shepp-Logan, 2880 views, 4096 bins) on one GPU; data = A(phantom)
from the library's own FP.  Prints one JSON line per method."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1907_10526_b200 as cbp  # noqa: E402
from paper_1907_10526_b200 import recon  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = W.geometry(cfg)
truth = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
y = cbp.forward(g, truth)
torch.cuda.synchronize()
for name, fn in (("sart", recon.sart), ("cgls", recon.cgls)):
    fn(g, y, 2)  # warm-up (tables, scratch pools)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x = fn(g, y, iters)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    err = float(torch.linalg.norm(x - truth) / torch.linalg.norm(truth))
    res = float(torch.linalg.norm(cbp.forward(g, x) - y) / torch.linalg.norm(y))
    print(json.dumps({"method": name, "config": cfg, "n": g["n"], "n_views": g["n_views"],
                      "n_det": g["n_det"], "iterations": iters, "total_ms": ms,
                      "ms_per_iteration": ms / iters, "rel_err_to_truth": err,
                      "rel_data_residual": res, "snr_db": -20 * np.log10(err),
                      "symmetry_fold": cbp.symmetry_fold(g)}), flush=True)
