"""Row f2 accuracy study on the GPU: the CNSF projector (cbp_forward, FP32)
against the paper's reference projector (cbp_ref_forward, FP64 exact chords
averaged over each bin), in the paper's settings:

* Fig. 5: 1 mm pixel at the origin, D_po = D_so = 3 mm,
  tau = 0.5 mm, 601 bins of 0.01 mm, angles 0/15/35/45 degrees;
* Fig. 6a: pixel at the origin, D_po = D_so = 200 mm,
  tau = Delta_s = 0.5 mm, 90 angles over 90 degrees;
* Fig. 6b: the pixel at (100.5, 50.5) mm, 360 angles over 360 degrees;
* Fig. 7: 128 mm Shepp-Logan, 409 bins of 1 mm, tau = 0.5 mm,
  D = 200/200 mm, 360 angles.

Eq. 15: e(u) = max_s |F(s, u) - F_ref(s, u)| per angle.  The paper prints no
values (its figures are lost), so the numbers here are the record, not a
comparison.  Writes one JSON document (default profiles/r01_accuracy_b200.json).

usage: python tools/accuracy_study.py [out.json]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402


def pair(g, img, views=None):
    dev = torch.device("cuda:0")
    x = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).to(dev)
    v0, nv = (0, g["n_views"]) if views is None else views
    t0 = time.perf_counter()
    y = cbp.forward(g, x, view_begin=v0, view_count=nv).double()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = cbp.ref_forward(g, x, view_begin=v0, view_count=nv)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return y.cpu().numpy(), r.cpu().numpy(), t1 - t0, t2 - t1


def per_angle(y, r):
    e = np.abs(y - r).max(axis=-1)
    peak = np.abs(r).max(axis=-1)
    return e, peak


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join("profiles", "r01_accuracy_b200.json")
    res = {"device": torch.cuda.get_device_name(0), "model": "CNSF cbp_forward (FP32) vs Ref cbp_ref_forward (FP64)"}

    g = W.FIG5
    y, r, _, _ = pair(g, np.ones((1, 1)))
    e, peak = per_angle(y, r)
    res["fig5"] = {
        "geometry": g,
        "angles_deg": [5 * v for v in W.FIG5_VIEWS],
        "max_error_mm": [float(e[v]) for v in W.FIG5_VIEWS],
        "peak_mm": [float(peak[v]) for v in W.FIG5_VIEWS],
    }

    g = W.FIG6
    y, r, _, _ = pair(g, np.ones((1, 1)), views=(0, 90))
    e, peak = per_angle(y, r)
    res["fig6a"] = {"geometry": g, "angles_deg": list(range(90)), "max_error_mm": e.tolist(),
                    "peak_mm": peak.tolist(), "worst": float(e.max()), "mean": float(e.mean())}

    g = dict(W.FIG6, n=204)  # pixel (51, 202) of a 204-grid is centred at (100.5, 50.5)
    y, r, _, _ = pair(g, W.single_pixel(204, 51, 202))
    e, peak = per_angle(y, r)
    res["fig6b"] = {"geometry": g, "pixel_mm": list(W.FIG6B_PIXEL), "angles_deg": list(range(360)),
                    "max_error_mm": e.tolist(), "peak_mm": peak.tolist(), "worst": float(e.max()),
                    "mean": float(e.mean())}

    g = W.FIG7
    img = W.shepp_logan(g["n"])
    y, r, tc, tr = pair(g, img)
    err = np.abs(y - r)
    res["fig7"] = {"geometry": g, "phantom": "Shepp-Logan (original intensities)",
                   "max_abs_error": float(err.max()), "mean_abs_error": float(err.mean()),
                   "sino_peak": float(np.abs(r).max()),
                   "max_rel_to_peak": float(err.max() / np.abs(r).max()),
                   "rel_l2": float(np.linalg.norm(y - r) / np.linalg.norm(r)),
                   "cnsf_seconds": tc, "ref_seconds": tr}
    # row f3 variants in the Fig. 6 setting: parallel beam (exact by Theorem 1:
    # only FP32 rounding remains) and the arc detector (D_ps = 400 mm)
    for name, extra in (("fig6a_parallel", dict(kind=cbp.PARALLEL)),
                        ("fig6a_arc", dict(kind=cbp.FAN_ARC))):
        g = dict(W.FIG6, **extra)
        y, r, _, _ = pair(g, np.ones((1, 1)), views=(0, 90))
        e, peak = per_angle(y, r)
        res[name] = {"geometry": g, "angles_deg": list(range(90)), "max_error_mm": e.tolist(),
                     "worst": float(e.max()), "mean": float(e.mean()), "peak_mm": float(peak.max())}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: ({kk: vv for kk, vv in v.items() if kk in ("worst", "mean", "max_error_mm", "max_rel_to_peak", "rel_l2", "ref_seconds")} if isinstance(v, dict) else v) for k, v in res.items()}))


if __name__ == "__main__":
    main()
