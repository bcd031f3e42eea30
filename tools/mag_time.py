"""Time FP and BP of both weight models (CNSF, magnified footprint) through
the Python binding, on the default stream and on a side stream."""
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402


def run(cfg, model, stream):
    g = dict(W.geometry(cfg), model=model)
    img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
    with torch.cuda.stream(stream):
        y = cbp.forward(g, img)
        c = cbp.back(g, y)
        for _ in range(3):  # warm-up (first calls of a process pay one-time host costs)
            cbp.forward(g, img, sino=y)
            cbp.back(g, y, image=c)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for _ in range(5):
            cbp.forward(g, img, sino=y)
        e[1].record()
        for _ in range(5):
            cbp.back(g, y, image=c)
        e[2].record()
        torch.cuda.synchronize()
    return {"cfg": cfg, "model": model, "stream": "default" if stream == torch.cuda.default_stream() else "side",
            "fp_ms": e[0].elapsed_time(e[1]) / 5, "bp_ms": e[1].elapsed_time(e[2]) / 5}


if __name__ == "__main__":
    if "--once" in sys.argv:  # one FP and one BP of the magnified model (for ncu)
        g = dict(W.geometry(sys.argv[1]), model=1)
        img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
        cbp.back(g, cbp.forward(g, img))
        torch.cuda.synchronize()
        sys.exit(0)
    cfgs = sys.argv[1:] or ["2"]
    for cfg in cfgs:
        for model in (0, 1):
            for st in (torch.cuda.default_stream(), torch.cuda.Stream()):
                print(json.dumps(run(cfg, model, st)), flush=True)
