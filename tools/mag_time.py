import torch, time, json, sys
sys.path.insert(0, '.')
import paper_1907_10526_b200 as cbp, workloads as W
for cfg in ("2",):
    for model in (0, 1):
        g = dict(W.geometry(cfg), model=model)
        img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
        y = cbp.forward(g, img); c = cbp.back(g, y); torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for _ in range(5): y = cbp.forward(g, img, sino=y)
        e[1].record()
        for _ in range(5): c = cbp.back(g, y, image=c)
        e[2].record(); torch.cuda.synchronize()
        print(json.dumps({"cfg": cfg, "model": model, "fp_ms": e[0].elapsed_time(e[1])/5, "bp_ms": e[1].elapsed_time(e[2])/5}))
