"""A/B timing of library builds on the view-sharded pair: for each
libcbp*.so, every rank's dihedral shard of a W-GPU run (FP + BP, warm L2,
CUDA events over 50 back-to-back pairs) in child processes, interleaved
rounds (clock drift hits every build alike), min over rounds per rank; prints
the slowest and mean rank per build.
usage: python tools/ab_shard.py CFG W lib1.so lib2.so ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json, torch
sys.path.insert(0, %r)
import paper_1907_10526_b200 as cbp, workloads as W
from paper_1907_10526_b200 import sharded
g = W.geometry(%r); world = %d
img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
y = torch.zeros((g["n_views"], g["n_det"]), device="cuda"); out = torch.empty_like(img)
res = []
for r in range(world):
    sh = sharded.make_shard(g["n_views"], r, world, dihedral=True)
    def pair():
        if sh.mode == "block":
            cbp.forward(g, img, sino=y); cbp.back(g, y, image=out)
        else:
            cbp.forward_dihedral(g, img, sh.begin, sh.count, sino=y)
            cbp.back_dihedral(g, y, sh.begin, sh.count, image=out)
    for _ in range(10): pair()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        a.record()
        for _ in range(50): pair()
        b.record(); b.synchronize()
        best = min(best, a.elapsed_time(b) / 50)
    res.append(best)
print(json.dumps(res))
'''

if __name__ == "__main__":
    cfg, world, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
    res = {lib: None for lib in libs}
    for rnd in range(3):
        for lib in libs:
            env = dict(os.environ, CBP_LIB_PATH=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg, world)], env=env, capture_output=True,
                                 text=True)
            if out.returncode != 0:
                print(lib, "FAILED", out.stderr[-800:])
                continue
            r = json.loads(out.stdout.strip().splitlines()[-1])
            res[lib] = r if res[lib] is None else [min(a, b) for a, b in zip(res[lib], r)]
    for lib, r in res.items():
        if r:
            print(json.dumps({"lib": os.path.basename(lib), "world": world, "slowest_ms": max(r),
                              "mean_ms": sum(r) / len(r), "ranks": [round(x, 4) for x in r]}))
