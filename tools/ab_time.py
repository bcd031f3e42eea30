"""A/B timing of library builds: for each libcbp*.so given, time the FP and
BP of one config (warm L2, CUDA events, interleaved rounds so clock drift
hits every build alike).  usage: [AB_BATCH=B] python tools/ab_time.py CFG lib1.so lib2.so ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json, statistics, torch
sys.path.insert(0, %r)
import paper_1907_10526_b200 as cbp, workloads as W
g = dict(W.geometry(%r), model=int(os.environ.get("AB_MODEL", "0")))
img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
if int(os.environ.get("AB_BATCH", "1")) > 1:  # a batch of slices (e.g. config 4: 64)
    img = img.expand(int(os.environ["AB_BATCH"]), -1, -1).contiguous()
y = cbp.forward(g, img); c = cbp.back(g, y)
def t(fn, reps=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps
fp = [t(lambda: cbp.forward(g, img, sino=y)) for _ in range(5)]
bp = [t(lambda: cbp.back(g, y, image=c)) for _ in range(5)]
print(json.dumps({"fp": statistics.median(fp), "bp": statistics.median(bp)}))
'''

if __name__ == "__main__":
    cfg, libs = sys.argv[1], sys.argv[2:]
    res = {lib: [] for lib in libs}
    for rnd in range(3):
        for lib in libs:
            env = dict(os.environ, CBP_LIB_PATH=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env, capture_output=True,
                                 text=True)
            if out.returncode != 0:
                print(lib, "FAILED", out.stderr[-800:])
                continue
            res[lib].append(json.loads(out.stdout.strip().splitlines()[-1]))
    for lib, r in res.items():
        if r:
            print(json.dumps({"lib": os.path.basename(lib), "fp_ms": min(x["fp"] for x in r),
                              "bp_ms": min(x["bp"] for x in r)}))
