"""Per-CTA timeline of the BP kernel (diagnostics): runs one
config's BP a few times on a -DCBP_BP_PROFILE build of the library
(libcbp_prof.so, built on first use) with CBP_BP_PROF set (each CTA records its
%globaltimer start / end and SM) and summarises the last launch: span, CTA
duration spread, slot occupancy over the span and the idle tail.
usage: python tools/bp_cta_prof.py CFG [out.txt [raw.jsonl]]  (raw: every CTA of the
last launch: start, end, SM, segments, covered-view bins, covered views, views)"""
import os
import statistics
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
import paper_1907_10526_b200 as cbp, workloads as W
g = W.geometry(%r)
img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
y = cbp.forward(g, img)
for _ in range(3):
    c = cbp.back(g, y)
torch.cuda.synchronize()
'''


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
    path = tempfile.mktemp(suffix=".txt")
    lib = os.path.join(ROOT, "paper_1907_10526_b200", "libcbp_prof.so")  # the timeline is compiled in here only
    if not os.path.exists(lib):
        sys.path.insert(0, ROOT)
        from paper_1907_10526_b200 import build
        build.build_variant(lib, ["CBP_BP_PROFILE"])
    env = dict(os.environ, CBP_BP_PROF=path, CBP_LIB_PATH=lib)
    subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env, check=True)
    launches, cur = [], None
    for line in open(path):
        if line.startswith("launch"):
            cur = []
            launches.append(cur)
        else:
            cur.append(tuple(int(x) for x in line.split()))
    rows = launches[-1]
    t0 = min(r[0] for r in rows)
    t1 = max(r[1] for r in rows)
    span = (t1 - t0) / 1e3
    dur = [(r[1] - r[0]) / 1e3 for r in rows]
    sms = sorted({r[2] for r in rows})
    busy = {}
    for r in rows:
        busy[r[2]] = busy.get(r[2], 0) + (r[1] - r[0])
    ends = sorted((r[1] - t0) / 1e3 for r in rows)
    out = {
        "config": cfg, "ctas": len(rows), "sms": len(sms), "span_us": span,
        "cta_us": {"min": min(dur), "median": statistics.median(dur), "max": max(dur),
                   "mean": statistics.mean(dur)},
        "slot_fill": sum(dur) / (span * len(sms) * 2),  # 2 resident CTAs per SM
        "sm_busy_us": {"min": min(busy.values()) / 1e3, "max": max(busy.values()) / 1e3},
        "first_sm_idle_us": min(max(r[1] for r in rows if r[2] == s) for s in sms) / 1e3 - t0 / 1e3,
        "ends_pct": {p: ends[int(p / 100 * (len(ends) - 1))] for p in (50, 90, 99)},
        "segments": sum(r[3] for r in rows),
    }
    import json
    print(json.dumps(out))
    if len(sys.argv) > 2:
        with open(sys.argv[2], "a") as f:
            f.write(json.dumps(out) + "\n")
    if len(sys.argv) > 3:
        with open(sys.argv[3], "w") as f:
            for r in rows:
                f.write(json.dumps(list(r)) + "\n")


if __name__ == "__main__":
    main()
