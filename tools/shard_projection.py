"""Strong-scaling projection of the view-sharded pair on ONE B200: for each
world size W, every rank's dihedral shard (sharded.make_shard, the bench's
N > 1 shape) is timed on this GPU (FP + BP, warm L2, CUDA events); the
projected step of W GPUs is the slowest shard (the ranks run concurrently
on their own GPUs), plus the BP all-reduce, which this one-GPU box cannot
measure (reported separately as not measured).  With CBP_PROJ_GRAPH=1 each
rank's pair is captured once in a CUDA graph and replayed (no host launch
overhead in the timed loop; the library's launches are graph nodes).  Usage:
  [PROJ_DIHEDRAL=0] python tools/shard_projection.py [config] [worlds...]   (0: orbit shards)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1907_10526_b200 as cbp  # noqa: E402
from paper_1907_10526_b200 import sharded  # noqa: E402
import workloads as W  # noqa: E402


def t_ms(fn, reps=20):
    if os.environ.get("CBP_PROJ_GRAPH") == "1":
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            fn()
        torch.cuda.synchronize()
        fn = gr.replay
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
    worlds = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
    g = W.geometry(cfg)
    img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
    y = torch.zeros((g["n_views"], g["n_det"]), device="cuda")
    out = torch.empty_like(img)
    for _ in range(10):  # warm-up: clocks, caches, the library's one-time set-up
        cbp.forward(g, img, sino=y)
        cbp.back(g, y, image=out)
    torch.cuda.synchronize()
    base = None
    dihedral = os.environ.get("PROJ_DIHEDRAL", "1") != "0"  # 0: orbit shards (4 rotations of a base block)
    for world in worlds:
        per_rank = []
        for r in range(world):
            sh = sharded.make_shard(g["n_views"], r, world, dihedral=dihedral)
            if sh.mode == "block":  # world 1: the library's own full-scan path
                def pair():
                    cbp.forward(g, img, sino=y)
                    cbp.back(g, y, image=out)
            elif sh.mode == "orbit":
                yo = torch.zeros((4, sh.count, g["n_det"]), device="cuda")

                def pair(sh=sh, yo=yo):
                    cbp.forward_orbit(g, img, sh.begin, sh.count, sino=yo)
                    cbp.back_orbit(g, yo, sh.begin, image=out)
            else:
                def pair(sh=sh):
                    cbp.forward_dihedral(g, img, sh.begin, sh.count, sino=y)
                    cbp.back_dihedral(g, y, sh.begin, sh.count, image=out)
            per_rank.append({"rank": r, "views": int(len(sh.views())), "ms": t_ms(pair)})
        slowest = max(p["ms"] for p in per_rank)
        if world == 1:
            base = slowest
        line = {"config": cfg, "world": world, "mode": sharded.make_shard(g["n_views"], 0, world, dihedral=dihedral).mode,
                "slowest_rank_ms": slowest, "mean_rank_ms": sum(p["ms"] for p in per_rank) / world,
                "max_views": max(p["views"] for p in per_rank),
                "projected_pairs_per_s_compute_only": 1e3 / slowest,
                "projected_efficiency_compute_only": base / (world * slowest) if base else None,
                "allreduce": "not measured (one GPU); add it to slowest_rank_ms", "ranks": per_rank}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
