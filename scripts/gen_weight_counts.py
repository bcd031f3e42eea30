"""Write tests/golden/weight_counts.json: the number of nonzero weights
(view, pixel, bin) per view -- the unit of algorithmic work --
counted by the FP64 oracle's exact support test (Eq. 14, ledger #15).
Calls only oracle/ (and the workloads geometry numbers)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "weight_counts.json")


def main(cfgs):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["_comment"] = ("nonzero (view, pixel, bin) weights per view, counted by "
                        "oracle.count_weights (scripts/gen_weight_counts.py)")
    for c in cfgs:
        g = W.geometry(c)
        t = time.time()
        per_view = [int(x) for x in O.count_weights_per_view(g)]
        data[c] = dict(geometry=g, per_view=per_view, total=sum(per_view),
                       per_view_pixel=sum(per_view) / (g["n"] ** 2 * g["n_views"]))
        print(c, sum(per_view), data[c]["per_view_pixel"], f"{time.time() - t:.1f}s", flush=True)
        json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["1", "2"])
