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


def per_view_counts(g, dihedral):
    """per-view counts; with `dihedral` (n_views % 8 == 0) only the base views
    [0, n_views/8] are counted and the rest filled from their orbits: the
    rotation by 90 degrees and the mirror map the square grid onto itself and
    a view's bins onto another view's bins, so the nonzero
    count of every view in an orbit is the same"""
    N = g["n_views"]
    if not dihedral:
        return [int(x) for x in O.count_weights_per_view(g)]
    base = [int(x) for x in O.count_weights_per_view(g, 0, N // 8 + 1)]
    out = [None] * N
    for v, cnt in enumerate(base):
        for m in (0, 1):
            for q in range(4):
                out[((N - v if m else v) + q * (N // 4)) % N] = cnt
    assert all(x is not None for x in out)
    return out


def main(cfgs):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["_comment"] = ("nonzero (view, pixel, bin) weights per view, counted by "
                        "oracle.count_weights (scripts/gen_weight_counts.py; configs 3, 5 and the "
                        "paper shapes p*: base views of the 8-fold symmetry, expanded over their orbits)")
    for c in cfgs:
        g = W.geometry(c)
        t = time.time()
        per_view = per_view_counts(g, dihedral=c not in ("1", "2") and g["n_views"] % 8 == 0)
        data[c] = dict(geometry=g, per_view=per_view, total=sum(per_view),
                       per_view_pixel=sum(per_view) / (g["n"] ** 2 * g["n_views"]))
        print(c, sum(per_view), data[c]["per_view_pixel"], f"{time.time() - t:.1f}s", flush=True)
        json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["1", "2"])
