"""Randomised sweeps of the CUDA path against the FP64 oracle beyond the
seeded draws of tests/test_gpu_fuzz.py (one-off hunts; the failures they
found are regression tests now: DESIGN.md 8).

  python tools/fuzz.py test  LO HI   # tests/test_gpu_fuzz.draw over more seeds
  python tools/fuzz.py wide  LO HI   # harder scanners: sources 1.05 field radii away, tau/Delta_s up to 6,
                                     # pixels 0.1..3 mm, batches up to 8
  python tools/fuzz.py big   LO HI   # n 100..520 (many BP tiles, ragged edges), 8..40 views (4-/8-fold paths)
  python tools/fuzz.py shards LO HI  # orbit / dihedral / block shard calls at 2, 3, 8 emulated ranks
  python tools/fuzz.py ref   LO HI   # the FP64 reference projector pair (row f2), relative 1e-9

Every check uses the parity bar of tests/test_gpu_parity.py, with ledger #23
for outputs that see only support-edge tails (tests/test_gpu_fuzz.py)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402
from paper_1907_10526_b200 import sharded  # noqa: E402
from tests.test_gpu_fuzz import DELTA_W, _mass  # noqa: E402
from tests.test_gpu_fuzz import draw as draw_test  # noqa: E402
from tests.test_gpu_parity import _metrics  # noqa: E402


def draw_wide(seed):
    rng = np.random.default_rng(90000 + seed)
    kind = int(rng.integers(0, 3))
    model = int(rng.random() < 0.3)
    n = int(rng.integers(1, 161))
    h = float(np.exp(rng.uniform(np.log(0.1), np.log(3.0))))
    n_views = int(rng.choice([1, 2, 4, 7, 8, 12, 16, 36, 60, 64, 100, 120]))
    pitch = float(np.exp(rng.uniform(np.log(0.2), np.log(4.0)))) * h
    R = n * h / np.sqrt(2.0)
    sid = float(R * np.exp(rng.uniform(np.log(1.05), np.log(20.0))) + 0.01 * h)
    sdd = float(sid * rng.uniform(1.0, 4.0))
    width = float(np.exp(rng.uniform(np.log(0.02), np.log(6.0)))) * pitch
    if kind != 1:
        width = min(width, 1.9 * sdd)
    span = 2 * R if kind == 1 else 2 * sdd * np.tan(np.arcsin(min(R / sid, 0.999)))
    n_det = max(1, min(2000, int(span / pitch * rng.uniform(0.5, 1.4)) + int(rng.integers(0, 5))))
    g = dict(n=n, pixel=h, n_views=n_views, n_det=n_det, det_pitch=pitch, det_width=width,
             sid=sid if kind != 1 else 0.0, sdd=sdd if kind != 1 else 0.0, kind=kind, model=model)
    while kind == 2 and g["n_det"] > 1 and cbp.validate(g) != cbp.CBP_OK:
        g["n_det"] -= 1
    batch = int(rng.choice([1, 1, 1, 2, 3, 4, 5, 8]))
    full = rng.random() < 0.6
    v0 = 0 if full else int(rng.integers(0, n_views))
    nv = n_views - v0 if full else int(rng.integers(1, n_views - v0 + 1))
    return g, batch, v0, nv


def draw_big(seed):
    rng = np.random.default_rng(70000 + seed)
    g, _, _, _ = draw_wide(seed)
    n = int(rng.integers(100, 521))
    h = g["pixel"]
    R = n * h / np.sqrt(2.0)
    kind = g["kind"]
    sid = float(R * np.exp(rng.uniform(np.log(1.15), np.log(15.0))))
    sdd = float(sid * rng.uniform(1.0, 3.0))
    pitch = float(np.exp(rng.uniform(np.log(0.3), np.log(3.0)))) * h
    width = float(np.exp(rng.uniform(np.log(0.2), np.log(4.0)))) * pitch
    span = 2 * R if kind == 1 else 2 * sdd * np.tan(np.arcsin(min(R / sid, 0.999)))
    n_det = max(1, min(3000, int(span / pitch * rng.uniform(0.7, 1.2))))
    g = dict(g, n=n, sid=sid if kind != 1 else 0.0, sdd=sdd if kind != 1 else 0.0, det_pitch=pitch,
             det_width=min(width, 1.9 * sdd) if kind != 1 else width, n_det=n_det,
             n_views=int(rng.choice([8, 12, 16, 24, 40])))
    while kind == 2 and g["n_det"] > 1 and cbp.validate(g) != cbp.CBP_OK:
        g["n_det"] -= 1
    return g, int(rng.choice([1, 1, 2, 4])), 0, g["n_views"]


def ok_parity(got, want, mass, h):
    """(ok, metrics): the parity bar, or ledger #23's absolute bound for tails"""
    if np.abs(want).max() == 0:
        return not np.any(got), (0.0, 0.0)
    r = _metrics(got, want)
    eps_abs = DELTA_W * np.sqrt(2.0) * h * mass
    if np.abs(want).max() < 1e4 * eps_abs:
        return float(np.abs(np.asarray(got, np.float64) - want).max()) <= eps_abs, r
    return r[0] <= 1e-5 and r[1] <= 1e-4, r


def check_fp_bp(seed, g, batch, v0, nv):
    n = g["n"]
    imgs = W.random_image(n, seed, batch=batch) if batch > 1 else W.random_image(n, seed)
    y = W.random_sino(nv, g["n_det"], seed + 7, batch=batch) if batch > 1 else W.random_sino(nv, g["n_det"], seed + 7)
    got = cbp.forward(g, torch.from_numpy(np.ascontiguousarray(imgs, dtype=np.float32)).cuda(),
                      view_begin=v0, view_count=nv).cpu().numpy()
    gotb = cbp.back(g, torch.from_numpy(y).cuda(), view_begin=v0).cpu().numpy()
    fails = []
    for what, a, b, mass in (("FP", got, O.forward(g, imgs, view_begin=v0, view_count=nv), _mass(imgs, batch)),
                             ("BP", gotb, O.back(g, y, view_begin=v0), _mass(y, batch))):
        ok, r = ok_parity(a, b, mass, g["pixel"])
        if not ok:
            fails.append((what, r))
    return fails


def check_shards(seed, g):
    N = g["n_views"]
    img = torch.from_numpy(W.random_image(g["n"], seed)).cuda()
    y = torch.from_numpy(W.random_sino(N, g["n_det"], seed + 1)).cuda()
    full_y, full_c = cbp.forward(g, img), cbp.back(g, y)
    fails = []
    for world in (2, 3, 8):
        for dihedral in (False, True):
            if dihedral and N % 8:
                continue
            total = torch.zeros_like(full_c)
            for r in range(world):
                sh = sharded.make_shard(N, r, world, dihedral=dihedral)
                if sh.count == 0:
                    continue
                rows = torch.as_tensor(sh.views(), device="cuda")
                if sh.mode == "dihedral":
                    ys = cbp.forward_dihedral(g, img, sh.begin, sh.count)[rows]
                    total += cbp.back_dihedral(g, y, sh.begin, sh.count)
                elif sh.mode == "orbit":
                    ys = cbp.forward_orbit(g, img, sh.begin, sh.count).reshape(-1, g["n_det"])
                    cbp.back_orbit(g, y[rows].reshape(4, sh.count, -1).contiguous(), sh.begin, image=total,
                                   accumulate=True)
                else:
                    ys = cbp.forward(g, img, view_begin=sh.begin, view_count=sh.count)
                    cbp.back(g, y[rows].contiguous(), image=total, view_begin=sh.begin, accumulate=True)
                if full_y[rows].abs().max() > 0:
                    r_fp = _metrics(ys.cpu().numpy(), full_y[rows].cpu().numpy())
                    if not (r_fp[0] <= 1e-5 and r_fp[1] <= 1e-4):
                        fails.append((f"FP shards x{world} dihedral={dihedral}", r_fp))
            torch.cuda.synchronize()
            if full_c.abs().max() > 0:
                r_bp = _metrics(total.cpu().numpy(), full_c.cpu().numpy())
                if not (r_bp[0] <= 1e-5 and r_bp[1] <= 1e-4):
                    fails.append((f"BP shards x{world} dihedral={dihedral}", r_bp))
    return fails


def check_ref(seed, g):
    img = W.random_image(g["n"], seed)
    want = O.ref_forward(g, img.astype(np.float64))
    got = cbp.ref_forward(g, torch.from_numpy(img).cuda()).cpu().numpy()
    y = W.random_sino(g["n_views"], g["n_det"], seed + 3).astype(np.float64)
    wb, gb = O.ref_back(g, y), cbp.ref_back(g, torch.from_numpy(y).cuda()).cpu().numpy()
    fails = []
    for what, a, b in (("ref FP", got, want), ("ref BP", gb, wb)):
        m = np.abs(b).max()
        err = np.abs(a - b).max() / m if m > 0 else np.abs(a).max()
        if not err <= 1e-9:
            fails.append((what, err))
    return fails


def main():
    mode, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    tried = bad = 0
    for seed in range(lo, hi):
        if mode == "test":
            g, batch, v0, nv, _ = draw_test(seed)
        elif mode == "big":
            g, batch, v0, nv = draw_big(seed)
        else:
            g, batch, v0, nv = draw_wide(seed)
        if cbp.validate(g) != cbp.CBP_OK:
            continue
        if mode == "shards":
            if g["n_views"] % 4:
                continue
            fails = check_shards(seed, g)
        elif mode == "ref":
            g = dict(g, n_views=min(g["n_views"], 12), n_det=min(g["n_det"], 200))
            if g["n"] > 24 or cbp.validate(g) != cbp.CBP_OK:
                continue
            fails = check_ref(seed, g)
        else:
            fails = check_fp_bp(seed, g, batch, v0, nv)
        tried += 1
        for what, r in fails:
            bad += 1
            print("FAIL", mode, seed, what, r, g, batch, v0, nv, flush=True)
    print("done", mode, tried, "draws, failures:", bad)


if __name__ == "__main__":
    main()
