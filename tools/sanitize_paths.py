"""One small call of every kernel path, for compute-sanitizer (memcheck /
racecheck / synccheck): CNSF FP/BP on the direct, batched (S = 2, 4),
4-fold and 8-fold symmetric paths, ragged grids, the parallel and arc
kinds, the magnified-footprint model (plain and 4-fold), orbit and dihedral
shards, the normal operator and its host pipeline, the FP64 reference pair,
the vector / TV kernels of the iterative loops, and (round 2) the precise
mode for narrow bins (CNSF and magnified, every kind, batches), the
one-slice BP over edge tiles the detector misses, the opt-in orbit-cluster
BP and rot_rows FP, and (v53) the opt-in persistent BP, the staged
4-rotation pad and the magnified model's pad-fed FP.  Run under the debug build (libcbp_debug.so:
CBP_DEBUG_CHECKS index checks and a sync + error check after each launch)
since compute-sanitizer is closed on this pool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1907_10526_b200 as cbp  # noqa: E402
from paper_1907_10526_b200 import sharded  # noqa: E402
import workloads as W  # noqa: E402


def pair(g, batch=1, v0=0, nv=None):
    n = g["n"]
    nv = g["n_views"] - v0 if nv is None else nv
    img = torch.from_numpy(W.random_image(n, 1, batch=batch) if batch > 1 else W.random_image(n, 1)).cuda()
    y = cbp.forward(g, img, view_begin=v0, view_count=nv)
    c = cbp.back(g, y, view_begin=v0)
    cbp.back(g, y, image=c, view_begin=v0, accumulate=True)


g1 = W.geometry("1")
for nvw in (90, 92, 88):                       # direct, 4-fold, 8-fold
    pair(dict(g1, n_views=nvw))
pair(g1, v0=13, nv=21)                         # view range
for b in (2, 3, 5):                            # batched S = 2 / 4, ragged batch
    pair(g1, batch=b)
pair(dict(g1, n_views=88), batch=3)            # batch over a full scan (per-image dihedral BP)
rag = dict(n=37, pixel=1.3, n_views=30, n_det=77, det_pitch=1.1, det_width=0.6, sid=120.0, sdd=260.0)
pair(rag)
pair(rag, batch=5)
pair(dict(rag, n_views=32))                    # ragged tiles with the symmetry
for kind in (cbp.PARALLEL, cbp.FAN_ARC):
    g = dict(g1, kind=kind, n_views=88) if kind == cbp.PARALLEL else \
        dict(n=64, pixel=1.0, n_views=88, n_det=160, det_pitch=1.2, det_width=1.0, sid=100.0, sdd=200.0, kind=kind)
    pair(g)
    pair(dict(g, n_views=90), batch=2)
for model_g in (dict(g1, model=1), dict(g1, model=1, n_views=88), dict(rag, model=1)):
    pair(model_g)
pair(dict(rag, model=1), batch=3)
# shards
g = dict(g1, n_views=88)
img = torch.from_numpy(W.random_image(64, 2)).cuda()
for dihedral in (False, True):
    for r in range(3):
        sh = sharded.make_shard(88, r, 3, dihedral=dihedral)
        if sh.mode == "orbit":
            y = cbp.forward_orbit(g, img, sh.begin, sh.count)
            cbp.back_orbit(g, y, sh.begin)
        else:
            y = cbp.forward_dihedral(g, img, sh.begin, sh.count)
            cbp.back_dihedral(g, y, sh.begin, sh.count)
# normal operator, device and host pipeline
cbp.normal(g1, img)
cbp.normal_stream(g1, np.stack([W.random_image(64, i) for i in range(3)]))
# round 2: the precise mode (narrow bins), every kind and model, batches
for kind in (cbp.FAN_FLAT, cbp.PARALLEL, cbp.FAN_ARC):
    for model in (0, 1):
        gn = dict(n=40, pixel=1.0, n_views=8, n_det=45 if kind == cbp.PARALLEL else 54,
                  det_pitch=1.0 if kind == cbp.PARALLEL else 2.0, det_width=0.01,
                  sid=0.0 if kind == cbp.PARALLEL else 100.0, sdd=0.0 if kind == cbp.PARALLEL else 200.0,
                  kind=kind, model=model)
        assert cbp.precise_mode(gn) == 1
        pair(gn)
        pair(gn, batch=3)
# the one-slice BP over edge tiles the detector does not cover, batch 8 (precise mode)
gw = dict(n=142, pixel=0.2931904994119643, n_views=100, n_det=444, det_pitch=0.0717829057628753,
          det_width=0.0032782721295456555, sid=0.0, sdd=0.0, kind=1, model=0)
pair(gw, batch=8)
# the opt-in orbit-cluster BP (n a multiple of 32; an odd tile grid) and rot_rows FP
os.environ["CBP_ORBIT"] = "1"
pair(dict(g1, n_views=88))
pair(dict(g1, n=96, n_det=192, n_views=48))
os.environ.pop("CBP_ORBIT")
# round 2 (v53): the opt-in persistent BP (both reductions: n a multiple of 32
# and ragged; many and few CTAs; a batch; a dihedral shard), the staged
# 4-rotation pad at a ragged size, the magnified model's 4-fold FP on its pad
os.environ["CBP_BP_SEG"] = "1"
pair(dict(g1, n_views=88))
pair(dict(rag, n_views=32))
pair(dict(g1, n_views=88), batch=3)
os.environ["CBP_BP_SEG_CTAS"] = "5"
pair(dict(g1, n=96, n_det=192, n_views=48))
os.environ["CBP_BP_SEG_CTAS"] = "3000"
pair(dict(g1, n_views=88))
os.environ.pop("CBP_BP_SEG_CTAS")
sh = sharded.make_shard(88, 1, 3, dihedral=True)
cbp.back_dihedral(dict(g1, n_views=88), cbp.forward(dict(g1, n_views=88), img), sh.begin, sh.count)
os.environ.pop("CBP_BP_SEG")
pair(dict(n=70, pixel=0.9, n_views=92, n_det=150, det_pitch=1.1, det_width=1.0, sid=200.0, sdd=400.0))
pair(dict(n=70, pixel=0.9, n_views=92, n_det=150, det_pitch=1.1, det_width=1.0, sid=200.0, sdd=400.0, model=1))
# v56: the 8-frame BP's wide chunk shape (the paper's timing shape; forced on a narrow geometry, a batch)
pair(dict(W.PAPER_TIMING[64]))
os.environ["CBP_BP_WIDE"] = "1"
pair(dict(g1, n_views=88))
pair(dict(g1, n_views=88), batch=3)
pair(dict(rag, n_views=32))
os.environ.pop("CBP_BP_WIDE")
# reference projector
gs = dict(g1, n=16, n_views=6, n_det=40)
yr = cbp.ref_forward(gs, torch.from_numpy(W.random_image(16, 3)).cuda())
cbp.ref_back(gs, yr)
# vector / TV kernels
x = torch.rand(64 * 64, device="cuda")
z = torch.rand(64 * 64, device="cuda")
d = torch.zeros(4, dtype=torch.float64, device="cuda")
cbp.dot(x, z, d[0:1])
cbp.tv_value(x.view(64, 64), d[1:2])
cbp.tv_gradient(x.view(64, 64), z.view(64, 64))
cbp.diff_norm2(x, z, d[2:3])
# SART / CGLS iterations (their vector kernels)
from paper_1907_10526_b200 import recon  # noqa: E402
yf = cbp.forward(g1, img)
recon.sart(g1, yf, 1)
recon.cgls(g1, yf, 1)
torch.cuda.synchronize()
print("sanitize paths ok, launches", cbp.launch_count())
