"""The kernels claim bitwise determinism (no atomics, fixed summation order;
DESIGN.md 5.3-5.4): repeated calls on the same inputs must agree bit for bit
on every path -- direct, batched (2 and 4 slices), 4- and 8-fold symmetric,
view ranges, ragged tiles and tiles the detector misses, the precise mode and
the magnified-footprint model.  (Round 2 found a header race in the
one-slice BP this way: tests/test_gpu_narrow.py.)"""
import numpy as np
import pytest

import paper_1907_10526_b200 as cbp
import workloads as W

from tests.test_gpu_parity import torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu

G1 = W.geometry("1")
# a detector narrower than the field of view: edge tiles see no bins for runs of views
NARROW_DET = dict(n=142, pixel=0.29, n_views=100, n_det=444, det_pitch=0.072, det_width=0.072,
                  sid=0.0, sdd=0.0, kind=1, model=0)
CASES = {
    "direct": (dict(G1, n_views=90), 1),
    "batch2": (dict(G1, n_views=90), 2),
    "batch5": (dict(G1, n_views=90), 5),
    "sym4": (dict(G1, n_views=92), 1),
    "sym8": (dict(G1, n_views=88), 1),
    "sym8_batch3": (dict(G1, n_views=88), 3),
    "ragged": (dict(n=37, pixel=1.3, n_views=30, n_det=77, det_pitch=1.1, det_width=0.6, sid=120.0, sdd=260.0), 1),
    "uncovered_tiles": (dict(NARROW_DET, n_views=99), 1),
    "uncovered_tiles_batch8": (NARROW_DET, 8),
    "precise": (dict(G1, n_views=90, det_width=0.01), 3),
    "mag": (dict(G1, n_views=88, model=1), 1),
    # config 2: 4 view groups x 8 frames = 32 planes, the reduce's four-lane path
    "sym8_config2": (W.geometry("2"), 1),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_repeated_calls_are_bitwise_equal(torch_cuda, name):
    torch = torch_cuda
    g, batch = CASES[name]
    img = torch.from_numpy(W.random_image(g["n"], 3, batch=batch) if batch > 1 else W.random_image(g["n"], 3)).cuda()
    ys = [cbp.forward(g, img) for _ in range(4)]
    cs = [cbp.back(g, ys[0]) for _ in range(4)]
    torch.cuda.synchronize()
    for y in ys[1:]:
        assert torch.equal(y, ys[0]), f"FP {name}"
    for c in cs[1:]:
        assert torch.equal(c, cs[0]), f"BP {name}"
    assert np.isfinite(cs[0].cpu().numpy()).all()
