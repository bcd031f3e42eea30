"""Time the FP paths on config 2 per slice: C4 symmetric (1 image), D4 FP,
batched S = 4 (4 images, all views), no-symmetry S = 1.  CUDA events, warm L2."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402


def t_ms(fn, reps=20):
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


g = W.geometry("2")
img1 = torch.from_numpy(W.shepp_logan(512)).cuda()
img4 = img1.expand(4, -1, -1).contiguous()
img8 = img1.expand(8, -1, -1).contiguous()
y1 = cbp.forward(g, img1)
y4 = cbp.forward(g, img4)
y8 = cbp.forward(g, img8)
print("fp C4 (1 image)        %.4f ms/slice" % t_ms(lambda: cbp.forward(g, img1, y1)))
print("fp batch S=4 (4 imgs)  %.4f ms/slice" % (t_ms(lambda: cbp.forward(g, img4, y4)) / 4))
print("fp batch S=4 (8 imgs)  %.4f ms/slice" % (t_ms(lambda: cbp.forward(g, img8, y8)) / 8))
print("fp C4 views 0..179     %.4f ms (orbit)" % t_ms(lambda: cbp.forward_orbit(g, img1, 0, 180)))
print("bp D4 (1 image)        %.4f ms/slice" % t_ms(lambda: cbp.back(g, y1)))
print("bp batch S=4 (4 imgs)  %.4f ms/slice" % (t_ms(lambda: cbp.back(g, y4)) / 4))
print("bp batch S=4 (8 imgs)  %.4f ms/slice" % (t_ms(lambda: cbp.back(g, y8)) / 8))
