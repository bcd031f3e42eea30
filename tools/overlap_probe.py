"""Does running the FP of one batch chunk concurrently with the BP of the
previous chunk (two streams) beat running them back to back?  Config 4."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402

g = W.geometry("4")
B = 64
imgs = torch.from_numpy(W.jittered_batch(g["n"], B, seed=7)).cuda()
sino = torch.empty((B, g["n_views"], g["n_det"]), device="cuda")
out = torch.empty_like(imgs)


def seq():
    cbp.forward(g, imgs, sino)
    cbp.back(g, sino, out)


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def pipelined(chunk):
    evs = []
    main = torch.cuda.current_stream()
    s1.wait_stream(main)
    s2.wait_stream(main)
    for c0 in range(0, B, chunk):
        with torch.cuda.stream(s1):
            cbp.forward(g, imgs[c0:c0 + chunk], sino[c0:c0 + chunk], stream=s1)
            e = torch.cuda.Event()
            e.record(s1)
        with torch.cuda.stream(s2):
            s2.wait_event(e)
            cbp.back(g, sino[c0:c0 + chunk], out[c0:c0 + chunk], stream=s2)
    main.wait_stream(s2)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


print("sequential %.3f ms" % t(seq))
for chunk in (32, 16, 8, 4):
    print("pipelined chunk %d: %.3f ms" % (chunk, t(lambda: pipelined(chunk))))
