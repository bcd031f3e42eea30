"""Worker of tests/test_gpu_multi.py (one process per GPU, torchrun): the
view-sharded normal operator A^T A c over NCCL -- dihedral / orbit / block
shards, the all-reduce, and (where the system has NVLink multicast) the BP
fused with the reduction through symmetric memory -- checked on rank 0
against the FP64 oracle.  Prints one JSON line per check on rank 0."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1907_10526_b200 as cbp  # noqa: E402
import workloads as W  # noqa: E402
from paper_1907_10526_b200 import sharded  # noqa: E402


def metrics(got, ref):
    d = got.astype(np.float64) - ref
    return float(np.linalg.norm(d) / np.linalg.norm(ref)), float(np.abs(d).max() / np.abs(ref).max())


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    out = []
    for n_views, dihedral in ((88, True), (88, False), (90, False)):
        g = dict(W.geometry("1"), n_views=n_views)
        img = W.random_image(g["n"], 5)
        want = O.back(g, O.forward(g, img)) if rank == 0 else None
        res = sharded.normal_sharded(g, torch.from_numpy(img).cuda(), dihedral=dihedral)
        torch.cuda.synchronize()
        if rank == 0:
            out.append(dict(check=f"nccl n_views={n_views} dihedral={dihedral}",
                            metrics=metrics(res.cpu().numpy(), want)))
    try:
        mm = sharded.MulticastImage(64)
    except Exception as e:  # noqa: BLE001
        mm = None
        if rank == 0:
            out.append(dict(check="multimem", skipped=str(e)[:200]))
    if mm is not None:
        g = dict(W.geometry("1"), n_views=88)
        img = W.random_image(g["n"], 6)
        y, sh = sharded.forward_sharded(g, torch.from_numpy(img).cuda(), dihedral=True)
        res = sharded.back_sharded(g, y, sh, multimem=mm)
        torch.cuda.synchronize()
        if rank == 0:
            out.append(dict(check="multimem dihedral", metrics=metrics(res.cpu().numpy(),
                                                                      O.back(g, O.forward(g, img)))))
    if rank == 0:
        for o in out:
            print(json.dumps(o), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
