"""Two processes on two GPUs over NCCL (runs only where >= 2 GPUs are
visible; the one-GPU box skips it): the sharded normal operator against the
FP64 oracle at the parity bar, through the NCCL all-reduce and, where the
system has NVLink multicast, through the BP fused with the reduction
(tests/_multi_worker.py)."""
import json
import os
import subprocess
import sys

import pytest

from tests.test_gpu_parity import MAX_REL, REL_L2

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_gpu_sharded_normal_operator():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "tests", "_multi_worker.py")]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(x) for x in res.stdout.splitlines() if x.startswith("{")]
    assert any(x["check"].startswith("nccl") for x in lines)
    for x in lines:
        if "metrics" in x:
            rl2, mr = x["metrics"]
            assert rl2 <= REL_L2 and mr <= MAX_REL, x
