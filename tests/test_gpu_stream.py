"""cbp_normal_stream: the copy / compute / copy pipeline over host buffers
returns, image by image, exactly what cbp_normal computes on the device (the
same kernels in the same order: bitwise), for pinned and pageable host
memory, batches, one input, and device buffers; mixed pointers are rejected."""
import numpy as np
import pytest

import paper_1907_10526_b200 as cbp
import workloads as W

from tests.test_gpu_parity import torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu


def _reference(torch, g, imgs):
    return np.stack([cbp.normal(g, torch.from_numpy(np.ascontiguousarray(x)).cuda()).cpu().numpy()
                     for x in imgs])


@pytest.mark.parametrize("cfg,count", [("1", 5), ("2", 4), ("1", 1)])
def test_stream_matches_normal(torch_cuda, cfg, count):
    torch = torch_cuda
    g = W.geometry(cfg)
    imgs = np.stack([W.random_image(g["n"], 60 + i) for i in range(count)])
    want = _reference(torch, g, imgs)
    # pageable numpy buffers
    got = cbp.normal_stream(g, imgs)
    np.testing.assert_array_equal(got, want)
    # pinned CPU tensors
    h = torch.from_numpy(imgs).pin_memory()
    out = torch.empty_like(h).pin_memory()
    cbp.normal_stream(g, h, out)
    np.testing.assert_array_equal(out.numpy(), want)
    # device tensors: back to back on the stream
    d = cbp.normal_stream(g, h.cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(d.cpu().numpy(), want)


def test_stream_batch_and_rejects_mixed(torch_cuda):
    torch = torch_cuda
    g = W.geometry("1")
    imgs = W.random_image(g["n"], 70, batch=6).reshape(3, 2, g["n"], g["n"])
    got = cbp.normal_stream(g, imgs)
    for i in range(3):
        want = cbp.normal(g, torch.from_numpy(imgs[i]).cuda()).cpu().numpy()
        np.testing.assert_array_equal(got[i], want)
    with pytest.raises(cbp.CbpError):
        cbp.normal_stream(g, imgs, torch.empty(imgs.shape, device="cuda"))
