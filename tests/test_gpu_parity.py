"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on
identical seeded inputs.

Bar (BASELINE.json north_star; DESIGN.md ledger #18):
  relL2  = |y_gpu - y_ref|_2 / |y_ref|_2        <= 1e-5
  maxrel = max|y_gpu - y_ref| / max|y_ref|       <= 1e-4
  adjoint defect |<Ac,y> - <c,A^T y>| / |<Ac,y>| <= 1e-5
"""
import numpy as np
import pytest

import oracle as O
import paper_1907_10526_b200 as cbp
import workloads as W

pytestmark = pytest.mark.gpu

REL_L2 = 1e-5
MAX_REL = 1e-4


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _metrics(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = got - ref
    return (float(np.linalg.norm(d) / max(np.linalg.norm(ref), 1e-300)),
            float(np.abs(d).max() / max(np.abs(ref).max(), 1e-300)))


def _assert_parity(got, ref, what=""):
    rl2, mr = _metrics(got, ref)
    assert rl2 <= REL_L2 and mr <= MAX_REL, f"{what}: relL2={rl2:.3e} maxrel={mr:.3e}"


def _fp(torch, g, img, view_begin=0, view_count=None):
    t = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).cuda()
    out = cbp.forward(g, t, view_begin=view_begin, view_count=view_count)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _bp(torch, g, sino, view_begin=0):
    t = torch.from_numpy(np.ascontiguousarray(sino, dtype=np.float32)).cuda()
    out = cbp.back(g, t, view_begin=view_begin)
    torch.cuda.synchronize()
    return out.cpu().numpy()


# ---------------------------------------------------------------- config 1
CFG1_IMAGES = {
    "shepp": lambda n: W.shepp_logan(n),
    "rand1": lambda n: W.random_image(n, 1),
    "rand2": lambda n: W.random_image(n, 2),
    "rand3": lambda n: W.random_image(n, 3),
    "ones": lambda n: W.ones(n),
}


@pytest.mark.parametrize("name", sorted(CFG1_IMAGES))
def test_forward_config1(torch_cuda, name):
    g = W.geometry("1")
    img = CFG1_IMAGES[name](g["n"])
    _assert_parity(_fp(torch_cuda, g, img), O.forward(g, img), f"FP cfg1 {name}")


@pytest.mark.parametrize("seed", [101, 102, 103])
def test_back_config1(torch_cuda, seed):
    g = W.geometry("1")
    y = W.random_sino(g["n_views"], g["n_det"], seed)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), f"BP cfg1 seed {seed}")


def test_back_of_forward_config1(torch_cuda):
    g = W.geometry("1")
    y = O.forward(g, W.shepp_logan(g["n"])).astype(np.float32)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), "BP(FP(shepp)) cfg1")


def test_adjoint_config1(torch_cuda):
    g = W.geometry("1")
    assert cbp.adjoint_check(g, seed=1) <= 1e-5
    c = W.random_image(g["n"], 1)
    y = W.random_sino(g["n_views"], g["n_det"], 101)
    lhs = float(np.sum(_fp(torch_cuda, g, c).astype(np.float64) * y))
    rhs = float(np.sum(c.astype(np.float64) * _bp(torch_cuda, g, y)))
    assert abs(lhs - rhs) / abs(lhs) <= 1e-5


# ---------------------------------------------- full sizes (sampled oracle)
def _frame_views(n_views, bases):
    """the views of base views `bases` under the 8 frames of the dihedral
    symmetry: every octant of the scan, each frame of the
    symmetric kernels' output"""
    N = n_views
    return sorted({((N - b if m else b) + q * (N // 4)) % N for b in bases for m in (0, 1) for q in range(4)})


# base views per config: the octant's ends (v = 0, N/8, the axis and diagonal
# views), its first view and interior ones -> 32-40 views over the 8 frames
FRAME_BASES = {"2": (0, 1, 37, 61, 90), "3": (0, 1, 71, 133, 180), "5": (0, 1, 97, 211, 359, 360)}


@pytest.mark.parametrize("cfg", ["2", "3", "5"])
def test_forward_full_size_sampled_views(torch_cuda, cfg):
    g = W.geometry(cfg)
    img = W.shepp_logan(g["n"])
    y = _fp(torch_cuda, g, img)  # all views, the launch bench.py times
    views = _frame_views(g["n_views"], FRAME_BASES[cfg])
    assert len(views) >= 32
    for v in views:
        _assert_parity(y[v], O.forward(g, img, view_begin=v, view_count=1)[0], f"FP cfg{cfg} v{v}")
    img_r = W.random_image(g["n"], 2)
    y = _fp(torch_cuda, g, img_r)
    for v in views[::3]:
        _assert_parity(y[v], O.forward(g, img_r, view_begin=v, view_count=1)[0],
                       f"FP cfg{cfg} rand v{v}")


def _bp_sample_pixels(n, nrand, seed=11):
    """BP check pixels: corners and edge midpoints of 32 x 32 tiles (the BP's
    tile anchors and ragged borders), both diagonals (the dihedral frames'
    fixed lines), the image corners, and random pixels"""
    rng = np.random.default_rng(seed)
    T = 32
    tiles = (n + T - 1) // T
    pts = set()
    for t in rng.choice(tiles * tiles, size=min(tiles * tiles, 16), replace=False):
        r0, c0 = (t // tiles) * T, (t % tiles) * T
        r1, c1 = min(r0 + T, n) - 1, min(c0 + T, n) - 1
        rm, cm = (r0 + r1) // 2, (c0 + c1) // 2
        pts |= {(r0, c0), (r0, c1), (r1, c0), (r1, c1), (r0, cm), (r1, cm), (rm, c0), (rm, c1)}
    d = np.linspace(0, n - 1, 128).astype(int)
    pts |= {(int(i), int(i)) for i in d} | {(int(i), int(n - 1 - i)) for i in d}
    pts |= {(0, 0), (0, n - 1), (n - 1, 0), (n - 1, n - 1), (n // 2, n // 2)}
    pts |= {(int(r), int(c)) for r, c in rng.integers(0, n, (nrand, 2))}
    pts = sorted(pts)
    return np.array([p[0] for p in pts]), np.array([p[1] for p in pts])


@pytest.mark.parametrize("cfg,nrand", [("2", 96), ("3", 128), ("5", 128)])
def test_back_full_size_sampled_pixels(torch_cuda, cfg, nrand):
    g = W.geometry(cfg)
    y = W.random_sino(g["n_views"], g["n_det"], 103)
    c = _bp(torch_cuda, g, y)
    rows, cols = _bp_sample_pixels(g["n"], nrand)
    assert len(rows) >= (512 if cfg == "5" else 256)
    ref = O.back_pixels(g, y, rows, cols)
    _assert_parity(c[rows, cols], ref, f"BP cfg{cfg} sampled")
    # invariant at any size: BP is nonnegative for a nonnegative sinogram
    assert c.min() >= 0.0


def test_adjoint_config2(torch_cuda):
    assert cbp.adjoint_check(W.geometry("2"), seed=7) <= 1e-5


# ------------------------------------------------------------- edge cases
EDGE = {
    # single pixel and the paper's accuracy set-ups
    "fig5": dict(W.FIG5),
    "fig6_origin": dict(W.FIG6, n_det=41),
    "fig7": dict(W.FIG7),
    "paper64": dict(W.PAPER_TIMING[64]),
    # ragged tiles and detector blocks
    "ragged": dict(n=37, pixel=1.3, n_views=17, n_det=97, det_pitch=1.1, det_width=0.9,
                   sid=120.0, sdd=260.0),
    # one view, one bin
    "one_view": dict(n=20, pixel=1.0, n_views=1, n_det=50, det_pitch=1.0, det_width=1.0,
                     sid=60.0, sdd=100.0),
    "one_bin": dict(n=8, pixel=1.0, n_views=12, n_det=1, det_pitch=4.0, det_width=4.0,
                    sid=60.0, sdd=100.0),
    # detector at the rotation centre (D_so = 0) and bins much wider than pixels
    "dso0_wide": dict(n=24, pixel=0.5, n_views=30, n_det=9, det_pitch=3.0, det_width=3.0,
                      sid=40.0, sdd=40.0),
    # large tau / pitch ratio and many bins per pixel (BP multi-pass)
    "fine_bins": dict(n=6, pixel=2.0, n_views=10, n_det=900, det_pitch=0.05, det_width=0.2,
                      sid=30.0, sdd=55.0),
}


@pytest.mark.parametrize("name", sorted(EDGE))
def test_edge_geometries(torch_cuda, name):
    g = EDGE[name]
    img = W.random_image(g["n"], 5)
    _assert_parity(_fp(torch_cuda, g, img), O.forward(g, img), f"FP {name}")
    y = W.random_sino(g["n_views"], g["n_det"], 105)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), f"BP {name}")


def test_single_pixel_image(torch_cuda):
    g = W.geometry("1")
    img = W.single_pixel(g["n"], 10, 50)
    _assert_parity(_fp(torch_cuda, g, img), O.forward(g, img), "FP single pixel")


def test_zero_inputs(torch_cuda):
    g = W.geometry("1")
    assert not _fp(torch_cuda, g, np.zeros((64, 64), np.float32)).any()
    assert not _bp(torch_cuda, g, np.zeros((90, 128), np.float32)).any()


def test_batch_and_view_ranges(torch_cuda):
    torch = torch_cuda
    g = W.geometry("1")
    imgs = W.random_image(g["n"], 3, batch=3)
    y = _fp(torch, g, imgs, view_begin=10, view_count=25)
    assert y.shape == (3, 25, g["n_det"])
    ref = O.forward(g, imgs, view_begin=10, view_count=25)
    for b in range(3):
        _assert_parity(y[b], ref[b], f"FP batch {b}")
    ys = W.random_sino(25, g["n_det"], 101, batch=2)
    c = _bp(torch, g, ys, view_begin=10)
    refc = O.back(g, ys, view_begin=10)
    for b in range(2):
        _assert_parity(c[b], refc[b], f"BP batch {b}")


def test_accumulate_and_shards(torch_cuda):
    torch = torch_cuda
    g = W.geometry("1")
    y = torch.from_numpy(W.random_sino(g["n_views"], g["n_det"], 102)).cuda()
    full = cbp.back(g, y)
    acc = cbp.back(g, y[:40].contiguous(), view_begin=0)
    cbp.back(g, y[40:].contiguous(), image=acc, view_begin=40, accumulate=True)
    torch.cuda.synchronize()
    _assert_parity(acc.cpu().numpy(), full.cpu().numpy(), "BP shards")


def test_deterministic(torch_cuda):
    torch = torch_cuda
    g = W.geometry("2")
    img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
    y1 = cbp.forward(g, img)
    y2 = cbp.forward(g, img)
    c1 = cbp.back(g, y1)
    c2 = cbp.back(g, y1)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and torch.equal(c1, c2)


def test_host_buffers_match_device(torch_cuda):
    torch = torch_cuda
    g = W.geometry("1")
    img = W.random_image(g["n"], 1)
    y_host = cbp.forward(g, img)  # numpy in, numpy out (staged)
    y_dev = cbp.forward(g, torch.from_numpy(img).cuda()).cpu().numpy()
    assert np.array_equal(y_host, y_dev)
    c_host = cbp.back(g, y_host)
    c_dev = cbp.back(g, torch.from_numpy(y_host).cuda()).cpu().numpy()
    assert np.array_equal(c_host, c_dev)
    assert np.isfinite(c_host).all()


@pytest.mark.parametrize("batch", [2, 3, 4, 5, 9])
def test_batched_slices(torch_cuda, batch):
    """Batches share each weight across S slices (S = 4, 2, 1 per group) --
    every slice must match the oracle, including ragged last groups."""
    g = W.geometry("1")
    imgs = W.random_image(g["n"], 7, batch=batch)
    y = _fp(torch_cuda, g, imgs)
    ref = O.forward(g, imgs)
    for b in range(batch):
        _assert_parity(y[b], ref[b], f"FP batch {batch} slice {b}")
    ys = W.random_sino(g["n_views"], g["n_det"], 107, batch=batch)
    c = _bp(torch_cuda, g, ys)
    refc = O.back(g, ys)
    for b in range(batch):
        _assert_parity(c[b], refc[b], f"BP batch {batch} slice {b}")


def test_batched_config4_sampled(torch_cuda):
    """config 4 (64 x 512^2, 720 views), sampled: views of slices 0, 33 and 63
    for FP; pixels of slices 5 and 62 for BP."""
    torch = torch_cuda
    g = W.geometry("4")
    imgs = W.jittered_batch(g["n"], 64, seed=7)
    y = cbp.forward(g, torch.from_numpy(imgs).cuda())
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    for b, v in [(0, 0), (33, 200), (63, 719)]:
        _assert_parity(y[b, v], O.forward(g, imgs[b], view_begin=v, view_count=1)[0],
                       f"FP cfg4 slice {b} view {v}")
    c = cbp.back(g, torch.from_numpy(y).cuda())
    torch.cuda.synchronize()
    c = c.cpu().numpy()
    rng = np.random.default_rng(12)
    rows, cols = rng.integers(0, g["n"], 24), rng.integers(0, g["n"], 24)
    for b in (5, 62):
        _assert_parity(c[b, rows, cols], O.back_pixels(g, y[b], rows, cols), f"BP cfg4 slice {b}")


@pytest.mark.parametrize("n_views,fold", [(88, 8), (92, 4), (360, 8)])
def test_rotational_symmetry_path(torch_cuda, n_views, fold):
    """A full scan with one image runs the symmetric path -- 8-fold (rotations
    and mirror) when N_v % 8 == 0, 4-fold (rotations) when N_v % 4 == 0 --
    partial view ranges run the direct path.  Both must match the oracle,
    and each other."""
    torch = torch_cuda
    g = dict(W.geometry("1"), n_views=n_views)
    assert cbp.symmetry_fold(g) == fold
    img = W.shepp_logan(g["n"])
    y_sym = _fp(torch, g, img)                       # full range: symmetric
    y_a = _fp(torch, g, img, view_begin=0, view_count=n_views // 2)
    y_b = _fp(torch, g, img, view_begin=n_views // 2, view_count=n_views // 2)
    ref = O.forward(g, img)
    _assert_parity(y_sym, ref, "FP symmetric")
    _assert_parity(np.concatenate([y_a, y_b]), ref, "FP direct")
    np.testing.assert_allclose(y_sym, np.concatenate([y_a, y_b]), rtol=2e-5, atol=1e-5 * ref.max())
    ys = W.random_sino(n_views, g["n_det"], 108)
    c_sym = _bp(torch, g, ys)
    c_dir = _bp(torch, g, ys[: n_views // 2], 0) + _bp(torch, g, ys[n_views // 2:], n_views // 2)
    refc = O.back(g, ys)
    _assert_parity(c_sym, refc, "BP symmetric")
    _assert_parity(c_dir, refc, "BP direct")
    # accumulate on the symmetric path
    t = torch.from_numpy(ys).cuda()
    acc = torch.from_numpy(c_dir).cuda()
    cbp.back(g, t, image=acc, accumulate=True)
    torch.cuda.synchronize()
    _assert_parity(acc.cpu().numpy(), 2 * refc, "BP symmetric accumulate")


def test_orbit_shards_sum_to_full(torch_cuda):
    """The orbit ABI (the multi-GPU shard shape): two 'ranks' run in sequence
    on one GPU, each FP-projects the 4 rotated copies of its base-view block
    and back-projects them; rows match the oracle and the partial images sum
    to the full back-projection (the all_reduce of row a7)."""
    torch = torch_cuda
    from paper_1907_10526_b200 import sharded
    g = W.geometry("2")
    img = torch.from_numpy(W.shepp_logan(g["n"])).cuda()
    total = torch.zeros((g["n"], g["n"]), device="cuda")
    ys = []
    for rank in range(2):
        sh = sharded.make_shard(g["n_views"], rank, 2)
        assert sh.mode == "orbit"
        y = cbp.forward_orbit(g, img, sh.begin, sh.count)
        cbp.back_orbit(g, y, sh.begin, image=total, accumulate=True)
        ys.append((sh, y))
    full_y = cbp.forward(g, img)
    full_c = cbp.back(g, full_y)
    torch.cuda.synchronize()
    for sh, y in ys:
        rows = torch.from_numpy(sh.views()).cuda()
        torch.testing.assert_close(y.reshape(-1, g["n_det"]), full_y[rows], rtol=1e-5, atol=1e-4)
    _assert_parity(total.cpu().numpy(), full_c.cpu().numpy(), "orbit shards summed")
    sh = sharded.make_shard(g["n_views"], 1, 2)
    for v in (int(sh.views()[0]), int(sh.views()[-1])):
        _assert_parity(full_y[v].cpu().numpy(), O.forward(g, W.shepp_logan(g["n"]), v, 1)[0],
                       f"FP view {v}")


def test_symmetry_ragged_odd_grid(torch_cuda):
    """8-fold path on an odd, ragged grid (n = 37: the pixel rotations and the
    mirror must map the grid onto itself exactly)."""
    g = dict(EDGE["ragged"], n_views=16)
    assert cbp.symmetry_fold(g) == 8
    img = W.random_image(g["n"], 9)
    _assert_parity(_fp(torch_cuda, g, img), O.forward(g, img), "FP ragged sym8")
    y = W.random_sino(g["n_views"], g["n_det"], 109)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), "BP ragged sym8")


@pytest.mark.parametrize("batch", [1, 5])
def test_close_source_ragged_tiles(torch_cuda, batch):
    """Regression: a ragged 5-column tile next to a close source (FOV radius 34
    of sid 40 mm) -- its circumscribed circle reaches behind the source, so the
    BP tile range must use the least pixel depth, not anchor depth - radius."""
    g = dict(n=37, n_views=30, n_det=101, pixel=1.3, det_pitch=1.87, det_width=1.1, sid=40.0, sdd=90.0)
    imgs = W.random_image(37, 7, batch=batch)
    _assert_parity(_fp(torch_cuda, g, imgs), O.forward(g, imgs), "FP close source")
    y = W.random_sino(30, 101, 8, batch=batch)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), "BP close source")
    assert cbp.adjoint_check(g, seed=2) <= 1e-5


@pytest.mark.parametrize("cfg,batch", [("1", 1), ("1", 3), ("2", 1)])
def test_normal_operator(torch_cuda, cfg, batch):
    """cbp_normal = A^T A over all views, device and host buffers, equals
    back(forward(.)) of the same library (and, at config 1, the oracle's)."""
    torch = torch_cuda
    g = W.geometry(cfg)
    img = W.random_image(g["n"], 21, batch=None if batch == 1 else batch)
    d = torch.from_numpy(img).cuda()
    got = cbp.normal(g, d)
    want = cbp.back(g, cbp.forward(g, d))
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    host = cbp.normal(g, torch.from_numpy(img).pin_memory())
    assert torch.equal(host, want.cpu())
    if cfg == "1":
        _assert_parity(host.numpy(), O.back(g, O.forward(g, img)), "normal cfg1")


@pytest.mark.parametrize("batch,n_views", [(3, 88), (5, 360)])
def test_batched_bp_uses_per_image_dihedral_symmetry(torch_cuda, batch, n_views):
    """A batch over a full scan with n_views % 8 == 0: the BP runs the 8 frames
    of each image (partial planes [images][groups][8]); parity per image."""
    g = dict(W.geometry("1"), n_views=n_views)
    assert cbp.symmetry_fold(g, batch) == 8
    y = W.random_sino(n_views, g["n_det"], 31, batch=batch)
    _assert_parity(_bp(torch_cuda, g, y), O.back(g, y), f"BP batch {batch} sym8")
    imgs = W.random_image(g["n"], 32, batch=batch)
    _assert_parity(_fp(torch_cuda, g, imgs), O.forward(g, imgs), f"FP batch {batch}")
    lhs = float(np.sum(_fp(torch_cuda, g, imgs).astype(np.float64) * y))
    rhs = float(np.sum(imgs.astype(np.float64) * _bp(torch_cuda, g, y)))
    assert abs(lhs - rhs) / abs(lhs) <= 1e-5


@pytest.mark.parametrize("n_views,world", [(88, 2), (88, 3), (720, 8)])
def test_dihedral_shards_sum_to_full(torch_cuda, n_views, world):
    """Dihedral shards (one GPU, shards run one after another): each shard's
    FP rows are the full FP's rows, and the partial BPs sum to the full BP."""
    from paper_1907_10526_b200 import sharded
    torch = torch_cuda
    g = dict(W.geometry("1"), n_views=n_views) if n_views == 88 else W.geometry("2")
    img = torch.from_numpy(W.random_image(g["n"], 51)).cuda()
    full_y = cbp.forward(g, img)
    y_rand = torch.from_numpy(W.random_sino(g["n_views"], g["n_det"], 52)).cuda()
    full_c = cbp.back(g, y_rand)
    total = torch.zeros_like(full_c)
    seen = []
    for r in range(world):
        sh = sharded.make_shard(g["n_views"], r, world, dihedral=True)
        assert sh.mode == "dihedral"
        rows = torch.as_tensor(sh.views(), device="cuda")
        y = cbp.forward_dihedral(g, img, sh.begin, sh.count)
        _assert_parity(y[rows].cpu().numpy(), full_y[rows].cpu().numpy(), f"FP dihedral shard {r}")
        total += cbp.back_dihedral(g, y_rand, sh.begin, sh.count)
        seen += sh.views().tolist()
    assert sorted(seen) == list(range(g["n_views"]))
    torch.cuda.synchronize()
    _assert_parity(total.cpu().numpy(), full_c.cpu().numpy(), "BP dihedral shards")


def test_rot_rows_fp_matches_oracle(torch_cuda, monkeypatch):
    # the opt-in rot_rows FP (CBP_ROTROWS=1, read once per process: run in a child)
    import subprocess
    import sys
    code = ("import sys, numpy as np, torch; sys.path.insert(0, '.');"
            "import oracle as O, paper_1907_10526_b200 as cbp, workloads as W;"
            "from tests.test_gpu_parity import _metrics;"
            "g = dict(W.geometry('1'), n_views=88); img = W.shepp_logan(64);"
            "y = cbp.forward(g, torch.from_numpy(img).cuda()).cpu().numpy();"
            "print(*_metrics(y, O.forward(g, img)))")
    import os
    env = dict(os.environ, CBP_ROTROWS="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    rl2, mr = (float(x) for x in out.stdout.split())
    assert rl2 <= REL_L2 and mr <= MAX_REL, (rl2, mr)


@pytest.mark.parametrize("wide", ["0", "1"])
def test_bp_chunk_shapes(torch_cuda, monkeypatch, wide):
    """The 8-frame BP's two chunk shapes (cbp::BPShape: 8 views x 80 bins, or
    4 views x 128 bins chosen for wide projected tiles such as the paper's
    timing shapes), each forced on a narrow and a wide geometry (CBP_BP_WIDE):
    one image, a batch of images (per-image frames), and dihedral shards
    summing to the full BP -- all against the oracle."""
    torch = torch_cuda
    from paper_1907_10526_b200 import sharded
    monkeypatch.setenv("CBP_BP_WIDE", wide)
    for g in (dict(W.geometry("1"), n_views=88), dict(W.PAPER_TIMING[64])):
        y = W.random_sino(g["n_views"], g["n_det"], 121)
        want = O.back(g, y)
        _assert_parity(_bp(torch, g, y), want, f"BP shape {wide} n_views {g['n_views']}")
        ys = W.random_sino(g["n_views"], g["n_det"], 122, batch=2)
        _assert_parity(_bp(torch, g, ys), np.stack([O.back(g, ys[b]) for b in range(2)]),
                       f"BP shape {wide} batch")
        yt = torch.from_numpy(y).cuda()
        total = torch.zeros((g["n"], g["n"]), device="cuda")
        for r in range(3):
            sh = sharded.make_shard(g["n_views"], r, 3, dihedral=True)
            total += cbp.back_dihedral(g, yt, sh.begin, sh.count)
        _assert_parity(total.cpu().numpy(), want, f"BP shape {wide} dihedral shards")


CLAMPED_FP = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1907_10526_b200 as cbp, workloads as W
g = %r
img = torch.from_numpy(W.random_image(g["n"], 77)).cuda()
np.save(%r, cbp.forward(g, img).cpu().numpy())
'''


@pytest.mark.parametrize("cfg", ["1", "2", "2v721"])
def test_fp_without_clamp_is_exact(torch_cuda, tmp_path, cfg):
    """The FP walks without its tau' clamp where the host proves tau' > 0 over
    the padded grid (fp_tau_positive); there the clamp (max(tau', 1e-30)) never
    acts, so the two kernels must agree bit for bit.  The clamped one is forced
    in a subprocess (CBP_FP_CLAMP is read once per process)."""
    import os
    import subprocess
    import sys
    torch = torch_cuda
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    g = W.geometry(cfg)
    out = str(tmp_path / "clamped.npy")
    res = subprocess.run([sys.executable, "-c", CLAMPED_FP % (root, g, out)], env=dict(os.environ, CBP_FP_CLAMP="1"),
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    img = torch.from_numpy(W.random_image(g["n"], 77)).cuda()
    assert np.array_equal(cbp.forward(g, img).cpu().numpy(), np.load(out))
