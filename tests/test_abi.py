"""The C-ABI library loads and exports every symbol include/cbp.h declares;
argument validation happens before any CUDA call (no GPU needed)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1907_10526_b200 as cbp
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "cbp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cbp_\w+)\s*\(", src)))


def test_header_declares_binding_names():
    assert _declared_functions() == sorted(cbp.ABI_FUNCTIONS)


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(cbp.LIB_PATH)
    for name in _declared_functions():
        assert hasattr(L, name), name
    assert cbp.version() == 140
    assert cbp.strerror(0) == "ok"
    assert "invalid" in cbp.strerror(-1)
    assert cbp.strerror(12345) == "unknown error"


def test_struct_layout_matches_header():
    # int32, (pad), double, int32, int32, double x4, int32, int32 -> 64 bytes on LP64
    assert ctypes.sizeof(cbp.cbp_geometry_t) == 64
    assert cbp.cbp_geometry_t.kind.offset == 56
    assert cbp.cbp_geometry_t.model.offset == 60
    assert cbp.cbp_geometry_t.pixel.offset == 8
    assert cbp.cbp_geometry_t.det_pitch.offset == 24


@pytest.mark.parametrize("field,value", [
    ("n", 0), ("pixel", 0.0), ("pixel", -1.0), ("n_views", 0), ("n_det", 0),
    ("det_pitch", 0.0), ("det_width", 0.0), ("det_width", -0.5), ("sid", 0.0),
    ("sdd", 400.0), ("pixel", float("nan")), ("sid", float("inf")),
    ("sid", 45.0),  # 64 mm FOV: circumscribed radius 45.25 mm must be < sid
    ("model", 2), ("model", -1), ("kind", 3),
])
def test_validate_rejects(field, value):
    g = W.geometry("1")
    g[field] = value
    assert cbp.validate(g) == cbp.CBP_EINVAL
    img = np.zeros((64, 64), np.float32)
    with pytest.raises(cbp.CbpError) as ei:
        cbp.forward(g, img, np.zeros((90, 128), np.float32)
                    if field not in ("n_views", "n_det") else None)
    assert ei.value.code == cbp.CBP_EINVAL


def test_validate_accepts_configs():
    for name in W.CONFIGS:
        assert cbp.validate(W.geometry(name)) == cbp.CBP_OK
    for g in W.PAPER_TIMING.values():
        assert cbp.validate(g) == cbp.CBP_OK
    for g in (W.FIG5, W.FIG6, W.FIG7):
        assert cbp.validate(g) == cbp.CBP_OK


def test_bad_arguments_rejected_before_cuda():
    g = W.geometry("1")
    L = cbp.lib()
    G = ctypes.byref(cbp.Geometry.from_dict(g).c_struct())
    img = np.zeros((64, 64), np.float32)
    sino = np.zeros((90, 128), np.float32)
    pi, ps = img.ctypes.data, sino.ctypes.data
    assert L.cbp_forward(G, None, ps, 1, 0, 90, None) == cbp.CBP_EINVAL
    assert L.cbp_forward(G, pi, None, 1, 0, 90, None) == cbp.CBP_EINVAL
    assert L.cbp_forward(G, pi, ps, 0, 0, 90, None) == cbp.CBP_EINVAL
    assert L.cbp_forward(G, pi, ps, 1, -1, 10, None) == cbp.CBP_EINVAL
    assert L.cbp_forward(G, pi, ps, 1, 85, 10, None) == cbp.CBP_EINVAL
    assert L.cbp_forward(G, pi, ps, 1, 0, 0, None) == cbp.CBP_EINVAL
    assert L.cbp_forward(G, pi + 1, ps, 1, 0, 90, None) == cbp.CBP_EINVAL
    assert L.cbp_back(G, ps, pi, 1, 0, 91, 0, None) == cbp.CBP_EINVAL
    assert L.cbp_back(None, ps, pi, 1, 0, 90, 0, None) == cbp.CBP_EINVAL
    out = ctypes.c_double()
    assert L.cbp_adjoint_check(G, 0, None) == cbp.CBP_EINVAL
    assert L.cbp_adjoint_check(None, 0, ctypes.byref(out)) == cbp.CBP_EINVAL


def test_binding_shape_checks():
    g = W.geometry("1")
    with pytest.raises(ValueError):
        cbp.forward(g, np.zeros((63, 64), np.float32))
    with pytest.raises(ValueError):
        cbp.back(g, np.zeros((90, 127), np.float32))
    with pytest.raises(ValueError):
        cbp.forward(g, np.zeros((64, 64), np.float64))


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(cbp, "_lib", None)
    monkeypatch.setattr(cbp, "LIB_PATH", str(tmp_path / "libcbp.so"))
    with pytest.raises(ImportError):
        cbp.lib()


def test_no_gpu_reports_cuda_error(cuda_available):
    if cuda_available:
        pytest.skip("a GPU is present")
    g = W.geometry("1")
    with pytest.raises(cbp.CbpError) as ei:
        cbp.forward(g, np.zeros((64, 64), np.float32))
    assert ei.value.code == cbp.CBP_ECUDA


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1907_10526_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", text).replace(
                    "no oracle", ""), f


def test_fuzz_draws_are_valid_scanners():
    """the randomised GPU parity test (test_gpu_fuzz.py) draws only valid
    scanners: cbp_validate makes no CUDA call"""
    from tests.test_gpu_fuzz import draw
    for s in range(160):
        g = draw(s)[0]
        assert cbp.validate(g) == cbp.CBP_OK, (s, g)


def test_narrow_ratio_bounds_tau_prime():
    """cbp_narrow_ratio is a lower bound on tau'/h over the (view, bin, pixel)
    triples with a nonzero weight, checked against the
    oracle's explicit Eq. 13 construction (oracle.effective_blur) at the
    pixels whose support the bin ray crosses."""
    import oracle as O
    rng = np.random.default_rng(5)
    for _ in range(12):
        kind = int(rng.integers(0, 3))
        n = int(rng.integers(4, 24))
        h = float(rng.uniform(0.3, 2.0))
        R = n * h / np.sqrt(2.0)
        sid = float(R * rng.uniform(1.1, 5.0))
        sdd = float(sid * rng.uniform(1.0, 2.5))
        pitch = float(rng.uniform(0.5, 2.0) * h)
        g = dict(n=n, pixel=h, n_views=6, n_det=int(2 * sdd * np.tan(np.arcsin(R / sid)) / pitch) + 3,
                 det_pitch=pitch, det_width=float(pitch * rng.uniform(0.01, 2.0)),
                 sid=sid if kind != 1 else 0.0, sdd=sdd if kind != 1 else 0.0, kind=kind, model=0)
        if kind == 2:
            while cbp.validate(g) != cbp.CBP_OK and g["n_det"] > 1:
                g["n_det"] -= 1
        assert cbp.validate(g) == cbp.CBP_OK, g
        bound = cbp.narrow_ratio(g)
        assert bound > 0
        worst = np.inf
        for v in range(g["n_views"]):
            th = O.view_angle(g, v)
            for j in range(g["n_det"]):
                s = O.bin_center(g, j)
                for r in range(n):
                    for c in range(n):
                        k = O.pixel_center(g, r, c)
                        if O.weight(g, th, s, k) != 0.0:
                            worst = min(worst, O.effective_blur(g, th, s, k) / h)
        assert worst >= 0.99 * bound, (g, worst, bound)


def test_validate_rejects_bins_below_the_precise_range():
    g = W.geometry("1")
    assert cbp.precise_mode(g) == 0 and cbp.narrow_ratio(g) > 0.25
    g["det_width"] = 1e-5 * g["pixel"]
    assert cbp.narrow_ratio(g) < 1e-4
    assert cbp.validate(g) == cbp.CBP_EINVAL
    g["det_width"] = 1e-3 * g["pixel"]
    assert cbp.validate(g) == cbp.CBP_OK and cbp.precise_mode(g) == 1


def test_precise_mode_env_override(monkeypatch):
    g = W.geometry("1")
    monkeypatch.setenv("CBP_PRECISE", "1")
    assert cbp.precise_mode(g) == 1
    g["det_width"] = 1e-3 * g["pixel"]
    monkeypatch.setenv("CBP_PRECISE", "0")
    assert cbp.precise_mode(g) == 0
