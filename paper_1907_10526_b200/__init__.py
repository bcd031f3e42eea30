"""B200-native CNSF fan-beam projector (arXiv 1907.10526): thin Python binding
of the C ABI in ``include/cbp.h`` (``libcbp.so``, built in-tree for sm_100a).

Argument marshalling only: every step of forward / back-projection runs in
the library's CUDA kernels.  There is no CPU fallback: if ``libcbp.so`` is
missing or fails to load, every call raises.

Tensors: ``torch.float32``, contiguous; CUDA tensors on the current device
run asynchronously on ``torch.cuda.current_stream()`` (or the given stream);
CPU tensors / numpy arrays go through the library's host-staging path
(synchronous).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, asdict

_HERE = os.path.dirname(os.path.abspath(__file__))
# CBP_LIB_PATH: load another build of the same library (A/B experiments)
LIB_PATH = os.environ.get("CBP_LIB_PATH") or os.path.join(_HERE, "libcbp.so")

CBP_OK, CBP_EINVAL, CBP_ECUDA, CBP_ENOMEM = 0, -1, -2, -3

# names declared in include/cbp.h
ABI_FUNCTIONS = ("cbp_validate", "cbp_forward", "cbp_back", "cbp_normal", "cbp_normal_stream", "cbp_symmetry_fold",
                 "cbp_forward_orbit", "cbp_back_orbit", "cbp_forward_dihedral", "cbp_back_dihedral",
                 "cbp_sart_residual", "cbp_sart_update",
                 "cbp_fill", "cbp_dot", "cbp_cgls_step", "cbp_cgls_direction", "cbp_ref_forward",
                 "cbp_ref_back", "cbp_tv_value", "cbp_tv_gradient", "cbp_diff_norm2", "cbp_tv_step",
                 "cbp_asd_adapt", "cbp_adjoint_check", "cbp_strerror", "cbp_version",
                 "cbp_launch_count", "cbp_precise_mode", "cbp_narrow_ratio")


class CbpError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {strerror(code)} ({code})")
        self.code = code


class cbp_geometry_t(ctypes.Structure):
    """mirror of ``cbp_geometry_t`` (include/cbp.h)."""
    _fields_ = [("n", ctypes.c_int32), ("pixel", ctypes.c_double),
                ("n_views", ctypes.c_int32), ("n_det", ctypes.c_int32),
                ("det_pitch", ctypes.c_double), ("det_width", ctypes.c_double),
                ("sid", ctypes.c_double), ("sdd", ctypes.c_double), ("kind", ctypes.c_int32),
                ("model", ctypes.c_int32)]


FAN_FLAT, PARALLEL, FAN_ARC = 0, 1, 2  # cbp_geometry_t.kind
MODEL_CNSF, MODEL_MAG = 0, 1  # cbp_geometry_t.model (the paper's weight; magnified footprint, row f3)


@dataclass(frozen=True)
class Geometry:
    """Scanner and grid, mm: see include/cbp.h."""
    n: int
    pixel: float
    n_views: int
    n_det: int
    det_pitch: float
    det_width: float
    sid: float
    sdd: float
    kind: int = FAN_FLAT
    model: int = MODEL_CNSF

    @classmethod
    def from_dict(cls, d: dict) -> "Geometry":
        return cls(**{k: d[k] for k in cls.__dataclass_fields__ if k in d})

    def c_struct(self) -> cbp_geometry_t:
        return cbp_geometry_t(int(self.n), float(self.pixel), int(self.n_views), int(self.n_det),
                              float(self.det_pitch), float(self.det_width), float(self.sid),
                              float(self.sdd), int(self.kind), int(self.model))

    def as_dict(self) -> dict:
        return asdict(self)


_lib = None


def lib() -> ctypes.CDLL:
    """Load libcbp.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run `python -m paper_1907_10526_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        G = ctypes.POINTER(cbp_geometry_t)
        vp, fp = ctypes.c_void_p, ctypes.c_void_p
        i32 = ctypes.c_int32
        L.cbp_validate.argtypes = [G]
        L.cbp_validate.restype = ctypes.c_int
        L.cbp_forward.argtypes = [G, fp, fp, i32, i32, i32, vp]
        L.cbp_forward.restype = ctypes.c_int
        L.cbp_back.argtypes = [G, fp, fp, i32, i32, i32, i32, vp]
        L.cbp_back.restype = ctypes.c_int
        L.cbp_normal.argtypes = [G, fp, fp, i32, vp]
        L.cbp_normal.restype = ctypes.c_int
        L.cbp_normal_stream.argtypes = [G, fp, fp, i32, i32, vp]
        L.cbp_normal_stream.restype = ctypes.c_int
        L.cbp_symmetry_fold.argtypes = [G, i32, i32, i32]
        L.cbp_symmetry_fold.restype = ctypes.c_int
        L.cbp_forward_orbit.argtypes = [G, fp, fp, i32, i32, vp]
        L.cbp_forward_orbit.restype = ctypes.c_int
        L.cbp_back_orbit.argtypes = [G, fp, fp, i32, i32, i32, vp]
        L.cbp_forward_dihedral.argtypes = [G, fp, fp, i32, i32, vp]
        L.cbp_forward_dihedral.restype = ctypes.c_int
        L.cbp_back_dihedral.argtypes = [G, fp, fp, i32, i32, i32, vp]
        L.cbp_back_dihedral.restype = ctypes.c_int
        L.cbp_back_orbit.restype = ctypes.c_int
        i64 = ctypes.c_int64
        L.cbp_sart_residual.argtypes = [fp, fp, fp, fp, i64, vp]
        L.cbp_sart_update.argtypes = [fp, fp, fp, ctypes.c_float, i32, i64, vp]
        L.cbp_fill.argtypes = [fp, ctypes.c_float, i64, vp]
        L.cbp_dot.argtypes = [fp, fp, i64, fp, vp]
        L.cbp_cgls_step.argtypes = [fp, fp, fp, fp, fp, fp, i64, i64, vp]
        L.cbp_cgls_direction.argtypes = [fp, fp, fp, fp, i64, vp]
        for name in ("cbp_sart_residual", "cbp_sart_update", "cbp_fill", "cbp_dot",
                     "cbp_cgls_step", "cbp_cgls_direction"):
            getattr(L, name).restype = ctypes.c_int
        L.cbp_ref_forward.argtypes = [G, fp, fp, i32, i32, i32, vp]
        L.cbp_ref_forward.restype = ctypes.c_int
        L.cbp_ref_back.argtypes = [G, fp, fp, i32, i32, i32, vp]
        L.cbp_ref_back.restype = ctypes.c_int
        f64 = ctypes.c_double
        L.cbp_tv_value.argtypes = [fp, i32, i32, f64, fp, vp]
        L.cbp_tv_gradient.argtypes = [fp, fp, i32, i32, f64, vp]
        L.cbp_diff_norm2.argtypes = [fp, fp, i64, fp, vp]
        L.cbp_tv_step.argtypes = [fp, fp, i64, fp, fp, fp, vp]
        L.cbp_asd_adapt.argtypes = [fp, fp, fp, f64, f64, vp]
        for name in ("cbp_tv_value", "cbp_tv_gradient", "cbp_diff_norm2", "cbp_tv_step", "cbp_asd_adapt"):
            getattr(L, name).restype = ctypes.c_int
        L.cbp_adjoint_check.argtypes = [G, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]
        L.cbp_adjoint_check.restype = ctypes.c_int
        L.cbp_strerror.argtypes = [ctypes.c_int]
        L.cbp_strerror.restype = ctypes.c_char_p
        L.cbp_version.argtypes = []
        L.cbp_version.restype = ctypes.c_int
        L.cbp_launch_count.argtypes = []
        L.cbp_launch_count.restype = ctypes.c_uint64
        L.cbp_precise_mode.argtypes = [G]
        L.cbp_precise_mode.restype = ctypes.c_int
        L.cbp_narrow_ratio.argtypes = [G]
        L.cbp_narrow_ratio.restype = ctypes.c_double
        _lib = L
    return _lib


def _geom(geom) -> cbp_geometry_t:
    if isinstance(geom, cbp_geometry_t):
        return geom
    if isinstance(geom, Geometry):
        return geom.c_struct()
    return Geometry.from_dict(geom).c_struct()


def _checked(geom) -> cbp_geometry_t:
    g = _geom(geom)
    rc = lib().cbp_validate(ctypes.byref(g))
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_validate")
    return g


def strerror(code: int) -> str:
    return lib().cbp_strerror(code).decode()


def version() -> int:
    return lib().cbp_version()


def launch_count() -> int:
    return int(lib().cbp_launch_count())


def validate(geom) -> int:
    return lib().cbp_validate(ctypes.byref(_geom(geom)))


def precise_mode(geom) -> int:
    """1 if calls with this geometry run the narrow-bin precise mode (include/cbp.h)."""
    return lib().cbp_precise_mode(ctypes.byref(_geom(geom)))


def narrow_ratio(geom) -> float:
    """the library's lower bound on tau'/h over the field of view (include/cbp.h)."""
    return float(lib().cbp_narrow_ratio(ctypes.byref(_geom(geom))))


def _check_dev(t, shape, what, device=None):
    """a contiguous float32 CUDA tensor of exactly `shape` (the orbit / dihedral
    calls take device buffers only, and their kernels trust the extents)"""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor")
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError(f"{what}: expected a contiguous float32 tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{what}: shape {tuple(t.shape)} != {tuple(shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{what}: on {t.device}, expected {device}")


def _ptr_and_stream(t, stream):
    """(data pointer, stream handle) of a torch tensor or numpy array."""
    import numpy as np
    if isinstance(t, np.ndarray):
        if t.dtype != np.float32 or not t.flags["C_CONTIGUOUS"]:
            raise ValueError("expected a C-contiguous float32 array")
        return t.ctypes.data, 0
    import torch
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError("expected a contiguous float32 tensor")
    if t.is_cuda:
        if stream is None:
            stream = torch.cuda.current_stream(t.device)
        return t.data_ptr(), int(stream.cuda_stream if hasattr(stream, "cuda_stream") else stream)
    return t.data_ptr(), int(stream or 0)


def forward(geom, image, sino=None, view_begin: int = 0, view_count: int | None = None,
            stream=None):
    """y = A c (Eq. 6) for views [view_begin, view_begin + view_count).

    image: [n, n] or [B, n, n] float32 (CUDA tensor, CPU tensor or numpy).
    Returns sino [B?, view_count, n_det] (allocated like `image` if not given).
    """
    g = _checked(geom)
    nv = g.n_views - view_begin if view_count is None else view_count
    squeeze = image.ndim == 2
    batch = 1 if squeeze else image.shape[0]
    if tuple(image.shape[-2:]) != (g.n, g.n):
        raise ValueError(f"image shape {tuple(image.shape)} does not match n={g.n}")
    shape = (nv, g.n_det) if squeeze else (batch, nv, g.n_det)
    if sino is None:
        sino = _empty_like(image, shape)
    elif tuple(sino.shape) != shape:
        raise ValueError(f"sino shape {tuple(sino.shape)} != {shape}")
    pi, st = _ptr_and_stream(image, stream)
    ps, _ = _ptr_and_stream(sino, stream)
    rc = lib().cbp_forward(ctypes.byref(g), pi, ps, batch, view_begin, nv, st)
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_forward")
    return sino


def normal(geom, image, out=None, stream=None):
    """out = A^T A image over all views (one FP+BP pair; the sinogram stays on
    the device).  image [n, n] or [B, n, n] float32: CUDA tensor, CPU tensor or
    numpy (host buffers: synchronous)."""
    g = _checked(geom)
    squeeze = image.ndim == 2
    batch = 1 if squeeze else image.shape[0]
    if tuple(image.shape[-2:]) != (g.n, g.n):
        raise ValueError(f"image shape {tuple(image.shape)} does not match n={g.n}")
    if out is None:
        out = _empty_like(image, tuple(image.shape))
    elif tuple(out.shape) != tuple(image.shape):
        raise ValueError("out must have the image's shape")
    pi, st = _ptr_and_stream(image, stream)
    po, _ = _ptr_and_stream(out, stream)
    rc = lib().cbp_normal(ctypes.byref(g), pi, po, batch, st)
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_normal")
    return out


def normal_stream(geom, images, out=None, stream=None):
    """out[i] = A^T A images[i] for a sequence of inputs (images [count, n, n]
    or [count, B, n, n]).  Host buffers (numpy / CPU tensors; pin them for
    overlap) go through the library's copy / compute / copy pipeline and the
    call returns with every result on the host; CUDA tensors run back to back
    on the stream."""
    g = _checked(geom)
    if images.ndim not in (3, 4) or tuple(images.shape[-2:]) != (g.n, g.n):
        raise ValueError(f"images shape {tuple(images.shape)}: expected [count, (B,) {g.n}, {g.n}]")
    count = int(images.shape[0])
    batch = 1 if images.ndim == 3 else int(images.shape[1])
    if out is None:
        out = _empty_like(images, tuple(images.shape))
    elif tuple(out.shape) != tuple(images.shape):
        raise ValueError("out must have the images' shape")
    pi, st = _ptr_and_stream(images, stream)
    po, _ = _ptr_and_stream(out, stream)
    rc = lib().cbp_normal_stream(ctypes.byref(g), pi, po, count, batch, st)
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_normal_stream")
    return out


def ref_forward(geom, image, sino=None, view_begin: int = 0, view_count: int | None = None,
                stream=None):
    """Row f2: the paper's reference projector -- exact chords
    averaged over each bin, FP64 -- for views [view_begin, view_begin + view_count).

    image: [n, n] or [B, n, n] float32 CUDA tensor.  Returns a float64 CUDA
    tensor [B?, view_count, n_det].
    """
    import torch
    g = _checked(geom)
    nv = g.n_views - view_begin if view_count is None else view_count
    squeeze = image.ndim == 2
    batch = 1 if squeeze else image.shape[0]
    if tuple(image.shape[-2:]) != (g.n, g.n):
        raise ValueError(f"image shape {tuple(image.shape)} does not match n={g.n}")
    if not (isinstance(image, torch.Tensor) and image.is_cuda):
        raise ValueError("ref_forward takes CUDA tensors")
    shape = (nv, g.n_det) if squeeze else (batch, nv, g.n_det)
    if sino is None:
        sino = torch.empty(shape, dtype=torch.float64, device=image.device)
    elif tuple(sino.shape) != shape or sino.dtype != torch.float64 or not sino.is_contiguous():
        raise ValueError(f"sino must be a contiguous float64 tensor of shape {shape}")
    pi, st = _ptr_and_stream(image, stream)
    rc = lib().cbp_ref_forward(ctypes.byref(g), pi, sino.data_ptr(), batch, view_begin, nv, st)
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_ref_forward")
    return sino


def back(geom, sino, image=None, view_begin: int = 0, accumulate: bool = False, stream=None):
    """c = A^T y over views [view_begin, view_begin + sino.shape[-2]).

    sino: [V, n_det] or [B, V, n_det] float32.  Returns image [B?, n, n];
    with accumulate=True adds into the given image.
    """
    g = _checked(geom)
    squeeze = sino.ndim == 2
    batch = 1 if squeeze else sino.shape[0]
    nv = sino.shape[-2]
    if sino.shape[-1] != g.n_det:
        raise ValueError(f"sino shape {tuple(sino.shape)} does not match n_det={g.n_det}")
    shape = (g.n, g.n) if squeeze else (batch, g.n, g.n)
    if image is None:
        if accumulate:
            raise ValueError("accumulate=True needs an image to add into")
        image = _empty_like(sino, shape)
    elif tuple(image.shape) != shape:
        raise ValueError(f"image shape {tuple(image.shape)} != {shape}")
    ps, st = _ptr_and_stream(sino, stream)
    pi, _ = _ptr_and_stream(image, stream)
    rc = lib().cbp_back(ctypes.byref(g), ps, pi, batch, view_begin, nv, 1 if accumulate else 0, st)
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_back")
    return image


ACC_OVERWRITE, ACC_ADD, ACC_MULTIMEM = 0, 1, 2  # the back-projections' accumulate modes


def back_multimem(geom, sino, mc_ptr: int, view_begin: int = 0, shard=None, stream=None):
    """Row a7 fused into the BP (CBP_ACC_MULTIMEM, include/cbp.h): add this
    rank's partial A_g^T y_g to every rank's copy of the image through the
    multicast address `mc_ptr` (an int: e.g. torch symmetric memory's
    multicast_ptr).  `sino` is a CUDA tensor: [V, n_det] for the views
    view_begin.. (shard None), or the sinogram of a sharded.Shard ("orbit":
    [4, base_count, n_det]; "dihedral": the natural [n_views, n_det]).  The
    caller zeroes every copy and fences before, and fences after."""
    g = _checked(geom)
    if shard is None or shard.mode == "block":
        _check_dev(sino, (sino.shape[0] if sino.ndim == 2 else -1, g.n_det), "back_multimem sino")
    elif shard.mode == "orbit":
        _check_dev(sino, (4, shard.count, g.n_det), "back_multimem sino")
    else:
        _check_dev(sino, (g.n_views, g.n_det), "back_multimem sino")
    ps, st = _ptr_and_stream(sino, stream)
    mc = ctypes.c_void_p(int(mc_ptr))
    if shard is None or shard.mode == "block":
        v0 = view_begin if shard is None else shard.begin
        rc = lib().cbp_back(ctypes.byref(g), ps, mc, 1, v0, sino.shape[-2], ACC_MULTIMEM, st)
        name = "cbp_back"
    elif shard.mode == "orbit":
        rc = lib().cbp_back_orbit(ctypes.byref(g), ps, mc, shard.begin, shard.count, ACC_MULTIMEM, st)
        name = "cbp_back_orbit"
    else:
        rc = lib().cbp_back_dihedral(ctypes.byref(g), ps, mc, shard.begin, shard.count, ACC_MULTIMEM, st)
        name = "cbp_back_dihedral"
    if rc != CBP_OK:
        raise CbpError(rc, name)


def symmetry_fold(geom, batch: int = 1, view_begin: int = 0, view_count: int | None = None) -> int:
    """views per BP weight evaluation: 8 (dihedral), 4 (rotations) or 1 (include/cbp.h)."""
    g = _checked(geom)
    nv = g.n_views - view_begin if view_count is None else view_count
    return lib().cbp_symmetry_fold(ctypes.byref(g), batch, view_begin, nv)


def forward_orbit(geom, image, base_begin: int, base_count: int, sino=None, stream=None):
    """Views {b + q n_views/4 : b in [base_begin, base_begin + base_count), q < 4}
    of one image (CUDA tensor [n, n]); returns sino [4, base_count, n_det]."""
    g = _checked(geom)
    _check_dev(image, (g.n, g.n), "forward_orbit image")
    shape = (4, base_count, g.n_det)
    if sino is None:
        sino = _empty_like(image, shape)
    _check_dev(sino, shape, "forward_orbit sino", image.device)
    pi, st = _ptr_and_stream(image, stream)
    ps, _ = _ptr_and_stream(sino, stream)
    rc = lib().cbp_forward_orbit(ctypes.byref(g), pi, ps, base_begin, base_count, st)
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_forward_orbit")
    return sino


def back_orbit(geom, sino, base_begin: int, image=None, accumulate: bool = False, stream=None):
    """Adjoint of forward_orbit: sino [4, base_count, n_det] -> image [n, n]."""
    g = _checked(geom)
    if sino.ndim != 3:
        raise ValueError(f"back_orbit sino: expected [4, base_count, n_det], got {tuple(sino.shape)}")
    _check_dev(sino, (4, sino.shape[1], g.n_det), "back_orbit sino")
    if image is None:
        if accumulate:
            raise ValueError("accumulate=True needs an image to add into")
        image = _empty_like(sino, (g.n, g.n))
    _check_dev(image, (g.n, g.n), "back_orbit image", sino.device)
    ps, st = _ptr_and_stream(sino, stream)
    pi, _ = _ptr_and_stream(image, stream)
    rc = lib().cbp_back_orbit(ctypes.byref(g), ps, pi, base_begin, sino.shape[1],
                              1 if accumulate else 0, st)
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_back_orbit")
    return image


# ---- row f1 building blocks (device tensors, current stream) ---------------
def _dev(t):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
        raise ValueError("expected a contiguous CUDA tensor")
    return t.data_ptr()


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def _call(name, *args):
    rc = getattr(lib(), name)(*args, _stream())
    if rc != CBP_OK:
        raise CbpError(rc, name)


def sart_residual(y, ay, rowsum, r):
    _call("cbp_sart_residual", _dev(y), _dev(ay), _dev(rowsum), _dev(r), y.numel())
    return r


def sart_update(c, bp, colsum, beta: float = 1.0, nonneg: bool = True):
    _call("cbp_sart_update", _dev(c), _dev(bp), _dev(colsum), ctypes.c_float(beta),
          1 if nonneg else 0, c.numel())
    return c


def fill(x, value: float):
    _call("cbp_fill", _dev(x), ctypes.c_float(value), x.numel())
    return x


def dot(a, b, out):
    """<a, b> into the device float64 tensor `out` (shape [1])."""
    _call("cbp_dot", _dev(a), _dev(b), a.numel(), _dev(out))
    return out


def cgls_step(x, p, r, q, num, den):
    _call("cbp_cgls_step", _dev(x), _dev(p), _dev(r), _dev(q), _dev(num), _dev(den), x.numel(),
          r.numel())


def cgls_direction(p, s, num, den):
    _call("cbp_cgls_direction", _dev(p), _dev(s), _dev(num), _dev(den), p.numel())


def dihedral_views(n_views: int, base_begin: int, base_count: int):
    """the views of a dihedral shard (sorted): the orbits of its base views"""
    N = n_views
    out = set()
    for v in range(base_begin, base_begin + base_count):
        for m in (0, 1):
            for q in range(4):
                out.add(((N - v if m else v) + q * (N // 4)) % N)
    return sorted(out)


def forward_dihedral(geom, image, base_begin: int, base_count: int, sino=None, stream=None):
    """This dihedral shard's rows of y = A c in a natural [n_views, n_det]
    sinogram (zero-filled when allocated here; other rows untouched)."""
    import torch
    g = _checked(geom)
    _check_dev(image, (g.n, g.n), "forward_dihedral image")
    if sino is None:
        sino = torch.zeros((g.n_views, g.n_det), dtype=torch.float32, device=image.device)
    _check_dev(sino, (g.n_views, g.n_det), "forward_dihedral sino", image.device)
    pi, st = _ptr_and_stream(image, stream)
    ps, _ = _ptr_and_stream(sino, stream)
    rc = lib().cbp_forward_dihedral(ctypes.byref(g), pi, ps, base_begin, base_count, st)
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_forward_dihedral")
    return sino


def back_dihedral(geom, sino, base_begin: int, base_count: int, image=None, accumulate: bool = False,
                  stream=None):
    """The partial adjoint over a dihedral shard's views (natural sinogram)."""
    g = _checked(geom)
    _check_dev(sino, (g.n_views, g.n_det), "back_dihedral sino")
    if image is None:
        if accumulate:
            raise ValueError("accumulate=True needs an image to add into")
        image = _empty_like(sino, (g.n, g.n))
    _check_dev(image, (g.n, g.n), "back_dihedral image", sino.device)
    ps, st = _ptr_and_stream(sino, stream)
    pi, _ = _ptr_and_stream(image, stream)
    rc = lib().cbp_back_dihedral(ctypes.byref(g), ps, pi, base_begin, base_count, 1 if accumulate else 0, st)
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_back_dihedral")
    return image


def ref_back(geom, sino, image=None, view_begin: int = 0):
    """Row f2/f4: A_ref^T y, the exact transpose of ref_forward (FP64 in and
    out, CUDA tensors).  sino [V, n_det] or [B, V, n_det]."""
    import torch
    g = _checked(geom)
    squeeze = sino.ndim == 2
    batch = 1 if squeeze else sino.shape[0]
    if sino.dtype != torch.float64 or sino.shape[-1] != g.n_det:
        raise ValueError("sino must be float64 [B?, V, n_det]")
    shape = (g.n, g.n) if squeeze else (batch, g.n, g.n)
    if image is None:
        image = torch.empty(shape, dtype=torch.float64, device=sino.device)
    _call_g("cbp_ref_back", g, _dev(sino), _dev(image), batch, view_begin, sino.shape[-2])
    return image


def _call_g(name, g, *args):
    rc = getattr(lib(), name)(ctypes.byref(g), *args, _stream())
    if rc != CBP_OK:
        raise CbpError(rc, name)


EPS_TV = 1e-8


def tv_value(x, out, eps: float = EPS_TV):
    """TV(x) (isotropic, forward differences, reflective boundary) summed over
    the batch, into the device float64 tensor `out` [1]."""
    n = x.shape[-1]
    _call("cbp_tv_value", _dev(x), n, x.numel() // (n * n), ctypes.c_double(eps), _dev(out))
    return out


def tv_gradient(x, grad, eps: float = EPS_TV):
    n = x.shape[-1]
    _call("cbp_tv_gradient", _dev(x), _dev(grad), n, x.numel() // (n * n), ctypes.c_double(eps))
    return grad


def diff_norm2(a, b, out):
    _call("cbp_diff_norm2", _dev(a), _dev(b), a.numel(), _dev(out))
    return out


def tv_step(x, g, gg, alpha, dp2):
    _call("cbp_tv_step", _dev(x), _dev(g), x.numel(), _dev(gg), _dev(alpha), _dev(dp2))
    return x


def asd_adapt(alpha, dp2, dg2, r_max: float, alpha_red: float):
    _call("cbp_asd_adapt", _dev(alpha), _dev(dp2), _dev(dg2), ctypes.c_double(r_max),
          ctypes.c_double(alpha_red))
    return alpha


def adjoint_check(geom, seed: int = 0) -> float:
    """relative adjoint defect |<Ac,y> - <c,A^T y>| / |<Ac,y>| on the current device."""
    out = ctypes.c_double()
    rc = lib().cbp_adjoint_check(ctypes.byref(_geom(geom)), ctypes.c_uint64(seed),
                                 ctypes.byref(out))
    if rc != CBP_OK:
        raise CbpError(rc, "cbp_adjoint_check")
    return out.value


def _empty_like(ref, shape):
    import numpy as np
    if isinstance(ref, np.ndarray):
        return np.empty(shape, dtype=np.float32)
    import torch
    return torch.empty(shape, dtype=torch.float32, device=ref.device)
