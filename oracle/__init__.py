"""FP64 CPU oracle of the CNSF fan-beam projector (arXiv 1907.10526).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1907_10526_b200``) never imports it and
shares no code with it; see ``oracle/cnsf_oracle.c`` for the algorithm and
its paper citations.

This module is argument marshalling for ``liboracle.so`` (plain C, FP64,
OpenMP over views / image rows).  ``build()`` compiles it with gcc.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cnsf_oracle.c")
_HDR = os.path.join(_HERE, "cnsf_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# ledger #16: FP64 round-to-nearest, no FMA contraction, no fast-math
CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
          "-fno-fast-math", "-Wall", "-Wextra"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc) if missing or older than its sources."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(src) > os.path.getmtime(_LIB) for src in (_SRC, _HDR))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Geometry(ctypes.Structure):
    """The oracle's own geometry record (oracle/cnsf_oracle.h: orc_geometry)."""
    _fields_ = [("n", ctypes.c_int32), ("pixel", ctypes.c_double),
                ("n_views", ctypes.c_int32), ("n_det", ctypes.c_int32),
                ("det_pitch", ctypes.c_double), ("det_width", ctypes.c_double),
                ("sid", ctypes.c_double), ("sdd", ctypes.c_double), ("kind", ctypes.c_int32),
                ("model", ctypes.c_int32)]

    @classmethod
    def from_dict(cls, d: dict) -> "Geometry":
        # kind: 0 fan beam / flat detector (default), 1 parallel beam, 2 arc detector;
        # model: 0 the paper's CNSF weight (default), 1 the magnified-footprint variant
        return cls(int(d["n"]), float(d["pixel"]), int(d["n_views"]), int(d["n_det"]),
                   float(d["det_pitch"]), float(d["det_width"]), float(d.get("sid", 0.0)),
                   float(d.get("sdd", 0.0)), int(d.get("kind", 0)), int(d.get("model", 0)))


_D2 = ctypes.c_double * 2
_PD = ctypes.POINTER(ctypes.c_double)
_PI32 = ctypes.POINTER(ctypes.c_int32)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            G = ctypes.POINTER(Geometry)
            sig = {
                "orc_view_frame": (None, [G, ctypes.c_double, _PD, _PD, _PD]),
                "orc_detector_point": (None, [G, ctypes.c_double, ctypes.c_double, _PD]),
                "orc_ray_frame": (None, [G, ctypes.c_double, ctypes.c_double, _PD, _PD]),
                "orc_perspective_project": (ctypes.c_double, [G, ctypes.c_double, _PD]),
                "orc_effective_blur": (ctypes.c_double, [G, ctypes.c_double, ctypes.c_double, _PD]),
                "orc_pixel_center": (None, [G, ctypes.c_int32, ctypes.c_int32, _PD]),
                "orc_bin_center": (ctypes.c_double, [G, ctypes.c_int32]),
                "orc_view_angle": (ctypes.c_double, [G, ctypes.c_int32]),
                "orc_canonicalize": (ctypes.c_int, [ctypes.c_int32, _PD, ctypes.c_double, _PD]),
                "orc_box_spline": (ctypes.c_double, [ctypes.c_int32, _PD, ctypes.c_double]),
                "orc_footprint": (ctypes.c_double, [G, ctypes.c_double, ctypes.c_double, _PD]),
                "orc_weight": (ctypes.c_double, [G, ctypes.c_double, ctypes.c_double, _PD]),
                "orc_forward": (ctypes.c_int, [G, _PD, _PD, ctypes.c_int32, ctypes.c_int32,
                                               ctypes.c_int32, ctypes.c_int32]),
                "orc_back": (ctypes.c_int, [G, _PD, _PD, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_int32, ctypes.c_int32]),
                "orc_back_pixels": (ctypes.c_int, [G, _PD, ctypes.c_int32, ctypes.c_int32,
                                                   ctypes.c_int32, _PI32, _PI32, ctypes.c_int32,
                                                   _PD, ctypes.c_int32]),
                "orc_set_candidate_margin_scale": (None, [ctypes.c_double]),
                "orc_count_weights": (ctypes.c_int64, [G, ctypes.c_int32, ctypes.c_int32,
                                                       ctypes.c_int32]),
                "orc_ref_chord": (ctypes.c_double, [G, ctypes.c_double, ctypes.c_double, _PD]),
                "orc_ref_weight": (ctypes.c_double, [G, ctypes.c_double, ctypes.c_double, _PD]),
                "orc_ref_forward": (ctypes.c_int, [G, _PD, _PD, ctypes.c_int32, ctypes.c_int32,
                                                   ctypes.c_int32, ctypes.c_int32]),
                "orc_ref_back": (ctypes.c_int, [G, _PD, _PD, ctypes.c_int32, ctypes.c_int32,
                                                ctypes.c_int32, ctypes.c_int32]),
                "orc_count_weights_per_view": (ctypes.c_int, [G, ctypes.c_int32, ctypes.c_int32,
                                                              ctypes.POINTER(ctypes.c_int64),
                                                              ctypes.c_int32]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _g(geom) -> Geometry:
    return geom if isinstance(geom, Geometry) else Geometry.from_dict(geom)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_PD)


# ---- scalar steps --------------------------------------------------------
def view_frame(geom, theta):
    u, e, p = _D2(), _D2(), _D2()
    lib().orc_view_frame(ctypes.byref(_g(geom)), theta, u, e, p)
    return np.array(u), np.array(e), np.array(p)


def detector_point(geom, theta, s):
    q = _D2()
    lib().orc_detector_point(ctypes.byref(_g(geom)), theta, s, q)
    return np.array(q)


def ray_frame(geom, theta, s):
    v, r = _D2(), _D2()
    lib().orc_ray_frame(ctypes.byref(_g(geom)), theta, s, v, r)
    return np.array(v), np.array(r)


def perspective_project(geom, theta, x):
    return lib().orc_perspective_project(ctypes.byref(_g(geom)), theta, _D2(*x))


def effective_blur(geom, theta, s, k):
    return lib().orc_effective_blur(ctypes.byref(_g(geom)), theta, s, _D2(*k))


def pixel_center(geom, row, col):
    k = _D2()
    lib().orc_pixel_center(ctypes.byref(_g(geom)), row, col, k)
    return np.array(k)


def bin_center(geom, j):
    return lib().orc_bin_center(ctypes.byref(_g(geom)), j)


def view_angle(geom, v):
    return lib().orc_view_angle(ctypes.byref(_g(geom)), v)


def canonicalize(raw, eps):
    raw = np.ascontiguousarray(raw, dtype=np.float64)
    out = np.zeros(len(raw))
    m = lib().orc_canonicalize(len(raw), _dp(raw), eps, _dp(out))
    return out[:m]


def box_spline(a, x):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().orc_box_spline(len(a), _dp(a), float(x))


def footprint(geom, theta, s, k):
    return lib().orc_footprint(ctypes.byref(_g(geom)), theta, s, _D2(*k))


def weight(geom, theta, s, k):
    return lib().orc_weight(ctypes.byref(_g(geom)), theta, s, _D2(*k))


# ---- projectors ----------------------------------------------------------
def forward(geom, image, view_begin=0, view_count=None, threads=0) -> np.ndarray:
    """y = A c (Eq. 6).  image [n,n] or [B,n,n] (any float dtype, promoted
    exactly to FP64); returns FP64 sino [B?, view_count, n_det]."""
    g = _g(geom)
    img = np.ascontiguousarray(image, dtype=np.float64)
    squeeze = img.ndim == 2
    if squeeze:
        img = img[None]
    nv = g.n_views - view_begin if view_count is None else view_count
    out = np.zeros((img.shape[0], nv, g.n_det))
    rc = lib().orc_forward(ctypes.byref(g), _dp(img), _dp(out), img.shape[0], view_begin, nv,
                           threads)
    if rc != 0:
        raise ValueError("orc_forward: invalid arguments")
    return out[0] if squeeze else out


def back(geom, sino, view_begin=0, threads=0) -> np.ndarray:
    """c = A^T y.  sino [nv, n_det] or [B, nv, n_det] covering views
    [view_begin, view_begin + nv); returns FP64 image [B?, n, n]."""
    g = _g(geom)
    y = np.ascontiguousarray(sino, dtype=np.float64)
    squeeze = y.ndim == 2
    if squeeze:
        y = y[None]
    out = np.zeros((y.shape[0], g.n, g.n))
    rc = lib().orc_back(ctypes.byref(g), _dp(y), _dp(out), y.shape[0], view_begin, y.shape[1],
                        threads)
    if rc != 0:
        raise ValueError("orc_back: invalid arguments")
    return out[0] if squeeze else out


def back_pixels(geom, sino, rows, cols, view_begin=0, threads=0) -> np.ndarray:
    g = _g(geom)
    y = np.ascontiguousarray(sino, dtype=np.float64)
    squeeze = y.ndim == 2
    if squeeze:
        y = y[None]
    r = np.ascontiguousarray(rows, dtype=np.int32)
    c = np.ascontiguousarray(cols, dtype=np.int32)
    out = np.zeros((y.shape[0], len(r)))
    rc = lib().orc_back_pixels(ctypes.byref(g), _dp(y), y.shape[0], view_begin, y.shape[1],
                               r.ctypes.data_as(_PI32), c.ctypes.data_as(_PI32), len(r),
                               _dp(out), threads)
    if rc != 0:
        raise ValueError("orc_back_pixels: invalid arguments")
    return out[0] if squeeze else out


def set_candidate_margin_scale(s: float) -> None:
    lib().orc_set_candidate_margin_scale(float(s))


def count_weights(geom, view_begin=0, view_count=None, threads=0) -> int:
    g = _g(geom)
    nv = g.n_views - view_begin if view_count is None else view_count
    return int(lib().orc_count_weights(ctypes.byref(g), view_begin, nv, threads))


def count_weights_per_view(geom, view_begin=0, view_count=None, threads=0) -> np.ndarray:
    g = _g(geom)
    nv = g.n_views - view_begin if view_count is None else view_count
    out = np.zeros(nv, dtype=np.int64)
    rc = lib().orc_count_weights_per_view(ctypes.byref(g), view_begin, nv,
                                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                          threads)
    if rc != 0:
        raise ValueError("orc_count_weights_per_view: invalid arguments")
    return out


# ---- row f2: the reference projector ---------------------------
def ref_chord(geom, theta, s, k):
    return lib().orc_ref_chord(ctypes.byref(_g(geom)), theta, s, _D2(*k))


def ref_weight(geom, theta, s, k):
    return lib().orc_ref_weight(ctypes.byref(_g(geom)), theta, s, _D2(*k))


def ref_forward(geom, image, view_begin=0, view_count=None, threads=0) -> np.ndarray:
    """y = A_ref c: exact bin-averaged chords (FP64), layout as forward()."""
    g = _g(geom)
    img = np.ascontiguousarray(image, dtype=np.float64)
    squeeze = img.ndim == 2
    if squeeze:
        img = img[None]
    nv = g.n_views - view_begin if view_count is None else view_count
    out = np.zeros((img.shape[0], nv, g.n_det))
    rc = lib().orc_ref_forward(ctypes.byref(g), _dp(img), _dp(out), img.shape[0], view_begin, nv,
                               threads)
    if rc != 0:
        raise ValueError("orc_ref_forward: invalid arguments")
    return out[0] if squeeze else out


def ref_back(geom, sino, view_begin=0, threads=0) -> np.ndarray:
    """c = A_ref^T y (FP64); sino [nv, n_det] or [B, nv, n_det]."""
    g = _g(geom)
    y = np.ascontiguousarray(sino, dtype=np.float64)
    squeeze = y.ndim == 2
    if squeeze:
        y = y[None]
    out = np.zeros((y.shape[0], g.n, g.n))
    rc = lib().orc_ref_back(ctypes.byref(g), _dp(y), _dp(out), y.shape[0], view_begin, y.shape[1],
                            threads)
    if rc != 0:
        raise ValueError("orc_ref_back: invalid arguments")
    return out[0] if squeeze else out
