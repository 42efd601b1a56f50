"""ctypes wrapper of oracle/grca_oracle.c (TEST INFRASTRUCTURE ONLY).

Functions follow the passages cited in grca_oracle.c:
  ray_table -> O1, cast -> O2/O3,
  ray_tri   -> single fp64 Moller-Trumbore query used by the comparator.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "grca_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def lib_path() -> str:
    return _LIB


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction: plain IEEE fp64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-pthread", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Em(C.Structure):
    _fields_ = [
        ("origin", C.c_float * 3),
        ("forward", C.c_float * 3),
        ("right", C.c_float * 3),
        ("up", C.c_float * 3),
        ("channel_elev_rad", C.POINTER(C.c_float)),
        ("n_channels", C.c_int32),
        ("rays_per_channel", C.c_int32),
        ("hfov_deg", C.c_int32),
        ("max_range", C.c_float),
        ("ray_azimuth_rad", C.POINTER(C.c_float)),
    ]


_lib = None


def _get():
    global _lib
    if _lib is None:
        build_oracle()
        L = C.CDLL(_LIB)
        L.oracle_n_rays.restype = C.c_int64
        L.oracle_n_rays.argtypes = [C.POINTER(_Em), C.c_int32]
        L.oracle_ray_table.restype = None
        L.oracle_ray_table.argtypes = [C.POINTER(_Em), C.c_int32, C.c_void_p]
        L.oracle_mt.restype = C.c_int
        L.oracle_mt.argtypes = [C.POINTER(C.c_double)] * 5 + [C.POINTER(C.c_double)] * 4
        L.oracle_ray_tri.restype = C.c_int
        L.oracle_ray_tri.argtypes = [C.POINTER(_Em), C.c_int32, C.c_int64, C.c_void_p, C.c_int32,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.oracle_near_edge_count.restype = C.c_int64
        L.oracle_near_edge_count.argtypes = [C.POINTER(_Em), C.c_int32, C.c_int64, C.c_void_p, C.c_int64, C.c_double]
        L.oracle_cast.restype = C.c_int
        L.oracle_cast.argtypes = [C.POINTER(_Em), C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                  C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p]
        _lib = L
    return _lib


class _EmArray:
    """Keeps the ctypes emitter array and its elevation buffers alive."""

    def __init__(self, emitters: Sequence):
        self.elevs = [np.ascontiguousarray(np.asarray(e.elev, dtype=np.float32)) for e in emitters]
        self.arr = (_Em * len(emitters))()
        for k, e in enumerate(emitters):
            s = self.arr[k]
            for name in ("origin", "forward", "right", "up"):
                v = np.asarray(getattr(e, name), dtype=np.float32)
                getattr(s, name)[:] = [float(x) for x in v]
            s.channel_elev_rad = self.elevs[k].ctypes.data_as(C.POINTER(C.c_float))
            s.n_channels = int(self.elevs[k].shape[0])
            s.rays_per_channel = int(e.rays_per_channel)
            s.hfov_deg = int(e.hfov_deg)
            s.max_range = float(e.max_range)
            az = getattr(e, "ray_azimuth", None)
            if az is not None:
                az = np.ascontiguousarray(np.asarray(az, dtype=np.float32))
                assert az.shape[0] == int(e.rays_per_channel)
                self.elevs.append(az)
                s.ray_azimuth_rad = az.ctypes.data_as(C.POINTER(C.c_float))
        self.n = len(emitters)


def n_rays(emitters) -> int:
    A = _EmArray(emitters)
    return int(_get().oracle_n_rays(A.arr, A.n))


def ray_table(emitters) -> np.ndarray:
    """O1: fp32 ray directions (n_rays, 3), channel-major per emitter (g = O_n + j*chi + i)."""
    A = _EmArray(emitters)
    L = _get()
    n = int(L.oracle_n_rays(A.arr, A.n))
    out = np.empty((n, 3), dtype=np.float32)
    L.oracle_ray_table(A.arr, A.n, out.ctypes.data)
    return out


def mt(o, d, v0, v1, v2):
    """Textbook fp64 Moller-Trumbore; returns (ok, t, u, v, dN) -- ok=False when det == 0."""
    arrs = [np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(3)) for x in (o, d, v0, v1, v2)]
    ptrs = [a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs]
    t, u, v, dN = C.c_double(), C.c_double(), C.c_double(), C.c_double()
    ok = _get().oracle_mt(*ptrs, C.byref(t), C.byref(u), C.byref(v), C.byref(dN))
    return bool(ok), t.value, u.value, v.value, dN.value


def ray_tri(emitters, g: int, tri9, faces: int = 0, _arr: Optional[_EmArray] = None):
    """fp64 query of global ray g against one triangle: (ok, t, u, v, hit)."""
    A = _arr or _EmArray(emitters)
    T = np.ascontiguousarray(np.asarray(tri9, dtype=np.float32).reshape(9))
    t, u, v, hit = C.c_double(), C.c_double(), C.c_double(), C.c_int32()
    ok = _get().oracle_ray_tri(A.arr, A.n, int(g), T.ctypes.data, int(faces), C.byref(t), C.byref(u),
                               C.byref(v), C.byref(hit))
    if ok < 0:
        raise IndexError(g)
    return bool(ok), t.value, u.value, v.value, bool(hit.value)


def near_edge_count(emitters, g: int, tris: np.ndarray, eps: float = 1e-6) -> int:
    """Triangles hit (t in (0, D_max]) by ray g within `eps` of their boundary (fp64 barycentric margin):
    by how much a per-ray all-hit count may legitimately differ (grca_oracle.c oracle_near_edge_count)."""
    A = _EmArray(emitters)
    T = np.ascontiguousarray(np.asarray(tris, dtype=np.float32).reshape(-1, 9))
    r = _get().oracle_near_edge_count(A.arr, A.n, int(g), T.ctypes.data if T.shape[0] else None, T.shape[0], float(eps))
    if r < 0:
        raise IndexError(g)
    return int(r)


def cast(emitters, tris: np.ndarray, ids: Optional[np.ndarray] = None, faces: int = 0,
         rays: Optional[np.ndarray] = None, threads: Optional[int] = None, want_t64: bool = False,
         want_allhits: bool = False) -> dict:
    """O2/O3 brute force: every (ray, triangle) pair, closest hit, ties -> smaller id.

    tris: (n, 3, 3) fp32.  rays: optional int64 global ray indices (sampled parity).
    Returns dict(t=float32[n_r], id=int32[n_r], t64=?, allhits=?, rays=int64[n_r]).
    """
    A = _EmArray(emitters)
    L = _get()
    T = np.ascontiguousarray(np.asarray(tris, dtype=np.float32).reshape(-1, 9))
    ntri = T.shape[0]
    idp = None
    if ids is not None:
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int32))
        assert ids.shape[0] == ntri
        idp = ids.ctypes.data
    if rays is None:
        nr = int(L.oracle_n_rays(A.arr, A.n))
        rp = None
        rays_out = np.arange(nr, dtype=np.int64)
    else:
        rays = np.ascontiguousarray(np.asarray(rays, dtype=np.int64))
        nr = rays.shape[0]
        rp = rays.ctypes.data
        rays_out = rays
    if threads is None:
        threads = os.cpu_count() or 1
    out_t = np.empty(nr, dtype=np.float32)
    out_id = np.empty(nr, dtype=np.int32)
    t64 = np.empty(nr, dtype=np.float64) if want_t64 else None
    ah = np.empty(nr, dtype=np.uint32) if want_allhits else None
    L.oracle_cast(A.arr, A.n, T.ctypes.data if ntri else None, idp, ntri, int(faces), rp, nr, int(threads),
                  out_t.ctypes.data, out_id.ctypes.data, t64.ctypes.data if t64 is not None else None,
                  ah.ctypes.data if ah is not None else None)
    return {"t": out_t, "id": out_id, "t64": t64, "allhits": ah, "rays": rays_out}
