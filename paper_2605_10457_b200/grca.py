"""Thin ctypes binding of include/grca.h (libgrca.so): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of csrc/grca.cu; this module
only converts Python/torch arguments to the C ABI.  There is no CPU fallback: if
the extension is missing or cannot be loaded, importing the library raises.
Function names follow the C ABI (grca_create -> Grca(), grca_cast -> Grca.cast, ...).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import Optional, Sequence

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GRCA_LIB") or os.path.join(_PKG, "libgrca.so")   # GRCA_LIB: A/B builds only

GRCA_OK, GRCA_E_INVALID, GRCA_E_STATE, GRCA_E_CAPACITY, GRCA_E_CUDA, GRCA_E_NCCL, GRCA_E_OOM = range(7)
FACES_TWO_SIDED, FACES_KEEP_POS, FACES_KEEP_NEG = 0, 1, 2
DEBUG_COUNT_ALL_HITS, DEBUG_NO_CULL, PROFILE_KERNELS, DEBUG_FORCE_FP64, DEBUG_SPLIT_REFINE, DEBUG_NO_REFINE = (
    1, 2, 4, 8, 16, 32)
L2_PERSIST = 64
DEBUG_NO_PACKED = 128
DEBUG_VIRTUAL_RANKS = 256
USE_CUDA_GRAPH = 512
SHARD_AUTO, SHARD_TRIANGLES, SHARD_EMITTERS = 0, 1, 2
MERGE_ALLREDUCE, MERGE_REDUCE_SCATTER, MERGE_NVLS = 0, 1, 2

EXPORTS = [
    "grca_create", "grca_destroy", "grca_set_emitters", "grca_update_triangles", "grca_cast",
    "grca_cast_packed", "grca_hits_packed", "grca_set_static_triangles", "grca_clear_static", "grca_unpack", "grca_get_stats", "grca_kernel_times", "grca_set_distance_noise",
    "grca_debug_all_hits", "grca_debug_large_list", "grca_debug_fast_atan2", "grca_get_layout", "grca_debug_ray_table", "grca_last_error", "grca_version",
    "grca_set_nvls", "grca_nvls_status", "grca_update_triangles_f3", "grca_update_scene",
    "grca_unpack_range", "grca_nccl_unique_id", "grca_get_shard", "grca_update_instances",
]


class GrcaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"grca status {status}: {msg}")
        self.status = status


class CreateInfo(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("stream", C.c_void_p), ("nranks", C.c_int32), ("rank", C.c_int32),
        ("nccl_uid", C.c_void_p), ("shard_mode", C.c_int32), ("merge", C.c_int32), ("gather_outputs", C.c_int32),
        ("max_triangles", C.c_int64), ("max_rays", C.c_int64), ("max_large_items", C.c_int64),
        ("faces", C.c_int32), ("debug_flags", C.c_uint32), ("small_max", C.c_int32),
        ("apparent_area_eps", C.c_float), ("reserved", C.c_int32 * 4),
    ]


class EmitterC(C.Structure):
    _fields_ = [
        ("origin", C.c_float * 3), ("forward", C.c_float * 3), ("right", C.c_float * 3), ("up", C.c_float * 3),
        ("channel_elev_rad", C.POINTER(C.c_float)), ("n_channels", C.c_int32),
        ("rays_per_channel", C.c_int32), ("hfov_deg", C.c_int32), ("max_range", C.c_float),
        ("ray_azimuth_rad", C.POINTER(C.c_float)),
    ]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "pairs", "range_culled", "channel_culled", "azimuth_culled", "survivors", "small_pairs", "large_pairs",
        "chunks", "rtic_tested", "rtic_brute", "fp64_fallbacks", "hits_recorded", "overflow_inline",
        "prefilter_survivors", "rtic_small", "sat_pairs", "bat_pairs", "area_culled", "hits_large")] + [
        ("overflow", C.c_int32), ("ms_total", C.c_float), ("ms_k", C.c_float * 8)]

    def as_dict(self) -> dict:
        d = {n: getattr(self, n) for n, _ in self._fields_ if n != "ms_k"}
        d["ms_k"] = list(self.ms_k)
        return d


_lib = None


def load(path: str = LIB_PATH):
    """Load libgrca.so (raises if missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libgrca.so not built at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    vp, i32, i64, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
    sig = {
        "grca_create": ([C.POINTER(CreateInfo), C.POINTER(vp)], C.c_int),
        "grca_destroy": ([vp], C.c_int),
        "grca_set_emitters": ([vp, C.POINTER(EmitterC), i32], C.c_int),
        "grca_update_triangles": ([vp, vp, i64, vp, i64, vp, i32], C.c_int),
        "grca_update_triangles_f3": ([vp, vp, i64, vp, i64, vp, i32], C.c_int),
        "grca_update_scene": ([vp, vp, i64, vp, i64, vp, i64, vp, i32], C.c_int),
        "grca_update_instances": ([vp, vp, i64, vp, i64, vp, i64], C.c_int),
        "grca_cast": ([vp, vp, vp, C.POINTER(Stats)], C.c_int),
        "grca_cast_packed": ([vp], C.c_int),
        "grca_set_static_triangles": ([vp, vp, i64, vp, i64, vp, i32], C.c_int),
        "grca_clear_static": ([vp], C.c_int),
        "grca_hits_packed": ([vp, C.POINTER(vp), C.POINTER(i64)], C.c_int),
        "grca_unpack": ([vp, vp, vp], C.c_int),
        "grca_unpack_range": ([vp, vp, i64, i64, vp, vp], C.c_int),
        "grca_get_stats": ([vp, C.POINTER(Stats)], C.c_int),
        "grca_set_distance_noise": ([vp, C.c_float, C.c_uint64], C.c_int),
        "grca_kernel_times": ([vp, i32, C.POINTER(C.c_float)], C.c_int),
        "grca_debug_all_hits": ([vp, C.POINTER(vp)], C.c_int),
        "grca_debug_large_list": ([vp, vp, i64, C.POINTER(i64)], C.c_int),
        "grca_debug_fast_atan2": ([vp, vp, vp, i64], C.c_int),
        "grca_get_layout": ([vp, C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "grca_debug_ray_table": ([vp, vp], C.c_int),
        "grca_set_nvls": ([vp, vp, vp, i32], C.c_int),
        "grca_nvls_status": ([vp, C.POINTER(i64), C.POINTER(i32)], C.c_int),
        "grca_last_error": ([vp], C.c_char_p),
        "grca_nccl_unique_id": ([vp], C.c_int),
        "grca_get_shard": ([vp, C.POINTER(i32), C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "grca_version": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("GRCA_AB_OLD_LIB") and not hasattr(L, name):   # tools/ab.py against an older build only
            continue
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def version() -> str:
    return load().grca_version().decode()


def nccl_unique_id() -> bytes:
    """grca_nccl_unique_id: 128 bytes for Grca(nccl_uid=...) (create on one rank, broadcast to the rest)."""
    buf = C.create_string_buffer(128)
    st = load().grca_nccl_unique_id(buf)
    if st != GRCA_OK:
        raise GrcaError(st, load().grca_last_error(None).decode())
    return buf.raw


def debug_fast_atan2(y, x):
    """Host evaluation of the cull's azimuth approximation (test-only)."""
    import numpy as np

    y = np.ascontiguousarray(np.asarray(y, dtype=np.float32))
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    out = np.empty_like(y)
    st = load().grca_debug_fast_atan2(y.ctypes.data, x.ctypes.data, out.ctypes.data, y.size)
    if st != GRCA_OK:
        raise GrcaError(st, "grca_debug_fast_atan2")
    return out


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory (no copy)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 2,
                                         "strides": None}


def _emitters_c(emitters: Sequence):
    keep = []
    arr = (EmitterC * len(emitters))()
    for k, e in enumerate(emitters):
        import numpy as np

        el = np.ascontiguousarray(np.asarray(e.elev, dtype=np.float32))
        keep.append(el)
        s = arr[k]
        for name in ("origin", "forward", "right", "up"):
            getattr(s, name)[:] = [float(x) for x in getattr(e, name)]
        s.channel_elev_rad = el.ctypes.data_as(C.POINTER(C.c_float))
        s.n_channels = int(el.shape[0])
        s.rays_per_channel = int(e.rays_per_channel)
        s.hfov_deg = int(e.hfov_deg)
        mr = float(e.max_range)
        s.max_range = mr if math.isfinite(mr) else float("inf")
        az = getattr(e, "ray_azimuth", None)
        if az is not None:
            az = np.ascontiguousarray(np.asarray(az, dtype=np.float32))
            keep.append(az)
            s.ray_azimuth_rad = az.ctypes.data_as(C.POINTER(C.c_float))
    return arr, keep


def _ptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


class Grca:
    """One handle (grca_t).  Tensors passed in must be CUDA tensors on ``device``."""

    def __init__(self, device: int = 0, stream=None, max_triangles: int = 1 << 20, max_rays: int = 1 << 20,
                 max_large_items: int = 0, faces: int = 0, debug_flags: int = 0, small_max: int = 0,
                 nranks: int = 1, rank: int = 0, apparent_area_eps: float = 0.0, nccl_uid: Optional[bytes] = None,
                 shard_mode: int = SHARD_AUTO, merge: int = MERGE_ALLREDUCE, gather_outputs: bool = False):
        import torch

        L = load()
        self._L = L
        self.device = int(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        ci = CreateInfo()
        ci.device = self.device
        ci.stream = C.c_void_p(int(stream.cuda_stream))
        ci.nranks, ci.rank = int(nranks), int(rank)
        ci.max_triangles, ci.max_rays, ci.max_large_items = int(max_triangles), int(max_rays), int(max_large_items)
        ci.faces, ci.debug_flags, ci.small_max = int(faces), int(debug_flags), int(small_max)
        ci.apparent_area_eps = float(apparent_area_eps)
        uid = None
        if nccl_uid is not None:
            assert len(nccl_uid) == 128
            uid = C.create_string_buffer(bytes(nccl_uid), 128)
            ci.nccl_uid = C.cast(uid, C.c_void_p)
        ci.shard_mode, ci.merge, ci.gather_outputs = int(shard_mode), int(merge), int(bool(gather_outputs))
        h = C.c_void_p()
        st = L.grca_create(C.byref(ci), C.byref(h))
        if st != GRCA_OK:
            raise GrcaError(st, L.grca_last_error(None).decode())
        self._h = h
        self.debug_flags = int(debug_flags)
        self.n_rays = 0
        self._tri_refs = ()

    def _check(self, st: int):
        if st != GRCA_OK:
            raise GrcaError(st, self._L.grca_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.grca_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- grca_set_emitters / grca_get_layout
    def set_emitters(self, emitters: Sequence):
        arr, keep = _emitters_c(emitters)
        self._check(self._L.grca_set_emitters(self._h, arr, len(emitters)))
        n = C.c_int64()
        offs = (C.c_int64 * (len(emitters) + 1))()
        self._check(self._L.grca_get_layout(self._h, C.byref(n), offs))
        self.n_rays = int(n.value)
        self.offsets = [int(x) for x in offs]
        return self

    # -- grca_update_triangles: vertices = float32 CUDA tensor [..., 4] (float4 rows)
    def update_triangles(self, vertices, indices=None, tri_ids=None, tri_id_base: int = 0, n_triangles=None):
        import torch

        # (n, 4) float4 vertices -> grca_update_triangles; (n, 3) packed float3 -> grca_update_triangles_f3
        assert vertices.is_cuda and vertices.dtype == torch.float32 and vertices.shape[-1] in (3, 4)
        assert vertices.is_contiguous()
        comps = vertices.shape[-1]
        nv = vertices.numel() // comps
        if indices is not None:
            assert indices.is_cuda and indices.dtype in (torch.int32, torch.uint32) and indices.is_contiguous()
            ntri = indices.numel() // 3
        else:
            ntri = nv // 3
        if n_triangles is not None:
            ntri = int(n_triangles)
        if tri_ids is not None:
            assert tri_ids.is_cuda and tri_ids.dtype == torch.int32 and tri_ids.is_contiguous()
        fn = self._L.grca_update_triangles_f3 if comps == 3 else self._L.grca_update_triangles
        self._check(fn(self._h, _ptr(vertices), nv, _ptr(indices), ntri, _ptr(tri_ids), int(tri_id_base)))
        self._tri_refs = (vertices, indices, tri_ids)
        self.n_triangles = ntri
        return self

    # -- grca_update_scene: soup = float32 CUDA [3 * n_soup, 4] (float4 triplets, triangles first),
    #    mesh_xyz = float32 CUDA [n_vertices, 3] with indices int32/uint32 [n_mesh, 3] (triangles after)
    def update_scene(self, soup=None, mesh_xyz=None, mesh_indices=None, tri_ids=None, tri_id_base: int = 0,
                     n_soup=None):
        import torch

        ns = 0
        if soup is not None:
            assert soup.is_cuda and soup.dtype == torch.float32 and soup.shape[-1] == 4 and soup.is_contiguous()
            ns = soup.numel() // 12 if n_soup is None else int(n_soup)
        nv = nm = 0
        if mesh_indices is not None:
            assert mesh_xyz is not None and mesh_xyz.is_cuda and mesh_xyz.dtype == torch.float32
            assert mesh_xyz.shape[-1] == 3 and mesh_xyz.is_contiguous()
            assert mesh_indices.is_cuda and mesh_indices.dtype in (torch.int32, torch.uint32)
            assert mesh_indices.is_contiguous()
            nv = mesh_xyz.numel() // 3
            nm = mesh_indices.numel() // 3
        if tri_ids is not None:
            assert tri_ids.is_cuda and tri_ids.dtype == torch.int32 and tri_ids.is_contiguous()
        self._check(self._L.grca_update_scene(self._h, _ptr(soup), ns, _ptr(mesh_xyz), nv, _ptr(mesh_indices), nm,
                                              _ptr(tri_ids), int(tri_id_base)))
        self._tri_refs = (soup, mesh_xyz, mesh_indices, tri_ids)
        self.n_triangles = ns + nm
        return self

    # -- grca_update_instances: local_xyz float32 CUDA [V, 3], faces int32/uint32 [F, 3], poses float32 CUDA
    #    [n_instances, 3, 4] (row-major 3x4 per instance); appended to the last update_scene / update_triangles set
    def update_instances(self, local_xyz, faces, poses):
        import torch

        assert local_xyz.is_cuda and local_xyz.dtype == torch.float32 and local_xyz.shape[-1] == 3
        assert faces.is_cuda and faces.dtype in (torch.int32, torch.uint32) and faces.is_contiguous()
        assert poses.is_cuda and poses.dtype == torch.float32 and poses.is_contiguous() and poses.shape[-2:] == (3, 4)
        assert local_xyz.is_contiguous()
        n_inst = poses.numel() // 12
        self._check(self._L.grca_update_instances(self._h, _ptr(local_xyz), local_xyz.numel() // 3, _ptr(faces),
                                                  faces.numel() // 3, _ptr(poses), n_inst))
        self._inst_refs = (local_xyz, faces, poses)
        self.n_triangles = getattr(self, "n_triangles", 0) + (faces.numel() // 3) * n_inst
        return self

    # -- grca_set_nvls / grca_nvls_status (NEXT-f3 fused NVLS merge on caller-bound buffers; the library binds
    #    its own NCCL symmetric window under merge=MERGE_NVLS)
    def set_nvls(self, uc_ptr, mc_ptr, n_ranks: int):
        self._check(self._L.grca_set_nvls(self._h, C.c_void_p(uc_ptr or None), C.c_void_p(mc_ptr or None),
                                          int(n_ranks)))

    def get_shard(self) -> dict:
        """grca_get_shard: the partition this rank casts and the output rays a cast writes."""
        mode, first, n = C.c_int32(), C.c_int64(), C.c_int64()
        self._check(self._L.grca_get_shard(self._h, C.byref(mode), C.byref(first), C.byref(n)))
        return {"shard_mode": mode.value, "first_ray": first.value, "n_written": n.value}

    def nvls_status(self) -> dict:
        need, to = C.c_int64(), C.c_int32()
        self._check(self._L.grca_nvls_status(self._h, C.byref(need), C.byref(to)))
        return {"bytes_needed": need.value, "timed_out": bool(to.value)}

    # -- grca_set_static_triangles / grca_clear_static (hybrid static/dynamic, NEXT-f2)
    def set_static_triangles(self, vertices, indices=None, tri_ids=None, tri_id_base: int = 0, n_triangles=None):
        import torch

        assert vertices.is_cuda and vertices.dtype == torch.float32 and vertices.shape[-1] == 4
        assert vertices.is_contiguous()
        nv = vertices.numel() // 4
        ntri = (indices.numel() // 3) if indices is not None else nv // 3
        if n_triangles is not None:
            ntri = int(n_triangles)
        self._check(self._L.grca_set_static_triangles(self._h, _ptr(vertices), nv, _ptr(indices), ntri, _ptr(tri_ids),
                                                      int(tri_id_base)))
        self._static_refs = (vertices, indices, tri_ids)
        return self

    def clear_static(self):
        self._check(self._L.grca_clear_static(self._h))
        self._static_refs = ()

    # -- grca_cast
    def cast(self, out_dist=None, out_tri=None, stats: bool = False):
        import torch

        if out_dist is None:
            out_dist = torch.empty(self.n_rays, dtype=torch.float32, device=f"cuda:{self.device}")
        if out_tri is None:
            out_tri = torch.empty(self.n_rays, dtype=torch.int32, device=f"cuda:{self.device}")
        s = Stats() if stats else None
        self._check(self._L.grca_cast(self._h, _ptr(out_dist), _ptr(out_tri), C.byref(s) if s is not None else None))
        return (out_dist, out_tri, s.as_dict()) if stats else (out_dist, out_tri)

    def cast_packed(self):
        self._check(self._L.grca_cast_packed(self._h))

    def hits_packed(self):
        """int64 CUDA tensor aliasing the packed hit buffer (t bits << 32 | id; >= 0 as int64)."""
        import torch

        p = C.c_void_p()
        n = C.c_int64()
        self._check(self._L.grca_hits_packed(self._h, C.byref(p), C.byref(n)))
        return torch.as_tensor(_CudaArray(int(p.value), int(n.value), "<i8"), device=f"cuda:{self.device}")

    def unpack(self, out_dist, out_tri):
        self._check(self._L.grca_unpack(self._h, _ptr(out_dist), _ptr(out_tri)))

    def unpack_range(self, keys, first_ray: int, out_dist, out_tri):
        """K5 over rays [first_ray, first_ray + n): keys = int64/uint64 CUDA tensor [n] of packed keys
        (e.g. this rank's reduce-scatter slice) or None for the handle's buffer (then n =
        out_dist/out_tri length); outputs are slice-local."""
        if keys is not None:
            assert keys.is_cuda and keys.element_size() == 8 and keys.is_contiguous()
            n = keys.numel()
        else:
            n = (out_dist if out_dist is not None else out_tri).numel()
        self._check(self._L.grca_unpack_range(self._h, _ptr(keys), int(first_ray), int(n), _ptr(out_dist),
                                              _ptr(out_tri)))

    def set_distance_noise(self, sigma: float, seed: int = 0):
        self._check(self._L.grca_set_distance_noise(self._h, float(sigma), int(seed)))

    def get_stats(self) -> dict:
        s = Stats()
        self._check(self._L.grca_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def kernel_times(self, n_last: int):
        ms = (C.c_float * 8)()
        self._check(self._L.grca_kernel_times(self._h, int(n_last), ms))
        return list(ms)

    def debug_all_hits(self):
        import torch

        p = C.c_void_p()
        self._check(self._L.grca_debug_all_hits(self._h, C.byref(p)))
        return torch.as_tensor(_CudaArray(int(p.value), self.n_rays, "<u4"), device=f"cuda:{self.device}")

    def debug_large_list(self, cap: int = 1 << 22):
        """Large-pair list of the last cast: int32 (n, 4) {tri, e | c_from << 8, c_to, r_lo | r_len << 16}."""
        import numpy as np

        out = np.empty((cap, 4), dtype=np.int32)
        n = C.c_int64()
        self._check(self._L.grca_debug_large_list(self._h, out.ctypes.data, cap, C.byref(n)))
        return out[: min(cap, int(n.value))]

    def debug_ray_table(self):
        import numpy as np

        out = np.empty((self.n_rays, 3), dtype=np.float32)
        self._check(self._L.grca_debug_ray_table(self._h, out.ctypes.data))
        return out


def tris_to_float4(tris, device="cuda"):
    """(n, 3, 3) float32 (numpy or torch) -> contiguous (3n, 4) float32 CUDA tensor (w = 0).
    Input marshalling for non-indexed triangle soups."""
    import torch

    t = torch.as_tensor(tris, dtype=torch.float32).reshape(-1, 3)
    out = torch.zeros((t.shape[0], 4), dtype=torch.float32, device=device)
    out[:, :3] = t.to(device)
    return out
