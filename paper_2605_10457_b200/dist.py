"""Multi-GPU partitioning and merge for the GRCA hot path.

One process per GPU, torch.distributed for the plumbing (NCCL on B200, gloo in CPU tests).

* Triangle sharding (default): triangles are independent units and the per-ray closest hit is a
  min over triangles (an associative, commutative lattice), so any partition of the triangles
  merges exactly by an element-wise min of the per-shard packed hit buffers.  Blocks of BLOCK
  consecutive triangles go to rank b mod P (heavy objects spread over ranks); global ids travel
  with the triangles.  The one exchange step is an in-place all-reduce(MIN) of the packed
  buffer (int64 view of (fp32 t bits << 32 | id): non-negative, so signed min == unsigned min).
* Sensor (emitter) sharding when Omega >= P: emitter n -> rank n mod P; every rank casts all
  triangles for its emitters; outputs are disjoint ray slices (no reduction for the cast; an
  optional all-gather assembles the full layout).

Nothing here computes any part of the method: it only partitions inputs and moves results.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

BLOCK = 4096
MISS_KEY = 0x7F800000FFFFFFFF


def shard_triangles(n_tri: int, rank: int, world: int, block: int = BLOCK) -> np.ndarray:
    """Global indices of the triangles owned by `rank` (block-interleaved)."""
    idx = np.arange(int(n_tri), dtype=np.int64)
    return idx[((idx // block) % world) == rank]


def shard_emitters(n_emitters: int, rank: int, world: int) -> List[int]:
    """Emitter indices owned by `rank` under sensor sharding (emitter n -> rank n mod P)."""
    return [n for n in range(int(n_emitters)) if n % world == rank]


def choose_mode(n_emitters: int, world: int) -> str:
    """'emitters' when every rank gets the same number of emitters (Omega >= P, P | Omega), else
    'triangles' (sensor sharding needs no reduction but re-reads all triangles)."""
    if world > 1 and n_emitters >= world and n_emitters % world == 0:
        return "emitters"
    return "triangles"


def mixed_partition(rank: int, world: int, groups: int):
    """2-D partition for `world` ranks: `groups` emitter groups x (world / groups) triangle shards.
    Rank r -> (emitter group g = r // T, triangle shard t = r mod T); ranks of one emitter group
    merge their packed keys (all-reduce MIN over a T-rank subgroup), different groups never talk."""
    assert groups >= 1 and world % groups == 0, (world, groups)
    T = world // groups
    return rank // T, rank % T, T


def merge_packed(hits, group=None):
    """In-place exact merge of per-shard packed hit buffers: all-reduce(MIN) over ranks.

    `hits` is an int64 tensor (CUDA with NCCL, CPU with gloo); returns it."""
    import torch
    import torch.distributed as dist

    assert hits.dtype == torch.int64
    dist.all_reduce(hits, op=dist.ReduceOp.MIN, group=group)
    return hits


def merge_packed_scatter(hits, group=None):
    """Exact merge with a ray-sharded result: rank r of the group receives the min over
    ranks of the keys of rays [r c, (r + 1) c), c = ceil(n / P) -- a reduce-scatter(MIN), half the
    traffic of the all-reduce.  Returns (keys slice, first ray); unpack it with Grca.unpack_range.
    NCCL: reduce_scatter_tensor; other backends (gloo tests): all-reduce then slice."""
    import torch
    import torch.distributed as dist

    assert hits.dtype == torch.int64
    P, r = dist.get_world_size(group), dist.get_rank(group)
    n = hits.numel()
    c = -(-n // P)
    src = hits if n == c * P else torch.cat([hits, torch.full((c * P - n,), MISS_KEY, dtype=hits.dtype,
                                                              device=hits.device)])
    first = r * c
    n_mine = max(0, min(c, n - first))
    if dist.get_backend(group) == "nccl":
        out = torch.empty(c, dtype=hits.dtype, device=hits.device)
        dist.reduce_scatter_tensor(out, src, op=dist.ReduceOp.MIN, group=group)
    else:
        tmp = src.clone()
        dist.all_reduce(tmp, op=dist.ReduceOp.MIN, group=group)
        out = tmp[first: first + c].clone()
    return out[:n_mine], first


def gather_emitter_slices(dist_slice, tri_slice, rank_emitters_rays: Sequence[Sequence[int]], offsets, group=None):
    """Assemble the full (dist, tri) layout from per-rank emitter slices (sensor sharding).

    rank_emitters_rays[r] lists the emitters of rank r; offsets are the global O_n (n_em + 1).
    Each rank passes its concatenated slices (in its emitter order)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n_total = int(offsets[-1])
    sizes = [sum(int(offsets[n + 1] - offsets[n]) for n in rank_emitters_rays[r]) for r in range(world)]
    mx = max(sizes)
    pad_d = torch.full((mx,), float("inf"), dtype=dist_slice.dtype, device=dist_slice.device)
    pad_t = torch.full((mx,), -1, dtype=tri_slice.dtype, device=tri_slice.device)
    pad_d[: dist_slice.numel()] = dist_slice
    pad_t[: tri_slice.numel()] = tri_slice
    gd = [torch.empty_like(pad_d) for _ in range(world)]
    gt = [torch.empty_like(pad_t) for _ in range(world)]
    dist.all_gather(gd, pad_d, group=group)
    dist.all_gather(gt, pad_t, group=group)
    out_d = torch.empty(n_total, dtype=dist_slice.dtype, device=dist_slice.device)
    out_t = torch.empty(n_total, dtype=tri_slice.dtype, device=tri_slice.device)
    for r in range(world):
        pos = 0
        for n in rank_emitters_rays[r]:
            a, b = int(offsets[n]), int(offsets[n + 1])
            out_d[a:b] = gd[r][pos: pos + (b - a)]
            out_t[a:b] = gt[r][pos: pos + (b - a)]
            pos += b - a
    return out_d, out_t


class ShardedCaster:
    """Triangle-sharded cast over a process group: each rank holds its shard's vertices (and
    their global ids); `cast()` runs K0..K4 locally, merges with all-reduce(MIN) and unpacks."""

    def __init__(self, grca, group=None):
        self.g = grca
        self.group = group

    def cast(self, out_dist, out_tri):
        self.g.cast_packed()
        merge_packed(self.g.hits_packed(), self.group)
        self.g.unpack(out_dist, out_tri)
        return out_dist, out_tri


# ----------------------------------------------------------- NEXT-f3 NVLS buffer --
def _ck(res):
    """cuda.bindings returns (err, *values); raise on error, return the value(s)."""
    from cuda.bindings import driver as cu

    err = res[0]
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver error {err}")
    return res[1] if len(res) == 2 else res[1:]


class NvlsBuffer:
    """Host plumbing of the fused NVLS merge (NEXT-f3; grca_set_nvls): one buffer of >= nbytes
    bound to a multicast object over the ranks of `group` (or a single-device multicast object
    when torch.distributed is not initialised), mapped twice on this rank:
      uc_ptr -- this rank's own copy (unicast), read by K0 / K5;
      mc_ptr -- the multicast view: a multimem reduction there lands in every rank's copy.
    Rank 0 creates the object and shares it as a fabric handle (broadcast over `group`); every
    rank adds its device, then binds its own physical memory, then maps both views.  Nothing
    here computes any part of the method."""

    def __init__(self, nbytes: int, device_index: int, group=None):
        import torch.distributed as dist
        from cuda.bindings import driver as cu

        self._cu = cu
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        _ck(cu.cuInit(0))
        dev = _ck(cu.cuDeviceGet(int(device_index)))
        if not _ck(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)):
            raise RuntimeError("multicast (NVLS) not supported on this device")
        fabric = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = self.world
        prop.handleTypes = fabric if self.world > 1 else cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE
        prop.size = int(nbytes)
        gran = int(_ck(cu.cuMulticastGetGranularity(
            prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)))
        aprop = cu.CUmemAllocationProp()
        aprop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        aprop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        aprop.location.id = int(device_index)
        agran = int(_ck(cu.cuMemGetAllocationGranularity(
            aprop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED)))
        align = max(gran, agran)
        self.size = (int(nbytes) + align - 1) // align * align
        prop.size = self.size
        if self.rank == 0:
            self.mc = _ck(cu.cuMulticastCreate(prop))
        if self.world > 1:   # share the object: fabric handle bytes over the process group
            payload = [bytes(_ck(cu.cuMemExportToShareableHandle(self.mc, fabric, 0)).data) if self.rank == 0
                       else None]
            dist.broadcast_object_list(payload, src=0, group=group)
            if self.rank != 0:
                fh = cu.CUmemFabricHandle()
                fh.data = payload[0]
                self.mc = _ck(cu.cuMemImportFromShareableHandle(fh, fabric))
        _ck(cu.cuMulticastAddDevice(self.mc, dev))
        if self.world > 1:
            dist.barrier(group)   # every device added before any memory is bound
        self.mem = _ck(cu.cuMemCreate(self.size, aprop, 0))
        _ck(cu.cuMulticastBindMem(self.mc, 0, self.mem, 0, self.size, 0))
        if self.world > 1:
            dist.barrier(group)
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = int(device_index)
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc_ptr = int(_ck(cu.cuMemAddressReserve(self.size, align, 0, 0)))
        _ck(cu.cuMemMap(self.uc_ptr, self.size, 0, self.mem, 0))
        _ck(cu.cuMemSetAccess(self.uc_ptr, self.size, [acc], 1))
        self.mc_ptr = int(_ck(cu.cuMemAddressReserve(self.size, align, 0, 0)))
        _ck(cu.cuMemMap(self.mc_ptr, self.size, 0, self.mc, 0))
        _ck(cu.cuMemSetAccess(self.mc_ptr, self.size, [acc], 1))
        _ck(cu.cuMemsetD8(self.uc_ptr, 0, self.size))
        _ck(cu.cuCtxSynchronize())
        self._dev = dev

    def close(self):
        cu = self._cu
        if getattr(self, "mc_ptr", 0):
            cu.cuCtxSynchronize()
            cu.cuMemUnmap(self.mc_ptr, self.size)
            cu.cuMemAddressFree(self.mc_ptr, self.size)
            cu.cuMemUnmap(self.uc_ptr, self.size)
            cu.cuMemAddressFree(self.uc_ptr, self.size)
            cu.cuMulticastUnbind(self.mc, self._dev, 0, self.size)
            cu.cuMemRelease(self.mem)
            cu.cuMemRelease(self.mc)
            self.mc_ptr = self.uc_ptr = 0
