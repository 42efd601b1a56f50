"""Multi-GPU plumbing for the GRCA hot path: partitions and the communicator id.

One process per GPU.  The collective itself lives in the library: a handle created with an NCCL
unique id (include/grca.h: grca_create_info.nccl_uid / shard_mode / merge / gather_outputs) owns its
NCCL communicator, and grca_cast merges in-stream between K4 and K5:

* Triangle sharding: each rank passes its own triangles (with their global ids).  The per-ray closest
  hit is a min over triangles (an associative, commutative lattice), so the shards merge exactly by an
  element-wise min of the packed (fp32 t bits << 32 | id) keys: ncclAllReduce(ncclUint64, ncclMin), a
  ncclReduceScatter (ray-sharded outputs, half the traffic), or the fused NVLS multimem.red.min into an
  NCCL symmetric window.
* Sensor (emitter) sharding when Omega >= P and P | Omega: every rank passes all triangles and the
  library casts emitters n mod P == rank; outputs are disjoint ray slices (optionally broadcast to all
  ranks, gather_outputs).

This module only decides partitions and moves the 128-byte communicator id; it computes no part of
the method and runs no data-path collective.
"""
from __future__ import annotations

from typing import List

import numpy as np

BLOCK = 4096
MISS_KEY = 0x7F800000FFFFFFFF


def shard_triangles(n_tri: int, rank: int, world: int, block: int = BLOCK) -> np.ndarray:
    """Global indices of the triangles owned by `rank` (blocks of `block` go to rank b mod P, so heavy
    objects spread over the ranks)."""
    idx = np.arange(int(n_tri), dtype=np.int64)
    return idx[((idx // block) % world) == rank]


def shard_emitters(n_emitters: int, rank: int, world: int) -> List[int]:
    """Emitters cast by `rank` under sensor sharding (the library's rule: emitter n -> rank n mod P)."""
    return [n for n in range(int(n_emitters)) if n % world == rank]


def choose_mode(n_emitters: int, world: int) -> str:
    """GRCA_SHARD_AUTO's rule: 'emitters' when every rank gets the same number of emitters (Omega >= P,
    P | Omega), else 'triangles' (sensor sharding needs no reduction but re-reads all triangles)."""
    if world > 1 and n_emitters >= world and n_emitters % world == 0:
        return "emitters"
    return "triangles"


def mixed_partition(rank: int, world: int, groups: int):
    """2-D partition for `world` ranks: `groups` emitter groups x (world / groups) triangle shards.
    Rank r -> (emitter group g = r // T, triangle shard t = r mod T); the T ranks of a group share one
    communicator (their own nccl_uid) and merge their keys; different groups never talk."""
    assert groups >= 1 and world % groups == 0, (world, groups)
    T = world // groups
    return rank // T, rank % T, T


def nccl_uid(group=None) -> bytes:
    """A fresh ncclUniqueId made by the group's first rank (grca_nccl_unique_id) and broadcast over the
    torch.distributed group: pass it to Grca(nccl_uid=..., nranks=group size, rank=group rank)."""
    import torch.distributed as dist

    from .grca import nccl_unique_id

    ranks = dist.get_process_group_ranks(group) if group is not None else list(range(dist.get_world_size()))
    payload = [nccl_unique_id() if dist.get_rank() == ranks[0] else None]
    dist.broadcast_object_list(payload, src=ranks[0], group=group)
    assert isinstance(payload[0], (bytes, bytearray)) and len(payload[0]) == 128
    return bytes(payload[0])
