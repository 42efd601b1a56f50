"""Multi-rank host logic on CPU (gloo, world sizes 2-4): the partitions of paper_2605_10457_b200.dist
and the library's collective steps reproduce the single-rank result exactly.  The per-shard hit
buffers come from the oracle (CPU), packed as (fp32 t bits << 32 | id) exactly like the library's K4
output; the library's in-stream NCCL steps (grca.cu launch_packed: ncclAllReduce / ncclReduceScatter
with ncclMin on uint64, one ncclBroadcast per emitter from rank n mod P) are modelled with the same
gloo collectives on int64 views (the keys are positive as int64, so a signed min is the unsigned
min).  The NCCL calls themselves run on the GPU (tests/test_gpu_parity.py, one-rank communicator)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import scenegen as sg
from paper_2605_10457_b200 import dist as D


# ---- models of the library's collective steps (same operation, gloo instead of NCCL) --------------
def merge_packed(hits, group=None):
    """GRCA_MERGE_ALLREDUCE: in-place all-reduce(MIN) of the packed keys."""
    dist.all_reduce(hits, op=dist.ReduceOp.MIN, group=group)
    return hits


def merge_packed_scatter(hits, group=None):
    """GRCA_MERGE_REDUCE_SCATTER: rank r keeps the min over ranks of rays [r c, r c + c), c = ceil(n / P);
    the keys are padded with MISS to c P (grca.cu K0 initialises the padding)."""
    P, r = dist.get_world_size(group), dist.get_rank(group)
    n = hits.numel()
    c = -(-n // P)
    src = torch.cat([hits, torch.full((c * P - n,), D.MISS_KEY, dtype=hits.dtype)])
    dist.all_reduce(src, op=dist.ReduceOp.MIN, group=group)
    first = r * c
    return src[first: first + max(0, min(c, n - first))].clone(), first


def gather_emitters(keys, offsets, world):
    """gather_outputs under emitter sharding: every emitter's keys broadcast from its owner n mod P."""
    for n in range(len(offsets) - 1):
        a, b = int(offsets[n]), int(offsets[n + 1])
        seg = keys[a:b].clone()
        dist.broadcast(seg, src=n % world)
        keys[a:b] = seg
    return keys


def _packed(res):
    t = res["t"].astype(np.float32).view(np.uint32).astype(np.uint64)
    i = res["id"].astype(np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    return ((t << np.uint64(32)) | i).astype(np.int64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ems, tris = sg.random_scene(77, n_tris=9000, n_emitters=2, gamma=8, chi=64, extent=8.0)
        # triangle sharding: block-interleaved (small block so both ranks own several blocks)
        own = D.shard_triangles(len(tris), rank, world, block=512)
        res = oracle.cast(ems, tris[own], ids=own.astype(np.int32), threads=2)
        hits = torch.as_tensor(_packed(res))
        merge_packed(hits)
        # sensor sharding: each rank casts its emitters (n mod P) with all triangles into the global layout
        # (other emitters' rays stay MISS), then every emitter's keys are broadcast from its owner
        mine = D.shard_emitters(len(ems), rank, world)
        offs = np.cumsum([0] + [e.n_rays for e in ems])
        keys = torch.full((int(offs[-1]),), D.MISS_KEY, dtype=torch.int64)
        for n in mine:
            keys[offs[n]: offs[n + 1]] = torch.as_tensor(_packed(oracle.cast([ems[n]], tris, threads=2)))
        gather_emitters(keys, offs, world)
        k = keys.numpy()
        d_full = (k >> 32).astype(np.uint32).view(np.float32)
        t_full = (k & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
        uid = D.nccl_uid()
        if rank == 0:
            q.put((hits.numpy(), d_full, t_full, uid))
        else:
            q.put(uid)
    finally:
        dist.destroy_process_group()


def test_two_rank_triangle_and_sensor_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    merged, d_full, t_full, uid0 = [x for x in got if isinstance(x, tuple)][0]
    uid1 = [x for x in got if not isinstance(x, tuple)][0]
    assert len(uid0) == 128 and uid0 == uid1      # the communicator id reached both ranks intact
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ems, tris = sg.random_scene(77, n_tris=9000, n_emitters=2, gamma=8, chi=64, extent=8.0)
    ref = oracle.cast(ems, tris, want_t64=True)
    full_key = _packed(ref)
    same = merged == full_key
    # keys may differ only on fp32-equal distances where fp64 order and id order disagree
    tie = (merged >> 32) == (full_key >> 32)
    assert np.all(same | tie)
    assert same.mean() > 0.999
    assert np.array_equal(t_full, ref["id"]) and np.array_equal(d_full.view(np.uint32), ref["t"].view(np.uint32))


def _worker_mixed(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ems, tris = sg.random_scene(78, n_tris=6000, n_emitters=2, gamma=8, chi=64, extent=8.0)
        G = 2
        g, t, T = D.mixed_partition(rank, world, G)
        subs = [dist.new_group(ranks=[gg * T + tt for tt in range(T)]) for gg in range(G)]
        mine_em = D.shard_emitters(len(ems), g, G)
        own = D.shard_triangles(len(tris), t, T, block=512)
        res = oracle.cast([ems[n] for n in mine_em], tris[own], ids=own.astype(np.int32), threads=2)
        hits = torch.as_tensor(_packed(res))
        merge_packed(hits, group=subs[g])   # merge only within this emitter group
        q.put((rank, mine_em, hits.numpy()))
    finally:
        dist.destroy_process_group()


def test_four_rank_mixed_partition():
    """2 emitter groups x 2 triangle shards (D.mixed_partition): each group's in-group min-merge
    equals the unsharded oracle for that group's emitters."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_mixed, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(4)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ems, tris = sg.random_scene(78, n_tris=6000, n_emitters=2, gamma=8, chi=64, extent=8.0)
    for rank, mine_em, hits in got:
        ref = _packed(oracle.cast([ems[n] for n in mine_em], tris, want_t64=True))
        same = hits == ref
        tie = (hits >> 32) == (ref >> 32)   # fp32-equal distances: fp64 order vs id order
        assert np.all(same | tie) and same.mean() > 0.999, rank


def _worker_scatter(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ems, tris = sg.random_scene(79, n_tris=5000, n_emitters=1, gamma=7, chi=61, extent=8.0)   # 427 rays
        own = D.shard_triangles(len(tris), rank, world, block=256)
        res = oracle.cast(ems, tris[own], ids=own.astype(np.int32), threads=2)
        hits = torch.as_tensor(_packed(res))
        sl, first = merge_packed_scatter(hits)
        q.put((rank, first, sl.numpy()))
    finally:
        dist.destroy_process_group()


def test_three_rank_reduce_scatter_merge():
    """Ray-sharded merge (reduce-scatter(MIN)) with a ray count not divisible by the
    ranks: the slices tile [0, n_rays) in rank order and equal the unsharded oracle's keys."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_scatter, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(3)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ems, tris = sg.random_scene(79, n_tris=5000, n_emitters=1, gamma=7, chi=61, extent=8.0)
    ref = _packed(oracle.cast(ems, tris, want_t64=True))
    assert [f for _, f, _ in got] == [0, 143, 286] and sum(len(s) for _, _, s in got) == len(ref) == 427
    merged = np.concatenate([s for _, _, s in got])
    same = merged == ref
    assert np.all(same | ((merged >> 32) == (ref >> 32))) and same.mean() > 0.999


def test_partition_helpers():
    n, world = 100_000, 4
    parts = [D.shard_triangles(n, r, world) for r in range(world)]
    allidx = np.sort(np.concatenate(parts))
    assert np.array_equal(allidx, np.arange(n))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= D.BLOCK
    assert D.shard_emitters(8, 1, 4) == [1, 5]
    assert D.choose_mode(8, 8) == "emitters" and D.choose_mode(2, 8) == "triangles" and D.choose_mode(8, 1) == "triangles"
    assert D.MISS_KEY == 0x7F800000FFFFFFFF and D.MISS_KEY < 2**63   # positive as int64: signed min works
    assert [D.mixed_partition(r, 8, 2) for r in (0, 3, 4, 7)] == [(0, 0, 4), (0, 3, 4), (1, 0, 4), (1, 3, 4)]
