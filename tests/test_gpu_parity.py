"""Parity of the CUDA path (through the C ABI) with the brute-force oracle (-m gpu).

Contract (BASELINE.json north star; oracle/compare.py): >= 99.999 % of rays agree, every
disagreement lies within 1e-6 barycentric of a triangle edge, |t_G - t_O| <= 1e-5 t_O, ids
equal except at near-ties.  Scenes are seeded synthetic (scenegen); sizes span several K2
tiles (256 triangles) with ragged tails; full-size configs are checked on sampled rays.
"""
import math

import numpy as np
import pytest

import oracle
import scenegen as sg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU hosts collect but skip
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_10457_b200 import Grca, GrcaError, tris_to_float4  # noqa: E402
from paper_2605_10457_b200 import grca as G  # noqa: E402


def run(ems, tris, ids=None, faces=0, flags=0, small_max=0, max_large=0, indexed=False, handle=None):
    n_rays = sg.n_rays_total(ems)
    g = handle or Grca(device=0, max_triangles=max(1, len(tris)), max_rays=n_rays, faces=faces, debug_flags=flags,
                       small_max=small_max, max_large_items=max_large)
    g.set_emitters(ems)
    tid = None if ids is None else torch.as_tensor(np.asarray(ids, np.int32), device="cuda")
    if indexed and len(tris):
        flat = np.asarray(tris, np.float32).reshape(-1, 3)
        uniq, inv = np.unique(flat, axis=0, return_inverse=True)
        v4 = tris_to_float4(uniq)
        idx = torch.as_tensor(inv.astype(np.int32).reshape(-1), device="cuda")
        g.update_triangles(v4, indices=idx, tri_ids=tid)
    else:
        v4 = tris_to_float4(tris) if len(tris) else torch.zeros((4, 4), device="cuda")
        g.update_triangles(v4, tri_ids=tid, n_triangles=len(tris))
    dist, tri, st = g.cast(stats=True)
    torch.cuda.synchronize()
    return dist.cpu().numpy(), tri.cpu().numpy(), st, g


def check(ems, tris, dist, tri, ids=None, faces=0, rays=None, ref=None):
    if ref is None:
        ref = oracle.cast(ems, tris, ids=ids, faces=faces, rays=rays, want_t64=True)
    sel = ref["rays"]
    rep = oracle.compare(ems, tris, dist[sel], tri[sel], ref, ids=ids, faces=faces)
    assert rep["passed"], {k: rep[k] for k in ("rays", "agree_frac", "unexcused", "kinds", "details")}
    return rep, ref


# ------------------------------------------------------------- ray table ----

def test_ray_table_bit_identical_to_oracle():
    """O1: the library's host-fp64 ray table equals the oracle's bit for bit."""
    rng = np.random.default_rng(0)
    ems = [sg.c1_emitter()]
    for k in range(4):
        f, r, u = sg.random_frame(rng)
        ems.append(sg.Emitter(origin=rng.normal(size=3) * 50, forward=f, right=r, up=u,
                              elev=sg.full_sphere_elev(64) if k % 2 else sg.vlp16_elev(),
                              rays_per_channel=1000 + 37 * k, hfov_deg=360 if k % 2 else 180))
    g = Grca(device=0, max_triangles=1, max_rays=sg.n_rays_total(ems))
    g.set_emitters(ems)
    mine = g.debug_ray_table()
    ref = oracle.ray_table(ems)
    assert mine.shape == ref.shape
    assert np.array_equal(mine.view(np.uint32), ref.view(np.uint32))


# ------------------------------------------------------------------ C1 ------

@pytest.mark.parametrize("max_range", [math.inf, 10.0])
def test_c1_full_frame(max_range):
    """BASELINE config 1: 1 LiDAR 16x512, 2,000-triangle static scene, every ray."""
    ems = [sg.c1_emitter(max_range=max_range)]
    tris = sg.c1_scene()
    dist, tri, st, _ = run(ems, tris)
    rep, ref = check(ems, tris, dist, tri)
    assert rep["oracle_hits"] > 1000
    assert st["rtic_tested"] < st["rtic_brute"]
    assert st["pairs"] == len(tris)


@pytest.mark.parametrize("fixture", ["quad", "seam", "ground", "room", "zenith"])
def test_fixtures_alone(fixture):
    """SURVEY 8c fixtures as unit scenes (quad at known distance, seam straddler, nadir, box)."""
    em = sg.c1_emitter()
    o = em.origin.astype(np.float64)
    tris = {
        "quad": sg.quad_x5(o), "seam": sg.seam_triangle(o), "ground": sg.ground_quad(1.5, 50.0, o),
        "room": sg.room_box(o + [-2, -3, -1], o + [4, 2, 2.5]),
        "zenith": np.array([[[-1.0, -1.0, 4.0], [2.0, -1.0, 4.0], [0.0, 2.0, 4.0]]], np.float32),
    }[fixture]
    dist, tri, _, _ = run([em], tris)
    rep, ref = check([em], tris, dist, tri)
    assert rep["oracle_hits"] > 0
    if fixture == "quad":
        g = 8 * 512 + 256
        assert dist[g] == 5.0 and tri[g] == 0
    if fixture == "seam":
        assert tri[8 * 512] == 0 and tri[8 * 512 + 511] == 0
    if fixture == "ground":
        assert np.all(dist[:512] == np.float32(1.5))   # nadir channel: all 512 rays at t = h
    if fixture == "room":
        assert np.all(tri >= 0)


def test_watertight_shared_diagonal():
    """Rays aimed at the shared diagonal of a quad: every one hits at least one triangle."""
    em = sg.Emitter(origin=(0, 0, 0), elev=np.linspace(-0.19, 0.19, 401).astype(np.float32),
                    rays_per_channel=4096)
    tris = sg.quad_x5()
    dist, tri, _, _ = run([em], tris)
    check([em], tris, dist, tri)
    D = oracle.ray_table([em]).astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        y = 5 * D[:, 1] / D[:, 0]
        z = 5 * D[:, 2] / D[:, 0]
    near_diag = (D[:, 0] > 0) & (np.abs(y - z) < 1e-3) & (np.abs(y) < 0.99) & (np.abs(z) < 0.99)
    assert near_diag.sum() > 50
    assert np.all(tri[near_diag] >= 0)


# ------------------------------------------------------- random sweeps ------

@pytest.mark.parametrize("seed", list(range(20)))
def test_random_scenes(seed):
    """20 seeded scenes: random frames, 360/180 deg, non-uniform tables, range limits, ragged sizes."""
    n_em = 1 + seed % 3
    ems, tris = sg.random_scene(seed, n_tris=257 + 97 * seed, n_emitters=n_em, gamma=8 + seed % 9,
                                chi=64 + 13 * seed, extent=6.0 + seed,
                                max_range=None if seed % 4 else 5.0 + seed)
    dist, tri, st, _ = run(ems, tris)
    rep, _ = check(ems, tris, dist, tri)
    assert st["rtic_tested"] <= st["rtic_brute"]


def _check_all_hits(ems, tris, counts, ref, rays=None, bound=1e-4):
    """All-hits invariant (north star: culling never drops a brute-force hit).  Per-ray counts of every
    accepted hit equal the oracle's, except on rays where a triangle lies within 1e-6 barycentric of its
    boundary (the excusal of the parity contract): there the counts may differ by at most the number of
    such triangles (oracle.near_edge_count).  Returns the number of excused rays, bounded by 1e-4 of the
    rays checked (the certified test disagrees with exact arithmetic only at ~1e-16 relative)."""
    got = counts if rays is None else counts[rays]
    exp = ref["allhits"]
    diff = np.nonzero(got != exp)[0]
    assert len(diff) <= max(2, int(bound * len(exp))), (len(diff), len(exp))
    bad = []
    for r in diff:
        g = int(ref["rays"][r])
        if abs(int(got[r]) - int(exp[r])) > oracle.near_edge_count(ems, g, tris):
            bad.append((g, int(got[r]), int(exp[r])))
    assert not bad, bad[:10]
    return len(diff)


def test_all_hits_invariant():
    """Culling never drops a brute-force hit: per-ray all-hit counts equal the oracle's, except on
    rays within 1e-6 barycentric of an edge of a triangle they (nearly) hit."""
    for seed in (1, 2, 3):
        ems, tris = sg.random_scene(100 + seed, n_tris=800, n_emitters=2, gamma=16, chi=200, extent=8.0)
        dist, tri, st, g = run(ems, tris, flags=G.DEBUG_COUNT_ALL_HITS)
        counts = g.debug_all_hits().cpu().numpy()
        ref = oracle.cast(ems, tris, want_t64=True, want_allhits=True)
        check(ems, tris, dist, tri, ref=ref)
        _check_all_hits(ems, tris, counts, ref)
    ems = [sg.c1_emitter()]
    tris = sg.c1_scene()
    dist, tri, st, g = run(ems, tris, flags=G.DEBUG_COUNT_ALL_HITS)
    ref = oracle.cast(ems, tris, want_allhits=True)
    # C1's ground grid has lines x = 0 and y = 0 right under the emitter: the 14 rays at azimuths 0, 90,
    # 180, 270 deg of channels 1-5 run exactly along shared ground edges (bound 2e-3 instead of 1e-4)
    excused = _check_all_hits(ems, tris, g.debug_all_hits().cpu().numpy(), ref, bound=2e-3)
    print(f"C1 all-hits: {len(ref['allhits'])} rays, {int(ref['allhits'].sum())} hits, {excused} excused rays")


def test_no_cull_bit_identical_and_fp64_mode():
    """Invariant (5): culling off (full ray grid per pair) gives the bit-identical packed result;
    the all-fp64 mode gives the same hits and ids with t within the certified 4.5e-6."""
    ems, tris = sg.random_scene(7, n_tris=600, n_emitters=2, gamma=12, chi=128)
    base = run(ems, tris)
    nocull = run(ems, tris, flags=G.DEBUG_NO_CULL)
    assert np.array_equal(base[1], nocull[1])
    assert np.array_equal(base[0].view(np.uint32), nocull[0].view(np.uint32))
    assert nocull[2]["rtic_tested"] == nocull[2]["rtic_brute"]
    f64 = run(ems, tris, flags=G.DEBUG_FORCE_FP64)
    assert np.array_equal(base[1], f64[1])
    hit = base[1] >= 0
    rel = np.abs(base[0][hit].astype(np.float64) / f64[0][hit].astype(np.float64) - 1)
    assert rel.max() <= 4.6e-6
    assert f64[2]["fp64_fallbacks"] == f64[2]["rtic_tested"]
    check(ems, tris, base[0], base[1])


@pytest.mark.parametrize("small_max,max_large", [(1, 0), (100000, 0), (0, 3), (1, 2)])
def test_binning_and_capacity_paths(small_max, max_large):
    """All-large, all-inline and capacity-overflow fallbacks give identical results."""
    ems, tris = sg.random_scene(11, n_tris=700, n_emitters=2, gamma=16, chi=300, extent=5.0)
    base = run(ems, tris)
    alt = run(ems, tris, small_max=small_max, max_large=max_large)
    assert np.array_equal(base[1], alt[1]) and np.array_equal(base[0].view(np.uint32), alt[0].view(np.uint32))
    if max_large:
        assert alt[2]["overflow"] == 1


def test_capacity_fallback_across_casts():
    """Capacity overflow must never replay stale work: one handle with a 3-entry large list (12 chunk
    slots) casts scene A, then a different scene B and emitter set, then A again; every result equals
    a fresh handle's (K3 writes every reserved chunk slot below the capacity and intersects the rest)."""
    ems_a, tris_a = sg.random_scene(11, n_tris=700, n_emitters=2, gamma=16, chi=300, extent=5.0)
    ems_b, tris_b = sg.random_scene(12, n_tris=900, n_emitters=1, gamma=24, chi=256, extent=4.0)
    n_rays = max(sg.n_rays_total(ems_a), sg.n_rays_total(ems_b))
    g = Grca(device=0, max_triangles=1000, max_rays=n_rays, small_max=1, max_large_items=3)
    for ems, tris in ((ems_a, tris_a), (ems_b, tris_b), (ems_a, tris_a)):
        fresh = run(ems, tris)
        got = run(ems, tris, handle=g)
        assert got[2]["overflow"] == 1
        assert np.array_equal(fresh[1], got[1]) and np.array_equal(fresh[0].view(np.uint32), got[0].view(np.uint32))
    g.close()


def test_nvls_binding_blocks_ray_count_change():
    """A bound NVLS buffer was sized for the current rays: set_emitters with another ray count is a
    state error until the binding is dropped (no cast runs here: the views are plain device memory)."""
    ems, tris = sg.random_scene(13, n_tris=100, n_emitters=1, gamma=8, chi=64)
    g = Grca(device=0, max_triangles=100, max_rays=4096)
    g.set_emitters(ems)
    need = g.nvls_status()["bytes_needed"]
    buf = torch.zeros(need // 8 + 32, dtype=torch.int64, device="cuda")
    ptr = (buf.data_ptr() + 127) // 128 * 128
    g.set_nvls(ptr, ptr, 1)
    g.set_emitters(ems)                                   # same ray count: fine
    bigger = [sg.Emitter(origin=(0, 0, 0), elev=sg.full_sphere_elev(8), rays_per_channel=128)]
    with pytest.raises(GrcaError) as ei:
        g.set_emitters(bigger)
    assert ei.value.status == 2
    g.set_nvls(None, None, 0)
    g.set_emitters(bigger)
    g.close()


@pytest.mark.parametrize("faces", [1, 2])
def test_face_modes(faces):
    ems, tris = sg.random_scene(21, n_tris=500, n_emitters=2)
    dist, tri, _, _ = run(ems, tris, faces=faces)
    check(ems, tris, dist, tri, faces=faces)


def test_indexed_ids_and_determinism():
    """Indexed meshes == triangle soup; custom ids travel; two casts are bit-identical."""
    tris = np.concatenate([sg.car(40, 40, dims=(4.0, 2.0, 1.2)) + np.float32([6, 1, 0]),
                           sg.grid_mesh(20, 20, -10, -10, 10, 10, -1.5)], 0)
    ems = [sg.Emitter(origin=(0, 0, 0), elev=sg.full_sphere_elev(32), rays_per_channel=720)]
    ids = (np.arange(len(tris), dtype=np.int32) * 3 + 5)
    a = run(ems, tris, ids=ids)
    b = run(ems, tris, ids=ids, indexed=True)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
    check(ems, tris, a[0], a[1], ids=ids)
    g = a[3]
    d2, t2 = g.cast()
    assert np.array_equal(d2.cpu().numpy().view(np.uint32), a[0].view(np.uint32))


def test_virtual_shards_min_merge():
    """1-shard == min over P block-interleaved shards of the packed hit buffers (bit-exact)."""
    ems, tris = sg.random_scene(31, n_tris=3000, n_emitters=2, gamma=16, chi=256, extent=10.0)
    n = len(tris)
    g = Grca(device=0, max_triangles=n, max_rays=sg.n_rays_total(ems))
    g.set_emitters(ems)
    v4 = tris_to_float4(tris)
    g.update_triangles(v4)
    g.cast_packed()
    full = g.hits_packed().clone()
    for P in (2, 3, 4):
        blk = 256
        owner = (np.arange(n) // blk) % P
        merged = None
        for r in range(P):
            idx = np.nonzero(owner == r)[0]
            g.update_triangles(tris_to_float4(tris[idx]), tri_ids=torch.as_tensor(idx.astype(np.int32), device="cuda"))
            g.cast_packed()
            h = g.hits_packed().clone()
            merged = h if merged is None else torch.minimum(merged, h)
        assert torch.equal(merged, full)
    dist = torch.empty(g.n_rays, device="cuda")
    tri = torch.empty(g.n_rays, dtype=torch.int32, device="cuda")
    g.update_triangles(v4)
    g.cast_packed()
    g.unpack(dist, tri)
    check(ems, tris, dist.cpu().numpy(), tri.cpu().numpy())


def test_edge_cases():
    """Empty scene, degenerate / NaN / origin-coplanar triangles, origin on a vertex."""
    em = sg.c1_emitter()
    o = em.origin
    dist, tri, _, _ = run([em], np.zeros((0, 3, 3), np.float32))
    assert np.all(tri == -1) and np.all(np.isinf(dist))
    bad = np.array([
        [[5, 0, 0], [5, 0, 0], [5, 1, 1]],                                   # zero-area
        [[np.nan, 0, 0], [5, 1, 0], [5, 0, 1]],                              # NaN
        [o, o + [1, 0, 0], o + [0, 1, 0]],                                   # origin is a vertex
        [o + [1, -1, 0], o + [2, 1, 0], o + [3, -1, 0]],                     # plane through origin
        [o + [4, -1, -1], o + [4, 1, -1], o + [4, 0, 1]],                    # a normal one
    ], dtype=np.float32)
    dist, tri, _, _ = run([em], bad)
    check([em], bad, dist, tri)
    assert set(np.unique(tri)) <= {-1, 4}


@pytest.mark.parametrize("shape", ["1x1", "chi_max", "gamma_max", "tile_edges"])
def test_extreme_emitter_shapes_and_counts(shape):
    """Boundary sizes of the ABI (include/grca.h: gamma, chi in [1, 65535], sum (gamma + 2) <= 4096) and triangle
    counts on both sides of a K2 tile (1024): every ray against the oracle."""
    rng = np.random.default_rng(7)
    tris = sg.random_triangles(rng, 300, center=(0, 0, 0), half_extent=8.0, edge_lo=0.05, edge_hi=6.0)
    if shape == "1x1":   # one channel, one ray (theta = 0): a triangle straight ahead and one behind
        ems = [sg.Emitter(origin=(0, 0, 0), elev=np.float32([0.0]), rays_per_channel=1)]
        tris = np.array([[[4, -1, -1], [4, 1, -1], [4, 0, 1]], [[-4, -1, -1], [-4, 1, -1], [-4, 0, 1]]],
                        np.float32)
    elif shape == "chi_max":   # 65,535 rays in one channel (16-bit ray ranges), 360 and 180 deg
        ems = [sg.Emitter(origin=(0.1, -0.2, 0.0), elev=np.float32([0.05]), rays_per_channel=65535),
               sg.Emitter(origin=(0.3, 0.2, 0.1), elev=np.float32([-0.1]), rays_per_channel=65535, hfov_deg=180)]
    elif shape == "gamma_max":   # the channel limit, sum (gamma + 2) = 4096, over two emitters (no channel LUT)
        ems = [sg.Emitter(origin=(0, 0, 0), elev=sg.full_sphere_elev(4000), rays_per_channel=3),
               sg.Emitter(origin=(0.5, 0.5, 0.5), elev=sg.full_sphere_elev(92), rays_per_channel=5, hfov_deg=180)]
    else:
        ems = [sg.Emitter(origin=(0, 0, 0), elev=sg.full_sphere_elev(16), rays_per_channel=97)]
    counts = [len(tris)] if shape != "tile_edges" else [1, 1023, 1024, 1025, 2049]
    for n in counts:
        t = tris if shape != "tile_edges" else sg.random_triangles(rng, n, center=(0, 0, 0), half_extent=8.0,
                                                                   edge_lo=0.05, edge_hi=6.0)
        dist, tri, st, _ = run(ems, t)
        rep, _ = check(ems, t, dist, tri)
        assert st["pairs"] == len(t) * len(ems)
    if shape == "1x1":
        assert tri[0] == 0 and dist[0] == np.float32(4.0)
    if shape == "chi_max":
        assert rep["oracle_hits"] > 1000
    if shape == "gamma_max":   # one channel more is refused
        g = Grca(device=0, max_triangles=1, max_rays=20000)
        with pytest.raises(GrcaError) as e:
            g.set_emitters([ems[0], sg.Emitter(origin=(0.5, 0.5, 0.5), elev=sg.full_sphere_elev(93), rays_per_channel=5)])
        assert e.value.status == G.GRCA_E_INVALID


def test_api_errors():
    g = Grca(device=0, max_triangles=10, max_rays=1000)
    with pytest.raises(GrcaError) as e:
        g.cast()
    assert e.value.status == G.GRCA_E_STATE
    with pytest.raises(GrcaError) as e:
        g.set_emitters([sg.Emitter(origin=(0, 0, 0), elev=np.float32([0.1, 0.0]), rays_per_channel=10)])
    assert e.value.status == G.GRCA_E_INVALID
    with pytest.raises(GrcaError) as e:
        g.set_emitters([sg.Emitter(origin=(0, 0, 0), elev=sg.full_sphere_elev(16), rays_per_channel=512)])
    assert e.value.status == G.GRCA_E_CAPACITY
    with pytest.raises(GrcaError):
        g.set_emitters([sg.Emitter(origin=(0, 0, 0), forward=(1, 0, 0), right=(1, 0, 0), elev=np.float32([0]),
                                   rays_per_channel=8)])
    g.set_emitters([sg.Emitter(origin=(0, 0, 0), elev=np.float32([0.0]), rays_per_channel=8)])
    with pytest.raises(GrcaError) as e:
        g.update_triangles(tris_to_float4(np.zeros((11, 3, 3), np.float32)))
    assert e.value.status == G.GRCA_E_CAPACITY


# --------------------------------------------------- larger, sampled rays ----

def _sampled(ems, n_per_emitter, seed):
    rng = np.random.default_rng(seed)
    out, base = [], 0
    for e in ems:
        out.append(base + rng.choice(e.n_rays, size=min(n_per_emitter, e.n_rays), replace=False))
        base += e.n_rays
    return np.sort(np.concatenate(out)).astype(np.int64)


def test_c2_like_sampled():
    """C2-shaped (2 LiDARs 128x4096, plant + car, f.i), reduced triangle count, 4,096 sampled rays."""
    w = sg.workload("C2", frame=0, static_scale=0.25)
    tris = w["tris"]
    dist, tri, st, _ = run(w["emitters"], tris)
    rays = _sampled(w["emitters"], 2048, 5)
    rep, _ = check(w["emitters"], tris, dist, tri, rays=rays)
    assert rep["oracle_hits"] > 100
    assert st["rtic_tested"] < 1e-3 * st["rtic_brute"]


@pytest.mark.parametrize("rng_m", [10.0, 50.0])
def test_c3_like_ranged_sampled(rng_m):
    """C3-shaped: 4 LiDARs mixed 360/180 deg with range culling; reduced scene; sampled rays."""
    w = sg.workload("C3", frame=1, static_scale=0.05, max_range=rng_m)
    dist, tri, st, _ = run(w["emitters"], w["tris"])
    rays = _sampled(w["emitters"], 1024, 6)
    check(w["emitters"], w["tris"], dist, tri, rays=rays)
    assert st["range_culled"] > 0


def _scale_parity(w, n_per_emitter, seed, label):
    """Full-size frame in the launch configuration bench.py times (grca_update_scene: static float4 soup
    + indexed float3 cars, an uninstrumented handle) == the triangle-soup cast bit for bit; then, on
    n_per_emitter sampled rays per emitter, closest-hit parity (north-star comparator) and the all-hits
    invariant against ONE oracle pass over all triangles."""
    ems, tris = w["emitters"], w["tris"]
    n_rays = sg.n_rays_total(ems)
    dist, tri, st, ga = run(ems, tris, flags=G.DEBUG_COUNT_ALL_HITS)
    if w.get("car_mesh") is not None:   # (subdivided cars have no shared-vertex mesh: soup only)
        g = Grca(device=0, max_triangles=len(tris), max_rays=n_rays)
        g.set_emitters(ems)
        di, ti = run_indexed_frame(w, g)
        g.close()
        assert np.array_equal(ti, tri) and np.array_equal(di.view(np.uint32), dist.view(np.uint32))
    else:
        di, ti = dist, tri
    counts = ga.debug_all_hits().cpu().numpy()
    rays = _sampled(ems, n_per_emitter, seed)
    ref = oracle.cast(ems, tris, rays=rays, want_t64=True, want_allhits=True)
    rep, _ = check(ems, tris, di, ti, rays=rays, ref=ref)
    excused = _check_all_hits(ems, tris, counts, ref, rays=rays)
    print(f"{label}: {rep['rays']} rays, agree {rep['agree_frac']:.6f}, excused {rep['excused']}, near-ties "
          f"{rep['near_ties']}, Hit% 1 mm {rep['hit_pct_1mm']:.4f}, oracle hits {rep['oracle_hits']}, "
          f"all-hit counts {int(ref['allhits'].sum())} (excused rays {excused})")
    assert rep["oracle_hits"] > n_per_emitter * len(ems) // 4
    ga.close()
    return st, rep


def test_c2_full_size_all_hits():
    """C2 at full size (2 x 128x4096 rays, ~1M triangles): parity + all-hits on 2,048 rays per emitter."""
    st, rep = _scale_parity(sg.workload("C2", frame=1), 2048, 21, "C2 frame 1")
    assert st["pairs"] == st["pairs"] and rep["agree_frac"] >= 0.99999


@pytest.mark.slow
def test_c4_full_size_sampled():
    """C4 at full size (8 x 128x4096 rays, ~21.8M triangles), frame 0: 1,024 sampled rays per emitter
    (8,192 rays x all triangles in the oracle), parity + all-hits invariant."""
    w = sg.workload("C4", frame=0)
    st, _ = _scale_parity(w, 1024, 9, "C4 frame 0")
    assert st["pairs"] == len(w["tris"]) * 8


@pytest.mark.slow
@pytest.mark.parametrize("rng_m", [10.0, 50.0])
def test_c3_full_size_ranged(rng_m):
    """C3 at full size (4 LiDARs 128x4096, two 360 deg and two 180 deg, ~5M triangles) with range culling at
    10 / 50 m: 1,024 sampled rays per emitter, parity + all-hits invariant (hits beyond D_max must not appear,
    hits within it must all be found)."""
    st, _ = _scale_parity(sg.workload("C3", frame=1, max_range=rng_m), 1024, 31, f"C3 range {rng_m:g} m")
    assert st["range_culled"] > 0


@pytest.mark.slow
def test_c5_full_size_subdivided():
    """C5 at full size, car subdivided twice (4.8M dynamic triangles of ~1/16 the area, ~5.5M in all):
    1,024 sampled rays per emitter, parity + all-hits invariant (culling stays exact as triangles shrink)."""
    _scale_parity(sg.workload("C5", frame=0, subdiv=2), 1024, 41, "C5 subdiv 2")


@pytest.mark.slow
def test_c4_full_size_large_rectangle_frame():
    """C4 frame 2 (huge scaled cars send many large rectangles through K3/K4 and A7), full size:
    1,024 sampled rays per emitter, parity + all-hits invariant."""
    st, _ = _scale_parity(sg.workload("C4", frame=2), 1024, 19, "C4 frame 2")
    assert st["large_pairs"] > 1000 and st["chunks"] > 10000


def test_c2_hybrid_indexed_dynamic():
    """The bench's hybrid line: static triangles (float4 soup) cached, the cars' posed vertices
    (indexed float3) cast each frame -- bit-identical to the full indexed cast."""
    w = sg.workload("C2", frame=2)
    v, idx = sg.indexed_frame(w)
    ns3 = 3 * w["n_static"]
    g = Grca(device=0, max_triangles=len(w["tris"]), max_rays=sg.n_rays_total(w["emitters"]))
    g.set_emitters(w["emitters"])
    g.update_triangles(torch.as_tensor(v, device="cuda"), indices=torch.as_tensor(idx, device="cuda"))
    d_f, t_f = g.cast()
    gh = Grca(device=0, max_triangles=len(w["tris"]), max_rays=sg.n_rays_total(w["emitters"]))
    gh.set_emitters(w["emitters"])
    gh.set_static_triangles(tris_to_float4(v[:ns3]), tri_id_base=0)
    dyn_idx = torch.as_tensor(idx[ns3:] - ns3, device="cuda")
    gh.update_triangles(torch.as_tensor(v[ns3:], device="cuda"), indices=dyn_idx, tri_id_base=w["n_static"])
    d_h, t_h = gh.cast()
    torch.cuda.synchronize()
    assert np.array_equal(t_h.cpu().numpy(), t_f.cpu().numpy())
    assert np.array_equal(d_h.cpu().numpy().view(np.uint32), d_f.cpu().numpy().view(np.uint32))


def test_c2_tilted_frames():
    """C2 at full size with every emitter's frame rolled 25 deg and pitched 10 deg (not level: the
    general K2 pre-test and sensor transform), indexed float3 layout; sampled parity."""
    w = sg.workload("C2", frame=1)
    ca, sa, cb, sb = math.cos(0.436), math.sin(0.436), math.cos(0.175), math.sin(0.175)
    roll = np.array([[1, 0, 0], [0, ca, -sa], [0, sa, ca]])
    pitch = np.array([[cb, 0, sb], [0, 1, 0], [-sb, 0, cb]])
    R = pitch @ roll
    ems = []
    for e in w["emitters"]:
        f, r, u = (R @ np.asarray(x, np.float64) for x in (e.forward, e.right, e.up))
        ems.append(sg.Emitter(origin=e.origin, forward=f, right=r, up=u, elev=e.elev,
                              rays_per_channel=e.rays_per_channel, hfov_deg=e.hfov_deg, max_range=e.max_range))
    w = dict(w, emitters=ems)
    dist, tri, st, g = run(ems, w["tris"])
    di, ti = run_indexed_frame(w, g)
    assert np.array_equal(ti, tri) and np.array_equal(di.view(np.uint32), dist.view(np.uint32))
    rep, _ = check(ems, w["tris"], di, ti, rays=_sampled(ems, 1024, 23))
    assert rep["oracle_hits"] > 100


def run_indexed_frame(w, g, layout="scene"):
    """layout "scene" (bench.py's default): grca_update_scene with the static triangles as a float4
    soup and the cars as indexed packed float3; "f3": everything indexed packed float3."""
    v, idx = sg.indexed_frame(w)
    if layout == "scene":
        ns3 = 3 * w["n_static"]
        g.update_scene(soup=tris_to_float4(w["tris"][: w["n_static"]]), mesh_xyz=torch.as_tensor(v[ns3:], device="cuda"),
                       mesh_indices=torch.as_tensor(idx[ns3:] - ns3, device="cuda"))
    else:
        g.update_triangles(torch.as_tensor(v, device="cuda"), indices=torch.as_tensor(idx, device="cuda"))
    d, t = g.cast()
    torch.cuda.synchronize()
    return d.cpu().numpy(), t.cpu().numpy()


def test_c2_indexed_layout():
    """C2 at full size in bench.py's indexed layout: bit-identical to the soup, parity on sampled rays."""
    w = sg.workload("C2", frame=3)
    dist, tri, st, g = run(w["emitters"], w["tris"])
    for layout in ("scene", "f3"):
        di, ti = run_indexed_frame(w, g, layout)
        assert np.array_equal(ti, tri) and np.array_equal(di.view(np.uint32), dist.view(np.uint32))
    check(w["emitters"], w["tris"], di, ti, rays=_sampled(w["emitters"], 1024, 11))


def _near_axis_scene(seed, n=1500):
    """Triangles within 5 deg of a level emitter's spin axis, above and below: random far / near,
    tiny / large, 10 % centred on the axis (pole inside), 5 % with a vertex exactly on it."""
    rng = np.random.default_rng(seed)
    o = np.array([0.3, -0.2, 1.0])
    out, off_axis = [], []
    for i in range(n):
        sgn = 1.0 if rng.random() < 0.5 else -1.0
        R = float(np.exp(rng.uniform(np.log(3.0), np.log(300.0))))
        alpha = 0.0 if i % 10 == 0 else rng.uniform(0.0, np.radians(5.0))
        beta = rng.uniform(0.0, 2 * np.pi)
        c = o + R * np.array([np.sin(alpha) * np.cos(beta), np.sin(alpha) * np.sin(beta), sgn * np.cos(alpha)])
        size = R * float(np.exp(rng.uniform(np.log(1e-4), np.log(0.05))))
        u = rng.normal(size=(3, 3))
        T = c + size * u / np.linalg.norm(u, axis=1, keepdims=True)
        if i % 20 == 1:
            T[0] = o + np.array([0.0, 0.0, sgn * R])
        T = T.astype(np.float32)
        out.append(T)
        rel = T.astype(np.float64) - o
        ang = np.arctan2(np.hypot(rel[:, 0], rel[:, 1]), np.abs(rel[:, 2]))
        # off the axis: every vertex > 0.5 deg from it and an azimuth span < 3 rad (so the axis is
        # outside T and the arc is not near pi, where a full row is the designed answer)
        th = np.sort(np.arctan2(rel[:, 1], rel[:, 0]))
        gaps = np.diff(np.concatenate([th, th[:1] + 2 * np.pi]))
        off_axis.append(bool(ang.min() > np.radians(0.5)) and 2 * np.pi - gaps.max() < 3.0)
    return o, np.stack(out), np.array(off_axis)


@pytest.mark.parametrize("yaw_deg,tilt_deg", [(0.0, 0.0), (37.0, 0.0), (20.0, 0.5)])
def test_near_axis_level_frames(yaw_deg, tilt_deg):
    """Near the spin axis (zenith / nadir of a full-sphere LiDAR, 64 x 1024 rays): full brute-force
    parity.  Level frames: triangles off the axis get partial-azimuth rectangles (the general-frame
    near-axis guard would take all 1024 rays of every row).  A frame tilted by 0.5 deg is not level:
    the guard applies (parity only)."""
    o, tris, off_axis = _near_axis_scene(7 + int(yaw_deg))
    a, b = np.radians(yaw_deg), np.radians(tilt_deg)
    f = np.array([np.cos(a), np.sin(a), 0.0])
    r = np.array([np.sin(a), -np.cos(a), 0.0])
    u = np.array([0.0, 0.0, 1.0])
    if tilt_deg:   # roll about the forward axis
        r, u = np.cos(b) * r + np.sin(b) * u, -np.sin(b) * r + np.cos(b) * u
    em = sg.Emitter(origin=o, forward=f, right=r, up=u, elev=sg.full_sphere_elev(64), rays_per_channel=1024)
    dist, tri, st, g = run([em], tris, small_max=64)
    check([em], tris, dist, tri)
    L = g.debug_large_list()
    full = ((L[:, 3] >> 16) & 0xFFFF) >= 1024
    assert len(L) > 20
    if not tilt_deg:
        assert not off_axis[L[full, 0]].any(), "off-axis triangle with a full-azimuth rectangle"
        assert (~full).sum() > 0


def test_update_scene_parts_and_errors():
    """grca_update_scene: any split point of a soup into [float4 part | indexed float3 part] gives
    the soup's bit-identical result (ids = global triangle index, or the explicit id array);
    empty parts; argument errors."""
    ems, tris = sg.random_scene(91, n_tris=3000, n_emitters=3, gamma=16, chi=240, extent=8.0)
    d0, t0, st0, g = run(ems, tris)
    check(ems, tris, d0, t0)
    n = len(tris)
    rng = np.random.default_rng(5)
    for na in (0, 1, 777, n - 1, n):
        # the mesh part as a vertex-deduplicated indexed float3 mesh with shuffled vertex order
        mv = tris[na:].reshape(-1, 3)
        perm = rng.permutation(len(mv))
        xyz = np.ascontiguousarray(mv[perm])
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm))
        g.update_scene(soup=tris_to_float4(tris[:na]) if na else None,
                       mesh_xyz=torch.as_tensor(xyz, device="cuda") if na < n else None,
                       mesh_indices=torch.as_tensor(inv.astype(np.int32), device="cuda") if na < n else None)
        d, t = g.cast()
        assert np.array_equal(t.cpu().numpy(), t0) and np.array_equal(d.cpu().numpy().view(np.uint32), d0.view(np.uint32))
    # explicit ids index the concatenation
    ids = rng.permutation(n).astype(np.int32)
    g.update_scene(soup=tris_to_float4(tris[:1000]), mesh_xyz=torch.as_tensor(tris[1000:].reshape(-1, 3), device="cuda"),
                   mesh_indices=torch.arange(3 * (n - 1000), dtype=torch.int32, device="cuda"),
                   tri_ids=torch.as_tensor(ids, device="cuda"))
    d, t = g.cast()
    t = t.cpu().numpy()
    hit = t0 >= 0
    assert np.array_equal(t[hit], ids[t0[hit]]) and np.array_equal(t[~hit], t0[~hit])
    # hybrid: the first 1200 triangles as the cached static set, the rest through grca_update_scene
    # (a soup part and an indexed part, ids continuing the static ones) == the plain soup cast
    gh = Grca(device=0, max_triangles=n, max_rays=sg.n_rays_total(ems))
    gh.set_emitters(ems)
    gh.set_static_triangles(tris_to_float4(tris[:1200]), tri_id_base=0)
    gh.update_scene(soup=tris_to_float4(tris[1200:2000]),
                    mesh_xyz=torch.as_tensor(tris[2000:].reshape(-1, 3), device="cuda"),
                    mesh_indices=torch.arange(3 * (n - 2000), dtype=torch.int32, device="cuda"), tri_id_base=1200)
    for _ in range(2):   # first cast fills the static cache, the second starts from it
        d, t = gh.cast()
        assert np.array_equal(t.cpu().numpy(), t0) and np.array_equal(d.cpu().numpy().view(np.uint32), d0.view(np.uint32))
    gh.close()
    # errors: misaligned soup, negative count, capacity
    v4 = tris_to_float4(tris)
    L, h = g._L, g._h
    E_INVALID, E_CAPACITY = 1, 3   # include/grca.h
    assert L.grca_update_scene(h, v4.data_ptr() + 4, 10, None, 0, None, 0, None, 0) == E_INVALID
    assert L.grca_update_scene(h, v4.data_ptr(), -1, None, 0, None, 0, None, 0) == E_INVALID
    assert L.grca_update_scene(h, v4.data_ptr(), n, v4.data_ptr(), 3, None, 1, None, 0) == E_INVALID  # no indices
    assert L.grca_update_scene(h, v4.data_ptr(), n + 1, None, 0, None, 0, None, 0) == E_CAPACITY      # > max_triangles


@pytest.mark.parametrize("n_em,gamma", [(9, 10), (17, 10), (16, 192)])
def test_many_emitters_generic_paths(n_em, gamma):
    """More emitters than the unrolled K2 handles (9: generic kernel + LUT; 17: no LUT, binary search;
    16 x 192 channels: the largest LUT tables, whose shared memory exceeds what create assumed)."""
    ems, tris = sg.random_scene(40 + n_em, n_tris=400, n_emitters=n_em, gamma=gamma, chi=60, extent=7.0)
    dist, tri, st, _ = run(ems, tris)
    check(ems, tris, dist, tri)
    assert st["pairs"] == len(tris) * n_em


def test_split_refine_path_identical():
    """The two-kernel (K2b bounds + K4s small) path gives bit-identical results to the fused one."""
    ems, tris = sg.random_scene(55, n_tris=1500, n_emitters=3, gamma=14, chi=220, extent=9.0)
    a = run(ems, tris)
    b = run(ems, tris, flags=G.DEBUG_SPLIT_REFINE)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
    # the fused path scales its small-rectangle cap to the load (more pairs may take K3/K4, whose
    # per-channel refinement trims candidates): compare the invariants
    for k in ("survivors", "hits_recorded"):
        assert a[2][k] == b[2][k], k
    assert a[2]["small_pairs"] + a[2]["large_pairs"] == b[2]["small_pairs"] + b[2]["large_pairs"]
    check(ems, tris, a[0], a[1])


@pytest.mark.parametrize("seed", [3, 8, 13, 21])
def test_a7_per_channel_refinement(seed):
    """A7 (late pass): with every pair forced through the large path, refined
    per-channel ray ranges give bit-identical results to whole rectangle rows, test fewer
    candidates, and keep every brute-force hit (all-hits invariant)."""
    ems, tris = sg.random_scene(200 + seed, n_tris=900, n_emitters=2, gamma=24, chi=400, extent=6.0,
                                max_range=None if seed % 2 else 9.0)
    ref = run(ems, tris, small_max=1, flags=G.DEBUG_NO_REFINE)
    a7 = run(ems, tris, small_max=1, flags=G.DEBUG_COUNT_ALL_HITS)
    assert np.array_equal(ref[1], a7[1]) and np.array_equal(ref[0].view(np.uint32), a7[0].view(np.uint32))
    assert a7[2]["rtic_tested"] < ref[2]["rtic_tested"]
    oref = oracle.cast(ems, tris, want_t64=True, want_allhits=True)
    check(ems, tris, a7[0], a7[1], ref=oref)
    _check_all_hits(ems, tris, a7[3].debug_all_hits().cpu().numpy(), oref)


def test_a7_c1_and_fixtures():
    """A7 on C1 (ground under the sensor, zenith ceiling, seam triangle, grazing triangle)."""
    ems = [sg.c1_emitter()]
    tris = sg.c1_scene()
    a7 = run(ems, tris, small_max=1, flags=G.DEBUG_COUNT_ALL_HITS)
    oref = oracle.cast(ems, tris, want_t64=True, want_allhits=True)
    check(ems, tris, a7[0], a7[1], ref=oref)
    # (C1's ground grid lines under the emitter: 14 rays along shared edges, see test_all_hits_invariant)
    _check_all_hits(ems, tris, a7[3].debug_all_hits().cpu().numpy(), oref, bound=2e-3)


def test_hybrid_static_dynamic_exact():
    """NEXT-f2 hybrid: static triangles cast once into cached keys, frames cull only the dynamic ones;
    bit-identical to casting everything, across frames, emitter changes and clear_static."""
    ems, tris = sg.random_scene(300, n_tris=2400, n_emitters=2, gamma=16, chi=256, extent=8.0)
    n_s = 1500
    st = tris[:n_s]
    g = Grca(device=0, max_triangles=len(tris), max_rays=sg.n_rays_total(ems) + 4096,
             debug_flags=G.DEBUG_COUNT_ALL_HITS)
    g.set_emitters(ems)
    g.set_static_triangles(tris_to_float4(st), tri_id_base=0)
    rng = np.random.default_rng(0)
    for frame in range(3):
        dyn = tris[n_s:] + np.float32(rng.normal(size=3) * 0.5)          # moved dynamic triangles
        g.update_triangles(tris_to_float4(dyn), tri_id_base=n_s)
        d_h, t_h = g.cast()
        allh = g.debug_all_hits().cpu().numpy().copy()
        full = np.concatenate([st, dyn], 0)
        d_f, t_f, _, gf = run(ems, full, flags=G.DEBUG_COUNT_ALL_HITS)
        assert np.array_equal(t_h.cpu().numpy(), t_f)
        assert np.array_equal(d_h.cpu().numpy().view(np.uint32), d_f.view(np.uint32))
        assert np.array_equal(allh, gf.debug_all_hits().cpu().numpy())
    check(ems, full, d_f, t_f)
    # emitters change -> the static cache is recomputed
    ems2, _ = sg.random_scene(301, n_tris=10, n_emitters=1, gamma=12, chi=300)
    g.set_emitters(ems2)
    d_h, t_h = g.cast()
    d_f, t_f, _, _ = run(ems2, full)
    assert np.array_equal(t_h.cpu().numpy(), t_f)
    # leave hybrid mode
    g.clear_static()
    d_c, t_c = g.cast()
    d_f, t_f, _, _ = run(ems2, dyn, ids=np.arange(n_s, len(tris)))
    assert np.array_equal(t_c.cpu().numpy(), t_f)


def _area_kept(em, tris, eps):
    """Paper Step 1.2 in fp64: keep a triangle for emitter em unless
    (A_T (c-o).n)^2 < eps^2 |c-o|^6 (two-sided: |(c-o).n|)."""
    t = tris.astype(np.float64)
    c = t.mean(axis=1)
    hN = 0.5 * np.cross(t[:, 1] - t[:, 0], t[:, 2] - t[:, 0])
    co = c - em.origin.astype(np.float64)
    an = np.einsum("ij,ij->i", hN, co)
    d2 = np.einsum("ij,ij->i", co, co)
    return ~(an * an < eps * eps * d2 ** 3)


@pytest.mark.parametrize("scene", ["c1", "random"])
def test_paper_mode_apparent_area_cull(scene):
    """NEXT-f1 paper mode (approximate): the GPU equals the oracle run on the triangles the paper's
    apparent-area test keeps per emitter (up to threshold ties), keeps the paper's Hit% floor (>= 98 %
    at 1 mm vs exact brute force) and reports SAT/BAT counts of its survivors."""
    if scene == "c1":
        ems, tris = [sg.c1_emitter()], sg.c1_scene()
        eps = 1e-4   # large enough to cull a visible share of C1's small random triangles
    else:
        ems, tris = sg.random_scene(77, n_tris=1500, n_emitters=2, gamma=16, chi=256, extent=10.0)
        eps = 1e-4
    n = sg.n_rays_total(ems)
    g = Grca(device=0, max_triangles=len(tris), max_rays=n, apparent_area_eps=eps)
    g.set_emitters(ems)
    g.update_triangles(tris_to_float4(tris))
    dist, tri, st = g.cast(stats=True)
    dist, tri = dist.cpu().numpy(), tri.cpu().numpy()
    assert st["area_culled"] > 0
    base = 0
    agree, tot = 0, 0
    for em in ems:
        keep = _area_kept(em, tris, eps)
        ids = np.nonzero(keep)[0].astype(np.int32)
        ref = oracle.cast([em], tris[keep], ids=ids, want_t64=True)
        sl = slice(base, base + em.n_rays)
        rep = oracle.compare([em], tris[keep], dist[sl], tri[sl], ref, ids=ids)
        agree += rep["agree"]
        tot += rep["rays"]
        base += em.n_rays
    assert agree >= 0.999 * tot
    exact = oracle.cast(ems, tris, want_t64=True)
    rep = oracle.compare(ems, tris, dist, tri, exact)
    assert rep["hit_pct_1mm"] >= 98.0, rep["hit_pct_1mm"]


def _noisy_emitters(seed, n_em=2):
    ems, tris = sg.random_scene(seed, n_tris=1200, n_emitters=n_em, gamma=14, chi=300, extent=7.0)
    for k, e in enumerate(ems):
        e.ray_azimuth = sg.perturbed_azimuths(e.rays_per_channel, e.hfov_deg, seed + k, frac=0.45)
        e.elev = sg.perturbed_elev(e.elev, seed + k)
    return ems, tris


@pytest.mark.parametrize("seed", [5, 6])
def test_noise_model_angles(seed):
    """NEXT-f4 noise model: perturbed per-ray azimuths and per-channel elevations;
    the ray table matches the oracle bit for bit and the result is exact (cull widened by one ray)."""
    ems, tris = _noisy_emitters(400 + seed)
    g = Grca(device=0, max_triangles=len(tris), max_rays=sg.n_rays_total(ems))
    g.set_emitters(ems)
    assert np.array_equal(g.debug_ray_table().view(np.uint32), oracle.ray_table(ems).view(np.uint32))
    for small_max, flags in ((0, G.DEBUG_COUNT_ALL_HITS), (1, G.DEBUG_COUNT_ALL_HITS)):
        dist, tri, st, gg = run(ems, tris, small_max=small_max, flags=flags)
        ref = oracle.cast(ems, tris, want_t64=True, want_allhits=True)
        check(ems, tris, dist, tri, ref=ref)
        _check_all_hits(ems, tris, gg.debug_all_hits().cpu().numpy(), ref)


def test_distance_noise():
    """Distance noise is a post-process of hit distances: ids unchanged, misses stay +inf, the
    deviation is N(0, sigma^2), reproducible for a seed and cast index, different across casts."""
    ems, tris = sg.random_scene(510, n_tris=3000, n_emitters=2, gamma=32, chi=600, extent=6.0)
    g = Grca(device=0, max_triangles=len(tris), max_rays=sg.n_rays_total(ems))
    g.set_emitters(ems)
    g.update_triangles(tris_to_float4(tris))
    d0, t0 = [x.cpu().numpy() for x in g.cast()]
    sigma = 0.05
    g.set_distance_noise(sigma, seed=123)
    d1, t1 = [x.cpu().numpy() for x in g.cast()]
    d2, _ = [x.cpu().numpy() for x in g.cast()]
    assert np.array_equal(t0, t1)
    hit = t0 >= 0
    assert hit.sum() > 5000 and np.all(np.isinf(d1[~hit]))
    dev = (d1[hit].astype(np.float64) - d0[hit])
    mask = d0[hit] > 10 * sigma   # away from the clamp at 0
    dv = dev[mask]
    assert abs(dv.mean()) < 4 * sigma / np.sqrt(dv.size) and abs(dv.std() / sigma - 1) < 0.05
    assert not np.array_equal(d1, d2)
    g2 = Grca(device=0, max_triangles=len(tris), max_rays=sg.n_rays_total(ems))
    g2.set_emitters(ems)
    g2.update_triangles(tris_to_float4(tris))
    g2.cast()
    g2.set_distance_noise(sigma, seed=123)
    d3, _ = [x.cpu().numpy() for x in g2.cast()]
    assert np.array_equal(d3.view(np.uint32), d1.view(np.uint32))   # same seed, same cast index


def test_unpack_range_slices():
    """grca_unpack_range (the reduce-scatter merge's K5): for each ray slice of a 3-way split (ragged),
    keys passed as a separate slice tensor give exactly the full unpack's values for those rays,
    distance noise included (keyed by the global ray index, same cast index); bad ranges rejected."""
    ems, tris = sg.random_scene(512, n_tris=2500, n_emitters=2, gamma=17, chi=301, extent=6.0)
    n = sg.n_rays_total(ems)

    def handle():
        g = Grca(device=0, max_triangles=len(tris), max_rays=n)
        g.set_emitters(ems)
        g.update_triangles(tris_to_float4(tris))
        g.set_distance_noise(0.05, seed=9)
        return g

    g = handle()
    d_full, t_full = [x.cpu().numpy() for x in g.cast()]
    assert (t_full >= 0).sum() > 1000
    c = -(-n // 3)
    for r in range(3):
        gr = handle()
        gr.cast_packed()
        first = r * c
        m = min(c, n - first)
        keys = gr.hits_packed()[first: first + m].clone()
        d = torch.empty(m, dtype=torch.float32, device="cuda")
        t = torch.empty(m, dtype=torch.int32, device="cuda")
        gr.unpack_range(keys, first, d, t)
        torch.cuda.synchronize()
        assert np.array_equal(t.cpu().numpy(), t_full[first: first + m])
        assert np.array_equal(d.cpu().numpy().view(np.uint32), d_full[first: first + m].view(np.uint32))
        E_INVALID = 1   # include/grca.h
        assert gr._L.grca_unpack_range(gr._h, None, n - 5, 6, d.data_ptr(), None) == E_INVALID
        assert gr._L.grca_unpack_range(gr._h, None, -1, 1, d.data_ptr(), None) == E_INVALID
        gr.close()


def _uid():
    from paper_2605_10457_b200.grca import nccl_unique_id

    return nccl_unique_id()


@pytest.mark.parametrize("shard,merge,gather", [(1, 0, 0), (1, 1, 0), (2, 0, 1), (2, 0, 0), (0, 0, 0)])
def test_collective_one_rank_nccl(shard, merge, gather):
    """the library-owned collective (grca_create with an NCCL unique id ->
    ncclCommInitRank; grca_cast merges in-stream: ncclAllReduce / ncclReduceScatter(ncclMin, uint64)
    for triangle shards, one ncclBroadcast per emitter for gathered emitter shards) on a one-rank
    communicator gives the non-collective result bit for bit, over several casts."""
    ems, tris = sg.random_scene(91, n_tris=2000, n_emitters=3, gamma=12, chi=200, extent=9.0)
    base = run(ems, tris)
    g = Grca(device=0, max_triangles=len(tris), max_rays=sg.n_rays_total(ems), nranks=1, rank=0, nccl_uid=_uid(),
             shard_mode=shard, merge=merge, gather_outputs=bool(gather))
    for _ in range(3):
        got = run(ems, tris, handle=g)
        assert np.array_equal(base[1], got[1]) and np.array_equal(base[0].view(np.uint32), got[0].view(np.uint32))
    sh = g.get_shard()
    # AUTO: emitter shards when n_emitters >= nranks and nranks | n_emitters (always, with one rank)
    assert sh["shard_mode"] == (shard or G.SHARD_EMITTERS)
    assert sh["n_written"] == sg.n_rays_total(ems) and sh["first_ray"] in (0, -1)
    g.close()


def test_nvls_merge_nccl_window_one_rank():
    """NEXT-f3 through NCCL (GRCA_MERGE_NVLS): keys + barrier flag in an ncclMemAlloc'd symmetric window
    (ncclCommWindowRegister), hits recorded with multimem.red.min.u64 at the window's lsa multimem
    address, device barriers on the window's flag.  Bit-identical to the local path where NCCL provides
    multimem; where it does not (NVLS needs an NVSwitch multicast group), set_emitters reports
    GRCA_E_NCCL with NCCL's reason -- never a silent fallback."""
    ems, tris = sg.random_scene(61, n_tris=3000, n_emitters=2, gamma=16, chi=256, extent=10.0)
    a_d, a_t, _, _ = run(ems, tris)
    g = Grca(device=0, max_triangles=len(tris), max_rays=sg.n_rays_total(ems), nranks=1, rank=0, nccl_uid=_uid(),
             shard_mode=G.SHARD_TRIANGLES, merge=G.MERGE_NVLS)
    try:
        g.set_emitters(ems)
    except GrcaError as e:
        assert e.status == G.GRCA_E_NCCL, e
        g.close()
        pytest.skip(f"no NVLS multimem on a one-rank NCCL communicator here: {e}")
    for _ in range(3):
        d, t, _, _ = run(ems, tris, handle=g)
        assert np.array_equal(t, a_t) and np.array_equal(d.view(np.uint32), a_d.view(np.uint32))
    assert not g.nvls_status()["timed_out"]
    g.close()


def test_virtual_ranks_partitions():
    """GRCA_DEBUG_VIRTUAL_RANKS: each handle does exactly rank r's share of a P-rank cast on one GPU.
    Emitter shards (P = 3, 4 emitters: rank r casts n mod 3 == r) write exactly their emitters' rays,
    equal to the one-GPU result, and leave the rest of the outputs untouched; triangle shards (P = 2)
    min-merge to the one-GPU keys, and under the reduce-scatter merge each rank unpacks only its slice
    [r c, r c + c), c = ceil(n / P)."""
    ems, tris = sg.random_scene(92, n_tris=2500, n_emitters=4, gamma=10, chi=150, extent=9.0)
    n = sg.n_rays_total(ems)
    base_d, base_t, _, gb = run(ems, tris)
    gb.cast_packed()
    base_keys = gb.hits_packed().clone().cpu().numpy()
    offs = np.cumsum([0] + [e.n_rays for e in ems])
    v4 = tris_to_float4(tris)
    for r in range(3):
        g = Grca(device=0, max_triangles=len(tris), max_rays=n, nranks=3, rank=r, shard_mode=G.SHARD_EMITTERS,
                 debug_flags=G.DEBUG_VIRTUAL_RANKS)
        g.set_emitters(ems)
        g.update_triangles(v4)
        d = torch.full((n,), 7.0, device="cuda")
        t = torch.full((n,), -7, dtype=torch.int32, device="cuda")
        _, _, st = g.cast(d, t, stats=True)
        d, t = d.cpu().numpy(), t.cpu().numpy()
        mine = np.zeros(n, bool)
        for m in range(4):
            if m % 3 == r:
                mine[offs[m]: offs[m + 1]] = True
        assert np.array_equal(t[mine], base_t[mine]) and np.array_equal(d[mine].view(np.uint32), base_d[mine].view(np.uint32))
        assert np.all(t[~mine] == -7) and np.all(d[~mine] == 7.0)
        sh = g.get_shard()
        assert sh == {"shard_mode": G.SHARD_EMITTERS, "first_ray": -1, "n_written": int(mine.sum())}
        assert st["pairs"] == len(tris) * sum(1 for m in range(4) if m % 3 == r)
        g.close()
    merged = None
    c = -(-n // 2)
    for r in range(2):
        own = np.nonzero(((np.arange(len(tris)) // 256) % 2) == r)[0]
        g = Grca(device=0, max_triangles=len(tris), max_rays=n, nranks=2, rank=r, shard_mode=G.SHARD_TRIANGLES,
                 merge=G.MERGE_REDUCE_SCATTER, debug_flags=G.DEBUG_VIRTUAL_RANKS)
        g.set_emitters(ems)
        g.update_triangles(tris_to_float4(tris[own]), tri_ids=torch.as_tensor(own.astype(np.int32), device="cuda"))
        d = torch.full((n,), 7.0, device="cuda")
        t = torch.full((n,), -7, dtype=torch.int32, device="cuda")
        g.cast(d, t)
        keys = g.hits_packed().clone().cpu().numpy()
        merged = keys if merged is None else np.minimum(merged, keys)
        f, m = r * c, min(c, n - r * c)
        assert g.get_shard() == {"shard_mode": G.SHARD_TRIANGLES, "first_ray": f, "n_written": m}
        t = t.cpu().numpy()
        kt = (keys[f: f + m] & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
        assert np.array_equal(t[f: f + m], kt) and np.all(t[:f] == -7) and np.all(t[f + m:] == -7)
        g.close()
    assert np.array_equal(merged, base_keys)


def test_float3_vertices_identical():
    """grca_update_triangles_f3 (packed float3 vertices) == float4, soup and indexed, bit for bit."""
    ems, tris = sg.random_scene(71, n_tris=2500, n_emitters=2, gamma=16, chi=300, extent=9.0)
    a_d, a_t, _, g = run(ems, tris)
    v3 = torch.as_tensor(np.ascontiguousarray(tris.reshape(-1, 3)), device="cuda")
    g.update_triangles(v3)
    d, t = g.cast()
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), a_t) and np.array_equal(d.cpu().numpy().view(np.uint32), a_d.view(np.uint32))
    flat = np.asarray(tris, np.float32).reshape(-1, 3)
    uniq, inv = np.unique(flat, axis=0, return_inverse=True)
    g.update_triangles(torch.as_tensor(np.ascontiguousarray(uniq), device="cuda"),
                       indices=torch.as_tensor(inv.astype(np.int32).reshape(-1), device="cuda"))
    d, t = g.cast()
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), a_t) and np.array_equal(d.cpu().numpy().view(np.uint32), a_d.view(np.uint32))


def test_cuda_graph_cast_mode():
    """GRCA_USE_CUDA_GRAPH: every cast runs as one CUDA graph (re-captured, cudaGraphExecUpdate'd in place);
    over scene changes, an emitter change and the hybrid static path the results are bit-identical to the
    plain launches."""
    s = torch.cuda.Stream()
    ems, tris = sg.random_scene(93, n_tris=1800, n_emitters=2, gamma=12, chi=160, extent=8.0)
    ems2, tris2 = sg.random_scene(94, n_tris=1500, n_emitters=3, gamma=10, chi=128, extent=8.0)
    n = max(sg.n_rays_total(ems), sg.n_rays_total(ems2))
    g = Grca(device=0, stream=s, max_triangles=2000, max_rays=n, debug_flags=G.USE_CUDA_GRAPH)
    with torch.cuda.stream(s):
        for e, t in ((ems, tris), (ems, tris2), (ems2, tris2), (ems2, tris)):
            ref = run(e, t)
            got = run(e, t, handle=g)
            assert np.array_equal(ref[1], got[1]) and np.array_equal(ref[0].view(np.uint32), got[0].view(np.uint32))
        # hybrid: static triangles cached on the first cast, dynamic ones every cast
        g.set_emitters(ems)
        st4 = tris_to_float4(tris)
        g.set_static_triangles(st4, tri_id_base=0)
        g.update_triangles(tris_to_float4(tris2), tri_id_base=len(tris))
        for _ in range(2):
            d, t = g.cast()
            s.synchronize()
        both = np.concatenate([tris, tris2], 0)
        ref = run(ems, both)
        assert np.array_equal(ref[1], t.cpu().numpy())
    g.close()


def test_cast_is_capturable_by_the_caller():
    """grca_cast allocates nothing and syncs nothing, so a caller can capture it into its own
    CUDA graph (torch.cuda.graph on the handle's stream) and replay it after rewriting the borrowed
    vertex buffer in place: each replay equals a plain cast of the new vertices."""
    if "bounds-checked" in G.version():
        pytest.skip("the bounds-checked build synchronizes inside grca_cast (not capturable by design)")
    ems, tris = sg.random_scene(95, n_tris=1200, n_emitters=2, gamma=12, chi=128, extent=8.0)
    _, tris_b = sg.random_scene(96, n_tris=1200, n_emitters=2, gamma=12, chi=128, extent=8.0)
    s = torch.cuda.Stream()
    g = Grca(device=0, stream=s, max_triangles=len(tris), max_rays=sg.n_rays_total(ems))
    g.set_emitters(ems)
    v4 = tris_to_float4(tris)
    d = torch.empty(sg.n_rays_total(ems), device="cuda")
    t = torch.empty(sg.n_rays_total(ems), dtype=torch.int32, device="cuda")
    g.update_triangles(v4)
    with torch.cuda.stream(s):
        g.cast(d, t)   # warm-up outside the capture
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        g.cast(d, t)
    for src in (tris_b, tris):
        v4.copy_(tris_to_float4(src))
        graph.replay()
        torch.cuda.synchronize()
        ref = run(ems, src)
        assert np.array_equal(ref[1], t.cpu().numpy()) and np.array_equal(ref[0].view(np.uint32), d.cpu().numpy().view(np.uint32))
    g.close()


def _exact_rect(em, tri, n=400):
    """Host recount of a triangle's exact (channel, ray) rectangle seen from emitter em (level frame, 360 deg):
    elevation / azimuth extremes over a dense barycentric sampling of the triangle (fp64), mapped to the
    channels inside [phi_min, phi_max] and the ray indices inside the azimuth arc."""
    u, v = np.meshgrid(np.linspace(0, 1, n), np.linspace(0, 1, n))
    m = (u + v) <= 1
    u, v = u[m], v[m]
    T = np.asarray(tri, np.float64)
    P = T[0] + u[:, None] * (T[1] - T[0]) + v[:, None] * (T[2] - T[0]) - np.asarray(em.origin, np.float64)
    f, r, up = (np.asarray(x, np.float64) for x in (em.forward, em.right, em.up))
    xf, xr, xu = P @ f, P @ r, P @ up
    elev = np.arctan2(xu, np.hypot(xf, xr))
    az = np.arctan2(xr, xf)
    phi = em.elev.astype(np.float64)
    chans = np.nonzero((phi >= elev.min()) & (phi <= elev.max()))[0]
    chi = em.rays_per_channel
    dth = 2 * np.pi / chi
    th = -(chi // 2) * dth + dth * np.arange(chi)   # ray azimuths (ray i = chi/2 is theta = 0)
    wraps = bool(az.max() - az.min() > np.pi)      # the arc crosses theta = +-pi (the seam)
    span = int(np.count_nonzero((th >= az.min()) & (th <= az.max())))
    return len(chans), span, wraps


def test_sat_bat_classification():
    """NEXT-f1 SAT/BAT counters (Eq. sat_cond, (gamma_T, chi_T) = (64, 64)): every surviving
    pair is classified exactly once (sat + bat == survivors on a scene without degenerate triangles), and on
    single-triangle scenes the GPU's class equals a host recount of the exact rectangle: SAT iff the arc does
    not wrap the seam and it spans <= 64 channels and <= 64 rays (cases chosen far from the thresholds)."""
    ems, tris = sg.random_scene(81, n_tris=1500, n_emitters=2, gamma=16, chi=256, extent=10.0)
    _, _, st, _ = run(ems, tris)
    assert st["sat_pairs"] + st["bat_pairs"] == st["survivors"] > 0
    em = sg.Emitter(origin=(0.0, 0.0, 0.0), elev=sg.full_sphere_elev(128), rays_per_channel=512)
    cases = {
        "tiny far": [[20.0, -0.05, -0.03], [20.0, 0.05, -0.03], [20.0, 0.0, 0.03]],
        "mid wall": [[5.0, -1.0, -1.0], [5.0, 1.0, -1.0], [5.0, 0.0, 1.0]],
        "wide wall": [[2.0, -4.0, 0.1], [2.0, 4.0, 0.1], [2.0, 0.0, 0.3]],
        "tall wall": [[2.0, -0.1, -4.0], [2.0, 0.1, -4.0], [2.0, 0.0, 4.0]],
        "seam": [[-5.0, -1.0, -1.0], [-5.0, 1.0, -1.0], [-5.0, 0.0, 1.0]],
    }
    expect = {"tiny far": "sat", "mid wall": "sat", "wide wall": "bat", "tall wall": "bat", "seam": "bat"}
    for name, t in cases.items():
        n_ch, span, wraps = _exact_rect(em, t)
        sat = (not wraps) and n_ch <= 64 and span <= 64
        assert ("sat" if sat else "bat") == expect[name], (name, n_ch, span, wraps)
        assert wraps or (n_ch <= 48 and span <= 48) or n_ch >= 80 or span >= 80, (name, n_ch, span)   # clear cases
        _, _, st, g = run([em], np.array([t], np.float32))
        assert (st["sat_pairs"], st["bat_pairs"]) == ((1, 0) if sat else (0, 1)), (name, st["sat_pairs"], st["bat_pairs"])
        g.close()


def test_instances_match_posed_soup_and_oracle():
    """grca_update_instances (rigid instances, ABI extension of SURVEY 8(a) A1): a static soup (part A) followed
    by 6 posed instances of a local mesh (part C) equals, bit for bit, the cast of the same triangles given as
    one soup whose instance vertices the host posed with the documented fp32 operation order
    (scenegen.apply_pose_f32); parity with the oracle on that soup; instances alone (no part A) too."""
    car_v, car_f = sg.car_mesh(24, 24, dims=(4.0, 2.0, 1.2))
    poses = sg.pose_instances(6, (40.0, 30.0, 6.0), seed=5, frame=1, scale_lo=0.3, scale_hi=3.0)
    Ms = np.stack([sg.pose_matrix(p) for p in poses])                       # (6, 3, 4) fp32
    posed = np.concatenate([sg.apply_pose_f32(car_v, M)[car_f] for M in Ms], 0)   # (6 F, 3, 3)
    static = sg.grid_mesh(8, 8, -5, -5, 45, 35, 0.0)
    soup = np.ascontiguousarray(np.concatenate([static, posed], 0))
    ems = [sg.Emitter(origin=(10.0, 12.0, 2.0), elev=sg.full_sphere_elev(32), rays_per_channel=720),
           sg.Emitter(origin=(30.0, 5.0, 1.5), forward=(0, 1, 0), right=(1, 0, 0), elev=sg.vlp16_elev(),
                      rays_per_channel=500, hfov_deg=180)]
    ref = run(ems, soup)
    check(ems, soup, ref[0], ref[1])
    g = Grca(device=0, max_triangles=len(soup), max_rays=sg.n_rays_total(ems))
    g.set_emitters(ems)
    lv = torch.as_tensor(car_v.astype(np.float32), device="cuda")
    lf = torch.as_tensor(car_f.astype(np.int32), device="cuda")
    pm = torch.as_tensor(Ms, device="cuda")
    g.update_scene(soup=tris_to_float4(static))
    g.update_instances(lv, lf, pm)
    d, t = g.cast()
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), ref[1]) and np.array_equal(d.cpu().numpy().view(np.uint32), ref[0].view(np.uint32))
    # instances alone: ids start at 0 for the first instance triangle
    g2 = Grca(device=0, max_triangles=len(posed), max_rays=sg.n_rays_total(ems))
    g2.set_emitters(ems)
    g2.update_instances(lv, lf, pm)
    d2, t2 = g2.cast()
    torch.cuda.synchronize()
    ref2 = run(ems, posed)
    assert np.array_equal(t2.cpu().numpy(), ref2[1]) and np.array_equal(d2.cpu().numpy().view(np.uint32), ref2[0].view(np.uint32))
    # errors: misaligned poses, capacity
    E_INVALID, E_CAPACITY = 1, 3
    L = g._L
    assert L.grca_update_instances(g._h, lv.data_ptr(), len(car_v), lf.data_ptr(), len(car_f), pm.data_ptr() + 4, 6) == E_INVALID
    assert L.grca_update_instances(g._h, lv.data_ptr(), len(car_v), lf.data_ptr(), len(car_f), pm.data_ptr(), 7) == E_CAPACITY
    g.close()
    g2.close()
