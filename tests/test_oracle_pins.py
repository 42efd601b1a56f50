"""Pins of the brute-force oracle against things other than itself (-m "not gpu").

Each test cites what fixes the expected value: a worked example printed in
SPEC.md/PAPER.md (tests/golden/spec_examples.json), a closed form, a library
routine (numpy.linalg.solve), an invariant, or brute force by hand.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import scenegen as sg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _em(**kw):
    base = dict(origin=(0, 0, 0), forward=(1, 0, 0), right=(0, -1, 0), up=(0, 0, 1))
    base.update(kw)
    return sg.Emitter(**base)


# ----------------------------------------------------------------- MT core --

def test_mt_spec_examples(oracle_lib):
    """t = 5.0; reversed direction -> miss; parallel -> det == 0."""
    g = GOLD["moller_trumbore"]
    v0, v1, v2 = g["triangle"]
    for case in g["cases"]:
        ok, t, u, v, _ = oracle.mt(g["origin"], case["dir"], v0, v1, v2)
        if case.get("det_zero"):
            assert not ok
            continue
        assert ok
        hit = u >= 0 and v >= 0 and u + v <= 1 and t > 0
        assert hit == case["hit"]
        if case["hit"]:
            assert t == case["t"]


def test_mt_matches_linear_solve(oracle_lib):
    """o + t d = v0 + u e1 + v e2 solved by LAPACK (numpy.linalg.solve) on random cases.

    Pins the textbook formulas against a transposed operand, wrong sign or index."""
    rng = np.random.default_rng(7)
    for _ in range(2000):
        o = rng.normal(size=3) * 3
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        v0, v1, v2 = rng.normal(size=(3, 3)) * 4 + rng.normal(size=3) * 10
        M = np.stack([-d, v1 - v0, v2 - v0], axis=1)
        if abs(np.linalg.det(M)) < 1e-6:
            continue
        t, u, v = np.linalg.solve(M, o - v0)
        ok, t2, u2, v2_, _ = oracle.mt(o, d, v0, v1, v2)
        assert ok
        np.testing.assert_allclose([t2, u2, v2_], [t, u, v], rtol=1e-8, atol=1e-9)


# ------------------------------------------------------- ray definition O1 --

def test_ray_direction_spec_examples(oracle_lib):
    """SPEC.md:50-52 on several frames: (0,0)->f, (pi/2,0)->r, (0,pi/2)->u."""
    rng = np.random.default_rng(3)
    for trial in range(5):
        f, r, u = sg.random_frame(rng) if trial else (np.float32([1, 0, 0]), np.float32([0, 1, 0]),
                                                      np.float32([0, 0, 1]))
        halfpi32 = np.float32(math.pi / 2)
        em = _em(forward=f, right=r, up=u, elev=np.array([0.0, halfpi32], np.float32), rays_per_channel=8)
        tab = oracle.ray_table([em])
        # chi = 8: theta0 = -pi, dtheta = pi/4 -> i = 4 is theta = 0, i = 6 is theta = pi/2
        np.testing.assert_array_equal(tab[0 * 8 + 4], f)                     # exact: cos 0 = 1, sin 0 = 0
        np.testing.assert_allclose(tab[0 * 8 + 6], r, atol=1e-12)           # cos(pi/2) ~ 6e-17
        np.testing.assert_allclose(tab[1 * 8 + 4], u, atol=1e-7)            # RN32(pi/2) overshoots by 4.4e-8


def test_demo_grid_middle_ray_is_forward(oracle_lib):
    """SPEC.md:161-163 / PAPER.md:435: gamma=4, chi=8 demo: ray (2,4) = f; 128x4096 -> 524,288 rays."""
    g = GOLD["demo_grid"]
    f = np.float32([0.6, 0.8, 0.0])
    em = _em(forward=f, right=(0.8, -0.6, 0.0), elev=sg.full_sphere_elev(g["gamma"]), rays_per_channel=g["chi"])
    tab = oracle.ray_table([em])
    j, i = g["ray"]
    np.testing.assert_array_equal(tab[j * g["chi"] + i], f)
    for chi in (7, 9, 1, 5):   # odd chi: theta0 = -floor(chi/2) dtheta puts ray floor(chi/2) on f
        odd = _em(forward=f, right=(0.8, -0.6, 0.0), elev=np.array([0.0], np.float32), rays_per_channel=chi)
        np.testing.assert_array_equal(oracle.ray_table([odd])[chi // 2], f)
    big = _em(elev=sg.full_sphere_elev(128), rays_per_channel=4096)
    assert oracle.n_rays([big]) == g["full_sphere_rays_128x4096"]


def test_ray_table_layout_and_unit_length(oracle_lib):
    """Channel-major layout g = O_n + j chi + i and |d| within 1e-6 of 1."""
    e1 = _em(elev=sg.full_sphere_elev(16), rays_per_channel=4096)
    e2 = _em(origin=(1, 2, 3), elev=sg.vlp16_elev(), rays_per_channel=100, hfov_deg=180)
    tab = oracle.ray_table([e1, e2])
    assert tab.shape == (16 * 4096 + 16 * 100, 3)
    nrm = np.linalg.norm(tab.astype(np.float64), axis=1)
    assert np.all(np.abs(nrm - 1) <= 1e-6)
    for c in GOLD["global_index"]["cases"]:
        g = c["j"] * c["chi"] + (c["R_from"] + c["i"]) % c["chi"] + c["O_n"]
        assert g == c["g"]
    # ray 8196 of emitter 0 is (j=2, i=4): closed-form angles
    dth = 2 * math.pi / 4096
    th = -(4096 // 2) * dth + 4 * dth
    ph = float(sg.full_sphere_elev(16)[2])
    d = np.array([math.cos(th) * math.cos(ph), -math.sin(th) * math.cos(ph), math.sin(ph)])
    np.testing.assert_allclose(tab[8196], d, atol=1e-7)
    # second emitter starts at O_1 = 16*4096; 180 deg: dtheta = pi/100, theta0 = -50 dtheta = -pi/2
    th = -math.pi / 2
    ph = float(sg.vlp16_elev()[0])
    d = np.array([math.cos(th) * math.cos(ph), -math.sin(th) * math.cos(ph), math.sin(ph)])
    np.testing.assert_allclose(tab[16 * 4096], d, atol=1e-7)


def test_eq1_worked_example():
    """1 x 128 x 4096 x 1e7 ~ 5.2e12 RTIC (the brute-force count the oracle performs)."""
    e = GOLD["eq1"]
    total = e["omega"] * e["gamma"] * e["chi"] * e["tau"]
    assert abs(total - e["approx"]) / e["approx"] < 0.01


# ------------------------------------------------------------- closed forms --

def _hits(res):
    return res["id"] >= 0


def test_quad_x5_closed_form(oracle_lib):
    """North-star fixture (i): square x = 5, |y|,|z| <= 1 -> t = 5/d_x inside, miss outside;
    the diagonal y = z is shared (watertight, tie -> id 0)."""
    em = sg.c1_emitter()
    o = em.origin.astype(np.float64)
    tris = sg.quad_x5(o)
    res = oracle.cast([em], tris, want_t64=True)
    D = oracle.ray_table([em]).astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.where(D[:, 0] > 0, (5.0 - 0.0) / D[:, 0], np.inf)
        y = t * D[:, 1]
        z = t * D[:, 2]
    inside = (D[:, 0] > 0) & (np.abs(y) <= 1) & (np.abs(z) <= 1)
    margin = np.minimum(1 - np.abs(y), 1 - np.abs(z))
    clear = ~np.isfinite(margin) | (np.abs(margin) > 1e-9)
    assert np.array_equal(_hits(res)[clear], inside[clear])
    assert inside.sum() > 50
    np.testing.assert_allclose(res["t64"][inside & clear], t[inside & clear], rtol=1e-12)
    # which triangle: T0 is the y >= z half, T1 the z >= y half (tie on the diagonal -> 0)
    sel = inside & clear & (np.abs(y - z) > 1e-9)
    exp_id = np.where(y[sel] > z[sel], 0, 1)
    assert np.array_equal(res["id"][sel], exp_id)
    # centre ray (channel 8, ray 256) is exactly f = (1,0,0): t = 5, on the diagonal -> id 0
    g = 8 * 512 + 256
    assert res["t"][g] == 5.0 and res["id"][g] == 0


def test_ground_plane_closed_form(oracle_lib):
    """Large quad at z = -h under an upright emitter: t = h / (-d_z) for d_z < 0 inside the quad,
    misses for d_z >= 0; the nadir channel (RN32(-pi/2), d_z = -1) hits at exactly t = h."""
    h = 1.5
    em = _em(elev=sg.full_sphere_elev(16), rays_per_channel=512)
    tris = sg.ground_quad(h, half=1000.0)
    res = oracle.cast([em], tris, want_t64=True)
    D = oracle.ray_table([em]).astype(np.float64)
    with np.errstate(divide="ignore"):
        t = np.where(D[:, 2] < 0, h / -D[:, 2], np.inf)
    x, y = t * D[:, 0], t * D[:, 1]
    inside = (D[:, 2] < 0) & (np.abs(x) <= 1000) & (np.abs(y) <= 1000)
    assert np.array_equal(_hits(res), inside)
    np.testing.assert_allclose(res["t64"][inside], t[inside], rtol=1e-12)
    assert np.all(res["t"][:512] == np.float32(h))          # channel 0 = nadir
    assert not _hits(res)[8 * 512:].any()                     # channels 8.. have d_z >= 0


def test_room_box_closed_form(oracle_lib):
    """Emitter inside an axis-aligned box: every ray hits, t = min over the 6 planes (two-sided)."""
    lo, hi = np.array([-2.0, -1.0, -1.5]), np.array([3.0, 4.0, 2.0])
    o = np.array([0.3, -0.2, 0.1], np.float32)
    rng = np.random.default_rng(11)
    f, r, u = sg.random_frame(rng)
    em = _em(origin=o, forward=f, right=r, up=u, elev=sg.full_sphere_elev(24), rays_per_channel=200)
    res = oracle.cast([em], sg.room_box(lo, hi), want_t64=True)
    D = oracle.ray_table([em]).astype(np.float64)
    o64 = o.astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        tp = np.where(D > 0, (hi - o64) / D, np.where(D < 0, (lo - o64) / D, np.inf))
    t = tp.min(axis=1)
    second = np.sort(tp, axis=1)[:, 1]
    clear = (second - t) > 1e-9 * t            # not within 1e-9 of a box edge/corner
    assert _hits(res).all()
    np.testing.assert_allclose(res["t64"], t, rtol=1e-12)
    face_axis = tp.argmin(axis=1)
    face_hi = D[np.arange(len(D)), face_axis] > 0
    # room_box face order: z-lo, z-hi, y-lo, y-hi, x-lo, x-hi (2 triangles each)
    face_idx = np.select([face_axis == 2, face_axis == 1, face_axis == 0], [0, 2, 4]) + face_hi.astype(int)
    assert np.array_equal(res["id"][clear] // 2, face_idx[clear])
    # all-hit count = 1 away from edges (each ray leaves a closed box exactly once)
    res2 = oracle.cast([em], sg.room_box(lo, hi), want_allhits=True)
    inner = clear & ((np.sort(np.abs(tp - t[:, None]) / t[:, None], axis=1)[:, 1]) > 1e-6)
    assert np.all(res2["allhits"][inner] >= 1)


def _point_in_tri_2d(p, a, b, c):
    def cr(o, x, y):
        return (x[..., 0] - o[..., 0]) * (y[..., 1] - o[..., 1]) - (x[..., 1] - o[..., 1]) * (y[..., 0] - o[..., 0])
    s1, s2, s3 = cr(a, b, p), cr(b, c, p), cr(c, a, p)
    inside = ((s1 >= 0) & (s2 >= 0) & (s3 >= 0)) | ((s1 <= 0) & (s2 <= 0) & (s3 <= 0))
    m = np.minimum(np.minimum(np.abs(s1), np.abs(s2)), np.abs(s3))
    return inside, m


def test_seam_triangle_wrap(oracle_lib):
    """North-star fixture (ii): triangle at x = -5 behind a 360 deg emitter straddles theta = +-pi:
    hits on rays i ~ 0 and i ~ chi-1 of the same channel; t = -5/d_x (2-D point-in-triangle)."""
    em = sg.c1_emitter()
    o = em.origin.astype(np.float64)
    tri = sg.seam_triangle(o)
    res = oracle.cast([em], tri, want_t64=True)
    D = oracle.ray_table([em]).astype(np.float64)
    with np.errstate(divide="ignore"):
        t = np.where(D[:, 0] < 0, -5.0 / D[:, 0], np.inf)
    P = np.stack([t * D[:, 1], t * D[:, 2]], -1)
    a, b, c = (np.array(v, np.float64) for v in ([-1, -1], [1, -1], [0, 1]))
    inside, m = _point_in_tri_2d(P, a, b, c)
    inside &= D[:, 0] < 0
    clear = m > 1e-9
    assert np.array_equal(_hits(res)[clear], inside[clear])
    np.testing.assert_allclose(res["t64"][inside], t[inside], rtol=1e-12)
    ch8 = _hits(res)[8 * 512:9 * 512]
    assert ch8[0] and ch8[511] and ch8[:9].all() and ch8[504:].all() and not ch8[100:400].any()
    assert res["t"][8 * 512] == 5.0     # ray (8, 0) is exactly -f


def test_d_max_straddler(oracle_lib):
    """0 < t <= D_max per ray: quad at x = 5 with D_max just below 5 -> no hits;
    D_max = 5.05 keeps exactly the rays with t <= 5.05."""
    base = sg.c1_emitter()
    tris = sg.quad_x5(base.origin.astype(np.float64))
    none = oracle.cast([sg.c1_emitter(max_range=4.99)], tris)
    assert not _hits(none).any()
    full = oracle.cast([sg.c1_emitter()], tris, want_t64=True)
    cut = oracle.cast([sg.c1_emitter(max_range=5.05)], tris)
    expect = _hits(full) & (full["t64"] <= np.float64(np.float32(5.05)))
    assert np.array_equal(_hits(cut), expect) and 0 < expect.sum() < _hits(full).sum()
    # closed interval: the centre ray has t = 5.0 exactly and D_max = 5.0 keeps it
    at = oracle.cast([sg.c1_emitter(max_range=5.0)], tris)
    g = 8 * 512 + 256
    assert at["id"][g] == 0 and at["t"][g] == 5.0 and _hits(at).sum() == 1


# --------------------------------------------------------- brute force, tiny --

def test_closest_and_tie_by_hand(oracle_lib):
    """Hand-enumerated: the closer of two triangles wins regardless of order; equal t -> smaller id;
    a triangle behind the emitter is never hit."""
    em = _em(elev=np.array([0.0], np.float32), rays_per_channel=4)   # ray i=2 is +x
    far = [[5, -1, -1], [5, 1, -1], [5, 0, 1]]
    near = [[3, -1, -1], [3, 1, -1], [3, 0, 1]]
    behind = [[-2, -1, -1], [-2, 1, -1], [-2, 0, 1]]
    for order, ids, exp_id in [([far, near], [0, 1], 1), ([near, far], [0, 1], 0)]:
        r = oracle.cast([em], np.array(order, np.float32), ids=np.array(ids))
        assert r["t"][2] == 3.0 and r["id"][2] == exp_id
    r = oracle.cast([em], np.array([far, far], np.float32), ids=np.array([7, 3]))
    assert r["t"][2] == 5.0 and r["id"][2] == 3
    r = oracle.cast([em], np.array([behind], np.float32))
    assert r["id"][2] == -1 and r["id"][0] == 0 and r["t"][0] == 2.0   # ray 0 is -x


def test_faces_modes(oracle_lib):
    """one-sided modes keep a hit iff sign(d.N) is + (mode 1) or - (mode 2).
    quad_x5 has N = +x for both triangles, rays travel +x -> d.N > 0."""
    em = sg.c1_emitter()
    tris = sg.quad_x5(em.origin.astype(np.float64))
    two = oracle.cast([em], tris, faces=0)
    pos = oracle.cast([em], tris, faces=1)
    neg = oracle.cast([em], tris, faces=2)
    assert np.array_equal(two["id"], pos["id"]) and _hits(two).sum() > 0
    assert not _hits(neg).any()
    flipped = tris[:, ::-1, :].copy()
    assert np.array_equal(_hits(oracle.cast([em], flipped, faces=2)), _hits(two))


def test_threads_and_permutation_invariance(oracle_lib):
    """Per-ray independence and the min-lattice: results do not depend on thread count or on
    triangle order (ids travel with triangles)."""
    ems, tris = sg.random_scene(5, n_tris=150)
    a = oracle.cast(ems, tris, threads=1, want_t64=True)
    b = oracle.cast(ems, tris, threads=5, want_t64=True)
    assert np.array_equal(a["t64"], b["t64"]) and np.array_equal(a["id"], b["id"])
    perm = np.random.default_rng(0).permutation(len(tris))
    c = oracle.cast(ems, tris[perm], ids=perm.astype(np.int32), want_t64=True)
    assert np.array_equal(a["t64"], c["t64"]) and np.array_equal(a["id"], c["id"])


def test_sampled_rays_match_full(oracle_lib):
    """Sampled-ray mode (used at full scale) returns exactly the full-frame rows."""
    ems, tris = sg.random_scene(9, n_tris=120)
    full = oracle.cast(ems, tris, want_t64=True, want_allhits=True)
    rays = np.random.default_rng(1).choice(len(full["t"]), 200, replace=False)
    s = oracle.cast(ems, tris, rays=rays, want_t64=True, want_allhits=True)
    assert np.array_equal(s["t64"], full["t64"][rays]) and np.array_equal(s["id"], full["id"][rays])
    assert np.array_equal(s["allhits"], full["allhits"][rays])


def test_allhits_translation_of_closed_form(oracle_lib):
    """Closed form for all-hit counts: a stack of k parallel quads in front of the emitter is hit
    k times by every ray through all of them."""
    em = _em(elev=np.array([-0.05, 0.0, 0.05], np.float32), rays_per_channel=64)
    quads = np.concatenate([sg.quad_x5((-float(k), 0, 0)) for k in range(3)], 0)   # x = 5, 4, 3
    r = oracle.cast([em], quads, want_allhits=True, want_t64=True)
    D = oracle.ray_table([em]).astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        inside5 = (D[:, 0] > 0) & (np.abs(5 * D[:, 1] / D[:, 0]) < 1 - 1e-9) & (np.abs(5 * D[:, 2] / D[:, 0]) < 1 - 1e-9)
    assert inside5.sum() > 0
    assert np.all(r["allhits"][inside5] >= 3)
    np.testing.assert_allclose(r["t64"][inside5], 3.0 / D[inside5, 0], rtol=1e-12)


def test_comparator_self_and_perturbed(oracle_lib):
    """The comparator accepts the oracle against itself and flags a wrong id / distance / miss."""
    ems, tris = sg.random_scene(2, n_tris=100)
    ref = oracle.cast(ems, tris, want_t64=True)
    rep = oracle.compare(ems, tris, ref["t"], ref["id"], ref)
    assert rep["passed"] and rep["disagree"] == 0
    hit_rays = np.nonzero(ref["id"] >= 0)[0]
    assert len(hit_rays) > 10
    t = ref["t"].copy()
    i = ref["id"].copy()
    t[hit_rays[0]] *= 1.001                     # distance off by 1e-3
    i[hit_rays[1]] = -1
    t[hit_rays[1]] = np.inf                     # a dropped hit (not near an edge in general)
    rep = oracle.compare(ems, tris, t, i, ref)
    assert not rep["passed"] and rep["kinds"]["dist"] == 1 and rep["kinds"]["gpu_miss"] == 1


def test_perturbed_azimuth_table(oracle_lib):
    """Noise model: a pre-stored per-ray azimuth table theta*_i replaces the grid
    angle of ray i.  Pins: the azimuth of every direction (in the frame) equals theta*_i within the fp32
    rounding of d, theta* = 0 gives f exactly, and a table equal to the grid reproduces the grid rays."""
    f, r, u = np.float32([1, 0, 0]), np.float32([0, -1, 0]), np.float32([0, 0, 1])
    az = sg.perturbed_azimuths(64, 360, seed=3)
    az[10] = 0.0
    em = _em(forward=f, right=r, up=u, elev=np.array([-0.3, 0.0, 0.4], np.float32), rays_per_channel=64)
    em.ray_azimuth = az
    tab = oracle.ray_table([em]).astype(np.float64)
    x_f, x_r = tab @ f.astype(np.float64), tab @ r.astype(np.float64)
    got = np.arctan2(x_r, x_f).reshape(3, 64)
    np.testing.assert_allclose(got, np.broadcast_to(az.astype(np.float64), (3, 64)), atol=3e-7)
    np.testing.assert_array_equal(tab[64 + 10], f)            # channel phi = 0, theta* = 0 -> f
    grid = _em(elev=np.array([0.2], np.float32), rays_per_channel=8, hfov_deg=180)
    g2 = _em(elev=np.array([0.2], np.float32), rays_per_channel=8, hfov_deg=180)
    g2.ray_azimuth = np.array([-(8 // 2) * (math.pi / 8) + i * (math.pi / 8) for i in range(8)], np.float64).astype(np.float32)
    a, b = oracle.ray_table([grid]), oracle.ray_table([g2])
    np.testing.assert_allclose(a, b, atol=2e-7)
