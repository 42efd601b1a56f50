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
    # a second emitter (180 deg, 0.75 m higher): its rays occupy g in [O_1, O_2) = [8192, 8192 + 12*300)
    # and follow the same closed form with its own height (PAPER.md:760-765 global index)
    em2 = _em(origin=(3.0, -2.0, 0.75), elev=sg.vlp16_elev()[:12], rays_per_channel=300, hfov_deg=180)
    res2 = oracle.cast([em, em2], tris, want_t64=True)
    D2 = oracle.ray_table([em2]).astype(np.float64)
    with np.errstate(divide="ignore"):
        t2 = np.where(D2[:, 2] < 0, (h + 0.75) / -D2[:, 2], np.inf)
    assert np.array_equal(res2["t64"][:8192], res["t64"])
    down = D2[:, 2] < 0
    assert down.sum() > 1000 and np.array_equal(_hits(res2)[8192:], down)
    np.testing.assert_allclose(res2["t64"][8192:][down], t2[down], rtol=1e-12)


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
    # all-hit count: a ray leaves a closed box exactly once, so away from face edges and from the face
    # diagonals (where two closed triangles share the point) it hits exactly ONE triangle.
    res2 = oracle.cast([em], sg.room_box(lo, hi), want_allhits=True)
    rows = np.arange(len(D))
    P = o64[None, :] + t[:, None] * D                              # exit point (closed form)
    ax_b = np.array([1, 0, 0])[face_axis]                         # the face's two in-plane axes
    ax_c = np.array([2, 2, 1])[face_axis]
    s_b = (P[rows, ax_b] - lo[ax_b]) / (hi - lo)[ax_b]            # normalised in-plane coordinates
    s_c = (P[rows, ax_c] - lo[ax_c]) / (hi - lo)[ax_c]
    # room_box splits every face (a, b, c, d) into (a, b, c) + (a, c, d): the diagonal is s_b == s_c
    inner = (np.minimum.reduce([s_b, 1 - s_b, s_c, 1 - s_c]) > 1e-6) & (np.abs(s_b - s_c) > 1e-6)
    assert inner.sum() > 0.9 * len(D)
    assert np.all(res2["allhits"][inner] == 1)
    assert np.all(res2["allhits"] >= 1)


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
    # t > 0 strictly -- a triangle through the origin meets every crossing ray at t = 0
    through = np.array([[[0, -1, -1], [0, 1, -1], [0, 0, 1]]], np.float32)   # plane x = 0 contains o
    r = oracle.cast([em], through)
    assert np.all(r["id"] == -1)
    # closed triangle: the ray +x meets (5, 0, 0), which lies exactly on the v1-v2 edge (u = v = 1/2,
    # u + v = 1) of this triangle -- exact in fp64 for these integer vertices, so it must hit at t = 5
    edge = np.array([[[5, -1, -1], [5, 1, -1], [5, -1, 1]]], np.float32)
    ok, t, u, v, _ = oracle.mt([0, 0, 0], [1, 0, 0], *edge[0])
    assert ok and u == 0.5 and v == 0.5
    r = oracle.cast([em], edge)
    assert r["id"][2] == 0 and r["t"][2] == 5.0


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
    """Closed form for all-hit counts: quads at x = 5, 4, 3 (|y|, |z| <= 1 each) in front of the emitter.
    A ray with slopes (y/x, z/x) = (a, b) crosses the quad at x = k iff k max(|a|, |b|) <= 1, so away from
    the quads' borders and their shared diagonals its all-hit count is EXACTLY #{k : k max(|a|,|b|) < 1}
    (3 inside the x = 5 cone, 1 or 2 in the rings between); behind the emitter it is 0.  The centre ray
    (1, 0, 0) lies on all three shared diagonals: both closed triangles of each quad -> exactly 6."""
    em = _em(elev=np.array([-0.3, -0.22, -0.1, 0.0, 0.05, 0.21, 0.3], np.float32), rays_per_channel=256)
    quads = np.concatenate([sg.quad_x5((-float(k), 0, 0)) for k in range(3)], 0)   # x = 5, 4, 3
    r = oracle.cast([em], quads, want_allhits=True, want_t64=True)
    D = oracle.ray_table([em]).astype(np.float64)
    fwd = D[:, 0] > 0
    with np.errstate(divide="ignore", invalid="ignore"):
        a, b = D[:, 1] / D[:, 0], D[:, 2] / D[:, 0]
    m = np.maximum(np.abs(a), np.abs(b))
    expect = np.where(fwd, sum((k * m < 1).astype(int) for k in (3, 4, 5)), 0)
    clear = ~fwd | ((np.min([np.abs(k * m - 1) for k in (3, 4, 5)], axis=0) > 1e-9) & (np.abs(a - b) > 1e-9))
    assert set(np.unique(expect[clear])) == {0, 1, 2, 3}
    assert np.array_equal(r["allhits"][clear], expect[clear].astype(np.uint32))
    inside5 = clear & (expect == 3)
    np.testing.assert_allclose(r["t64"][inside5], 3.0 / D[inside5, 0], rtol=1e-12)
    g = 3 * 256 + 128                                              # channel phi = 0, theta = 0: d = (1, 0, 0)
    assert np.array_equal(D[g], [1.0, 0.0, 0.0])
    assert r["allhits"][g] == 6 and r["t"][g] == 3.0 and r["id"][g] == 4   # tie on x = 3 -> smaller id


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


# ------------------------------------------------- comparator, constructed --

def _tri_with_margin(p, margin):
    """Right triangle in the plane x = p_x whose barycentric margin min(u, v, 1-u-v) at the point p is
    `margin` (u = margin along the +y leg, v = 0.5 along the +z leg): v0 = p - (0, 2 margin, 1), legs
    of length 2.  p lies inside for margin > 0 (fp32 vertex rounding moves u by <= 2e-8)."""
    v0 = np.array([p[0], p[1] - 2.0 * margin, p[2] - 1.0])
    return np.array([[v0, v0 + [0, 2, 0], v0 + [0, 0, 2]]]).astype(np.float32)


def _fake(ref):
    return ref["t"].copy(), ref["id"].copy()


def test_comparator_excusal_boundary(oracle_lib):
    """SURVEY 8(c) comparator, excusal branch: a dropped hit is excused iff the oracle's triangle has
    |margin| <= 1e-6 for that ray.  Constructed cases around the threshold (margins 5e-7 -> excused,
    2e-6 and 1e-3 -> unexcused) and the exact shared-diagonal ray of quad x = 5 (margin 0 -> excused)."""
    em = _em(elev=np.array([-0.07, 0.0, 0.09], np.float32), rays_per_channel=64)
    D = oracle.ray_table([em]).astype(np.float64)
    g = 2 * 64 + 33                                      # phi = 0.09, theta = dtheta: a generic ray
    p = 5.0 * D[g] / D[g, 0]
    for margin, excused in [(5e-7, True), (2e-6, False), (1e-3, False)]:
        tri = _tri_with_margin(p, margin)
        ref = oracle.cast([em], tri, want_t64=True)
        assert ref["id"][g] == 0
        ok, t, u, v, hit = oracle.ray_tri([em], g, tri[0])
        assert hit and abs(min(u, v, 1 - u - v) - margin) < 0.05 * margin
        t_g, i_g = _fake(ref)
        t_g[g], i_g[g] = np.inf, -1                      # "GPU" drops the hit
        rep = oracle.compare([em], tri, t_g, i_g, ref)
        assert rep["disagree"] == 1 and rep["kinds"]["gpu_miss"] == 1
        assert rep["excused"] == int(excused) and rep["unexcused"] == int(not excused)
        assert not rep["passed"] or excused
        # the all-hits excusal counter agrees: the triangle is within 1e-6 of its boundary iff excused
        assert oracle.near_edge_count([em], g, tri) == int(excused)
        # the mirror case: the GPU reports a hit on a triangle the oracle misses (ray just outside)
        out = _tri_with_margin(p, -margin)
        ref2 = oracle.cast([em], out, want_t64=True)
        assert ref2["id"][g] == -1
        t_g, i_g = _fake(ref2)
        t_g[g], i_g[g] = np.float32(t), 0
        rep = oracle.compare([em], out, t_g, i_g, ref2)
        assert rep["kinds"]["gpu_extra"] == 1 and rep["excused"] == int(excused)
    # the shared diagonal of quad x = 5: the centre ray (1, 0, 0) hits both closed triangles (u = 0 in T0)
    em = sg.c1_emitter()
    tris = sg.quad_x5(em.origin.astype(np.float64))
    ref = oracle.cast([em], tris, want_t64=True)
    g = 8 * 512 + 256
    t_g, i_g = _fake(ref)
    t_g[g], i_g[g] = np.inf, -1
    rep = oracle.compare([em], tris, t_g, i_g, ref)
    assert rep["excused"] == 1 and rep["unexcused"] == 0 and rep["kinds"]["gpu_miss"] == 1
    assert not rep["passed"]                             # 8191 / 8192 = 99.988 % < 99.999 %
    assert oracle.near_edge_count([em], g, tris) == 2 and oracle.near_edge_count([em], g - 6, tris) == 0
    # ... while the same excused drop among 103,424 rays passes (1 - 1/103424 >= 99.999 %) and an
    # unexcused one (a 1e-4 relative distance error) does not
    elev = np.concatenate([np.linspace(-0.3, -0.006, 50), [0.0], np.linspace(0.006, 0.3, 50)]).astype(np.float32)
    big = _em(origin=(0, 0, 0), elev=elev, rays_per_channel=1024)
    tris = sg.quad_x5()
    ref = oracle.cast([big], tris, want_t64=True)
    g = 50 * 1024 + 512                                  # phi = 0, theta = 0: d = (1, 0, 0), the diagonal
    assert np.array_equal(oracle.ray_table([big])[g], [1, 0, 0]) and ref["id"][g] == 0
    t_g, i_g = _fake(ref)
    t_g[g], i_g[g] = np.inf, -1
    rep = oracle.compare([big], tris, t_g, i_g, ref)
    assert rep["rays"] == 103424 and rep["excused"] == 1 and rep["passed"]
    t_g, i_g = _fake(ref)
    t_g[g] = np.float32(ref["t64"][g] * (1 + 1e-4))
    rep = oracle.compare([big], tris, t_g, i_g, ref)
    assert rep["disagree"] == 1 and rep["unexcused"] == 1 and not rep["passed"]


def test_comparator_near_tie_and_swaps(oracle_lib):
    """SURVEY 8(c) comparator, near-tie branch.  (a) Two identical triangles (ids 0, 1): the oracle
    takes id 0; a GPU answer of id 1 at the same t is a near-tie (agrees).  (b) Two parallel quads 2e-4
    apart (relative): reporting the farther id is NOT a near-tie (its fp64 t is 2e-4 > 1e-5 away) and
    not excused.  (c) An id whose triangle the ray misses entirely: unexcused.  (d) A distance off by
    2e-5 relative with the right id: a 'dist' disagreement, never excused."""
    em = _em(elev=np.array([0.0, 0.05], np.float32), rays_per_channel=64)
    q = sg.quad_x5()
    twin = np.concatenate([q[:1], q[:1], q[1:]], 0)     # ids 0 and 1 identical, id 2 the other half
    ref = oracle.cast([em], twin, want_t64=True)
    hit0 = np.nonzero(ref["id"] == 0)[0]
    assert len(hit0) >= 3
    g = int(hit0[0])
    t_g, i_g = _fake(ref)
    i_g[g] = 1
    rep = oracle.compare([em], twin, t_g, i_g, ref)
    assert rep["passed"] and rep["near_ties"] == 1 and rep["disagree"] == 0
    # (b) parallel quads at x = 5 and x = 5.001
    two = np.concatenate([q, sg.quad_x5((0.001, 0, 0))], 0)  # ids 0, 1 near; 2, 3 far
    ref = oracle.cast([em], two, want_t64=True)
    g = int(np.nonzero(ref["id"] == 0)[0][0])
    t_g, i_g = _fake(ref)
    i_g[g] = 2
    rep = oracle.compare([em], two, t_g, i_g, ref)
    assert rep["near_ties"] == 0 and rep["kinds"]["id"] == 1 and rep["unexcused"] == 1
    # (c) swap to a triangle behind the emitter
    scene = np.concatenate([q, sg.seam_triangle()], 0)   # id 2 is at x = -5
    ref = oracle.cast([em], scene, want_t64=True)
    g = int(np.nonzero(ref["id"] == 0)[0][0])
    t_g, i_g = _fake(ref)
    i_g[g] = 2
    rep = oracle.compare([em], scene, t_g, i_g, ref)
    assert rep["near_ties"] == 0 and rep["kinds"]["id"] == 1 and rep["unexcused"] == 1
    # (d) distance tolerance 1e-5 relative: 2e-5 fails, 5e-6 passes
    t_g, i_g = _fake(ref)
    t_g[g] = np.float32(ref["t64"][g] * (1 + 2e-5))
    rep = oracle.compare([em], scene, t_g, i_g, ref)
    assert rep["kinds"]["dist"] == 1 and rep["unexcused"] == 1
    t_g[g] = np.float32(ref["t64"][g] * (1 + 5e-6))
    assert oracle.compare([em], scene, t_g, i_g, ref)["passed"]
    # (e) sentinels: a miss must carry (+inf, -1); a finite distance with id -1 is a disagreement
    t_g, i_g = _fake(ref)
    miss = int(np.nonzero(ref["id"] == -1)[0][0])
    t_g[miss] = 3.0
    rep = oracle.compare([em], scene, t_g, i_g, ref)
    assert rep["kinds"]["sentinel"] == 1 and rep["unexcused"] == 1


# ------------------------------------------------- grazing (north star iii) --

def test_grazing_edge_planes(oracle_lib):
    """SURVEY 8(c) hand-built (iii): rays within ~1e-7 rad of an edge plane.  A vertical edge in the
    plane x = 5 at y = y_e is crossed by ray d at y = 5 d_y / d_x (closed form); the triangle lies on
    the y <= y_e side, so the ray hits iff 5 d_y / d_x <= y_e.  Edges placed 5e-7 m (1e-7 rad at 5 m)
    on either side of each aimed point: exactly the inside ones hit, at t = 5 / d_x."""
    em = _em(elev=np.array([-0.2, 0.0, 0.13], np.float32), rays_per_channel=128)
    D = oracle.ray_table([em]).astype(np.float64)
    gs = [g for g in range(len(D)) if D[g, 0] > 0.9]
    for g in gs[::7]:
        y = 5.0 * D[g, 1] / D[g, 0]
        z = 5.0 * D[g, 2] / D[g, 0]
        for off in (5e-7, -5e-7):
            ye = np.float32(y + off)
            tri = np.array([[[5, ye, z - 2], [5, ye, z + 2], [5, ye - 3, z]]], np.float32)
            r = oracle.cast([em], tri, rays=np.array([g]), want_t64=True)
            inside = y <= np.float64(ye)
            assert inside == (off > 0)
            assert (r["id"][0] == 0) == inside, (g, off)
            if inside:
                assert abs(r["t64"][0] - 5.0 / D[g, 0]) <= 1e-12 * r["t64"][0]


def test_grazing_incidence_and_flush_plane(oracle_lib):
    """SURVEY 8(c) hand-built (iii): triangles at |cos| < 1e-3 to the ray.  Plane z - 1.5 = 2^-11 (x - 10)
    (exact fp32 vertices), emitter at (0, 0, 1.5): every horizontal ray (phi = 0: d_z = 0 exactly) meets
    it at x = 10, so t = 10 / d_x and it hits iff -1 <= 10 d_y / d_x <= 3 (the triangle's cross-section
    at x = 10); |d.n| = 2^-11 / sqrt(1 + 2^-22) < 1e-3.  Then the paper's absolute plane guard
    (PAPER.md:2471-2474 skips planes within 1e-4 m of o): a ground plane 2^-15 m below the emitter is
    still hit by every downward ray, at t = 2^-15 / -d_z (the plain definition has no such guard)."""
    s = 2.0 ** -11
    tri = np.array([[[2, -1, 1.5 - 8 * s], [18, -1, 1.5 + 8 * s], [10, 3, 1.5]]], np.float32)
    assert np.array_equal(tri.astype(np.float64), np.array([[[2, -1, 1.5 - 8 * s], [18, -1, 1.5 + 8 * s], [10, 3, 1.5]]]))
    em = _em(origin=(0, 0, 1.5), elev=np.array([-0.4, 0.0, 0.4], np.float32), rays_per_channel=720)
    D = oracle.ray_table([em]).astype(np.float64)
    r = oracle.cast([em], tri, want_t64=True)
    row = slice(720, 1440)                                   # the phi = 0 channel
    assert np.all(D[row, 2] == 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        y = 10.0 * D[row, 1] / D[row, 0]
    fwd = D[row, 0] > 0
    inside = fwd & (y >= -1) & (y <= 3)
    clear = ~fwd | ((np.abs(y + 1) > 1e-9) & (np.abs(y - 3) > 1e-9))
    assert inside.sum() > 20
    assert np.array_equal((r["id"][row] == 0)[clear], inside[clear])
    np.testing.assert_allclose(r["t64"][row][inside & clear], 10.0 / D[row][inside & clear, 0], rtol=1e-12)
    ncos = s / math.sqrt(1 + s * s)
    assert ncos < 1e-3
    # flush plane
    h = 2.0 ** -15
    em2 = _em(origin=(0, 0, 1.5), elev=sg.full_sphere_elev(16), rays_per_channel=256)
    ground = sg.ground_quad(h, half=100.0, offset=(0, 0, 1.5))
    assert np.all(ground[..., 2] == np.float32(1.5 - h))
    r = oracle.cast([em2], ground, want_t64=True)
    D = oracle.ray_table([em2]).astype(np.float64)
    down = D[:, 2] < -1e-3
    assert np.all(r["id"][down] >= 0)
    np.testing.assert_allclose(r["t64"][down], h / -D[down, 2], rtol=1e-9)
    assert np.all(r["id"][D[:, 2] >= 0] == -1)


def test_mutations_named_by_the_review_are_killed(tmp_path):
    """tools/mutate_oracle.py on the slips that survived the round-1 pins (all-hit count before the
    accept test, BARY_EPS = 1e9) plus the near-tie branch: each must now fail a pin.  The full list
    (28 mutations) is run by the tool itself (profiles/r02_oracle_mutations.md)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "mutate_oracle.py"), "--out",
                        str(tmp_path / "m.md"), "--only", "count before,BARY_EPS = 1e9,no near-tie"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "3/3 killed" in r.stdout
