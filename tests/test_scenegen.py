"""Input generators (no method arithmetic): sizes and seeding of the SURVEY 8(d) recipes."""
import numpy as np

import scenegen as sg


def test_car_triangle_count():
    """388 x 388 superellipsoid grid -> 2*388*388 = 301,088 triangles (PAPER.md:940 ~300,603)."""
    c = sg.car()
    assert c.shape == (301088, 3, 3) and c.dtype == np.float32
    ext = c.reshape(-1, 3).max(0) - c.reshape(-1, 3).min(0)
    np.testing.assert_allclose(ext, [4.57, 2.28, 1.08], rtol=1e-3)
    v, f = sg.car_mesh()
    assert v.shape == (389 * 389, 3) and f.shape == (301088, 3) and f.dtype == np.int32
    assert np.array_equal(v[f], c)                      # the soup is the indexed mesh, same order
    assert np.array_equal(f[0], [0, 389, 390]) and np.array_equal(f[1], [0, 390, 1])   # quad pairs adjacent


def test_plant_exact_count_and_area():
    t = sg.plant(50000, bbox=(60.0, 30.0, 20.0), seed=3)
    assert t.shape == (50000, 3, 3)
    e1 = t[:, 1] - t[:, 0]
    e2 = t[:, 2] - t[:, 0]
    area = 0.5 * np.linalg.norm(np.cross(e1.astype(np.float64), e2.astype(np.float64)), axis=1)
    assert 0.01 < area.mean() < 0.2       # ~384 cm^2 recipe
    assert np.array_equal(t, sg.plant(50000, bbox=(60.0, 30.0, 20.0), seed=3))


def test_c1_scene_and_emitter():
    s = sg.c1_scene()
    assert s.shape == (2000, 3, 3)
    e = sg.c1_emitter()
    assert e.n_rays == 16 * 512
    el = sg.full_sphere_elev(16)
    assert el[0] == np.float32(-np.pi / 2) and np.all(np.diff(el) > 0)


def test_pose_and_swd_seeded():
    a = sg.pose_instances(3, (10, 10, 10), seed=1, frame=2)
    b = sg.pose_instances(3, (10, 10, 10), seed=1, frame=2)
    assert all(np.array_equal(x.rotation, y.rotation) for x, y in zip(a, b))
    R = a[0].rotation
    np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-12)
    tris = sg.random_triangles(np.random.default_rng(0), 50, (0, 0, 0), 5.0)
    w = sg.swd(tris, (10, 10, 10), seed=1, frame=0)
    # rigid per-triangle scatter: edge vectors preserved
    np.testing.assert_allclose(w[:, 1] - w[:, 0], tris[:, 1] - tris[:, 0], atol=1e-4)


def test_indexed_frame_reproduces_the_soup():
    """The bench's indexed layout (trivial static indices + shared car vertices) is the same list
    of triangles as the workload soup, bit for bit."""
    w = sg.workload("C2", static_scale=0.02, n_cars=2)
    v, idx = sg.indexed_frame(w)
    assert idx.shape == (3 * len(w["tris"]),) and v.shape[0] == 3 * w["n_static"] + 2 * 389 * 389
    assert np.array_equal(v[idx].reshape(-1, 3, 3), w["tris"])


def test_pose_f32_matches_definition():
    """scenegen.apply_pose_f32 is grca_update_instances' documented fp32 order (include/grca.h): per row,
    ((m0 x + m1 y) + m2 z) + m3 with every product and sum rounded; it agrees with the fp64 pose to fp32
    accuracy, and equals an element-by-element Python-float32 evaluation bit for bit."""
    import numpy as np
    import scenegen as sg

    v, f = sg.car_mesh(12, 12)
    p = sg.pose_instances(1, (50.0, 40.0, 10.0), seed=3, frame=2)[0]
    M = sg.pose_matrix(p)
    a = sg.apply_pose_f32(v, M)
    b = sg.apply_pose(v, p)
    np.testing.assert_allclose(a, b, rtol=0, atol=2e-5 * (1 + np.abs(b).max()))
    f32 = np.float32
    for k in (0, 7, len(v) - 1):
        x, y, z = (f32(c) for c in v[k])
        for r in range(3):
            want = f32(f32(f32(f32(M[r, 0] * x) + f32(M[r, 1] * y)) + f32(M[r, 2] * z)) + M[r, 3])
            assert a[k, r] == want
