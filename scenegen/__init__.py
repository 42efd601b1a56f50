"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds *inputs only*: emitter descriptions, triangle soups and the
workload recipes of SURVEY.md 8(d).  It contains none of the method's
arithmetic (no ray directions, no culling, no intersection), so both the
oracle (oracle/) and the product (paper_2605_10457_b200/) may consume it
without sharing code with each other.

Recipes:
  * ``full_sphere_elev(g)``   -- the paper's uniform full-sphere channel grid
    phi_j = -pi/2 + j*pi/g, rounded to fp32.
  * ``vlp16_elev()``          -- a non-uniform 16-channel table -15..+15 deg.
  * ``plant(...)``            -- ground grid + seeded tessellated boxes,
    mean triangle area ~ 384 cm^2.
  * ``car(...)``              -- superellipsoid "sports car", 388x388 grid ->
    301,088 triangles, 4.57 x 2.28 x 1.08 m.
  * ``pose_instances(...)``   -- motion f.i: per-frame uniform position,
    uniform rotation, per-axis scale U[0.001, 30] (Q18).
  * ``swd(...)``              -- per-triangle rigid scatter of dynamic
    triangles into the world box.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

INF = float("inf")


@dataclass
class Emitter:
    """One spinning LiDAR (ray origin).  All vectors are fp32 world space.

    PAPER.md:411-435 (frame f,r,u; grid); north star ABI ``grca_emitter``.
    """

    origin: Sequence[float]
    forward: Sequence[float] = (1.0, 0.0, 0.0)
    right: Sequence[float] = (0.0, -1.0, 0.0)
    up: Sequence[float] = (0.0, 0.0, 1.0)
    elev: np.ndarray = field(default_factory=lambda: full_sphere_elev(16))
    rays_per_channel: int = 512
    hfov_deg: int = 360
    max_range: float = INF
    ray_azimuth: Optional[np.ndarray] = None   # noise model: pre-stored perturbed azimuths (chi,)

    def __post_init__(self):
        self.origin = np.asarray(self.origin, dtype=np.float32).reshape(3)
        self.forward = np.asarray(self.forward, dtype=np.float32).reshape(3)
        self.right = np.asarray(self.right, dtype=np.float32).reshape(3)
        self.up = np.asarray(self.up, dtype=np.float32).reshape(3)
        self.elev = np.ascontiguousarray(np.asarray(self.elev, dtype=np.float32))

    @property
    def n_channels(self) -> int:
        return int(self.elev.shape[0])

    @property
    def n_rays(self) -> int:
        return self.n_channels * int(self.rays_per_channel)


def n_rays_total(emitters: Sequence[Emitter]) -> int:
    return int(sum(e.n_rays for e in emitters))


def full_sphere_elev(n_channels: int) -> np.ndarray:
    """phi_j = phi0 + j*dphi with dphi = pi/g, phi0 = -floor(g/2)*dphi.

    For even g this is -pi/2 + j*pi/g; channel 0 is the nadir.
    """
    g = int(n_channels)
    dphi = math.pi / g
    phi0 = -(g // 2) * dphi
    return np.array([phi0 + j * dphi for j in range(g)], dtype=np.float64).astype(np.float32)


def perturbed_azimuths(chi: int, hfov_deg: int, seed: int, frac: float = 0.45) -> np.ndarray:
    """Noise-model input: per-ray azimuths theta*_i = theta_i + U(-frac, frac) dtheta
    around the nominal scan pattern theta_i = -floor(chi/2) dtheta + i dtheta (frac < 0.5: no ray
    crosses its neighbour), rounded to fp32."""
    rng = np.random.default_rng([int(seed), 0xA21])
    H = 2 * math.pi if hfov_deg == 360 else math.pi
    dth = H / chi
    th = np.array([-(chi // 2) * dth + i * dth for i in range(chi)])
    return (th + rng.uniform(-frac, frac, size=chi) * dth).astype(np.float32)


def perturbed_elev(elev: np.ndarray, seed: int, frac: float = 0.3) -> np.ndarray:
    """Noise-model input: per-channel perturbed elevations phi*_j, each moved by at
    most frac of its gap to the neighbours (order kept), clipped to [-RN32(pi/2), RN32(pi/2)]."""
    rng = np.random.default_rng([int(seed), 0xE1E])
    e = np.asarray(elev, dtype=np.float64)
    gaps = np.diff(e)
    lo = np.concatenate([[gaps[0] if len(gaps) else 0.01], gaps])
    hi = np.concatenate([gaps, [gaps[-1] if len(gaps) else 0.01]])
    step = np.minimum(lo, hi) * frac
    out = e + rng.uniform(-1, 1, size=e.shape) * step
    lim = float(np.float32(math.pi / 2))
    return np.clip(out, -lim, lim).astype(np.float32)


def vlp16_elev() -> np.ndarray:
    """VLP-16-like table: -15..+15 degrees in 2 degree steps (non-uniform test case)."""
    return np.radians(np.arange(-15.0, 15.0 + 1e-9, 2.0)).astype(np.float32)


def yaw_frame(yaw: float):
    """Level frame (u = +z) rotated by yaw about +z; r is f rotated -90 deg (clockwise from above)."""
    c, s = math.cos(yaw), math.sin(yaw)
    f = np.array([c, s, 0.0], dtype=np.float64)
    r = np.array([s, -c, 0.0], dtype=np.float64)
    u = np.array([0.0, 0.0, 1.0])
    return f.astype(np.float32), r.astype(np.float32), u.astype(np.float32)


def random_frame(rng: np.random.Generator):
    """A random orthonormal (f, r, u) frame, rounded to fp32."""
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    R = _quat_to_mat(q)
    return (R[:, 0].astype(np.float32), R[:, 1].astype(np.float32), R[:, 2].astype(np.float32))


def _quat_to_mat(q) -> np.ndarray:
    w, x, y, z = q
    return np.array(
        [
            [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
            [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
            [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
        ]
    )


# --------------------------------------------------------------------------
# Hand-built fixtures (SURVEY 8c "What pins each part", north star)
# --------------------------------------------------------------------------

def quad_x5(offset=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Axis-aligned square x = 5, |y|,|z| <= 1 as two triangles sharing the (-1,-1)-(1,1) diagonal."""
    o = np.asarray(offset, dtype=np.float64)
    t = np.array(
        [
            [[5, -1, -1], [5, 1, -1], [5, 1, 1]],
            [[5, -1, -1], [5, 1, 1], [5, -1, 1]],
        ],
        dtype=np.float64,
    )
    return (t + o).astype(np.float32)


def seam_triangle(offset=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Triangle behind a 360 deg emitter straddling the azimuth wrap theta = +-pi."""
    o = np.asarray(offset, dtype=np.float64)
    t = np.array([[[-5, -1, -1], [-5, 1, -1], [-5, 0, 1]]], dtype=np.float64)
    return (t + o).astype(np.float32)


def ground_quad(h: float, half: float = 1000.0, offset=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Large square at z = -h (relative to offset) as two triangles."""
    o = np.asarray(offset, dtype=np.float64)
    z = -h
    t = np.array(
        [
            [[-half, -half, z], [half, -half, z], [half, half, z]],
            [[-half, -half, z], [half, half, z], [-half, half, z]],
        ],
        dtype=np.float64,
    )
    return (t + o).astype(np.float32)


def room_box(lo, hi) -> np.ndarray:
    """Closed axis-aligned box [lo, hi] as 12 triangles."""
    x0, y0, z0 = lo
    x1, y1, z1 = hi
    P = np.array(
        [[x0, y0, z0], [x1, y0, z0], [x1, y1, z0], [x0, y1, z0],
         [x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]], dtype=np.float64)
    faces = [(0, 1, 2, 3), (4, 5, 6, 7), (0, 1, 5, 4), (3, 2, 6, 7), (0, 3, 7, 4), (1, 2, 6, 5)]
    tris = []
    for a, b, c, d in faces:
        tris.append([P[a], P[b], P[c]])
        tris.append([P[a], P[c], P[d]])
    return np.array(tris, dtype=np.float64).astype(np.float32)


def grid_mesh(nx: int, ny: int, x0, y0, x1, y1, z: float) -> np.ndarray:
    """Horizontal tessellated rectangle (2*nx*ny triangles) at height z."""
    xs = np.linspace(x0, x1, nx + 1)
    ys = np.linspace(y0, y1, ny + 1)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    Z = np.full_like(X, z)
    P = np.stack([X, Y, Z], -1)
    a = P[:-1, :-1].reshape(-1, 3)
    b = P[1:, :-1].reshape(-1, 3)
    c = P[1:, 1:].reshape(-1, 3)
    d = P[:-1, 1:].reshape(-1, 3)
    t1 = np.stack([a, b, c], 1)
    t2 = np.stack([a, c, d], 1)
    return np.concatenate([t1, t2], 0).astype(np.float32)


def random_triangles(rng: np.random.Generator, n: int, center, half_extent: float,
                     edge_lo: float = 0.02, edge_hi: float = 3.0) -> np.ndarray:
    """n random triangles, centroids uniform in a cube, edge lengths log-uniform [edge_lo, edge_hi]."""
    c = np.asarray(center, dtype=np.float64) + rng.uniform(-half_extent, half_extent, size=(n, 3))
    size = np.exp(rng.uniform(math.log(edge_lo), math.log(edge_hi), size=(n, 1, 1)))
    dirs = rng.normal(size=(n, 3, 3))
    dirs /= np.linalg.norm(dirs, axis=2, keepdims=True)
    v = dirs * size * 0.577
    v -= v.mean(axis=1, keepdims=True)
    return (v + c[:, None, :]).astype(np.float32)


# --------------------------------------------------------------------------
# Benchmark-shaped generators (SURVEY 8d "Reference generator parameters")
# --------------------------------------------------------------------------

def plant(n: int, bbox=(611.0, 186.0, 249.0), e: float = 0.28, seed: int = 0) -> np.ndarray:
    """Power-Plant-like static scene: ground grid (cell 3e) + seeded tessellated boxes.

    Box size per axis exp(N(ln 6 m, 0.8)), height doubled and capped at Z, yaw uniform,
    faces tessellated into right-triangle pairs with edge e*exp(N(0, 0.5)) per box.
    Truncated to exactly n triangles.
    """
    rng = np.random.default_rng(seed)
    X, Y, Z = bbox
    cell = 3.0 * e
    nx = max(1, int(X / cell))
    ny = max(1, int(Y / cell))
    parts = [grid_mesh(nx, ny, 0.0, 0.0, X, Y, 0.0)]
    total = parts[0].shape[0]
    while total < n:
        sz = np.exp(rng.normal(math.log(6.0), 0.8, size=3))
        sz[2] = min(2.0 * sz[2], Z)
        sz[0] = min(sz[0], X)
        sz[1] = min(sz[1], Y)
        cx = rng.uniform(0.0, X)
        cy = rng.uniform(0.0, Y)
        yaw = rng.uniform(-math.pi, math.pi)
        edge = e * math.exp(rng.normal(0.0, 0.5))
        box = _tess_box(sz, edge)
        c, s = math.cos(yaw), math.sin(yaw)
        R = np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])
        box = box.astype(np.float64) @ R.T + np.array([cx, cy, sz[2] / 2.0])
        parts.append(box.astype(np.float32))
        total += box.shape[0]
    out = np.concatenate(parts, 0)[:n]
    return np.ascontiguousarray(out)


def _tess_box(size, edge: float) -> np.ndarray:
    """Box centred at 0 with the given size; each face split into right-triangle pairs."""
    sx, sy, sz = (float(s) for s in size)
    tris = []
    hx, hy, hz = sx / 2, sy / 2, sz / 2
    # (axis u, axis v, normal axis, normal sign)
    faces = [
        ((0, sx), (1, sy), 2, +hz), ((0, sx), (1, sy), 2, -hz),
        ((0, sx), (2, sz), 1, +hy), ((0, sx), (2, sz), 1, -hy),
        ((1, sy), (2, sz), 0, +hx), ((1, sy), (2, sz), 0, -hx),
    ]
    for (au, lu), (av, lv), an, off in faces:
        nu = max(1, int(round(lu / edge)))
        nv = max(1, int(round(lv / edge)))
        us = np.linspace(-lu / 2, lu / 2, nu + 1)
        vs = np.linspace(-lv / 2, lv / 2, nv + 1)
        U, V = np.meshgrid(us, vs, indexing="ij")
        P = np.zeros(U.shape + (3,))
        P[..., au] = U
        P[..., av] = V
        P[..., an] = off
        a = P[:-1, :-1].reshape(-1, 3)
        b = P[1:, :-1].reshape(-1, 3)
        c = P[1:, 1:].reshape(-1, 3)
        d = P[:-1, 1:].reshape(-1, 3)
        tris.append(np.stack([a, b, c], 1))
        tris.append(np.stack([a, c, d], 1))
    return np.concatenate(tris, 0)


def car_mesh(n_theta: int = 388, n_psi: int = 388, dims=(4.57, 2.28, 1.08), exponent: float = 4.0):
    """Superellipsoid 'sports car' in its local frame as an indexed mesh: a (n_theta+1) x (n_psi+1)
    vertex grid and 2*n_theta*n_psi triangles, the two of each quad adjacent in the list.

    x = (L/2) sgn(sin t cos p)|sin t cos p|^(2/exponent) etc.  The pole rows give
    zero-area triangles (never hit).  Returns (vertices (V, 3) fp32, faces (F, 3) int32).
    """
    L, W, H = dims
    k = 2.0 / exponent
    th = np.linspace(0.0, math.pi, n_theta + 1)
    ps = np.linspace(-math.pi, math.pi, n_psi + 1)
    T, P = np.meshgrid(th, ps, indexing="ij")

    def sp(x):
        return np.sign(x) * np.abs(x) ** k

    X = (L / 2) * sp(np.sin(T) * np.cos(P))
    Yv = (W / 2) * sp(np.sin(T) * np.sin(P))
    Zv = (H / 2) * sp(np.cos(T))
    verts = np.stack([X, Yv, Zv], -1).reshape(-1, 3).astype(np.float32)
    i, j = np.meshgrid(np.arange(n_theta), np.arange(n_psi), indexing="ij")
    i, j = i.reshape(-1), j.reshape(-1)
    a = i * (n_psi + 1) + j
    b = (i + 1) * (n_psi + 1) + j
    c = (i + 1) * (n_psi + 1) + j + 1
    d = i * (n_psi + 1) + j + 1
    faces = np.stack([np.stack([a, b, c], 1), np.stack([a, c, d], 1)], 1).reshape(-1, 3).astype(np.int32)
    return verts, faces


def car(n_theta: int = 388, n_psi: int = 388, dims=(4.57, 2.28, 1.08), exponent: float = 4.0) -> np.ndarray:
    """The car_mesh triangles as a (F, 3, 3) fp32 soup (same triangles, same order)."""
    verts, faces = car_mesh(n_theta, n_psi, dims, exponent)
    return np.ascontiguousarray(verts[faces])


def subdivide(tris: np.ndarray, levels: int) -> np.ndarray:
    """Split every triangle into 4**levels (midpoint subdivision)."""
    t = tris.astype(np.float64)
    for _ in range(levels):
        a, b, c = t[:, 0], t[:, 1], t[:, 2]
        ab, bc, ca = (a + b) / 2, (b + c) / 2, (c + a) / 2
        t = np.concatenate([
            np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
            np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)], 0)
    return t.astype(np.float32)


@dataclass
class InstancePose:
    rotation: np.ndarray  # 3x3 fp64
    scale: np.ndarray     # 3 fp64
    position: np.ndarray  # 3 fp64


def pose_instances(n: int, bbox, seed: int, frame: int, scale_lo: float = 0.001,
                   scale_hi: float = 30.0) -> List[InstancePose]:
    """Motion f.i: per frame, uniform position in the bbox (z >= 0), uniform random rotation,
    per-axis scale U[scale_lo, scale_hi]."""
    rng = np.random.default_rng([int(seed), int(frame), 0xCA5])
    out = []
    X, Y, Z = bbox
    for _ in range(n):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        s = rng.uniform(scale_lo, scale_hi, size=3)
        p = np.array([rng.uniform(0, X), rng.uniform(0, Y), rng.uniform(0, Z)])
        out.append(InstancePose(_quat_to_mat(q), s, p))
    return out


def apply_pose(local: np.ndarray, pose: InstancePose) -> np.ndarray:
    """World vertices v = R (s * v_local) + p."""
    v = local.astype(np.float64) * pose.scale
    v = v @ pose.rotation.T + pose.position
    return v.astype(np.float32)


def pose_matrix(pose: InstancePose) -> np.ndarray:
    """The instance's row-major 3x4 fp32 matrix [R diag(s) | p] (grca_update_instances), rounded once from fp64."""
    M = np.concatenate([pose.rotation * pose.scale[None, :], pose.position[:, None]], axis=1)
    return M.astype(np.float32)


def apply_pose_f32(local: np.ndarray, M: np.ndarray) -> np.ndarray:
    """World vertices of an instance exactly as grca_update_instances defines them: per row r,
    ((m_r0 x + m_r1 y) + m_r2 z) + m_r3 in IEEE fp32, every product and sum rounded (numpy float32 ops)."""
    v = np.asarray(local, dtype=np.float32)
    M = np.asarray(M, dtype=np.float32)
    out = np.empty(v.shape, dtype=np.float32)
    for r in range(3):
        out[..., r] = ((M[r, 0] * v[..., 0] + M[r, 1] * v[..., 1]) + M[r, 2] * v[..., 2]) + M[r, 3]
    return out


def swd(tris: np.ndarray, bbox, seed: int, frame: int) -> np.ndarray:
    """Scene-wide deformation: each triangle keeps its shape; its centroid is redrawn
    uniformly in the world bbox."""
    rng = np.random.default_rng([int(seed), int(frame), 0x5D])
    t = tris.astype(np.float64)
    c = t.mean(axis=1, keepdims=True)
    X, Y, Z = bbox
    nc = np.stack([rng.uniform(0, X, len(t)), rng.uniform(0, Y, len(t)), rng.uniform(0, Z, len(t))], -1)
    return (t - c + nc[:, None, :]).astype(np.float32)


# --------------------------------------------------------------------------
# Workload presets (BASELINE.json configs)
# --------------------------------------------------------------------------

def c1_emitter(max_range: float = INF, elev: Optional[np.ndarray] = None) -> Emitter:
    """C1 sensor: 1 LiDAR, 16 channels full sphere, 512 rays, 360 deg, at (0, 0, 1.5)."""
    return Emitter(origin=(0.0, 0.0, 1.5), elev=full_sphere_elev(16) if elev is None else elev,
                   rays_per_channel=512, hfov_deg=360, max_range=max_range)


def c1_scene(seed: int = 1) -> np.ndarray:
    """C1: 2,000 triangles: ground 40x40 m at z=0 (200 tris), fixtures placed relative to
    the emitter at (0,0,1.5), random triangles in a 30 m cube; total exactly 2,000."""
    rng = np.random.default_rng(seed)
    o = (0.0, 0.0, 1.5)
    ground = grid_mesh(10, 10, -20.0, -20.0, 20.0, 20.0, 0.0)  # 200
    fixtures = [
        quad_x5(o),                                   # 2
        seam_triangle(o),                             # 1
        np.array([[[-1.0, -1.0, 4.0], [2.0, -1.0, 4.0], [0.0, 2.0, 4.0]]], np.float32),  # zenith ceiling
        np.array([[[0.0, 8.0, 0.3], [3.0, 8.0, 0.3], [1.5, 8.0, 3.0]]], np.float32),     # facing +y
        np.array([[[7.0, 7.0, 1.5], [9.0, 7.2, 1.5], [8.0, 9.0, 1.5002]]], np.float32),  # grazing, ~horizon plane
    ]
    fix = np.concatenate(fixtures, 0)
    n_rand = 2000 - ground.shape[0] - fix.shape[0]
    rand = random_triangles(rng, n_rand, center=(0.0, 0.0, 1.5), half_extent=15.0)
    return np.ascontiguousarray(np.concatenate([ground, fix, rand], 0))


def random_scene(seed: int, n_tris: int = 300, n_emitters: int = 2, gamma: int = 12, chi: int = 96,
                 extent: float = 12.0, max_range: Optional[float] = None):
    """Small random scene for parity sweeps: random frames, mixed 360/180 emitters,
    optional range limits, random triangle soup around the emitters."""
    rng = np.random.default_rng([int(seed), 0xA11])
    ems = []
    for k in range(n_emitters):
        f, r, u = random_frame(rng) if k % 2 else yaw_frame(rng.uniform(-math.pi, math.pi))
        elev = full_sphere_elev(gamma) if k % 3 != 2 else np.sort(
            rng.uniform(-1.2, 1.2, size=gamma)).astype(np.float32)
        ems.append(Emitter(origin=rng.uniform(-2, 2, size=3), forward=f, right=r, up=u, elev=elev,
                           rays_per_channel=chi + 7 * k, hfov_deg=360 if k % 2 == 0 else 180,
                           max_range=(INF if max_range is None else max_range * (1 + k))))
    tris = random_triangles(rng, n_tris, center=(0, 0, 0), half_extent=extent, edge_lo=0.05, edge_hi=6.0)
    return ems, tris


def place_emitters(n: int, bbox, seed: int, gamma: int = 128, chi: int = 4096, hfovs=None,
                   max_range: Optional[float] = 1000.0, height: float = 2.0) -> List[Emitter]:
    """seeded uniform positions inside the bbox footprint at 2 m above ground,
    yaw uniform, level (u = +z); the paper's full-sphere grid."""
    rng = np.random.default_rng([int(seed), 0xE317])
    X, Y, _ = bbox
    out = []
    for k in range(n):
        pos = (rng.uniform(0.1 * X, 0.9 * X), rng.uniform(0.1 * Y, 0.9 * Y), height)
        f, r, u = yaw_frame(rng.uniform(-math.pi, math.pi))
        out.append(Emitter(origin=pos, forward=f, right=r, up=u, elev=full_sphere_elev(gamma), rays_per_channel=chi,
                           hfov_deg=(hfovs[k] if hfovs else 360),
                           max_range=INF if max_range is None else float(max_range)))
    return out


WORKLOADS = {
    # name: (n_emitters, hfovs, bbox, n_static, n_cars, default range, car scale range)
    "C2": (2, None, (240.0, 80.0, 60.0), 700_000, 1, None, (0.001, 30.0)),
    "C3": (4, [360, 360, 180, 180], (400.0, 150.0, 120.0), 3_500_000, 5, 50.0, (0.001, 30.0)),
    "C4": (8, None, (611.0, 186.0, 249.0), 12_759_246, 30, 1000.0, (0.001, 30.0)),
    "C5": (2, None, (240.0, 80.0, 60.0), 700_000, 1, None, (1.0, 1.0)),
}


def indexed_frame(w: dict):
    """The bench's indexed representation of a workload frame (ND motion, no subdivision): vertices =
    [static triangles' own vertices, 3 each] + [each car instance's posed grid vertices], indices =
    [0 .. 3 n_static - 1] + [the cars' faces offset per instance].  verts[idx] reproduces w["tris"]
    exactly (same per-vertex posing).  Returns (verts (V, 3) fp32, idx (3 T,) int32)."""
    car_v, car_f = w["car_mesh"]
    ns = w["n_static"]
    static_v = w["tris"][:ns].reshape(-1, 3)
    inst_v = [apply_pose(car_v, p) for p in w["poses"]]
    verts = np.concatenate([static_v] + inst_v, 0)
    off = 3 * ns + np.arange(len(inst_v), dtype=np.int64)[:, None, None] * len(car_v)
    dyn_idx = (car_f[None].astype(np.int64) + off).reshape(-1)
    idx = np.concatenate([np.arange(3 * ns, dtype=np.int64), dyn_idx]).astype(np.int32)
    return np.ascontiguousarray(verts.astype(np.float32)), idx


def workload(name: str, frame: int = 0, deformation: str = "ND", static_scale: float = 1.0,
             max_range=-1.0, subdiv: int = 0, n_cars: Optional[int] = None) -> dict:
    """BASELINE.json configs as concrete seeded scenes.

    Returns dict(emitters, tris = static + dynamic (n, 3, 3) fp32, n_static, n_dynamic, bbox,
    poses).  Scene seed = config id; motion seed = (config id, frame).
    """
    if name == "C1":
        return {"emitters": [c1_emitter()], "tris": c1_scene(), "n_static": 2000, "n_dynamic": 0,
                "bbox": (40.0, 40.0, 30.0), "poses": []}
    n_em, hfovs, bbox, n_static, cars, rng_default, (slo, shi) = WORKLOADS[name]
    seed = int(name[1:])
    if n_cars is not None:
        cars = n_cars
    rng_m = rng_default if (max_range is not None and max_range < 0) else max_range
    ems = place_emitters(n_em, bbox, seed, hfovs=hfovs, max_range=rng_m)
    static = plant(max(1, int(n_static * static_scale)), bbox=bbox, seed=seed)
    car_v, car_f = car_mesh()
    local = np.ascontiguousarray(car_v[car_f])
    if subdiv:
        local = subdivide(local, subdiv)
    poses = pose_instances(cars, bbox, seed, frame, scale_lo=slo, scale_hi=shi)
    dyn = [apply_pose(local, p) for p in poses]
    dynamic = np.concatenate(dyn, 0) if dyn else np.zeros((0, 3, 3), np.float32)
    if deformation == "SWD":
        dynamic = swd(dynamic, bbox, seed, frame)
    tris = np.ascontiguousarray(np.concatenate([static, dynamic], 0))
    return {"emitters": ems, "tris": tris, "n_static": static.shape[0], "n_dynamic": dynamic.shape[0],
            "bbox": bbox, "poses": poses, "car_local": local,
            "car_mesh": None if subdiv else (car_v, car_f)}
