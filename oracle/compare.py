"""Parity comparator (TEST INFRASTRUCTURE ONLY) -- the north-star contract.

SURVEY 8(c) "Comparator": for every ray r with GPU result G = (t_G, id_G) and
oracle result O = (t_O, id_O) the ray AGREES iff
  * both miss; or
  * both hit, |t_G - t_O| <= 1e-5 t_O and id_G == id_O; or
  * both hit with different ids and the oracle's fp64 t of (r, id_G) is within
    1e-5 t_O (a near-tie), with |t_G - t_O| <= 1e-5 t_O.
Any other ray is a disagreement; it is EXCUSED iff the triangle that one side
hit and the other did not has fp64 barycentric margin within 1e-6 of its
boundary for r (min(u, v, 1-u-v) in [-1e-6, 1e-6]).  Pass = agreement >=
99.999 % of rays and every disagreement excused.  Also reports the paper's
Hit% at 0.001 m.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import oracle as _o

REL_T = 1e-5
BARY_EPS = 1e-6
AGREE_FRAC = 0.99999


def _margin(emitters, g, tri9, faces, arr):
    ok, t, u, v, hit = _o.ray_tri(emitters, g, tri9, faces, _arr=arr)
    if not ok:
        return None, False, t
    return min(u, v, 1.0 - u - v), hit, t


def compare(emitters, tris: np.ndarray, gpu_t: np.ndarray, gpu_id: np.ndarray, ref: dict,
            ids: Optional[np.ndarray] = None, faces: int = 0, max_detail: int = 20) -> dict:
    """Compare GPU outputs (for the rays ref['rays']) with an oracle result ``ref``."""
    rays = ref["rays"]
    o_t = ref["t64"] if ref.get("t64") is not None else ref["t"].astype(np.float64)
    o_id = ref["id"]
    g_t = np.asarray(gpu_t, dtype=np.float64)
    g_id = np.asarray(gpu_id, dtype=np.int32)
    assert g_t.shape == o_t.shape == g_id.shape == o_id.shape
    T9 = np.asarray(tris, dtype=np.float32).reshape(-1, 9)
    if ids is None:
        index_of = None
    else:
        index_of = {int(v): k for k, v in enumerate(np.asarray(ids))}

    def tri_of(i):
        k = int(i) if index_of is None else index_of.get(int(i))
        if k is None or k < 0 or k >= T9.shape[0]:
            return None
        return T9[k]

    arr = _o._EmArray(emitters)
    n = rays.shape[0]
    g_miss = g_id < 0
    o_miss = o_id < 0
    both_miss = g_miss & o_miss
    both_hit = ~g_miss & ~o_miss
    with np.errstate(invalid="ignore"):
        t_ok = np.abs(g_t - o_t) <= REL_T * o_t
    agree = both_miss | (both_hit & (g_id == o_id) & t_ok)
    # also: GPU miss flags must carry +inf and -1 consistently
    bad_sentinel = (g_miss & ~np.isinf(g_t)) | (~g_miss & ~np.isfinite(g_t))
    agree &= ~bad_sentinel
    kinds = {"dist": 0, "id": 0, "gpu_miss": 0, "gpu_extra": 0, "sentinel": int(bad_sentinel.sum())}
    excused = {"dist": 0, "id": 0, "gpu_miss": 0, "gpu_extra": 0, "sentinel": 0}
    near_ties = 0
    details = []
    for r in np.nonzero(~agree)[0]:
        g = int(rays[r])
        kind, exc = None, False
        if bad_sentinel[r]:
            kind = "sentinel"
        elif both_hit[r] and g_id[r] == o_id[r]:
            kind = "dist"
        elif both_hit[r]:
            tri = tri_of(g_id[r])
            m, hit, tq = _margin(emitters, g, tri, faces, arr) if tri is not None else (None, False, 0.0)
            if hit and abs(tq - o_t[r]) <= REL_T * o_t[r] and t_ok[r]:
                near_ties += 1
                agree[r] = True
                continue
            kind = "id"
            if not hit:
                exc = m is not None and abs(m) <= BARY_EPS   # GPU hit a triangle the oracle misses
            else:
                tri_o = tri_of(o_id[r])                      # GPU missed the oracle's closer triangle
                mo, _, _ = _margin(emitters, g, tri_o, faces, arr)
                exc = mo is not None and abs(mo) <= BARY_EPS
        elif g_miss[r]:
            kind = "gpu_miss"
            tri_o = tri_of(o_id[r])
            mo, _, _ = _margin(emitters, g, tri_o, faces, arr)
            exc = mo is not None and abs(mo) <= BARY_EPS
        else:
            kind = "gpu_extra"
            tri = tri_of(g_id[r])
            m, hit, _ = _margin(emitters, g, tri, faces, arr) if tri is not None else (None, False, 0.0)
            exc = (not hit) and m is not None and abs(m) <= BARY_EPS
        if kind != "sentinel":
            kinds[kind] += 1
        if exc:
            excused[kind] += 1
        if len(details) < max_detail:
            details.append({"ray": g, "kind": kind, "excused": bool(exc), "gpu": (float(g_t[r]), int(g_id[r])),
                            "oracle": (float(o_t[r]), int(o_id[r]))})
    n_agree = int(agree.sum())
    n_dis = n - n_agree
    n_exc = int(sum(excused.values()))
    frac = n_agree / n if n else 1.0
    # paper-style Hit% at 0.001 m: oracle hits reproduced within 1 mm
    o_hits = ~o_miss
    with np.errstate(invalid="ignore"):
        hit_mm = o_hits & ~g_miss & (np.abs(g_t - o_t) <= 1e-3)
    hit_pct = 100.0 * hit_mm.sum() / max(1, o_hits.sum())
    return {
        "rays": int(n),
        "agree": n_agree,
        "agree_frac": frac,
        "disagree": n_dis,
        "excused": n_exc,
        "unexcused": n_dis - n_exc,
        "kinds": kinds,
        "excused_kinds": excused,
        "near_ties": near_ties,
        "oracle_hits": int(o_hits.sum()),
        "hit_pct_1mm": float(hit_pct),
        "passed": bool(frac >= AGREE_FRAC and n_dis == n_exc),
        "details": details,
    }
