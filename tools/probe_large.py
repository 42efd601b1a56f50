"""Where do the large-path (K3/K4) items of a C4 frame come from?  (dev tooling, GPU)

    PYTHONPATH=. python tools/probe_large.py [--frames 0,1,2,3]

Per frame: the large-pair list (grca_debug_large_list), split into full-azimuth rectangles
(r_len == chi: no A7 refinement) and partial ones; rectangle items before A7 vs the items K4
actually tested; the biggest rectangles with their triangle's size and distance.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as sg  # noqa: E402


def main():
    import torch

    from paper_2605_10457_b200 import Grca, tris_to_float4

    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", default="0,1,2,3")
    ap.add_argument("--config", default="C4")
    args = ap.parse_args()
    for f in [int(x) for x in args.frames.split(",")]:
        w = sg.workload(args.config, frame=f)
        ems, tris = w["emitters"], w["tris"]
        g = Grca(device=0, max_triangles=len(tris), max_rays=sg.n_rays_total(ems))
        g.set_emitters(ems)
        v4 = tris_to_float4(tris)
        g.update_triangles(v4)
        d, t = g.cast()
        torch.cuda.synchronize()
        st = g.get_stats()
        L = g.debug_large_list()
        tri = L[:, 0]
        e = L[:, 1] & 255
        c_from = (L[:, 1] >> 8) & 0xFFFFFF
        c_to = L[:, 2]
        r_lo = L[:, 3] & 0xFFFF
        r_len = (L[:, 3] >> 16) & 0xFFFF
        chi = np.array([ems[k].rays_per_channel for k in e])
        rows = c_to - c_from + 1
        full = r_len >= chi
        items = rows * r_len
        large_items = st["rtic_tested"] - st["rtic_small"]
        print(f"frame {f}: large pairs {len(L)}, full-azimuth {int(full.sum())} "
              f"({items[full].sum() / 1e6:.2f}M rect items), partial {int((~full).sum())} "
              f"({items[~full].sum() / 1e6:.2f}M rect items before A7); K4 tested {large_items / 1e6:.2f}M, "
              f"hits (all paths) {st['hits_recorded'] / 1e6:.2f}M, chunks {st['chunks']}")
        o = np.stack([np.asarray(ems[k].origin, np.float64) for k in e])
        T = tris[tri].astype(np.float64)
        dist = np.linalg.norm(T.mean(1) - o, axis=1)
        area = 0.5 * np.linalg.norm(np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0]), axis=1)
        dyn = tri >= w["n_static"]
        print(f"   dynamic (car) pairs {int(dyn.sum())} items {items[dyn].sum() / 1e6:.2f}M; static {int((~dyn).sum())} "
              f"items {items[~dyn].sum() / 1e6:.2f}M")
        # full-azimuth pairs: horizontal distance of the triangle from the emitter's spin axis
        up = np.stack([np.asarray(ems[k].up, np.float64) for k in e])
        rel = T - o[:, None, :]
        zc = np.einsum("nkd,nd->nk", rel, up)
        hor = rel - zc[..., None] * up[:, None, :]
        rho = np.linalg.norm(hor, axis=2)
        emax = np.max(np.linalg.norm(T - np.roll(T, 1, axis=1), axis=2), axis=1)
        for name, m in (("full car", full & dyn), ("full static", full & ~dyn), ("partial", ~full)):
            if m.sum():
                print(f"   {name}: n {int(m.sum())} items {items[m].sum() / 1e6:.2f}M  min-rho median {np.median(rho[m].min(1)):.3f} m "
                      f"(p10 {np.percentile(rho[m].min(1), 10):.3f}, p90 {np.percentile(rho[m].min(1), 90):.3f})  |dz| median "
                      f"{np.median(np.abs(zc[m]).min(1)):.3f} m  edge median {np.median(emax[m]):.4f} m  rows median {np.median(rows[m])}")
        top = np.argsort(-items)[:8]
        for i in top:
            print(f"   tri {tri[i]:9d} {'car' if dyn[i] else 'static'} em {e[i]} rows {rows[i]:3d} r_len {r_len[i]:5d} "
                  f"full {bool(full[i])} items {items[i]:7d} dist {dist[i]:6.2f} m area {area[i]:.4f} m2")
        g.close()


if __name__ == "__main__":
    main()
