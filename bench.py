"""bench.py -- GRCA hot path on B200: rays/s & frame ms (device-timed, max over ranks), RTIC culled %.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

One step = one LiDAR frame of BASELINE config C4 (8 LiDARs 128x4096 = 4,194,304 rays,
~21.8M triangles of which ~9.0M dynamic, 1000 m range): K0 init -> K2 cull -> fused refine +
small-rectangle intersection -> K3 bin -> K4 intersect -> K5 unpack.  Inputs are resident in HBM
(grca_update_scene: the static scenery as one float4 soup, the cars as indexed float3 meshes with
4 posed frames cycled; every step streams 0.78 GB, > L2).  With N>1 (torchrun) the emitters are
sharded across ranks (sensor sharding, no reduction; --shard triangles|mixed adds the library's
in-stream NCCL min-merge of the packed hit keys: all-reduce, reduce-scatter or the fused NVLS path --
the handle owns its communicator, grca_cast is collective).  `e2e`
repeats the measurement through the public API with the frame's car vertices copied from pinned
host memory and the outputs copied back inside the timed region.  `--impl reference` times the
brute-force oracle (the reference arm of this tier) on host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import scenegen as sg  # noqa: E402

N_FRAMES = 4   # distinct resident frames cycled through (each > L2)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "src_hbm": "measured (MEASURED_PEAKS.json hbm_gbs, copy b/w)",
                "sm_max_mhz": float(d.get("sm_max_mhz", 1965))}
    except Exception:
        return {"hbm_gbs": 6650.0, "src_hbm": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- scene --
class Scene:
    """Resident C-config frames on the GPU (harness: input generation, not the hot path).

    mesh="indexed" (default when the cars are plain meshes, i.e. ND motion and no subdivision):
    grca_update_scene's two parts -- the static triangles as one resident float4-triplet soup
    shared by all frames, then the cars as one packed-float3 vertex buffer per frame (shared grid
    vertices) with one index buffer shared by all frames (their faces).  Same triangles, same order
    and ids as the soup; a frame's per-step input is then only the car vertices.  mesh="soup":
    float4 triplets per triangle, one buffer per frame (static part copied into each)."""

    def __init__(self, config: str, rank: int, world: int, device, deformation: str = "ND", shard: str = "triangles",
                 max_range=-1.0, subdiv: int = 0, car_scale=None, mesh: str = "indexed", w=None):
        import torch

        from paper_2605_10457_b200 import dist as D
        from paper_2605_10457_b200 import tris_to_float4

        if w is None:
            w = sg.workload(config, frame=0, deformation=deformation, max_range=max_range, subdiv=subdiv)
        self.w = w
        self.scale = car_scale or sg.WORKLOADS.get(config, (0,) * 7)[6] if config != "C1" else (1.0, 1.0)
        self.emitters = w["emitters"]
        n_static, n_dyn = w["n_static"], w["n_dynamic"]
        self.n_tri_global = n_static + n_dyn
        own = np.zeros(self.n_tri_global, dtype=bool)
        if shard.startswith("mixed"):   # emitter groups x triangle shards (D.mixed_partition)
            g, t, T = D.mixed_partition(rank, world, int(shard.split(":")[1]))
            own[D.shard_triangles(self.n_tri_global, t, T)] = True
            self.emitters = [self.emitters[n] for n in D.shard_emitters(len(self.emitters), g, world // T)]
        elif shard == "triangles":
            own[D.shard_triangles(self.n_tri_global, rank, world)] = True
        else:   # sensor sharding: every rank holds all triangles, casts its own emitters
            own[:] = True
            self.emitters = [self.emitters[n] for n in D.shard_emitters(len(self.emitters), rank, world)]
        self.own_static = np.nonzero(own[:n_static])[0]
        self.own_dyn = np.nonzero(own[n_static:])[0]
        self.ids = torch.as_tensor(np.concatenate([self.own_static, n_static + self.own_dyn]).astype(np.int32),
                                   device=device)
        self.n_tri = int(self.ids.numel())
        # every triangle in its global order (one GPU, sensor shards): ids are the identity, so the
        # library derives them (tri_id_base) instead of gathering an id array per survivor
        self.identity = self.n_tri == self.n_tri_global
        self.ids_arg = None if self.identity else self.ids
        self.n_static_local = len(self.own_static)
        self.ns3 = 3 * self.n_static_local
        static = torch.as_tensor(w["tris"][:n_static][self.own_static].reshape(-1, 3), device=device)
        self.n_cars = len(w["poses"])
        self.bbox = w["bbox"]
        self.config = config
        self.deformation = deformation
        self.device = device
        cm = w.get("car_mesh")
        self.indexed = mesh in ("indexed", "instances") and cm is not None and deformation == "ND" and n_dyn > 0
        # rigid instances (grca_update_instances): a frame is one 3x4 matrix per car; needs whole instances in
        # order on this rank (one GPU or sensor shards)
        self.instanced = self.indexed and mesh == "instances" and self.identity
        self.mesh = "instances" if self.instanced else "indexed" if self.indexed else "soup"
        self.idx_dyn = self.static_soup = None
        if self.indexed:
            car_v, car_f = cm
            nv_car, nf_car = len(car_v), len(car_f)
            self.car_v_np = np.asarray(car_v, dtype=np.float32)   # (V, 3) local
            inst, f = self.own_dyn // nf_car, self.own_dyn % nf_car
            rel = (inst.astype(np.int64) * nv_car)[:, None] + car_f[f].astype(np.int64)
            self.idx_dyn = torch.as_tensor(rel.astype(np.int32).reshape(-1), device=device)
            self.n_dyn_vert = self.n_cars * nv_car
            self.static_soup = tris_to_float4(static, device=device)   # part A of grca_update_scene (resident)
            # Algorithmic K2 read per cast: static 48 B (3 float4); cars 12 B indices per triangle +
            # 12 B per shared float3 vertex
            self.tri_bytes = self.n_static_local * 48 + len(self.own_dyn) * 12 + self.n_dyn_vert * 12
            if self.instanced:   # local mesh (faces + vertices) once, 48 B of matrix per instance
                self.car_v_dev = torch.as_tensor(self.car_v_np, device=device)
                self.car_f_np = np.asarray(car_f, dtype=np.int32)
                self.car_f_dev = torch.as_tensor(self.car_f_np, device=device)
                self.tri_bytes = self.n_static_local * 48 + nf_car * 12 + nv_car * 12 + self.n_cars * 48
        else:
            self.car_np = np.asarray(w.get("car_local", np.zeros((0, 3, 3))), dtype=np.float32)   # (m, 3, 3) local
            self.tri_bytes = self.n_tri * 48
        # frame buffers: soup = [static | dynamic] float4 rows; indexed = the car vertices only; instances = the
        # cars' 3x4 matrices as rows of 4 floats (3 per car)
        self.fs = 0 if self.indexed else self.ns3   # static rows at the head of a frame buffer
        self.frames = []
        for fr in range(N_FRAMES if self.instanced else 0):
            poses = sg.pose_instances(self.n_cars, self.bbox, int(self.config[1:]), fr, scale_lo=self.scale[0],
                                      scale_hi=self.scale[1])
            Ms = np.stack([sg.pose_matrix(p) for p in poses]).reshape(-1, 4)
            self.frames.append(torch.as_tensor(np.ascontiguousarray(Ms), device=device))
        for fr in range(0 if self.instanced else N_FRAMES):
            nd = self.n_dyn_vert if self.indexed else 3 * (self.n_tri - self.n_static_local)
            buf = torch.zeros((self.fs + nd, 3 if self.indexed else 4), dtype=torch.float32, device=device)
            buf[: self.fs, :3] = static[: self.fs]
            buf[self.fs:, :3] = self.dynamic(fr)
            self.frames.append(buf)
        del static
        torch.cuda.synchronize()

    def bind(self, g, buf, n_triangles=None):
        """Point handle g at one frame buffer (public API: grca_update_scene / grca_update_triangles /
        grca_update_instances)."""
        if self.instanced:
            g.update_scene(soup=self.static_soup, tri_ids=self.ids_arg)
            g.update_instances(self.car_v_dev, self.car_f_dev, buf.view(-1, 3, 4))
        elif self.indexed:
            g.update_scene(soup=self.static_soup, mesh_xyz=buf, mesh_indices=self.idx_dyn, tri_ids=self.ids_arg)
        else:
            g.update_triangles(buf, tri_ids=self.ids_arg, n_triangles=n_triangles)

    def frame_tris(self, frame: int, w_tris):
        """The triangles frame `frame` casts, on the host (the oracle's input): scenegen's frame, except that
        instanced cars are posed with the documented fp32 order of grca_update_instances."""
        if not self.instanced:
            return w_tris
        Ms = self.frames[frame].cpu().numpy().reshape(-1, 3, 4)
        cars = [sg.apply_pose_f32(self.car_v_np, M)[self.car_f_np] for M in Ms]
        return np.ascontiguousarray(np.concatenate([w_tris[: self.n_static_local]] + cars, 0))

    def dynamic(self, frame: int):
        """Motion f.i: per-frame random pose/scale of every car instance; world
        v = R (s * v_local) + p, posed with scenegen.apply_pose (host fp64, rounded once), so every frame
        equals scenegen.workload(config, frame) bit for bit and the oracle can check it.  Indexed: the
        posed car vertices (n_cars * V, 3); soup: the own dynamic triangles' vertices (3 * n_own_dyn, 3)."""
        import torch

        poses = sg.pose_instances(self.n_cars, self.bbox, int(self.config[1:]), frame, scale_lo=self.scale[0],
                                  scale_hi=self.scale[1])
        if not poses:
            return torch.zeros((0, 3), dtype=torch.float32, device=self.device)
        if self.indexed:
            v = np.concatenate([sg.apply_pose(self.car_v_np, p) for p in poses], 0)
            return torch.as_tensor(v, device=self.device)
        v = np.concatenate([sg.apply_pose(self.car_np, p) for p in poses], 0)
        if self.deformation == "SWD":
            v = sg.swd(v, self.bbox, int(self.config[1:]), frame)
        return torch.as_tensor(np.ascontiguousarray(v[self.own_dyn].reshape(-1, 3)), device=self.device)


# ------------------------------------------------------------- reference --
def oracle_sample(emitters, tris, n_rays_sample: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    tot = sg.n_rays_total(emitters)
    return np.sort(rng.choice(tot, size=min(n_rays_sample, tot), replace=False)).astype(np.int64)


def time_oracle(emitters, tris, target_s: float = 12.0, max_rays: int = 4096):
    """Time the brute-force oracle (as it stands) on this host's cores on a bounded ray sample of
    the same workload; returns rays/s of full Eq.-1 brute force."""
    import oracle

    threads = os.cpu_count() or 1
    n = max(threads, 8)
    t0 = time.perf_counter()
    oracle.cast(emitters, tris, rays=oracle_sample(emitters, tris, n, 1), threads=threads)
    dt = time.perf_counter() - t0
    rate = n / max(dt, 1e-9)
    n2 = int(min(max_rays, max(n, rate * target_s)))
    rays = oracle_sample(emitters, tris, n2, 2)
    t0 = time.perf_counter()
    ref = oracle.cast(emitters, tris, rays=rays, threads=threads, want_t64=True)
    dt = time.perf_counter() - t0
    return {"value": n2 / dt, "unit": "rays/s", "cores": threads, "kind": "oracle",
            "sample": f"{n2} seeded rays x all {len(tris)} triangles (fp64 brute force, Eq. 1), {dt:.1f} s",
            "tests_per_s": n2 * len(tris) / dt, "frame_ms_extrapolated": 1e3 * dt * sg.n_rays_total(emitters) / n2,
            "frame_ms_kind": "extrapolated: measured sample time x rays per frame / sampled rays"}, ref


KERNELS = ["K0_init", "K2_cull", "K2b_refine", "K4s_small", "K3_bin", "K4_large", "K5_unpack"]
# (fused default: "K4s_small" is the fused K2b+K4s kernel k_refine_small and "K2b_refine" is ~0)
NCU_NAME = {"K2_cull": "k_cull_fixed", "K2b_refine": "k_refine(", "K4s_small": "k_refine_small", "K4_large": "k_isect",
            "K0_init": "k_init", "K3_bin": "k_bin", "K5_unpack": "k_unpack"}
# Algorithmic work per unit, SURVEY.md 8(d) "Algorithmic work" (midpoints of its ranges):
#   per (triangle, emitter) pair: quick reject ~40-60 instructions -> 50
#   per K2 survivor: exact bounds ~250-400 instructions -> 325 (the fused kernel's per-survivor work)
#   per candidate (RTIC performed): ~20 fp32 flops + compares -> 25 lane-instructions, and one u64 RED.MIN
#   per improving hit; per ray 8 B init (K0) + 8 B read + 8 B written (K5); per triangle its vertex bytes
ALU_PER_PAIR = 50
ALU_PER_SURVIVOR = 325
ALU_PER_CANDIDATE = 25
BYTES_K0_PER_RAY = 8
BYTES_K5_PER_RAY = 16


def ncu_traffic():
    """DRAM bytes per launch from the latest committed `ncu --set full` capture (profiles/)."""
    import glob

    import re

    def order(path):   # rNN<letter>_traffic.json: mid-round snapshots (r02b) before the round's final r02_
        m = re.match(r"r(\d+)([a-z]*)_traffic\.json$", os.path.basename(path))
        return (int(m.group(1)), m.group(2) == "", m.group(2)) if m else (-1, False, "")

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), key=order)
    if not files:
        return {}, None
    d = json.load(open(files[-1]))
    out = {}
    for k, v in d.get("per_kernel", {}).items():
        for ours, nm in NCU_NAME.items():
            if nm in k:
                out[ours] = v
    return out, os.path.basename(files[-1])


def measured_peaks():
    """Denominators measured live on this GPU (tools/peaks.cu: FFMA lane-instruction rate, u64 RED.MIN rate
    into an L2-resident 33.5 MB buffer) plus MEASURED_PEAKS.json's HBM copy bandwidth; the committed
    profiles/r02_peaks.json if the live run fails."""
    pk = peaks()
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import peaks as P   # noqa: E402

        m = P.measure()
        m["src"] = "measured live (tools/peaks.cu)"
    except Exception as e:  # noqa: BLE001
        m = json.load(open(os.path.join(ROOT, "profiles", "r02_peaks.json")))
        m["src"] = f"profiles/r02_peaks.json (live measurement failed: {e})"
    pk.update(m)
    return pk


def kernel_rooflines(kernel_ms, st, n_rays, pk, tri_bytes, split=False):
    """Per-kernel achieved / peak with SURVEY 8(d)'s per-unit counts (see the constants above)."""
    traffic, src = ncu_traffic()
    small_items = st["rtic_small"]
    large_items = st["rtic_tested"] - small_items
    alu_peak = pk["ffma_lane_instr_per_s"] / 1e12
    work = {
        "K0_init": ("hbm", BYTES_K0_PER_RAY * n_rays, f"{BYTES_K0_PER_RAY} B x rays"),
        "K2_cull": ("alu", ALU_PER_PAIR * st["pairs"], f"{ALU_PER_PAIR} x pairs"),
        "K2b_refine": ("alu", ALU_PER_SURVIVOR * st["prefilter_survivors"] if split else 0,
                       f"{ALU_PER_SURVIVOR} x K2 survivors (split mode only)"),
        "K4s_small": ("alu", ALU_PER_CANDIDATE * small_items + (0 if split else ALU_PER_SURVIVOR * st["prefilter_survivors"]),
                      f"{ALU_PER_SURVIVOR} x K2 survivors + {ALU_PER_CANDIDATE} x small-rectangle candidates"),
        "K3_bin": ("hbm", 32 * max(1, st["large_pairs"]), "32 B x large pairs (not an 8(d) unit; context)"),
        "K4_large": ("alu", ALU_PER_CANDIDATE * large_items, f"{ALU_PER_CANDIDATE} x large-rectangle candidates"),
        "K5_unpack": ("hbm", BYTES_K5_PER_RAY * n_rays, f"{BYTES_K5_PER_RAY} B x rays"),
    }
    reds = {"K4s_small": st["hits_recorded"] - st["hits_large"], "K4_large": st["hits_large"]}
    out = {}
    for k, (bound, amount, unit_src) in work.items():
        t = max(kernel_ms[k], 1e-9) / 1e3
        if bound == "hbm":
            ach, peak, unit = amount / t / 1e9, pk["hbm_gbs"], "GB/s"
            psrc = pk["src_hbm"]
        else:
            ach, peak, unit = amount / t / 1e12, alu_peak, "T lane-instr/s"
            psrc = "FFMA lane-instruction rate, " + pk["src"]
        tr = traffic.get(k, {})
        out[k] = {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                  "traffic": tr.get("dram_bytes"), "algorithmic_per_launch": amount, "algorithmic_units": unit_src,
                  # context from the same ncu capture: fraction of cycles an instruction issued
                  # (a latency-bound kernel sits well below 1 even when its ALU fraction is low)
                  "ncu_issue_slots_busy": (tr["issue_slots_busy_pct"] / 100.0) if "issue_slots_busy_pct" in tr else None,
                  "peak_src": psrc, "traffic_src": src}
        if k in reds:   # closest-hit key updates: u64 RED.MIN per accepted hit
            out[k]["red_min_per_s"] = reds[k] / t
            out[k]["red_min_frac"] = reds[k] / t / pk["red_min_u64_random_per_s"]
    # K2 also streams the triangles once: its HBM fraction beside the ALU one
    t2 = max(kernel_ms["K2_cull"], 1e-9) / 1e3
    out["K2_cull"]["hbm_achieved_gbs"] = tri_bytes / t2 / 1e9
    out["K2_cull"]["hbm_frac"] = out["K2_cull"]["hbm_achieved_gbs"] / pk["hbm_gbs"]
    return out


def frame_roofline(roof, ms_step, n_rays, tri_bytes, pk):
    """Whole-frame bound: t_HBM = (triangle bytes + 24 B per ray) / HBM peak, t_ALU = all kernels'
    algorithmic lane-instructions / FFMA lane-instruction peak; frac = max(t_HBM, t_ALU) / t_measured."""
    t_hbm = (tri_bytes + 24 * n_rays) / (pk["hbm_gbs"] * 1e9) * 1e3
    alu = sum(v["algorithmic_per_launch"] for v in roof.values() if v["bound"] == "alu")
    t_alu = alu / pk["ffma_lane_instr_per_s"] * 1e3
    return {"t_hbm_floor_ms": t_hbm, "t_alu_floor_ms": t_alu, "t_measured_ms": ms_step,
            "frac": max(t_hbm, t_alu) / ms_step, "alu_lane_instr": alu, "hbm_bytes": tri_bytes + 24 * n_rays}


# ------------------------------------------------------------------ main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--deformation", default="ND", choices=["ND", "SWD"])
    ap.add_argument("--impl", default="grca", choices=["grca", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-hybrid", action="store_true")
    ap.add_argument("--small-max", type=int, default=0)
    ap.add_argument("--max-range", type=float, default=-1.0, help="metres; -1 = config default, 0 = unlimited")
    ap.add_argument("--subdiv", type=int, default=0, help="C5: car subdivision level (4^L triangles each)")
    ap.add_argument("--car-scale", default=None, help="lo,hi per-axis car scale (C5 'large triangles' variant)")
    ap.add_argument("--split-refine", action="store_true", help="K2b and K4s as two kernels (A/B)")
    ap.add_argument("--l2-persist", action="store_true", help="A/B: persisting L2 window (opt-in)")
    ap.add_argument("--no-packed", action="store_true", help="A/B: K2 without packed fp32x2 math")
    ap.add_argument("--emulate-world", type=int, default=0, help="do rank --emulate-rank's share of a W-rank run "
                    "on this one GPU (sensor shards: ranks never wait on one another); see tools/emulate_ranks.py")
    ap.add_argument("--emulate-rank", type=int, default=0)
    ap.add_argument("--merge", choices=["allreduce", "reduce_scatter", "nvls"], default="allreduce",
                    help="triangle-shard merge inside grca_cast: NCCL all-reduce(MIN) of the packed keys, "
                         "reduce-scatter(MIN) (each rank keeps its ray slice; half the traffic), or the fused NVLS "
                         "multimem.red.min into an NCCL symmetric window (NEXT-f3; needs NVLS multicast)")
    ap.add_argument("--no-graph", action="store_true", help="plain launches instead of GRCA_USE_CUDA_GRAPH (each cast "
                    "as one CUDA graph, the default: C4 1.053 vs 1.064 ms, C2 0.105 vs 0.115 ms)")
    ap.add_argument("--logic-check", action="store_true", help="N > 1 on one GPU over gloo with virtual-rank handles: "
                    "a check of the multi-rank host logic, not a measurement")
    ap.add_argument("--collective", action="store_true", help="N=1: cast through a one-rank NCCL communicator "
                    "(the library's collective path, merge included) instead of a plain handle")
    ap.add_argument("--e2e-vertices", action="store_true", help="e2e uploads the posed car vertices (54.5 MB per C4 "
                    "frame) instead of one 3x4 matrix per car")
    ap.add_argument("--instances", action="store_true", help="cars as rigid instances (grca_update_instances): a frame's "
                    "input is one 3x4 matrix per car (e2e upload 1.4 KB instead of 54.5 MB of posed vertices)")
    ap.add_argument("--soup", action="store_true", help="triangle-soup scene (float4 triplets) instead of the indexed "
                    "car meshes (same triangles; the e2e upload is then every dynamic triangle's vertices)")
    ap.add_argument("--shard", default="auto", choices=["auto", "triangles", "emitters", "mixed"])
    ap.add_argument("--emitter-groups", type=int, default=2, help="--shard mixed: emitter groups (each split "
                    "into world / groups triangle shards merged within the group)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        w = sg.workload(args.config, frame=0, deformation=args.deformation)
        n_rays = sg.n_rays_total(w["emitters"])
        import oracle

        threads = os.cpu_count() or 1
        cal, _ = time_oracle(w["emitters"], w["tris"], target_s=2.0, max_rays=256)
        per_step = max(1, int(cal["value"] * 120.0 / max(1, args.steps + args.warmup)))
        vals = []
        for k in range(args.warmup + args.steps):
            rays = oracle_sample(w["emitters"], w["tris"], per_step, 100 + k)
            t0 = time.perf_counter()
            oracle.cast(w["emitters"], w["tris"], rays=rays, threads=threads)
            dt = time.perf_counter() - t0
            if k >= args.warmup:
                vals.append(per_step / dt)
        v = float(np.median(vals))
        steps = [{"kind": "oracle", "cores": threads,
                  "sample": f"{per_step} seeded rays per step x all {len(w['tris'])} triangles (fp64 brute force)"}]
        line = {
            "impl": "reference", "metric": "rays/s", "value": v, "unit": "rays/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * n_rays / v,
            "ms_per_step_kind": (f"extrapolated: each step times {per_step} sampled rays of the frame; ms_per_step = "
                                 f"{n_rays} rays per frame / the median sampled rate"),
            "sampled_rays_per_step": per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "rays_per_frame": n_rays, "triangles": int(len(w["tris"])),
                       "deformation": args.deformation},
            "cpu_baseline": {k: steps[-1][k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": "rays/s"},
            "e2e": {"value": v, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist

    from paper_2605_10457_b200 import build as B
    if local_rank == 0:
        B.build()   # no-op when libgrca.so is up to date; a fresh checkout compiles it (nvcc, sm_100a)
    else:
        for _ in range(600):   # the other local ranks wait for rank 0's build
            if os.path.exists(B.LIB):
                break
            time.sleep(1.0)
    from paper_2605_10457_b200 import Grca, tris_to_float4
    from paper_2605_10457_b200 import dist as D
    from paper_2605_10457_b200 import grca as G

    # --logic-check: several ranks on ONE GPU over gloo, handles in virtual-rank mode (no NCCL: it refuses two
    # ranks on one device) -- exercises the N > 1 host logic (partitions, e2e split / all-gather / readback
    # ranges, timing); not a measurement, and triangle shards are left unmerged
    logic = world > 1 and args.logic_check
    dev_index = local_rank % max(1, torch.cuda.device_count()) if logic else local_rank
    if world > 1:
        torch.cuda.set_device(dev_index)
        if logic:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev_index}"))
    device = torch.device(f"cuda:{dev_index}")
    torch.cuda.set_device(device)
    # one non-default stream for everything (scene set-up, casts, events): a stream the library can capture
    # into a CUDA graph (--graph), unlike the legacy default stream
    torch.cuda.set_stream(torch.cuda.Stream(device))
    # --emulate-world W --emulate-rank R: this process does exactly rank R's share of a W-rank run
    # (its shard of the scene, no process group).  Valid for sensor shards, whose ranks never wait on
    # one another; tools/emulate_ranks.py runs every rank and takes the slowest (projected frame).
    s_rank, s_world = (args.emulate_rank, args.emulate_world) if args.emulate_world > 1 else (rank, world)
    if args.emulate_world > 1:
        args.no_e2e = args.no_hybrid = args.no_cpu_baseline = True
    n_em_total = len(sg.workload(args.config)["emitters"]) if args.config == "C1" else sg.WORKLOADS[args.config][0]
    shard = args.shard if args.shard != "auto" else (D.choose_mode(n_em_total, s_world) if s_world > 1 else "triangles")
    if shard == "mixed":
        shard = f"mixed:{args.emitter_groups}"

    car_scale = tuple(float(x) for x in args.car_scale.split(",")) if args.car_scale else None
    scene = Scene(args.config, s_rank, s_world, device, args.deformation, shard=shard,
                  max_range=(None if args.max_range == 0 else args.max_range), subdiv=args.subdiv, car_scale=car_scale,
                  mesh="soup" if args.soup else "instances" if args.instances else "indexed")
    # The library casts the partition itself: sensor shards pass EVERY emitter (the handle casts n mod P),
    # triangle shards pass every emitter and their own triangles, a mixed partition passes its group's
    # emitters and its triangle shard; grca_cast is collective and merges in-stream (NCCL).
    ems = scene.emitters                               # the emitters this rank casts
    ems_lib = scene.w["emitters"] if shard == "emitters" else ems
    n_rays = sg.n_rays_total(ems_lib)                   # output layout of the handle
    n_rays_job = sg.n_rays_total(scene.w["emitters"])
    mode_flags = ((G.DEBUG_SPLIT_REFINE if args.split_refine else 0) | (G.L2_PERSIST if args.l2_persist else 0)
                  | (G.DEBUG_NO_PACKED if args.no_packed else 0) | (0 if args.no_graph else G.USE_CUDA_GRAPH))
    shard_mode = G.SHARD_EMITTERS if shard == "emitters" else G.SHARD_TRIANGLES
    merge_mode = {"allreduce": G.MERGE_ALLREDUCE, "reduce_scatter": G.MERGE_REDUCE_SCATTER, "nvls": G.MERGE_NVLS}[args.merge]
    coll_group, c_ranks, c_rank = None, 1, 0
    if world > 1:
        c_ranks, c_rank = world, rank
        if shard.startswith("mixed"):   # one communicator per emitter group (its T triangle shards)
            n_groups = int(shard.split(":")[1])
            gi, ti, T = D.mixed_partition(rank, world, n_groups)
            subs = [dist.new_group(ranks=[gg * T + t for t in range(T)]) for gg in range(n_groups)]
            coll_group, c_ranks, c_rank = subs[gi], T, ti
        if logic:
            mode_flags |= G.DEBUG_VIRTUAL_RANKS
    elif args.emulate_world > 1:        # this rank's exact share, no collective (library virtual ranks)
        c_ranks, c_rank = s_world, s_rank
        mode_flags |= G.DEBUG_VIRTUAL_RANKS
    collective = (world > 1 and not logic) or args.collective

    def new_handle(flags):
        uid = None
        if world > 1 and not logic:
            uid = D.nccl_uid(coll_group)
        elif args.collective:
            uid = G.nccl_unique_id()
        h = Grca(device=dev_index, max_triangles=scene.n_tri, max_rays=n_rays, debug_flags=flags,
                 small_max=args.small_max, nranks=c_ranks, rank=c_rank, nccl_uid=uid, shard_mode=shard_mode,
                 merge=merge_mode if (collective or c_ranks > 1) else G.MERGE_ALLREDUCE)
        h.set_emitters(ems_lib)
        return h

    # the timed handle is uninstrumented (what a user runs); the per-kernel breakdown comes from a
    # second, profiled handle afterwards (CUDA events around every kernel)
    g = new_handle(mode_flags)
    shard_info = g.get_shard()
    nvls = collective and args.merge == "nvls" and shard_mode == G.SHARD_TRIANGLES
    dist_out = torch.empty(n_rays, dtype=torch.float32, device=device)
    tri_out = torch.empty(n_rays, dtype=torch.int32, device=device)

    def cast_once(dout=dist_out, tout=tri_out):
        g.cast(dout, tout)   # collective with a communicator: K0..K4, in-stream merge, K5

    def step(k):
        scene.bind(g, scene.frames[k % N_FRAMES])
        cast_once()

    stream = torch.cuda.current_stream(device)
    pk = measured_peaks()   # roofline denominators, measured on this GPU before the timed region
    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    stats = g.get_stats()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.15)
    barrier()
    # per-frame events on the launch stream (frame pacing) inside the timed region
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for k in range(args.steps):
        step(k)
        evs[k + 1].record(stream)
    barrier()
    clk = clocks.stop()
    ms = evs[0].elapsed_time(evs[-1])
    frame_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    if args.steps < 50:   # the pacing statistics use >= 50 frames (the paper's 50-frame sections)
        extra = [torch.cuda.Event(enable_timing=True) for _ in range(50 - args.steps + 1)]
        extra[0].record(stream)
        for k in range(len(extra) - 1):
            step(args.steps + k)
            extra[k + 1].record(stream)
        torch.cuda.synchronize()
        frame_ms += [extra[k].elapsed_time(extra[k + 1]) for k in range(len(extra) - 1)]
    fm = np.asarray(frame_ms)
    mu = float(fm.mean())
    pacing = {"frames": int(fm.size), "median_ms": float(np.median(fm)), "mean_ms": mu,
              "p95_ms": float(np.percentile(fm, 95)), "min_ms": float(fm.min()), "max_ms": float(fm.max()),
              "within_20pct_of_mean": float(np.mean(np.abs(fm - mu) <= 0.2 * mu)),
              "below_mean": float(np.mean(fm < mu)),
              "note": "per-frame CUDA events on the launch stream; +-20 % and < mu as in PAPER.md Table frame_pacing "
                      "(P:1588-1614); frames beyond --steps (if < 50) are timed after the headline region"}
    # per-kernel breakdown: the same casts on a profiled handle (not part of the timed region)
    gp = new_handle(mode_flags | G.PROFILE_KERNELS)
    n_last = min(max(args.steps, 8), 64)
    for k in range(n_last + 2):
        scene.bind(gp, scene.frames[k % N_FRAMES])
        gp.cast(dist_out, tri_out)
    torch.cuda.synchronize()
    kt = gp.kernel_times(n_last)
    kms = [x / n_last for x in kt]
    gp.close()
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    rays_s = n_rays_job * args.steps / (ms / 1e3)   # whole job: every rank's rays of the frame

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region.
    # Pipelined over frames with double buffers: the H2D of frame k+1 (copy stream) and the D2H of
    # frame k-1's (dist, id) (second copy stream) overlap the cast of frame k; every step's copies
    # are inside the timed region (which starts before the first H2D and ends after the last D2H).
    e2e = None
    if not args.no_e2e:
        # rigid cars: the e2e input is one 3x4 matrix per car per frame (grca_update_instances), the natural host
        # input for the paper's rigid dynamic instances; --e2e-vertices (or a layout without whole instances on
        # this rank) uploads the posed vertices instead
        es = scene
        if not args.e2e_vertices and scene.indexed and scene.identity:
            es = Scene(args.config, s_rank, s_world, device, args.deformation, shard=shard,
                       max_range=(None if args.max_range == 0 else args.max_range), subdiv=args.subdiv,
                       car_scale=car_scale, mesh="instances", w=scene.w)
        # N > 1: each rank uploads 1/N of the dynamic vertices over its own PCIe link and an
        # all-gather over NVLink assembles the rest (inside the timed region); each rank reads back
        # only its own results (sensor shards: its emitters' rays; triangle shards: 1/N of the rays)
        ns3 = es.fs                                  # static rows carried in a frame buffer
        comps = es.frames[0].shape[1]
        n_dyn = es.frames[0].shape[0] - ns3          # dynamic vertices per frame
        # split only when every rank needs the same dynamic data (indexed scene: all car vertices;
        # sensor shards: all triangles); a triangle-sharded soup holds per-rank data
        split = world > 1 and (es.indexed or shard == "emitters")
        nsplit = world if split else 1
        chunk = -(-n_dyn // nsplit)                     # per-rank upload slice (padded)
        lo_v = (rank if split else 0) * chunk
        n_mine = max(0, min(chunk, n_dyn - lo_v))
        host_dyn = []
        for f in range(N_FRAMES):
            hs = torch.zeros((chunk, comps), dtype=torch.float32)
            hs[:n_mine] = es.frames[f][ns3 + lo_v: ns3 + lo_v + n_mine].cpu()
            host_dyn.append(hs.pin_memory())
        dev_bufs = []
        for _ in range(2):   # static part resident; dynamic part (padded to world * chunk) uploaded
            db = torch.zeros((ns3 + chunk * nsplit, comps), dtype=torch.float32, device=device)
            db[:ns3] = es.frames[0][:ns3]
            dev_bufs.append(db)
        outs = [(torch.empty(n_rays, dtype=torch.float32, device=device),
                 torch.empty(n_rays, dtype=torch.int32, device=device)) for _ in range(2)]
        # rays this rank reads back (grca_get_shard): emitter shards their emitters' slices, a reduce-scatter
        # its merged slice, an all-reduce group 1/T of the merged rays each, one GPU everything
        if shard_info["first_ray"] == -1:
            ranges = [(g.offsets[m], g.offsets[m + 1] - g.offsets[m]) for m in range(len(ems_lib)) if m % c_ranks == c_rank]
        elif shard_info["n_written"] < n_rays:
            ranges = [(shard_info["first_ray"], shard_info["n_written"])]
        elif c_ranks > 1:
            rch = -(-n_rays // c_ranks)
            ranges = [(c_rank * rch, max(0, min(rch, n_rays - c_rank * rch)))]
        else:
            ranges = [(0, n_rays)]
        r_n = sum(n for _, n in ranges)
        host_out = [(torch.empty(r_n, dtype=torch.float32).pin_memory(),
                     torch.empty(r_n, dtype=torch.int32).pin_memory()) for _ in range(2)]
        cs, ds = torch.cuda.Stream(device), torch.cuda.Stream(device)
        ev_h2d = [torch.cuda.Event() for _ in range(2)]
        ev_cast = [torch.cuda.Event() for _ in range(2)]
        ev_d2h = [torch.cuda.Event() for _ in range(2)]
        k_e2e = max(50, min(args.steps, 200))   # >= 50 frames, like the headline pacing

        def issue_h2d(k):
            b = k % 2
            with torch.cuda.stream(cs):
                if k >= 2:
                    cs.wait_event(ev_cast[b])   # cast k-2 has released buffer b
                dyn = dev_bufs[b][ns3:]
                mine = dyn[lo_v: lo_v + chunk]
                mine.copy_(host_dyn[k % N_FRAMES], non_blocking=True)
                if split:   # in place: this rank's slice sits at rank * chunk of the output
                    dist.all_gather_into_tensor(dyn, mine)
                ev_h2d[b].record(cs)

        def run_e2e(n):
            for k in range(n):
                b = k % 2
                if k == 0:
                    issue_h2d(0)
                stream.wait_event(ev_h2d[b])
                if k >= 2:
                    stream.wait_event(ev_d2h[b])   # host copy of step k-2 done with outs[b]
                es.bind(g, dev_bufs[b], n_triangles=es.n_tri)
                cast_once(*outs[b])
                ev_cast[b].record(stream)
                if k + 1 < n:
                    issue_h2d(k + 1)
                with torch.cuda.stream(ds):
                    ds.wait_event(ev_cast[b])
                    pos = 0
                    for lo, nn in ranges:
                        host_out[b][0][pos: pos + nn].copy_(outs[b][0][lo: lo + nn], non_blocking=True)
                        host_out[b][1][pos: pos + nn].copy_(outs[b][1][lo: lo + nn], non_blocking=True)
                        pos += nn
                    ev_d2h[b].record(ds)
            stream.wait_stream(cs)
            stream.wait_stream(ds)

        run_e2e(4)   # warm-up
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        cs.wait_stream(stream)
        ds.wait_stream(stream)
        run_e2e(k_e2e)
        f1.record(stream)
        barrier()
        ems_e2e = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([ems_e2e], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems_e2e = float(t.item())
        # the host results are the cast's (checked on the last step), and the gathered frame equals
        # the resident one
        last = (k_e2e - 1) % 2
        assert torch.equal(host_out[last][1], torch.cat([outs[last][1][lo: lo + nn] for lo, nn in ranges]).cpu())
        fr = (k_e2e - 1) % N_FRAMES
        assert torch.equal(dev_bufs[last][ns3: ns3 + n_dyn], es.frames[fr][ns3:])
        e2e = {"value": n_rays_job * k_e2e / (ems_e2e / 1e3), "unit": "rays/s", "ms_per_step": ems_e2e / k_e2e,
               "h2d_bytes_per_step": int(chunk * comps * 4), "d2h_bytes_per_step": int(r_n * 8), "steps": k_e2e,
               "bytes_scope": "per rank" if world > 1 else "job",
               "what": (f"pinned H2D of this frame's car poses (one 3x4 matrix per car: rigid instances, "
                        f"grca_update_instances" if es.instanced else
                        f"pinned H2D of this frame's dynamic vertices ({es.mesh} mesh") +
                       f"{', 1/N per rank + NVLink all-gather' if split else ''}) + grca_cast + D2H of "
                       "(dist, id) per ray; pipelined over frames (double buffers, H2D/D2H on two copy "
                       "streams overlap the previous/next cast)"}
        del dev_bufs
        if es is not scene:
            del es

    # ---- hybrid static/dynamic (NEXT-f2; NOT the headline: static triangles cached across frames)
    hybrid = None
    if world == 1 and not args.no_hybrid and scene.n_static_local > 0:
        gh = Grca(device=dev_index, max_triangles=scene.n_tri, max_rays=n_rays)
        gh.set_emitters(ems)
        ns3 = scene.fs
        st4 = scene.static_soup if scene.indexed else scene.frames[0][:ns3]   # float4 triplets
        if scene.identity:
            gh.set_static_triangles(st4, tri_id_base=0)
            dyn_ids, dyn_base = None, scene.n_static_local
        else:
            gh.set_static_triangles(st4, tri_ids=scene.ids[: scene.n_static_local])
            dyn_ids, dyn_base = scene.ids[scene.n_static_local:], 0

        def hstep(k):
            if scene.instanced:   # the dynamic set is only the instances (ids after the static ones)
                gh.update_scene(tri_id_base=dyn_base)
                gh.update_instances(scene.car_v_dev, scene.car_f_dev, scene.frames[k % N_FRAMES].view(-1, 3, 4))
            else:
                gh.update_triangles(scene.frames[k % N_FRAMES][ns3:], indices=scene.idx_dyn, tri_ids=dyn_ids,
                                    tri_id_base=dyn_base)
            gh.cast(dist_out, tri_out)

        for k in range(3):
            hstep(k)
        barrier()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kh = max(4, min(args.steps, 100))
        h0.record(stream)
        for k in range(kh):
            hstep(k)
        h1.record(stream)
        barrier()
        hms = h0.elapsed_time(h1) / kh
        hybrid = {"ms_per_step": hms, "value": n_rays_job / (hms / 1e3), "unit": "rays/s", "steps": kh,
                  "static_triangles": int(scene.n_static_local), "dynamic_triangles": int(scene.n_tri - scene.n_static_local),
                  "note": "static triangles cast once into cached per-ray keys (emitters static); each frame culls "
                          "only the dynamic ones -- exact (min-lattice); context, not the headline (PAPER.md:2077-2085)"}
        gh.close()

    # our kernels per cast (cf. the ncu launch list): K0, K2, fused K2b+K4s (split: K2b and K4s),
    # K3, K4, K5; the fused NVLS merge adds its two barrier kernels
    launches_per_cast = 6 + (1 if args.split_refine else 0) + (2 if nvls else 0)
    # ---- per-kernel roofline (per-kernel CUDA events on the launch stream, last <= 64 steps)
    kernel_ms = {n: kms[i] for i, n in enumerate(KERNELS)}
    roof = kernel_rooflines(kernel_ms, stats, n_rays, pk, scene.tri_bytes, split=args.split_refine)
    froof = frame_roofline(roof, ms_step, n_rays, scene.tri_bytes, pk)
    dom = max(roof, key=lambda n: kernel_ms[n])
    roofline = dict(roof[dom])
    roofline["kernel"] = dom

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        # the GPU result of frame 0 (the frame the oracle sample below is drawn from: scene frames equal
        # scenegen.workload(config, frame) bit for bit), cast by the timed handle
        scene.bind(g, scene.frames[0])
        cast_once()
        torch.cuda.synchronize()
        gd, gt = dist_out.cpu().numpy(), tri_out.cpu().numpy()
        tris_np = scene.frame_tris(0, scene.w["tris"])
        cpu, ref = time_oracle(ems_lib, tris_np, target_s=15.0)
        rep = oracle.compare(ems_lib, tris_np, gd[ref["rays"]], gt[ref["rays"]], ref)
        parity = {k: rep[k] for k in ("rays", "agree_frac", "disagree", "excused", "unexcused", "near_ties",
                                      "oracle_hits", "hit_pct_1mm", "passed")}
        parity["what"] = ("frame 0 of the timed handle vs the cpu_baseline's oracle rays (same sample), north-star "
                          "comparator (oracle/compare.py)")

    if rank == 0:
        culled = 1.0 - stats["rtic_tested"] / max(1, stats["rtic_brute"])
        line = {
            "metric": "rays/s", "value": rays_s, "unit": "rays/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": args.config, "emitters": len(scene.w["emitters"]), "rays_per_frame": n_rays_job,
                       "triangles": scene.n_tri_global, "dynamic_triangles": int(scene.w["n_dynamic"]),
                       "deformation": args.deformation, "max_range_m": float(ems[0].max_range),
                       "subdiv": args.subdiv, "car_scale": list(scene.scale), "mesh": scene.mesh,
                       "sharding": ("none" if world == 1 else
                                    f"triangles block-interleaved ({D.BLOCK}) + "
                                    f"{'fused NVLS multimem.red.min' if nvls else 'reduce-scatter(MIN), ray-sharded output' if args.merge == 'reduce_scatter' else 'all-reduce(MIN)'} x {world}"
                                    if shard == "triangles" else
                                    f"{shard.split(':')[1]} emitter groups x {world // int(shard.split(':')[1])} "
                                    f"triangle shards, all-reduce(MIN) within a group"
                                    if shard.startswith("mixed") else f"emitters (n mod P) x {world}, no reduction"),
                       "l2": (f"inputs > L2: every cast streams the resident {scene.static_soup.numel() * 4 / 1e9:.2f} GB "
                              f"static float4 soup; the cars are rigid instances of one local mesh ("
                              f"{(scene.car_v_np.nbytes + scene.car_f_np.nbytes) / 1e6:.1f} MB) posed by one of {N_FRAMES} "
                              f"cycled sets of {scene.n_cars} 3x4 matrices"
                              if scene.instanced else
                              f"inputs > L2: every cast streams the resident {scene.static_soup.numel() * 4 / 1e9:.2f} GB "
                              f"static float4 soup + {scene.idx_dyn.numel() * 4 / 1e9:.3f} GB car indices + one of "
                              f"{N_FRAMES} cycled {scene.frames[0].numel() * 4 / 1e9:.3f} GB car-vertex frames"
                              if scene.indexed else
                              f"inputs > L2: {N_FRAMES} resident frame buffers of "
                              f"{scene.frames[0].numel() * 4 / 1e9:.2f} GB cycled")},
            "frame_ms": ms_step, "rtic_culled_frac": culled,
            "rtic_tested_per_frame": stats["rtic_tested"], "rtic_brute_per_frame": stats["rtic_brute"],
            "rtic_per_s": stats["rtic_tested"] / (ms_step / 1e3),
            "rtic_effective_per_s": n_rays_job * scene.n_tri_global / (ms_step / 1e3),
            "stats_scope": "rank 0" if world > 1 else "job",
            "kernel_ms": kernel_ms,
            "kernel_roofline": {k: {kk: v[kk] for kk in ("bound", "achieved", "unit", "frac", "hbm_achieved_gbs",
                                                         "hbm_frac", "red_min_per_s", "red_min_frac") if kk in v}
                                for k, v in roof.items()},
            "frame_roofline": froof, "frame_pacing": pacing,
            "peaks": {k: pk[k] for k in ("hbm_gbs", "src_hbm", "ffma_lane_instr_per_s", "ffma2_lane_instr_per_s",
                                         "red_min_u64_random_per_s", "red_min_u64_coalesced_per_s", "src") if k in pk},
            "stats": {k: stats[k] for k in ("prefilter_survivors", "rtic_small",
                "pairs", "range_culled", "channel_culled", "azimuth_culled", "survivors", "small_pairs", "large_pairs",
                "chunks", "fp64_fallbacks", "hits_recorded", "hits_large", "overflow")},
            "roofline": roofline, "gpu_launches": launches_per_cast * args.steps, "clocks": clk,
            "e2e": e2e, "cpu_baseline": cpu, "parity": parity, "hybrid_static_cache": hybrid,
            "emulated": ({"rank": s_rank, "world": s_world, "shard": shard, "rank_rays": n_rays,
                          "note": "this rank's share of a W-rank run on one GPU (no merge timed)"}
                         if args.emulate_world > 1 else None),
            "context": "paper (PAPER.md:1758-1762): GRCA_GPU 10.7 ms/frame on RTX 5090 for PP30 Omega=8 "
                       "(3.9e8 rays/s), 1.98x OptiX 9.1; other hardware, not a target",
        }
        print(json.dumps(line))
    torch.cuda.synchronize()
    g.close()   # (its NCCL communicator, if any, before the process group)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
