"""bench.py's roofline arithmetic on CPU (no GPU): the per-kernel and frame fractions follow SURVEY 8(d)'s
per-unit counts and can be recomputed by hand from the printed inputs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _inputs():
    kms = {"K0_init": 0.0105, "K2_cull": 0.4845, "K2b_refine": 0.0027, "K4s_small": 0.5084, "K3_bin": 0.0222,
           "K4_large": 0.0315, "K5_unpack": 0.0145}
    st = {"pairs": 174335088, "prefilter_survivors": 8532271, "rtic_small": 26029994, "rtic_tested": 28726612,
          "large_pairs": 2457, "hits_recorded": 7675336, "hits_large": 500000}
    pk = json.load(open(os.path.join(ROOT, "profiles", "r02_peaks.json")))
    pk.update(bench.peaks())
    pk["src"] = "test"
    return kms, st, pk


def test_kernel_rooflines_follow_8d_units():
    kms, st, pk = _inputs()
    n_rays, tri_bytes = 4194304, 774_000_000
    roof = bench.kernel_rooflines(kms, st, n_rays, pk, tri_bytes)
    alu = pk["ffma_lane_instr_per_s"]
    k2 = roof["K2_cull"]
    assert k2["algorithmic_per_launch"] == 50 * st["pairs"]
    assert abs(k2["frac"] - 50 * st["pairs"] / (kms["K2_cull"] * 1e-3) / alu) < 1e-12
    fused = roof["K4s_small"]
    assert fused["algorithmic_per_launch"] == 325 * st["prefilter_survivors"] + 25 * st["rtic_small"]
    assert abs(fused["frac"] - fused["algorithmic_per_launch"] / (kms["K4s_small"] * 1e-3) / alu) < 1e-12
    assert abs(fused["red_min_per_s"] - (st["hits_recorded"] - st["hits_large"]) / (kms["K4s_small"] * 1e-3)) < 1
    assert roof["K4_large"]["algorithmic_per_launch"] == 25 * (st["rtic_tested"] - st["rtic_small"])
    assert roof["K5_unpack"]["algorithmic_per_launch"] == 16 * n_rays and roof["K5_unpack"]["unit"] == "GB/s"
    assert abs(k2["hbm_frac"] - tri_bytes / (kms["K2_cull"] * 1e-3) / 1e9 / pk["hbm_gbs"]) < 1e-12
    fr = bench.frame_roofline(roof, 1.06, n_rays, tri_bytes, pk)
    alu_total = sum(v["algorithmic_per_launch"] for v in roof.values() if v["bound"] == "alu")
    assert abs(fr["t_alu_floor_ms"] - alu_total / alu * 1e3) < 1e-12
    assert abs(fr["t_hbm_floor_ms"] - (tri_bytes + 24 * n_rays) / (pk["hbm_gbs"] * 1e9) * 1e3) < 1e-12
    assert abs(fr["frac"] - max(fr["t_alu_floor_ms"], fr["t_hbm_floor_ms"]) / 1.06) < 1e-12
    assert 0 < fr["frac"] < 1


def test_traffic_from_the_latest_full_capture():
    # the round's final capture (rNN_) outranks its mid-round snapshots (rNNb_, ...) and every earlier round
    _, src = bench.ncu_traffic()
    names = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_traffic.json"))
    last_round = max(int(f[1:3]) for f in names)
    assert src == f"r{last_round:02d}_traffic.json" or (src.startswith(f"r{last_round:02d}")
                                                        and f"r{last_round:02d}_traffic.json" not in names)
