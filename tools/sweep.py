"""Config sweeps of BASELINE.json configs C2/C3/C5: frame time, rays/s, culling.

    python tools/sweep.py [--steps 20] [--out profiles/rNN_sweeps.md]

Runs bench.py once per point (1 GPU, device-timed, no CPU baseline / e2e) and tabulates
  * C5: car subdivision 0..3 at scale 1 (0.3M..19.3M dynamic triangles) + the large-triangle
    variant (scale U[1,30]) -- culling efficiency vs triangle size (PAPER.md:1358-1416 analog);
  * C3: 4 LiDARs mixed 360/180 deg, range 10 / 50 / 100 m / unlimited (PAPER.md:1503-1578 analog);
  * C2: ND vs SWD deformation.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

POINTS = [
    ("C5 subdiv 0 (scale 1)", ["--config", "C5", "--subdiv", "0"]),
    ("C5 subdiv 1 (scale 1)", ["--config", "C5", "--subdiv", "1"]),
    ("C5 subdiv 2 (scale 1)", ["--config", "C5", "--subdiv", "2"]),
    ("C5 subdiv 3 (scale 1)", ["--config", "C5", "--subdiv", "3"]),
    ("C5 large triangles (scale U[1,30])", ["--config", "C5", "--car-scale", "1,30"]),
    ("C3 range 10 m", ["--config", "C3", "--max-range", "10"]),
    ("C3 range 50 m", ["--config", "C3", "--max-range", "50"]),
    ("C3 range 100 m", ["--config", "C3", "--max-range", "100"]),
    ("C3 unlimited", ["--config", "C3", "--max-range", "0"]),
    ("C2 ND", ["--config", "C2"]),
    ("C2 SWD", ["--config", "C2", "--deformation", "SWD"]),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweeps.md"))
    args = ap.parse_args()
    rows = []
    for name, extra in POINTS:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(args.steps), "--warmup", "3",
               "--no-cpu-baseline", "--no-e2e"] + extra
        p = subprocess.run(cmd, capture_output=True, text=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("{")]
        if p.returncode or not line:
            rows.append((name, None, p.stderr[-300:]))
            continue
        rows.append((name, json.loads(line[-1]), ""))
        print(name, "done", flush=True)
    out = ["# Config sweeps (1 B200, device-timed; bench.py per point)", "",
           "| point | triangles | rays | ms/frame | rays/s | culled vs Eq. 1 | K2 survivors | final survivors | "
           "candidates | cand./survivor |", "|---|---|---|---|---|---|---|---|---|---|"]
    for name, d, err in rows:
        if d is None:
            out.append(f"| {name} | failed: {err.strip()[:80]} | | | | | | | | |")
            continue
        st = d["stats"]
        cps = d["rtic_tested_per_frame"] / max(1, st["survivors"])
        out.append(f"| {name} | {d['config']['triangles']:,} | {d['config']['rays_per_frame']:,} | {d['ms_per_step']:.3f} | "
                   f"{d['value']:.3e} | {100 * d['rtic_culled_frac']:.5f} % | {st['prefilter_survivors']:,} | "
                   f"{st['survivors']:,} | {d['rtic_tested_per_frame']:,} | {cps:.1f} |")
    open(args.out, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
