"""Projected multi-GPU frame times on one GPU (dev tooling).

    python tools/emulate_ranks.py [--worlds 2,4,8] [--steps 300] [--shard emitters] [--out profiles/....md]

For each W, runs bench.py --emulate-world W --emulate-rank r for every rank r (sequentially, one
process at a time, nothing waiting on anything): each run times exactly that rank's share of the C4
frame.  Under sensor sharding (the default for C4 at W | 8) the ranks never exchange data, so the
projected W-GPU frame time is the slowest rank's.  Triangle shards additionally need the
all-reduce(MIN) merge (not timed here).  A projection for planning, not a multi-GPU measurement.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--shard", default="auto")
    ap.add_argument("--emitter-groups", type=int, default=2)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows, data = [], {}
    base = None
    for W in [1] + [int(x) for x in args.worlds.split(",")]:
        per = []
        for r in range(W):
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", args.config, "--steps", str(args.steps),
                   "--warmup", "5", "--no-cpu-baseline", "--no-e2e", "--no-hybrid", "--shard", args.shard if W > 1 else "auto",
                   "--emitter-groups", str(args.emitter_groups)]
            if W > 1:
                cmd += ["--emulate-world", str(W), "--emulate-rank", str(r)]
            p = subprocess.run(cmd, capture_output=True, text=True)
            line = [l for l in p.stdout.splitlines() if l.startswith("{")]
            if p.returncode or not line:
                raise SystemExit(f"W={W} r={r} failed: {p.stderr[-400:]}")
            d = json.loads(line[-1])
            per.append(d["ms_per_step"])
            n_rays_job = d["config"]["rays_per_frame"]
            shard = (d.get("emulated") or {}).get("shard", "none")
        worst = max(per)
        base = base or worst
        data[W] = {"per_rank_ms": per, "frame_ms": worst, "rays_per_s": n_rays_job / (worst / 1e3), "shard": shard}
        rows.append(f"| {W} | {shard} | {worst:.3f} | {n_rays_job / (worst / 1e3):.3e} | {base / worst / W:.2f} | "
                    f"{', '.join(f'{x:.3f}' for x in per)} |")
        print(W, data[W], flush=True)
    md = ["# Projected multi-GPU frame times (one B200, ranks emulated one at a time)", "",
          f"`tools/emulate_ranks.py --config {args.config} --steps {args.steps}`: each rank's share timed alone "
          "(sensor shards never exchange data: the projected frame is the slowest rank). Not a multi-GPU "
          "measurement.", "",
          "| GPUs | sharding | projected frame ms | rays/s | efficiency | per-rank ms |", "|---|---|---|---|---|---|"] + rows
    if args.out:
        open(args.out, "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
