"""Per-source-line totals of one kernel from an `ncu --import-source on` report (dev tooling):

    python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> [--top 40] [--per N]

Aggregates the cuda,sass source view: warp instructions executed and warp-stall samples of every SASS
instruction, attributed to the CUDA source line it belongs to (file:line), sorted by instructions.
--per N divides instruction counts by N (e.g. the number of 32-survivor rounds)."""
import argparse
import collections
import csv
import io
import os
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--per", type=float, default=0)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          "regex:" + a.kernel], capture_output=True, text=True).stdout
    agg = collections.defaultdict(lambda: [0, 0, ""])
    fname, line, src = "?", "?", ""
    cols = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = os.path.basename(row[1])
            continue
        if row[0] == "Line No":
            cols = row
            continue
        if cols is None or len(row) < 8:
            continue
        if row[0]:
            line, src = row[0], row[1]
            continue
        if row[2] in ("...", "-"):
            continue
        d = dict(zip(cols[2:], row[2:]))
        try:
            ie = float(d.get("Instructions Executed", "0") or 0)
            ss = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        k = f"{fname}:{line}"
        agg[k][0] += ie
        agg[k][1] += ss
        agg[k][2] = src.strip()[:90]
    tot_i = sum(v[0] for v in agg.values()) or 1
    tot_s = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
    print(f"{'line':28s} {'instr %':>8s} {'per unit':>9s} {'stall %':>8s}  source")
    for k, (i, s_, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: a.top]:
        per = f"{i / a.per:9.1f}" if a.per else ""
        print(f"{k:28s} {100 * i / tot_i:8.2f} {per:>9s} {100 * s_ / tot_s:8.2f}  {src}")


if __name__ == "__main__":
    main()
