"""Summarize ncu captures into profiles/ (dev tooling; reads gpurun_out/ artifacts).

    python tools/ncu_summarize.py launches <launches.csv> <out.md>
    python tools/ncu_summarize.py full <prof.ncu-rep> <out.md> [<traffic.json>]
"""
import collections
import re
import csv
import json
import subprocess
import sys

KEEP = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Executed Instructions", "Avg. Active Threads Per Warp", "Eligible Warps Per Scheduler",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       # L2 atomics / reductions (the closest-hit RED.MIN keys): sectors and requests
       "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_requests_srcunit_tex_op_red.sum",
       "lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed",
       "lts__t_sectors_srcunit_tex_op_atom.sum", "smsp__inst_executed_op_global_red.sum"]


def launches(path, out, cmd="bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-hybrid"):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        agg.setdefault(name, []).append(float(d["Metric Value"]))
    # the library's kernels (namespace grca); bench.py's measured-peak microbenchmarks (tools/peaks.cu) excluded
    ours = {k: v for k, v in agg.items() if re.match(r"(void )?grca::k_", k)}
    med = {k: sorted(v)[len(v) // 2] for k, v in ours.items()}
    step_ns = sum(med.values())
    lines = [f"# ncu launch list ({path.split('/')[-1]})", "",
             f"`ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_` over `{cmd}`;",
             "cold-cache, serialized launches: compare SHARES of the step, not absolutes.", "",
             "| kernel | launches | median us | min us | max us | share of step (medians) |", "|---|---|---|---|---|---|"]
    for k, v in ours.items():
        lines.append(f"| {k} | {len(v)} | {med[k] / 1e3:.1f} | {min(v) / 1e3:.1f} | {max(v) / 1e3:.1f} | "
                     f"{100 * med[k] / step_ns:.1f} % |")
    lines.append(f"| **step (sum of medians)** | | {step_ns / 1e3:.1f} | | | 100 % |")
    others = sum(len(v) for k, v in agg.items() if k not in ours)
    lines += ["", f"Other (harness / torch) launches in the capture: {others}."]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, traffic_json=None):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(det.splitlines()))
    hdr = r[0]
    per = collections.OrderedDict()
    for row in r[1:]:
        d = dict(zip(hdr, row))
        k = (d["ID"], d["Kernel Name"].split("(")[0])
        if d["Metric Name"] in KEEP:
            per.setdefault(k, {})[d["Metric Name"]] = f'{d["Metric Value"]} {d.get("Metric Unit", "")}'.strip()
    rr = list(csv.reader(raw.splitlines()))
    rh = rr[0]
    units = dict(zip(rh, rr[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rawd = {}
    for row in rr[2:]:
        d = dict(zip(rh, row))
        k = (d["ID"], d["Kernel Name"].split("(")[0])
        rawd[k] = {m: f"{d.get(m)} {units.get(m, '')}".strip() for m in RAW}
        rawd[k]["_bytes"] = sum(float(d[m]) * scale.get(units.get(m, "byte"), 1.0)
                                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum") if d.get(m))
        stalls = []
        for kk, v in d.items():
            if kk.startswith("smsp__average_warps_issue_stalled_") and kk.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), kk[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        rawd[k]["top_stalls"] = ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:5])
    lines = [f"# ncu --set full summary ({rep.split('/')[-1]})", ""]
    traffic = {}
    for k, m in per.items():
        lines.append(f"## {k[1]} (capture ID {k[0]})")
        for name in KEEP:
            if name in m:
                lines.append(f"- {name}: {m[name]}")
        for name, v in rawd.get(k, {}).items():
            if not name.startswith("_"):
                lines.append(f"- {name}: {v}")
        if k in rawd:
            lines.append(f"- DRAM traffic per launch (read + write): {rawd[k]['_bytes'] / 1e6:.1f} MB")
            traffic[k[1]] = {"dram_bytes": rawd[k]["_bytes"]}
            for name, key in (("Issue Slots Busy", "issue_slots_busy_pct"), ("Executed Ipc Active", "ipc_active")):
                if name in m:
                    try:
                        traffic[k[1]][key] = float(m[name].split()[0].replace(",", ""))
                    except ValueError:
                        pass
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json:
        json.dump({"source": rep.split("/")[-1], "per_kernel": traffic}, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], *sys.argv[4:5])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
