"""Instruction mix of one kernel from an `ncu --set full --import-source on` report (dev tooling).

    python tools/sass_profile.py <report.ncu-rep> <kernel-regex> [--per N --unit pair] [--out f.md]

Reads the SASS source page (`ncu -i ... --page source --csv --print-source sass`), which carries
every instruction's execution count (warp level), and prints
  * warp instructions by class (fp32, packed fp32x2, fp64, MUFU, conversions, integer/moves,
    shared, global/constant, control, warp-level), per unit of work when --per gives the number
    of units (thread instructions per unit = warp instructions x 32 / N);
  * the instructions grouped by execution count (e.g. once per round vs once per loop step);
  * the top opcodes.
"""
import argparse
import collections
import csv
import io
import subprocess

CLASSES = [
    ("fp32x2", ("FFMA2", "FADD2", "FMUL2")),
    ("fp32", ("FFMA", "FMUL", "FADD", "FSETP", "FMNMX", "FMNMX3", "FSEL", "FCHK", "FSWZADD")),
    ("fp64", ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX")),
    ("mufu", ("MUFU",)),
    ("cvt", ("F2F", "F2I", "I2F", "I2FP", "F2IP", "FRND")),
    ("spill", ("LDL", "STL")),
    ("shared", ("LDS", "STS", "LDSM", "ATOMS")),
    ("global/const", ("LDG", "STG", "RED", "REDG", "ATOM", "ATOMG", "LDC", "LDCU", "LD", "ST")),
    ("control", ("BRA", "BSSY", "BSYNC", "BREAK", "WARPSYNC", "EXIT", "CALL", "RET", "PLOP3", "BAR", "BMOV",
                 "NOP", "YIELD")),
    ("warp", ("SHFL", "VOTE", "VOTEU", "MATCH", "REDUX", "POPC", "FLO", "BREV", "S2R", "S2UR", "UPOPC")),
]


def opcode(text: str) -> str:
    parts = text.split()
    if not parts:
        return "?"
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    return op.rstrip(";")


def klass(op: str) -> str:
    base = op.split(".")[0]
    for name, ops in CLASSES:
        if base in ops:
            return name
    return "int/mov"


def read_sass(rep: str, kernel: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kernel}"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ie, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[hdr_i + 1:]:
        if not r or r[0] == "Kernel Name":   # a second kernel instance: keep the first
            break
        data.append((opcode(r[isrc]), int(r[ie] or 0), int(r[iss] or 0)))
    return data


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--per", type=float, default=0.0, help="units of work in the launch (e.g. pairs)")
    ap.add_argument("--unit", default="unit")
    ap.add_argument("--warp-units", action="store_true",
                    help="units are warp-level (e.g. 32-survivor rounds): report warp instructions per unit")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    data = read_sass(a.report, a.kernel)
    lanes = 1 if a.warp_units else 32
    kind = "warp" if a.warp_units else "thread"
    tot = sum(e for _, e, _ in data)
    stall = sum(s for _, _, s in data) or 1
    lines = [f"# SASS instruction mix: `{a.kernel}` in `{a.report.split('/')[-1]}`", "",
             f"{tot / 1e6:.1f} M warp instructions executed" +
             (f"; {tot * lanes / a.per:.1f} {kind} instructions per {a.unit} ({a.per:.4g} {a.unit}s)" if a.per else ""),
             "", "| class | share | " + (f"per {a.unit} |" if a.per else "") + " stall samples |",
             "|---|---|" + ("---|" if a.per else "") + "---|"]
    c, cs = collections.Counter(), collections.Counter()
    for op, e, s in data:
        c[klass(op)] += e
        cs[klass(op)] += s
    for k, v in c.most_common():
        lines.append(f"| {k} | {v / tot * 100:.1f} % | " + (f"{v * lanes / a.per:.1f} |" if a.per else "") +
                     f" {cs[k] / stall * 100:.1f} % |")
    # execution-count groups (instructions run once per X)
    g = collections.Counter()
    for _, e, _ in data:
        if e:
            g[round(e, -3)] += e
    lines += ["", "Largest execution-count groups (instructions executed the same number of times, e.g. once per "
              "round or once per loop step):", "", "| executions per instruction | share of instructions |", "|---|---|"]
    for k, v in sorted(g.items(), key=lambda kv: -kv[1])[:8]:
        lines.append(f"| {k:,.0f} | {v / tot * 100:.1f} % |")
    o = collections.Counter()
    for op, e, _ in data:
        o[op] += e
    lines += ["", "Top opcodes:", "", "| opcode | share |" + (f" per {a.unit} |" if a.per else ""),
              "|---|---|" + ("---|" if a.per else "")]
    for k, v in o.most_common(20):
        lines.append(f"| `{k}` | {v / tot * 100:.1f} % |" + (f" {v * lanes / a.per:.2f} |" if a.per else ""))
    text = "\n".join(lines) + "\n"
    if a.out:
        open(a.out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
