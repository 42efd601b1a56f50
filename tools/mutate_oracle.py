"""Mutation check of the oracle pins (tests/test_oracle_pins.py): every plausible slip in the oracle
or the comparator must fail at least one pin, otherwise that part of the oracle is not pinned.

    python tools/mutate_oracle.py [--out profiles/r02_oracle_mutations.md]

Each mutation is applied to a scratch copy of oracle/ (+ scenegen/, the pins and their golden files),
the oracle is rebuilt there and the pins are run against the copy.  Nothing in the repository is
modified.  Exit status 1 if any mutation survives.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C = "oracle/grca_oracle.c"
P = "oracle/compare.py"

# (name, file, old, new): each a slip a careful reader could make when writing the oracle from the paper
MUTATIONS = [
    ("drop u + v <= 1 (open wedge instead of triangle)", C,
     "if (!(u >= 0.0 && v >= 0.0 && u + v <= 1.0)) return 0;", "if (!(u >= 0.0 && v >= 0.0)) return 0;"),
    ("u + v < 1 (half-open triangle)", C, "u + v <= 1.0", "u + v < 1.0"),
    ("u > 0 (open edge)", C, "if (!(u >= 0.0 && v >= 0.0 && u + v <= 1.0))", "if (!(u > 0.0 && v >= 0.0 && u + v <= 1.0))"),
    ("v > 0 (open edge)", C, "if (!(u >= 0.0 && v >= 0.0 && u + v <= 1.0))", "if (!(u >= 0.0 && v > 0.0 && u + v <= 1.0))"),
    ("t >= 0 instead of t > 0", C, "if (!(t > 0.0 && t <= dmax)) return 0;", "if (!(t >= 0.0 && t <= dmax)) return 0;"),
    ("t < D_max instead of t <= D_max", C, "if (!(t > 0.0 && t <= dmax)) return 0;",
     "if (!(t > 0.0 && t < dmax)) return 0;"),
    ("theta step flipped", C, "theta0 + (double)i * dtheta", "theta0 - (double)i * dtheta"),
    ("ceil(chi/2) instead of floor(chi/2)", C, "-(double)(e->rays_per_channel / 2) * dtheta",
     "-(double)((e->rays_per_channel + 1) / 2) * dtheta"),
    ("cos <-> sin of theta", C, "const double ct = cos(theta), st = sin(theta);",
     "const double ct = sin(theta), st = cos(theta);"),
    ("right term sign flipped", C, "st * cp * (double)e->right[c]", "-st * cp * (double)e->right[c]"),
    ("180 deg / 360 deg span swapped", C, "const double H = (e->hfov_deg == 180) ? M_PI : 2.0 * M_PI;",
     "const double H = (e->hfov_deg == 180) ? 2.0 * M_PI : M_PI;"),
    ("cross-product operands swapped (p = e2 x d)", C, "cross3(d, e2, p);", "cross3(e2, d, p);"),
    ("q = e1 x s instead of s x e1", C, "cross3(s, e1, q);", "cross3(e1, s, q);"),
    ("ray kept in fp64 (not RN32)", C, "d[k] = (double)d32[k]; /* the ray is the fp32 direction */",
     "d[k] = d64[k];"),
    ("tie -> larger id", C, "(t == best_t && id < best_id)", "(t == best_t && id > best_id)"),
    ("tie -> last triangle (t <= best)", C, "if (t < best_t || (t == best_t && id < best_id)) {",
     "if (t <= best_t) {"),
    ("all-hit count before the accept test", C,
     "if (!hit_accept(t, u, v, dN, dmax, J->faces)) continue;\n                ++nhits;",
     "++nhits;\n                if (!hit_accept(t, u, v, dN, dmax, J->faces)) continue;"),
    ("face modes swapped", C, "if (faces == 1 && !(dN > 0.0)) return 0;", "if (faces == 1 && !(dN < 0.0)) return 0;"),
    ("ray offset O_n not accumulated", C, "        base += cnt;\n    }\n    return -1;", "    }\n    return -1;"),
    ("comparator: BARY_EPS = 1e9 (excuse everything)", P, "BARY_EPS = 1e-6", "BARY_EPS = 1e9"),
    ("comparator: BARY_EPS = 1e-7", P, "BARY_EPS = 1e-6", "BARY_EPS = 1e-7"),
    ("comparator: BARY_EPS = 1e-5", P, "BARY_EPS = 1e-6", "BARY_EPS = 1e-5"),
    ("comparator: REL_T = 1e-4", P, "REL_T = 1e-5", "REL_T = 1e-4"),
    ("comparator: no near-tie branch", P,
     "if hit and abs(tq - o_t[r]) <= REL_T * o_t[r] and t_ok[r]:", "if False:"),
    ("comparator: near-tie without the t check", P,
     "if hit and abs(tq - o_t[r]) <= REL_T * o_t[r] and t_ok[r]:", "if hit:"),
    ("comparator: id swap excused when the GPU's triangle is not hit", P,
     "exc = m is not None and abs(m) <= BARY_EPS   # GPU hit a triangle the oracle misses",
     "exc = True"),
    ("comparator: sentinel check dropped", P, "agree &= ~bad_sentinel", "pass"),
    ("comparator: agreement threshold 99.9 %", P, "AGREE_FRAC = 0.99999", "AGREE_FRAC = 0.999"),
]


def run_one(name, path, old, new, scratch):
    src = os.path.join(scratch, path)
    text = open(src).read()
    if text.count(old) != 1:
        return name, "NOT APPLIED (pattern count %d)" % text.count(old), []
    open(src, "w").write(text.replace(old, new))
    for so in ("oracle/liboracle.so",):
        p = os.path.join(scratch, so)
        if os.path.exists(p):
            os.remove(p)
    env = dict(os.environ, PYTHONPATH=scratch, PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x", "--tb=no",
                        "-rf", "-k", "not mutations_named", os.path.join(scratch, "tests", "test_oracle_pins.py")],
                       cwd=scratch, env=env, capture_output=True, text=True, timeout=900)
    failed = [ln.split("::")[-1].split(" ")[0] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
    open(src, "w").write(text)
    return name, ("killed" if r.returncode != 0 else "SURVIVED"), failed


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_oracle_mutations.md"))
    ap.add_argument("--only", default="", help="comma-separated substrings: run only matching mutations")
    args = ap.parse_args()
    muts = [m for m in MUTATIONS if not args.only or any(k in m[0] for k in args.only.split(","))]
    scratch = tempfile.mkdtemp(prefix="mut_oracle_")
    try:
        for d in ("oracle", "scenegen"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(scratch, d),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        os.makedirs(os.path.join(scratch, "tests"))
        for f in ("conftest.py", "test_oracle_pins.py"):
            shutil.copy(os.path.join(ROOT, "tests", f), os.path.join(scratch, "tests", f))
        shutil.copytree(os.path.join(ROOT, "tests", "golden"), os.path.join(scratch, "tests", "golden"))
        rows = []
        env = dict(os.environ, PYTHONPATH=scratch)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--tb=short", "-k", "not mutations_named",
                            os.path.join(scratch, "tests", "test_oracle_pins.py")], cwd=scratch, env=env,
                           capture_output=True, text=True)
        if r.returncode != 0:
            print(r.stdout[-3000:])
            raise SystemExit("unmutated pins fail in the scratch copy")
        for m in muts:
            rows.append(run_one(*m, scratch))
            print(f"{rows[-1][1]:>10}  {rows[-1][0]}  {','.join(rows[-1][2])}", flush=True)
    finally:
        shutil.rmtree(scratch, ignore_errors=True)
    survived = [r for r in rows if r[1] != "killed"]
    with open(args.out, "w") as f:
        f.write("# Oracle mutation check (tools/mutate_oracle.py)\n\n")
        f.write("Each row is one slip applied to a scratch copy of `oracle/` and run against "
                "`tests/test_oracle_pins.py` (stops at the first failing pin).\n\n")
        f.write("| mutation | file | result | first failing pin |\n|---|---|---|---|\n")
        for (name, path, _, _), (_, res, failed) in zip(muts, rows):
            f.write(f"| {name} | `{path}` | {res} | {', '.join(failed) or '-'} |\n")
        f.write(f"\n{len(rows) - len(survived)} of {len(rows)} mutations killed.\n")
    print(f"{len(rows) - len(survived)}/{len(rows)} killed -> {args.out}")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
