"""Same-box A/B of compile-time variants of libgrca.so (dev tooling).

    python tools/ab.py build NAME=DEF1,DEF2 [NAME2=...]      # here: nvcc into build/ab/lib_NAME.so
    python tools/ab.py run [--steps 300] [--passes 2] [--config C4] NAME ...   # on the GPU box

`build` compiles each variant (the base sources with extra -D macros; `base=` for none).  `run` times
bench.py (device-timed, no CPU baseline / e2e / hybrid) once per variant per pass, interleaved
A B A B so clock or thermal drift hits every variant alike, and prints ms/frame per variant and pass,
plus the per-kernel times of the last pass.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build", "ab")


def main():
    if sys.argv[1] == "build":
        sys.path.insert(0, ROOT)
        from paper_2605_10457_b200.build import build_variant

        os.makedirs(OUT, exist_ok=True)
        for spec in sys.argv[2:]:
            name, _, defs = spec.partition("=")
            build_variant(os.path.join(OUT, f"lib_{name}.so"), [d for d in defs.split(",") if d])
            print("built", name, defs)
        return
    args = sys.argv[2:]
    steps, passes, config, extra = "300", 2, "C4", []
    names = []
    i = 0
    while i < len(args):
        if args[i] == "--steps":
            steps = args[i + 1]; i += 2
        elif args[i] == "--passes":
            passes = int(args[i + 1]); i += 2
        elif args[i] == "--config":
            config = args[i + 1]; i += 2
        elif args[i] == "--extra":
            extra = args[i + 1].split(); i += 2
        else:
            names.append(args[i]); i += 1
    res = {n: [] for n in names}
    kms, sts = {}, {}
    for p in range(passes):
        for n in names:
            env = dict(os.environ, GRCA_LIB=os.path.join(OUT, f"lib_{n}.so"), GRCA_AB_OLD_LIB="1")
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", steps, "--warmup", "10",
                   "--no-cpu-baseline", "--no-e2e", "--no-hybrid"] + extra
            r = subprocess.run(cmd, env=env, capture_output=True, text=True)
            line = [l for l in r.stdout.splitlines() if l.startswith("{")]
            if r.returncode or not line:
                res[n].append(None)
                print(n, "FAILED", r.stderr[-500:], flush=True)
                continue
            d = json.loads(line[-1])
            res[n].append(d["ms_per_step"])
            kms[n] = d["kernel_ms"]
            sts[n] = {k: d["stats"][k] for k in ("prefilter_survivors", "survivors", "hits_recorded")}
            print(f"pass {p} {n}: {d['ms_per_step']:.4f} ms", flush=True)
    for n in names:
        print(f"{n:16s} ms/frame {res[n]}  kernels " + " ".join(f"{k}={v:.4f}" for k, v in kms.get(n, {}).items()))
    # a variant must do the same work (culling is exact-conservative: survivors may only grow, hits never change)
    ref = sts.get(names[0])
    for n in names[1:]:
        if ref and n in sts and sts[n]["hits_recorded"] != ref["hits_recorded"]:
            print(f"WARNING {n}: hits_recorded {sts[n]['hits_recorded']} != {ref['hits_recorded']} ({names[0]})")
        if ref and n in sts:
            print(f"{n}: stats {sts[n]} vs {names[0]} {ref}")


if __name__ == "__main__":
    main()
