"""Measured roofline denominators on this GPU (tools/peaks.cu):

    python tools/peaks.py [--out profiles/r02_peaks.json]

FP32 FFMA and packed FFMA2 lane-instruction rates (the issue-rate peak the GRCA kernels' lane-instruction
counts are divided by) and u64 RED.MIN rates into an L2-resident 33.5 MB buffer (the C4 hit keys), random
and lane-consecutive addresses.  bench.py calls measure() live (about a second) so the denominators come
from the same box and clocks as the timed region.
"""
import ctypes as C
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "peaks.cu")
LIB = os.path.join(HERE, "libpeaks.so")


def build() -> str:
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = f"{LIB}.{os.getpid()}.tmp"   # per process: ranks building at once never share a partial file
        subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                               "-Xcompiler", "-fPIC", "-shared", SRC, "-o", tmp])
        os.replace(tmp, LIB)
    return LIB


def measure() -> dict:
    import torch

    torch.cuda.init()
    L = C.CDLL(build())
    L.peaks_run.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    out = {}
    for kind, name in ((0, "ffma_lane_instr_per_s"), (1, "ffma2_lane_instr_per_s"),
                       (2, "red_min_u64_random_per_s"), (3, "red_min_u64_coalesced_per_s")):
        v, ms = C.c_double(), C.c_double()
        rc = L.peaks_run(kind, C.byref(v), C.byref(ms))
        if rc != 0:
            raise RuntimeError(f"peaks_run({kind}) failed: {rc}")
        out[name] = v.value
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    out["implied_sm_mhz_from_ffma"] = out["ffma_lane_instr_per_s"] / (n_sm * 128) / 1e6
    out["how"] = ("tools/peaks.cu: 148 SMs x 8 blocks x 256 threads; FFMA/FFMA2 with 8 independent chains per "
                  "thread (lane-instructions/s); atomicMin u64 with unused result (RED.MIN) into 4,194,304 keys "
                  "(33.5 MB, L2-resident), random or lane-consecutive addresses (ops/s); CUDA events, 5 reps")
    return out


if __name__ == "__main__":
    res = measure()
    print(json.dumps(res, indent=1))
    if "--out" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--out") + 1], "w"), indent=1)
