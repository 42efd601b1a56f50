"""Bounds-checked build of libgrca.so (the substitute for compute-sanitizer, which is closed on this GPU pool):

    python tools/check_build.py                      # here: nvcc -DGRCA_CHECK -> build/check/libgrca.so
    GRCA_LIB=build/check/libgrca.so python -m pytest tests -m gpu -q   # on the GPU box

Every global index of the hot path (survivor writes, ray-table / hit-key indices, mesh vertex indices,
triangle indices) is checked against its buffer's extent inside the kernels; a violation sets a site bit
and is redirected (no fault), and grca_cast synchronizes and returns GRCA_E_CUDA with the site mask, so
every GPU test doubles as an out-of-bounds test.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_10457_b200.build import build_variant  # noqa: E402

if __name__ == "__main__":
    out = os.path.join(ROOT, "build", "check", "libgrca.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    print(build_variant(out, ["GRCA_CHECK"]))
