"""CPU checks of arithmetic shortcuts the kernels rely on (no GPU): each is a claim in a csrc/ comment that
an exhaustive or worst-case sweep can settle."""
import numpy as np


def _nudge(x, n):
    """x moved n float32 ulps up (n > 0) or down (n < 0)."""
    for _ in range(abs(n)):
        x = np.nextafter(x, np.float32(np.inf if n > 0 else -np.inf), dtype=np.float32)
    return x


def test_fused_row_from_reciprocal_needs_no_correction():
    """grca.cu KF_ROWCOL_EXACT: row = trunc(((float)local + 0.5f) * rcp(len)) equals local // len for every item
    of a small rectangle (rows x len <= small_max <= 1023), even with the reciprocal and the product off by a
    few ulp (__fdividef(1, len) is within 2 ulp; the product adds 0.5 ulp; checked here at +-4 ulp each)."""
    f32 = np.float32
    for ln in range(1, 1024):
        local = np.arange((1023 // ln) * ln, dtype=np.int64)
        for k in (-4, 0, 4):
            inv = _nudge(f32(1.0) / f32(ln), k)
            prod = (local.astype(np.float32) + f32(0.5)) * inv
            for j in (-4, 4):
                row = np.trunc(_nudge(prod, j)).astype(np.int64)
                assert np.array_equal(row, local // ln), (ln, k, j)


def test_k2_lut_bin_saturating_conversion():
    """grca_device.cuh K2_BIN_U32: the bin (unsigned)((lo + 1) * 1024) needs no clamp: lo < 1 keeps it <= 2047 and
    a negative product converts (saturating, like cvt.rzi.u32.f32) to 0, i.e. bin 0 -- the same bin as the clamped
    form max(lo, -1)."""
    f32 = np.float32
    lo = np.concatenate([np.linspace(-1.5, 1 - 3e-6, 200001, dtype=np.float32),
                         np.float32([-1.0, -0.9999999, 1 - 3e-6, -100.0])])
    prod = lo * f32(1024) + f32(1024)
    sat = np.where(prod < 0, 0, np.trunc(prod)).astype(np.int64)   # cvt.rzi.u32 saturates negatives to 0
    clamped = np.trunc(np.maximum(lo, f32(-1)) * f32(1024) + f32(1024)).astype(np.int64)
    assert sat.max() <= 2047 and sat.min() >= 0
    assert np.array_equal(sat, clamped)
