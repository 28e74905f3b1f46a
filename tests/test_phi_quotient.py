"""CPU: the phi kernel's division-free quotient rule (mstep.cu phi_quotient) is exact.

The reference computes bhat = f32((cnt + beta) / denom) with a correctly rounded double
division (counts.cpp:58-60).  The kernel multiplies by RN(1/denom) instead and falls back to
the division only when the product is within 64 double ulps of an f32 rounding boundary or
outside the f32 normal range.  This numpy replica of the same rule (IEEE double, round to
nearest) must never disagree with the division on the fast path -- on random inputs of the
shapes the trainer produces and on quotients placed exactly at f32 midpoints.
"""
import numpy as np


def _fast_path(x, den):
    y = x * (1.0 / den)
    b = y.view(np.uint64)
    lo = (b & np.uint64(0x1FFFFFFF)).astype(np.uint32)
    ex = ((b >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.uint32)
    near_mid = (lo - np.uint32(0x10000000 - 64)) <= np.uint32(128)
    out_of_range = (ex - np.uint32(898)) > np.uint32(1149 - 898)
    return y.astype(np.float32), ~(near_mid | out_of_range)


def test_fast_quotient_matches_division_on_trainer_shapes():
    rng = np.random.default_rng(7)
    for beta in (0.01, 0.1, 1e-3, 0.5):
        n = 2_000_000
        cnt = rng.integers(1, 1 << 22, n).astype(np.float64)
        den = rng.integers(0, 1 << 34, n).astype(np.float64) + 141_000 * beta
        x = cnt + beta
        got, fast = _fast_path(x, den)
        exact = (x / den).astype(np.float32)
        assert not np.any((got != exact) & fast)
        assert fast.mean() > 0.9999


def test_fast_quotient_never_decides_a_midpoint():
    rng = np.random.default_rng(8)
    f = rng.random(500_000).astype(np.float32).astype(np.float64)
    mid = f + np.spacing(f.astype(np.float32)).astype(np.float64) / 2
    den = rng.integers(1, 1 << 20, mid.size).astype(np.float64)
    x = mid * den
    got, fast = _fast_path(x, den)
    exact = (x / den).astype(np.float32)
    assert not np.any((got != exact) & fast)
