"""Host check of the summation-order identity k_mass relies on (DESIGN.md §5,
k_mass): for 32 fp32 lane values, the lane-31 result of the Hillis-Steele
inclusive scan (shfl_up by 1, 2, 4, 8, 16; k_locate's sub-tile totals) equals
bit for bit the reduce-scatter over lane bits 0..3 followed by an xor-16 step
(k_mass's 16-shuffle warp totals).  Both add the same aligned binary tree;
IEEE addition is commutative.  Simulated in numpy float32 (round to nearest,
as FADD)."""
import numpy as np


def scan_lane31(x):
    v = x.astype(np.float32).copy()
    o = 1
    while o < 32:
        t = np.roll(v, o)                       # t[i] = v[i - o]
        v = np.where(np.arange(32) >= o, (v + t).astype(np.float32), v)
        o <<= 1
    return v[31]


def reduce_scatter(vals):                       # vals: [32 lanes][16 sub-tiles]
    v = vals.astype(np.float32).copy()
    lanes = np.arange(32)
    m, n = 1, 8
    while m <= 8:
        hi = (lanes & m) != 0
        keep = np.where(hi[:, None], v[:, n:2 * n], v[:, :n])
        send = np.where(hi[:, None], v[:, :n], v[:, n:2 * n])
        v = (keep + send[lanes ^ m]).astype(np.float32)
        m, n = m << 1, n >> 1
    v = (v[:, 0] + v[lanes ^ 16, 0]).astype(np.float32)
    s = ((lanes & 1) << 3) | ((lanes & 2) << 1) | ((lanes & 4) >> 1) | ((lanes & 8) >> 3)
    out = np.empty(16, np.float32)
    for lane in range(16):
        out[s[lane]] = v[lane]
    assert np.array_equal(v[:16], v[16:])       # the xor-16 step leaves both halves equal
    return out


def test_reduce_scatter_equals_scan_lane31():
    rng = np.random.default_rng(0)
    for trial in range(300):
        scale = 10.0 ** rng.uniform(-30, 3)
        w = (rng.exponential(1.0, (16, 32)) * scale).astype(np.float32)
        w[rng.random((16, 32)) < 0.3] = 0.0      # residual max(0, p - q) zeros
        if trial % 7 == 0:
            w[:, rng.integers(0, 32)] *= np.float32(1e7)   # wide dynamic range
        got = reduce_scatter(w.T)
        want = np.array([scan_lane31(w[s]) for s in range(16)], np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), trial


def test_sequential_order_differs():
    """Sanity: the check can fail -- a left-to-right sum is a different tree."""
    rng = np.random.default_rng(1)
    diff = 0
    for _ in range(200):
        w = (rng.exponential(1.0, 32) * 1e-3).astype(np.float32)
        seq = np.float32(0)
        for x in w:
            seq = np.float32(seq + x)
        diff += seq != scan_lane31(w)
    assert diff > 0
