"""The split-fp16 operand encoding of the tcgen05 GEMMs (DESIGN.md §3,
kernels_simt.cuh put16), restated in numpy on the CPU:

    s = x 2^sigma,  hi = fp16_rn(s),  lo = fp16_rn(s - hi)

* s - hi is exact in fp32 and hi + lo carries 22 significant bits: the
  relative error of (hi + lo) 2^-sigma is below 2^-22 for s in fp16's normal
  range;
* the error is below max(2^-22 |x|, 2^-25 2^-sigma) at any sigma that keeps
  max|s| inside fp16 — relative where lo is a normal fp16, lo's subnormal
  spacing below (the engine targets max|s| in [2^12, 2^13));
* the three products hi*hi + hi*lo + lo*hi reproduce an fp32 product to
  ~2^-21 relative (lo*lo is below it);
* the engine's sigma target (h16_sigma_for: 12 - floor(log2 max)) lands every
  maximum in [2^12, 2^13).
"""
import numpy as np


def split(x, sigma):
    s = (x.astype(np.float32) * np.float32(2.0 ** sigma)).astype(np.float32)
    hi = s.astype(np.float16)
    lo = (s - hi.astype(np.float32)).astype(np.float16)
    return hi, lo


def join(hi, lo, sigma):
    return ((hi.astype(np.float32) + lo.astype(np.float32)) * np.float32(2.0 ** -sigma)).astype(np.float32)


def sigma_for(m):
    return 12 - int(np.floor(np.log2(m)))


def test_residual_exact_and_22_bits():
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(200000) * 10.0 ** rng.uniform(-3, 3, 200000)).astype(np.float32)
    sigma = sigma_for(np.abs(x).max())
    s = (x * np.float32(2.0 ** sigma)).astype(np.float32)
    hi, lo = split(x, sigma)
    # s - hi is exactly representable (the fp32 subtraction loses nothing)
    r = s.astype(np.float64) - hi.astype(np.float64)
    assert np.array_equal(r.astype(np.float32).astype(np.float64), r)
    # 22-bit accuracy where lo is a normal fp16 (|s| >= 2^-3)
    big = np.abs(s) >= 2.0 ** -3
    rel = np.abs(join(hi, lo, sigma).astype(np.float64) - x) / np.abs(x.astype(np.float64))
    assert rel[big].max() <= 2.0 ** -22
    # below that the absolute error stays under the subnormal spacing 2^-25 (scaled)
    err = np.abs(join(hi, lo, sigma).astype(np.float64) - x) * 2.0 ** sigma
    assert err[~big].max() <= 2.0 ** -25


def test_error_bound_at_every_sigma_of_the_band():
    """|x - (hi + lo) 2^-sigma| <= max(2^-22 |x|, 2^-25 2^-sigma): relative where
    lo is a normal fp16, absolute (lo's subnormal spacing) below — for any sigma
    that keeps max|s| inside fp16, so a far-off sigma costs only elements tiny
    against the tensor's max.  (The bits themselves depend on sigma through
    lo's subnormal rounding; sigma is global state, identical on every rank.)"""
    rng = np.random.default_rng(2)
    x = (rng.standard_normal(50000) * 10.0 ** rng.uniform(-4, 0, 50000)).astype(np.float32)
    s0 = sigma_for(np.abs(x).max())
    for ds in (-8, -4, -2, 0, 1):
        sig = s0 + ds
        err = np.abs(join(*split(x, sig), sig).astype(np.float64) - x)
        bound = np.maximum(2.0 ** -22 * np.abs(x.astype(np.float64)), 2.0 ** (-25 - sig))
        assert np.all(err <= bound), ds


def test_three_products_match_fp32():
    rng = np.random.default_rng(3)
    a = rng.standard_normal(100000).astype(np.float32)
    b = rng.standard_normal(100000).astype(np.float32)
    sa, sb = sigma_for(np.abs(a).max()), sigma_for(np.abs(b).max())
    ah, al = split(a, sa)
    bh, bl = split(b, sb)
    f = lambda h: h.astype(np.float64)
    p3 = (f(ah) * f(bh) + f(ah) * f(bl) + f(al) * f(bh)) * 2.0 ** -(sa + sb)
    exact = a.astype(np.float64) * b.astype(np.float64)
    rel = np.abs(p3 - exact) / np.abs(exact)
    ok = (np.abs(a) * 2.0 ** sa >= 2.0 ** -3) & (np.abs(b) * 2.0 ** sb >= 2.0 ** -3)
    assert rel[ok].max() < 2.0 ** -20


def test_sigma_target_band():
    for m in np.float32([1e-30, 3.7e-5, 0.25, 1.0, 1.5, 4095.0, 7.9e20]):
        x = float(m) * 2.0 ** sigma_for(float(m))
        assert 2.0 ** 12 <= x < 2.0 ** 13, (m, x)
