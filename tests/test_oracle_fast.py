"""Pins for the FAST-mode oracle (oracle_escape_fma_*: the FMA-contracted sequence on the
doubled state X = 2x, Y = 2y that defines FP32_FAST / FP64_FAST, DESIGN.md §5 "State
representation", reading c-10).

What fixes it, independent of its own code:
  * exact dyadic orbits: every operation is exact, so fused and unfused agree and the
    counts are the hand-traced ones of test_oracle_pins (count definition, strict '>',
    fencepost);
  * closed forms and invariants that survive correct rounding: C = 0, the C = -2 real
    segment, the Mandelbrot regions, the 180-degree / conjugate symmetries (fma and
    round-to-nearest are sign-symmetric), cap monotonicity;
  * a brute force in exact rational arithmetic with its own round-to-nearest-even to
    binary32 / binary64 (no libm fma), on tiny grids, of BOTH the doubled sequence (the
    definition) and the unscaled contraction of reading c-9's iteration (the doubled one
    is its exact power-of-two rescaling while no unscaled product is subnormal);
  * that the sequence is really fused: on a 1080p-shaped frame it differs from the
    strict oracle on a small, nonzero fraction of pixels.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import numpy_ref
from paper_1611_03079_b200 import workloads as W

from test_oracle_pins import JULIA_EXACT, MANDEL_EXACT

PRECS = (32, 64)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("z0,c,expected", JULIA_EXACT)
def test_fast_exact_orbits_julia(oracle_mod, prec, z0, c, expected):
    assert oracle.escape_time(z0, c, 100, prec, fast=True) == expected
    assert oracle.escape_time(-z0, c, 100, prec, fast=True) == expected


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("c,expected", MANDEL_EXACT)
def test_fast_exact_orbits_mandelbrot(oracle_mod, prec, c, expected):
    assert oracle.escape_time(0j, c, 100, prec, fast=True) == expected


@pytest.mark.parametrize("prec", PRECS)
def test_fast_c_zero_closed_form(oracle_mod, prec):
    """C = 0 (as test_oracle_pins.test_c_zero_closed_form): |Z_0| < 1 never escapes,
    |Z_0| > 2 escapes at n = 0, and in between n = floor(log2(ln 4 / ln|Z_0|)) away from
    integer arguments."""
    n = 257
    g = oracle.julia(0j, 0j, 2.5, 2.5, n, n, 100, prec, fast=True).astype(np.int64)
    re, im = numpy_ref.axes(0j, 2.5, 2.5, n, n)
    dt = np.float32 if prec == 32 else np.float64
    r = np.hypot(re.astype(dt).astype(np.float64)[None, :],
                 im.astype(dt).astype(np.float64)[:, None]) * np.ones((n, 1))
    assert (g[r < 1 - 1e-6] == 100).all()
    assert (g[r > 2 + 1e-6] == 0).all()
    ann = (r > 1 + 1e-6) & (r <= 2 - 1e-6)
    arg = np.log2(np.log(4.0) / np.log(r[ann]))
    ok = np.abs(arg - np.round(arg)) > 1e-9
    np.testing.assert_array_equal(g[ann][ok], np.minimum(np.floor(arg), 100)[ok])


@pytest.mark.parametrize("prec", PRECS)
def test_fast_c_minus_two_real_segment(oracle_mod, prec):
    """C = -2: on the real axis yy = 0, so the fused steps are fl(x^2) and fl(x^2 - 2)
    as in the strict reading: |x| <= 2 stays bounded; everything off the axis escapes."""
    w, h = 257, 129
    g = oracle.julia(-2 + 0j, 0j, 2.5, 2.5 * h / w, w, h, 100, prec, fast=True)
    re, im = numpy_ref.axes(0j, 2.5, 2.5 * h / w, w, h)
    dt = np.float32 if prec == 32 else np.float64
    expected = np.zeros((h, w), dtype=bool)
    for py in range(h):
        if dt(im[py]) == 0:
            expected[py] = np.abs(re.astype(dt)) <= 2
    np.testing.assert_array_equal(g == 100, expected)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("c", list(W.FIG2_C) + [-0.8 + 0.156j])
def test_fast_symmetries(oracle_mod, prec, c):
    g = oracle.julia(c, 0j, 1.7, 1.3, 333, 255, 100, prec, fast=True)
    np.testing.assert_array_equal(g, g[::-1, ::-1])
    a = oracle.julia(c, 0.1 + 0j, 1.5, 1.2, 200, 151, 100, prec, fast=True)
    b = oracle.julia(c.conjugate(), 0.1 + 0j, 1.5, 1.2, 200, 151, 100, prec, fast=True)
    np.testing.assert_array_equal(a, b[::-1])
    m = oracle.mandelbrot(-0.5 + 0j, 1.5, 1.5, 257, 257, 200, prec, fast=True)
    np.testing.assert_array_equal(m, m[::-1])


@pytest.mark.parametrize("prec", PRECS)
def test_fast_mandelbrot_known_regions(oracle_mod, prec):
    n = 513
    g = oracle.mandelbrot(-0.5 + 0j, 2.2, 2.2, n, n, 1000, prec, fast=True)
    re, im = numpy_ref.axes(-0.5 + 0j, 2.2, 2.2, n, n)
    dt = np.float32 if prec == 32 else np.float64
    c = re.astype(dt).astype(np.float64)[None, :] + 1j * im.astype(dt).astype(np.float64)[:, None]
    far = np.abs(c) > 2.01
    assert far.sum() > 1000 and (g[far] == 1).all()
    card = np.abs(1 - np.sqrt(1 - 4 * c)) < 0.99
    disc = np.abs(c + 1) < 0.24
    assert (g[card] == 1000).all() and (g[disc] == 1000).all()


@pytest.mark.parametrize("prec", PRECS)
def test_fast_cap_monotonicity(oracle_mod, prec):
    c = W.FIG2_C[2]
    g2 = oracle.julia(c, 0j, 1.6, 1.2, 160, 120, 1000, prec, fast=True).astype(np.int64)
    for m1 in (1, 2, 7, 100, 999):
        g1 = oracle.julia(c, 0j, 1.6, 1.2, 160, 120, m1, prec, fast=True).astype(np.int64)
        np.testing.assert_array_equal(g1, np.minimum(g2, m1))


# ------------------------------------------------------------------ exact-rational brute force
_FMT = {32: (24, -126), 64: (53, -1022)}  # (significand bits, minimum normal exponent)


def _rn(q: Fraction, prec: int) -> Fraction:
    """Round-to-nearest-even of an exact rational to binary32 / binary64 (subnormals
    included; no overflow on these orbits)."""
    if q == 0:
        return Fraction(0)
    p, emin = _FMT[prec]
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    quantum = Fraction(2) ** (max(e, emin) - (p - 1))
    r = round(a / quantum) * quantum  # round() of a Fraction: half to even
    return r if q > 0 else -r


def _brute_fast(z0: complex, c: complex, mi: int, prec: int) -> int:
    R = lambda v: _rn(v, prec)  # noqa: E731
    x, y = R(Fraction(z0.real)), R(Fraction(z0.imag))
    cr, ci = R(Fraction(c.real)), R(Fraction(c.imag))
    for n in range(mi):
        yy = R(y * y)
        if R(x * x + yy) > 4:       # fused: x*x + yy rounded once
            return n
        t = R(x * x - yy)            # fused
        x, y = R(t + cr), R(2 * x * y + ci)  # y: fused 2x*y + ci
    return mi


def _brute_fast_doubled(z0: complex, c: complex, mi: int, prec: int) -> int:
    """The FAST definition as written (doubled state): YY = Y*Y; M = fma(X,X,YY) > 16?;
    T = fma(X,X,-YY); Y' = fma(X,Y,CI); X' = fma(T,1/2,CR), every fused op rounded once."""
    R = lambda v: _rn(v, prec)  # noqa: E731
    X, Y = 2 * R(Fraction(z0.real)), 2 * R(Fraction(z0.imag))
    CR, CI = 2 * R(Fraction(c.real)), 2 * R(Fraction(c.imag))
    for n in range(mi):
        YY = R(Y * Y)
        if R(X * X + YY) > 16:
            return n
        T = R(X * X - YY)
        X, Y = R(T / 2 + CR), R(X * Y + CI)
    return mi


@pytest.mark.parametrize("prec", PRECS)
def test_fast_oracle_matches_doubled_brute_force(oracle_mod, prec):
    """The definition itself: the oracle's doubled FMA sequence against an exact-rational
    evaluation of the same sequence with its own rounding, on tiny fuzz grids."""
    for c, win, w, h, mi in W.fuzz_cases(5, max_side=9, seed=12):
        mi = min(mi, 120)
        g = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec, fast=True)
        m = oracle.mandelbrot(win.center, win.half_w, win.half_h, w, h, mi, prec, fast=True)
        for py in range(h):
            for px in range(w):
                z = oracle.pixel_to_complex(win.center, win.half_w, win.half_h, w, h, px, py)
                if prec == 32:
                    z = complex(np.float32(z.real), np.float32(z.imag))
                assert g[py, px] == _brute_fast_doubled(z, c, mi, prec), (c, px, py)
                assert m[py, px] == _brute_fast_doubled(0j, z, mi, prec), (z, px, py)


@pytest.mark.parametrize("prec", PRECS)
def test_doubled_equals_unscaled_contraction(oracle_mod, prec):
    """Away from subnormal products the doubled FAST sequence is the unscaled FMA
    contraction of reading c-9's iteration rescaled by 2 (every rounding commutes with
    the scaling): the two oracle functions agree orbit for orbit on fuzz starts, and on
    a 1080p-shaped frame's worth of sampled pixels."""
    rng = np.random.default_rng(77)
    for _ in range(3000):
        z0 = complex(*rng.uniform(-2.2, 2.2, 2))
        c = complex(*rng.uniform(-1.5, 1.5, 2))
        mi = int(rng.choice([7, 100, 1000]))
        assert (oracle.escape_time(z0, c, mi, prec, fast=True)
                == oracle.escape_time_fast_unscaled(z0, c, mi, prec)), (z0, c, mi)


def test_doubled_differs_only_through_subnormals():
    """Where an unscaled product is subnormal the doubled one keeps bits: y = 3 * 2^-75 in
    binary32 has y*y = 4.5 subnormal quanta (2^-149), rounded to 4, while 4y^2 = 18
    quanta is exact, so fl(4 y^2) != 4 fl(y^2) (reading c-10's stated exception to the
    equivalence above)."""
    y = Fraction(3, 2 ** 75)
    assert _rn(4 * y * y, 32) != 4 * _rn(y * y, 32)
    y = Fraction(3, 2 ** 40)  # normal range: the scaling commutes
    assert _rn(4 * y * y, 32) == 4 * _rn(y * y, 32)


@pytest.mark.parametrize("prec", PRECS)
def test_fast_oracle_matches_exact_rational_brute_force(oracle_mod, prec):
    for c, win, w, h, mi in W.fuzz_cases(5, max_side=9, seed=11):
        mi = min(mi, 120)
        g = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec, fast=True)
        m = oracle.mandelbrot(win.center, win.half_w, win.half_h, w, h, mi, prec, fast=True)
        for py in range(h):
            for px in range(w):
                z = oracle.pixel_to_complex(win.center, win.half_w, win.half_h, w, h, px, py)
                if prec == 32:
                    z = complex(np.float32(z.real), np.float32(z.imag))
                assert g[py, px] == _brute_fast(z, c, mi, prec), (c, px, py)
                assert m[py, px] == _brute_fast(0j, z, mi, prec), (z, px, py)


def test_rn_helper_against_numpy():
    """The brute force's rounding against numpy's float32 / float64 conversion (both
    correctly rounded from an exactly representable double / a Fraction)."""
    rng = np.random.default_rng(5)
    for v in rng.standard_normal(2000) * 10.0 ** rng.integers(-40, 5, 2000):
        assert float(_rn(Fraction(float(v)), 32)) == float(np.float32(v))
        q = Fraction(float(v)) / 3
        assert float(_rn(q, 64)) == float(q)


@pytest.mark.parametrize("prec", PRECS)
def test_fast_is_really_fused(oracle_mod, prec):
    """A 1080p-shaped Julia frame: the fused sequence differs from the strict one on a
    small nonzero fraction of pixels (an unfused 'fast' would differ on none)."""
    win = W.julia_window(480, 270)
    c = -0.7269 + 0.1889j
    mi = 300 if prec == 32 else 1000  # binary64 needs longer orbits to show it
    s = oracle.julia(c, win.center, win.half_w, win.half_h, 480, 270, mi, prec)
    f = oracle.julia(c, win.center, win.half_w, win.half_h, 480, 270, mi, prec, fast=True)
    frac = float(np.mean(s != f))
    assert 0 < frac < 0.05, frac
    # on pixels where fusion decides the count, the exact-rational fused brute force
    # agrees with the fast oracle
    py, px = np.nonzero(s != f)
    for k in np.linspace(0, len(px) - 1, 6).astype(int):
        z = oracle.pixel_to_complex(win.center, win.half_w, win.half_h, 480, 270, px[k], py[k])
        if prec == 32:
            z = complex(np.float32(z.real), np.float32(z.imag))
        assert f[py[k], px[k]] == _brute_fast(z, c, mi, prec)
