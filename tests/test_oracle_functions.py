"""NEXT-3 oracle pins: the Figure 4 family of iteration maps (reading c-14)."""
import numpy as np
import pytest

import oracle
from paper_1611_03079_b200 import workloads as W

PRECS = (32, 64)


@pytest.mark.parametrize("prec", PRECS)
def test_z2_variant_equals_main_definition(oracle_mod, prec):
    for c, win, w, h, mi in W.fuzz_cases(6, max_side=64, seed=3):
        a = oracle.julia_fn("z2", c, win.center, win.half_w, win.half_h, w, h, mi, prec)
        b = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec)
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("prec", PRECS)
def test_exact_orbits_quartic(oracle_mod, prec):
    """Dyadic hand iterations (exact in both precisions); 2^4 + 1 = 17."""
    assert oracle.escape_time_fn("z4", 0j, 1 + 0j, 100, prec) == 3    # 0 -> 1 -> 2 (|.|^2 = 4) -> 17
    assert oracle.escape_time_fn("z4", 0j, 0j, 100, prec) == 100
    assert oracle.escape_time_fn("z4", 1 + 0j, 0j, 100, prec) == 100  # 1 is fixed
    assert oracle.escape_time_fn("z4", 1.5 + 0j, 0j, 100, prec) == 1  # 1.5^4 = 5.0625
    assert oracle.escape_time_fn("z4", 1j, -1 + 0j, 100, prec) == 100  # i -> 0 -> -1 -> 0
    assert oracle.escape_time_fn("z4", 0j, -2 + 0j, 100, prec) == 2    # 0 -> -2 -> 14


@pytest.mark.parametrize("prec", PRECS)
def test_exact_orbits_rational_and_pole(oracle_mod, prec):
    """z^4 + (z^2+1)/(z^2-1) + c: at z = +-1 the pole sends Z to infinity."""
    assert oracle.escape_time_fn("z4_rational", 1 + 0j, 0j, 100, prec) == 1
    assert oracle.escape_time_fn("z4_rational", -1 + 0j, 0j, 100, prec) == 1
    # 0 -> 0 + (1/-1) = -1 -> pole -> inf
    assert oracle.escape_time_fn("z4_rational", 0j, 0j, 100, prec) == 2
    # i: w = -1, q = 0/(-2) = 0, z^4 = 1 -> Z_1 = 1 + c; with c = -1: 0 -> -1 -> pole
    assert oracle.escape_time_fn("z4_rational", 1j, -1 + 0j, 100, prec) == 3


@pytest.mark.parametrize("prec", PRECS)
def test_quartic_four_fold_symmetry(oracle_mod, prec):
    """(iz)^4 = z^4 exactly in RN arithmetic (w -> -w), so on a square grid centred at
    0 the z^4 + c frame is invariant under 90-degree rotation; the rational map keeps
    the 180-degree symmetry (w unchanged under z -> -z)."""
    n = 129
    for c in (W.FIG4_C, 0.5 + 0.3j, -0.7 + 0.0j):
        g = oracle.julia_fn("z4", c, 0j, 1.6, 1.6, n, n, 100, prec)
        np.testing.assert_array_equal(g, np.rot90(g))
        r = oracle.julia_fn("z4_rational", c, 0j, 2.0, 2.0, n, n, 100, prec)
        np.testing.assert_array_equal(r, r[::-1, ::-1])


@pytest.mark.parametrize("prec", PRECS)
def test_quartic_c_zero_closed_form(oracle_mod, prec):
    """C = 0: Z_n = Z_0^(4^n): |Z_0| < 1 never escapes, |Z_0| > 2 escapes at 0, and for
    1 < r <= 2 the count is floor(log4(ln 4 / ln r)) + 1 (first n with r^(2*4^n) > 4)."""
    for r in (1.05, 1.2, 1.3, 1.5, 1.9):
        z0 = complex(r, 0)
        n = int(np.floor(np.log(np.log(2.0) / np.log(r)) / np.log(4.0))) + 1
        assert oracle.escape_time_fn("z4", z0, 0j, 100, prec) == n
    assert oracle.escape_time_fn("z4", 0.9 + 0.1j, 0j, 100, prec) == 100
    assert oracle.escape_time_fn("z4", 2.5j, 0j, 100, prec) == 0


@pytest.mark.parametrize("prec", PRECS)
def test_rational_orbit_with_complex_w(oracle_mod, prec):
    """A hand-traced orbit where Im(w) != 0, so every term of q = (w+1)/(w-1) matters
    (S:35 reading of Fig. 4).  Z_0 = 1 + i: w = Z_0^2 = 2i, z^4 = w^2 = -4,
    q = (1 + 2i)/(-1 + 2i) = (1 + 2i)(-1 - 2i)/5 = (3 - 4i)/5.  With C = 2.4 + 1.8i:
    Z_1 = -4 + 0.6 + 2.4 + (-0.8 + 1.8)i = -1 + i (|Z_1|^2 = 2), then w = (-1 + i)^2 = -2i,
    z^4 = -4, q = (1 - 2i)/(-1 - 2i) = (3 + 4i)/5, Z_2 = -1 + 2.6i (|Z_2|^2 = 7.76 > 4):
    count 2.  A slip in q moves Z_1 by 1.6 (sign of Im q: Z_1 = -1 + 2.6i; the b*d term
    of Re q with the wrong sign: Z_1 = -2.6 + i), both outside radius 2 -> count 1.  The
    margins (|Z|^2 = 2 and 7.76 against 4) dwarf any rounding of 0.6, 0.8, 2.4, 1.8."""
    c = 2.4 + 1.8j
    assert oracle.escape_time_fn("z4_rational", 1 + 1j, c, 100, prec) == 2
    assert oracle.escape_time_fn("z4_rational", 1 - 1j, c.conjugate(), 100, prec) == 2
    # the same first step reached from the conjugate side and from -Z_0 (w unchanged)
    assert oracle.escape_time_fn("z4_rational", -1 - 1j, c, 100, prec) == 2


def _exact_fn_orbit(fn, z0, c, mi):
    """The map evaluated in exact rational arithmetic from the binary64 start values (no
    rounding at all): returns the list of |Z_n|^2 for n = 0 .. until escape or mi-1, and
    the minimum |w - 1|^2 seen (pole proximity)."""
    from fractions import Fraction as Fr
    x, y = Fr(z0.real), Fr(z0.imag)
    cr, ci = Fr(c.real), Fr(c.imag)
    mags, pole = [], None
    for _ in range(mi):
        m = x * x + y * y
        mags.append(m)
        if m > 4:
            break
        wx, wy = x * x - y * y, 2 * x * y
        fx, fy = wx * wx - wy * wy, 2 * wx * wy
        if fn == "z4_rational":
            den = (wx - 1) ** 2 + wy ** 2
            pole = den if pole is None else min(pole, den)
            if den == 0:
                return mags, Fr(0)
            # (w + 1)/(w - 1) = (w + 1) * conj(w - 1) / |w - 1|^2
            fx += ((wx + 1) * (wx - 1) + wy * wy) / den
            fy += (wy * (wx - 1) - (wx + 1) * wy) / den
        x, y = fx + cr, fy + ci
    return mags, pole


@pytest.mark.parametrize("fn", ["z4", "z4_rational"])
def test_fn_maps_against_exact_rational_orbits(oracle_mod, fn):
    """Brute force in exact rationals (the map's definition, no operation order) on random
    starts with Im(w) != 0: wherever every exact |Z_n|^2 is at least 1e-6 (relative) away
    from the bailout 4 and the orbit stays away from the pole, the binary64 oracle count
    equals the exact count.  Catches a dropped term or a sign slip anywhere in q."""
    rng = np.random.default_rng(4067)
    checked = 0
    for _ in range(400):
        z0 = complex(*rng.uniform(-1.5, 1.5, 2))
        c = complex(*rng.uniform(-1.2, 1.2, 2))
        mi = 4
        mags, pole = _exact_fn_orbit(fn, z0, c, mi)
        if any(abs(float(m) - 4.0) < 4e-6 for m in mags):
            continue
        if pole is not None and float(pole) < 0.05:
            continue
        want = len(mags) - 1 if float(mags[-1]) > 4 else mi
        assert oracle.escape_time_fn(fn, z0, c, mi, 64) == want, (z0, c)
        checked += 1
    assert checked > 250
