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
