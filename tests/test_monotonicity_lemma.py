"""The escape-monotonicity lemma that kernel A and the amortised P2
rely on: if |C| <= 1.989 and the computed |Z_n|^2 > 4, every later computed |Z_m|^2
is > 4 (or the orbit has overflowed to inf/NaN, which the unordered block-end test also
flags).  Checked here in the strict IEEE operation sequence (reading c-9) with numpy
binary32 / binary64 scalars-as-arrays, on adversarial orbits: starts just outside
|Z| = 2 in every direction, C on and inside the |C| = 1.989 circle (including C
pointing against Z), plus random orbits that escape from inside."""
import numpy as np
import pytest


def _strict_orbit_escapes_stay(dt, z_re, z_im, c_re, c_im, steps):
    x, y = z_re.astype(dt), z_im.astype(dt)
    cr, ci = c_re.astype(dt), c_im.astype(dt)
    escaped = np.zeros(x.shape, dtype=bool)
    with np.errstate(over="ignore", invalid="ignore"):
        for _ in range(steps):
            xx, yy = x * x, y * y
            m = xx + yy
            now = ~(m <= dt(4))  # unordered: inf / NaN count as escaped
            assert not (escaped & ~now).any(), "an escaped orbit came back inside"
            escaped |= now
            xy = x * y
            x, y = (xx - yy) + cr, (xy + xy) + ci
    return escaped


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_escaped_orbits_never_return(dt):
    rng = np.random.default_rng(1611)
    n = 200_000
    # starts just outside radius 2 (relative margins down to one ulp)
    th = rng.uniform(0, 2 * np.pi, n)
    eps = 10.0 ** rng.uniform(-7 if dt is np.float32 else -15, -1, n)
    r0 = 2.0 * (1 + eps)
    # C with |C| <= 1.989, half of them anti-aligned with Z_0^2 (the worst case)
    rc = 1.989 * np.sqrt(rng.uniform(0, 1, n))
    rc[: n // 4] = 1.989
    phi = rng.uniform(0, 2 * np.pi, n)
    phi[: n // 2] = 2 * th[: n // 2] + np.pi
    esc = _strict_orbit_escapes_stay(dt, r0 * np.cos(th), r0 * np.sin(th), rc * np.cos(phi),
                                     rc * np.sin(phi), 60)
    assert esc.all()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_orbits_escaping_from_inside(dt):
    rng = np.random.default_rng(3079)
    n = 200_000
    z = rng.uniform(-2, 2, (2, n))
    rc = 1.989 * np.sqrt(rng.uniform(0, 1, n))
    phi = rng.uniform(0, 2 * np.pi, n)
    esc = _strict_orbit_escapes_stay(dt, z[0], z[1], rc * np.cos(phi), rc * np.sin(phi), 300)
    assert esc.mean() > 0.5  # most of these orbits do escape: the check is exercised


def test_bound_is_needed():
    """Negative control: with |C| = 2.2 anti-aligned to Z_0^2 an orbit that was outside
    radius 2 comes back inside (Z_0 = 2.01 -> 4.04 - 2.2 = 1.84), so the check above has
    teeth and the host-side precondition is not decorative."""
    with pytest.raises(AssertionError, match="came back inside"):
        _strict_orbit_escapes_stay(np.float64, np.array([2.01]), np.array([0.0]),
                                   np.array([-2.2]), np.array([0.0]), 5)


# ---------------------------------------------------------------------------------------
# The same lemma for the FAST sequence the amortised kernels actually run (kernel A, the
# amortised P1/P2; DESIGN.md §5 "State representation", reading c-10): doubled state
# X = 2x, Y = 2y, one iteration YY = Y*Y; T = fma(X,X,-YY); Y' = fma(X,Y,CI);
# X' = fma(T,1/2,CR), escape test fma(X,X,YY) > 16.
#
# binary32: an exact fma emulated in binary64 -- the product of two binary32 values is
# exact in binary64, the sum is rounded to ODD in binary64 (TwoSum error + sticky last
# bit), and rounding that to binary32 is then correctly rounded (53 >= 24 + 2).
# binary64: exact rational arithmetic with its own round-to-nearest-even (the helper of
# test_oracle_fast), on fewer orbits.
# ---------------------------------------------------------------------------------------
def _fma32(a, b, c):
    p = a.astype(np.float64) * b.astype(np.float64)  # exact (48 significant bits)
    cc = c.astype(np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        s = p + cc
        bp = s - p
        ap = s - bp
        e = (p - ap) + (cc - bp)  # TwoSum: p + cc = s + e exactly (finite s)
        odd = (s.view(np.int64) & 1) == 1
        fix = np.isfinite(s) & (e != 0) & ~odd
        s = np.where(fix, np.nextafter(s, np.where(e > 0, np.inf, -np.inf)), s)
        return s.astype(np.float32)


def test_fma32_emulation_is_correctly_rounded():
    """The emulation against exact rational rounding (test_oracle_fast's _rn) on random
    operands, including results in binary32's subnormal range and exact ties."""
    from fractions import Fraction
    from test_oracle_fast import _rn
    rng = np.random.default_rng(99)
    n = 3000
    a = (rng.standard_normal(n) * 10.0 ** rng.integers(-22, 8, n)).astype(np.float32)
    b = (rng.standard_normal(n) * 10.0 ** rng.integers(-22, 8, n)).astype(np.float32)
    c = (rng.standard_normal(n) * 10.0 ** rng.integers(-44, 14, n)).astype(np.float32)
    c[:300] = -(a[:300].astype(np.float64) * b[:300]).astype(np.float32)  # cancellation
    got = _fma32(a, b, c)
    for i in range(n):
        want = _rn(Fraction(float(a[i])) * Fraction(float(b[i])) + Fraction(float(c[i])), 32)
        assert Fraction(float(got[i])) == want, (a[i], b[i], c[i])


def _fast_orbit_escapes_stay_f32(z_re, z_im, c_re, c_im, steps):
    f32 = np.float32
    X = (z_re.astype(f32) * f32(2)).astype(f32)
    Y = (z_im.astype(f32) * f32(2)).astype(f32)
    CR = (c_re.astype(f32) * f32(2)).astype(f32)
    CI = (c_im.astype(f32) * f32(2)).astype(f32)
    half = np.full(X.shape, 0.5, dtype=f32)
    escaped = np.zeros(X.shape, dtype=bool)
    with np.errstate(over="ignore", invalid="ignore"):
        for _ in range(steps):
            YY = Y * Y
            M = _fma32(X, X, YY)
            now = ~(M <= f32(16))  # unordered: inf / NaN count as escaped
            assert not (escaped & ~now).any(), "an escaped orbit came back inside"
            escaped |= now
            T = _fma32(X, X, -YY)
            X, Y = _fma32(T, half, CR), _fma32(X, Y, CI)
    return escaped


def _adversarial_starts(rng, n, eps_lo):
    th = rng.uniform(0, 2 * np.pi, n)
    r0 = 2.0 * (1 + 10.0 ** rng.uniform(eps_lo, -1, n))
    rc = 1.989 * np.sqrt(rng.uniform(0, 1, n))
    rc[: n // 4] = 1.989
    phi = rng.uniform(0, 2 * np.pi, n)
    phi[: n // 2] = 2 * th[: n // 2] + np.pi  # C against Z_0^2: the worst case
    return r0 * np.cos(th), r0 * np.sin(th), rc * np.cos(phi), rc * np.sin(phi)


def test_fast_sequence_escaped_orbits_never_return_f32():
    rng = np.random.default_rng(1612)
    zr, zi, cr, ci = _adversarial_starts(rng, 200_000, -7)
    assert _fast_orbit_escapes_stay_f32(zr, zi, cr, ci, 60).all()
    z = rng.uniform(-2, 2, (2, 200_000))
    rc = 1.989 * np.sqrt(rng.uniform(0, 1, 200_000))
    phi = rng.uniform(0, 2 * np.pi, 200_000)
    esc = _fast_orbit_escapes_stay_f32(z[0], z[1], rc * np.cos(phi), rc * np.sin(phi), 300)
    assert esc.mean() > 0.5


def test_fast_sequence_escaped_orbits_never_return_f64():
    """binary64 FAST sequence in exact rationals with round-to-nearest-even; an orbit is
    followed until |X|^2 + |Y|^2 passes 2^400 (far past any rounding effect: the next
    modulus is at least its square minus 4|C| minus a relative 2^-50)."""
    from fractions import Fraction
    from test_oracle_fast import _rn
    rng = np.random.default_rng(1613)
    zr, zi, cr, ci = _adversarial_starts(rng, 1500, -15)
    R = lambda v: _rn(v, 64)  # noqa: E731
    big = Fraction(2) ** 400
    for k in range(zr.size):
        X, Y = 2 * Fraction(float(zr[k])), 2 * Fraction(float(zi[k]))
        CR, CI = 2 * Fraction(float(cr[k])), 2 * Fraction(float(ci[k]))
        escaped = False
        for _ in range(60):
            YY = R(Y * Y)
            M = R(X * X + YY)
            now = M > 16
            assert not (escaped and not now), ("came back inside", k)
            escaped = escaped or now
            if M > big:
                break
            T = R(X * X - YY)
            X, Y = R(T / 2 + CR), R(X * Y + CI)
        assert escaped, k


def test_fast_sequence_bound_is_needed():
    """Negative control for the FAST sequence, as test_bound_is_needed."""
    with pytest.raises(AssertionError, match="came back inside"):
        _fast_orbit_escapes_stay_f32(np.array([2.01]), np.array([0.0]), np.array([-2.2]),
                                     np.array([0.0]), 5)
