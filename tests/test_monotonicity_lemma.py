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
