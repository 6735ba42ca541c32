"""Pins for the CPU oracle against facts fixed by the paper and by mathematics.

Each test names what pins the oracle; none re-types the oracle's own formula.
Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import numpy_ref
from paper_1611_03079_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PRECS = (32, 64)


def _hash(a):
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4").tobytes()).hexdigest()[:16]


# ------------------------------------------------------------------ FP environment
def test_fp_environment_and_contraction_canary(oracle_mod):
    """DESIGN.md reading c-9: no FTZ/DAZ, no FMA contraction in the oracle build."""
    assert oracle.fp_env_ok()
    # a*b = 1 + 2^-29 + 2^-60 exactly; unfused rounding drops 2^-60 -> 0, fused keeps it.
    a = 1.0 + 2.0 ** -30
    assert oracle.mul_add(a, a, -(1.0 + 2.0 ** -29), 64) == 0.0
    af = 1.0 + 2.0 ** -13  # exact in binary32; a*a = 1 + 2^-12 + 2^-26
    assert oracle.mul_add(af, af, -(1.0 + 2.0 ** -12), 32) == 0.0


# ------------------------------------------------------------------ exact orbits
# All values are small dyadics: every operation is exact in binary32 and binary64, so
# the count is fixed by hand iteration (proof by exact arithmetic).  These pin the
# count definition, the strict '>' (|Z|=2 does not escape) and the
# fencepost (Z_0 tested as n = 0).
JULIA_EXACT = [
    # (z0, C, expected)
    (2 + 0j, 0j, 1),        # |2|^2 = 4 not > 4; Z1 = 4 -> 16 > 4
    (1 + 0j, 0j, 100),      # fixed point 1
    (1j, 0j, 100),          # i -> -1 -> 1 -> 1 ...
    (1 + 1j, 0j, 2),        # 1+i -> 2i (|.|^2 = 4, not >) -> -4
    (1.5 + 0j, 0j, 1),      # 2.25 -> 5.0625
    (3 + 0j, 0j, 0),        # |3|^2 = 9 > 4 at n = 0
    (2 + 0j, -2 + 0j, 100),  # 2 -> 2 (fixed point of z^2 - 2)
    (0.5j, -2 + 0j, 1),     # 0.5i -> -2.25 -> escapes at n = 1
    (0j, 1j, 100),          # 0 -> i -> -1+i -> -i -> -1+i ... (period 2)
    (0j, 1 + 0j, 3),        # 0 -> 1 -> 2 -> 5
    (0j, 0j, 100),
    (0j, -1 + 0j, 100),     # 0 -> -1 -> 0
]
MANDEL_EXACT = [  # c with Z_0 = 0
    (1 + 0j, 3), (-2 + 0j, 100), (1j, 100), (2j, 2), (-1 + 0j, 100), (0.25 + 0j, 100),
    (-2.25 + 0j, 1), (0.5 + 0j, 5),
]


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("z0,c,expected", JULIA_EXACT)
def test_exact_orbits_julia(oracle_mod, prec, z0, c, expected):
    assert oracle.escape_time(z0, c, 100, prec) == expected
    # the negated start point gives the same count (Z^2 kills the sign)
    assert oracle.escape_time(-z0, c, 100, prec) == expected


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("c,expected", MANDEL_EXACT)
def test_exact_orbits_mandelbrot(oracle_mod, prec, c, expected):
    assert oracle.escape_time(0j, c, 100, prec) == expected


def test_mandelbrot_pixel_hits_exact_point(oracle_mod):
    """a Mandelbrot pixel whose centre is 1+0i has count 3.  Window centre 1,
    odd size: the centre pixel maps to the centre exactly."""
    for prec in PRECS:
        g = oracle.mandelbrot(1 + 0j, 1.0, 1.0, 5, 5, 100, prec)
        assert g[2, 2] == 3
        # 1x1 grid centred on 0.5: 0 -> 0.5 -> 0.75 -> 1.0625 -> 1.62890625 -> escapes
        assert oracle.mandelbrot(0.5 + 0j, 0.5, 0.5, 1, 1, 100, prec)[0, 0] == 5


# ------------------------------------------------------------------ SPEC examples
def test_spec_pixel_to_complex_examples(oracle_mod):
    """S:111-112 (4x4 grid, span 4) and the odd-grid centre property."""
    assert oracle.pixel_to_complex(0j, 2.0, 2.0, 4, 4, 2, 2) == 0.5 - 0.5j
    assert oracle.pixel_to_complex(0j, 2.0, 2.0, 4, 4, 0, 0) == -1.5 + 1.5j
    z = oracle.pixel_to_complex(0.3 - 0.7j, 1.25, 1.25, 5, 5, 2, 2)
    assert z == 0.3 - 0.7j


def test_spec_render_sequential_3x3(oracle_mod):
    """Julia C=0, centre 0, span 4, 3x3, max 100 -> corners escape early,
    centre 100.  Hand iteration: corner z0 = (-4/3, 4/3): |z0|^2 = 32/9 <= 4,
    z1 = -32/9 i escapes (count 1); edge z0 = 4/3 i: z1 = -16/9, z2 = 256/81,
    |z2|^2 > 4 (count 2)."""
    expected = np.array([[1, 2, 1], [2, 100, 2], [1, 2, 1]])
    for prec in PRECS:
        g = oracle.julia(0j, 0j, 2.0, 2.0, 3, 3, 100, prec)
        np.testing.assert_array_equal(g, expected)


def test_one_pixel_grid(oracle_mod):
    """1x1 grid whose centre is 3+0i with C = 0 -> [0]."""
    assert oracle.julia(0j, 3 + 0j, 1.0, 1.0, 1, 1, 100, 32)[0, 0] == 0


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("prec", PRECS)
def test_c_zero_closed_form(oracle_mod, prec):
    """C = 0: Z_n = Z_0^(2^n).  |Z_0| < 1 never escapes; |Z_0| > 2 escapes at n = 0;
    for 1 < |Z_0| <= 2 the first n with |Z_0|^(2^(n+1)) > 4 is
    n = floor(log2(ln 4 / ln|Z_0|)) (strict >).  Pixels whose real-valued argument is
    within 1e-9 of an integer are skipped (rounding decides them)."""
    n = 257
    g = oracle.julia(0j, 0j, 2.5, 2.5, n, n, 100, prec).astype(np.int64)
    re, im = numpy_ref.axes(0j, 2.5, 2.5, n, n)
    dt = np.float32 if prec == 32 else np.float64
    zr = re.astype(dt).astype(np.float64)[None, :]
    zi = im.astype(dt).astype(np.float64)[:, None]
    r = np.hypot(zr, zi) * np.ones((n, 1))
    inner = r < 1 - 1e-6
    assert (g[inner] == 100).all()
    outer = r > 2 + 1e-6
    assert (g[outer] == 0).all()
    ann = (r > 1 + 1e-6) & (r <= 2 - 1e-6)
    arg = np.log2(np.log(4.0) / np.log(r[ann]))
    ok = np.abs(arg - np.round(arg)) > 1e-9
    expect = np.minimum(np.floor(arg), 100).astype(np.int64)
    assert ok.sum() > 0.99 * ann.sum() and ann.sum() > 10000
    np.testing.assert_array_equal(g[ann][ok], expect[ok])


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("size", [(65, 65), (257, 129), (64, 64), (1921, 1081)])
def test_c_minus_two_only_real_segment_bounded(oracle_mod, prec, size):
    """C = -2: the filled Julia set of z^2 - 2 is exactly [-2, 2].  Real stays real and
    for x in [-2, 2], fl(x^2) in [0, 4] and fl(x^2 - 2) in [-2, 2], so pixels on the
    im == 0 row with |re| <= 2 never escape; every other pixel escapes within the
    limit.  Centre 0: an odd height has such a row, an even height has none."""
    w, h = size
    g = oracle.julia(-2 + 0j, 0j, 2.5, 2.5 * h / w, w, h, 100, prec)
    re, im = numpy_ref.axes(0j, 2.5, 2.5 * h / w, w, h)
    dt = np.float32 if prec == 32 else np.float64
    expected = np.zeros((h, w), dtype=bool)
    for py in range(h):
        if dt(im[py]) == 0:
            expected[py] = np.abs(re.astype(dt)) <= 2
    np.testing.assert_array_equal(g == 100, expected)
    assert expected.any() == (h % 2 == 1)


# ------------------------------------------------------------------ symmetries
@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("c", list(W.FIG2_C) + [-0.8 + 0.156j, 0.285 + 0.01j])
@pytest.mark.parametrize("size", [(257, 257), (333, 777), (64, 48)])
def test_julia_rot180_symmetry(oracle_mod, prec, c, size):
    """count(Z_0) = count(-Z_0) and the pixel-centre map is exactly antisymmetric
    about a zero centre, so the grid is invariant under 180-degree rotation."""
    w, h = size
    g = oracle.julia(c, 0j, 1.7, 1.7 * h / w, w, h, 100, prec)
    np.testing.assert_array_equal(g, g[::-1, ::-1])


@pytest.mark.parametrize("prec", PRECS)
def test_julia_conjugate_flip(oracle_mod, prec):
    """conj(Z)^2 + conj(C) = conj(Z^2 + C): render(conj C) = flipud(render(C)) for a
    window centred on the real axis."""
    for c in W.FIG2_C:
        a = oracle.julia(c, 0.1 + 0j, 1.5, 1.2, 200, 151, 100, prec)
        b = oracle.julia(c.conjugate(), 0.1 + 0j, 1.5, 1.2, 200, 151, 100, prec)
        np.testing.assert_array_equal(a, b[::-1])


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("h", [257, 256])
def test_mandelbrot_vertical_flip(oracle_mod, prec, h):
    """Mandelbrot map with centre on the real axis is invariant under flipud."""
    g = oracle.mandelbrot(-0.5 + 0j, 1.5, 1.5 * h / 257, 257, h, 200, prec)
    np.testing.assert_array_equal(g, g[::-1])


# ------------------------------------------------------------------ Mandelbrot regions
@pytest.mark.parametrize("prec", PRECS)
def test_mandelbrot_known_regions(oracle_mod, prec):
    """|c| > 2 escapes at n = 1 exactly (Z_1 = c); the main cardioid
    (|1 - sqrt(1-4c)| < 1) and the period-2 disc (|c + 1| < 1/4) are inside M, so they
    never escape (margins 0.99 / 0.24 keep away from their boundaries)."""
    n = 513
    g = oracle.mandelbrot(-0.5 + 0j, 2.2, 2.2, n, n, 1000, prec)
    re, im = numpy_ref.axes(-0.5 + 0j, 2.2, 2.2, n, n)
    dt = np.float32 if prec == 32 else np.float64
    c = re.astype(dt).astype(np.float64)[None, :] + 1j * im.astype(dt).astype(np.float64)[:, None]
    far = np.abs(c) > 2.01
    assert far.sum() > 1000 and (g[far] == 1).all()
    card = np.abs(1 - np.sqrt(1 - 4 * c)) < 0.99
    disc = np.abs(c + 1) < 0.24
    assert card.sum() > 1000 and (g[card] == 1000).all()
    assert disc.sum() > 100 and (g[disc] == 1000).all()


# ------------------------------------------------------------------ cap monotonicity
@pytest.mark.parametrize("prec", PRECS)
def test_cap_monotonicity(oracle_mod, prec):
    """count(m1) = min(count(m2), m1) for m1 < m2 (the loop is the same prefix)."""
    c = W.FIG2_C[2]
    g2 = oracle.julia(c, 0j, 1.6, 1.2, 160, 120, 1000, prec).astype(np.int64)
    for m1 in (1, 2, 7, 100, 999):
        g1 = oracle.julia(c, 0j, 1.6, 1.2, 160, 120, m1, prec).astype(np.int64)
        np.testing.assert_array_equal(g1, np.minimum(g2, m1))


# ------------------------------------------------------------------ independent implementations
@pytest.mark.parametrize("case", range(24))
def test_oracle_matches_independent_numpy(oracle_mod, case):
    """The C oracle and the separately written numpy implementation agree exactly on
    seeded fuzz cases (both precisions, Julia and Mandelbrot, ragged sizes)."""
    c, win, w, h, mi = W.fuzz_cases(24, max_side=96)[case]
    mi = min(mi, 300)
    for prec in PRECS:
        a = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec)
        b = numpy_ref.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec)
        np.testing.assert_array_equal(a, b)
        a = oracle.mandelbrot(win.center, win.half_w, win.half_h, w, h, mi, prec)
        b = numpy_ref.mandelbrot(win.center, win.half_w, win.half_h, w, h, mi, prec)
        np.testing.assert_array_equal(a, b)


def _brute(z0, c, mi):
    """Python complex (binary64) with the operations spelled as in S:55-58."""
    x, y = z0.real, z0.imag
    for n in range(mi):
        xx, yy = x * x, y * y
        if xx + yy > 4.0:
            return n
        x, y = (xx - yy) + c.real, (x * y + x * y) + c.imag
    return mi


def test_oracle_matches_brute_force_tiny(oracle_mod):
    """Pure-Python brute force on tiny fp64 grids (every pixel)."""
    for c, win, w, h, mi in W.fuzz_cases(6, max_side=12, seed=7):
        g = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, 64)
        for py in range(h):
            for px in range(w):
                z0 = oracle.pixel_to_complex(win.center, win.half_w, win.half_h, w, h, px, py)
                assert g[py, px] == _brute(z0, c, mi)


def test_sampled_pixels_match_full_grid(oracle_mod):
    rng = np.random.default_rng(3)
    for kind in ("julia", "mandelbrot"):
        for prec in PRECS:
            w, h = 123, 77
            full = (oracle.julia(W.FIG3_C[0], 0.1j, 1.9, 1.2, w, h, 300, prec) if kind == "julia"
                    else oracle.mandelbrot(-0.6 + 0.1j, 1.9, 1.2, w, h, 300, prec))
            px = rng.integers(0, w, 500)
            py = rng.integers(0, h, 500)
            s = oracle.pixels(kind, W.FIG3_C[0], (0.1j if kind == "julia" else -0.6 + 0.1j), 1.9,
                              1.2, w, h, 300, prec, px, py)
            np.testing.assert_array_equal(s, full[py, px])


def test_survey_probe_values(oracle_mod):
    """Σcounts / interior / hash of an independent survey-time
    re-implementation under the same readings (cross-check, not paper facts)."""
    gold = json.load(open(os.path.join(GOLDEN, "survey_probe_values.json")))
    for g in gold["grids"]:
        a = oracle.julia(complex(*g["c"]), complex(*g["center"]), g["half_w"], g["half_h"],
                         g["width"], g["height"], g["max_iter"], g["precision"])
        assert int(a.sum(dtype=np.int64)) == g["sum"], g["name"]
        assert int((a == g["max_iter"]).sum()) == g["interior"], g["name"]
        assert _hash(a) == g["hash"], g["name"]
        if g["name"] == "cfg1":
            assert a[0, 0] == 0 and a[31, 31] == 100
    path = W.circle_path(4096)
    win = W.julia_window(1920, 1080)
    for f in gold["cfg4_frames"]["frames"]:
        a = oracle.julia(complex(path[f["k"]]), win.center, win.half_w, win.half_h, 1920, 1080,
                         100, 32)
        assert int(a.sum(dtype=np.int64)) == f["sum"]
        assert _hash(a) == f["hash"]


# ------------------------------------------------------------------ colour levels
def test_colorize_spec_examples(oracle_mod):
    """count = max_iter -> interior; 0 -> entries[0]; len+1 -> entries[1]."""
    pal, interior = W.palette("classic")
    n = len(pal)
    counts = np.array([100, 0, n + 1, 5, 99], dtype=np.uint16)
    out = oracle.colorize(counts, 100, pal, interior)
    np.testing.assert_array_equal(out[0], interior)
    np.testing.assert_array_equal(out[1], pal[0])
    np.testing.assert_array_equal(out[2], pal[1])
    np.testing.assert_array_equal(out[3], pal[5])
    np.testing.assert_array_equal(out[4], pal[99 % n])


def test_colorize_is_a_pure_per_pixel_map(oracle_mod):
    """permuting two cells permutes exactly those two output pixels."""
    rng = np.random.default_rng(11)
    pal, interior = W.palette("fire")
    counts = rng.integers(0, 301, size=(37, 41)).astype(np.uint16)
    out = oracle.colorize(counts, 300, pal, interior)
    sw = counts.copy()
    sw[3, 4], sw[20, 30] = counts[20, 30], counts[3, 4]
    out2 = oracle.colorize(sw, 300, pal, interior)
    exp = out.copy()
    exp[3, 4], exp[20, 30] = out[20, 30].copy(), out[3, 4].copy()
    np.testing.assert_array_equal(out2, exp)
    assert (out[counts == 300] == interior).all()


# ------------------------------------------------------------------ cardioid path
def test_cardioid_boundary_identity(oracle_mod):
    """"the border of the main cardioid of the Mandelbrot set is this function
    when a = 4": |1 - sqrt(1 - 4 f(t, 4))| = 1; with a = 3.9 the point lies just
    outside (> 1)."""
    for t in np.linspace(-math.pi, math.pi, 1001)[1:-1]:
        c4 = oracle.cardioid_point(t, 4.0)
        assert abs(abs(1 - np.sqrt(1 - 4 * c4)) - 1) < 1e-9
        c39 = oracle.cardioid_point(t, 3.9)
        assert abs(1 - np.sqrt(1 - 4 * c39)) > 1
    assert oracle.cardioid_point(0.0, 3.9) == pytest.approx(1 / 3.9)
    assert oracle.cardioid_point(math.pi, 3.9) == pytest.approx(-3 / 3.9)
    assert oracle.cardioid_point(math.pi / 2, 4.0) == pytest.approx(0.25 + 0.5j)


def test_fig2_parameters_lie_on_the_a39_cardioid(oracle_mod):
    """P:43 + P:53: the four Figure 2 C values were taken on the a = 3.9 cardioid; each
    is within caption rounding (2.5e-7) of f(t, 3.9) for some t, and in caption order
    t decreases (clockwise traversal)."""
    ts = []
    for c in W.FIG2_C:
        grid = np.linspace(-2 * math.pi, math.pi, 20001)
        d = [abs(oracle.cardioid_point(t, 3.9) - c) for t in grid]
        t = grid[int(np.argmin(d))]
        lo, hi = t - 1e-3, t + 1e-3
        for _ in range(80):  # golden-section refine
            m1, m2 = lo + (hi - lo) * 0.382, lo + (hi - lo) * 0.618
            if abs(oracle.cardioid_point(m1, 3.9) - c) < abs(oracle.cardioid_point(m2, 3.9) - c):
                hi = m2
            else:
                lo = m1
        t = 0.5 * (lo + hi)
        assert abs(oracle.cardioid_point(t, 3.9) - c) < 2.5e-7
        ts.append(t)
    unwrapped = np.unwrap(ts)
    assert (np.diff(unwrapped) < 0).all()


# ------------------------------------------------------------------ fast-mode tolerance tools
def test_distance_estimate_closed_form_c_zero(oracle_mod):
    """C = 0: Z_n = Z_0^(2^n), Z'_n = 2^n Z_0^(2^n - 1), so DE = |Z_0| ln|Z_0| exactly for
    every n; the true distance to K = unit disc is |Z_0| - 1 >= DE/2 (Koebe)."""
    for r, th in [(1.5, 0.3), (1.01, 2.0), (3.0, -1.0), (1.0001, 0.7)]:
        z0 = r * complex(math.cos(th), math.sin(th))
        de = oracle.distance_estimate("julia", z0, 0j)
        assert de == pytest.approx(r * math.log(r), rel=1e-9)
        assert de / 2 <= r - 1 + 1e-15
    assert oracle.distance_estimate("julia", 0.5 + 0j, 0j) == 0.0  # inside: never escapes


def test_distance_estimate_mandelbrot_real_axis(oracle_mod):
    """For real c > 1/4 the nearest point of M lies on the main-cardioid border
    e^{it}/2 - e^{2it}/4 (the rightmost part of M), so that distance d must satisfy the
    Koebe-type bounds DE/2 <= d <= 2 DE."""
    t = np.linspace(-math.pi, math.pi, 400001)
    border = np.exp(1j * t) / 2 - np.exp(2j * t) / 4
    for c in (0.3, 0.5, 1.0, 2.5):
        de = oracle.distance_estimate("mandelbrot", 0j, complex(c, 0))
        d = np.abs(border - c).min()
        assert de / 2 <= d <= 2 * de
    assert oracle.distance_estimate("mandelbrot", 0j, -1 + 0j, 10000) == 0.0


def test_nudged_pixels(oracle_mod):
    """nudge = 0 reproduces the sampled strict counts exactly; a 1-ulp nudge of Z_0
    changes some, but few, counts at max_iter 1000 (the problem's own sensitivity)."""
    rng = np.random.default_rng(5)
    px, py = rng.integers(0, 640, 4000), rng.integers(0, 360, 4000)
    args = ("julia", -0.7269 + 0.1889j, 0j, 2.0, 1.125, 640, 360, 1000)
    for prec in PRECS:
        a = oracle.pixels(*args, prec, px, py)
        np.testing.assert_array_equal(a, oracle.pixels_nudged(*args, prec, px, py, 0))
        c = oracle.pixels_nudged(*args, prec, px, py, 1)
        assert (a != c).sum() < 0.1 * a.size
        if prec == 32:
            assert (a != c).sum() > 0


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("kind", ["julia", "mandelbrot"])
@pytest.mark.parametrize("nudge", [1, 3])
def test_nudge_is_exactly_n_ulps(oracle_mod, prec, kind, nudge):
    """The nudge of reading c-10's sensitivity bound moves the start value's real part
    (Julia Z_0, Mandelbrot C) by exactly `nudge` ulps of the working precision toward
    +inf: each sampled count equals the plain escape time of the start value stepped
    with numpy's nextafter, pixel by pixel (a 4-ulp nudge in place of 1 would fail)."""
    rng = np.random.default_rng(8)
    w, h, mi = 320, 180, 1000
    px, py = rng.integers(0, w, 300), rng.integers(0, h, 300)
    c = -0.7269 + 0.1889j
    center, hw, hh = (0j, 2.0, 1.125) if kind == "julia" else (-0.5 + 0j, 1.5, 0.85)
    got = oracle.pixels_nudged(kind, c, center, hw, hh, w, h, mi, prec, px, py, nudge)
    dt = np.float32 if prec == 32 else np.float64
    differs = 0
    for k in range(px.size):
        z = oracle.pixel_to_complex(center, hw, hh, w, h, int(px[k]), int(py[k]))
        re = dt(z.real)
        for _ in range(nudge):
            re = np.nextafter(re, dt(np.inf))
        start = complex(float(re), float(dt(z.imag)))
        want = (oracle.escape_time(start, c, mi, prec) if kind == "julia"
                else oracle.escape_time(0j, start, mi, prec))
        assert got[k] == want, (kind, px[k], py[k])
        differs += int(want != oracle.escape_time(z if kind == "julia" else 0j,
                                                  c if kind == "julia" else z, mi, prec))
    if prec == 32:
        assert differs > 0  # the nudge is not a no-op at this sensitivity
