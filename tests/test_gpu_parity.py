"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

STRICT modes: bit-exact counts on every BASELINE config (full frames where the oracle
finishes in seconds, sampled pixels at cfg4/cfg5 full size), fuzzed windows, ragged
and degenerate sizes, bands and C-paths.  FAST modes: the DESIGN.md reading c-10
tolerance -- the differing fraction is at most max(1e-4, 4 x the oracle's own 1-ulp
sensitivity) and every differing pixel lies within one pixel of a boundary: of a count
level set (its fast count occurs in the strict 3x3 neighbourhood) or of the set itself
(distance estimate DE/2 <= sqrt(2) * pitch).
"""
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from paper_1611_03079_b200 import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def fr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1611_03079_b200 import binding
    binding.load()
    return binding


def np16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def sample16(t, py, px):
    """t[py, px] for a uint16 CUDA tensor (indexed through an int16 view)."""
    v = t.view(torch.int16)[torch.as_tensor(py, device=t.device), torch.as_tensor(px, device=t.device)]
    return v.cpu().numpy().view(np.uint16)


def strict(prec, fr):
    return fr.Mode.FP32_STRICT if prec == 32 else fr.Mode.FP64_STRICT


def fast(prec, fr):
    return fr.Mode.FP32_FAST if prec == 32 else fr.Mode.FP64_FAST


def _sentinel_outputs(fr, w, h, mi, bands, palette):
    """Output buffers pre-filled with a value no correct render leaves (count mi + 1;
    RGBA 0x5A bytes), so a pixel a kernel never writes fails the comparison instead of
    passing on stale memory from the caching allocator (a dropped-work bug once hid
    behind exactly that)."""
    rows = h if bands is fr.FULL_FRAME else fr.band_local_rows(h, bands)
    s = (mi + 1) & 0xFFFF
    out = torch.full((rows, w), s - 65536 if s >= 32768 else s, dtype=torch.int16,
                     device="cuda").view(torch.uint16)
    rgba = (torch.full((rows, w, 4), 0x5A, dtype=torch.uint8, device="cuda")
            if palette is not None else None)
    return out, rgba


def gpu_julia(fr, c, win, w, h, mi, mode, bands=None, palette=None):
    bands = bands or fr.FULL_FRAME
    out, rgba = _sentinel_outputs(fr, w, h, mi, bands, palette)
    r = fr.julia_render_ex(c, win, w, h, mi, mode, bands, out=out, palette=palette,
                           out_rgba=rgba)
    torch.cuda.synchronize()
    if palette is not None:
        return np16(r[0]), r[1].cpu().numpy()
    return np16(r)


def gpu_mandel(fr, win, w, h, mi, mode, bands=None):
    bands = bands or fr.FULL_FRAME
    out, _ = _sentinel_outputs(fr, w, h, mi, bands, None)
    r = fr.mandelbrot_param_map(win, w, h, mi, mode, bands, out=out)
    torch.cuda.synchronize()
    return np16(r)


def test_native_library_is_loaded(fr):
    maps = open("/proc/self/maps").read()
    assert "libfractal.so" in maps
    assert "sm_100a" in fr.version()
    assert torch.cuda.get_device_capability() == (10, 0)


# ------------------------------------------------------------------ strict, full frames
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_strict_configs_full_frame(fr, name):
    cfg = W.configs()[name]
    win = cfg.window
    ref = oracle.julia(cfg.c, win.center, win.half_w, win.half_h, cfg.width, cfg.height,
                       cfg.max_iter, cfg.precision)
    if cfg.colorize:
        pal = W.palette("classic")
        got, rgba = gpu_julia(fr, cfg.c, win, cfg.width, cfg.height, cfg.max_iter,
                              strict(cfg.precision, fr), palette=pal)
        np.testing.assert_array_equal(rgba, oracle.colorize(ref, cfg.max_iter, *pal))
    else:
        got = gpu_julia(fr, cfg.c, win, cfg.width, cfg.height, cfg.max_iter,
                        strict(cfg.precision, fr))
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("c", list(W.FIG2_C) + list(W.FIG3_C))
def test_strict_paper_parameters(fr, prec, c):
    """Figure 2 and Figure 3 parameter values at 256^2."""
    win = W.julia_window(256, 256)
    ref = oracle.julia(c, win.center, win.half_w, win.half_h, 256, 256, 100, prec)
    np.testing.assert_array_equal(gpu_julia(fr, c, win, 256, 256, 100, strict(prec, fr)), ref)


# ------------------------------------------------------------------ non-monotone regime
# |C| > 1.989: the escape-monotonicity lemma does not hold, an orbit can
# leave radius 2 and come back (SURVEY c-11: C = -5, z = sqrt 5 -> 0), so the host must
# keep these frames on the per-iteration-test kernels.  max_iter 100 runs the static
# kernels, 300 and 1000 the heavy-tail scheduler (two phases or refill).
NONMONO_C = (-2 + 0j, -2.1 + 0j, 2j, -5 + 0j, 3 + 1j, 1.995 + 0j, -1.4 - 1.4j)


@pytest.mark.parametrize("c", NONMONO_C)
@pytest.mark.parametrize("mi", [100, 300, 1000])
def test_nonmonotone_julia_strict(fr, c, mi):
    w, h = 241, 161  # odd H: one row lies on the real axis
    win = W.Window(0j, 2.6, 2.6 * h / w)
    for prec in (32, 64):
        ref = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec)
        np.testing.assert_array_equal(gpu_julia(fr, c, win, w, h, mi, strict(prec, fr)), ref)


def test_nonmonotone_c_minus_two_segment(fr):
    """C = -2 through the kernels: exactly the pixels of the im == 0 row with |re| <= 2
    stay bounded (proof in test_oracle_pins), strict and fast, both precisions."""
    w, h = 401, 201
    win = W.Window(0j, 2.5, 2.5 * h / w)
    re = np.array([oracle.pixel_to_complex(0j, win.half_w, win.half_h, w, h, px, 0).real
                   for px in range(w)])
    for mi in (100, 1000):
        for mode in ("FP32_STRICT", "FP32_FAST", "FP64_STRICT", "FP64_FAST"):
            dt = np.float32 if "32" in mode else np.float64
            g = gpu_julia(fr, -2 + 0j, win, w, h, mi, fr.Mode[mode])
            expected = np.zeros((h, w), dtype=bool)
            expected[h // 2] = np.abs(re.astype(dt)) <= 2
            np.testing.assert_array_equal(g == mi, expected, err_msg=f"{mode} mi={mi}")


def test_nonmonotone_c_zero_closed_form(fr):
    """C = 0 through the kernels: |z0| < 1 never escapes, |z0| > 2 escapes at 0, and
    count = floor(log2(ln 4 / ln|z0|)) in between (away from integer arguments)."""
    n = 257
    re, im = (np.array([oracle.pixel_to_complex(0j, 2.5, 2.5, n, n, k, k).real
                        for k in range(n)]),
              np.array([oracle.pixel_to_complex(0j, 2.5, 2.5, n, n, k, k).imag
                        for k in range(n)]))
    for mode, dt in (("FP32_STRICT", np.float32), ("FP32_FAST", np.float32),
                     ("FP64_STRICT", np.float64), ("FP64_FAST", np.float64)):
        for mi in (100, 1000):
            g = gpu_julia(fr, 0j, W.Window(0j, 2.5, 2.5), n, n, mi, fr.Mode[mode]).astype(np.int64)
            r = np.hypot(re.astype(dt).astype(np.float64)[None, :],
                         im.astype(dt).astype(np.float64)[:, None])
            assert (g[r < 1 - 1e-6] == mi).all() and (g[r > 2 + 1e-6] == 0).all()
            ann = (r > 1 + 1e-6) & (r <= 2 - 1e-6)
            arg = np.log2(np.log(4.0) / np.log(r[ann]))
            ok = np.abs(arg - np.round(arg)) > 1e-9
            np.testing.assert_array_equal(g[ann][ok], np.floor(arg)[ok])


@pytest.mark.parametrize("case", range(96))
def test_strict_fuzz(fr, case):
    c, win, w, h, mi = W.fuzz_cases(96, max_side=300)[case]
    for prec in (32, 64):
        ref = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec)
        np.testing.assert_array_equal(gpu_julia(fr, c, win, w, h, mi, strict(prec, fr)), ref)
        ref = oracle.mandelbrot(win.center, win.half_w, win.half_h, w, h, mi, prec)
        np.testing.assert_array_equal(gpu_mandel(fr, win, w, h, mi, strict(prec, fr)), ref)


@pytest.mark.parametrize("case", range(32))
def test_strict_fuzz_large(fr, case):
    """A second seeded set with larger, ragged frames (up to 600 px a side) and
    max_iter in {100, 300, 1000}: the two-phase path (P1 + P2) and S2 on many windows,
    strict fp32 and fp64, Julia and Mandelbrot, bit-exact."""
    c, win, w, h, _ = W.fuzz_cases(32, max_side=600, seed=W.FUZZ_SEED + 1)[case]
    mi = (100, 300, 1000)[case % 3]
    for prec in (32, 64):
        ref = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec)
        np.testing.assert_array_equal(gpu_julia(fr, c, win, w, h, mi, strict(prec, fr)), ref)
        ref = oracle.mandelbrot(win.center, win.half_w, win.half_h, w, h, mi, prec)
        np.testing.assert_array_equal(gpu_mandel(fr, win, w, h, mi, strict(prec, fr)), ref)


@pytest.mark.parametrize("size", [(1, 1), (1, 37), (37, 1), (33, 9), (31, 7), (257, 129),
                                  (8, 4), (32, 8), (65, 17)])
@pytest.mark.parametrize("mi", [1, 2, 7, 100])
def test_strict_ragged_and_degenerate(fr, size, mi):
    w, h = size
    c = W.FIG2_C[2]
    win = W.julia_window(w, h, span_re=3.2)
    for prec in (32, 64):
        ref = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec)
        np.testing.assert_array_equal(gpu_julia(fr, c, win, w, h, mi, strict(prec, fr)), ref)
        ref = oracle.mandelbrot(-0.5 + 0j, 1.5, 1.5 * h / w, w, h, mi, prec)
        got = gpu_mandel(fr, (-0.5 + 0j, 1.5, 1.5 * h / w), w, h, mi, strict(prec, fr))
        np.testing.assert_array_equal(got, ref)


def test_max_iter_65535(fr):
    """The uint16 limit: interior pixels report 65535."""
    win = W.julia_window(24, 16)
    for prec in (32, 64):
        ref = oracle.julia(-0.12 + 0.75j, win.center, win.half_w, win.half_h, 24, 16, 65535, prec)
        assert (ref == 65535).any()
        got = gpu_julia(fr, -0.12 + 0.75j, win, 24, 16, 65535, strict(prec, fr))
        np.testing.assert_array_equal(got, ref)


def test_every_pixel_written_once(fr):
    """Sentinel-filled output: nothing left unwritten, nothing written outside."""
    w, h = 333, 77
    buf = torch.full((h * w + 64,), -1, dtype=torch.int16, device="cuda").view(torch.uint16)
    out = buf[: h * w].view(h, w)
    fr.julia_render_ex(0.285 + 0.01j, W.julia_window(w, h), w, h, 100, fr.Mode.FP32_STRICT,
                       out=out)
    torch.cuda.synchronize()
    a = np16(buf)
    assert (a[: h * w] != 0xFFFF).all()
    assert (a[h * w:] == 0xFFFF).all()


def test_largest_frame(fr):
    """W*H = 2^31 (the S:182 limit): 64-bit offsets; corners and a sample match."""
    w, h = 65536, 32768
    out = torch.full((h, w), -1, dtype=torch.int16, device="cuda").view(torch.uint16)
    win = W.julia_window(w, h)
    fr.julia_render_ex(-0.8 + 0.156j, win, w, h, 3, fr.Mode.FP32_STRICT, out=out)
    torch.cuda.synchronize()
    assert not bool((out.view(torch.int16) == -1).any())
    rng = np.random.default_rng(1)
    px = np.r_[0, w - 1, 0, w - 1, rng.integers(0, w, 2000)]
    py = np.r_[0, 0, h - 1, h - 1, rng.integers(0, h, 2000)]
    ref = oracle.pixels("julia", -0.8 + 0.156j, win.center, win.half_w, win.half_h, w, h, 3, 32,
                        px, py)
    got = sample16(out, py, px)
    np.testing.assert_array_equal(got, ref)
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["FP32_STRICT", "FP32_FAST", "FP64_STRICT"])
def test_tall_frame_linear_grid(fr, mode):
    """More than 65535 tile rows: kernels S/S2 fall back from the (x, y[, z]) grid to
    linear tiles with a division (tile_of), with a ragged 37-pixel width.  Every pixel is
    written, and the sampled pixels are bit-exact: strict modes against the strict
    oracle, fast mode (kernel S2) against the FAST oracle."""
    w, h = 37, 1_100_000  # S: 137,500 tile rows; S2: 68,750 (both > 65535)
    m = fr.Mode[mode]
    out = torch.full((h, w), -1, dtype=torch.int16, device="cuda").view(torch.uint16)
    win = W.julia_window(w, h, span_re=1.0e-4)  # half_h = 1.49: a thin column through the set
    c = -0.8 + 0.156j
    fr.julia_render_ex(c, win, w, h, 60, m, out=out)
    torch.cuda.synchronize()
    assert not bool((out.view(torch.int16) == -1).any())
    rng = np.random.default_rng(2)
    px = np.r_[0, w - 1, 0, w - 1, rng.integers(0, w, 3000)]
    py = np.r_[0, 0, h - 1, h - 1, rng.integers(0, h, 3000)]
    got = sample16(out, py, px)
    prec = 64 if mode.startswith("FP64") else 32
    ref = oracle.pixels("julia", c, win.center, win.half_w, win.half_h, w, h, 60, prec, px, py,
                        fast=mode.endswith("FAST"))
    np.testing.assert_array_equal(got, ref)
    del out
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ paths (cfg4)
def test_path_equals_single_frames(fr):
    """julia_render_path(C[])[k] == julia_render_ex(C[k]) byte-exactly, across the
    1024-frame launch chunk boundary, in fast and strict modes."""
    cs = W.circle_path(1100)
    w, h = 48, 27
    win = W.julia_window(w, h)
    # max_iter 100: whole vote blocks; 99: the tail block after the last whole one
    for mode, mi in ((fr.Mode.FP32_FAST, 100), (fr.Mode.FP32_FAST, 99),
                     (fr.Mode.FP32_STRICT, 100), (fr.Mode.FP64_FAST, 100)):
        pal = W.palette("fire")
        frames = torch.full((len(cs), h, w), mi + 1, dtype=torch.int16,
                            device="cuda").view(torch.uint16)  # sentinel: never a count
        rgba = torch.full((len(cs), h, w, 4), 0x5A, dtype=torch.uint8, device="cuda")
        frames, rgba = fr.julia_render_path(cs, win, w, h, mi, mode, out=frames, palette=pal,
                                            out_rgba=rgba)
        torch.cuda.synchronize()
        frames = np16(frames)
        rgba = rgba.cpu().numpy()
        for k in (0, 1, 511, 1023, 1024, 1099):
            one, one_rgba = gpu_julia(fr, complex(cs[k]), win, w, h, mi, mode, palette=pal)
            np.testing.assert_array_equal(frames[k], one)
            np.testing.assert_array_equal(rgba[k], one_rgba)


def test_cfg4_strict_all_frames(fr):
    """cfg4 at full size, ALL of it (north_star "bit-exact strict-mode counts on
    all five configs"): 4096 frames of 1080p rendered in one call (64-bit offsets, 17 GB
    of counts), every frame compared with the oracle's frame (5.4e10 oracle iterations,
    spread over the host cores while the next frame is copied back)."""
    cfg = W.configs()["cfg4"]
    cs = W.circle_path(cfg.n_frames)
    win = cfg.window
    out = fr.julia_render_path(cs, win, cfg.width, cfg.height, cfg.max_iter, fr.Mode.FP32_STRICT)
    torch.cuda.synchronize()

    def ref(k):
        return oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, cfg.width,
                            cfg.height, cfg.max_iter, 32, threads=2)

    nthreads = max(1, oracle.default_threads() // 2)
    bad = []
    with ThreadPoolExecutor(nthreads) as ex:
        step = 64
        for k0 in range(0, cfg.n_frames, step):
            refs = list(ex.map(ref, range(k0, min(k0 + step, cfg.n_frames))))
            got = out[k0:k0 + len(refs)].view(torch.int16).cpu().numpy().view(np.uint16)
            for i, r in enumerate(refs):
                if not np.array_equal(got[i], r):
                    bad.append(k0 + i)
    assert not bad, f"{len(bad)} frames differ, first {bad[:8]}"
    del out
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ Mandelbrot cfg5
def test_cfg5_strict_full_size_sampled(fr):
    """cfg5: 16384^2, max_iter 10000, fp64 deep zoom, full render on the GPU; 6000
    random pixels plus one full row compared with the oracle."""
    cfg = W.configs()["cfg5"]
    win = cfg.window
    got = fr.mandelbrot_param_map(win, cfg.width, cfg.height, cfg.max_iter, fr.Mode.FP64_STRICT)
    torch.cuda.synchronize()
    rng = np.random.default_rng(55)
    px = np.r_[rng.integers(0, cfg.width, 6000), np.arange(0, cfg.width, 4)]
    py = np.r_[rng.integers(0, cfg.height, 6000), np.full(cfg.width // 4, 8191)]
    ref = oracle.pixels("mandelbrot", 0j, win.center, win.half_w, win.half_h, cfg.width,
                        cfg.height, cfg.max_iter, 64, px, py)
    np.testing.assert_array_equal(sample16(got, py, px), ref)
    del got
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["FP64_STRICT", "FP64_FAST"])
def test_cfg5_full_frame_hash(fr, mode):
    """cfg5 at full size, ALL of it: the GPU frame (16384^2, max_iter 10000, fp64) hashed
    block by block against tests/golden/cfg5_oracle.json, which the committed
    oracle-only script tools/oracle_cfg5_golden.py computed (parallel render ==
    sequential render, bit for bit).  FP64_FAST compares against the FAST oracle's
    hashes when they are present."""
    import hashlib
    import json
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                         "cfg5_oracle.json")))
    if mode not in golden:
        pytest.skip(f"no oracle hashes for {mode} in cfg5_oracle.json")
    ref = golden[mode]
    cfg = W.configs()["cfg5"]
    got = fr.mandelbrot_param_map(cfg.window, cfg.width, cfg.height, cfg.max_iter,
                                  fr.Mode[mode])
    torch.cuda.synchronize()
    a = got.view(torch.int16).cpu().numpy().view(np.uint16)
    del got
    torch.cuda.empty_cache()
    br = ref["block_rows"]
    bad = [i for i, h in enumerate(ref["blocks"])
           if hashlib.sha256(a[i * br:(i + 1) * br].astype("<u2").tobytes()).hexdigest() != h]
    assert not bad, f"row blocks differing from the oracle: {bad}"
    assert int(a.sum(dtype=np.int64)) == ref["sum_counts"]
    assert int((a == cfg.max_iter).sum()) == ref["interior"]
    assert hashlib.sha256(a.astype("<u2").tobytes()).hexdigest() == ref["sha256"]


# ------------------------------------------------------------------ bands
@pytest.mark.parametrize("n_ranks", [2, 4, 8])
def test_bands_equal_rows_of_full_render(fr, n_ranks):
    w, h, br = 960, 547, 15
    win = W.julia_window(w, h)
    c = -0.7269 + 0.1889j
    pal = W.palette("classic")
    full, full_rgba = gpu_julia(fr, c, win, w, h, 1000, fr.Mode.FP32_FAST, palette=pal)
    mfull = gpu_mandel(fr, (-0.6 + 0j, 1.6, 1.6 * h / w), w, h, 500, fr.Mode.FP64_STRICT)
    rows_seen = []
    for rank in range(n_ranks):
        b = fr.Bands(br, n_ranks, rank)
        rows = [fr.band_global_row(h, b, i) for i in range(fr.band_local_rows(h, b))]
        rows_seen += rows
        part, part_rgba = gpu_julia(fr, c, win, w, h, 1000, fr.Mode.FP32_FAST, bands=b,
                                    palette=pal)
        np.testing.assert_array_equal(part, full[rows])
        np.testing.assert_array_equal(part_rgba, full_rgba[rows])
        mpart = gpu_mandel(fr, (-0.6 + 0j, 1.6, 1.6 * h / w), w, h, 500, fr.Mode.FP64_STRICT,
                           bands=b)
        np.testing.assert_array_equal(mpart, mfull[rows])
    assert sorted(rows_seen) == list(range(h))


# ------------------------------------------------------------------ colour levels
@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 1000, 12345, 1 << 20])
@pytest.mark.parametrize("offset", [0, 1])
def test_colorize_standalone(fr, n, offset):
    rng = np.random.default_rng(n + offset)
    counts = rng.integers(0, 1001, size=n + offset).astype(np.uint16)
    counts[::97] = 1000
    t = torch.from_numpy(counts.view(np.int16)).cuda().view(torch.uint16)[offset:]
    for name in ("classic", "fire"):
        pal = W.palette(name)
        got = fr.colorize(t, 1000, pal)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy(), oracle.colorize(counts[offset:], 1000, *pal))
    odd = (np.arange(7 * 4, dtype=np.uint8).reshape(7, 4), np.array([9, 8, 7, 6], np.uint8))
    got = fr.colorize(t, 1000, odd)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), oracle.colorize(counts[offset:], 1000, *odd))


_COLORIZE_GRID = r"""
import numpy as np, torch, sys
import oracle
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
n = 3 * (1 << 20) + 4321  # > 4 blocks of 256 pixels per warp of the forced 1-CTA/SM grid
rng = np.random.default_rng(5)
counts = rng.integers(0, 1001, size=n).astype(np.uint16)
counts[::89] = 1000
t = torch.from_numpy(counts.view(np.int16)).cuda().view(torch.uint16)
pal = W.palette("fire")
rgba = fr.colorize(t, 1000, pal)
torch.cuda.synchronize()
ok = np.array_equal(rgba.cpu().numpy().reshape(-1, 4), oracle.colorize(counts, 1000, *pal).reshape(-1, 4))
sys.exit(0 if ok else 1)
"""


@pytest.mark.parametrize("ctas", ["1", "3"])
def test_colorize_grid_stride(ctas):
    """The warp-contiguous colorize kernel with a forced small grid (FRACTAL_COLORIZE_CTAS):
    every warp runs its unrolled 4-block loop, the remainder loop and the ragged tail."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, FRACTAL_COLORIZE_CTAS=ctas)
    r = subprocess.run([sys.executable, "-c", _COLORIZE_GRID], cwd=root, env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("name,mode,pal_name", [("cfg2", "FP32_FAST", "fire"),
                                               ("cfg3", "FP32_FAST", "classic"),
                                               ("cfg3", "FP64_STRICT", "fire")])
def test_fused_colorize_matches_standalone(fr, name, mode, pal_name):
    """Fused colour levels (S2 at max_iter < 256, P1 + P2 above; palettes read from the
    device copy or shared memory) equal the standalone colorize of the same counts."""
    cfg = W.configs()[name]
    pal = W.palette(pal_name)
    counts, rgba = gpu_julia(fr, cfg.c, cfg.window, cfg.width, cfg.height, cfg.max_iter,
                             fr.Mode[mode], palette=pal)
    t = torch.from_numpy(counts.view(np.int16)).cuda().view(torch.uint16)
    again = fr.colorize(t, cfg.max_iter, pal)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(again.cpu().numpy(), rgba)


def test_two_palettes_alternating(fr):
    """The device palette cache keys on content: alternating palettes never mix."""
    cfg = W.configs()["cfg2"]
    for pal_name in ("fire", "classic", "fire"):
        pal = W.palette(pal_name)
        counts, rgba = gpu_julia(fr, cfg.c, cfg.window, 480, 270, cfg.max_iter,
                                 fr.Mode.FP32_FAST, palette=pal)
        t = torch.from_numpy(counts.view(np.int16)).cuda().view(torch.uint16)
        again = fr.colorize(t, cfg.max_iter, pal)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(again.cpu().numpy(), rgba)


# ------------------------------------------------------------------ fast-mode tolerance
def _within_one_pixel_of_a_boundary(kind, c, win, w, h, mi, prec, px, py, fast_vals):
    """DESIGN.md reading c-10: a differing pixel p passes iff it lies within one pixel of
    (b) a count level-set boundary -- its fast count occurs among the strict counts of its
    3x3 neighbourhood (the escape test |Z_n|^2 > 4 is a knife edge there) -- or of
    (a) the set boundary -- distance estimate DE(p)/2 <= sqrt(2) * pitch (Koebe: the true
    distance is >= DE/2).  Returns (all_pass, n_level, n_de, worst_de_px)."""
    px = np.asarray(px, np.int64)
    py = np.asarray(py, np.int64)
    offs = [(dx, dy) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    nx = np.clip(px[:, None] + np.array([o[0] for o in offs])[None, :], 0, w - 1)
    ny = np.clip(py[:, None] + np.array([o[1] for o in offs])[None, :], 0, h - 1)
    neigh = oracle.pixels(kind, c, win.center, win.half_w, win.half_h, w, h, mi, prec,
                          nx.ravel(), ny.ravel()).reshape(nx.shape)
    level = (neigh == np.asarray(fast_vals)[:, None]).any(axis=1)
    rest = ~level
    worst = 0.0
    de_ok = np.ones(px.shape, bool)
    if rest.any():
        pitch = 2.0 * max(win.half_w / w, win.half_h / h)
        idx = np.flatnonzero(rest)
        chunks = np.array_split(idx, max(1, min(64, idx.size // 16)))
        with ThreadPoolExecutor(max_workers=oracle.default_threads()) as ex:
            parts = list(ex.map(lambda ii: oracle.distance_pixels(
                kind, c, win.center, win.half_w, win.half_h, w, h, px[ii], py[ii]), chunks))
        de = np.concatenate(parts)
        de_ok[idx] = de / 2 <= math.sqrt(2) * pitch
        worst = float((de / 2 / pitch).max())
    return bool((level | de_ok).all()), int(level.sum()), int(rest.sum()), worst


def _sensitivity(kind, c, win, w, h, mi, prec, n=None, seed=9):
    """Fraction of pixels whose strict count changes when the start value moves by one
    ulp (over the whole frame, or n random pixels)."""
    if n is None:
        py, px = np.divmod(np.arange(w * h, dtype=np.int64), w)
    else:
        rng = np.random.default_rng(seed)
        px, py = rng.integers(0, w, n), rng.integers(0, h, n)
    a = oracle.pixels(kind, c, win.center, win.half_w, win.half_h, w, h, mi, prec, px, py)
    b = oracle.pixels_nudged(kind, c, win.center, win.half_w, win.half_h, w, h, mi, prec, px, py, 1)
    return float((a != b).mean())


def _check_fast_frame(kind, c, win, w, h, mi, prec, got, ref, label, sample=20000):
    diff = np.argwhere(got != ref)
    frac = diff.shape[0] / ref.size
    sens = _sensitivity(kind, c, win, w, h, mi, prec)
    print(f"{label}: fast-vs-strict {frac:.3e}, 1-ulp sensitivity {sens:.3e}")
    assert frac <= max(1e-4, 4 * sens)
    if diff.size:
        sel = diff if diff.shape[0] <= sample else diff[np.random.default_rng(0).choice(
            diff.shape[0], sample, replace=False)]
        ok, nl, nd, worst = _within_one_pixel_of_a_boundary(
            kind, c, win, w, h, mi, prec, sel[:, 1], sel[:, 0], got[sel[:, 0], sel[:, 1]])
        print(f"{label}: {nl} level-set, {nd} DE-checked, worst DE/2 {worst:.3f} px")
        assert ok


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_fast_mode_tolerance_julia(fr, name):
    cfg = W.configs()[name]
    win = cfg.window
    ref = oracle.julia(cfg.c, win.center, win.half_w, win.half_h, cfg.width, cfg.height,
                       cfg.max_iter, cfg.precision)
    got = gpu_julia(fr, cfg.c, win, cfg.width, cfg.height, cfg.max_iter, fast(cfg.precision, fr))
    _check_fast_frame("julia", cfg.c, win, cfg.width, cfg.height, cfg.max_iter, cfg.precision,
                      got, ref, name)


def test_fast_mode_tolerance_cfg4_frames(fr):
    cfg = W.configs()["cfg4"]
    cs = W.circle_path(cfg.n_frames)
    ks = [0, 700, 1365, 2047, 3000]
    out = fr.julia_render_path(cs[ks], cfg.window, cfg.width, cfg.height, cfg.max_iter,
                               fr.Mode.FP32_FAST)
    torch.cuda.synchronize()
    win = cfg.window
    for i, k in enumerate(ks):
        ref = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, cfg.width,
                           cfg.height, cfg.max_iter, 32)
        _check_fast_frame("julia", complex(cs[k]), win, cfg.width, cfg.height, cfg.max_iter, 32,
                          np16(out[i]), ref, f"cfg4 frame {k}")


def test_bench_launch_fast_frames(fr):
    """The exact launch bench.py times (512 frames of the |C| = 0.7885 circle path of
    F = 512, 1080p, max_iter 100, FP32_FAST, one julia_render_path call): sampled frames
    are byte-identical to independent single-frame renders (kernel S2; FAST is one
    arithmetic across kernels) and within reading c-10 of the strict oracle."""
    cfg = W.configs()["cfg4"]
    cs = W.circle_path(512, 0.7885)
    win = W.julia_window(1920, 1080)
    out = torch.full((512, 1080, 1920), 101, dtype=torch.int16, device="cuda").view(torch.uint16)
    fr.julia_render_path(cs, win, 1920, 1080, 100, fr.Mode.FP32_FAST, out=out)
    torch.cuda.synchronize()
    assert not bool((out.view(torch.int16) == 101).any()), "unwritten pixels"
    for k in (0, 1, 127, 256, 383, 511):
        one = gpu_julia(fr, complex(cs[k]), win, 1920, 1080, 100, fr.Mode.FP32_FAST)
        np.testing.assert_array_equal(np16(out[k]), one)
        ref = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, 1920, 1080,
                           100, 32)
        _check_fast_frame("julia", complex(cs[k]), win, 1920, 1080, 100, 32, one, ref,
                          f"bench frame {k}")
    del out
    torch.cuda.empty_cache()


def test_fast_mode_tolerance_cfg5_sampled(fr):
    cfg = W.configs()["cfg5"]
    win = cfg.window
    got = fr.mandelbrot_param_map(win, cfg.width, cfg.height, cfg.max_iter, fr.Mode.FP64_FAST)
    torch.cuda.synchronize()
    rng = np.random.default_rng(77)
    px, py = rng.integers(0, cfg.width, 3000), rng.integers(0, cfg.height, 3000)
    ref = oracle.pixels("mandelbrot", 0j, win.center, win.half_w, win.half_h, cfg.width,
                        cfg.height, cfg.max_iter, 64, px, py)
    g = sample16(got, py, px)
    bad = g != ref
    sens = _sensitivity("mandelbrot", 0j, win, cfg.width, cfg.height, cfg.max_iter, 64, n=3000)
    print(f"cfg5: fast-vs-strict {bad.mean():.3e}, 1-ulp sensitivity {sens:.3e}")
    assert bad.mean() <= max(1e-4, 4 * sens)
    if bad.any():
        ok, nl, nd, worst = _within_one_pixel_of_a_boundary(
            "mandelbrot", 0j, win, cfg.width, cfg.height, cfg.max_iter, 64, px[bad], py[bad],
            g[bad])
        print(f"cfg5: {nl} level-set, {nd} DE-checked, worst DE/2 {worst:.3f} px")
        assert ok
    del got
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ streams / launches
def test_side_stream_and_launch_count(fr):
    cfg = W.configs()["cfg1"]
    before = fr.launch_count()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a = fr.julia_render_ex(cfg.c, cfg.window, 64, 64, 100, fr.Mode.FP32_STRICT)
    s.synchronize()
    b = gpu_julia(fr, cfg.c, cfg.window, 64, 64, 100, fr.Mode.FP32_STRICT)
    np.testing.assert_array_equal(np16(a), b)
    # one launch per render for the static kernel; the refill path may add a pre-pass
    # and a continuation launch (FRACTAL_SCHED forced in the scheduler runs)
    assert 2 <= fr.launch_count() - before <= 6


def test_concurrent_host_threads_and_streams(fr):
    """Reentrancy (include/fractal.h "Async"): four host threads, each on its own CUDA
    stream, render heavy-tailed frames (P1 + P2 with their per-stream queue and survivor
    buffer), paths (SX) and refill / amortised frames at the same time, several rounds;
    every result equals the same render done alone on the default stream."""
    import threading
    c3 = -0.7269 + 0.1889j
    win = W.julia_window(640, 360)
    mwin = W.Window(-0.3 + 0.1j, 0.4, 0.225)
    cs = W.circle_path(24)
    jobs = [("twophase", lambda out: fr.julia_render_ex(c3, win, 640, 360, 1000,
                                                         fr.Mode.FP32_FAST, out=out)),
            ("twophase64", lambda out: fr.julia_render_ex(c3, win, 640, 360, 1000,
                                                           fr.Mode.FP64_FAST, out=out)),
            ("path", lambda out: fr.julia_render_path(cs, win, 640, 360, 100,
                                                      fr.Mode.FP32_FAST, out=out)),
            ("amort", lambda out: fr.mandelbrot_param_map(mwin, 640, 360, 2000,
                                                          fr.Mode.FP64_FAST, out=out))]
    shapes = {"path": (24, 360, 640)}
    ref = {}
    for name, fn in jobs:
        out = torch.empty(shapes.get(name, (360, 640)), dtype=torch.uint16, device="cuda")
        fn(out)
        torch.cuda.synchronize()
        ref[name] = np16(out)
    errors = []

    def worker(name, fn):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(4):
                    out = torch.empty(shapes.get(name, (360, 640)), dtype=torch.uint16,
                                      device="cuda")
                    fn(out)
                    st.synchronize()
                    if not np.array_equal(np16(out), ref[name]):
                        errors.append(name)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(f"{name}: {e!r}")

    threads = [threading.Thread(target=worker, args=j) for j in jobs]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_c_abi_demo_program(fr, tmp_path):
    """examples/c_abi_demo.c: a plain C program renders cfg4-path frames through
    julia_render_path_host (host output, no CUDA calls of its own); its file equals the
    oracle frame by frame, strict and fast."""
    import subprocess
    import sys as _sys
    _sys.path.insert(0, os.path.dirname(__file__))
    from test_abi import _build_c_demo
    exe = _build_c_demo(tmp_path)
    w, h, n = 96, 54, 6
    cs = W.circle_path(n)
    win = W.julia_window(w, h)
    for mode, fast in ((1, False), (0, True)):
        out = tmp_path / f"counts{mode}.bin"
        r = subprocess.run([str(exe), str(w), str(h), str(n), "100", str(mode), str(out)],
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        got = np.fromfile(out, dtype="<u2").reshape(n, h, w)
        for k in range(n):
            ref = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, w, h, 100,
                               32, fast=fast)
            np.testing.assert_array_equal(got[k], ref)


# ------------------------------------------------------------------ NEXT-2: cardioid path
def test_cardioid_path_frames_strict(fr):
    """The paper's own dynamic workload: Julia frames along the a = 3.9 cardioid
    with the shrinking-a sweep, strict fp32, equal to the oracle frame by frame."""
    cs = fr.cardioid_path(1300)[::20]  # 65 frames over two revolutions
    w, h = 320, 180
    win = W.julia_window(w, h)
    out = fr.julia_render_path(cs, win, w, h, 100, fr.Mode.FP32_STRICT)
    torch.cuda.synchronize()
    got = np16(out)
    for k in range(len(cs)):
        ref = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, w, h, 100, 32)
        np.testing.assert_array_equal(got[k], ref)


# ------------------------------------------------------------------ NEXT-3: other maps
@pytest.mark.parametrize("fn", ["z4", "z4_rational"])
@pytest.mark.parametrize("case", range(12))
def test_function_variants_bit_exact(fr, fn, case):
    """Figure 4 family (reading c-14): GPU == oracle bit for bit, both precisions,
    fuzzed windows, plus the Figure 4 parameter value."""
    c, win, w, h, mi = W.fuzz_cases(12, max_side=200, seed=44)[case]
    if case == 0:
        c, win, w, h, mi = W.FIG4_C, W.julia_window(256, 256, span_re=3.0), 256, 256, 100
    f = {"z4": fr.Function.Z4, "z4_rational": fr.Function.Z4_RATIONAL}[fn]
    for prec, mode in ((32, fr.Mode.FP32_STRICT), (64, fr.Mode.FP64_STRICT), (32, fr.Mode.FP32_FAST)):
        ref = oracle.julia_fn(fn, c, win.center, win.half_w, win.half_h, w, h, mi, prec)
        got = fr.julia_render_fn(f, c, win, w, h, mi, mode)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(np16(got), ref)


def test_path_uint8_counts(fr):
    """julia_render_path8: the same counts as uint8 (max_iter <= 255), fast and strict."""
    cs = W.circle_path(40)
    w, h = 96, 54
    win = W.julia_window(w, h)
    for mode in (fr.Mode.FP32_FAST, fr.Mode.FP32_STRICT):
        a = fr.julia_render_path(cs, win, w, h, 255, mode)
        b = fr.julia_render_path(cs, win, w, h, 255, mode,
                                 out=torch.empty((40, h, w), dtype=torch.uint8, device="cuda"))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(np16(a), b.cpu().numpy().astype(np.uint16))
    with pytest.raises(fr.FractalError):
        fr.julia_render_path(cs, win, w, h, 256, fr.Mode.FP32_FAST,
                             out=torch.empty((40, h, w), dtype=torch.uint8, device="cuda"))


# ------------------------------------------------------------------ write extents (canaries)
def _guarded(n, dtype, guard=256):
    """A buffer with `guard` canary elements on both sides; returns (full, view)."""
    full = torch.full((n + 2 * guard,), -1 if dtype == torch.int16 else 0xAB,
                      dtype=dtype, device="cuda")
    return full, full[guard:guard + n]


def _check_canaries(full, n, dtype, guard=256):
    a = full.cpu().numpy()
    fill = -1 if dtype == torch.int16 else 0xAB
    assert (a[:guard] == fill).all(), "write before the output"
    assert (a[guard + n:] == fill).all(), "write past the output"
    return a[guard:guard + n]


@pytest.mark.parametrize("size", [(37, 5), (65, 17), (1, 1), (100, 33)])
def test_outputs_written_exactly_in_bounds(fr, size):
    """Every kernel family writes every output element exactly within its buffer: counts,
    rgba, bands, paths (uint16 and uint8), map variants, standalone colorize.  (Stands in
    for compute-sanitizer, which is closed on this pool.)"""
    w, h = size
    win = W.julia_window(w, h)
    pal = W.palette("fire")
    # max_iter 50: S2 (fp32) / S (fp64); 300 and 1200: P1 + P2; the monotone Mandelbrot
    # window at 1200: kernel A; fast and strict modes
    cases = [(mi, kind, strict_m) for mi in (50, 300, 1200) for kind in ("julia", "mandelbrot")
             for strict_m in (False, True)] + [(1200, "mandel_mono", False),
                                               (1200, "mandel_mono", True)]
    for mi, kind, strict_m in cases:
        for bands in (fr.FULL_FRAME, fr.Bands(4, 3, 1)):
            rows = fr.band_local_rows(h, bands)
            fc, vc = _guarded(rows * w, torch.int16)
            fr_, vr = _guarded(rows * w * 4, torch.uint8)
            cnt = vc.view(torch.uint16)
            if kind == "julia":
                m = fr.Mode.FP32_STRICT if strict_m else fr.Mode.FP32_FAST
                fr.julia_render_ex(0.285 + 0.01j, win, w, h, mi, m, bands,
                                   out=cnt, palette=pal, out_rgba=vr)
            else:
                m = fr.Mode.FP64_STRICT if strict_m else fr.Mode.FP64_FAST
                mw = ((-0.5 + 0j, 1.5, 1.5 * h / w) if kind == "mandelbrot"
                      else (-0.3 + 0.1j, 0.4, 0.4 * h / w))  # |C| <= 1.989: kernel A
                fr.mandelbrot_param_map(mw, w, h, mi, m, bands, out=cnt, palette=pal,
                                        out_rgba=vr)
            torch.cuda.synchronize()
            body = _check_canaries(fc, rows * w, torch.int16)
            assert (body != -1).all()
            _check_canaries(fr_, rows * w * 4, torch.uint8)
    n = 3
    fc, vc = _guarded(n * h * w, torch.int16)
    fr.julia_render_path(W.circle_path(n), win, w, h, 100, fr.Mode.FP32_FAST, out=vc.view(torch.uint16))
    fb, vb = _guarded(n * h * w, torch.uint8)
    fr.julia_render_path(W.circle_path(n), win, w, h, 100, fr.Mode.FP32_FAST, out=vb)
    ff, vf = _guarded(h * w, torch.int16)
    fr.julia_render_fn(fr.Function.Z4_RATIONAL, W.FIG4_C, win, w, h, 100, fr.Mode.FP32_STRICT,
                       out=vf.view(torch.uint16))
    counts = torch.randint(0, 300, (h * w,), dtype=torch.int32).to(torch.int16).cuda().view(torch.uint16)
    fz, vz = _guarded(h * w * 4, torch.uint8)
    fr.colorize(counts, 299, pal, out_rgba=vz)
    torch.cuda.synchronize()
    assert (_check_canaries(fc, n * h * w, torch.int16) != -1).all()
    _check_canaries(fb, n * h * w, torch.uint8)
    assert (_check_canaries(ff, h * w, torch.int16) != -1).all()
    _check_canaries(fz, h * w * 4, torch.uint8)


def test_path_to_host_buffers(fr):
    """julia_render_path_host: the same counts as the device path, delivered to host
    memory (pinned and pageable, uint8 and uint16), across several staging chunks."""
    cs = W.circle_path(70)
    w, h = 1920, 1080
    win = W.julia_window(w, h)
    ref = np16(fr.julia_render_path(cs, win, w, h, 100, fr.Mode.FP32_FAST))
    pinned = torch.empty((70, h, w), dtype=torch.uint8, pin_memory=True)
    fr.julia_render_path_host(cs, win, w, h, 100, fr.Mode.FP32_FAST, out=pinned)
    np.testing.assert_array_equal(pinned.numpy().astype(np.uint16), ref)
    page16 = np.empty((70, h, w), dtype=np.uint16)
    fr.julia_render_path_host(cs, win, w, h, 100, fr.Mode.FP32_FAST, out=page16)
    np.testing.assert_array_equal(page16, ref)


def test_graph_capture_contract(fr):
    """fractal.h 'Memory': library caches are created outside graph capture.  A palette
    first seen inside a capture fails cleanly (FractalError, nothing launched); once used
    outside capture, the same coloured render captures and replays, and the replay equals
    an eager render."""
    cfg = W.configs()["cfg2"]
    w, h = 320, 180
    win = W.julia_window(w, h)
    fresh = (np.arange(4 * 7, dtype=np.uint8).reshape(7, 4) * 9 + 3, (1, 2, 3, 255))
    out = torch.empty((h, w), dtype=torch.uint16, device="cuda")
    rgba = torch.empty((h, w, 4), dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(fr.FractalError):
        with torch.cuda.graph(g, stream=side):
            fr.julia_render_ex(cfg.c, win, w, h, 100, fr.Mode.FP32_FAST, out=out,
                               palette=fresh, out_rgba=rgba)
    torch.cuda.synchronize()
    # eager first use creates the device copy; then capture works
    want_c, want_rgba = gpu_julia(fr, cfg.c, win, w, h, 100, fr.Mode.FP32_FAST, palette=fresh)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=side):
        fr.julia_render_ex(cfg.c, win, w, h, 100, fr.Mode.FP32_FAST, out=out, palette=fresh,
                           out_rgba=rgba)
    out.zero_()
    rgba.zero_()
    g2.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(np16(out), want_c)
    np.testing.assert_array_equal(rgba.cpu().numpy(), want_rgba)


def test_graph_replays_of_self_resetting_kernels(fr):
    """The queue of P1 + P2, kernel R's chunk counter and kernel A reset themselves at the
    end of each launch, so a CUDA graph of them replays correctly any number of times
    (include/fractal.h "Graphs").  And the round-1 review's use-after-free scenario: a
    graph captured with a small survivor buffer still replays correctly after a larger
    frame made the buffer grow on the same stream (outgrown buffers are kept alive)."""
    side = torch.cuda.Stream()
    c3 = -0.7269 + 0.1889j
    w, h = 480, 270
    win = W.julia_window(w, h)
    mwin = W.Window(-0.3 + 0.1j, 0.4, 0.225)
    pal = W.palette("classic")
    out1 = torch.empty((h, w), dtype=torch.uint16, device="cuda")
    rgba1 = torch.empty((h, w, 4), dtype=torch.uint8, device="cuda")
    out2 = torch.empty((h, w), dtype=torch.uint16, device="cuda")
    out3 = torch.empty((h, w), dtype=torch.uint16, device="cuda")

    def frame():
        fr.julia_render_ex(c3, win, w, h, 1000, fr.Mode.FP32_FAST, out=out1, palette=pal,
                           out_rgba=rgba1)                                    # P1 + P2
        fr.julia_render_ex(c3, win, w, h, 1000, fr.Mode.FP64_STRICT, out=out2)  # P1 + P2
        fr.mandelbrot_param_map(mwin, w, h, 2000, fr.Mode.FP32_FAST, out=out3)  # kernel A

    with torch.cuda.stream(side):
        frame()  # eager first use on this stream: workspaces, queue, palette copy
    torch.cuda.synchronize()
    want = [np16(out1), rgba1.cpu().numpy(), np16(out2), np16(out3)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        frame()
    # grow the survivor buffer of this stream with a larger eager frame
    with torch.cuda.stream(side):
        big = fr.julia_render_ex(c3, W.julia_window(1920, 1080), 1920, 1080, 1000,
                                 fr.Mode.FP32_FAST)
    torch.cuda.synchronize()
    del big
    for _ in range(12):
        for t in (out1, out2, out3):
            t.view(torch.int16).fill_(-1)
        rgba1.zero_()
        g.replay()
        torch.cuda.synchronize()
        got = [np16(out1), rgba1.cpu().numpy(), np16(out2), np16(out3)]
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a, b)
