"""GPU parity of the FAST modes against the FAST oracle, bit for bit.

FP32_FAST / FP64_FAST are defined (DESIGN.md §5 "State representation", reading c-10)
as the escape-time iteration carried out with one FMA-contracted operation sequence;
oracle/escape_oracle.c's oracle_escape_fma_* writes that sequence (doubled state,
C99 fmaf/fma) plainly, independent of the kernels.
Because both are the same sequence of correctly rounded operations, the counts must
agree exactly -- a stronger check than the tolerance test_gpu_parity.py applies
against the strict oracle, which stays as the statement of how far FAST is from the
exact-IEEE reading.
"""
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
    v = t.view(torch.int16)[torch.as_tensor(py, device=t.device),
                            torch.as_tensor(px, device=t.device)]
    return v.cpu().numpy().view(np.uint16)


def fast(prec, fr):
    return fr.Mode.FP32_FAST if prec == 32 else fr.Mode.FP64_FAST


def _sentinel(w, h, mi):
    s = (mi + 1) & 0xFFFF
    return torch.full((h, w), s - 65536 if s >= 32768 else s, dtype=torch.int16,
                      device="cuda").view(torch.uint16)


def gpu_julia(fr, c, win, w, h, mi, mode, palette=None):
    out = _sentinel(w, h, mi)
    r = fr.julia_render_ex(c, win, w, h, mi, mode, out=out, palette=palette)
    torch.cuda.synchronize()
    if palette is not None:
        return np16(r[0]), r[1].cpu().numpy()
    return np16(r)


def gpu_mandel(fr, win, w, h, mi, mode):
    r = fr.mandelbrot_param_map(win, w, h, mi, mode, out=_sentinel(w, h, mi))
    torch.cuda.synchronize()
    return np16(r)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_fast_configs_full_frame(fr, name, prec):
    cfg = W.configs()[name]
    win = cfg.window
    ref = oracle.julia(cfg.c, win.center, win.half_w, win.half_h, cfg.width, cfg.height,
                       cfg.max_iter, prec, fast=True)
    if cfg.colorize:
        pal = W.palette("classic")
        got, rgba = gpu_julia(fr, cfg.c, win, cfg.width, cfg.height, cfg.max_iter,
                              fast(prec, fr), palette=pal)
        np.testing.assert_array_equal(rgba, oracle.colorize(ref, cfg.max_iter, *pal))
    else:
        got = gpu_julia(fr, cfg.c, win, cfg.width, cfg.height, cfg.max_iter, fast(prec, fr))
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("mi", [100, 256, 1000, 3000])
def test_fast_mandelbrot_full_frame(fr, prec, mi):
    """max_iter 100 -> static tiles, 256 -> two-phase, >= 1000 on a window inside
    |C| <= 1.989 -> kernel A (amortised test + replay)."""
    win = W.mandel_window(640, 480, span_re=2.4, center=-0.5 + 0j)  # |C| <= 1.92
    ref = oracle.mandelbrot(win.center, win.half_w, win.half_h, 640, 480, mi, prec, fast=True)
    np.testing.assert_array_equal(gpu_mandel(fr, win, 640, 480, mi, fast(prec, fr)), ref)


@pytest.mark.parametrize("case", range(96))
def test_fast_fuzz(fr, case):
    c, win, w, h, mi = W.fuzz_cases(96, max_side=300)[case]
    for prec in (32, 64):
        ref = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec, fast=True)
        np.testing.assert_array_equal(gpu_julia(fr, c, win, w, h, mi, fast(prec, fr)), ref)
        ref = oracle.mandelbrot(win.center, win.half_w, win.half_h, w, h, mi, prec, fast=True)
        np.testing.assert_array_equal(gpu_mandel(fr, win, w, h, mi, fast(prec, fr)), ref)


@pytest.mark.parametrize("case", range(24))
def test_fast_fuzz_large(fr, case):
    c, win, w, h, _ = W.fuzz_cases(24, max_side=600, seed=W.FUZZ_SEED + 2)[case]
    mi = (100, 300, 1000)[case % 3]
    for prec in (32, 64):
        ref = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec, fast=True)
        np.testing.assert_array_equal(gpu_julia(fr, c, win, w, h, mi, fast(prec, fr)), ref)


def test_fast_bench_launch_frames(fr):
    """The launch bench.py times (512 frames of the |C| = 0.7885 circle, 1080p,
    max_iter 100, FP32_FAST, one julia_render_path call): sampled whole frames equal the
    FAST oracle."""
    cs = W.circle_path(512, 0.7885)
    win = W.julia_window(1920, 1080)
    out = torch.full((512, 1080, 1920), 101, dtype=torch.int16, device="cuda").view(torch.uint16)
    fr.julia_render_path(cs, win, 1920, 1080, 100, fr.Mode.FP32_FAST, out=out)
    torch.cuda.synchronize()
    for k in (0, 1, 127, 256, 383, 511):
        ref = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, 1920, 1080, 100,
                           32, fast=True)
        np.testing.assert_array_equal(np16(out[k]), ref)
    del out
    torch.cuda.empty_cache()


def test_fast_path_fp64_and_tail_block(fr):
    cs = W.circle_path(300)
    w, h = 96, 54
    win = W.julia_window(w, h)
    for mode, prec, mi in ((fr.Mode.FP64_FAST, 64, 100), (fr.Mode.FP32_FAST, 32, 99),
                           (fr.Mode.FP32_FAST, 32, 1)):
        out = fr.julia_render_path(cs, win, w, h, mi, mode)
        torch.cuda.synchronize()
        for k in (0, 77, 150, 299):
            ref = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, w, h, mi,
                               prec, fast=True)
            np.testing.assert_array_equal(np16(out[k]), ref)


def test_fast_cfg5_sampled(fr):
    """cfg5 at full size (16384^2, max_iter 10000, FP64_FAST): 3000 sampled pixels."""
    cfg = W.configs()["cfg5"]
    win = cfg.window
    got = fr.mandelbrot_param_map(win, cfg.width, cfg.height, cfg.max_iter, fr.Mode.FP64_FAST)
    torch.cuda.synchronize()
    rng = np.random.default_rng(78)
    px, py = rng.integers(0, cfg.width, 3000), rng.integers(0, cfg.height, 3000)
    ref = oracle.pixels("mandelbrot", 0j, win.center, win.half_w, win.half_h, cfg.width,
                        cfg.height, cfg.max_iter, 64, px, py, fast=True)
    np.testing.assert_array_equal(sample16(got, py, px), ref)
    del got
    torch.cuda.empty_cache()


NONMONO_C = (-2 + 0j, -2.1 + 0j, 2j, -5 + 0j, 3 + 1j, 1.995 + 0j, -1.4 - 1.4j)


@pytest.mark.parametrize("c", NONMONO_C)
@pytest.mark.parametrize("mi", [100, 300, 1000])
def test_fast_nonmonotone_julia(fr, c, mi):
    """|C| > 1.989 (no escape monotonicity): FAST counts equal the FAST oracle whatever
    kernel the host routes to (the amortised ones must not be used here)."""
    w, h = 241, 161
    win = W.Window(0j, 2.6, 2.6 * h / w)
    for prec in (32, 64):
        ref = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec, fast=True)
        np.testing.assert_array_equal(gpu_julia(fr, c, win, w, h, mi, fast(prec, fr)), ref)


@pytest.mark.parametrize("prec", [32, 64])
def test_fast_nonmonotone_mandelbrot_window(fr, prec):
    """A Mandelbrot window reaching |c| = 2.6 (corners outside the monotone bound)."""
    win = W.Window(-0.3 + 0.1j, 2.3, 1.4)
    for mi in (100, 1000):
        ref = oracle.mandelbrot(win.center, win.half_w, win.half_h, 301, 183, mi, prec, fast=True)
        np.testing.assert_array_equal(gpu_mandel(fr, win, 301, 183, mi, fast(prec, fr)), ref)


@pytest.mark.parametrize("w,h", [(37, 5), (48, 9), (65, 17), (130, 7), (1, 1)])
@pytest.mark.parametrize("offset", [0, 1])
def test_fast_path_kernel_sx_layouts(fr, w, h, offset):
    """Kernel SX (FP32_FAST C-paths: x-adjacent pixel pairs, 4-byte count stores and
    8-byte RGBA stores when the pair is whole and aligned): odd widths, an output pointer
    one element off alignment (scalar stores), uint16 and uint8 counts, fused colour --
    every frame equal to the FAST oracle, nothing written outside the buffers."""
    cs = W.circle_path(37)
    win = W.julia_window(w, h)
    pal = W.palette("fire")
    n = len(cs)
    g = 64
    base16 = torch.full((n * h * w + 2 * g + offset,), -1, dtype=torch.int16, device="cuda")
    out16 = base16[g + offset:g + offset + n * h * w].view(torch.uint16).view(n, h, w)
    base8 = torch.full((n * h * w + 2 * g + offset,), 0xAB, dtype=torch.uint8, device="cuda")
    out8 = base8[g + offset:g + offset + n * h * w].view(n, h, w)
    baser = torch.full((4 * (n * h * w + 2 * g + offset),), 0x5A, dtype=torch.uint8,
                       device="cuda")
    rgba = baser[4 * (g + offset):4 * (g + offset + n * h * w)].view(n, h, w, 4)
    fr.julia_render_path(cs, win, w, h, 100, fr.Mode.FP32_FAST, out=out16, palette=pal,
                         out_rgba=rgba)
    fr.julia_render_path(cs, win, w, h, 100, fr.Mode.FP32_FAST, out=out8)
    torch.cuda.synchronize()
    a16 = base16.cpu().numpy()
    assert (a16[:g + offset] == -1).all() and (a16[g + offset + n * h * w:] == -1).all()
    a8 = base8.cpu().numpy()
    assert (a8[:g + offset] == 0xAB).all() and (a8[g + offset + n * h * w:] == 0xAB).all()
    ar = baser.cpu().numpy()
    assert (ar[:4 * (g + offset)] == 0x5A).all() and (ar[4 * (g + offset + n * h * w):] == 0x5A).all()
    got16, got8, gotr = np16(out16), out8.cpu().numpy(), rgba.cpu().numpy()
    for k in range(n):
        ref = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, w, h, 100, 32,
                           fast=True)
        np.testing.assert_array_equal(got16[k], ref)
        np.testing.assert_array_equal(got8[k], ref.astype(np.uint8))
        np.testing.assert_array_equal(gotr[k], oracle.colorize(ref, 100, *pal))


def test_fast_cfg4_all_frames(fr):
    """cfg4 in FP32_FAST at full size, ALL 4096 frames (kernel SX, the bench kernel)
    against the FAST oracle, frame by frame."""
    from concurrent.futures import ThreadPoolExecutor
    cfg = W.configs()["cfg4"]
    cs = W.circle_path(cfg.n_frames)
    win = cfg.window
    out = fr.julia_render_path(cs, win, cfg.width, cfg.height, cfg.max_iter, fr.Mode.FP32_FAST)
    torch.cuda.synchronize()

    def ref(k):
        return oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, cfg.width,
                            cfg.height, cfg.max_iter, 32, threads=2, fast=True)

    bad = []
    with ThreadPoolExecutor(max(1, oracle.default_threads() // 2)) as ex:
        for k0 in range(0, cfg.n_frames, 64):
            refs = list(ex.map(ref, range(k0, min(k0 + 64, cfg.n_frames))))
            got = out[k0:k0 + len(refs)].view(torch.int16).cpu().numpy().view(np.uint16)
            bad += [k0 + i for i, r in enumerate(refs) if not np.array_equal(got[i], r)]
    assert not bad, f"{len(bad)} frames differ, first {bad[:8]}"
    del out
    torch.cuda.empty_cache()
