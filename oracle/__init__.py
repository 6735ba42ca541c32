"""CPU oracle for the escape-time hot path of arXiv 1611.03079 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  It shares no code with the
CUDA path in ``paper_1611_03079_b200/`` and never imports it.

The arithmetic lives in ``escape_oracle.c`` (plain scalar C, built with
``-ffp-contract=off``, no FTZ/DAZ), loaded here with ctypes.  ``numpy_ref.py`` is a
second, independent numpy implementation used to cross-check it on small grids.

Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "escape_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-pthread", "-Wall", "-Werror"]
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (contraction off).  Returns the path."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = ctypes.CDLL(build())
        i64, i32, f64, f32 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_float
        vp = ctypes.c_void_p
        lib.oracle_fp_env_ok.restype = i32
        lib.oracle_mul_add_f64.argtypes = [f64, f64, f64]
        lib.oracle_mul_add_f64.restype = f64
        lib.oracle_mul_add_f32.argtypes = [f32, f32, f32]
        lib.oracle_mul_add_f32.restype = f32
        lib.oracle_pixel_re.argtypes = [f64, f64, i64, i64]
        lib.oracle_pixel_re.restype = f64
        lib.oracle_pixel_im.argtypes = [f64, f64, i64, i64]
        lib.oracle_pixel_im.restype = f64
        lib.oracle_escape_f32.argtypes = [f32, f32, f32, f32, i32]
        lib.oracle_escape_f32.restype = i32
        lib.oracle_escape_f64.argtypes = [f64, f64, f64, f64, i32]
        lib.oracle_escape_f64.restype = i32
        lib.oracle_julia.argtypes = [f64, f64, f64, f64, f64, f64, i64, i64, i32, i32, vp, i32]
        lib.oracle_julia.restype = i32
        lib.oracle_mandel.argtypes = [f64, f64, f64, f64, i64, i64, i32, i32, vp, i32]
        lib.oracle_mandel.restype = i32
        lib.oracle_pixels.argtypes = [i32, f64, f64, f64, f64, f64, f64, i64, i64, i32, i32,
                                      vp, vp, i64, vp, i32]
        lib.oracle_pixels.restype = i32
        lib.oracle_colorize.argtypes = [vp, i64, i32, vp, i32, vp, vp]
        lib.oracle_colorize.restype = i32
        lib.oracle_cardioid_point.argtypes = [f64, f64, ctypes.POINTER(f64), ctypes.POINTER(f64)]
        lib.oracle_cardioid_point.restype = None
        lib.oracle_distance_estimate.argtypes = [i32, f64, f64, f64, f64, ctypes.c_long]
        lib.oracle_distance_estimate.restype = f64
        lib.oracle_distance_pixels.argtypes = [i32, f64, f64, f64, f64, f64, f64, i64, i64, vp, vp,
                                               i64, ctypes.c_long, vp]
        lib.oracle_distance_pixels.restype = i32
        lib.oracle_pixels_nudged.argtypes = [i32, f64, f64, f64, f64, f64, f64, i64, i64, i32, i32,
                                             vp, vp, i64, i32, vp, i32]
        lib.oracle_pixels_nudged.restype = i32
        lib.oracle_escape_fn_f32.argtypes = [i32, f32, f32, f32, f32, i32]
        lib.oracle_escape_fn_f32.restype = i32
        lib.oracle_escape_fn_f64.argtypes = [i32, f64, f64, f64, f64, i32]
        lib.oracle_escape_fn_f64.restype = i32
        lib.oracle_julia_fn.argtypes = [i32, f64, f64, f64, f64, f64, f64, i64, i64, i32, i32, vp]
        lib.oracle_julia_fn.restype = i32
        lib.oracle_escape_fma_f32.argtypes = [f32, f32, f32, f32, i32]
        lib.oracle_escape_fma_f32.restype = i32
        lib.oracle_escape_fma_f64.argtypes = [f64, f64, f64, f64, i32]
        lib.oracle_escape_fma_f64.restype = i32
        lib.oracle_escape_fma_unscaled_f32.argtypes = [f32, f32, f32, f32, i32]
        lib.oracle_escape_fma_unscaled_f32.restype = i32
        lib.oracle_escape_fma_unscaled_f64.argtypes = [f64, f64, f64, f64, i32]
        lib.oracle_escape_fma_unscaled_f64.restype = i32
        lib.oracle_frame_fma.argtypes = [i32, f64, f64, f64, f64, f64, f64, i64, i64, i32, i32,
                                         vp, i32]
        lib.oracle_frame_fma.restype = i32
        lib.oracle_pixels_fma.argtypes = [i32, f64, f64, f64, f64, f64, f64, i64, i64, i32, i32,
                                          vp, vp, i64, vp, i32]
        lib.oracle_pixels_fma.restype = i32
        _lib = lib
        return lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _prec(precision) -> int:
    p = {32: 32, 64: 64, "f32": 32, "f64": 64, "fp32": 32, "fp64": 64}.get(precision)
    if p is None:
        raise ValueError(f"precision must be 32 or 64, got {precision!r}")
    return p


# --------------------------------------------------------------------------- scalar API
def fp_env_ok() -> bool:
    """MXCSR FTZ and DAZ both clear (denormals preserved)."""
    return bool(_load().oracle_fp_env_ok())


def mul_add(a: float, b: float, c: float, precision=64) -> float:
    """Contraction canary: a*b+c as two separately rounded ops."""
    lib = _load()
    return (lib.oracle_mul_add_f32 if _prec(precision) == 32 else lib.oracle_mul_add_f64)(a, b, c)


def pixel_to_complex(center: complex, half_w: float, half_h: float, width: int, height: int,
                     px: int, py: int) -> complex:
    """Region-covering map, pixel centre (reading c-3), in binary64."""
    lib = _load()
    return complex(lib.oracle_pixel_re(center.real, half_w, width, px),
                   lib.oracle_pixel_im(center.imag, half_h, height, py))


def escape_time(z0: complex, c: complex, max_iter: int = 100, precision=64,
                fast: bool = False) -> int:
    """Smallest n in [0, max_iter-1] with |Z_n|^2 > 4, else max_iter.
    For precision 32 the inputs are rounded to binary32 first.  fast=True iterates the
    FMA-contracted sequence that defines the *_FAST modes (reading c-10)."""
    lib = _load()
    if fast:
        f = lib.oracle_escape_fma_f32 if _prec(precision) == 32 else lib.oracle_escape_fma_f64
    else:
        f = lib.oracle_escape_f32 if _prec(precision) == 32 else lib.oracle_escape_f64
    return int(f(z0.real, z0.imag, c.real, c.imag, int(max_iter)))


def escape_time_fast_unscaled(z0: complex, c: complex, max_iter: int = 100,
                              precision=64) -> int:
    """The unscaled FMA contraction of the strict iteration (yy = y*y; m = fma(x,x,yy);
    t = fma(x,x,-yy); y = fma(2x,y,ci); x = t + cr): equal to the FAST (doubled-state)
    sequence unless an unscaled product is subnormal.  For the equivalence pin only."""
    lib = _load()
    f = (lib.oracle_escape_fma_unscaled_f32 if _prec(precision) == 32
         else lib.oracle_escape_fma_unscaled_f64)
    return int(f(z0.real, z0.imag, c.real, c.imag, int(max_iter)))


def cardioid_point(t: float, a: float) -> complex:
    """f(t) = ((2cos t - cos 2t)/a, (2 sin t - sin 2t)/a)."""
    re, im = ctypes.c_double(), ctypes.c_double()
    _load().oracle_cardioid_point(float(t), float(a), ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


# --------------------------------------------------------------------------- grid API
def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def julia(c: complex, center: complex, half_w: float, half_h: float, width: int, height: int,
          max_iter: int = 100, precision=32, threads: int | None = None,
          fast: bool = False) -> np.ndarray:
    """Julia frame of Z^2 + C: uint16 counts [height, width], row 0 = top."""
    out = np.empty((height, width), dtype=np.uint16)
    if fast:
        return _frame_fma(0, c, center, half_w, half_h, width, height, max_iter, precision,
                          threads, out)
    rc = _load().oracle_julia(c.real, c.imag, center.real, center.imag, half_w, half_h, width,
                              height, max_iter, _prec(precision), _ptr(out),
                              threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_julia: invalid arguments")
    return out


def mandelbrot(center: complex, half_w: float, half_h: float, width: int, height: int,
               max_iter: int = 100, precision=64, threads: int | None = None,
               fast: bool = False) -> np.ndarray:
    """Mandelbrot parameter map: C from the pixel, Z_0 = 0."""
    out = np.empty((height, width), dtype=np.uint16)
    if fast:
        return _frame_fma(1, 0j, center, half_w, half_h, width, height, max_iter, precision,
                          threads, out)
    rc = _load().oracle_mandel(center.real, center.imag, half_w, half_h, width, height, max_iter,
                               _prec(precision), _ptr(out), threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_mandel: invalid arguments")
    return out


def pixels(kind: str, c: complex, center: complex, half_w: float, half_h: float, width: int,
           height: int, max_iter: int, precision, px, py, threads: int | None = None,
           fast: bool = False) -> np.ndarray:
    """Counts of selected pixels (px[i], py[i]) of a width x height grid; kind 'julia' or
    'mandelbrot'.  Lets parity run at full BASELINE sizes on a sample."""
    px = np.ascontiguousarray(px, dtype=np.int64)
    py = np.ascontiguousarray(py, dtype=np.int64)
    if px.shape != py.shape:
        raise ValueError("px/py shape mismatch")
    out = np.empty(px.shape, dtype=np.uint16)
    mandel = {"julia": 0, "mandelbrot": 1}[kind]
    lib = _load()
    fn = lib.oracle_pixels_fma if fast else lib.oracle_pixels
    rc = fn(mandel, c.real, c.imag, center.real, center.imag, half_w, half_h,
            width, height, max_iter, _prec(precision), _ptr(px), _ptr(py), px.size, _ptr(out),
            threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_pixels: invalid arguments")
    return out


def _frame_fma(mandel, c, center, half_w, half_h, width, height, max_iter, precision, threads,
               out):
    rc = _load().oracle_frame_fma(mandel, c.real, c.imag, center.real, center.imag, half_w,
                                  half_h, width, height, max_iter, _prec(precision), _ptr(out),
                                  threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_frame_fma: invalid arguments")
    return out


def colorize(counts: np.ndarray, max_iter: int, palette: np.ndarray, interior) -> np.ndarray:
    """Colour levels: count==max_iter -> interior, else palette[count % n].
    palette: uint8 [n, 4] RGBA.  Returns uint8 [..., 4]."""
    counts = np.ascontiguousarray(counts, dtype=np.uint16)
    pal = np.ascontiguousarray(palette, dtype=np.uint8).reshape(-1, 4)
    inter = np.ascontiguousarray(np.asarray(interior, dtype=np.uint8).reshape(4))
    out = np.empty(counts.shape + (4,), dtype=np.uint8)
    rc = _load().oracle_colorize(_ptr(counts), counts.size, max_iter, _ptr(pal), pal.shape[0],
                                 _ptr(inter), _ptr(out))
    if rc != 0:
        raise ValueError("oracle_colorize: invalid arguments")
    return out


# --------------------------------------------------------------------------- fast-mode tools
def distance_estimate(kind: str, z0: complex, c: complex, max_iter: int = 1_000_000) -> float:
    """Exterior distance estimate |Z| ln|Z| / |Z'| (binary64, bailout 1e10); 0 if the
    orbit does not escape (reading c-10).  kind 'julia' (derivative in Z_0)
    or 'mandelbrot' (derivative in c, Z_0 = 0)."""
    m = {"julia": 0, "mandelbrot": 1}[kind]
    return float(_load().oracle_distance_estimate(m, z0.real, z0.imag, c.real, c.imag, max_iter))


def distance_pixels(kind: str, c: complex, center: complex, half_w: float, half_h: float,
                    width: int, height: int, px, py, max_iter: int = 1_000_000) -> np.ndarray:
    px = np.ascontiguousarray(px, dtype=np.int64)
    py = np.ascontiguousarray(py, dtype=np.int64)
    out = np.empty(px.shape, dtype=np.float64)
    m = {"julia": 0, "mandelbrot": 1}[kind]
    rc = _load().oracle_distance_pixels(m, c.real, c.imag, center.real, center.imag, half_w,
                                        half_h, width, height, _ptr(px), _ptr(py), px.size,
                                        max_iter, _ptr(out))
    if rc != 0:
        raise ValueError("oracle_distance_pixels: invalid arguments")
    return out


def pixels_nudged(kind: str, c: complex, center: complex, half_w: float, half_h: float,
                  width: int, height: int, max_iter: int, precision, px, py,
                  nudge: int = 1, threads: int | None = None) -> np.ndarray:
    """Strict counts with the start value's real part moved by `nudge` ulps."""
    px = np.ascontiguousarray(px, dtype=np.int64)
    py = np.ascontiguousarray(py, dtype=np.int64)
    out = np.empty(px.shape, dtype=np.uint16)
    m = {"julia": 0, "mandelbrot": 1}[kind]
    rc = _load().oracle_pixels_nudged(m, c.real, c.imag, center.real, center.imag, half_w, half_h,
                                      width, height, max_iter, _prec(precision), _ptr(px),
                                      _ptr(py), px.size, nudge, _ptr(out),
                                      threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_pixels_nudged: invalid arguments")
    return out


# --------------------------------------------------------------------------- NEXT-3 maps
FUNCTIONS = {"z2": 0, "z4": 1, "z4_rational": 2}


def escape_time_fn(fn: str, z0: complex, c: complex, max_iter: int = 100, precision=64) -> int:
    """Escape time under z^2+c ('z2'), z^4+c ('z4') or z^4+(z^2+1)/(z^2-1)+c
    ('z4_rational'; pole -> +inf), reading c-14."""
    lib = _load()
    f = lib.oracle_escape_fn_f32 if _prec(precision) == 32 else lib.oracle_escape_fn_f64
    return int(f(FUNCTIONS[fn], z0.real, z0.imag, c.real, c.imag, int(max_iter)))


def julia_fn(fn: str, c: complex, center: complex, half_w: float, half_h: float, width: int,
             height: int, max_iter: int = 100, precision=32) -> np.ndarray:
    out = np.empty((height, width), dtype=np.uint16)
    rc = _load().oracle_julia_fn(FUNCTIONS[fn], c.real, c.imag, center.real, center.imag, half_w,
                                 half_h, width, height, max_iter, _prec(precision), _ptr(out))
    if rc != 0:
        raise ValueError("oracle_julia_fn: invalid arguments")
    return out
