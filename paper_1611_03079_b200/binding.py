"""Thin Python binding over libfractal (include/fractal.h): argument marshalling only.

Every step of the hot path runs inside libfractal's sm_100a kernels; torch supplies
device memory (tensors) and streams.  There is no CPU fallback: if libfractal.so is
missing or a call fails, a FractalError is raised.

Names follow the C ABI: julia_render, julia_render_ex, julia_render_path,
mandelbrot_param_map, colorize (P:31, P:47, P:53 of the paper).
"""
from __future__ import annotations

import ctypes
import enum
import os
import threading
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libfractal.so")
_lock = threading.Lock()
_lib = None


class FractalError(RuntimeError):
    pass


class Mode(enum.IntEnum):
    FP32_FAST = 0
    FP32_STRICT = 1
    FP64_FAST = 2
    FP64_STRICT = 3


class Function(enum.IntEnum):
    """Iteration maps (NEXT-3; Figure 4, reading c-14)."""
    Z2 = 0
    Z4 = 1
    Z4_RATIONAL = 2


class _Complex(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class _Window(ctypes.Structure):
    _fields_ = [("center_re", ctypes.c_double), ("center_im", ctypes.c_double),
                ("half_w", ctypes.c_double), ("half_h", ctypes.c_double)]


class _Palette(ctypes.Structure):
    _fields_ = [("rgba", ctypes.c_void_p), ("n", ctypes.c_int32),
                ("interior", ctypes.c_uint8 * 4)]


class _Bands(ctypes.Structure):
    _fields_ = [("band_rows", ctypes.c_int32), ("n_ranks", ctypes.c_int32),
                ("rank", ctypes.c_int32)]


@dataclass(frozen=True)
class Bands:
    """Cyclic row bands: global band b -> rank b % n_ranks (band_rows 0 = whole frame)."""
    band_rows: int = 0
    n_ranks: int = 1
    rank: int = 0

    def _c(self):
        return _Bands(self.band_rows, self.n_ranks, self.rank)


FULL_FRAME = Bands()
STATUS = {0: "FR_OK", 1: "FR_ERR_INVALID_ARG", 2: "FR_ERR_TOO_LARGE", 3: "FR_ERR_UNSUPPORTED",
          4: "FR_ERR_CUDA"}

# Functions declared in include/fractal.h (checked by tests/test_abi.py).
EXPORTS = ("julia_render", "julia_render_ex", "julia_render_path", "mandelbrot_param_map",
           "julia_render_path8", "julia_render_path_host", "colorize", "julia_render_fn", "fr_cardioid_path", "fr_band_local_rows", "fr_band_global_row", "fr_status_str",
           "fr_last_cuda_error", "fr_launch_count", "fr_version", "fr_debug_refill_trace")


def load():
    """dlopen libfractal.so (in-tree).  Raises FractalError if it is not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = LIB_PATH
        alt = os.environ.get("FRACTAL_LIB")  # diagnostic: a build.build_variant library
        if alt:
            alt = os.path.realpath(alt)
            if os.path.dirname(alt) != os.path.join(os.path.dirname(LIB_PATH), "variants"):
                raise FractalError(f"FRACTAL_LIB must name a library under variants/: {alt}")
            path = alt
        if not os.path.exists(path):
            raise FractalError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; "
                               "g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        st, vp, i32, i64 = ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        P = ctypes.POINTER
        lib.julia_render.argtypes = [_Complex, _Window, i32, i32, i32, vp, vp]
        lib.julia_render_ex.argtypes = [_Complex, _Window, i32, i32, i32, st, _Bands, vp,
                                        P(_Palette), vp, vp]
        lib.julia_render_path.argtypes = [vp, i32, _Window, i32, i32, i32, st, vp, P(_Palette),
                                          vp, vp]
        lib.julia_render_path8.argtypes = [vp, i32, _Window, i32, i32, i32, st, vp, P(_Palette),
                                           vp, vp]
        lib.julia_render_path8.restype = st
        lib.julia_render_path_host.argtypes = [vp, i32, _Window, i32, i32, i32, st, i32, vp, vp]
        lib.julia_render_path_host.restype = st
        lib.mandelbrot_param_map.argtypes = [_Window, i32, i32, i32, st, _Bands, vp, P(_Palette),
                                             vp, vp]
        lib.colorize.argtypes = [vp, i64, i32, P(_Palette), vp, vp]
        lib.julia_render_fn.argtypes = [st, _Complex, _Window, i32, i32, i32, st, vp, P(_Palette),
                                        vp, vp]
        lib.julia_render_fn.restype = st
        for f in ("julia_render", "julia_render_ex", "julia_render_path", "mandelbrot_param_map",
                  "colorize"):
            getattr(lib, f).restype = st
        f64 = ctypes.c_double
        lib.fr_cardioid_path.argtypes = [f64, f64, f64, f64, f64, i32, vp]
        lib.fr_cardioid_path.restype = st
        lib.fr_band_local_rows.argtypes = [i32, _Bands]
        lib.fr_band_local_rows.restype = i64
        lib.fr_band_global_row.argtypes = [i32, _Bands, i64]
        lib.fr_band_global_row.restype = i64
        lib.fr_status_str.argtypes = [st]
        lib.fr_status_str.restype = ctypes.c_char_p
        lib.fr_last_cuda_error.restype = i32
        lib.fr_launch_count.restype = ctypes.c_uint64
        lib.fr_version.restype = ctypes.c_char_p
        lib.fr_debug_refill_trace.argtypes = [vp]
        lib.fr_debug_refill_trace.restype = st
        _lib = lib
        return lib


# --------------------------------------------------------------------------- helpers
def _check(rc: int, what: str):
    if rc != 0:
        lib = load()
        msg = lib.fr_status_str(rc).decode()
        if rc == 4:
            msg += f" (cudaError {lib.fr_last_cuda_error()})"
        raise FractalError(f"{what}: {msg}")


def _window(win) -> _Window:
    if hasattr(win, "center"):
        c = complex(win.center)
        return _Window(c.real, c.imag, float(win.half_w), float(win.half_h))
    center, half_w, half_h = win
    c = complex(center)
    return _Window(c.real, c.imag, float(half_w), float(half_h))


def _stream(stream):
    if stream is None:
        import torch
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:  # no Stream object per call (host overhead of small frames)
            return ctypes.c_void_p(raw(torch.cuda.current_device()))
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _dev_ptr(t, dtype_name: str, numel: int, what: str):
    import torch
    want = {"uint16": torch.uint16, "uint8": torch.uint8}[dtype_name]
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise FractalError(f"{what} must be a CUDA tensor")
    if t.dtype != want:
        raise FractalError(f"{what} must have dtype {want}, got {t.dtype}")
    if not t.is_contiguous():
        raise FractalError(f"{what} must be contiguous")
    if t.numel() < numel:
        raise FractalError(f"{what} holds {t.numel()} elements, needs {numel}")
    return ctypes.c_void_p(t.data_ptr())


_PAL_CACHE = {}


def _pal(palette):
    """Host palette struct, cached by the palette's CONTENT (entries and interior bytes),
    so a palette edited in place is never served stale."""
    entries, interior = palette
    ent = np.ascontiguousarray(np.asarray(entries, dtype=np.uint8).reshape(-1, 4))
    inter = np.ascontiguousarray(np.asarray(interior, dtype=np.uint8).reshape(4))
    key = ent.tobytes() + inter.tobytes()
    hit = _PAL_CACHE.get(key)
    if hit is not None:
        return hit
    h = _PalHolder(ent, inter)
    if len(_PAL_CACHE) > 64:
        _PAL_CACHE.clear()
    _PAL_CACHE[key] = h
    return h


class _PalHolder:
    """Keeps the host palette buffer alive for the duration of a call."""

    def __init__(self, ent, inter):
        ent = ent.copy()  # owned: the caller may edit its arrays after the call
        self.buf = ent
        self.c = _Palette(ent.ctypes.data, ent.shape[0], (ctypes.c_uint8 * 4)(*inter.tolist()))


def cardioid_path(n: int, t0: float = 0.0, a0: float = 3.9, dt: float = 2 * np.pi / 600,
                  da_per_rev: float = 0.05, a_floor: float = 3.5) -> np.ndarray:
    """The paper's cardioid C-path with the shrinking-a sweep: complex128 [n]
    (host; feed it to julia_render_path).  Defaults: SPEC S:321 (600 frames per
    revolution, a from 3.9 down by 0.05 per revolution to 3.5)."""
    out = np.empty(max(n, 0), dtype=np.complex128)
    rc = load().fr_cardioid_path(float(t0), float(a0), float(dt), float(da_per_rev),
                                 float(a_floor), int(n), ctypes.c_void_p(out.ctypes.data))
    _check(rc, "fr_cardioid_path")
    return out


def band_local_rows(height: int, bands: Bands = FULL_FRAME) -> int:
    r = load().fr_band_local_rows(int(height), bands._c())
    if r < 0:
        raise FractalError(f"invalid bands {bands} for height {height}")
    return int(r)


def band_global_row(height: int, bands: Bands, local_row: int) -> int:
    return int(load().fr_band_global_row(int(height), bands._c(), int(local_row)))


def launch_count() -> int:
    return int(load().fr_launch_count())


def version() -> str:
    return load().fr_version().decode()


# --------------------------------------------------------------------------- API
def julia_render(c: complex, win, width: int, height: int, max_iter: int = 100, out=None,
                 stream=None):
    """Julia frame, FP32 fast, full frame -> uint16 [height, width] on the GPU."""
    import torch
    if out is None:
        out = torch.empty((height, width), dtype=torch.uint16, device="cuda")
    p = _dev_ptr(out, "uint16", width * height, "out")
    rc = load().julia_render(_Complex(complex(c).real, complex(c).imag), _window(win), width,
                             height, max_iter, p, _stream(stream))
    _check(rc, "julia_render")
    return out


def julia_render_ex(c: complex, win, width: int, height: int, max_iter: int = 100,
                    mode: Mode = Mode.FP32_FAST, bands: Bands = FULL_FRAME, out=None,
                    palette=None, out_rgba=None, stream=None):
    """Julia frame with mode, cyclic bands and optional fused colour levels."""
    import torch
    rows = height if bands is FULL_FRAME else band_local_rows(height, bands)
    if out is None:
        out = torch.empty((rows, width), dtype=torch.uint16, device="cuda")
    pal = _pal(palette) if palette is not None else None
    if pal is not None and out_rgba is None:
        out_rgba = torch.empty((rows, width, 4), dtype=torch.uint8, device="cuda")
    p = _dev_ptr(out, "uint16", rows * width, "out")
    q = _dev_ptr(out_rgba, "uint8", rows * width * 4, "out_rgba") if out_rgba is not None else None
    rc = load().julia_render_ex(_Complex(complex(c).real, complex(c).imag), _window(win), width,
                                height, max_iter, int(mode), bands._c(), p,
                                ctypes.byref(pal.c) if pal else None, q, _stream(stream))
    _check(rc, "julia_render_ex")
    return (out, out_rgba) if pal is not None else out


def julia_render_path(cs, win, width: int, height: int, max_iter: int = 100,
                      mode: Mode = Mode.FP32_FAST, out=None, palette=None, out_rgba=None,
                      stream=None):
    """Julia frames along a path of C values: uint16 [n, height, width]
    (or uint8 when `out` is a uint8 tensor; needs max_iter <= 255)."""
    import torch
    arr = np.ascontiguousarray(np.asarray(cs, dtype=np.complex128).reshape(-1))
    n = arr.shape[0]
    if out is None:
        out = torch.empty((n, height, width), dtype=torch.uint16, device="cuda")
    pal = _pal(palette) if palette is not None else None
    if pal is not None and out_rgba is None:
        out_rgba = torch.empty((n, height, width, 4), dtype=torch.uint8, device="cuda")
    u8 = getattr(out, "dtype", None) is not None and str(out.dtype) == "torch.uint8"
    p = _dev_ptr(out, "uint8" if u8 else "uint16", n * width * height, "out")
    q = (_dev_ptr(out_rgba, "uint8", n * width * height * 4, "out_rgba")
         if out_rgba is not None else None)
    fn = load().julia_render_path8 if u8 else load().julia_render_path
    rc = fn(ctypes.c_void_p(arr.ctypes.data), n, _window(win), width, height, max_iter,
            int(mode), p, ctypes.byref(pal.c) if pal else None, q, _stream(stream))
    _check(rc, "julia_render_path8" if u8 else "julia_render_path")
    return (out, out_rgba) if pal is not None else out


def mandelbrot_param_map(win, width: int, height: int, max_iter: int = 100,
                         mode: Mode = Mode.FP64_FAST, bands: Bands = FULL_FRAME, out=None,
                         palette=None, out_rgba=None, stream=None):
    """Mandelbrot parameter map: C from the pixel, Z_0 = 0."""
    import torch
    rows = height if bands is FULL_FRAME else band_local_rows(height, bands)
    if out is None:
        out = torch.empty((rows, width), dtype=torch.uint16, device="cuda")
    pal = _pal(palette) if palette is not None else None
    if pal is not None and out_rgba is None:
        out_rgba = torch.empty((rows, width, 4), dtype=torch.uint8, device="cuda")
    p = _dev_ptr(out, "uint16", rows * width, "out")
    q = _dev_ptr(out_rgba, "uint8", rows * width * 4, "out_rgba") if out_rgba is not None else None
    rc = load().mandelbrot_param_map(_window(win), width, height, max_iter, int(mode), bands._c(),
                                     p, ctypes.byref(pal.c) if pal else None, q, _stream(stream))
    _check(rc, "mandelbrot_param_map")
    return (out, out_rgba) if pal is not None else out


def colorize(counts, max_iter: int, palette, out_rgba=None, stream=None):
    """Colour levels of a uint16 CUDA tensor -> uint8 [..., 4]."""
    import torch
    n = counts.numel()
    if out_rgba is None:
        out_rgba = torch.empty(tuple(counts.shape) + (4,), dtype=torch.uint8, device=counts.device)
    pal = _pal(palette)
    p = _dev_ptr(counts, "uint16", n, "counts")
    q = _dev_ptr(out_rgba, "uint8", 4 * n, "out_rgba")
    rc = load().colorize(p, n, max_iter, ctypes.byref(pal.c), q, _stream(stream))
    _check(rc, "colorize")
    return out_rgba


def julia_render_fn(fn, c: complex, win, width: int, height: int, max_iter: int = 100,
                    mode: Mode = Mode.FP32_STRICT, out=None, palette=None, out_rgba=None,
                    stream=None):
    """Julia frame of another iteration map (z^4 + c, z^4 + (z^2+1)/(z^2-1) + c)."""
    import torch
    if out is None:
        out = torch.empty((height, width), dtype=torch.uint16, device="cuda")
    pal = _pal(palette) if palette is not None else None
    if pal is not None and out_rgba is None:
        out_rgba = torch.empty((height, width, 4), dtype=torch.uint8, device="cuda")
    p = _dev_ptr(out, "uint16", height * width, "out")
    q = _dev_ptr(out_rgba, "uint8", height * width * 4, "out_rgba") if out_rgba is not None else None
    rc = load().julia_render_fn(int(fn), _Complex(complex(c).real, complex(c).imag), _window(win),
                                width, height, max_iter, int(mode), p,
                                ctypes.byref(pal.c) if pal else None, q, _stream(stream))
    _check(rc, "julia_render_fn")
    return (out, out_rgba) if pal is not None else out


def julia_render_path_host(cs, win, width: int, height: int, max_iter: int = 100,
                           mode: Mode = Mode.FP32_FAST, out=None, stream=None):
    """Julia frames along a C-path with the counts delivered to HOST memory (native
    chunked render + overlapped device->host copies; synchronous).  `out`: a host
    numpy array or CPU torch tensor of uint8 (max_iter <= 255) or uint16, shape
    [n, height, width]; pinned torch memory gives overlapped copies."""
    arr = np.ascontiguousarray(np.asarray(cs, dtype=np.complex128).reshape(-1))
    n = arr.shape[0]
    if out is None:
        out = np.empty((n, height, width), dtype=np.uint8 if max_iter <= 255 else np.uint16)
    if hasattr(out, "data_ptr"):  # torch CPU tensor
        if out.is_cuda or not out.is_contiguous():
            raise FractalError("out must be a contiguous host tensor")
        nbytes, ptr = out.element_size(), out.data_ptr()
        numel = out.numel()
    else:
        if not out.flags["C_CONTIGUOUS"]:
            raise FractalError("out must be C-contiguous")
        nbytes, ptr, numel = out.dtype.itemsize, out.ctypes.data, out.size
    if nbytes not in (1, 2) or numel < n * width * height:
        raise FractalError("out must hold n*height*width uint8/uint16 counts")
    rc = load().julia_render_path_host(ctypes.c_void_p(arr.ctypes.data), n, _window(win), width,
                                       height, max_iter, int(mode), nbytes, ctypes.c_void_p(ptr),
                                       _stream(stream))
    _check(rc, "julia_render_path_host")
    return out


class FramePlan:
    """Latency path for repeated renders of one frame shape (the interactive case of
    P:39 and the small frames of Fig. 1): every argument but C is validated and
    marshalled ONCE -- output pointers, window, bands, palette and stream are kept as
    ready ctypes objects -- so `render(c)` is one C-ABI call (julia_render_ex, or
    mandelbrot_param_map for kind='mandelbrot', where C is ignored) plus the C value.
    The output tensors are owned by the plan (`out`, `out_rgba`).  The calls it makes
    are ordinary C-ABI calls, so a plan can also be captured into a CUDA graph (after
    one eager render on the stream: the library's workspaces are created outside
    capture, include/fractal.h "Memory")."""

    def __init__(self, kind: str, win, width: int, height: int, max_iter: int = 100,
                 mode: Mode = Mode.FP32_FAST, bands: Bands = FULL_FRAME, palette=None,
                 out=None, out_rgba=None, stream=None):
        import torch
        if kind not in ("julia", "mandelbrot"):
            raise FractalError(f"kind must be 'julia' or 'mandelbrot', got {kind!r}")
        rows = height if bands is FULL_FRAME else band_local_rows(height, bands)
        self.out = out if out is not None else torch.empty((rows, width), dtype=torch.uint16,
                                                           device="cuda")
        self._pal = _pal(palette) if palette is not None else None
        if self._pal is not None and out_rgba is None:
            out_rgba = torch.empty((rows, width, 4), dtype=torch.uint8, device="cuda")
        self.out_rgba = out_rgba
        self._p = _dev_ptr(self.out, "uint16", rows * width, "out")
        self._q = (_dev_ptr(out_rgba, "uint8", rows * width * 4, "out_rgba")
                   if out_rgba is not None else None)
        self._palp = ctypes.byref(self._pal.c) if self._pal is not None else None
        self._win = _window(win)
        self._bands = bands._c()
        self._stream = _stream(stream)
        self._args = (width, height, max_iter, int(mode))
        self._c = _Complex(0.0, 0.0)
        lib = load()
        self._fn = lib.julia_render_ex if kind == "julia" else lib.mandelbrot_param_map
        self._julia = kind == "julia"

    def render(self, c: complex = 0j):
        """Enqueue the frame for C = c on the plan's stream; returns the output tensor(s)."""
        if self._julia:
            self._c.re = c.real
            self._c.im = c.imag
            rc = self._fn(self._c, self._win, *self._args, self._bands, self._p, self._palp,
                          self._q, self._stream)
        else:
            rc = self._fn(self._win, *self._args, self._bands, self._p, self._palp, self._q,
                          self._stream)
        if rc:
            _check(rc, "FramePlan.render")
        return (self.out, self.out_rgba) if self._pal is not None else self.out
