"""Independent numpy cross-check of the C oracle -- TEST INFRASTRUCTURE ONLY.

Written separately from ``escape_oracle.c`` (no shared code) so that each pins the
other on small grids.  numpy ufuncs round every multiply and add separately (no
fused multiply-add), so with the same operation order the results are IEEE
identical to the C oracle built with ``-ffp-contract=off``.

P:31 (iteration, region-covering, limit), P:47 (Mandelbrot: C from pixel, Z_0 = 0),
S:58/S:73-75 (count definition, strict bailout > 4).
"""
from __future__ import annotations

import numpy as np


def axes(center: complex, half_w: float, half_h: float, width: int, height: int):
    """Pixel-centre coordinates in float64: re[width], im[height] (reading c-3)."""
    hx = np.float64(half_w) / np.float64(width)
    hy = np.float64(half_h) / np.float64(height)
    kx = (2 * np.arange(width, dtype=np.int64) + 1 - width).astype(np.float64)
    ky = (height - 1 - 2 * np.arange(height, dtype=np.int64)).astype(np.float64)
    return np.float64(center.real) + kx * hx, np.float64(center.imag) + ky * hy


def escape_grid(z_re, z_im, c_re, c_im, max_iter: int, dtype) -> np.ndarray:
    """Vectorised escape time: first n with x^2 + y^2 > 4 (else max_iter)."""
    x = np.array(z_re, dtype=dtype, copy=True)
    y = np.array(z_im, dtype=dtype, copy=True)
    x, y = np.broadcast_arrays(x, y)
    x, y = x.copy(), y.copy()
    cr = np.broadcast_to(np.asarray(c_re, dtype=dtype), x.shape)
    ci = np.broadcast_to(np.asarray(c_im, dtype=dtype), x.shape)
    count = np.full(x.shape, max_iter, dtype=np.int64)
    alive = np.ones(x.shape, dtype=bool)
    four = dtype(4)
    with np.errstate(over="ignore", invalid="ignore"):
        for n in range(max_iter):
            xx = x * x
            yy = y * y
            m = xx + yy
            esc = alive & (m > four)
            count[esc] = n
            alive &= ~esc
            if not alive.any():
                break
            xy = x * y
            x = (xx - yy) + cr
            y = (xy + xy) + ci
    return count


def julia(c: complex, center: complex, half_w: float, half_h: float, width: int, height: int,
          max_iter: int = 100, precision: int = 32) -> np.ndarray:
    dtype = np.float32 if precision == 32 else np.float64
    re, im = axes(center, half_w, half_h, width, height)
    zr = re.astype(dtype)[None, :]
    zi = im.astype(dtype)[:, None]
    cr = dtype(np.float64(c.real))
    ci = dtype(np.float64(c.imag))
    return escape_grid(zr, zi, cr, ci, max_iter, dtype).astype(np.uint16)


def mandelbrot(center: complex, half_w: float, half_h: float, width: int, height: int,
               max_iter: int = 100, precision: int = 64) -> np.ndarray:
    dtype = np.float32 if precision == 32 else np.float64
    re, im = axes(center, half_w, half_h, width, height)
    cr = np.broadcast_to(re.astype(dtype)[None, :], (height, width))
    ci = np.broadcast_to(im.astype(dtype)[:, None], (height, width))
    zero = np.zeros((height, width), dtype=dtype)
    return escape_grid(zero, zero, cr, ci, max_iter, dtype).astype(np.uint16)
