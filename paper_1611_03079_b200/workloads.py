"""Seeded, synthetic inputs shaped like the paper's workloads.

This module holds NO escape-time arithmetic: only input recipes (windows, C values,
C-paths, palettes as data, fuzz generators).  It is the one module that both the CUDA
path's tests/bench and the CPU oracle's tests draw inputs from.

Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, BJ = BASELINE.json.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

FUZZ_SEED = 161103079  # numpy.random.default_rng(161103079)


@dataclass(frozen=True)
class Window:
    """Region covered ("region-covering routine"): centre and half extents."""
    center: complex
    half_w: float
    half_h: float


def julia_window(width: int, height: int, span_re: float = 4.0, center: complex = 0j) -> Window:
    """SPEC default Julia viewport: centre 0, real span 4, square pixels
    (reading c-4): half_w = span/2, half_h = half_w * H / W."""
    half_w = span_re / 2.0
    return Window(center, half_w, half_w * height / width)


def mandel_window(width: int, height: int, span_re: float = 3.0, center: complex = -0.5 + 0j) -> Window:
    """SPEC default Mandelbrot viewport: centre -0.5, span 3, square pixels."""
    half_w = span_re / 2.0
    return Window(center, half_w, half_w * height / width)


# ---------------------------------------------------------------- paper parameter values
# Figure 2: four C values "traversing the main cardioid", caption order.
FIG2_C = (0.320564 - 0.0391827j, -0.454038 - 0.572187j, -0.763667 + 0.0870413j,
          0.137384 + 0.600803j)
# Figure 3: two very close C values from a Mandelbrot deep zoom.
FIG3_C = (0.177078 + 0.577384j, 0.185723 + 0.588104j)
# Figure 4: the alternate-function parameter (NEXT-3; not on the hot path).
FIG4_C = 0.862085 + 0.64695j
# "zoom on Julia set" (Figure 4 caption): the paper gives no window; this 1080p zoom on
# the rational map's set boundary (centre 0.65625+0.65625i, real span 0.375) is chosen
# for orbits of cfg4-like length (mean count ~15, ~7% interior at max_iter 100).
FIG4_ZOOM_CENTER = 0.65625 + 0.65625j
FIG4_ZOOM_SPAN = 0.375
# Cardioid path divisor: a = 3.9 (a = 4 is the main-cardioid border).
CARDIOID_A = 3.9

# Deep-zoom anchor for config 5 (reading c-7): where the boundary of M
# crosses the segment between the two Figure 3 parameters.
CFG5_CENTER = 0.179562260547786 + 0.580464540552026j
CFG5_HALF = 1e-9


def circle_path(n_frames: int, radius: float = 0.7885) -> np.ndarray:
    """Config 4's C-path (reading c-6): C_k = r (cos th_k, sin th_k),
    th_k = 2 pi k / n_frames, computed once on the host in double with libm
    (math.cos/math.sin); complex128 [n_frames]."""
    out = np.empty(n_frames, dtype=np.complex128)
    for k in range(n_frames):
        th = 2.0 * math.pi * k / n_frames
        out[k] = complex(radius * math.cos(th), radius * math.sin(th))
    return out


# ---------------------------------------------------------------- BASELINE configs
@dataclass(frozen=True)
class Config:
    name: str
    kind: str          # "julia" | "path" | "mandelbrot"
    width: int
    height: int
    max_iter: int
    precision: int     # 32 | 64
    window: Window
    c: complex = 0j    # Julia C (kind == "julia")
    n_frames: int = 1  # kind == "path"
    colorize: bool = False
    band_rows: int = 0
    note: str = ""
    path: tuple = field(default=(), repr=False)

    @property
    def pixels(self) -> int:
        return self.width * self.height * self.n_frames


def configs() -> dict:
    """The five BASELINE.json configs as concrete synthetic inputs."""
    return {
        "cfg1": Config("cfg1", "julia", 64, 64, 100, 32, Window(0j, 1.5, 1.5), c=-0.8 + 0.156j,
                       note="BJ configs[0]: Julia C=-0.8+0.156i, 64x64, [-1.5,1.5]^2, mi 100, fp32"),
        "cfg2": Config("cfg2", "julia", 1920, 1080, 100, 32, julia_window(1920, 1080),
                       c=-0.7269 + 0.1889j,
                       note="BJ configs[1]: Julia C=-0.7269+0.1889i, 1920x1080, mi 100, fp32"),
        "cfg3": Config("cfg3", "julia", 3840, 2160, 1000, 32, julia_window(3840, 2160),
                       c=-0.7269 + 0.1889j, colorize=True, band_rows=15,
                       note="BJ configs[2]: Julia 3840x2160, mi 1000, fp32 + fused colorize, bands"),
        "cfg4": Config("cfg4", "path", 1920, 1080, 100, 32, julia_window(1920, 1080),
                       n_frames=4096,
                       note="BJ configs[3]: 4096 frames 1080p, C on |C|=0.7885, mi 100, fp32"),
        "cfg5": Config("cfg5", "mandelbrot", 16384, 16384, 10000, 64,
                       Window(CFG5_CENTER, CFG5_HALF, CFG5_HALF), band_rows=16,
                       note="BJ configs[4]: Mandelbrot 16384^2, mi 10000, fp64 deep zoom, bands"),
    }


# ---------------------------------------------------------------- palettes (data)
def _rn(v: float) -> int:
    return int(math.floor(v + 0.5))


def palette(name: str = "classic"):
    """Built-in palettes as DATA (reading c-12).
    Returns (entries uint8 [16, 4] RGBA, interior uint8 [4])."""
    if name == "classic":  # dark blue -> white ramp
        ent = [(_rn(255 * i / 15), _rn(255 * i / 15), 128 + _rn(127 * i / 15), 255) for i in range(16)]
    elif name == "fire":  # black -> red -> yellow ramp
        ent = [(_rn(255 * i / 7), 0, 0, 255) if i < 8 else (255, _rn(255 * (i - 8) / 7), 0, 255)
               for i in range(16)]
    else:
        raise KeyError(f"unknown palette {name!r}")
    return np.array(ent, dtype=np.uint8), np.array([0, 0, 0, 255], dtype=np.uint8)


# ---------------------------------------------------------------- fuzzing
def fuzz_cases(n: int, max_side: int = 512, seed: int = FUZZ_SEED):
    """Seeded random (C, window, W, H, max_iter) cases: C near the Mandelbrot boundary
    region |C| <= 1.2 for 4 cases in 5, and 1.2 < |C| <= 2.5 for the fifth -- past the
    escape-monotonicity bound |C| <= 1.989 of the amortised kernels,
    where an orbit can leave radius 2 and come back -- windows of random centre/scale,
    ragged sizes."""
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n):
        r = 1.2 * math.sqrt(rng.uniform())
        if k % 5 == 4:
            r = float(rng.uniform(1.2, 2.5))
        th = rng.uniform(0, 2 * math.pi)
        c = complex(r * math.cos(th), r * math.sin(th))
        w = int(rng.integers(1, max_side + 1))
        h = int(rng.integers(1, max_side + 1))
        half_w = float(10 ** rng.uniform(-3, 0.5))
        center = complex(rng.uniform(-1.0, 1.0), rng.uniform(-1.0, 1.0))
        mi = int(rng.choice([1, 2, 7, 100, 257, 1000]))
        out.append((c, Window(center, half_w, half_w * h / w), w, h, mi))
    return out
