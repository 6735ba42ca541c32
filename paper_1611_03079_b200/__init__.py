"""B200-native escape-time engine for arXiv 1611.03079 (Julia frames, C-paths,
Mandelbrot parameter maps, colour levels).

The compute path is ``libfractal.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/fractal.h``); ``binding`` marshals torch tensors to it.  Importing this
package does not load the library; the first call does, and fails loudly if the
library is missing (there is no CPU fallback).
"""
from importlib import import_module as _imp

__all__ = ["julia_render", "julia_render_ex", "julia_render_path", "mandelbrot_param_map",
           "colorize", "FractalError", "Mode", "Bands", "FULL_FRAME", "band_local_rows",
           "band_global_row", "launch_count", "version", "cardioid_path", "julia_render_fn", "Function", "julia_render_path_host", "workloads"]


def __getattr__(name):
    if name == "workloads":
        return _imp(".workloads", __name__)
    if name in __all__:
        return getattr(_imp(".binding", __name__), name)
    raise AttributeError(name)
