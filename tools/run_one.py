"""Run one config render a few times (for ncu / sanitizer captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
name = sys.argv[1]; reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = fr.Mode[sys.argv[3]] if len(sys.argv) > 3 else None
c = W.configs()[name]
mode = mode or (fr.Mode.FP32_FAST if c.precision == 32 else fr.Mode.FP64_FAST)
for _ in range(reps):
    if c.kind == "julia":
        fr.julia_render_ex(c.c, c.window, c.width, c.height, c.max_iter, mode,
                           palette=W.palette("classic") if c.colorize else None)
    elif c.kind == "path":
        fr.julia_render_path(W.circle_path(4096)[::8], c.window, c.width, c.height, c.max_iter, mode)
    else:
        w = c.width if len(sys.argv) <= 4 else int(sys.argv[4])
        fr.mandelbrot_param_map(c.window, w, w, c.max_iter, mode)
torch.cuda.synchronize()
print("ok")
