"""Small renders through every kernel family for compute-sanitizer (memcheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
pal = W.palette("classic")
for (w, h) in [(1, 1), (37, 5), (65, 17), (100, 33)]:
    win = W.julia_window(w, h)
    for mode in fr.Mode:
        fr.julia_render_ex(0.285 + 0.01j, win, w, h, 300, mode, palette=pal)
        fr.julia_render_ex(0.285 + 0.01j, win, w, h, 50, mode, fr.Bands(4, 3, 1), palette=pal)
        fr.mandelbrot_param_map((-0.5 + 0j, 1.5, 1.5 * h / w), w, h, 1200, mode, palette=pal)
        fr.mandelbrot_param_map((-0.5 + 0j, 1.5, 1.5 * h / w), w, h, 300, mode, fr.Bands(3, 2, 0))
        fr.julia_render_path(W.circle_path(5), win, w, h, 100, mode, palette=pal)
        fr.julia_render_path(W.circle_path(3), win, w, h, 100, mode,
                             out=torch.empty((3, h, w), dtype=torch.uint8, device="cuda"))
        for fn in (fr.Function.Z4, fr.Function.Z4_RATIONAL):
            fr.julia_render_fn(fn, W.FIG4_C, win, w, h, 100, mode, palette=pal)
    t = torch.randint(0, 301, (w * h,), dtype=torch.int32).to(torch.int16).cuda().view(torch.uint16)
    fr.colorize(t, 300, pal)
    fr.colorize(t[1:], 300, pal)
torch.cuda.synchronize()
print("sanitize workload done")
