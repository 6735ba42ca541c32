"""Time kernel A on a 4096^2 part of the cfg5 deep-zoom window (quarter half-widths, same
centre, max_iter 10000, FP64_FAST): a short stand-in for ncu captures of cfg5's kernel."""
import sys, torch
sys.path.insert(0, '.')
from paper_1611_03079_b200 import binding as fr, workloads as W
fr.load()
c = W.configs()['cfg5']
w = 4096
win = W.Window(c.window.center, c.window.half_w / 4, c.window.half_h / 4)
out = torch.empty((w, w), dtype=torch.uint16, device='cuda')
for _ in range(2):
    fr.mandelbrot_param_map(win, w, w, c.max_iter, fr.Mode.FP64_FAST, out=out)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(); fr.mandelbrot_param_map(win, w, w, c.max_iter, fr.Mode.FP64_FAST, out=out); b.record(); b.synchronize()
s = int(out.view(torch.int16).to(torch.int64).bitwise_and(0xFFFF).sum())
print("ms", a.elapsed_time(b), "iters", s, "Gpix-iter/s", s / a.elapsed_time(b) / 1e6)
