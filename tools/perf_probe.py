"""Quick per-config timing probe (not the bench contract): CUDA-event time per render,
Gpixel-iter/s from the rendered counts, for fast and strict modes."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W

def total(t):
    return int((t.view(torch.int16).to(torch.int64) & 0xFFFF).sum().item())

def timeit(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts)), float(min(ts))

res = {}
cf = W.configs()
only = sys.argv[1:] or ["cfg1","cfg2","cfg3","cfg4","cfg5"]
for name in only:
    c = cf[name]
    for mode in ([fr.Mode.FP32_FAST, fr.Mode.FP32_STRICT] if c.precision == 32 else [fr.Mode.FP64_FAST, fr.Mode.FP64_STRICT]):
        pal = W.palette("classic") if c.colorize else None
        if c.kind == "julia":
            out = torch.empty((c.height, c.width), dtype=torch.uint16, device="cuda")
            rgba = torch.empty((c.height, c.width, 4), dtype=torch.uint8, device="cuda") if pal else None
            fn = lambda: fr.julia_render_ex(c.c, c.window, c.width, c.height, c.max_iter, mode, out=out, palette=pal, out_rgba=rgba)
        elif c.kind == "path":
            nf = 512
            cs = W.circle_path(4096)[::8]
            out = torch.empty((nf, c.height, c.width), dtype=torch.uint16, device="cuda")
            fn = lambda: fr.julia_render_path(cs, c.window, c.width, c.height, c.max_iter, mode, out=out)
        else:
            out = torch.empty((c.height, c.width), dtype=torch.uint16, device="cuda")
            fn = lambda: fr.mandelbrot_param_map(c.window, c.width, c.height, c.max_iter, mode, out=out)
        reps = 3 if name == "cfg5" else 20
        med, mn = timeit(fn, reps=reps, warm=1 if name == "cfg5" else 3)
        s = total(out)
        lanes = 64 if c.precision == 64 else 128
        frac = s * 6 / (med * 1e-3) / (148 * lanes * 1.965e9)
        res[f"{name}/{mode.name}"] = dict(ms=med, ms_min=mn, sum=s, gpix_iter_s=s / (med * 1e-3) / 1e9, frac_1965=frac)
        print(name, mode.name, json.dumps(res[f"{name}/{mode.name}"]), flush=True)
