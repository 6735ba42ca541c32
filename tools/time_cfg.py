"""Time one config's single-frame render (CUDA events, back-to-back, after warm-up).
usage: python tools/time_cfg.py cfg2 [reps] [MODE]   -> one JSON line (ms per call)
(GRAPH=1: replays of a CUDA graph of 50 calls)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
c = W.configs()[name]
mode = fr.Mode[sys.argv[3]] if len(sys.argv) > 3 else (
    fr.Mode.FP32_FAST if c.precision == 32 else fr.Mode.FP64_FAST)
pal = W.palette("classic") if c.colorize and not os.environ.get("NOCOLOR") else None
out = torch.empty((c.height, c.width), dtype=torch.uint16, device="cuda")
rgba = torch.empty((c.height, c.width, 4), dtype=torch.uint8, device="cuda") if pal else None


def call():
    if c.kind == "julia":
        fr.julia_render_ex(c.c, c.window, c.width, c.height, c.max_iter, mode, out=out,
                           palette=pal, out_rgba=rgba)
    else:
        fr.mandelbrot_param_map(c.window, c.width, c.height, c.max_iter, mode, out=out)


for _ in range(5):
    call()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if os.environ.get("GRAPH") == "1":  # replay a CUDA graph of 50 calls
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        call()
    torch.cuda.current_stream().wait_stream(side)
    with torch.cuda.graph(g):
        for _ in range(50):
            call()
    g.replay()
    torch.cuda.synchronize()
    n_rep = max(1, reps // 50)
    a.record()
    for _ in range(n_rep):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / (50 * n_rep)
else:
    a.record()
    for _ in range(reps):
        call()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
iters = int(out.view(torch.int16).to(torch.int64).bitwise_and(0xFFFF).sum())
print(json.dumps({"cfg": name, "sched": os.environ.get("FRACTAL_SCHED", "default"),
                  "ms": ms, "gpix_iter_s": iters / ms / 1e6}))
