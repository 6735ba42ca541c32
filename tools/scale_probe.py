"""Does per-launch drain matter?  cfg3's window rendered at 1x, 2x, 4x pixels (same
work per pixel): time per pixel-iteration should be constant if not."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
c = W.configs()["cfg3"]
pal = W.palette("classic")
for s in (1, 2, 4):
    w, h = c.width * s // 2 if s == 1 else c.width * s // 2, c.height * s // 2 if s == 1 else c.height * s // 2
    for (w, h) in [(c.width * s, c.height * s)] if s > 1 else [(c.width // 2, c.height // 2), (c.width, c.height)]:
        out = torch.empty((h, w), dtype=torch.uint16, device="cuda")
        rgba = torch.empty((h, w, 4), dtype=torch.uint8, device="cuda")
        fn = lambda: fr.julia_render_ex(c.c, c.window, w, h, c.max_iter, fr.Mode.FP32_FAST, out=out, palette=pal, out_rgba=rgba)
        fn(); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): fn()
        b.record(); b.synchronize()
        ms = a.elapsed_time(b) / 10
        tot = int((out.view(torch.int16).to(torch.int64) & 0xFFFF).sum())
        print(json.dumps({"w": w, "h": h, "ms": ms, "gpix_iter_s": tot / ms / 1e6}), flush=True)
