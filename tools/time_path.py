"""Time julia_render_path on the bench workload (512 x 1080p frames, mi 100) in one mode.
usage: python tools/time_path.py [MODE] [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
mode = fr.Mode[sys.argv[1]] if len(sys.argv) > 1 else fr.Mode.FP32_FAST
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
mi = int(sys.argv[3]) if len(sys.argv) > 3 else 100
cs = W.circle_path(512)
win = W.julia_window(1920, 1080)
out = torch.empty((512, 1080, 1920), dtype=torch.uint16, device="cuda")
for _ in range(2):
    fr.julia_render_path(cs, win, 1920, 1080, mi, mode, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    fr.julia_render_path(cs, win, 1920, 1080, mi, mode, out=out)
b.record()
torch.cuda.synchronize()
print(json.dumps({"mode": mode.name, "max_iter": mi, "ms": a.elapsed_time(b) / reps}))
