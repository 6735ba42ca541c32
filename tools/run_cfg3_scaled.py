"""cfg3's window at scale s (pixels x s^2), for side-by-side ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
s = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = W.configs()["cfg3"]
for _ in range(reps):
    fr.julia_render_ex(c.c, c.window, c.width * s, c.height * s, c.max_iter, fr.Mode.FP32_FAST)
torch.cuda.synchronize(); print("ok")
