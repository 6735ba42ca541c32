import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
n = 128 * 1920 * 1080
counts = torch.randint(0, 101, (n,), dtype=torch.int32, device="cuda").to(torch.int16).view(torch.uint16)
rgba = torch.empty((n, 4), dtype=torch.uint8, device="cuda")
for _ in range(3):
    fr.colorize(counts, 100, W.palette("classic"), out_rgba=rgba)
torch.cuda.synchronize(); print("ok")
