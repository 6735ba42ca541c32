"""Time the NEXT-3 Figure 4 maps (bench.fig4_maps_rate) with the library named by
FRACTAL_LIB (or the default); prints one JSON line.  usage: python tools/time_fig4.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W

fr.load()
r = bench.fig4_maps_rate(fr, W, torch, 1965.0)
print(json.dumps({k: round(v["ms"], 4) if isinstance(v, dict) else v for k, v in r.items()}))
