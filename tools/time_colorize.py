"""Standalone colorize bandwidth (bench.colorize_bandwidth) with the library named by
FRACTAL_LIB (or the default); prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W

fr.load()
r = bench.colorize_bandwidth(fr, W, torch)
print(json.dumps({"ms": round(r["ms"], 4), "GB_per_s": round(r["GB_per_s"], 1), "frac": round(r["frac"], 4)}))
