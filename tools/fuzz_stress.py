"""One-off parity stress (not part of the default suite): N seeded random cases (C,
window, ragged W x H up to MAX_SIDE, max_iter in {1, 3, 50, 100, 255, 256, 300, 1000}),
Julia and Mandelbrot, all four modes.  Strict modes must equal the oracle bit for bit;
fast modes must equal the FAST (FMA-sequence) oracle bit for bit, and their distance
from the strict oracle is compared with reading c-10's fraction bound (max(1e-4, 4 x
the oracle's 1-ulp sensitivity, estimated on the frame)).  Prints one JSON summary line.
usage: python tools/fuzz_stress.py [N] [MAX_SIDE] [SEED]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
max_side = int(sys.argv[2]) if len(sys.argv) > 2 else 800
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 20261018
rng = np.random.default_rng(seed)
mis = [1, 3, 50, 100, 255, 256, 300, 1000]


def np16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


t0 = time.time()
strict_bad, fast_bad, fast_exact_bad, checked = [], [], [], 0
for i in range(n):
    r = 1.2 * np.sqrt(rng.uniform())
    th = rng.uniform(0, 2 * np.pi)
    c = complex(r * np.cos(th), r * np.sin(th))
    w = int(rng.integers(1, max_side + 1))
    h = int(rng.integers(1, max_side + 1))
    hw = float(10 ** rng.uniform(-4, 0.4))
    center = complex(rng.uniform(-1.2, 0.6), rng.uniform(-1.0, 1.0))
    win = W.Window(center, hw, hw * h / w)
    mi = int(rng.choice(mis))
    for kind in ("julia", "mandelbrot"):
        for mode in fr.Mode:
            prec = 64 if mode.name.startswith("FP64") else 32
            strict = mode.name.endswith("STRICT")
            if kind == "julia":
                got = np16(fr.julia_render_ex(c, win, w, h, mi, mode))
                ref = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec)
            else:
                got = np16(fr.mandelbrot_param_map(win, w, h, mi, mode))
                ref = oracle.mandelbrot(win.center, win.half_w, win.half_h, w, h, mi, prec)
            checked += 1
            frac = float(np.mean(got != ref))
            if strict and frac > 0:
                strict_bad.append((i, kind, mode.name, w, h, mi, frac))
            if not strict:
                if kind == "julia":
                    ref_f = oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, prec,
                                         fast=True)
                else:
                    ref_f = oracle.mandelbrot(win.center, win.half_w, win.half_h, w, h, mi, prec,
                                              fast=True)
                if (got != ref_f).any():
                    fast_exact_bad.append((i, kind, mode.name, w, h, mi,
                                           float(np.mean(got != ref_f))))
            if not strict and frac > 0:
                py, px = np.divmod(np.arange(w * h, dtype=np.int64), w)
                nud = oracle.pixels_nudged(kind, c, win.center, win.half_w, win.half_h, w, h,
                                           mi, prec, px, py).reshape(h, w)
                sens = float(np.mean(nud != ref))
                if frac > max(1e-4, 4 * sens) and frac > 2.0 / (w * h):
                    # pitch relative to binary32 spacing at the window: < ~100 ulps per
                    # pixel is the ill-conditioned regime for fp32
                    ulp = np.spacing(np.float32(max(abs(win.center.real), abs(win.center.imag),
                                                    win.half_w, 1e-30)))
                    pitch_ulps = float(2 * win.half_w / w / ulp)
                    fast_bad.append((i, kind, mode.name, w, h, mi, round(frac, 5),
                                     round(sens, 5), round(pitch_ulps, 1)))
torch.cuda.synchronize()
fast_renders = checked // 2
print(json.dumps({"cases": n, "renders_checked": checked, "strict_mismatches": strict_bad[:10],
                  "fast_renders": fast_renders,
                  "fast_vs_fast_oracle_mismatches": fast_exact_bad[:10],
                  "fast_over_bound_count": len(fast_bad),
                  "fast_over_bound": sorted(fast_bad, key=lambda x: x[-1])[:12],
                  "max_pitch_ulps_over_bound": max([x[-1] for x in fast_bad], default=None),
                  "seconds": round(time.time() - t0, 1),
                  "seed": seed, "max_side": max_side}))
