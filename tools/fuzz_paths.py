"""One-off parity stress for C-paths (not part of the default suite): N seeded random
paths -- 1..300 frames, C on random arcs (radius up to 2.3, so some paths leave the
escape-monotonicity bound |C| <= 1.989), ragged W x H up to MAX_SIDE, max_iter from a
list around the vote block, all four modes, uint16 or uint8 counts, with or without fused
colour -- every frame compared with the oracle: strict modes bit for bit with the strict
oracle, fast modes bit for bit with the FAST oracle.  Prints one JSON summary line.
usage: python tools/fuzz_paths.py [N] [MAX_SIDE] [SEED]"""
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
max_side = int(sys.argv[2]) if len(sys.argv) > 2 else 160
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 20261019
rng = np.random.default_rng(seed)
mis = [1, 2, 3, 4, 7, 8, 50, 99, 100, 255]
pal = W.palette("fire")

t0 = time.time()
bad, frames_checked = [], 0
for i in range(n):
    nf = int(rng.integers(1, 301))
    r = float(rng.uniform(0.0, 2.3))
    th0, dth = rng.uniform(0, 2 * np.pi), rng.uniform(-0.5, 0.5)
    cs = np.array([r * np.exp(1j * (th0 + dth * k / max(nf, 1))) for k in range(nf)])
    w = int(rng.integers(1, max_side + 1))
    h = int(rng.integers(1, max_side // 2 + 1))
    win = W.julia_window(w, h)
    mi = int(rng.choice(mis))
    mode = list(fr.Mode)[int(rng.integers(0, 4))]
    prec = 64 if mode.name.startswith("FP64") else 32
    fast = mode.name.endswith("FAST")
    u8 = bool(rng.integers(0, 2)) and mi <= 255
    colour = bool(rng.integers(0, 2))
    kw = {}
    if colour:
        kw = dict(palette=pal)
    if u8:
        out = torch.empty((nf, h, w), dtype=torch.uint8, device="cuda")
        res = fr.julia_render_path(cs, win, w, h, mi, mode, out=out, **kw)
        got = out.cpu().numpy()
        rgba = res[1].cpu().numpy() if colour else None
    else:
        res = fr.julia_render_path(cs, win, w, h, mi, mode, **kw)
        if colour:
            cnt_t, rgba_t = res
            got = cnt_t.view(torch.int16).cpu().numpy().view(np.uint16)
            rgba = rgba_t.cpu().numpy()
        else:
            got = res.view(torch.int16).cpu().numpy().view(np.uint16)
            rgba = None
    torch.cuda.synchronize()
    for k in range(nf):
        ref = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, w, h, mi, prec,
                           fast=fast)
        want = ref.astype(np.uint8) if u8 else ref
        ok = np.array_equal(got[k], want)
        if ok and rgba is not None:
            ok = np.array_equal(rgba[k], oracle.colorize(ref, mi, *pal))
        frames_checked += 1
        if not ok:
            bad.append((i, k, mode.name, w, h, mi, nf, round(r, 3), u8, colour))
            break
print(json.dumps({"paths": n, "frames_checked": frames_checked, "mismatches": bad[:10],
                  "n_mismatch_paths": len(bad), "seconds": round(time.time() - t0, 1),
                  "seed": seed, "max_side": max_side}))
