"""Write tests/golden/cfg5_oracle.json: hashes of the FULL cfg5 frame computed by the CPU
oracle only (no CUDA code is imported).

cfg5 = BASELINE.json configs[4]: Mandelbrot parameter map 16384 x 16384,
max_iter 10000, fp64, deep-zoom window of DESIGN.md reading c-7.  The oracle cannot
run it inside a GPU test (about 2.4e12 binary64 iterations, ~25 min on 8 host cores),
so this committed script computes it once and stores, per precision mode,
  sha256 of the whole frame (little-endian uint16, row-major, row 0 = top), the
  sha256 of every block of 1024 rows (so a mismatch is localised), sum of counts and
  the interior count.
tests/test_gpu_parity.py::test_cfg5_full_frame_hash compares the GPU frame with it
(the parallel render equals the sequential one bit for bit).

usage: python tools/oracle_cfg5_golden.py [strict|fast ...]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1611_03079_b200 import workloads as W  # noqa: E402  (input recipes only)

OUT = os.path.join(ROOT, "tests", "golden", "cfg5_oracle.json")
BLOCK = 1024


def render_rows(cfg, r0, r1, fast):
    """Rows r0..r1-1 of the full frame: the oracle's pixel list over those rows (the
    region-covering map of the FULL frame, so rows are bit-identical to a whole render)."""
    w = cfg.width
    py, px = np.meshgrid(np.arange(r0, r1, dtype=np.int64), np.arange(w, dtype=np.int64),
                         indexing="ij")
    win = cfg.window
    v = oracle.pixels("mandelbrot", 0j, win.center, win.half_w, win.half_h, w, cfg.height,
                      cfg.max_iter, 64, px.ravel(), py.ravel(), fast=fast)
    return v.reshape(r1 - r0, w)


def main(modes):
    cfg = W.configs()["cfg5"]
    doc = json.load(open(OUT)) if os.path.exists(OUT) else {}
    doc["_about"] = ("cfg5 (BASELINE configs[4]) computed by oracle/ only via "
                     "tools/oracle_cfg5_golden.py: sha256 of little-endian uint16 counts, "
                     "row-major, row 0 = top; blocks of 1024 rows")
    for mode in modes:
        fast = mode == "fast"
        t0 = time.time()
        h_all = hashlib.sha256()
        blocks, total, interior = [], 0, 0
        for r0 in range(0, cfg.height, BLOCK):
            rows = render_rows(cfg, r0, min(r0 + BLOCK, cfg.height), fast)
            b = rows.astype("<u2").tobytes()
            h_all.update(b)
            blocks.append(hashlib.sha256(b).hexdigest())
            total += int(rows.sum(dtype=np.int64))
            interior += int((rows == cfg.max_iter).sum())
            print(f"{mode} rows {r0}..{r0 + BLOCK} {time.time() - t0:.0f}s", flush=True)
        doc["FP64_FAST" if fast else "FP64_STRICT"] = {
            "sha256": h_all.hexdigest(), "block_rows": BLOCK, "blocks": blocks,
            "sum_counts": total, "interior": interior,
            "oracle_seconds": round(time.time() - t0, 1),
            "oracle_threads": oracle.default_threads()}
        with open(OUT, "w") as f:
            json.dump(doc, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1:] or ["strict"])
