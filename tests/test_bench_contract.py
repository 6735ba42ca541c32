"""bench.py's JSON-line contract (the CPU oracle arm runs here; the GPU arm on a B200)
and the seeded workload recipes shared by both sides."""
import json
import math
import os
import subprocess
import sys

import numpy as np

from paper_1611_03079_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]


def test_configs_match_baseline_json():
    bj = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    cf = W.configs()
    assert len(bj["configs"]) == len(cf) == 5
    c1, c2, c3, c4, c5 = (cf[f"cfg{i}"] for i in range(1, 6))
    assert (c1.width, c1.height, c1.max_iter, c1.c) == (64, 64, 100, -0.8 + 0.156j)
    assert (c1.window.half_w, c1.window.half_h) == (1.5, 1.5)
    assert (c2.width, c2.height, c2.max_iter, c2.c) == (1920, 1080, 100, -0.7269 + 0.1889j)
    assert (c3.width, c3.height, c3.max_iter, c3.colorize) == (3840, 2160, 1000, True)
    assert (c4.n_frames, c4.width, c4.height, c4.max_iter) == (4096, 1920, 1080, 100)
    assert (c5.width, c5.height, c5.max_iter, c5.precision, c5.kind) == (16384, 16384, 10000, 64, "mandelbrot")


def test_circle_path_recipe():
    cs = W.circle_path(4096)
    assert np.allclose(np.abs(cs), 0.7885, rtol=0, atol=1e-15)
    assert cs[0] == 0.7885 and abs(cs[1024] - 0.7885j) < 1e-15
    th = np.unwrap(np.angle(cs))
    assert np.allclose(np.diff(th), 2 * math.pi / 4096)


def test_palette_data():
    pal, inter = W.palette("classic")
    assert pal.shape == (16, 4) and (pal[:, 3] == 255).all() and list(inter) == [0, 0, 0, 255]
    assert list(pal[0][:3]) == [0, 0, 128] and list(pal[15][:3]) == [255, 255, 255]
    fire, _ = W.palette("fire")
    assert list(fire[7][:3]) == [255, 0, 0] and list(fire[15][:3]) == [255, 255, 0]


def test_fuzz_cases_are_seeded():
    a, b = W.fuzz_cases(10), W.fuzz_cases(10)
    assert [x[0] for x in a] == [x[0] for x in b]
    assert all(1 <= w <= 512 and 1 <= h <= 512 for _, _, w, h, _ in a)
