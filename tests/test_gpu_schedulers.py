"""Every kernel family, whatever the default dispatch picks: a parity subset re-run in
subprocesses with FRACTAL_SCHED forced to static (kernel S), refill (kernel R), amort
(kernel A) and twophase (kernels P1 + P2, at several phase-1 budgets), with the
persistent / CTA-local refill grids, and with programmatic dependent launch off."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SUBSET = ("test_strict_configs_full_frame or test_strict_fuzz or test_strict_ragged or "
          "test_bands or test_max_iter_65535 or test_every_pixel or test_fast_mode_tolerance_julia "
          "or test_nonmonotone")


@pytest.mark.parametrize("env", [{"FRACTAL_SCHED": "static"}, {"FRACTAL_SCHED": "refill"},
                                 {"FRACTAL_SCHED": "amort"}, {"FRACTAL_SCHED": "twophase"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_BUDGET": "4"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_BUDGET": "48",
                                  "FRACTAL_P2_OCC": "1"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P1_TILES": "2"},
                                 {"FRACTAL_SCHED": "refill", "FRACTAL_REFILL_CPC": "16"},
                                 {"FRACTAL_SCHED": "amort", "FRACTAL_REFILL_CPC": "0"},
                                 {"FRACTAL_PDL": "0"}])
def test_parity_under_forced_scheduler(env):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-m", "gpu", "-q", "-x", "-k", SUBSET, "-p", "no:cacheprovider"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


_HASH_SCRIPT = r"""
import hashlib, sys
import torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
out = []
for mode in ("FP32_FAST", "FP64_FAST", "FP32_STRICT"):
    c3 = W.configs()["cfg3"]
    win = W.julia_window(960, 540)
    a = fr.julia_render_ex(c3.c, win, 960, 540, 1000, fr.Mode[mode])
    m = fr.mandelbrot_param_map(W.mandel_window(640, 360), 640, 360, 700, fr.Mode[mode])
    torch.cuda.synchronize()
    for t in (a, m):
        out.append(hashlib.sha256(t.view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:16])
print(" ".join(out))
"""


def test_fast_mode_identical_across_schedulers():
    """FAST modes are one arithmetic (the contracted doubled-state step), whichever kernel
    runs it: S/S2 (PTX vote loops), P1 + P2, R and A must give bit-identical counts for the
    same frame, not merely counts within reading c-10."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    hashes = {}
    for sched in ("static", "refill", "twophase", "twophase_exact", "twophase_p1a4",
                  "twophase_p1a8", "twophase_p1a8pre16", "amort"):
        # twophase: amortised P2 where the precondition holds; twophase_exact: P2 with
        # the per-iteration test; _p1aK: amortised P1 with sub-blocks of K
        e = dict(os.environ, FRACTAL_SCHED=sched.split("_")[0],
                 FRACTAL_P2_AMORT="0" if sched.endswith("exact") else "1")
        if "_p1a" in sched:
            e["FRACTAL_P1_AMORT"] = sched.split("_p1a")[1][0]
            if "pre" in sched:
                e["FRACTAL_P1_PRE"] = sched.split("pre")[1]
        r = subprocess.run([sys.executable, "-c", _HASH_SCRIPT], cwd=ROOT, env=e,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        hashes[sched] = r.stdout.split()
    ref = hashes["static"]
    for sched, h in hashes.items():
        assert h == ref, (sched, h, ref)


@pytest.mark.parametrize("env", [{"FRACTAL_SCHED": "twophase"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P2_AMORT": "0"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_BUDGET": "8",
                                  "FRACTAL_P2_OCC": "1"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P1_AMORT": "4"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P1_AMORT": "8"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P1_AMORT": "8",
                                  "FRACTAL_BUDGET": "8"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P1_AMORT": "4",
                                  "FRACTAL_P1_PRE": "8"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P1_AMORT": "8",
                                  "FRACTAL_P1_PRE": "16"},
                                 {"FRACTAL_VOTE_K": "4"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P1_AMORT": "0"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P1_TILES": "2"},
                                 {"FRACTAL_SCHED": "refill"}, {"FRACTAL_SCHED": "amort"},
                                 {"FRACTAL_SCHED": "static"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P2S": "1"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P2S": "1",
                                  "FRACTAL_P2S_K": "16"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P2S": "1",
                                  "FRACTAL_P2S_K": "64"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_P2S": "1",
                                  "FRACTAL_BUDGET": "8", "FRACTAL_P2_OCC": "1"}])
def test_fast_exact_under_forced_scheduler(env):
    """FAST counts equal the FAST oracle bit for bit under every kernel family, including
    P2 with the amortised block-end test and with the exact test."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest",
                        os.path.join(ROOT, "tests", "test_gpu_fast_exact.py"), "-m", "gpu", "-q",
                        "-x", "-k", "fast_configs or fast_fuzz or fast_mandelbrot or fast_nonmonotone",
                        "-p", "no:cacheprovider"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
