"""Every kernel family, whatever the default dispatch picks: a parity subset re-run in
subprocesses with FRACTAL_SCHED forced to static (kernel S), refill (kernel R), amort
(kernel A) and twophase (kernels P1 + P2, at several phase-1 budgets), and with the
persistent / CTA-local refill grids."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SUBSET = ("test_strict_configs_full_frame or test_strict_fuzz or test_strict_ragged or "
          "test_bands or test_max_iter_65535 or test_every_pixel or test_fast_mode_tolerance_julia")


@pytest.mark.parametrize("env", [{"FRACTAL_SCHED": "static"}, {"FRACTAL_SCHED": "refill"},
                                 {"FRACTAL_SCHED": "amort"}, {"FRACTAL_SCHED": "twophase"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_BUDGET": "4"},
                                 {"FRACTAL_SCHED": "twophase", "FRACTAL_BUDGET": "48",
                                  "FRACTAL_P2_OCC": "1"},
                                 {"FRACTAL_SCHED": "refill", "FRACTAL_REFILL_CPC": "16"},
                                 {"FRACTAL_SCHED": "amort", "FRACTAL_REFILL_CPC": "0"}])
def test_parity_under_forced_scheduler(env):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-m", "gpu", "-q", "-x", "-k", SUBSET, "-p", "no:cacheprovider"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
