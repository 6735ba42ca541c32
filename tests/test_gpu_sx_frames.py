"""Kernel SX's frame loop: the frame-independent first iteration
hoisted out of the frame loop (sx_pre), the uint16 frame loop as one PTX block with the
chunk's C values staged in shared memory (sx_frames_u16), and the host's VEC choice.
Every frame is compared with the FAST oracle, bit for bit, at the edges of that code:
iteration limits around the vote block (1, 2, 3, 4, odd and even), paths longer than one
shared-memory chunk (128 frames) with frame groups that end inside a chunk, odd widths
(no VEC) and pixels outside the frame."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_1611_03079_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1611_03079_b200 import binding
    binding.load()
    return binding


def _check_path(fr, cs, w, h, mi):
    win = W.julia_window(w, h)
    out = fr.julia_render_path(cs, win, w, h, mi, fr.Mode.FP32_FAST)
    torch.cuda.synchronize()
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    for k in range(len(cs)):
        ref = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, w, h, mi, 32,
                           fast=True)
        np.testing.assert_array_equal(got[k], ref, err_msg=f"frame {k} mi {mi} {w}x{h}")


@pytest.mark.parametrize("mi", [1, 2, 3, 4, 5, 100, 101, 256])
@pytest.mark.parametrize("w,h", [(64, 8), (66, 10), (63, 9)])
def test_sx_iteration_limits(fr, mi, w, h):
    """max_iter 1 (no vote block: the scalar tail), 2 (the hoisted block only), odd limits
    (tail after the vote loop), even limits (PTX frame loop); even and odd widths."""
    _check_path(fr, W.circle_path(19), w, h, mi)


_CHUNK_SCRIPT = r"""
import sys
import numpy as np, torch
import oracle
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
n, w, h, mi = 300, 34, 6, 60
cs = W.circle_path(n)
win = W.julia_window(w, h)
out = fr.julia_render_path(cs, win, w, h, mi, fr.Mode.FP32_FAST)
torch.cuda.synchronize()
got = out.view(torch.int16).cpu().numpy().view(np.uint16)
bad = [k for k in range(n) if not np.array_equal(
    got[k], oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, w, h, mi, 32,
                         fast=True))]
print("BAD", bad[:10])
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("fpc", ["1", "3", "127", "128", "129", "300"])
def test_sx_frame_groups_and_chunks(fpc):
    """Frames per CTA (FRACTAL_FPC) below, at and above the 128-frame shared-memory chunk
    of the PTX frame loop, and groups that end inside a chunk: all 300 frames exact."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    e = dict(os.environ, FRACTAL_FPC=fpc)
    r = subprocess.run([sys.executable, "-c", _CHUNK_SCRIPT], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
