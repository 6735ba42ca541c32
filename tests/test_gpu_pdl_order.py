"""Ordering of back-to-back single-frame calls: single-frame kernels are
launched with programmatic dependent launch, so the next call's CTAs compute while the
previous kernel finishes.  Whatever the overlap, stream order must hold for every memory
effect: after a run of calls into ONE buffer, the buffer holds exactly the last call's
frame (write-after-write), also when the footprint changes in between (other sizes,
Mandelbrot maps, strict frames through the same pointer), with fused colour, and inside
a CUDA graph."""
import numpy as np
import pytest

import oracle
from paper_1611_03079_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def fr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1611_03079_b200 import binding
    binding.load()
    return binding


def np16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


CS = [-0.7269 + 0.1889j, -0.8 + 0.156j, 0.285 + 0.01j, -0.4 + 0.6j, 0.0 + 0.0j]


def ref(c, w, h, mi):
    win = W.julia_window(w, h)
    return oracle.julia(c, win.center, win.half_w, win.half_h, w, h, mi, 32, fast=True)


@pytest.mark.parametrize("w,h", [(1920, 1080), (333, 97)])
def test_last_call_wins(fr, w, h):
    """200 calls alternating five C values into one buffer: it ends as the last frame."""
    win = W.julia_window(w, h)
    out = torch.empty((h, w), dtype=torch.uint16, device="cuda")
    for rep in range(3):
        order = [CS[(k * 3 + rep) % len(CS)] for k in range(200)]
        for c in order:
            fr.julia_render_ex(c, win, w, h, 100, fr.Mode.FP32_FAST, out=out)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(np16(out), ref(order[-1], w, h, 100))


def test_last_call_wins_with_colour(fr):
    w, h = 1920, 1080
    win = W.julia_window(w, h)
    pal = W.palette("fire")
    out = torch.empty((h, w), dtype=torch.uint16, device="cuda")
    rgba = torch.empty((h, w, 4), dtype=torch.uint8, device="cuda")
    order = [CS[k % 3] for k in range(100)] + [CS[4]]
    for c in order:
        fr.julia_render_ex(c, win, w, h, 100, fr.Mode.FP32_FAST, out=out, palette=pal,
                           out_rgba=rgba)
    torch.cuda.synchronize()
    r = ref(order[-1], w, h, 100)
    np.testing.assert_array_equal(np16(out), r)
    np.testing.assert_array_equal(rgba.cpu().numpy(), oracle.colorize(r, 100, *pal))


def test_footprint_changes_into_one_buffer(fr):
    """Frames of different sizes (and a Mandelbrot map, and a strict frame) written through
    the same base pointer, interleaved: every call's own region is exact at the end of its
    turn, and the final full-size frame covers everything."""
    big_w, big_h = 1280, 720
    base = torch.empty((big_h * big_w,), dtype=torch.uint16, device="cuda")
    sizes = [(1280, 720), (640, 360), (1280, 720), (1000, 500), (1280, 720)]
    for k in range(40):
        w, h = sizes[k % len(sizes)]
        out = base[:w * h].view(h, w)
        c = CS[k % len(CS)]
        if k % 7 == 3:
            mwin = W.mandel_window(w, h)
            fr.mandelbrot_param_map(mwin, w, h, 100, fr.Mode.FP32_FAST, out=out)
        else:
            mode = fr.Mode.FP32_STRICT if k % 5 == 2 else fr.Mode.FP32_FAST
            fr.julia_render_ex(c, W.julia_window(w, h), w, h, 100, mode, out=out)
    torch.cuda.synchronize()
    # last call: k = 39 -> sizes[4] = full frame, C = CS[4], fast
    np.testing.assert_array_equal(np16(base.view(big_h, big_w)), ref(CS[39 % len(CS)], big_w, big_h, 100))


def test_graph_of_alternating_frames(fr):
    """A CUDA graph of 30 alternating-C calls into one buffer (programmatic edges between
    the captured launches): each replay leaves the last call's frame."""
    w, h = 1920, 1080
    win = W.julia_window(w, h)
    out = torch.empty((h, w), dtype=torch.uint16, device="cuda")
    s = torch.cuda.Stream()
    order = [CS[k % 4] for k in range(29)] + [CS[4]]
    with torch.cuda.stream(s):
        for c in order[:3]:
            fr.julia_render_ex(c, win, w, h, 100, fr.Mode.FP32_FAST, out=out, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for c in order:
            fr.julia_render_ex(c, win, w, h, 100, fr.Mode.FP32_FAST, out=out, stream=s)
    want = ref(order[-1], w, h, 100)
    for _ in range(3):
        out.fill_(0)
        g.replay()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(np16(out), want)
    # an eager call after the replays, then the graph again
    fr.julia_render_ex(CS[0], win, w, h, 100, fr.Mode.FP32_FAST, out=out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(np16(out), ref(CS[0], w, h, 100))
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(np16(out), want)
