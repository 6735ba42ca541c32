"""The multi-GPU code path on the one GPU available: an NCCL process group of world
size 1 runs render_path_sharded / render_bands (partition + torch.distributed.gather
over NCCL with uint8 views) and must reproduce the single-call renders byte for byte.
World sizes > 1 are covered on CPU with gloo (tests/test_distributed.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    store = dist.TCPStore("127.0.0.1", _port(), 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def _np16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def test_render_path_sharded_nccl(nccl):
    from paper_1611_03079_b200 import binding as fr
    from paper_1611_03079_b200 import distributed as D
    from paper_1611_03079_b200 import workloads as W
    cs = W.circle_path(24)
    win = W.julia_window(320, 180)
    full = D.render_path_sharded(cs, win, 320, 180, 100, fr.Mode.FP32_STRICT)
    ref = fr.julia_render_path(cs, win, 320, 180, 100, fr.Mode.FP32_STRICT)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_np16(full), _np16(ref))


@pytest.mark.parametrize("kind", ["julia", "mandelbrot"])
def test_render_bands_nccl(nccl, kind):
    from paper_1611_03079_b200 import binding as fr
    from paper_1611_03079_b200 import distributed as D
    from paper_1611_03079_b200 import workloads as W
    w, h = 480, 270
    win = W.julia_window(w, h) if kind == "julia" else W.mandel_window(w, h)
    img = D.render_bands(kind, win, w, h, 300, 15, c=-0.7269 + 0.1889j)
    if kind == "julia":
        ref = fr.julia_render_ex(-0.7269 + 0.1889j, win, w, h, 300, fr.Mode.FP32_FAST)
    else:
        ref = fr.mandelbrot_param_map(win, w, h, 300, fr.Mode.FP64_FAST)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_np16(img), _np16(ref))


@pytest.mark.parametrize("chunk", [1, 5, 64])
def test_deliver_path_nccl(nccl, chunk):
    """Pipelined render + gather (distributed.deliver_path) on the real renderer: the
    delivered frames equal one julia_render_path call (uint8 counts), ragged last chunk
    included."""
    from paper_1611_03079_b200 import binding as fr
    from paper_1611_03079_b200 import distributed as D
    from paper_1611_03079_b200 import workloads as W
    cs = W.circle_path(23)
    win = W.julia_window(320, 180)
    got = D.deliver_path(cs, win, 320, 180, 100, fr.Mode.FP32_STRICT, chunk=chunk)
    ref = fr.julia_render_path(cs, win, 320, 180, 100, fr.Mode.FP32_STRICT,
                               out=torch.empty((23, 180, 320), dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.to_path_order().cpu().numpy(), ref.cpu().numpy())
    for k in (0, 11, 22):
        np.testing.assert_array_equal(got.frame(k).cpu().numpy(), ref[k].cpu().numpy())


def test_render_bands_with_palette_nccl(nccl):
    """cfg3-style bands with the fused palette (BASELINE configs[2]: "fp32 + fused
    colorize, row bands"): counts and RGBA gathered equal one full render."""
    from paper_1611_03079_b200 import binding as fr
    from paper_1611_03079_b200 import distributed as D
    from paper_1611_03079_b200 import workloads as W
    w, h, br = 640, 361, 15
    win = W.julia_window(w, h)
    pal = W.palette("classic")
    c = -0.7269 + 0.1889j
    counts, rgba = D.render_bands("julia", win, w, h, 1000, br, c=c, mode=fr.Mode.FP32_FAST,
                                  palette=pal)
    full, full_rgba = fr.julia_render_ex(c, win, w, h, 1000, fr.Mode.FP32_FAST, palette=pal)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_np16(counts), _np16(full))
    np.testing.assert_array_equal(rgba.cpu().numpy(), full_rgba.cpu().numpy())


def test_bench_exchange_branches_at_n1():
    """bench.py --force-exchange runs the N > 1 measurements (plain gather, pipelined
    delivery, cfg3/cfg5 row bands) over an NCCL group of one: every branch reports
    without an `error` key (BASELINE configs[2..4])."""
    import json
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "2",
                        "--warmup", "3", "--no-extra", "--cpu-seconds", "0.5",
                        "--force-exchange"], cwd=root, env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("gather_to_rank0", "delivered_to_rank0", "bands"):
        assert key in line, key
    assert "error" not in line["gather_to_rank0"], line["gather_to_rank0"]
    assert "error" not in line["delivered_to_rank0"], line["delivered_to_rank0"]
    for name in ("cfg3", "cfg5"):
        assert "error" not in line["bands"][name], line["bands"][name]
    assert line["bands"]["cfg3"]["colour"] == "fused classic palette"
