"""Multi-rank partition + gather logic on CPU (gloo, world size 2 and 3), and the
pure partition/assembly functions against the band/frame definitions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_03079_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,world", [(4096, 8), (10, 3), (7, 2), (1, 4), (0, 2)])
def test_frame_partition_covers_path(n, world):
    allk = np.concatenate([D.frame_indices(n, world, r) for r in range(world)])
    assert sorted(allk.tolist()) == list(range(n))
    assert max(len(D.frame_indices(n, world, r)) for r in range(world)) == D.frames_per_rank(n, world)


@pytest.mark.parametrize("h,br,world", [(2160, 15, 8), (16384, 16, 8), (1081, 16, 8), (7, 3, 4), (5, 16, 2)])
def test_band_partition_covers_frame(h, br, world):
    rows = np.concatenate([D.band_rows_of(h, br, world, r) for r in range(world)])
    assert sorted(rows.tolist()) == list(range(h))
    for r in range(world):
        rr = D.band_rows_of(h, br, world, r)
        assert all((x // br) % world == r for x in rr)  # cyclic rule


def test_assemble_roundtrip_single_process():
    frames = torch.arange(11 * 3 * 2, dtype=torch.int16).view(11, 3, 2)
    world = 3
    per = D.frames_per_rank(11, world)
    parts = []
    for r in range(world):
        k = D.frame_indices(11, world, r)
        p = torch.zeros((per, 3, 2), dtype=torch.int16)
        p[: len(k)] = frames[torch.as_tensor(k)]
        parts.append(p)
    assert torch.equal(D.assemble_frames(parts, 11), frames)
    img = torch.arange(37 * 5, dtype=torch.int16).view(37, 5)
    mx = D.max_band_rows(37, 4, world)
    parts = []
    for r in range(world):
        rows = D.band_rows_of(37, 4, world, r)
        p = torch.zeros((mx, 5), dtype=torch.int16)
        p[: len(rows)] = img[torch.as_tensor(rows)]
        parts.append(p)
    assert torch.equal(D.assemble_bands(parts, 37, 4), img)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # frames: rank-local cyclic frames tagged with their global index (uint16 as int16 view)
        n = 13
        k = D.frame_indices(n, world, rank)
        local = torch.stack([torch.full((4, 6), int(i) * 7 + 1, dtype=torch.int16) for i in k]) \
            if len(k) else torch.empty((0, 4, 6), dtype=torch.int16)
        full = D.gather_frames(local.view(torch.uint16), n)
        # bands: rank-local rows tagged with their global row
        h, br = 29, 4
        rows = D.band_rows_of(h, br, world, rank)
        bl = torch.tensor(rows, dtype=torch.int16)[:, None].repeat(1, 5) if len(rows) else \
            torch.empty((0, 5), dtype=torch.int16)
        img = D.gather_bands(bl.view(torch.uint16), h, br)
        if rank == 0:
            ok_f = torch.equal(full.view(torch.int16),
                               torch.stack([torch.full((4, 6), i * 7 + 1, dtype=torch.int16) for i in range(n)]))
            ok_b = torch.equal(img.view(torch.int16),
                               torch.arange(h, dtype=torch.int16)[:, None].repeat(1, 5))
            q.put((ok_f, ok_b))
        else:
            assert full is None and img is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_frames_and_bands_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ok_f, ok_b = q.get(timeout=10)
    assert ok_f and ok_b


def _deliver_worker(rank, world, port, q, n, chunk, dtype):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cs = np.arange(n, dtype=np.float64) + 0j  # C_k = k tags the frame

        def render(c, out):  # frame k -> every pixel (7k + 1) mod 251, rank-local shape
            v = torch.as_tensor((7 * np.real(c).astype(np.int64) + 1) % 251, dtype=out.dtype)
            out[: len(c)] = v[:, None, None]

        got = D.deliver_path(cs, None, 5, 3, 100, chunk=chunk, render=render, dtype=dtype)
        if rank == 0:
            want = torch.stack([torch.full((3, 5), (7 * k + 1) % 251, dtype=dtype) for k in range(n)])
            ok = torch.equal(got.to_path_order(), want) and all(
                torch.equal(got.frame(k), want[k]) for k in range(n))
            q.put(ok)
        else:
            assert got is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,chunk,dtype", [(2, 13, 2, torch.uint8), (3, 13, 4, torch.int16),
                                                 (2, 3, 8, torch.uint8), (3, 2, 1, torch.uint8)])
def test_deliver_path_pipelined_gloo(world, n, chunk, dtype):
    """Chunked render + gather to rank 0 (SURVEY §8(e) plan 1): every frame arrives, in
    path order through the zero-copy view, including ranks with no frames and ragged
    last chunks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_deliver_worker, args=(r, world, port, q, n, chunk, dtype))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10)
