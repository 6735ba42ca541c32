"""Multi-GPU partitioning of the escape-time path, one process per GPU.

Frames of a C-path and row bands of a frame are independent, so every rank renders
its own share with no data-path collective:

* frames: cyclic, frame k -> rank k % world (balanced: per-frame work varies ~10x along
  the |C| = 0.7885 circle; contiguous blocks were measured 1.74x imbalanced);
* bands: cyclic bands of `band_rows` rows, global band b -> rank b % world, rendered
  with GLOBAL row indices so band pixels are bit-identical to the full frame
  (`fr_bands` in include/fractal.h).

The one exchange step -- delivering the frames/bands to rank 0 -- is a
`torch.distributed.gather` (NCCL over NVLink/NVSwitch on the GPU box, gloo in the CPU
tests).  NCCL has no 16-bit integer type, so tensors travel as uint8 views; every
rank contributes the same padded size.
"""
from __future__ import annotations

import contextlib
import math

import numpy as np
import torch
import torch.distributed as dist


# --------------------------------------------------------------------------- partition
def frame_indices(n_frames: int, world: int, rank: int) -> np.ndarray:
    """Frames rendered by `rank`: k = rank, rank + world, ... (cyclic)."""
    return np.arange(rank, n_frames, world, dtype=np.int64)


def frames_per_rank(n_frames: int, world: int) -> int:
    return math.ceil(n_frames / world)


def band_rows_of(height: int, band_rows: int, world: int, rank: int) -> np.ndarray:
    """Global rows held by `rank` under cyclic bands (same rule as fr_band_global_row)."""
    if band_rows <= 0:
        return np.arange(height) if rank == 0 else np.arange(0)
    rows = []
    for b in range(rank, math.ceil(height / band_rows), world):
        rows.append(np.arange(b * band_rows, min((b + 1) * band_rows, height)))
    return np.concatenate(rows) if rows else np.arange(0)


def max_band_rows(height: int, band_rows: int, world: int) -> int:
    return max(len(band_rows_of(height, band_rows, world, r)) for r in range(world))


# --------------------------------------------------------------------------- assembly
_VIEW = {torch.uint16: torch.int16, torch.uint32: torch.int32}  # index_put lacks uints


def _iv(t: torch.Tensor) -> torch.Tensor:
    return t.view(_VIEW[t.dtype]) if t.dtype in _VIEW else t


def assemble_frames(parts, n_frames: int):
    """parts[r] = rank r's frames (padded to ceil(n/world)) -> frames in path order."""
    world = len(parts)
    per = parts[0].shape[0]
    out = parts[0].new_empty((n_frames,) + tuple(parts[0].shape[1:]))
    for r, p in enumerate(parts):
        k = frame_indices(n_frames, world, r)
        _iv(out)[torch.as_tensor(k, device=out.device)] = _iv(p)[: len(k)]
    assert per >= frames_per_rank(n_frames, world)
    return out


def assemble_bands(parts, height: int, band_rows: int):
    """parts[r] = rank r's band rows (padded) -> the full frame."""
    world = len(parts)
    out = parts[0].new_empty((height,) + tuple(parts[0].shape[1:]))
    for r, p in enumerate(parts):
        rows = band_rows_of(height, band_rows, world, r)
        if len(rows):
            _iv(out)[torch.as_tensor(rows, device=out.device)] = _iv(p)[: len(rows)]
    return out


# --------------------------------------------------------------------------- collectives
def _as_bytes(t: torch.Tensor) -> torch.Tensor:
    return t.contiguous().view(torch.uint8)


def gather_padded(local: torch.Tensor, rows: int, dst: int = 0, group=None):
    """Pad `local` ([n, ...]) to `rows` leading entries and gather to dst.
    Returns the list of per-rank tensors on dst, None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    pad = local.new_zeros((rows,) + tuple(local.shape[1:]))
    if local.shape[0]:
        _iv(pad)[: local.shape[0]] = _iv(local)
    send = _as_bytes(pad)
    if rank == dst:
        recv = [torch.empty_like(send) for _ in range(world)]
        dist.gather(send, gather_list=recv, dst=dst, group=group)
        return [r.view(local.dtype).view(pad.shape) for r in recv]
    dist.gather(send, dst=dst, group=group)
    return None


def gather_frames(local: torch.Tensor, n_frames: int, dst: int = 0, group=None):
    """Rank-local cyclic frames -> all frames in path order on dst (None elsewhere)."""
    world = dist.get_world_size(group)
    parts = gather_padded(local, frames_per_rank(n_frames, world), dst, group)
    return assemble_frames(parts, n_frames) if parts is not None else None


def gather_bands(local: torch.Tensor, height: int, band_rows: int, dst: int = 0, group=None):
    """Rank-local cyclic bands -> the full frame on dst (None elsewhere)."""
    world = dist.get_world_size(group)
    parts = gather_padded(local, max_band_rows(height, band_rows, world), dst, group)
    return assemble_bands(parts, height, band_rows) if parts is not None else None


# --------------------------------------------------------------------------- pipelined delivery
class Delivered:
    """Frames delivered to rank dst by `deliver_path`: the receive buffer
    [n_chunks, world, chunk, H, W] as NCCL filled it.  Frame k (path order) is
    buf[j, r, i] with r = k % world and k // world = j * chunk + i, so path order is the
    zero-copy view buf.permute(0, 2, 1, 3, 4) ("rank 0 un-interleaves with
    a view or one HBM-bound copy")."""

    def __init__(self, buf: torch.Tensor, n_frames: int, world: int, chunk: int):
        self.buf, self.n_frames, self.world, self.chunk = buf, n_frames, world, chunk

    def frame(self, k: int) -> torch.Tensor:
        idx, r = divmod(k, self.world)
        j, i = divmod(idx, self.chunk)
        return self.buf[j, r, i]

    def path_view(self) -> torch.Tensor:
        """[n_chunks, chunk, world, H, W] view whose flattening is path order (padded)."""
        return self.buf.permute(0, 2, 1, 3, 4)

    def to_path_order(self) -> torch.Tensor:
        """The frames in path order as one contiguous tensor (one HBM-bound copy)."""
        v = self.path_view()
        return v.reshape((-1,) + tuple(v.shape[3:]))[: self.n_frames]


def deliver_path(cs, win, width: int, height: int, max_iter: int = 100, mode=None,
                 chunk: int = 64, dst: int = 0, group=None, dtype=torch.uint8, render=None,
                 device=None):
    """Render this rank's cyclic frames of the path in chunks of `chunk` frames and
    gather every chunk to `dst` while the next chunk renders (SURVEY §8(e) plan 1):
    render on the current stream into one of two buffers, gather on a separate
    communication stream; a buffer is rendered again only after its previous gather
    finished (CUDA events).  uint8 counts (max_iter <= 255) halve the bytes on the wire.

    `render(cs_chunk, out)` fills out[:len(cs_chunk)] (default: libfractal's
    julia_render_path on `out`'s device); the CPU tests pass a synthetic one under gloo.
    Returns a `Delivered` on dst, None elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cs = np.asarray(cs, dtype=np.complex128).reshape(-1)
    n = len(cs)
    if dtype == torch.uint8 and max_iter > 255:
        raise ValueError("uint8 delivery needs max_iter <= 255")
    if render is None:
        from . import binding as fr
        md = fr.Mode.FP32_FAST if mode is None else mode

        def render(c, out):
            fr.julia_render_path(c, win, width, height, max_iter, md, out=out)
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device("cpu") if device is None else torch.device(device)
    k_local = frame_indices(n, world, rank)
    n_chunks = max(1, math.ceil(frames_per_rank(n, world) / chunk))
    bufs = [torch.zeros((chunk, height, width), dtype=dtype, device=device) for _ in range(2)]
    recv = (torch.empty((n_chunks, world, chunk, height, width), dtype=dtype, device=device)
            if rank == dst else None)
    cuda = device.type == "cuda"
    comp = torch.cuda.current_stream(device) if cuda else None
    comm = torch.cuda.Stream(device) if cuda else None
    done = [None, None]
    for j in range(n_chunks):
        b = j % 2
        lo, hi = j * chunk, min((j + 1) * chunk, len(k_local))
        if cuda and done[b] is not None:
            comp.wait_event(done[b])
        if hi > lo:
            render(cs[k_local[lo:hi]], bufs[b][: hi - lo])
        if cuda:
            ready = torch.cuda.Event()
            ready.record(comp)
            comm.wait_event(ready)
        with torch.cuda.stream(comm) if cuda else contextlib.nullcontext():
            send = bufs[b].reshape(-1).view(torch.uint8)
            if rank == dst:
                gl = [recv[j, r].reshape(-1).view(torch.uint8) for r in range(world)]
                dist.gather(send, gather_list=gl, dst=dst, group=group)
            else:
                dist.gather(send, dst=dst, group=group)
            if cuda:
                done[b] = torch.cuda.Event()
                done[b].record(comm)
    if cuda:
        comp.wait_stream(comm)
    return Delivered(recv, n, world, chunk) if rank == dst else None


# --------------------------------------------------------------------------- GPU renders
def render_path_sharded(cs, win, width: int, height: int, max_iter: int = 100, mode=None,
                        group=None, gather: bool = True, dst: int = 0):
    """Each rank renders frames k = rank (mod world) of the path with libfractal; with
    gather=True the frames are delivered to dst in path order."""
    from . import binding as fr
    mode = fr.Mode.FP32_FAST if mode is None else mode
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cs = np.asarray(cs, dtype=np.complex128)
    k = frame_indices(len(cs), world, rank)
    local = torch.empty((len(k), height, width), dtype=torch.uint16, device="cuda")
    if len(k):
        fr.julia_render_path(cs[k], win, width, height, max_iter, mode, out=local)
    if not gather:
        return local
    return gather_frames(local, len(cs), dst, group)


def render_bands(kind: str, win, width: int, height: int, max_iter: int, band_rows: int,
                 c: complex = 0j, mode=None, group=None, gather: bool = True, dst: int = 0,
                 palette=None):
    """Each rank renders its cyclic bands of a Julia ('julia') or Mandelbrot
    ('mandelbrot') frame, with the colour levels fused when `palette` is given (cfg3:
    "fp32 + fused colorize, row bands"); with gather=True the frame (and its RGBA image)
    is assembled on dst.  Returns counts, or (counts, rgba) with a palette; None for
    both on ranks other than dst when gathering."""
    from . import binding as fr
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bands = fr.Bands(band_rows, world, rank)
    if kind == "julia":
        mode = fr.Mode.FP32_FAST if mode is None else mode
        local = fr.julia_render_ex(c, win, width, height, max_iter, mode, bands,
                                   palette=palette)
    else:
        mode = fr.Mode.FP64_FAST if mode is None else mode
        local = fr.mandelbrot_param_map(win, width, height, max_iter, mode, bands,
                                        palette=palette)
    if not gather:
        return local
    if palette is None:
        return gather_bands(local, height, band_rows, dst, group)
    counts = gather_bands(local[0], height, band_rows, dst, group)
    rgba = gather_bands(local[1], height, band_rows, dst, group)
    return (counts, rgba) if counts is not None else (None, None)
