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
                 c: complex = 0j, mode=None, group=None, gather: bool = True, dst: int = 0):
    """Each rank renders its cyclic bands of a Julia ('julia') or Mandelbrot
    ('mandelbrot') frame; with gather=True the frame is assembled on dst."""
    from . import binding as fr
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bands = fr.Bands(band_rows, world, rank)
    if kind == "julia":
        mode = fr.Mode.FP32_FAST if mode is None else mode
        local = fr.julia_render_ex(c, win, width, height, max_iter, mode, bands)
    else:
        mode = fr.Mode.FP64_FAST if mode is None else mode
        local = fr.mandelbrot_param_map(win, width, height, max_iter, mode, bands)
    if not gather:
        return local
    return gather_bands(local, height, band_rows, dst, group)
