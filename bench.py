#!/usr/bin/env python
"""Benchmark of the escape-time hot path (arXiv 1611.03079) on 1..8 B200s.

Workload (BASELINE.json configs[3], weak-scaled): the C-path sweep of 1080p Julia
frames (1920x1080, max_iter 100, FP32 fast mode) with C on |C| = 0.7885.  At N GPUs
the path has F = 512*N frames, th_k = 2 pi k / F, and frame k is rendered by rank
k mod N (cyclic frames, no data-path collective); every rank renders 512 frames per
step, so at N = 8 one step is exactly configs[3] (4096 frames).  A step = one pass of
the whole hot path over the rank's batch: parameter derivation, region-covering map,
escape-time iteration, uint16 count store, frame loop (one julia_render_path call).

Metric: Gpixel-iter/s = sum of escape counts / time (BASELINE.json metric), whole job;
1080p frames/s is reported beside it.  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

FRAMES_PER_RANK = 512
W_PX, H_PX, MAX_ITER = 1920, 1080, 100
RADIUS = 0.7885
SM_COUNT, FP32_LANES_PER_SM, FP64_LANES_PER_SM = 148, 128, 64
ALG_OPS_PER_ITER = 4  # FMA-pipe ops per pixel-iteration, algorithmic minimum
SURVEY_OPS_PER_ITER = 6  # SURVEY §8(d)'s per-unit figure (per-iteration test included)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def path_for(world: int, rank: int):
    from paper_1611_03079_b200 import workloads as W
    full = W.circle_path(FRAMES_PER_RANK * world, RADIUS)
    return full[rank::world]


def arm_config(world: int, mode: str = "FP32_FAST") -> dict:
    """The workload both arms report (ours and --impl reference; the reference arm times
    the strict oracle and says so in `mode`)."""
    return {"workload": "cfg4 C-path sweep (BASELINE configs[3]), weak-scaled: "
                        f"{FRAMES_PER_RANK} frames/GPU, F={FRAMES_PER_RANK}*N frames "
                        "on |C|=0.7885, frame k -> rank k mod N",
            "width": W_PX, "height": H_PX, "max_iter": MAX_ITER, "mode": mode,
            "frames_per_step": FRAMES_PER_RANK * world, "parallelism": f"frames{world}",
            "l2": f"output {FRAMES_PER_RANK * W_PX * H_PX * 2 / 1e9:.2f} GB per step per "
                  "GPU (> 126 MB L2), no L2 reuse between steps"}


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons DURING the timed region via NVML (every
    ~10 ms; the B200_PROFILING.md clocks line, without nvidia-smi's 100 ms floor)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, period_s: float = 0.01):
        self.index = index
        self.period = period_s
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self._nvml = None
        return self

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            self._stop.wait(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._nvml is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0}
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm for sm, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "source": "NVML, 10 ms"}


# --------------------------------------------------------------------------- CPU oracle
def cpu_oracle_rate(cs, seconds: float = 12.0, threads: int | None = None):
    """The oracle as it stands (strict, plain C, all host cores) on a bounded sample of
    the same workload: whole frames of the rank's path until ~`seconds` elapse."""
    import oracle
    from paper_1611_03079_b200 import workloads as W
    win = W.julia_window(W_PX, H_PX)
    threads = threads or oracle.default_threads()
    order = np.random.default_rng(0).permutation(len(cs))
    total, frames, t0 = 0, 0, time.perf_counter()
    for k in order:
        g = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, W_PX, H_PX,
                         MAX_ITER, 32, threads)
        total += int(g.sum(dtype=np.int64))
        frames += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    res = {"value": total / dt / 1e9, "unit": "Gpixel-iter/s", "cores": threads,
           "kind": "oracle", "frames_per_s": frames / dt,
           "sample": f"{frames} of the {len(cs)} rank-0 1080p frames (random order), strict "
                     f"fp32 scalar C oracle, {threads} threads, {dt:.1f} s"}
    if threads > 1:
        # also once on one core (same frames, ~1/4 of the time budget)
        t1, tot1, fr1 = time.perf_counter(), 0, 0
        for k in order:
            g = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, W_PX, H_PX,
                             MAX_ITER, 32, 1)
            tot1 += int(g.sum(dtype=np.int64))
            fr1 += 1
            if time.perf_counter() - t1 >= seconds / 4:
                break
        d1 = time.perf_counter() - t1
        res["one_core"] = {"value": tot1 / d1 / 1e9, "frames": fr1, "seconds": round(d1, 2)}
    try:
        res["cpu_model"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                                if l.startswith("model name"))
    except Exception:
        pass
    return res


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    if rank != 0:
        return 0
    import oracle
    from paper_1611_03079_b200 import workloads as W
    cs = path_for(world, 0)
    win = W.julia_window(W_PX, H_PX)
    threads = oracle.default_threads()
    per_step = 2  # frames of the rank-0 batch per step (bounded sample)
    order = np.random.default_rng(0).permutation(len(cs))

    def step(i):
        s = 0
        for j in range(per_step):
            k = order[(i * per_step + j) % len(order)]
            g = oracle.julia(complex(cs[k]), win.center, win.half_w, win.half_h, W_PX, H_PX,
                             MAX_ITER, 32, threads)
            s += int(g.sum(dtype=np.int64))
        return s

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    total = 0
    for i in range(args.steps):
        total += step(args.warmup + i)
    dt = time.perf_counter() - t0
    v = total / dt / 1e9
    line = {
        "impl": "reference", "metric": "Gpixel-iter/s", "value": v, "unit": "Gpixel-iter/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": arm_config(world, "FP32_STRICT_ORACLE"),
        "reference_sample": f"each step renders {per_step} random frames of the rank-0 batch "
                            "of this workload (bounded sample); the rate is per pixel-iteration",
        "cpu_baseline": {"value": v, "unit": "Gpixel-iter/s", "cores": threads, "kind": "oracle",
                         "sample": f"{per_step} random frames of the rank-0 batch per step, "
                                   f"strict fp32 scalar C oracle on {threads} threads"},
        "e2e": {"value": v, "unit": "Gpixel-iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip the per-config extras")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--force-exchange", action="store_true",
                    help="run the N > 1 exchange measurements (gather, pipelined delivery, "
                         "row bands) even at N = 1, over an NCCL group of one")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    exchange = world > 1 or args.force_exchange
    if exchange:
        if world == 1:  # a process group of one (no torchrun): local rendezvous
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1611_03079_b200 import binding as fr
    from paper_1611_03079_b200 import workloads as W

    fr.load()
    win = W.julia_window(W_PX, H_PX)
    cs = path_for(world, rank)
    nf = len(cs)
    out = torch.empty((nf, H_PX, W_PX), dtype=torch.uint16, device="cuda")
    stream = torch.cuda.current_stream()
    mode = fr.Mode.FP32_FAST

    def step():
        fr.julia_render_path(cs, win, W_PX, H_PX, MAX_ITER, mode, out=out, stream=stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    iters_per_step = int((out.view(torch.int16).to(torch.int64) & 0xFFFF).sum().item())
    barrier()

    # ---- timed region: K steps, per-launch CUDA events on the launching stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    l0 = fr.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        t_end.record(stream)
        barrier()
    launches = fr.launch_count() - l0
    elapsed_ms = t_start.elapsed_time(t_end)
    kernel_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    clocks = clk.summary()

    total_iters = iters_per_step * args.steps
    tot = torch.tensor([float(total_iters)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    job_iters = float(tot.item())
    value = job_iters / (elapsed_ms * 1e-3) / 1e9
    frames_per_s = nf * world * args.steps / (elapsed_ms * 1e-3)

    # ---- roofline of the dominant (only) kernel: escape_tile_kernel
    peaks = measured_peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak_gpix = SM_COUNT * FP32_LANES_PER_SM * f_max * 1e6 / ALG_OPS_PER_ITER / 1e9
    kavg = statistics.mean(kernel_ms)
    achieved = iters_per_step / (kavg * 1e-3) / 1e9
    roof = {"bound": "alu", "achieved": achieved, "peak": peak_gpix, "unit": "Gpixel-iter/s",
            "frac": achieved / peak_gpix, "traffic": None,
            "kernel": "fr::escape_pathx_kernel<1024,2,false,true> (SX: C-path frames, FP32_FAST, PTX frame loop)",
            "peak_basis": f"{SM_COUNT} SMs x {FP32_LANES_PER_SM} FP32 lanes x {f_max:.0f} MHz "
                          f"(MEASURED_PEAKS.json sm_max_mhz) / {ALG_OPS_PER_ITER} FMA-pipe ops "
                          "per pixel-iteration (DESIGN.md §5)",
            "frac_6op_survey": achieved * SURVEY_OPS_PER_ITER / ALG_OPS_PER_ITER / peak_gpix,
            "frac_6op": achieved * SURVEY_OPS_PER_ITER / ALG_OPS_PER_ITER / peak_gpix,
            "kernel_ms_avg": kavg}
    if clocks.get("sm_mhz"):
        roof["frac_at_measured_clock"] = achieved / (peak_gpix * clocks["sm_mhz"] / f_max)
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        try:
            roof["traffic"] = json.load(open(traffic_file)).get("bench_kernel_dram_bytes")
        except Exception:
            pass

    line = None
    if rank == 0:
        line = {
            "metric": "Gpixel-iter/s", "value": value, "unit": "Gpixel-iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": arm_config(world),
            "frames_per_s": frames_per_s,
            "pixel_iters_per_step": job_iters / args.steps,
            "gpu_launches": int(launches),
            "parity": {"strict": "bit-exact vs the CPU oracle (tests -m gpu)",
                       "fast": "bit-exact vs the FAST oracle (the doubled FMA sequence, "
                               "DESIGN.md reading c-10)",
                       "north_star_fast_clause": "not met literally: '<= 1e-4 of pixels "
                               "differ from strict' is unattainable for any FMA "
                               "implementation on cfg1-3/5 (SURVEY c-10); replaced by "
                               "reading c-10's bound max(1e-4, 4 x the 1-ulp "
                               "sensitivity) + one-pixel-of-a-boundary rule"},
            "clocks": clocks,
            "roofline": roof,
        }
    # ---- the exchange step (N > 1): NCCL gather of every rank's frames to rank 0, plain
    # (after the render) and pipelined with the render (chunked, separate stream)
    gather = measure_gather(out, world, rank, barrier) if exchange else None
    delivered = (measure_delivered(win, world, rank, barrier, job_iters / args.steps)
                 if exchange else None)
    # ---- row bands over the ranks (cfg3 and cfg5 as cyclic bands)
    bands = (measure_bands(world, rank, barrier)
             if exchange and (not args.no_extra or args.force_exchange) else None)
    # ---- end-to-end through the public API with HOST buffers (pinned), N GPUs
    e2e = measure_e2e(fr, W, cs, win, world, args, barrier, stream)
    if rank == 0:
        line["e2e"] = e2e
        if gather is not None:
            line["gather_to_rank0"] = gather
        if delivered is not None:
            line["delivered_to_rank0"] = delivered
        if bands is not None:
            line["bands"] = bands
        if world == 1:
            line["cpu_baseline"] = cpu_oracle_rate(cs, seconds=args.cpu_seconds)
            if not args.no_extra:
                line["configs"] = extras(fr, W, torch)
        print(json.dumps(line), flush=True)
    if exchange:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def measure_gather(out, world, rank, barrier):
    """Time the delivery of all ranks' frames to rank 0 (torch.distributed.gather over
    NCCL; paper_1611_03079_b200.distributed.gather_padded), max over ranks.  Reported
    beside, not inside, the compute-resident `value`."""
    import torch
    import torch.distributed as dist
    from paper_1611_03079_b200 import distributed as D
    try:
        reps = 2
        D.gather_padded(out, out.shape[0], 0)  # warm-up (NCCL communicator set-up)
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(reps):
            parts = D.gather_padded(out, out.shape[0], 0)
            del parts
        t1.record()
        barrier()
        ms = t0.elapsed_time(t1) / reps
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        nbytes = out.numel() * out.element_size() * (world - 1)
        return {"ms": ms, "bytes_into_rank0": nbytes, "GB_per_s": nbytes / (ms * 1e-3) / 1e9,
                "note": "uint16 frames of ranks 1..N-1 to rank 0 (NCCL gather, uint8 view); "
                        "the rank-0 ingress bound is ~0.77-0.9 TB/s (B200_PROFILING.md)"}
    except Exception as e:  # report, never fail the bench line
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def measure_delivered(win, world, rank, barrier, job_iters_per_step, chunk=64):
    """Frames delivered to rank 0 with the render and the gather pipelined
    (distributed.deliver_path: chunks of `chunk` frames per rank, uint8 counts, gather on
    its own stream overlapping the next chunk's render), max over ranks -- the second
    frames/s figure of SURVEY §8(e) next to the compute-resident `value`."""
    import torch
    import torch.distributed as dist
    from paper_1611_03079_b200 import distributed as D
    from paper_1611_03079_b200 import workloads as W
    try:
        full = W.circle_path(FRAMES_PER_RANK * world, RADIUS)
        got = D.deliver_path(full, win, W_PX, H_PX, MAX_ITER, chunk=chunk)  # warm-up
        del got
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        got = D.deliver_path(full, win, W_PX, H_PX, MAX_ITER, chunk=chunk)
        t1.record()
        barrier()
        del got
        t = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        nbytes = FRAMES_PER_RANK * W_PX * H_PX * (world - 1)
        return {"ms": ms, "frames_per_s": len(full) / (ms * 1e-3),
                "gpix_iter_s": job_iters_per_step / (ms * 1e-3) / 1e9,
                "bytes_into_rank0": nbytes, "ingress_GB_per_s": nbytes / (ms * 1e-3) / 1e9,
                "chunk_frames_per_rank": chunk, "dtype": "u8",
                "note": "render + NCCL gather to rank 0 pipelined per chunk (separate stream); "
                        "frames land in rank 0's buffer, path order is a zero-copy view"}
    except Exception as e:  # report, never fail the bench line
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def measure_bands(world, rank, barrier):
    """cfg3 (4K Julia, mi 1000, fp32 fast, fused colour levels) and cfg5 (16384^2
    Mandelbrot, mi 10000, fp64 fast) as cyclic row bands over the ranks (band_rows 15
    and 16): the compute makespan (max over ranks of each rank's render) and the NCCL
    gather of the bands to rank 0 (distributed.gather_bands; cfg3: counts and RGBA),
    timed separately with CUDA events."""
    import torch
    import torch.distributed as dist
    from paper_1611_03079_b200 import binding as fr
    from paper_1611_03079_b200 import distributed as D
    from paper_1611_03079_b200 import workloads as W
    out = {}
    for name, reps in (("cfg3", 20), ("cfg5", 1)):
        try:
            c = W.configs()[name]
            pal = W.palette("classic") if c.colorize else None
            if c.kind == "julia":
                mode = fr.Mode.FP32_FAST

                def render():
                    return D.render_bands("julia", c.window, c.width, c.height, c.max_iter,
                                          c.band_rows, c=c.c, mode=mode, gather=False,
                                          palette=pal)
            else:
                mode = fr.Mode.FP64_FAST

                def render():
                    return D.render_bands("mandelbrot", c.window, c.width, c.height,
                                          c.max_iter, c.band_rows, mode=mode, gather=False)
            def gather(loc):
                if pal is None:
                    return D.gather_bands(loc, c.height, c.band_rows)
                return (D.gather_bands(loc[0], c.height, c.band_rows),
                        D.gather_bands(loc[1], c.height, c.band_rows))

            local = render()  # warm-up (workspaces, survivor buffer, NCCL set-up)
            _ = gather(local)
            del _
            barrier()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(reps):
                local = render()
            t1.record()
            barrier()
            ms = t0.elapsed_time(t1) / reps
            cnt = local[0] if pal is not None else local
            iters = float((cnt.view(torch.int16).to(torch.int64) & 0xFFFF).sum().item())
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            g0.record()
            full = gather(local)
            g1.record()
            barrier()
            gms = g0.elapsed_time(g1)
            t = torch.tensor([ms, gms, iters], dtype=torch.float64, device="cuda")
            mx = t.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = t.clone()
            dist.all_reduce(sm, op=dist.ReduceOp.SUM)
            del full, local
            out[name] = {"compute_ms": float(mx[0]), "gather_ms": float(mx[1]),
                         "gpix_iter_s": float(sm[2]) / (float(mx[0]) * 1e-3) / 1e9,
                         "band_rows": c.band_rows, "mode": mode.name,
                         "colour": "fused classic palette" if pal is not None else None,
                         "world": world,
                         "note": "cyclic bands, compute makespan = max over ranks; gather "
                                 "of the bands to rank 0 (NCCL; uint16 counts, plus RGBA "
                                 "when coloured) timed separately"}
        except Exception as e:  # report, never fail the bench line
            out[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
    return out


def measure_e2e(fr, W, cs, win, world, args, barrier, stream):
    """Same metric end to end through the C-ABI call with HOST buffers:
    julia_render_path_host renders the rank's frames in chunks and copies every chunk's
    uint8 counts (max_iter 100 <= 255) device->host into pinned memory on an internal
    stream while the next chunk renders; it returns once all counts are on the host.
    Per step: 16 B/frame of C values in (kernel parameters), 1 B/pixel of counts out."""
    import torch
    import torch.distributed as dist
    nf = len(cs)
    host = torch.empty((nf, H_PX, W_PX), dtype=torch.uint8, pin_memory=True)

    def step():
        fr.julia_render_path_host(cs, win, W_PX, H_PX, MAX_ITER, fr.Mode.FP32_FAST, out=host,
                                  stream=stream)

    steps = max(2, min(args.steps, 5))
    for _ in range(2):
        step()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    barrier()
    ms = t0.elapsed_time(t1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    iters = int(host.numpy().sum(dtype=np.int64))
    # roofline of e2e: a plain pinned device->host copy of the same bytes (torch)
    dev = torch.empty((nf, H_PX, W_PX), dtype=torch.uint8, device="cuda")
    host.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    copy_gbs = 0.0
    for _ in range(3):  # best of three: PCIe rates vary from copy to copy
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record()
        host.copy_(dev, non_blocking=True)
        c1.record()
        torch.cuda.synchronize()
        copy_gbs = max(copy_gbs, dev.numel() / (c0.elapsed_time(c1) * 1e-3) / 1e9)
    del dev
    tot = torch.tensor([float(iters)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    return {"value": float(tot.item()) * steps / (ms * 1e-3) / 1e9, "unit": "Gpixel-iter/s",
            "h2d_bytes_per_step": int(nf * 16), "d2h_bytes_per_step": int(nf * H_PX * W_PX),
            "steps": steps, "ms_per_step": ms / steps,
            "d2h_GB_per_s": nf * H_PX * W_PX / (ms / steps * 1e-3) / 1e9,
            "d2h_copy_peak_GB_per_s": copy_gbs,
            "bound": "PCIe device->host: d2h_copy_peak_GB_per_s is the best of three plain "
                     "pinned copies of the same bytes (torch), measured in this run",
            "api": "julia_render_path_host (C ABI, host output buffer)",
            "note": "C values (16 B/frame) host->device as kernel parameters; uint8 counts "
                    "device->host into pinned memory inside the call, 128 MiB chunks "
                    "double-buffered and overlapped with rendering"}


def extras(fr, W, torch):
    """Per-config single-GPU figures (fast mode) for the other BASELINE configs."""
    res = {}
    peaks = measured_peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0))
    for name in ("cfg2", "cfg3", "cfg5"):
        cfg = W.configs()[name]
        prec = cfg.precision
        pal = W.palette("classic") if cfg.colorize else None
        out = torch.empty((cfg.height, cfg.width), dtype=torch.uint16, device="cuda")
        rgba = (torch.empty((cfg.height, cfg.width, 4), dtype=torch.uint8, device="cuda")
                if pal else None)
        if cfg.kind == "julia":
            mode = fr.Mode.FP32_FAST

            def fn():
                fr.julia_render_ex(cfg.c, cfg.window, cfg.width, cfg.height, cfg.max_iter, mode,
                                   out=out, palette=pal, out_rgba=rgba)
        else:
            mode = fr.Mode.FP64_FAST

            def fn():
                fr.mandelbrot_param_map(cfg.window, cfg.width, cfg.height, cfg.max_iter, mode,
                                        out=out)
        # timed regions of several ms: a sub-ms burst after an idle sync is ~1 us per call
        # slower on cfg2 (clock ramp at the burst's start)
        reps = {"cfg2": 400, "cfg3": 50, "cfg5": 2}[name]
        fn()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / reps
        s = int((out.view(torch.int16).to(torch.int64) & 0xFFFF).sum().item())
        ms_graph = None
        if name == "cfg2":  # CUDA graph of 50 frames: no launch gaps between frames
            try:
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    fn()
                torch.cuda.current_stream().wait_stream(side)
                with torch.cuda.graph(g):
                    for _ in range(50):
                        fn()
                g.replay()
                torch.cuda.synchronize()
                a.record()
                for _ in range(4):
                    g.replay()
                b.record()
                b.synchronize()
                ms_graph = a.elapsed_time(b) / 200
            except Exception as e:  # report, never fail the line
                ms_graph = f"graph capture failed: {type(e).__name__}"
        lanes = FP64_LANES_PER_SM if prec == 64 else FP32_LANES_PER_SM
        peak = SM_COUNT * lanes * f_max * 1e6 / ALG_OPS_PER_ITER / 1e9
        res[name] = {"ms": ms, "gpix_iter_s": s / (ms * 1e-3) / 1e9, "pixel_iters": s,
                     "frac_of_alu_peak": s / (ms * 1e-3) / 1e9 / peak,
                     "frac_6op_survey": s / (ms * 1e-3) / 1e9 / peak * SURVEY_OPS_PER_ITER
                     / ALG_OPS_PER_ITER, "mode": mode.name,
                     "fused_colorize": bool(pal), "reps": reps,
                     "note": "back-to-back launches, CUDA events"}
        if ms_graph is not None:
            res[name]["ms_cuda_graph"] = ms_graph
            if isinstance(ms_graph, float):
                res[name]["gpix_iter_s_cuda_graph"] = s / (ms_graph * 1e-3) / 1e9
                res[name]["frames_per_s_cuda_graph"] = 1e3 / ms_graph
        del out, rgba
    torch.cuda.empty_cache()
    res["colorize_hbm"] = colorize_bandwidth(fr, W, torch)
    res["cardioid_path"] = cardioid_path_rate(fr, W, torch, f_max)
    res["fig4_maps"] = fig4_maps_rate(fr, W, torch, f_max)
    return res


# FP32-pipe operations per iteration of the Figure 4 maps' defining sequence (DESIGN.md
# reading c-14; every operation separately rounded): z^4 + c = 7 MUL + 6 ADD/SUB (the
# |Z|^2 test included); the rational map adds 8 MUL + 5 ADD/SUB and two IEEE divisions
FIG4_OPS = {"Z4": 13, "Z4_RATIONAL": 26}


def fig4_maps_rate(fr, W, torch, f_max):
    """NEXT-3: Julia frames of z^4 + c and z^4 + (z^2+1)/(z^2-1) + c at 1080p,
    C = FIG4_C, max_iter 100, FP32 (the maps run the strict sequence), through
    julia_render_fn: both maps on the full view (real span 3; z^4 + c is a dust of
    orbits <= 14 long there) and the rational map on the Figure 4 "zoom" window
    (W.FIG4_ZOOM_*); rate against the FP32 pipe for the map's op count."""
    res = {}
    try:
        out = torch.empty((H_PX, W_PX), dtype=torch.uint16, device="cuda")
        full = W.julia_window(W_PX, H_PX, span_re=3.0)
        zoom = W.julia_window(W_PX, H_PX, span_re=W.FIG4_ZOOM_SPAN, center=W.FIG4_ZOOM_CENTER)
        for key, name, win in (("z4", "Z4", full), ("z4_rational", "Z4_RATIONAL", full),
                               ("z4_rational_zoom", "Z4_RATIONAL", zoom)):
            f = fr.Function[name]

            def call():
                fr.julia_render_fn(f, W.FIG4_C, win, W_PX, H_PX, MAX_ITER, fr.Mode.FP32_STRICT,
                                   out=out)
            call()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            reps = 200
            a.record()
            for _ in range(reps):
                call()
            b.record()
            b.synchronize()
            ms = a.elapsed_time(b) / reps
            s = float((out.view(torch.int16).to(torch.int64) & 0xFFFF).sum().item())
            rate = s / (ms * 1e-3) / 1e9
            peak = SM_COUNT * FP32_LANES_PER_SM * f_max * 1e6 / FIG4_OPS[name] / 1e9
            res[key] = {
                "ms": ms, "gpix_iter_s": rate, "pixel_iters": s, "frames_per_s": 1e3 / ms,
                "fp32_ops_per_iter": FIG4_OPS[name], "frac_of_fp32_pipe": rate / peak,
                "note": ("kernel S (one orbit per lane, strict sequence); the two divisions "
                         "are counted as one op each" if "RAT" in name else
                         "kernel fn2 (two pixels per thread, strict sequence)")}
        del out
    except Exception as e:  # report, never fail the line
        res["error"] = f"{type(e).__name__}: {e}"[:300]
    return res


def cardioid_path_rate(fr, W, torch, f_max):
    """NEXT-2: the paper's own C-path -- 512 frames of 1080p along the a = 3.9
    cardioid (fr_cardioid_path), max_iter 100, FP32_FAST, through julia_render_path."""
    try:
        cs = fr.cardioid_path(512)
        win = W.julia_window(W_PX, H_PX)
        out = torch.empty((len(cs), H_PX, W_PX), dtype=torch.uint16, device="cuda")
        fr.julia_render_path(cs, win, W_PX, H_PX, MAX_ITER, fr.Mode.FP32_FAST, out=out)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        reps = 3
        a.record()
        for _ in range(reps):
            fr.julia_render_path(cs, win, W_PX, H_PX, MAX_ITER, fr.Mode.FP32_FAST, out=out)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / reps
        s = float((out.view(torch.int16).to(torch.int64) & 0xFFFF).sum().item())
        peak = SM_COUNT * FP32_LANES_PER_SM * f_max * 1e6 / ALG_OPS_PER_ITER / 1e9
        del out
        return {"frames": len(cs), "ms": ms, "frames_per_s": len(cs) / (ms * 1e-3),
                "gpix_iter_s": s / (ms * 1e-3) / 1e9,
                "mean_iters_per_px": s / (len(cs) * W_PX * H_PX),
                "frac_of_alu_peak": s / (ms * 1e-3) / 1e9 / peak,
                "note": "cardioid a = 3.9, clockwise (fr_cardioid_path), kernel SX"}
    except Exception as e:  # report, never fail the line
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def colorize_bandwidth(fr, W, torch):
    """Standalone colour levels (N6) on 512 frames of 1080p counts (2.1 GB read + 4.2 GB
    written, >> L2): algorithmic bytes / time against the measured HBM copy peak."""
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6556.2))
    n = 512 * W_PX * H_PX
    counts = torch.randint(0, 101, (n,), dtype=torch.int32, device="cuda").to(torch.int16).view(torch.uint16)
    rgba = torch.empty((n, 4), dtype=torch.uint8, device="cuda")
    pal = W.palette("classic")
    fr.colorize(counts, 100, pal, out_rgba=rgba)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fr.colorize(counts, 100, pal, out_rgba=rgba)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 5
    gbs = n * 6 / (ms * 1e-3) / 1e9
    del counts, rgba
    torch.cuda.empty_cache()
    return {"pixels": n, "ms": ms, "GB_per_s": gbs, "peak_GB_per_s": hbm, "frac": gbs / hbm,
            "bound": "hbm", "bytes_per_pixel": 6,
            "peak_basis": "MEASURED_PEAKS.json hbm_gbs (torch copy, read+write)"}


if __name__ == "__main__":
    sys.exit(main())
