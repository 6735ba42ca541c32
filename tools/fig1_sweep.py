"""NEXT-1: the paper's Figure 1 experiment on B200 -- generation time of a
square Julia frame against its side, GPU (libfractal, compute only, display excluded as
in P:37) vs the CPU oracle (1 thread, and all host threads).  Writes a JSON list."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from paper_1611_03079_b200 import binding as fr

C = -0.8 + 0.156j          # CUDA by Example's constant (P:37 cites [7]); window [-1.5, 1.5]^2
SIDES = [10, 32, 100, 316, 1000, 3162, 10000]
MAX_ITER = 100

def gpu_ms(n, mode, reps):
    out = torch.empty((n, n), dtype=torch.uint16, device="cuda")
    fn = lambda: fr.julia_render_ex(C, (0j, 1.5, 1.5), n, n, MAX_ITER, mode, out=out)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts)), int((out.view(torch.int16).to(torch.int64) & 0xFFFF).sum())

def cpu_ms(n, threads, budget_s=20.0):
    t0 = time.perf_counter(); reps = 0
    while True:
        oracle.julia(C, 0j, 1.5, 1.5, n, n, MAX_ITER, 32, threads)
        reps += 1
        if time.perf_counter() - t0 > min(budget_s, 0.5) or reps >= 5:
            break
    return (time.perf_counter() - t0) / reps * 1e3

res = []
allt = oracle.default_threads()
for n in SIDES:
    g_fast, s = gpu_ms(n, fr.Mode.FP32_FAST, 20)
    g_strict, _ = gpu_ms(n, fr.Mode.FP32_STRICT, 20)
    c1 = cpu_ms(n, 1) if n <= 3162 else None
    cn = cpu_ms(n, allt)
    row = {"side": n, "pixel_iters": s, "gpu_fast_ms": g_fast, "gpu_strict_ms": g_strict,
           "cpu_1thread_ms": c1, f"cpu_{allt}threads_ms": cn,
           "speedup_vs_1thread": (c1 / g_fast) if c1 else None, "speedup_vs_allthreads": cn / g_fast}
    res.append(row); print(json.dumps(row), flush=True)
json.dump({"experiment": "Figure 1 (P:35-39): square Julia frame, C=-0.8+0.156i, [-1.5,1.5]^2, max_iter 100, fp32; GPU timed with CUDA events around the ABI call (includes launch), CPU = strict oracle",
           "host_threads": allt, "rows": res}, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fig1.json", "w"), indent=1)
