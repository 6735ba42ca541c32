"""Host submission latency of small frames (NEXT-1 / NEXT-4 regime): per-call
time of julia_render_ex (generic binding) and FramePlan.render (arguments marshalled
once), measured (a) as in tools/fig1_sweep.py -- CUDA events around ONE call, median --
and (b) back to back, N calls between two events (the submission rate)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1611_03079_b200 import binding as fr

C = -0.8 + 0.156j
res = {}
for n in (10, 100, 316, 1000):
    out = torch.empty((n, n), dtype=torch.uint16, device="cuda")
    plan = fr.FramePlan("julia", (0j, 1.5, 1.5), n, n, 100, fr.Mode.FP32_FAST, out=out)
    calls = {"julia_render_ex": lambda: fr.julia_render_ex(C, (0j, 1.5, 1.5), n, n, 100,
                                                           fr.Mode.FP32_FAST, out=out),
             "plan": lambda: plan.render(C)}
    row = {}
    for name, fn in calls.items():
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(200):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        for _ in range(2000):
            fn()
        b.record()
        host_us = (time.perf_counter() - t0) / 2000 * 1e6
        b.synchronize()
        row[name] = {"one_call_us_median": float(np.median(ts)),
                     "back_to_back_us": a.elapsed_time(b) * 1e3 / 2000,
                     "host_submit_us": host_us}
    # the plan's call captured once into a CUDA graph (fixed C), replayed back to back
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        gplan = fr.FramePlan("julia", (0j, 1.5, 1.5), n, n, 100, fr.Mode.FP32_FAST, out=out,
                             stream=s)
        gplan.render(C)  # eager first call on the stream (workspaces, outside capture)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            gplan.render(C)
    torch.cuda.synchronize()
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(2000):
        g.replay()
    b.record()
    b.synchronize()
    row["plan_graph_replay"] = {"back_to_back_us": a.elapsed_time(b) * 1e3 / 2000}
    res[n] = row
    print(json.dumps({"side": n, **row}), flush=True)
