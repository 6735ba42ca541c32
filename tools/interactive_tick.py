"""NEXT-4: the paper's interactive application -- per tick, a full-screen
1920x1080 Julia frame (fused colour levels) plus a 240x180 Mandelbrot minimap, with C
moving along the cardioid path; each tick is launched and synchronised (as a display
would need it).  Reports ms/tick and ticks/s against the paper's ">50 frames per second"."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W

TICKS = 600
cs = fr.cardioid_path(TICKS)
pal = W.palette("classic")
jw = W.julia_window(1920, 1080)
mw = W.mandel_window(240, 180)
jc = torch.empty((1080, 1920), dtype=torch.uint16, device="cuda")
jr = torch.empty((1080, 1920, 4), dtype=torch.uint8, device="cuda")
mc = torch.empty((180, 240), dtype=torch.uint16, device="cuda")
mr = torch.empty((180, 240, 4), dtype=torch.uint8, device="cuda")
res = {}
plans = {}
for variant, mode in (("", fr.Mode.FP32_FAST), ("", fr.Mode.FP32_STRICT),
                      ("plan", fr.Mode.FP32_FAST)):
    if variant == "plan":  # arguments marshalled once (binding.FramePlan)
        jp = fr.FramePlan("julia", jw, 1920, 1080, 100, mode, palette=pal, out=jc, out_rgba=jr)
        mp = fr.FramePlan("mandelbrot", mw, 240, 180, 100, mode, palette=pal, out=mc,
                          out_rgba=mr)
        stream = torch.cuda.current_stream()

        def tick(k):
            jp.render(complex(cs[k]))
            mp.render()
            stream.synchronize()
    else:
        def tick(k):
            fr.julia_render_ex(complex(cs[k]), jw, 1920, 1080, 100, mode, palette=pal, out=jc,
                               out_rgba=jr)
            fr.mandelbrot_param_map(mw, 240, 180, 100, mode, palette=pal, out=mc, out_rgba=mr)
            torch.cuda.current_stream().synchronize()
    for k in range(10): tick(k)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(TICKS + 1)]
    import time
    t0 = time.perf_counter()
    ev[0].record()
    for k in range(TICKS):
        tick(k)
        ev[k + 1].record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / TICKS * 1e3
    gpu = [ev[k].elapsed_time(ev[k + 1]) for k in range(TICKS)]
    name = mode.name + ("_plan" if variant else "")
    res[name] = {"ms_per_tick_wall": wall, "ticks_per_s_wall": 1e3 / wall,
                      "ms_per_tick_gpu_median": float(np.median(gpu)),
                      "ms_per_tick_gpu_p99": float(np.percentile(gpu, 99))}
    print(name, json.dumps(res[name]), flush=True)
json.dump({"experiment": "interactive tick (P:39 '>50 frames per second', P:49 minimap): Julia 1920x1080 + colour levels, Mandelbrot minimap 240x180 + colour levels, C on the a=3.9 cardioid, max_iter 100, each tick synchronised; display excluded",
           "results": res}, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tick.json", "w"), indent=1)
