"""Per-warp timeline of the lane-refill kernel on cfg3 (entry, supply exhaustion, exit)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes, numpy as np, torch
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
c = W.configs()["cfg3"]
s = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lib = fr.load()
tr = torch.zeros(200000 * 3, dtype=torch.int64, device="cuda")
fr.julia_render_ex(c.c, c.window, c.width * s, c.height * s, c.max_iter, fr.Mode.FP32_FAST)
torch.cuda.synchronize()
lib.fr_debug_refill_trace(ctypes.c_void_p(tr.data_ptr()))
fr.julia_render_ex(c.c, c.window, c.width * s, c.height * s, c.max_iter, fr.Mode.FP32_FAST)
torch.cuda.synchronize()
lib.fr_debug_refill_trace(None)
t = tr.cpu().numpy().reshape(-1, 3)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
st, ex, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
q = lambda a: [round(float(np.percentile(a, p)), 1) for p in (0, 10, 50, 90, 99, 100)]
print(json.dumps({"scale": s, "warps": int(len(t)), "start_us_pct": q(st), "exhaust_us_pct": q(ex),
                  "end_us_pct": q(en), "drain_us_pct": q(en - ex)}))
# utilisation: fraction of warp-time after exhaustion
tot = (en - st).sum(); print(json.dumps({"frac_warp_time_after_exhaustion": float((en - ex).sum() / tot)}))
