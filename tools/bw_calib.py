"""Calibrate the colorize roofline: bandwidth of plain torch ops with colorize's byte
pattern (read 2 B, write 4 B per element) next to the 1:1 copy of MEASURED_PEAKS.json."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
n = 1 << 30
src16 = torch.randint(0, 1000, (n,), dtype=torch.int16, device="cuda")
dst32 = torch.empty(n, dtype=torch.int32, device="cuda")
a16 = torch.empty_like(src16)
def timeit(fn, bytes_, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    return bytes_ / (best * 1e-3) / 1e9
res = {
    "copy_int16_GBps (1:1)": timeit(lambda: a16.copy_(src16), 4 * n),
    "int16_to_int32_GBps (1:2, colorize pattern)": timeit(lambda: dst32.copy_(src16), 6 * n),
    "fill_int32_GBps (write only)": timeit(lambda: dst32.fill_(7), 4 * n),
}
from paper_1611_03079_b200 import binding as fr
from paper_1611_03079_b200 import workloads as W
counts = (src16[: n // 2].view(torch.uint16))
rgba = torch.empty((n // 2, 4), dtype=torch.uint8, device="cuda")
pal = W.palette("classic")
res["colorize_GBps (1:2)"] = timeit(lambda: fr.colorize(counts, 1000, pal, out_rgba=rgba), 6 * (n // 2))
print(json.dumps(res, indent=1))
