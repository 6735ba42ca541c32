"""Instruction accounting of an escape kernel from an ncu report's SASS source page
(needs a capture with --import-source; per-instruction 'Instructions Executed').

Finds the hot vote loop (the backward branch right after a VOTE with the most executed
instructions), and reports
  * the share of executed warp-instructions inside that loop vs outside (setup, stores),
  * the hardware-measured SIMT efficiency of the loop: for the predicated count
    increments (@P IADD/VIADD), predicated-on threads / threads = the fraction of lanes
    whose orbit was still alive when the iteration ran,
  * the top stall-sampled instructions.
usage: python tools/ncu_loop_share.py report.ncu-rep [kernel-substring]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
blocks, cur = [], None
for line in out:
    if line.startswith('"Kernel Name"'):
        cur = {"name": next(csv.reader([line]))[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(line)
for b in blocks:
    if want and want not in b["name"]:
        continue
    rows = list(csv.reader(b["rows"]))
    h = rows[0]
    ia, isrc = h.index("Address"), h.index("Source")
    iex, ith = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    ipo = h.index("Predicated-On Thread Instructions Executed")
    ist = h.index("Warp Stall Sampling (All Samples)")
    ins = []
    for r in rows[1:]:
        if len(r) <= ist:
            continue
        try:
            ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ith] or 0),
                        int(r[ipo] or 0), int(r[ist] or 0)))
        except ValueError:
            continue
    addr = [i[0] for i in ins]
    # candidate loops: backward branches preceded (within 3) by a VOTE
    best = None
    for k, (a, src, ex, th, po, st) in enumerate(ins):
        m = re.search(r"BRA(?:\.\w+)?\s.*?(0x[0-9a-f]+)", src)
        if not m or "VOTE" not in " ".join(x[1] for x in ins[max(0, k - 3):k]):
            continue
        tgt = int(m.group(1), 16) + addr[0] if int(m.group(1), 16) < addr[0] else int(m.group(1), 16)
        if tgt >= a:
            continue
        lo = next((j for j, x in enumerate(ins) if x[0] >= tgt), None)
        if lo is None:
            continue
        tot = sum(x[2] for x in ins[lo:k + 1])
        if best is None or tot > best[2]:
            best = (lo, k, tot)
    total = sum(x[2] for x in ins)
    print(f"kernel: {b['name'][:110]}")
    print(f"  executed warp-instructions: {total:.4g}")
    if best:
        lo, hi, tot = best
        inc = [x for x in ins[lo:hi + 1] if re.match(r"@!?P\d\s+(IADD3|VIADD)", x[1])]
        th = sum(x[3] for x in inc)
        po = sum(x[4] for x in inc)
        print(f"  hot loop: {hi - lo + 1} SASS instructions, {tot / total:.3f} of executed"
              f" warp-instructions")
        if th:
            print(f"  SIMT efficiency of the loop (alive lanes per count increment): {po / th:.3f}")
        st_all = sum(x[5] for x in ins)
        st_loop = sum(x[5] for x in ins[lo:hi + 1])
        if st_all:
            print(f"  stall samples inside the loop: {st_loop / st_all:.3f} of {st_all}")
    top = sorted(ins, key=lambda x: -x[5])[:6]
    print("  top stall-sampled instructions:")
    for a, src, ex, th, po, st in top:
        print(f"    {st:8d}  {src[:70]}")
