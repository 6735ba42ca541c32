"""Static checks on the built sm_100a code (cuobjdump, no GPU): the escape kernels are
compiled for sm_100a, do not spill to local memory, and the fast fp32 loops keep the
constant 0.5 of X' = T * 0.5 + CR2 as an FFMA immediate.  ptxas rematerialises 0.5
with an extra ALU move every iteration when C sits in a uniform register (DESIGN.md
§5, "SASS guard"); that cost +18% instructions on the bench kernel before it was
caught, so it is pinned here."""
import os
import re
import shutil
import subprocess

import pytest

from paper_1611_03079_b200 import build

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="no cuobjdump")


@pytest.fixture(scope="module")
def sass():
    build.build()
    out = subprocess.run(["cuobjdump", "-sass", build.LIB], capture_output=True, text=True,
                         check=True).stdout
    funcs, name = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            funcs[name] = []
            continue
        if name is not None:
            ins = re.sub(r"/\*\s*0x[0-9a-f]+\s*\*/", "", line)  # drop encoding words
            ins = re.sub(r"^\s*/\*[0-9a-f]+\*/", "", ins).strip()
            if ins:
                funcs[name].append(ins)
    return out, funcs


def _fast_f32(name):
    # escape_tile / escape_refill / escape_budget / escape_cont kernels with T = float,
    # STRICT = false; escape_tile2_kernel<STRICT = false, ...>
    return (re.search(r"escape_(tile|refill|budget|cont)_kernelIfLb0E", name) is not None
            or "escape_tile2_kernelILb0E" in name or "escape_pathx_kernel" in name)


def test_sm100a(sass):
    out, funcs = sass
    assert "arch = sm_100a" in out
    assert any("escape_tile_kernel" in f for f in funcs)
    assert any("colorize_kernel" in f for f in funcs)


def test_no_local_memory_spills(sass):
    _, funcs = sass
    for name, ins in funcs.items():
        if "escape" in name or "colorize" in name:
            bad = [i for i in ins if re.search(r"\b(LDL|STL)\b", i)]
            assert not bad, (name, bad[:3])


def test_half_stays_an_immediate(sass):
    _, funcs = sass
    fast = [n for n in funcs if _fast_f32(n)]
    assert len(fast) >= 10
    for name in fast:
        remat = [i for i in funcs[name] if re.search(r"MOV.*0x3f000000", i)]
        assert not remat, (name, remat[:3])
        assert any(re.search(r"FFMA2? .*, 0\.5, ", i) for i in funcs[name]), name


def _tile_fn_param(name):
    """FN template argument of escape_tile_kernel<T, STRICT, MANDEL, COLOR, K, NC, FN, ES>
    (the Figure 4 map variants; FN = 2 divides)."""
    m = re.search(r"escape_tile_kernelI[fd](?:Lb[01]E){3}Li(\d+)ELi(\d+)ELi(\d+)E", name)
    return int(m.group(3)) if m else 0


def _strict(name):
    # escape_fn2_kernel: the Figure 4 map z^4 + c (FN = 1), strict sequence only
    return (re.search(r"escape_(tile|refill|budget|cont)_kernelI[fd]Lb1E", name) is not None
            or "escape_tile2_kernelILb1E" in name
            or re.search(r"escape_fn2_kernelI[fd]Li1E", name) is not None)


def test_strict_kernels_never_fuse(sass):
    """Reading c-9: STRICT runs every multiply and add separately rounded.  ptxas may
    contract separately written packed or scalar .rn ops (it does so for mul.rn.f32x2 +
    add.rn.f32x2), so the strict kernels are checked for fused instructions: none, except
    in the map variant with the rational term (FN = 2), whose correctly rounded division
    routine uses FMAs internally.  (HFMA2 -RZ, RZ is ptxas's register-zeroing idiom, not
    arithmetic, and fp16 is not used.)"""
    _, funcs = sass
    strict = [n for n in funcs if _strict(n)]
    assert len(strict) >= 10
    for name in strict:
        if _tile_fn_param(name) == 2:
            continue
        fused = [i for i in funcs[name] if re.search(r"\b(FFMA2?|DFMA)\b", i)]
        assert not fused, (name, fused[:3])


def test_fast_two_orbit_loops_are_packed(sass):
    """The two-orbit fast fp32 vote loops (S frame pairs, S2, exact P1) run on packed
    FFMA2 / FMUL2 (sm_100): both orbits per instruction."""
    _, funcs = sass
    names = [n for n in funcs
             if "escape_tile2_kernelILb0E" in n
             or re.search(r"escape_budget_kernelIfLb0ELb[01]ELb[01]ELi0ELi0E", n)
             or re.search(r"escape_tile_kernelIfLb0ELb0ELb[01]ELi4ELi1024E", n)
             or "escape_pathx_kernel" in n]
    assert len(names) >= 14
    for name in names:
        assert sum("FFMA2" in i for i in funcs[name]) >= 8, name
        assert any("FMUL2" in i for i in funcs[name]), name


def _loops(ins):
    """Backward-branch loops of a function's SASS: (first, last) index pairs."""
    addr = []
    for i in ins:
        m = re.match(r"/\*([0-9a-f]{4,})\*/", i)
        addr.append(int(m.group(1), 16) if m else None)
    out = []
    for k, i in enumerate(ins):
        m = re.search(r"BRA (?:P\d, )?0x([0-9a-f]+)", i)
        if m and addr[k] is not None and int(m.group(1), 16) < addr[k]:
            t = int(m.group(1), 16)
            first = next(j for j, a in enumerate(addr) if a is not None and a >= t)
            out.append((first, k))
    return out


def test_sx_frame_loop_vote_blocks_are_move_free(sass):
    """Kernel SX's uint16 PTX frame loop: every vote loop of its frame
    loops is the 23-instruction packed block -- 10 FFMA2/FMUL2, 4 FSETP, 4 count
    increments, vote, loop test -- with no register moves.  Register budgets that make
    ptxas add 2-3 moves per block measured 4-10% slower (profiles/r02/ab_sx_regs.txt)."""
    _, funcs = sass
    raw = subprocess.run(["cuobjdump", "-sass", build.LIB], capture_output=True, text=True,
                         check=True).stdout
    name = next(n for n in funcs if re.search(r"escape_pathx_kernelILi1024ELi2ELb0ELb1E", n))
    body = raw.split("Function : " + name, 1)[1].split("Function :", 1)[0]
    ins = [re.sub(r"/\*\s*0x[0-9a-f]+\s*\*/", "", l).strip() for l in body.splitlines()]
    ins = [i for i in ins if re.match(r"/\*[0-9a-f]{4,}\*/", i)]
    # the PTX frame loop of the first C chunk (the one every frame group of <= 128 frames
    # runs; nvcc unrolls the chunk loop, and later copies are not pinned): the first outer
    # loop that loads C from shared memory (LDS) and stores; the innermost vote loops
    # inside it (one VOTE, no store)
    loops = _loops(ins)
    frame_loops = [(a, b) for a, b in loops
                   if any("LDS" in x for x in ins[a:b + 1]) and any("STG" in x for x in ins[a:b + 1])]
    assert frame_loops, name
    frame_loops = [min(frame_loops)]
    vote_loops = [(a, b) for a, b in loops
                  if sum("VOTE" in x for x in ins[a:b + 1]) == 1
                  and not any("STG" in x for x in ins[a:b + 1])
                  and any(fa <= a and b <= fb for fa, fb in frame_loops)]
    assert vote_loops, name
    for a, b in vote_loops:
        blk = ins[a:b + 1]
        assert sum(bool(re.search(r"\b(FFMA2|FMUL2)\b", x)) for x in blk) == 10, blk
        assert not [x for x in blk if re.search(r"\bMOV\b|IMAD\.MOV", x)], blk
        assert len(blk) <= 23, (len(blk), blk)
