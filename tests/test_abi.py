"""The C-ABI boundary on CPU: libfractal loads, exports every function declared in
include/fractal.h, and its synchronous validation returns the documented statuses
without launching anything (no GPU needed for these paths)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1611_03079_b200 import binding as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1611_03079_b200 import build
    build.build()
    return B.load()


def _declared():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            for m in re.finditer(r"^[A-Za-z_][\w \*]*?\b(\w+)\s*\(", src, flags=re.M):
                if m.group(1) not in ("defined",):
                    names.add(m.group(1))
    return names


def test_every_declared_symbol_is_exported(lib):
    declared = _declared()
    assert {"julia_render", "julia_render_path", "mandelbrot_param_map", "colorize"} <= declared
    assert declared == set(B.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_version_and_status_strings(lib):
    assert "sm_100a" in B.version()
    for s, name in B.STATUS.items():
        assert lib.fr_status_str(s).decode().startswith(name)


W = B._Window(0.0, 0.0, 2.0, 1.125)
C = B._Complex(-0.7269, 0.1889)
NOPAL = None
DUMMY = ctypes.c_void_p(0x1000)  # never dereferenced: validation fails first
STREAM = ctypes.c_void_p(0)


@pytest.mark.parametrize("args,expected", [
    (dict(width=0), 1), (dict(height=-3), 1), (dict(max_iter=0), 1), (dict(max_iter=65536), 3),
    (dict(width=65536, height=32769), 2), (dict(c=B._Complex(float("nan"), 0.0)), 1),
    (dict(c=B._Complex(0.0, float("inf"))), 1), (dict(win=B._Window(0.0, 0.0, 0.0, 1.0)), 1),
    (dict(win=B._Window(0.0, 0.0, 1.0, -1.0)), 1), (dict(win=B._Window(float("inf"), 0.0, 1.0, 1.0)), 1),
    (dict(out=None), 1), (dict(mode=7), 3), (dict(bands=B._Bands(4, 2, 2)), 1),
    (dict(bands=B._Bands(-1, 1, 0)), 1), (dict(bands=B._Bands(0, 2, 0)), 1),
    (dict(rgba=DUMMY), 1),
])
def test_julia_render_ex_validation(lib, args, expected):
    a = dict(c=C, win=W, width=1920, height=1080, max_iter=100, mode=0, bands=B._Bands(0, 1, 0),
             out=DUMMY, pal=None, rgba=None)
    a.update(args)
    before = lib.fr_launch_count()
    rc = lib.julia_render_ex(a["c"], a["win"], a["width"], a["height"], a["max_iter"], a["mode"],
                             a["bands"], a["out"], a["pal"], a["rgba"], STREAM)
    assert rc == expected
    assert lib.fr_launch_count() == before  # nothing launched on error


def test_palette_validation(lib):
    ent = np.zeros((1, 4), np.uint8)
    bad = B._Palette(ent.ctypes.data, 1, (ctypes.c_uint8 * 4)(0, 0, 0, 255))
    rc = lib.julia_render_ex(C, W, 64, 64, 100, 0, B._Bands(0, 1, 0), DUMMY, ctypes.byref(bad),
                             DUMMY, STREAM)
    assert rc == 1
    big = B._Palette(ent.ctypes.data, 257, (ctypes.c_uint8 * 4)(0, 0, 0, 255))
    assert lib.colorize(DUMMY, 10, 100, ctypes.byref(big), DUMMY, STREAM) == 1
    assert lib.colorize(DUMMY, 10, 100, None, DUMMY, STREAM) == 1
    assert lib.colorize(DUMMY, -1, 100, None, DUMMY, STREAM) == 1
    ok = np.zeros((4, 4), np.uint8)
    pal = B._Palette(ok.ctypes.data, 4, (ctypes.c_uint8 * 4)(0, 0, 0, 255))
    before = lib.fr_launch_count()
    assert lib.colorize(None, 0, 100, ctypes.byref(pal), None, STREAM) == 0  # no-op
    assert lib.colorize(DUMMY, 10, 70000, ctypes.byref(pal), DUMMY, STREAM) == 3
    assert lib.fr_launch_count() == before


def test_path_validation(lib):
    cs = np.array([0.1 + 0.2j, np.nan], dtype=np.complex128)
    before = lib.fr_launch_count()
    assert lib.julia_render_path(None, 0, W, 64, 64, 100, 0, None, None, None, STREAM) == 0
    assert lib.julia_render_path(cs.ctypes.data, 2, W, 64, 64, 100, 0, DUMMY, None, None, STREAM) == 1
    assert lib.julia_render_path(cs.ctypes.data, -1, W, 64, 64, 100, 0, DUMMY, None, None, STREAM) == 1
    assert lib.julia_render_path(None, 3, W, 64, 64, 100, 0, DUMMY, None, None, STREAM) == 1
    assert lib.julia_render_path(cs.ctypes.data, 1, W, 64, 64, 100, 9, DUMMY, None, None, STREAM) == 3
    assert lib.fr_launch_count() == before


def test_mandelbrot_validation(lib):
    before = lib.fr_launch_count()
    assert lib.mandelbrot_param_map(W, 0, 10, 100, 2, B._Bands(0, 1, 0), DUMMY, None, None, STREAM) == 1
    assert lib.mandelbrot_param_map(W, 10, 10, 100, 2, B._Bands(0, 1, 0), None, None, None, STREAM) == 1
    # a rank that holds no band is a valid no-op
    assert lib.mandelbrot_param_map(W, 10, 10, 100, 2, B._Bands(16, 2, 1), DUMMY, None, None, STREAM) == 0
    assert lib.fr_launch_count() == before


def _bands_reference(height, band_rows, n_ranks, rank):
    """Global rows of a rank, written out from the definition."""
    if band_rows == 0:
        return list(range(height))
    rows = []
    b = 0
    while b * band_rows < height:
        if b % n_ranks == rank:
            rows.extend(range(b * band_rows, min((b + 1) * band_rows, height)))
        b += 1
    return rows


@pytest.mark.parametrize("height,band_rows,n_ranks", [(2160, 15, 8), (2160, 15, 1), (1081, 16, 8),
                                                      (7, 3, 4), (5, 16, 2), (16384, 16, 8),
                                                      (100, 1, 3)])
def test_band_row_mapping(lib, height, band_rows, n_ranks):
    seen = []
    for rank in range(n_ranks):
        bands = B.Bands(band_rows, n_ranks, rank)
        ref = _bands_reference(height, band_rows, n_ranks, rank)
        assert B.band_local_rows(height, bands) == len(ref)
        got = [B.band_global_row(height, bands, i) for i in range(len(ref))]
        assert got == ref
        assert B.band_global_row(height, bands, len(ref)) == -1
        seen.extend(ref)
    assert sorted(seen) == list(range(height))  # the ranks partition the frame


def test_python_api_rejects_cpu_tensors(lib):
    import torch
    with pytest.raises(B.FractalError):
        B.julia_render(0.1 + 0.2j, (0j, 2.0, 2.0), 8, 8, 100, out=torch.empty((8, 8), dtype=torch.uint16))


def test_function_variant_validation(lib):
    before = lib.fr_launch_count()
    assert lib.julia_render_fn(7, C, W, 64, 64, 100, 1, DUMMY, None, None, STREAM) == 3
    assert lib.julia_render_fn(1, C, W, 0, 64, 100, 1, DUMMY, None, None, STREAM) == 1
    assert lib.julia_render_fn(2, B._Complex(float("nan"), 0), W, 8, 8, 100, 1, DUMMY, None, None, STREAM) == 1
    assert lib.fr_launch_count() == before


def test_rank_without_bands_is_a_noop(lib):
    """A rank whose cyclic bands are all past the last row holds 0 rows: FR_OK, nothing
    launched, null outputs accepted (an empty torch tensor has a null data_ptr)."""
    before = lib.fr_launch_count()
    assert B.band_local_rows(1, B.Bands(4, 3, 1)) == 0
    assert lib.julia_render_ex(C, W, 64, 1, 100, 0, B._Bands(4, 3, 1), None, None, None, STREAM) == 0
    assert lib.mandelbrot_param_map(W, 64, 4, 100, 2, B._Bands(4, 2, 1), None, None, None, STREAM) == 0
    assert lib.fr_launch_count() == before


def _build_c_demo(tmp_path):
    """Compile examples/c_abi_demo.c (plain C11 against include/fractal.h, linked to
    libfractal.so only) -- the C ABI without Python or torch."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    from paper_1611_03079_b200 import build
    build.build()
    exe = tmp_path / "c_abi_demo"
    pkg = os.path.dirname(build.LIB)
    subprocess.run([cc, "-std=c11", "-Wall", "-Wextra", "-Werror",
                    "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", pkg, "-lfractal",
                    "-lm", f"-Wl,-rpath,{pkg}", "-Wl,--allow-shlib-undefined", "-o", str(exe)],
                   check=True)
    return exe


def test_c_abi_demo_builds(tmp_path):
    """The demo compiles warning-free and, without a GPU, fails cleanly with FR_ERR_CUDA
    through fr_status_str (no crash, exit code 1)."""
    import subprocess
    exe = _build_c_demo(tmp_path)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present: the run is covered by the -m gpu test")
    r = subprocess.run([str(exe), "8", "8", "2", "100", "1", str(tmp_path / "x.bin")],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 1, (r.returncode, r.stdout, r.stderr)
    assert "FR_ERR_CUDA" in r.stderr
