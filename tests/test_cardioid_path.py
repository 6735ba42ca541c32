"""NEXT-2: the paper's cardioid C-path -- host generator in the C ABI against the
oracle's f(t, a) and the SPEC step rule."""
import math

import numpy as np
import pytest

import oracle
from paper_1611_03079_b200 import binding as B
from paper_1611_03079_b200 import workloads as W


@pytest.fixture(scope="module")
def lib():
    from paper_1611_03079_b200 import build
    build.build()
    return B.load()


def _spec_path(n, t0, a0, dt, da, floor):
    """t' = t - dt; on passing -2 pi: t' += 2 pi, a' = max(a - da, floor)."""
    out, t, a = [], t0, a0
    for _ in range(n):
        out.append(oracle.cardioid_point(t, a))
        t -= dt
        if t <= -2 * math.pi:
            t += 2 * math.pi
            a = max(a - da, floor)
    return np.array(out)


@pytest.mark.parametrize("args", [(1500, 0.0, 3.9, 2 * math.pi / 600, 0.05, 3.5),
                                  (100, 1.0, 4.0, 0.1, 0.0, 3.5), (7, -0.5, 3.9, 0.0, 0.05, 3.5),
                                  (5000, 0.0, 3.9, 2 * math.pi / 360, 0.1, 3.6)])
def test_cardioid_path_matches_oracle(lib, args):
    got = B.cardioid_path(*args)
    ref = _spec_path(*args)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-15)


def test_cardioid_path_properties(lib):
    c = B.cardioid_path(600 * 9)
    assert c[0] == pytest.approx(1 / 3.9)  # t = 0: (2 - 1)/a
    # a shrinks by 0.05 per revolution down to the floor 3.5: |C| at t = 0 is 1/a
    for rev, a in [(1, 3.85), (2, 3.8), (8, 3.5)]:
        assert c[600 * rev].real == pytest.approx(1 / a, rel=1e-9)
    # every point stays outside the main cardioid (a < 4: "just outside the main body")
    assert (np.abs(1 - np.sqrt(1 - 4 * c)) > 1).all()
    # clockwise: the first steps move from t = 0 toward negative t (Im C < 0)
    assert c[1].imag < 0 and c[5].imag < 0
    # the four Figure 2 parameters are visited (within the caption's rounding + step)
    for fc in W.FIG2_C:
        assert np.abs(c[:600] - fc).min() < 0.02


def test_cardioid_path_validation(lib):
    assert lib.fr_cardioid_path(0.0, 0.0, 0.1, 0.0, 3.5, 3, None) == 1
    assert lib.fr_cardioid_path(0.0, 3.9, -0.1, 0.0, 3.5, 3, None) == 1
    assert lib.fr_cardioid_path(0.0, 3.9, 0.1, 0.0, 3.5, -1, None) == 1
    assert lib.fr_cardioid_path(float("nan"), 3.9, 0.1, 0.0, 3.5, 1, None) == 1
    assert lib.fr_cardioid_path(0.0, 3.9, 0.1, 0.0, 3.5, 0, None) == 0
    assert len(B.cardioid_path(0)) == 0
