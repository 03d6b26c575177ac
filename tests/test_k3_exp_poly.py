"""The FMA-pipe exp2 of K3 (ptx.cuh ex2_poly2), restated in float32 numpy with
the constants parsed from the header: relative error far below bf16's 2^-9
over the softmax range (x <= 8 under lazy rescaling), no exponent wrap below."""
import pathlib
import re

import numpy as np

HDR = pathlib.Path(__file__).resolve().parents[1] / "paper_2404_02015_b200/csrc/kernels/ptx.cuh"


def _consts():
    src = HDR.read_text()
    body = src[src.index("void ex2_poly2"):]
    m = re.search(r"c0 = ([0-9.e+-]+)f, c1 = ([0-9.e+-]+)f, c2 = ([0-9.e+-]+)f, c3 = ([0-9.e+-]+)f", body)
    assert m, "ex2_poly2 constants not found"
    return [np.float32(v) for v in m.groups()]


def _ex2_poly(x):
    c0, c1, c2, c3 = _consts()
    shift = np.float32(12582912.0)
    x = np.maximum(x.astype(np.float32), np.float32(-126.0))
    t = (x + shift).astype(np.float32)
    r = (t - shift).astype(np.float32)
    f = (x - r).astype(np.float32)
    # fused multiply-adds: evaluate in float64 and round once, as FFMA2 does
    p = np.float32(np.float64(f) * np.float64(c3) + np.float64(c2))
    p = np.float32(np.float64(p) * np.float64(f) + np.float64(c1))
    p = np.float32(np.float64(p) * np.float64(f) + np.float64(c0))
    bits = (p.view(np.uint32).astype(np.uint64) + ((t.view(np.uint32).astype(np.uint64) << 23) & 0xFFFFFFFF)) & 0xFFFFFFFF
    return bits.astype(np.uint32).view(np.float32)


def test_relative_error_in_softmax_range():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-120, 8, 1 << 20), np.linspace(-30, 8, 200001)]).astype(np.float32)
    got = _ex2_poly(x).astype(np.float64)
    want = np.exp2(x.astype(np.float64))
    assert (np.abs(got - want) / want).max() < 1e-4  # bf16 P keeps 2^-9 = 2e-3


def test_underflow_stays_tiny_and_positive():
    x = np.array([-126.5, -127, -150, -1e4, -np.inf], np.float32)
    got = _ex2_poly(x)
    assert np.all(got >= 0) and np.all(got < 2e-38)


def test_integers_exact_enough():
    x = np.arange(-100, 9, dtype=np.float32)
    got = _ex2_poly(x).astype(np.float64)
    assert np.allclose(got, np.exp2(x.astype(np.float64)), rtol=1e-4, atol=0)
