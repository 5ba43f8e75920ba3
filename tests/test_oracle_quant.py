"""Pins for the oracle's quantizer (O5) and lo() (O6) against exact rational
arithmetic and the paper's worked example."""
import math
from fractions import Fraction

import numpy as np
import pytest

from tests.exact import BINMAX, exact_bin, exact_lo


def test_paper_worked_example(ref):
    # "with an ABS error bound of 0.1, the quantizer maps all values
    # between 0.95 and 1.05 to bin number 10".
    for v in (0.951, 0.96, 0.99, 1.0, 1.01, 1.04, 1.0499):
        assert ref.bin_of(v, 0.1, 1) == 10
        assert ref.bin_of(float(np.float32(v)), 0.1, 0) == 10
    # Boundary ownership is the G6 reading (half-up, exact): the double 0.95 is
    # below 9.5 * 0.1 exactly, so it falls in bin 9; 1.05 is below 10.5 * 0.1.
    assert Fraction(0.95) < Fraction(19, 2) * Fraction(0.1)
    assert ref.bin_of(0.95, 0.1, 1) == 9
    assert ref.bin_of(1.05, 0.1, 1) == 10
    assert ref.bin_of(0.0, 0.1, 1) == 0
    assert ref.bin_of(-0.05, 0.1, 1) == exact_bin(-0.05, 0.1)
    assert ref.bin_of(0.05, 0.1, 1) == exact_bin(0.05, 0.1) == 1


def test_lo_worked_values(ref):
    assert ref.lo(10, 0.1, 1) == 0.9500000000000001 == math.nextafter(0.95, 1)
    assert ref.lo(11, 0.1, 1) == 1.0500000000000003
    assert ref.lo(10, 0.1, 0) == 0.9500000476837158
    for b in (-3, 0, 1, 10, 11, 12345):
        for dt in (np.float32, np.float64):
            assert ref.lo(b, 0.1, 0 if dt == np.float32 else 1) == exact_lo(b, 0.1, dt)


def _rand_eps(rng):
    return float(rng.uniform(1, 2) * 2.0 ** rng.integers(-30, 12))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_lo_exact_random(ref, dt):
    rng = np.random.default_rng(11)
    code = 0 if dt == np.float32 else 1
    for _ in range(1500):
        eps = _rand_eps(rng)
        lim = 2**24 if dt == np.float32 else 2**45
        b = int(rng.integers(-lim, lim))
        assert ref.lo(b, eps, code) == exact_lo(b, eps, dt), (b, eps)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_bin_exact_near_boundaries(ref, dt):
    """Values within +-2 ulps of every bin edge, half-points, zeros."""
    rng = np.random.default_rng(12)
    code = 0 if dt == np.float32 else 1
    finfo = np.finfo(dt)
    for _ in range(1200):
        eps = _rand_eps(rng)
        lim = 2**20
        b = int(rng.integers(-lim, lim))
        edge = dt(exact_lo(b, eps, dt))
        cands = [edge]
        for k in (1, 2):
            cands.append(np.nextafter(edge, dt(np.inf), dtype=dt) if k == 1 else
                         np.nextafter(np.nextafter(edge, dt(np.inf), dtype=dt), dt(np.inf), dtype=dt))
            cands.append(np.nextafter(edge, dt(-np.inf), dtype=dt))
        cands.append(dt(b * eps))
        for x in cands:
            x = float(x)
            if not math.isfinite(x):
                continue
            want = exact_bin(x, eps)
            got = ref.bin_of(x, eps, code)
            if abs(want) <= BINMAX[dt]:
                assert got == want, (x, eps, got, want)
            else:
                assert got is None
    # escapes: non-finite and |b| > BINMAX (G8/G9)
    assert ref.bin_of(math.inf, 1.0, code) is None
    assert ref.bin_of(-math.inf, 1.0, code) is None
    assert ref.bin_of(math.nan, 1.0, code) is None
    bm = BINMAX[dt]
    eps = 1.0
    top = float(dt(bm)) if float(dt(bm)) <= bm else float(np.nextafter(dt(bm), dt(0), dtype=dt))
    assert ref.bin_of(top, eps, code) == exact_bin(top, eps) == int(top)
    assert ref.bin_of(-top, eps, code) == -int(top)
    over = top
    while exact_bin(over, eps) <= bm:
        over = float(np.nextafter(dt(over), dt(np.inf), dtype=dt))
    assert exact_bin(over, eps) > bm and ref.bin_of(over, eps, code) is None
    assert ref.bin_of(float(finfo.max), 1e-3, code) is None


def test_bin_monotone(ref):
    rng = np.random.default_rng(13)
    x = np.sort(rng.standard_normal(3000).astype(np.float32))
    eps = 0.0137
    b = [ref.bin_of(float(v), eps, 0) for v in x]
    assert all(b[i] <= b[i + 1] for i in range(len(b) - 1))


def test_quantize_field_matches_scalar(ref):
    rng = np.random.default_rng(14)
    x = rng.standard_normal((5, 7)).astype(np.float32)
    x[1, 2] = np.inf
    x[3, 3] = np.nan
    q = ref.quantize(x, 0.1)
    for i, v in enumerate(x.ravel()):
        e = ref.bin_of(float(v), 0.1, 0)
        assert q.ravel()[i] == (e if e is not None else np.iinfo(np.int64).min)


def test_ord_pins(ref):
    import oracle

    L = oracle.lib()
    # ord is monotone in value and maps -0.0 and +0.0 to 0 (O3, G13)
    vals = np.array([-np.inf, -3.5, -1e-45, -0.0, 0.0, 1e-45, 2.0, np.inf], np.float32)
    o = [L.lopc_ref_ord(int(v), 0) for v in vals.view(np.uint32)]
    assert o[3] == o[4] == 0
    assert all(o[i] < o[i + 1] for i in range(len(o) - 1) if i != 3)
    # adjacent floats differ by exactly one in ord (decode rule P:314 "next lowest")
    a = np.float32(1.5)
    assert L.lopc_ref_ord(int(np.nextafter(a, np.float32(2)).view(np.uint32)), 0) - L.lopc_ref_ord(
        int(a.view(np.uint32)), 0) == 1
    assert L.lopc_ref_ord(int(np.float32(-1e-45).view(np.uint32)), 0) == -1
