"""The paper's guarantees, checked by brute force on the oracle's round trip:
error bound, full local order, critical points and
their types (Table III: LOPC 0/0/0), stability (proof (v) in
DESIGN.md), and a 'teeth' test that the checkers catch a degraded decode."""
import math
from fractions import Fraction

import numpy as np
import pytest

from synth.fields import CONFIGS, eps_noa, random_field
from tests.exact import fp_fn_ft


def _exact_bound_ok(x, y, eps):
    for a, b in zip(x.ravel(), y.ravel()):
        if not np.isfinite(a):
            if a.tobytes() != b.tobytes():
                return False
            continue
        if abs(Fraction(float(a)) - Fraction(float(b))) > Fraction(eps):
            return False
    return True


CASES = [(seed, kind, rel) for seed in range(8) for kind in ("noise", "smooth", "ties", "plateau", "grid16", "signed_zero_subnormal")
         for rel in (0.1, 0.01)]


@pytest.mark.parametrize("seed,kind,rel", CASES)
def test_round_trip_guarantees(ref, seed, kind, rel):
    rng = np.random.default_rng(seed)
    dims = (12, 12) if seed % 2 == 0 else (5, 6, 6)
    dt = "f32" if seed % 4 != 3 else "f64"
    x = random_field(dims, dt, kind, seed + 77)
    eps = eps_noa(x, rel)
    stream = ref.compress(x, eps)
    y = ref.decompress(stream)
    assert y.shape == x.shape and y.dtype == x.dtype
    assert _exact_bound_ok(x, y, eps)
    assert ref.bound_violations(x, y, eps) == 0
    assert ref.order_violations(x, y) == 0
    fp, fn, ft, pairs = fp_fn_ft(x, y)
    assert (fp, fn, ft, pairs) == (0, 0, 0, 0)
    # decompress(compress(x)) is exactly the O10 reconstruction of the fixpoint
    s = ref.subbins(x, eps)
    assert ref.reconstruct(x, eps, s).tobytes() == y.tobytes()
    # one-sided error (proof (i)): lo(b) <= x^ <= x
    fin = np.isfinite(x)
    assert (y[fin] <= x[fin]).all()


def test_config1_guarantees(ref):
    cfg = CONFIGS["cfg1"]
    x = cfg.generate()
    eps = eps_noa(x, cfg.rel)
    y = ref.decompress(ref.compress(x, eps))
    assert ref.bound_violations(x, y, eps) == 0
    assert ref.order_violations(x, y) == 0
    assert fp_fn_ft(x, y) == (0, 0, 0, 0)
    s = ref.subbins(x, eps)
    assert s.max() > 0  # the eps/16 snap makes the repair do work


def test_teeth_midbin_decode_is_caught(ref):
    """Decoding every point to its bin centre without subbins (the
    'normal' decode) must break order and critical points on a noisy field —
    proves the checkers detect errors."""
    x = random_field((12, 12), "f32", "noise", 5)
    eps = eps_noa(x, 0.1)
    b = ref.quantize(x, eps)
    y = (b.astype(np.float64) * eps).astype(np.float32)
    assert ref.order_violations(x, y) > 0
    fp, fn, ft, pairs = fp_fn_ft(x, y)
    assert fp + fn + ft > 0 and pairs > 0


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_stability_with_escapes(ref, dt):
    """C(D(C(x))) == C(x) byte-for-byte and D(C(D(C(x)))) == D(C(x))."""
    x = random_field((9, 11), dt, "noise", 3)
    x.ravel()[[3, 17, 40]] = [np.inf, -np.inf, np.nan]
    x.ravel()[50] = np.finfo(x.dtype).max  # |b| > BINMAX -> escaped (G8)
    eps = 0.05
    c1 = ref.compress(x, eps)
    y1 = ref.decompress(c1)
    assert y1.ravel()[[3, 17, 40, 50]].tobytes() == x.ravel()[[3, 17, 40, 50]].tobytes()
    c2 = ref.compress(y1, eps)
    assert c1 == c2
    y2 = ref.decompress(c2)
    assert y1.tobytes() == y2.tobytes()
    assert ref.order_violations(x, y1) == 0


def test_negative_zero_decodes_positive(ref):
    x = np.array([[-0.0, 0.0, 1e-3]], np.float32)
    y = ref.decompress(ref.compress(x, 1.0))
    assert ref.bound_violations(x, y, 1.0) == 0
    assert ref.order_violations(x, y) == 0
