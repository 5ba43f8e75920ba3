"""cfg5's input generator (synth/turbulence.py) on the CPU: seeded, pointwise
in global coordinates (any z-range alone gives the same values), the blocked
DGEMM factorisation equals the direct mode sum, and the mode amplitudes follow
the Kolmogorov recipe of DESIGN.md §6 (a_m ~ k_m^(-1/3) at log spacing, unit
variance)."""
import math

import numpy as np

from synth import turbulence as turb


def test_modes_are_seeded_and_kolmogorov():
    k1, p1, a1 = turb.modes(5)
    k2, p2, a2 = turb.modes(5)
    assert np.array_equal(k1, k2) and np.array_equal(p1, p2) and np.array_equal(a1, a2)
    k3, _, _ = turb.modes(6)
    assert not np.array_equal(k1, k3)
    kmag = np.linalg.norm(k1, axis=1)
    assert np.allclose(kmag[0], 2 * math.pi / 2048) and np.allclose(kmag[-1], math.pi / 2)
    # log-spaced: constant ratio; amplitudes ~ k^(-1/3); unit variance
    r = kmag[1:] / kmag[:-1]
    assert np.allclose(r, r[0])
    slope = np.polyfit(np.log(kmag), np.log(a1), 1)[0]
    assert abs(slope + 1.0 / 3.0) < 1e-9
    assert abs(0.5 * float(np.sum(a1 * a1)) - 1.0) < 1e-12
    assert np.all((p1 >= 0) & (p1 < 2 * math.pi))


def test_blocked_product_equals_mode_sum_and_is_pointwise():
    a = turb.planes_torch(30, 35, 17, 23, device="cpu").numpy()
    b = turb.planes_numpy(30, 35, 17, 23)
    assert np.abs(a - b).max() < 1e-11
    # a sub-range built alone equals the same planes of a larger build
    c = turb.planes_torch(32, 34, 17, 23, device="cpu").numpy()
    assert np.abs(c - a[2:4]).max() < 1e-11


def test_eps_from_range():
    assert turb.eps_noa_range(-2.0, 3.0, 1e-5) == np.float64(1e-5) * np.float64(5.0)
    assert turb.eps_noa_range(1.0, 1.0, 1e-5) == 1e-5
