"""Row a0 (NOA): the oracle's finite min/max and eps = rel * range,
pinned to numpy's own reductions (an independent library routine) and to
special cases."""
import numpy as np
import pytest

from synth.fields import CONFIGS, eps_noa, random_field


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("seed", range(6))
def test_range_matches_numpy(ref, dt, seed):
    rng = np.random.default_rng(seed)
    x = random_field((int(rng.integers(1, 40)), int(rng.integers(1, 60))), dt, "noise", seed) * 1e3
    flat = x.reshape(-1)
    k = int(rng.integers(0, max(1, flat.size // 3)))
    pos = rng.choice(flat.size, size=k, replace=False)
    flat[pos] = rng.choice([np.nan, np.inf, -np.inf], size=k)
    lo, hi, n = ref.value_range(x)
    fin = flat[np.isfinite(flat)]
    assert n == fin.size
    if fin.size:
        assert lo == float(np.min(fin)) and hi == float(np.max(fin))
        r = float(np.max(fin)) - float(np.min(fin))
        assert ref.noa_eps(x, 1e-3) == (1e-3 * r if r > 0 else 1e-3)


def test_special_cases(ref):
    assert ref.value_range(np.full((3, 4), np.nan, np.float32))[2] == 0
    assert ref.noa_eps(np.full((3, 4), np.nan, np.float32), 0.25) == 0.25  # no finite value: eps = rel
    assert ref.noa_eps(np.full((5, 5), 7.0), 0.1) == 0.1  # zero range
    x = np.array([[-2.5, 1.5], [np.inf, 0.0]], np.float32)
    assert ref.value_range(x) == (-2.5, 1.5, 3)
    assert ref.noa_eps(x, 0.5) == 2.0  # 0.5 * (1.5 - (-2.5)), exact
    z = np.array([[-0.0, 0.0]], np.float64)
    assert ref.noa_eps(z, 0.3) == 0.3


@pytest.mark.parametrize("name", ["cfg1", "cfg4"])
def test_configs_agree_with_caller_helper(ref, name):
    """synth.eps_noa (the caller-side a0 used by the bench and tests) and the
    oracle's a0 give the same double."""
    x = CONFIGS[name].generate()
    assert ref.noa_eps(x, CONFIGS[name].rel) == eps_noa(x, CONFIGS[name].rel)
