"""NEXT f4: the OpenMP CPU baseline (oracle/lopc_omp.c) must produce the
single-thread oracle's bytes (same definitions, parallel schedule; G14)."""
import numpy as np
import pytest

from synth.fields import CONFIGS, eps_noa, random_field


@pytest.mark.parametrize("seed,kind", [(s, k) for s in range(4) for k in ("noise", "smooth", "ties", "grid16")])
def test_omp_equals_oracle(ref, seed, kind):
    rng = np.random.default_rng(300 + seed)
    dims = (int(rng.integers(1, 16)), int(rng.integers(1, 30)), int(rng.integers(1, 70))) if seed % 2 else \
        (int(rng.integers(1, 70)), int(rng.integers(1, 120)))
    dt = "f64" if seed == 2 else "f32"
    x = random_field(dims, dt, kind, seed)
    x.reshape(-1)[:3] = [np.nan, np.inf, 1e30] if x.size >= 3 else x.reshape(-1)[:3]
    eps = eps_noa(x, [1e-1, 1e-2, 1e-3, 1.0][seed])
    st, sweeps = ref.omp_compress(x, eps, threads=4)
    assert st == ref.compress(x, eps)
    assert sweeps >= 1


def test_omp_chain_and_config(ref):
    x = (1.0 - 1e-6 * np.arange(400)).astype(np.float32).reshape(1, 400)
    st, sweeps = ref.omp_compress(x, 1.0, threads=3)
    assert st == ref.compress(x, 1.0)
    cfg = CONFIGS["cfg4"]
    y = cfg.generate((180, 360))
    eps = eps_noa(y, cfg.rel)
    assert ref.omp_compress(y, eps)[0] == ref.compress(y, eps)
