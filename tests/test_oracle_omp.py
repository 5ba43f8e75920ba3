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


def test_omp_check_chunks_teeth(ref):
    """lopc_omp_check_chunks (the whole-stream check used for the cfg5 rank
    slab) accepts the oracle's stream and finds a flipped payload byte, a
    wrong subbin and a wrong header field."""
    import struct

    from synth.fields import CONFIGS, eps_noa

    x = CONFIGS["cfg2"].generate((20, 100, 100))
    eps = eps_noa(x, 1e-3)
    st = ref.compress(x, eps)
    s = ref.subbins(x, eps)
    assert ref.omp_check_chunks(x, eps, s, st) == (0, None)
    b = bytearray(st)
    b[-5] ^= 1
    assert ref.omp_check_chunks(x, eps, s, bytes(b)) == (1, 48)
    s2 = s.copy()
    s2.ravel()[5000] += 1
    assert ref.omp_check_chunks(x, eps, s2, st) == (1, 1)
    h = bytearray(st)
    struct.pack_into("<d", h, 32, eps * 2)
    assert ref.omp_check_chunks(x, eps, s, bytes(h))[0] == 1


def test_omp_decompress_equals_oracle(ref):
    """The OpenMP decompress (chunks in parallel through the oracle's own
    per-chunk decoder) gives the oracle's bits; corrupt streams fail."""
    from synth.fields import CONFIGS, eps_noa, random_field

    for x in (CONFIGS["cfg2"].generate((20, 100, 100)), random_field((70, 300), "f64", "smooth", 3)):
        eps = eps_noa(x, 1e-3)
        st = ref.compress(x, eps)
        assert ref.omp_decompress(st).tobytes() == ref.decompress(st).tobytes()
        import oracle

        with pytest.raises(oracle.OracleError):
            ref.omp_decompress(st[:-4])
