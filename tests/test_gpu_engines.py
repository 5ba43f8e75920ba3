"""Every repair engine and index width reaches the oracle's least fixpoint
(reading G14: any monotone relaxation schedule gives the unique least
fixpoint O9), hence the oracle's bytes:

  engine 0  tile fixpoints over alternating half-shifted tilings (k_tiles,
            subbin bit planes; the default), with its 8-plane overflow
            falling back to engine 2;
  engine 2  round 1's dense tile pass + point worklist (k_sweep, u32);
  index64   k_quant_flags / k_sweep in their int64 index builds (otherwise
            used only from N >= 2^31 - 2^24: cfg5 slabs at N > 1).
(Engine 1, the paper's own point worklist, is tests/test_gpu_engine.py.)"""
import numpy as np
import pytest

from synth.fields import CONFIGS, eps_noa, random_field

pytestmark = pytest.mark.gpu

MODES = [(0, False), (0, True), (2, False), (2, True)]


@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: -m gpu tests must run on a B200")
    import paper_2603_26968_b200 as lopc

    lopc.load()
    yield lopc
    lopc.set_repair_engine(0)
    lopc.set_index64(False)


def _t(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _mode(gpu, engine, i64):
    gpu.set_repair_engine(engine)
    gpu.set_index64(i64)


CASES = [(s, k) for s in range(6) for k in ("noise", "smooth", "ties", "grid16", "signed_zero_subnormal")]


@pytest.mark.parametrize("engine,i64", MODES)
@pytest.mark.parametrize("seed,kind", CASES[::3])
def test_engines_equal_oracle(ref, gpu, engine, i64, seed, kind):
    _mode(gpu, engine, i64)
    rng = np.random.default_rng(1300 + seed)
    dims = (int(rng.integers(1, 24)), int(rng.integers(1, 40)), int(rng.integers(1, 100))) if seed % 2 else \
        (int(rng.integers(1, 90)), int(rng.integers(1, 170)))
    dt = "f64" if seed % 3 == 0 else "f32"
    x = random_field(dims, dt, kind, seed)
    if seed == 4:
        x.ravel()[:: max(1, x.size // 7)] = np.inf  # escapes inside tiles
    eps = eps_noa(x, [1e-1, 1e-2, 1e-3, 1.0, 1e-2, 1e-1][seed])
    f, s = gpu.repair(_t(x), eps)
    assert np.array_equal(f.cpu().numpy().view(np.uint16), ref.flags(x, eps))
    assert np.array_equal(s.cpu().numpy().view(np.uint32), ref.subbins(x, eps))
    assert gpu.compress(_t(x), eps).cpu().numpy().tobytes() == ref.compress(x, eps)


@pytest.mark.parametrize("engine,i64", MODES)
def test_engines_config_shaped(ref, gpu, engine, i64):
    _mode(gpu, engine, i64)
    for name, small in (("cfg2", (20, 100, 100)), ("cfg3", (48, 64, 64)), ("cfg4", (180, 360))):
        cfg = CONFIGS[name]
        x = cfg.generate(small)
        eps = eps_noa(x, cfg.rel)
        assert gpu.compress(_t(x), eps).cpu().numpy().tobytes() == ref.compress(x, eps), name


def test_tile_engine_plane_overflow_falls_back(ref, gpu):
    """A subbin above 254 does not fit the tile engine's 8 planes: the call
    re-runs on the u32 engine and still returns the oracle's bytes (a
    decreasing chain of 700 points in one bin: subbins 699..0)."""
    _mode(gpu, 0, False)
    x = (1.0 - 1e-6 * np.arange(700)).astype(np.float32).reshape(1, 700)
    assert gpu.compress(_t(x), 1.0).cpu().numpy().tobytes() == ref.compress(x, 1.0)
    assert gpu.last_stats()["max_subbin"] == 699
    y = (1.0 - 1e-6 * np.arange(200)).astype(np.float32).reshape(1, 200)  # fits: stays on the tile engine
    assert gpu.compress(_t(y), 1.0).cpu().numpy().tobytes() == ref.compress(y, 1.0)
    assert gpu.last_stats()["max_subbin"] == 199


@pytest.mark.parametrize("decoder", [1, 2])
def test_decoders_equal_oracle(ref, gpu, decoder):
    """Both decoders (one CTA per chunk; 2-CTA clusters) give the oracle's
    bits on f32 / f64 fields with escapes, raw chunks and ragged tails, from
    device and host streams; a truncated stream is E_CORRUPT for both."""
    import torch

    gpu.set_repair_engine(0)
    gpu.set_decoder(decoder)
    try:
        fields = [CONFIGS["cfg2"].generate((20, 100, 100)), random_field((70, 300), "f64", "smooth", 3),
                  random_field((9, 31, 77), "f32", "noise", 5) * np.float32(1e6)]
        fields[1].ravel()[::97] = np.nan
        for x in fields:
            eps = eps_noa(x, 1e-3)
            st = ref.compress(x, eps)
            y = ref.decompress(st).tobytes()
            dev = torch.from_numpy(np.frombuffer(st, np.uint8).copy()).cuda()
            assert gpu.decompress(dev).cpu().numpy().tobytes() == y
            host = torch.from_numpy(np.frombuffer(st, np.uint8).copy()).pin_memory()
            out = torch.empty(x.shape, dtype=torch.float32 if x.dtype == np.float32 else torch.float64).pin_memory()
            assert gpu.decompress(host, out=out).numpy().tobytes() == y
            with pytest.raises(gpu.LopcError):
                gpu.decompress(dev[:-4])
    finally:
        gpu.set_decoder(1)
