"""Row a0 / NEXT f1 on the GPU: k_value_range (finite min/max in one read)
and lopc_compress_noa against the oracle's a0 and stream."""
import numpy as np
import pytest

from synth.fields import CONFIGS, random_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: -m gpu tests must run on a B200")
    import paper_2603_26968_b200 as lopc

    lopc.load()
    return lopc


def _t(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("seed", range(5))
def test_value_range(ref, gpu, dt, seed):
    rng = np.random.default_rng(seed)
    shape = (int(rng.integers(1, 30)), int(rng.integers(1, 50)), int(rng.integers(1, 90)))
    x = random_field(shape, dt, "noise", seed) * 100
    flat = x.reshape(-1)
    k = int(rng.integers(0, max(1, flat.size // 4)))
    flat[rng.choice(flat.size, size=k, replace=False)] = rng.choice([np.nan, np.inf, -np.inf], size=k)
    assert gpu.value_range(_t(x)) == ref.value_range(x)


def test_value_range_edges(ref, gpu):
    for x in [np.full((4, 5), np.nan, np.float32), np.full((3, 3, 3), -0.0), np.array([[np.inf, 2.0]], np.float32),
              np.arange(7, dtype=np.float32).reshape(1, 7)[:, 1:]]:
        assert gpu.value_range(_t(x)) == ref.value_range(x)


@pytest.mark.parametrize("name", ["cfg1", "cfg4", "cfg2"])
def test_compress_noa(ref, gpu, name):
    cfg = CONFIGS[name]
    x = cfg.generate()
    st, eps = gpu.compress_noa(_t(x), cfg.rel)
    assert eps == ref.noa_eps(x, cfg.rel)
    if x.size <= 7_000_000:
        assert st.cpu().numpy().tobytes() == ref.compress(x, eps)
    else:
        assert st.cpu().numpy().tobytes() == gpu.compress(_t(x), eps).cpu().numpy().tobytes()
