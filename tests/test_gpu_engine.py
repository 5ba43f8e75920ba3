"""NEXT f2: the paper's point-worklist schedule as the GPU repair
engine must reach the same least fixpoint as the default tile engine and the
oracle (G14), hence the same bytes."""
import numpy as np
import pytest

from synth.fields import CONFIGS, eps_noa, random_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: -m gpu tests must run on a B200")
    import paper_2603_26968_b200 as lopc

    lopc.load()
    lopc.set_repair_engine(1)
    yield lopc
    lopc.set_repair_engine(0)


def _t(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("seed,kind", [(s, k) for s in range(4) for k in ("noise", "smooth", "ties", "grid16")])
def test_worklist_engine_equals_oracle(ref, gpu, seed, kind):
    rng = np.random.default_rng(900 + seed)
    dims = (int(rng.integers(1, 20)), int(rng.integers(1, 40)), int(rng.integers(1, 90))) if seed % 2 else \
        (int(rng.integers(1, 80)), int(rng.integers(1, 150)))
    dt = "f64" if seed == 3 else "f32"
    x = random_field(dims, dt, kind, seed)
    eps = eps_noa(x, [1e-1, 1e-2, 1e-3, 1.0][seed])
    _, s = gpu.repair(_t(x), eps)
    assert np.array_equal(s.cpu().numpy().view(np.uint32), ref.subbins(x, eps))
    assert gpu.compress(_t(x), eps).cpu().numpy().tobytes() == ref.compress(x, eps)


def test_worklist_engine_chains_and_config(ref, gpu):
    x = (1.0 - 1e-6 * np.arange(3000)).astype(np.float32).reshape(1, 3000)
    assert gpu.compress(_t(x), 1.0).cpu().numpy().tobytes() == ref.compress(x, 1.0)
    st = gpu.last_stats()
    assert st["max_subbin"] == 2999 and st["pass_items"][1] == 3000
    cfg = CONFIGS["cfg4"]
    y = cfg.generate((180, 360))
    eps = eps_noa(y, cfg.rel)
    assert gpu.compress(_t(y), eps).cpu().numpy().tobytes() == ref.compress(y, eps)
