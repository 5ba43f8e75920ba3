"""k_check on the GPU: order and bound violation counts equal
the oracle's checkers (O13) exactly, on clean decodes (0/0) and on decodes
damaged on purpose (teeth); error statistics against numpy."""
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
    return lopc


def _t(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("shape,dt,kind", [((12, 20, 40), "f32", "smooth"), ((9, 17, 33), "f64", "ties"),
                                           ((70, 90), "f32", "noise"), ((50, 64), "f64", "plateau")])
def test_counts_equal_oracle(ref, gpu, shape, dt, kind):
    x = random_field(shape, dt, kind, 4)
    x.reshape(-1)[[3, 50]] = [np.nan, np.inf]
    eps = eps_noa(x, 1e-2)
    y = ref.decompress(ref.compress(x, eps))
    r = gpu.check(_t(x), _t(y), eps)
    assert r["order_violations"] == 0 and r["bound_violations"] == 0
    reg = np.isfinite(x)
    d = (x.astype(np.float64) - y.astype(np.float64))[reg]
    assert r["max_abs_err"] == float(np.max(d)) and r["n_regular"] == int(reg.sum())
    assert np.isclose(r["sum_sq_err"], float(np.sum(d * d)), rtol=1e-12)
    # teeth: mid-bin / shuffled decodes must be caught with the oracle's exact counts
    rng = np.random.default_rng(1)
    z = y.copy()
    flat = z.reshape(-1)
    idx = rng.choice(flat.size, size=flat.size // 7, replace=False)
    flat[idx] = flat[rng.permutation(idx)]
    z2 = (y + np.asarray(eps * 0.6, y.dtype) * rng.standard_normal(y.shape).astype(y.dtype)).astype(y.dtype)
    for bad in (z, z2):
        r = gpu.check(_t(x), _t(bad), eps)
        assert r["order_violations"] == ref.order_violations(x, bad)
        assert r["bound_violations"] == ref.bound_violations(x, bad, eps)
        assert r["order_violations"] > 0 and r["bound_violations"] > 0


def test_config2_clean(ref, gpu):
    cfg = CONFIGS["cfg2"]
    x = cfg.generate()
    eps = eps_noa(x, cfg.rel)
    xt = _t(x)
    y = gpu.decompress(gpu.compress(xt, eps))
    r = gpu.check(xt, y, eps)
    assert r["order_violations"] == 0 and r["bound_violations"] == 0 and r["max_abs_err"] < eps
