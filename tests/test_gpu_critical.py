"""NEXT f3: the GPU critical-point verifier (k_critical) against the brute
force of tests/exact.py (explicit Kuhn simplices, link graphs, union-find;
Table III semantics P:396) on small grids — clean decodes (0/0/0) and damaged
ones (teeth) — and 0/0/0 on full-size configs."""
import numpy as np
import pytest

from synth.fields import CONFIGS, eps_noa, random_field
from tests.exact import classify, fp_fn_ft

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


@pytest.mark.parametrize("shape,dt,kind", [((5, 6, 7), "f32", "smooth"), ((4, 5, 9), "f64", "ties"),
                                           ((12, 15), "f32", "noise"), ((9, 11), "f64", "plateau"),
                                           ((3, 1, 8), "f32", "noise")])
def test_equals_brute_force(ref, gpu, shape, dt, kind):
    x = random_field(shape, dt, kind, 6)
    eps = eps_noa(x, 0.05)
    y = ref.decompress(ref.compress(x, eps))
    rng = np.random.default_rng(2)
    bad = (y + np.asarray(eps * 2, y.dtype) * rng.standard_normal(y.shape).astype(y.dtype)).astype(y.dtype)
    for z in (y, bad):
        fp, fn, ft, pm = fp_fn_ft(x, z)
        r = gpu.critical_points(_t(x), _t(z))
        assert (r["false_positives"], r["false_negatives"], r["false_types"], r["pair_mismatches"]) == (fp, fn, ft, pm)
        tx, _ = classify(x)
        assert r["critical_x"] == sum(t != "regular" for t in tx)
    assert fp_fn_ft(x, y)[:3] == (0, 0, 0)


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_configs_preserve_critical_points(gpu, name):
    cfg = CONFIGS[name]
    x = cfg.generate()
    eps = eps_noa(x, cfg.rel)
    xt = _t(x)
    y = gpu.decompress(gpu.compress(xt, eps))
    r = gpu.critical_points(xt, y)
    assert (r["false_positives"], r["false_negatives"], r["false_types"], r["pair_mismatches"]) == (0, 0, 0, 0)
    assert r["critical_x"] > 0
