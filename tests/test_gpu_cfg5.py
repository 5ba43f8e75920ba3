"""cfg5 (BASELINE.json configs[4]: 3D f64 2048^3 turbulence, NOA 1e-5, sharded
as z-slabs across 8 B200) on one B200.

The whole field (64 GiB) is an 8-GPU workload; what one GPU runs of it is one
rank's slab, 2048 x 2048 x 256 f64 (1.07 G points, 8.6 GB, 524,288 chunks).
Parity at that size is proven without the oracle compressing 1 G points:
  * the GPU subbins satisfy the Bellman equation at every point
    (oracle lopc_ref_certify), so they ARE the unique least fixpoint (O9);
  * the decoded field equals the oracle's O10 reconstruction bit for bit;
  * EVERY chunk of the stream equals the oracle's chunk encoder byte for byte
    (lopc_omp_check_chunks, plus the header, size table and total length);
  * zero order / bound violations (oracle checkers).
The 8-way slab decomposition (halo rounds across slab boundaries) is checked on
a 64-plane crop of the same field in 8 slabs: byte-identical to the
single-GPU stream of the crop, which is certified the same way.
eps is cfg5's: 1e-5 x the range of the full 2048^3 field (found block by block
on the device, never materialised)."""
import numpy as np
import pytest

from synth import turbulence as turb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: -m gpu tests must run on a B200")
    import paper_2603_26968_b200 as lopc

    lopc.load()
    return lopc


@pytest.fixture(scope="module")
def eps5():
    lo, hi = turb.field_range(*turb.CFG5_DIMS)
    return turb.eps_noa_range(lo, hi, turb.CFG5_REL)


def test_generator_is_the_mode_sum():
    """The GPU generator (blocked DGEMM factorisation) equals the direct mode
    sum on a crop that straddles a block boundary."""
    a = turb.planes_torch(14, 19, 33, 70).cpu().numpy()
    b = turb.planes_numpy(14, 19, 33, 70)
    assert np.abs(a - b).max() < 1e-11


def _certify_field(ref, gpu, xt, eps):
    """Certificate-based parity of one field at any size (see module doc)."""
    x = xt.cpu().numpy()
    _, s = gpu.repair(xt, eps)
    s = s.cpu().numpy().view(np.uint32)
    assert ref.certify(x, eps, s) == 0
    st = gpu.compress(xt, eps)
    y = gpu.decompress(st)
    yh = y.cpu().numpy()
    del y
    assert yh.tobytes() == ref.reconstruct(x, eps, s).tobytes()
    if x.size <= (1 << 28):
        assert ref.order_violations(x, yh) == 0
        assert ref.bound_violations(x, yh, eps) == 0
    else:  # 1 G points: the device checker (k_check == the oracle checkers, test_gpu_check.py)
        chk = gpu.check(xt, gpu.decompress(st), eps)
        assert chk["order_violations"] == 0 and chk["bound_violations"] == 0
    stb = st.cpu().numpy().tobytes()
    # every chunk (and the header, table and total length) against the
    # oracle's chunk encoder on the certified subbins, all host cores
    assert ref.omp_check_chunks(x, eps, s, stb) == (0, None)
    return stb


@pytest.mark.slow
def test_cfg5_rank_slab_full_size(ref, gpu, eps5):
    """One rank's slab of the 8-GPU cfg5 layout (planes 768..1023), at full
    per-GPU size."""
    import torch

    xt = turb.planes_torch(768, 1024, 2048, 2048)
    stb = _certify_field(ref, gpu, xt, eps5)
    assert len(stb) < xt.numel() * 8  # compresses
    del xt
    torch.cuda.empty_cache()


def test_cfg5_eight_slabs_crop(ref, gpu, eps5):
    """8 slabs of 8 planes (the cfg5 partition pattern: whole 2048^2 planes,
    chunk-aligned) through the slab algorithm == the single-GPU stream, which
    is certified."""
    import torch

    xt = turb.planes_torch(0, 64, 2048, 2048)
    bounds = gpu.slab_partition(tuple(xt.shape), torch.float64, 8)
    P = 2048 * 2048
    assert all(b % P == 0 for b in bounds)
    st8 = gpu.compress_slabs_local(xt, eps5, bounds).cpu().numpy().tobytes()
    st1 = _certify_field(ref, gpu, xt, eps5)
    assert st8 == st1
