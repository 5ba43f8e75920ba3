"""GPU parity of the multi-GPU slab mode on one B200: the slab
algorithm (box + ghosts + per-round halo exchange + injection + sparse
re-sweeps, then per-slab encode and offset assembly) through
lopc_compress_slabs_local (device copies instead of NCCL, same code) and
lopc_compress_slab (world 1, with and without an NCCL communicator) must give
the oracle's single stream byte for byte; lopc_decompress_slab must give the
oracle's decoded values for every range."""
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


CASES = [((24, 40, 50), "f32", "smooth", 2), ((24, 40, 50), "f64", "ties", 3), ((30, 60, 70), "f32", "noise", 4),
         ((400, 300), "f32", "smooth", 3), ((600, 130), "f64", "plateau", 2), ((40, 64, 64), "f32", "grid16", 4)]


@pytest.fixture
def engine(gpu, request):
    """Slab mode on the tile engine (0, the default) or the u32 engine (2)."""
    gpu.set_repair_engine(request.param)
    yield request.param
    gpu.set_repair_engine(0)


@pytest.mark.parametrize("engine", [0, 2], indirect=True)
@pytest.mark.parametrize("shape,dt,kind,world", CASES)
def test_slabs_local_equal_oracle(ref, gpu, engine, shape, dt, kind, world):
    x = random_field(shape, dt, kind, 11)
    eps = eps_noa(x, 1e-2)
    st_ref = ref.compress(x, eps)
    import torch

    tdt = torch.float32 if dt == "f32" else torch.float64
    bounds = gpu.slab_partition(shape, tdt, world)
    st = gpu.compress_slabs_local(_t(x), eps, bounds).cpu().numpy().tobytes()
    assert st == st_ref


@pytest.mark.parametrize("engine", [0, 2], indirect=True)
def test_chains_cross_slab_boundaries(ref, gpu, engine):
    """Decreasing ramps along the linear order: subbins n-1..0 must flow
    across every slab boundary (several exchange rounds).  Subbins reach
    23999: on the tile engine the call overflows the 8 subbin planes and
    every slab re-runs on the u32 engine (same bytes)."""
    x = (1.0 - 1e-7 * np.arange(30 * 20 * 40)).astype(np.float32).reshape(30, 20, 40)
    for world in (2, 3, 5):
        import torch

        bounds = gpu.slab_partition(x.shape, torch.float32, world)
        st = gpu.compress_slabs_local(_t(x), 1.0, bounds).cpu().numpy().tobytes()
        assert st == ref.compress(x, 1.0)
        assert gpu.last_stats()["inner_iters"] >= 2  # repair rounds
    y = (1.0 - 1e-6 * np.arange(500 * 33)).astype(np.float32).reshape(500, 33)
    bounds = gpu.slab_partition(y.shape, torch.float32, 4)
    assert gpu.compress_slabs_local(_t(y), 1.0, bounds).cpu().numpy().tobytes() == ref.compress(y, 1.0)


@pytest.mark.parametrize("engine", [0, 2], indirect=True)
@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_slab_escapes(ref, gpu, engine, dt):
    """NaN, +-Inf and out-of-range values (escapes, G8-G11) in several slabs,
    one beside a slab boundary: the slab encoder (planes mode on the tile
    engine) must store them raw exactly as the oracle does."""
    import torch

    x = random_field((24, 40, 50), dt, "smooth", 8)
    eps = eps_noa(x, 1e-2)
    big = 3e38 if dt == "f32" else 1e300
    n = x.size
    for i, v in zip([0, 7, n // 3, n // 2 - 1, n // 2, 2 * n // 3 + 5, n - 1],
                    [np.nan, np.inf, -np.inf, big, np.nan, -big, np.inf]):
        x.ravel()[i] = v
    tdt = torch.float32 if dt == "f32" else torch.float64
    for world in (2, 3):
        bounds = gpu.slab_partition(x.shape, tdt, world)
        st = gpu.compress_slabs_local(_t(x), eps, bounds).cpu().numpy().tobytes()
        assert st == ref.compress(x, eps), world


@pytest.mark.parametrize("engine", [0, 2], indirect=True)
def test_short_chains_cross_slab_boundaries(ref, gpu, engine):
    """Repeated decreasing ramps of 200 points (subbins 199..0: they fit the
    tile engine's planes) cut by every slab boundary: ghosts raised over
    several rounds, injected into the planes and re-swept from the marked
    tiles, must give the oracle's bytes."""
    import torch

    x = (1.0 - 1e-7 * (np.arange(24 * 30 * 40) % 200)).astype(np.float32).reshape(24, 30, 40)
    y = (1.0 - 1e-6 * (np.arange(300 * 70) % 230)).astype(np.float32).reshape(300, 70)
    for z in (x, y):
        st_ref = ref.compress(z, 1.0)
        for world in (2, 3, 5):
            bounds = gpu.slab_partition(z.shape, torch.float32, world)
            st = gpu.compress_slabs_local(_t(z), 1.0, bounds).cpu().numpy().tobytes()
            assert st == st_ref, (z.shape, world)
            assert gpu.last_stats()["max_subbin"] < 255


@pytest.mark.parametrize("name,world", [("cfg2s", 3), ("cfg4s", 2), ("cfg2", 4)])
def test_slabs_local_configs(ref, gpu, name, world):
    import torch

    small = {"cfg2s": (20, 100, 100), "cfg4s": (180, 360), "cfg2": None}[name]
    cfg = CONFIGS[name[:4]]
    x = cfg.generate(small)
    eps = eps_noa(x, cfg.rel)
    bounds = gpu.slab_partition(x.shape, torch.float32, world)
    st = gpu.compress_slabs_local(_t(x), eps, bounds).cpu().numpy().tobytes()
    if small is None:  # full size: equal to the single-GPU call (itself oracle-equal, test_gpu_parity)
        assert st == gpu.compress(_t(x), eps).cpu().numpy().tobytes()
    else:
        assert st == ref.compress(x, eps)


def test_compress_slab_world1_and_nccl(ref, gpu):
    import torch

    x = random_field((20, 50, 60), "f32", "smooth", 5)
    eps = eps_noa(x, 1e-3)
    xt = _t(x)
    full = gpu.compress(xt, eps).cpu().numpy().tobytes()
    loc, po, tot = gpu.compress_slab(None, xt.reshape(-1), x.shape, eps, 0, x.size)
    hdr = gpu.write_header(x.shape, torch.float32, eps, tot)
    assert hdr + loc.cpu().numpy().tobytes() == full and po == 64 + 8 * ((x.size + 4095) // 4096)
    comm = gpu.Comm(1, 0, gpu.comm_unique_id())
    try:
        loc2, po2, tot2 = gpu.compress_slab(comm, xt.reshape(-1), x.shape, eps, 0, x.size)
        assert (po2, tot2) == (po, tot) and torch.equal(loc2, loc)
    finally:
        comm.close()


@pytest.mark.parametrize("shape,dt,world", [((24, 40, 50), "f32", 3), ((600, 130), "f64", 2)])
def test_decompress_slab_ranges(ref, gpu, shape, dt, world):
    import torch

    from paper_2603_26968_b200 import dist as ldist

    x = random_field(shape, dt, "smooth", 9)
    eps = eps_noa(x, 1e-2)
    st = ref.compress(x, eps)
    y_ref = ref.decompress(st).reshape(-1)
    tdt = torch.float32 if dt == "f32" else torch.float64
    b = gpu.slab_partition(shape, tdt, world)
    W = 16384 // x.itemsize
    sizes = ref.chunk_sizes(st)
    C = len(sizes)
    pay_off = 64 + 8 * C + np.concatenate([[0], np.cumsum(sizes.sum(axis=1))])
    for r in range(world):
        c0, c1 = b[r] // W, -(-b[r + 1] // W)
        local = st[64 + 8 * c0:64 + 8 * c1] + st[int(pay_off[c0]):int(pay_off[c1])]
        tab, pay = ldist.split_local(local, c1 - c0)
        assert len(tab) == 8 * (c1 - c0)
        y = gpu.decompress_slab(st[:64], _t(np.frombuffer(local, np.uint8).copy()), b[r], b[r + 1], tdt)
        assert y.cpu().numpy().tobytes() == y_ref[b[r]:b[r + 1]].tobytes()
