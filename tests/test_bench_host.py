"""bench.py host helpers (CPU): the bounded oracle crop, the weak-scaling
tiling of a config along z (mirrored copies keep the field continuous and the
value range, hence the NOA eps, unchanged), and the workload table."""
import numpy as np

import bench
from synth.fields import CONFIGS, eps_noa


def test_workloads_cover_every_config():
    assert set(bench.WORKLOAD) == set(CONFIGS)


def test_crop_is_bounded():
    for shape in [(100, 500, 500), (512, 512, 512), (1800, 3600), (1, 2048, 2048), (64, 64)]:
        x = np.zeros(shape, np.float32)
        p = bench.crop_planes(x)
        assert 1 <= p <= shape[0]
        assert p * int(np.prod(shape[1:])) <= max(2 << 20, int(np.prod(shape[1:])))


def test_tiled_slabs_are_mirrored_copies():
    base = np.arange(3 * 4 * 5, dtype=np.float32).reshape(3, 4, 5)
    shape = (9, 4, 5)  # 3 copies along z
    full = bench.slab_values(base, shape, 0, 9 * 20).reshape(shape)
    assert np.array_equal(full[0:3], base)
    assert np.array_equal(full[3:6], base[::-1])  # mirrored: plane 2 meets plane 2
    assert np.array_equal(full[6:9], base)
    assert eps_noa(full, 1e-3) == eps_noa(base, 1e-3)
    # any element range equals the same slice of the whole field
    for e0, e1 in [(0, 1), (7, 61), (59, 121), (100, 180)]:
        assert np.array_equal(bench.slab_values(base, shape, e0, e1), full.reshape(-1)[e0:e1])
