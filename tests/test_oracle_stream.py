"""Pins for the lossless stages and the container: worked
examples, closed forms of negabinary and the bit transpose,
inverse round trips, level sizes, raw fallback and corrupt-stream handling."""
import struct

import numpy as np
import pytest

from synth.fields import eps_noa, random_field


def negabinary_value(u: int, bits: int) -> int:
    """Value of a word read as negabinary digits: sum_i d_i (-2)^i."""
    return sum(((u >> i) & 1) * (-2) ** i for i in range(bits))


def test_negabinary_closed_form(ref):
    # NB(-1) = 0x3, NB(2) = 0x6, NB(-2) = 0x2, NB(3) = 0x7
    w = np.array([-1, 0, 1, 2, -2, 3], np.int32).view(np.uint32)
    u = ref.diffnb(np.concatenate([[0], np.cumsum(w.astype(np.uint64)) % 2**32]).astype(np.uint32))[1:]
    assert list(u) == [0x3, 0x0, 0x1, 0x6, 0x2, 0x7]
    rng = np.random.default_rng(0)
    v = rng.integers(-2**20, 2**20, size=200)
    words = (np.cumsum(v) % 2**32).astype(np.uint32)
    enc = ref.diffnb(words)
    d = np.diff(np.concatenate([[0], words.astype(np.int64)])) % 2**32
    for ui, di in zip(enc, d):
        assert negabinary_value(int(ui), 32) % 2**32 == int(di)


def test_delta_examples(ref):
    # [5,5,5] -> [5,0,0]; [0,1,3] -> [0,1,2] (then negabinary)
    nb = lambda v: negabinary_value  # noqa: E731
    a = ref.diffnb(np.array([5, 5, 5], np.uint32))
    assert negabinary_value(int(a[0]), 32) == 5 and a[1] == 0 and a[2] == 0
    b = ref.diffnb(np.array([0, 1, 3], np.uint32))
    assert [negabinary_value(int(t), 32) for t in b] == [0, 1, 2]
    for dt in (np.uint32, np.uint64):
        r = np.random.default_rng(1).integers(0, 2**31, size=512).astype(dt)
        assert (ref.undiffnb(ref.diffnb(r)) == r).all()


def test_bitshuffle_pins(ref):
    # a single word 0x1 -> plane 0 bit 0 only
    w = np.zeros(8, np.uint32)
    w[0] = 1
    b = ref.bitshuffle(w)
    assert b[0] == 1 and b[1:].sum() == 0
    # independent transpose with numpy: plane j = bit j of every word, LSB-first
    rng = np.random.default_rng(2)
    for dt in (np.uint32, np.uint64):
        words = rng.integers(0, 2**32, size=256).astype(dt) * (dt(3) if dt == np.uint64 else dt(1))
        k = words.itemsize
        bits = np.unpackbits(words.view(np.uint8).reshape(-1, k), axis=1, bitorder="little")  # [W, 8k]
        planes = np.packbits(bits.T, axis=1, bitorder="little").ravel()
        assert (ref.bitshuffle(words) == planes).all()
        assert (ref.unbitshuffle(ref.bitshuffle(words), dt) == words).all()


def test_rze_example_and_sizes(ref):
    # [5,0,0,7] -> bitmap 1001b, payload [5,7]
    assert ref.rze(bytes([5, 0, 0, 7]), 1) == bytes([0b1001, 5, 7])
    # all-zero 16384-byte chunk: bitmap levels 2048 -> 256 -> 32 -> 4 bytes, all zero
    assert ref.rze(bytes(16384), 1) == bytes(4)
    # g = 4: 512 -> 64 -> 8 bytes
    assert ref.rze(bytes(16384), 4) == bytes(8)
    assert ref.rze(bytes(16384), 8) == bytes(4)  # 256 -> 32 -> 4
    # one non-zero byte at position 100 of 16384 (g = 1)
    d = bytearray(16384)
    d[100] = 9
    e = ref.rze(bytes(d), 1)
    # B0[12] = 0x10; B1 bits 12, 13 set (B0 changes at 12 and back at 13);
    # B2 bit 1 (B1[1] != B1[0]) and bit 2? B1[1] = 0x30, B1[2] = 0 -> bits 1,2;
    # B3 bit 0 (B2[0] = 0x06 != 0)... check by decoding instead of by hand:
    out, used = ref.unrze(e, 16384, 1)
    assert out == bytes(d) and used == len(e)
    assert e[-1] == 9


@pytest.mark.parametrize("g", [1, 4, 8])
def test_rze_round_trip_fuzz(ref, g):
    rng = np.random.default_rng(g)
    for trial in range(60):
        L = int(rng.integers(1, 300)) * g if trial % 3 else 16384
        kind = trial % 4
        if kind == 0:
            a = np.zeros(L, np.uint8)
        elif kind == 1:
            a = rng.integers(0, 256, L).astype(np.uint8)
        elif kind == 2:
            a = (rng.random(L) < 0.05) * rng.integers(1, 256, L)
        else:
            a = np.repeat(rng.integers(0, 3, L // g + 1), g)[:L]
        data = a.astype(np.uint8).tobytes()
        enc = ref.rze(data, g)
        out, used = ref.unrze(enc, L, g)
        assert out == data and used == len(enc)
        if len(enc) > 1:
            bad, rc = ref.unrze(enc[:-1], L, g)
            assert rc == -1


def _roundtrip(ref, x, eps):
    st = ref.compress(x, eps)
    y = ref.decompress(st)
    return st, y


def test_container_header_and_table(ref):
    x = random_field((70, 130), "f32", "smooth", 4)  # 9100 elements -> 3 chunks
    eps = eps_noa(x, 1e-2)
    st, y = _roundtrip(ref, x, eps)
    assert st[:4] == b"LOPC"
    ver, dt, nd = struct.unpack_from("<HBB", st, 4)
    assert (ver, dt, nd) == (1, 0, 2)
    d0, d1, d2 = struct.unpack_from("<QQQ", st, 8)
    assert (d0, d1, d2) == (1, 70, 130)
    (e,) = struct.unpack_from("<d", st, 32)
    assert e == eps
    n, cb, C, total = struct.unpack_from("<QIIQ", st, 40)
    assert (n, cb, C, total) == (9100, 16384, 3, len(st))
    sizes = ref.chunk_sizes(st)
    assert sizes.shape == (3, 2)
    assert 64 + 8 * 3 + int(sizes.sum()) == len(st)
    assert all(4 <= v <= 16384 and v % 4 == 0 for v in sizes.ravel())


def test_all_zero_and_raw_fallback(ref):
    z = np.zeros((64, 64), np.float32)
    st = ref.compress(z, 1.0)
    assert list(ref.chunk_sizes(st)[0]) == [4, 4]  # A.6: 4 B bins, 3 B -> 4 B subbins
    # subbin 0 decodes to the lowest value of bin 0 = lo(0) = -eps/2
    assert (ref.decompress(st) == np.float32(-0.5)).all()
    # incompressible: random bins everywhere -> raw bins
    r = random_field((64, 64), "f32", "noise", 9) * np.float32(1e6)
    st = ref.compress(r, 1e-3)
    assert ref.chunk_sizes(st)[0][0] == 16384
    y = ref.decompress(st)
    assert ref.bound_violations(r, y, 1e-3) == 0


@pytest.mark.parametrize("shape,dt", [((1, 1), "f32"), ((1, 4097), "f32"), ((64, 64), "f32"),
                                      ((2, 2048), "f64"), ((3, 5, 7), "f64"), ((0, 5), "f32")])
def test_edge_shapes(ref, shape, dt):
    x = random_field(shape, dt, "noise", 1) if 0 not in shape else np.zeros(shape, np.float32)
    st, y = _roundtrip(ref, x, 0.1)
    assert y.shape == x.shape
    if x.size:
        assert ref.bound_violations(x, y, 0.1) == 0
        assert ref.order_violations(x, y) == 0
    else:
        assert len(st) == 64


def test_errors(ref):
    import oracle

    x = random_field((16, 16), "f32", "noise", 2)
    for bad in (0.0, -1.0, float("inf"), float("nan"), 1e-300):
        with pytest.raises(oracle.OracleError) as e:
            ref.compress(x, bad)
        assert e.value.code == -1
    st = ref.compress(x, 0.01)
    assert ref.decompress_rc(st, x.shape, x.dtype) == 0
    assert ref.decompress_rc(st[:-4], x.shape, x.dtype) == -4      # truncated
    assert ref.decompress_rc(b"XOPC" + st[4:], x.shape, x.dtype) == -4
    v2 = bytearray(st)
    v2[4] = 2
    assert ref.decompress_rc(bytes(v2), x.shape, x.dtype) == -5
    t = bytearray(st)
    struct.pack_into("<I", t, 64, 6)  # bin size no longer matches the payload
    assert ref.decompress_rc(bytes(t), x.shape, x.dtype) == -4
    assert ref.decompress_rc(st[:10], x.shape, x.dtype) == -4
