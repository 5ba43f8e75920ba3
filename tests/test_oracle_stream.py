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


def test_rze_two_level_hand_vector(ref):
    """RZE_1 of 1024 bytes, zero except d[100] = 0x09, d[900] = 0x41,
    d[901] = 0x42, derived by hand from the format text (reading G21):
      B0 (128 B): B0[12] = 0x10 (word 100), B0[112] = 0x30 (words 900, 901)
      B1 (16 B):  B0 changes at t = 12, 13, 112, 113 -> B1[1] = 0x30, B1[14] = 0x03
      K0 = B0[12], B0[13], B0[112], B0[113] = 10 00 30 00
      B2 (2 B):   B1 changes at t = 1, 2, 14, 15 -> B2 = 06 c0 (|B2| <= 8: top)
      K1 = B1[1], B1[2], B1[14], B1[15] = 30 00 03 00
      output = B2 | K1 | K0 | words = 06 c0 | 30 00 03 00 | 10 00 30 00 | 09 41 42
    B0[13] = 0 is kept only because it differs from B0[12]: a "!= 0" repeat
    test would drop it."""
    from tests.exact import rze_spec

    d = bytearray(1024)
    d[100], d[900], d[901] = 0x09, 0x41, 0x42
    want = bytes.fromhex("06c0" "30000300" "10003000" "094142")
    assert rze_spec(bytes(d), 1) == want
    assert ref.rze(bytes(d), 1) == want
    out, used = ref.unrze(want, 1024, 1)
    assert out == bytes(d) and used == len(want)


@pytest.mark.parametrize("g", [1, 4, 8])
def test_rze_matches_spec(ref, g):
    """The oracle's RZE_g equals the independent restatement (tests/exact.py
    rze_spec) on 16384-byte inputs whose bitmap levels have non-empty K_1 /
    K_2 (clustered runs of non-zero words at several densities), plus short
    inputs; >= 100 cases per g."""
    from tests.exact import rze_spec

    rng = np.random.default_rng(100 + g)
    deep = 0
    for trial in range(110):
        L = 16384 if trial % 4 else int(rng.integers(1, 600)) * g
        n = L // g
        kind = trial % 5
        w = np.zeros((n, g), np.uint8)
        if kind == 0:      # sparse isolated words
            idx = rng.choice(n, size=max(1, n // 200), replace=False)
            w[idx] = rng.integers(1, 256, (idx.size, g))
        elif kind == 1:    # runs of non-zero words (B0 bytes 0xff inside runs)
            for _ in range(int(rng.integers(1, 20))):
                a = int(rng.integers(0, n))
                w[a:a + int(rng.integers(1, 300))] = rng.integers(1, 256, g)
        elif kind == 2:    # dense random words with zero holes
            w[:] = rng.integers(0, 256, (n, g))
            w[rng.random(n) < 0.3] = 0
        elif kind == 3:    # periodic patterns (B0 repeats a non-zero byte)
            per = int(rng.integers(2, 17))
            w[::per] = rng.integers(1, 256, g)
        else:              # mostly zero with a few partially-zero words
            idx = rng.choice(n, size=max(1, n // 50), replace=False)
            w[idx, int(rng.integers(0, g))] = rng.integers(1, 256, idx.size)
        data = w.tobytes()
        enc = ref.rze(data, g)
        assert enc == rze_spec(data, g), (g, trial, kind)
        nb0 = -(-n // 8)
        if nb0 > 64:
            deep += 1
    assert deep >= 60  # most cases recurse at least twice (|B0| > 64 bytes)


def test_bound_violations_teeth(ref):
    """The exact bound checker (O13; proof (i): 0 <= x - x^ <= eps)
    fires one ulp past the bound, on the wrong side, and on a changed escape;
    the TwoSum term decides a difference that rounds to exactly eps."""
    up, dn = (lambda v: np.nextafter(v, np.inf)), (lambda v: np.nextafter(v, -np.inf))
    x = np.array([1.0])
    assert ref.bound_violations(x, np.array([0.75]), 0.25) == 0          # exactly eps below
    assert ref.bound_violations(x, np.array([dn(0.75)]), 0.25) == 1      # one ulp past eps
    assert ref.bound_violations(x, np.array([1.0]), 0.25) == 0
    assert ref.bound_violations(x, np.array([up(1.0)]), 0.25) == 1       # above x: one-sided error
    # 8 - (-2^-60) = 8 + 2^-60 rounds to 8 = eps but exceeds it; 8 - 2^-60 does not
    assert ref.bound_violations(np.array([8.0]), np.array([-2.0 ** -60]), 8.0) == 1
    assert ref.bound_violations(np.array([8.0]), np.array([2.0 ** -60]), 8.0) == 0
    # f32: one f32 ulp past eps
    xf = np.array([1.0], np.float32)
    assert ref.bound_violations(xf, np.array([0.75], np.float32), 0.25) == 0
    assert ref.bound_violations(xf, np.array([np.nextafter(np.float32(0.75), np.float32(0))]), 0.25) == 1
    # escapes must come back bitwise
    xe = np.array([np.inf, np.nan, 1e300])
    assert ref.bound_violations(xe, xe.copy(), 1e-3) == 0
    assert ref.bound_violations(xe, np.array([np.inf, np.nan, up(1e300)]), 1e-3) == 1
    assert ref.bound_violations(xe, np.array([-np.inf, np.nan, 1e300]), 1e-3) == 1
    # counts add up over points
    xs = np.array([1.0, 2.0, 3.0])
    assert ref.bound_violations(xs, np.array([dn(0.75), 2.0, up(3.0)]), 0.25) == 2
