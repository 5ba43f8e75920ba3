"""CPU oracle for the LOPC hot path — TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper around ``oracle/liblopc_ref.so`` (plain C, built from
``oracle/lopc_ref.c``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  The product path (``paper_2603_26968_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(_HERE, "liblopc_ref.so")
SRC = os.path.join(_HERE, "lopc_ref.c")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < max(
        os.path.getmtime(SRC), os.path.getmtime(os.path.join(_HERE, "lopc_ref.h"))
    ):
        subprocess.check_call(["gcc", *CFLAGS, "-o", SO, SRC, "-lm"])
    return SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(SO)
        P, U64P, I64, D, I, SZ = C.c_void_p, C.POINTER(C.c_uint64), C.c_int64, C.c_double, C.c_int, C.c_size_t
        L.lopc_ref_bin.argtypes = [D, D, I, C.POINTER(C.c_int64)]
        L.lopc_ref_bin.restype = I
        L.lopc_ref_lo.argtypes = [I64, D, I]
        L.lopc_ref_lo.restype = D
        L.lopc_ref_ord.argtypes = [C.c_uint64, I]
        L.lopc_ref_ord.restype = I64
        for name in ("lopc_ref_quantize", "lopc_ref_flags", "lopc_ref_subbins"):
            getattr(L, name).argtypes = [P, I, U64P, I, D, P]
            getattr(L, name).restype = I
        for name in ("lopc_ref_subbins_alg12", "lopc_ref_subbins_jacobi"):
            getattr(L, name).argtypes = [P, I, U64P, I, D, P, U64P]
            getattr(L, name).restype = I
        L.lopc_ref_reconstruct.argtypes = [P, I, U64P, I, D, P, P]
        L.lopc_ref_reconstruct.restype = I
        L.lopc_ref_compress_bound.argtypes = [I, U64P, I]
        L.lopc_ref_compress_bound.restype = SZ
        L.lopc_ref_compress.argtypes = [P, I, U64P, I, D, P, C.POINTER(C.c_size_t)]
        L.lopc_ref_compress.restype = I
        L.lopc_ref_decompress.argtypes = [P, SZ, P, SZ]
        L.lopc_ref_decompress.restype = I
        L.lopc_ref_stream_info.argtypes = [P, SZ, C.POINTER(I), U64P, C.POINTER(I), C.POINTER(D), U64P,
                                           C.POINTER(C.c_uint32)]
        L.lopc_ref_stream_info.restype = I
        L.lopc_ref_chunk_sizes.argtypes = [P, SZ, P, C.c_uint32]
        L.lopc_ref_chunk_sizes.restype = I
        for name in ("lopc_ref_diffnb", "lopc_ref_undiffnb", "lopc_ref_bitshuffle", "lopc_ref_unbitshuffle"):
            getattr(L, name).argtypes = [P, SZ, I, P]
            getattr(L, name).restype = None
        L.lopc_ref_rze.argtypes = [P, SZ, I, P]
        L.lopc_ref_rze.restype = SZ
        L.lopc_ref_unrze.argtypes = [P, SZ, SZ, I, P]
        L.lopc_ref_unrze.restype = C.c_long
        L.lopc_ref_order_violations.argtypes = [P, P, I, U64P, I]
        L.lopc_ref_order_violations.restype = C.c_uint64
        L.lopc_ref_bound_violations.argtypes = [P, P, C.c_uint64, I, D]
        L.lopc_ref_bound_violations.restype = C.c_uint64
        L.lopc_ref_encode_chunk.argtypes = [P, C.c_uint64, I, D, P, C.c_uint64, P, P]
        L.lopc_ref_encode_chunk.restype = I
        L.lopc_ref_certify.argtypes = [P, I, U64P, I, D, P]
        L.lopc_ref_certify.restype = C.c_uint64
        L.lopc_ref_value_range.argtypes = [P, C.c_uint64, I, C.POINTER(D), C.POINTER(D)]
        L.lopc_ref_value_range.restype = C.c_uint64
        L.lopc_ref_noa_eps.argtypes = [P, C.c_uint64, I, D]
        L.lopc_ref_noa_eps.restype = D
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what} failed with code {code}")
        self.code = code


def _dt(x: np.ndarray) -> int:
    if x.dtype == np.float32:
        return 0
    if x.dtype == np.float64:
        return 1
    raise TypeError(x.dtype)


def _dims(x: np.ndarray):
    d = (C.c_uint64 * 3)(*([int(v) for v in x.shape] + [0] * (3 - x.ndim)))
    return d


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _chk(rc, what):
    if rc != 0:
        raise OracleError(rc, what)


def bin_of(x: float, eps: float, dtype: int = 1):
    b = C.c_int64()
    ok = lib().lopc_ref_bin(float(x), float(eps), dtype, C.byref(b))
    return int(b.value) if ok else None


def lo(b: int, eps: float, dtype: int = 1) -> float:
    return lib().lopc_ref_lo(int(b), float(eps), dtype)


def quantize(x: np.ndarray, eps: float) -> np.ndarray:
    x = np.ascontiguousarray(x)
    out = np.empty(x.size, np.int64)
    _chk(lib().lopc_ref_quantize(_ptr(x), x.ndim, _dims(x), _dt(x), eps, _ptr(out)), "quantize")
    return out.reshape(x.shape)


def flags(x: np.ndarray, eps: float) -> np.ndarray:
    x = np.ascontiguousarray(x)
    out = np.empty(x.size, np.uint16)
    _chk(lib().lopc_ref_flags(_ptr(x), x.ndim, _dims(x), _dt(x), eps, _ptr(out)), "flags")
    return out.reshape(x.shape)


def subbins(x: np.ndarray, eps: float, method: str = "dp"):
    x = np.ascontiguousarray(x)
    out = np.empty(x.size, np.uint32)
    st = (C.c_uint64 * 4)()
    if method == "dp":
        _chk(lib().lopc_ref_subbins(_ptr(x), x.ndim, _dims(x), _dt(x), eps, _ptr(out)), "subbins")
        return out.reshape(x.shape)
    fn = {"alg12": lib().lopc_ref_subbins_alg12, "jacobi": lib().lopc_ref_subbins_jacobi}[method]
    _chk(fn(_ptr(x), x.ndim, _dims(x), _dt(x), eps, _ptr(out), st), method)
    return out.reshape(x.shape), tuple(int(v) for v in st)


def reconstruct(x: np.ndarray, eps: float, s: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x)
    s = np.ascontiguousarray(s, dtype=np.uint32)
    out = np.empty_like(x)
    _chk(lib().lopc_ref_reconstruct(_ptr(x), x.ndim, _dims(x), _dt(x), eps, _ptr(s), _ptr(out)), "reconstruct")
    return out


def compress_bound(shape, dtype) -> int:
    d = (C.c_uint64 * 3)(*([int(v) for v in shape] + [0] * (3 - len(shape))))
    return int(lib().lopc_ref_compress_bound(len(shape), d, 0 if np.dtype(dtype) == np.float32 else 1))


def compress(x: np.ndarray, eps: float) -> bytes:
    x = np.ascontiguousarray(x)
    cap = compress_bound(x.shape, x.dtype)
    out = np.empty(max(cap, 1), np.uint8)
    n = C.c_size_t(cap)
    _chk(lib().lopc_ref_compress(_ptr(x), x.ndim, _dims(x), _dt(x), eps, _ptr(out), C.byref(n)), "compress")
    return out[: n.value].tobytes()


def stream_info(stream: bytes):
    buf = np.frombuffer(stream, np.uint8)
    nd, dt, e = C.c_int(), C.c_int(), C.c_double()
    d3 = (C.c_uint64 * 3)()
    n, c = C.c_uint64(), C.c_uint32()
    rc = lib().lopc_ref_stream_info(_ptr(buf), len(stream), C.byref(nd), d3, C.byref(dt), C.byref(e), C.byref(n),
                                    C.byref(c))
    _chk(rc, "stream_info")
    dims = tuple(int(v) for v in d3)
    shape = dims[1:] if nd.value == 2 else dims
    return {"ndims": nd.value, "shape": shape, "dtype": dt.value, "eps": e.value, "n": n.value, "chunks": c.value}


def chunk_sizes(stream: bytes) -> np.ndarray:
    info = stream_info(stream)
    buf = np.frombuffer(stream, np.uint8)
    out = np.empty(2 * max(info["chunks"], 1), np.uint32)
    _chk(lib().lopc_ref_chunk_sizes(_ptr(buf), len(stream), _ptr(out), info["chunks"]), "chunk_sizes")
    return out[: 2 * info["chunks"]].reshape(-1, 2)


def decompress(stream: bytes) -> np.ndarray:
    info = stream_info(stream)
    dt = np.float32 if info["dtype"] == 0 else np.float64
    out = np.empty(info["shape"], dt)
    buf = np.frombuffer(stream, np.uint8)
    _chk(lib().lopc_ref_decompress(_ptr(buf), len(stream), _ptr(out), out.nbytes), "decompress")
    return out


def decompress_rc(stream: bytes, shape, dtype) -> int:
    """Return the oracle's error code for a (possibly corrupt) stream."""
    out = np.empty(shape, dtype)
    buf = np.frombuffer(stream, np.uint8) if len(stream) else np.zeros(1, np.uint8)
    return int(lib().lopc_ref_decompress(_ptr(buf), len(stream), _ptr(out), out.nbytes))


# --- stages -----------------------------------------------------------------
def diffnb(words: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(words)
    out = np.empty_like(w)
    lib().lopc_ref_diffnb(_ptr(w), w.size, w.itemsize, _ptr(out))
    return out


def undiffnb(u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u)
    out = np.empty_like(u)
    lib().lopc_ref_undiffnb(_ptr(u), u.size, u.itemsize, _ptr(out))
    return out


def bitshuffle(words: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(words)
    out = np.empty(w.nbytes, np.uint8)
    lib().lopc_ref_bitshuffle(_ptr(w), w.size, w.itemsize, _ptr(out))
    return out


def unbitshuffle(b: np.ndarray, dtype) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.uint8)
    k = np.dtype(dtype).itemsize
    out = np.empty(b.size // k, dtype)
    lib().lopc_ref_unbitshuffle(_ptr(b), out.size, k, _ptr(out))
    return out


def rze(data: bytes, g: int) -> bytes:
    a = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
    out = np.empty(len(data) + len(data) // g + 64, np.uint8)
    n = lib().lopc_ref_rze(_ptr(a), len(data), g, _ptr(out))
    return out[:n].tobytes()


def unrze(enc: bytes, L: int, g: int):
    a = np.frombuffer(enc, np.uint8).copy() if len(enc) else np.zeros(1, np.uint8)
    out = np.empty(max(L, 1), np.uint8)
    used = lib().lopc_ref_unrze(_ptr(a), len(enc), L, g, _ptr(out))
    if used < 0:
        return None, -1
    return out[:L].tobytes(), int(used)


# --- checkers ---------------------------------------------------------------
def order_violations(x: np.ndarray, y: np.ndarray) -> int:
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y, dtype=x.dtype)
    return int(lib().lopc_ref_order_violations(_ptr(x), _ptr(y), x.ndim, _dims(x), _dt(x)))


def bound_violations(x: np.ndarray, y: np.ndarray, eps: float) -> int:
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y, dtype=x.dtype)
    return int(lib().lopc_ref_bound_violations(_ptr(x), _ptr(y), x.size, _dt(x), eps))


def encode_chunk(x: np.ndarray, eps: float, s: np.ndarray, c: int):
    x = np.ascontiguousarray(x)
    s = np.ascontiguousarray(s, dtype=np.uint32)
    out = np.empty(2 * 16384, np.uint8)
    sz = (C.c_uint32 * 2)()
    _chk(lib().lopc_ref_encode_chunk(_ptr(x), x.size, _dt(x), eps, _ptr(s), c, _ptr(out), sz), "encode_chunk")
    return out[: sz[0]].tobytes(), out[sz[0]: sz[0] + sz[1]].tobytes()


def certify(x: np.ndarray, eps: float, s: np.ndarray) -> int:
    x = np.ascontiguousarray(x)
    s = np.ascontiguousarray(s, dtype=np.uint32)
    return int(lib().lopc_ref_certify(_ptr(x), x.ndim, _dims(x), _dt(x), eps, _ptr(s)))


def value_range(x: np.ndarray):
    """Row a0: (min, max, count) over the finite values, as doubles."""
    x = np.ascontiguousarray(x)
    lo, hi = C.c_double(), C.c_double()
    n = lib().lopc_ref_value_range(_ptr(x), x.size, _dt(x), C.byref(lo), C.byref(hi))
    return lo.value, hi.value, int(n)


def noa_eps(x: np.ndarray, rel: float) -> float:
    """Row a0: eps = rel * (max - min) over the finite values."""
    x = np.ascontiguousarray(x)
    return float(lib().lopc_ref_noa_eps(_ptr(x), x.size, _dt(x), float(rel)))


# ---- NEXT f4: multi-core CPU baseline (oracle/lopc_omp.c, OpenMP) ----------
OMP_SO = os.path.join(_HERE, "liblopc_omp.so")
_omp = None


def build_omp(force: bool = False) -> str:
    src = os.path.join(_HERE, "lopc_omp.c")
    deps = [src, SRC, os.path.join(_HERE, "lopc_ref.h")]
    if force or not os.path.exists(OMP_SO) or os.path.getmtime(OMP_SO) < max(os.path.getmtime(p) for p in deps):
        subprocess.check_call(["gcc", *CFLAGS, "-fopenmp", "-o", OMP_SO, src, SRC, "-lm"])
    return OMP_SO


def omp_compress(x: np.ndarray, eps: float, threads: int = 0):
    """(stream bytes, relaxation sweeps): the OpenMP baseline, all cores by default."""
    global _omp
    if _omp is None:
        build_omp()
        _omp = C.CDLL(OMP_SO)
        _omp.lopc_omp_compress.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_uint64), C.c_int, C.c_double,
                                           C.c_void_p, C.POINTER(C.c_size_t), C.c_int, C.POINTER(C.c_uint64)]
        _omp.lopc_omp_compress.restype = C.c_int
    x = np.ascontiguousarray(x)
    cap = compress_bound(x.shape, x.dtype)
    out = C.create_string_buffer(cap)
    nb = C.c_size_t(cap)
    sw = C.c_uint64()
    rc = _omp.lopc_omp_compress(_ptr(x), x.ndim, _dims(x), _dt(x), float(eps), out, C.byref(nb), int(threads),
                                C.byref(sw))
    if rc:
        raise OracleError(rc, "omp_compress")
    return out.raw[: nb.value], int(sw.value)


def omp_check_chunks(x: np.ndarray, eps: float, s: np.ndarray, stream) -> tuple:
    """(mismatching chunks, first bad chunk or None): every chunk of `stream`
    against the oracle's chunk encoder on (x, eps, s), all host cores
    (lopc_omp_check_chunks).  s must be certified first (certify(x, eps, s)
    == 0), which makes the expected bytes the oracle's stream."""
    global _omp
    if _omp is None:
        omp_compress(np.zeros((1, 1), np.float32), 1.0)  # loads the library
    f = _omp.lopc_omp_check_chunks
    f.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_uint64,
                  C.POINTER(C.c_uint64)]
    f.restype = C.c_uint64
    x = np.ascontiguousarray(x)
    s = np.ascontiguousarray(s, dtype=np.uint32)
    st = np.frombuffer(stream, np.uint8) if isinstance(stream, (bytes, bytearray)) else np.ascontiguousarray(stream)
    first = C.c_uint64()
    bad = int(f(_ptr(x), x.size, _dt(x), float(eps), _ptr(s), _ptr(st), st.size, C.byref(first)))
    return bad, (None if first.value == 2**64 - 1 else int(first.value))


def omp_decompress(stream: bytes, threads: int = 0) -> np.ndarray:
    """The OpenMP decompress (every chunk in parallel by lopc_ref_decode_chunk)."""
    global _omp
    if _omp is None:
        omp_compress(np.zeros((1, 1), np.float32), 1.0)
    f = _omp.lopc_omp_decompress
    f.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int]
    f.restype = C.c_int
    info = stream_info(stream)
    out = np.empty(info["shape"], np.float32 if info["dtype"] == 0 else np.float64)
    buf = np.frombuffer(stream, np.uint8)
    rc = f(_ptr(buf), len(stream), _ptr(out), out.nbytes, int(threads))
    if rc:
        raise OracleError(rc, "omp_decompress")
    return out
