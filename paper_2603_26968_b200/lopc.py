"""Thin ctypes binding of liblopc.so (include/lopc.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of ``csrc/``.  PyTorch provides device memory (workspaces, outputs)
and the current CUDA stream.  There is no CPU fallback: if ``liblopc.so`` is
missing or no GPU is visible, every call raises.
"""
from __future__ import annotations

import ctypes as C
import threading
import os
import re

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("LOPC_LIB") or os.path.join(_HERE, "liblopc.so")  # LOPC_LIB: variant builds (tools)
HEADER = os.path.join(os.path.dirname(_HERE), "include", "lopc.h")

F32, F64 = 0, 1
ERRORS = {0: "OK", -1: "E_ARG", -2: "E_SHAPE", -3: "E_NOSPACE", -4: "E_CORRUPT", -5: "E_VERSION",
          -6: "E_CUDA", -7: "E_NCCL", -8: "E_INTERNAL"}


class LopcError(RuntimeError):
    def __init__(self, code: int, what: str, detail: str = ""):
        msg = f"{what}: {ERRORS.get(code, code)}"
        if detail:
            msg += f" ({detail})"
        super().__init__(msg)
        self.code = code


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("n_elems", "n_chunks", "n_tiles", "sweep_passes", "worklist_points",
                                          "inner_iters", "escapes", "bin_bytes", "sub_bytes", "total_bytes")] + [
        ("max_subbin", C.c_uint32), ("timing_valid", C.c_uint32)] + [
        (n, C.c_float) for n in ("ms_h2d", "ms_quant_repair", "ms_sweep", "ms_encode", "ms_decode", "ms_d2h",
                                 "ms_total")] + [("raised", C.c_uint64), ("pass_items", C.c_uint32 * 16), ("phase_cycles", C.c_uint64 * 16),
        ("ms_place", C.c_float), ("launches", C.c_uint32), ("pass_us", C.c_float * 16),
        ("tma", C.c_uint32)]


_lib = None


def declared_symbols() -> list[str]:
    """Function names declared in include/lopc.h."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lopc_[a-z0-9_]+)\s*\(", src)))


def load(require_gpu: bool = True):
    """Load liblopc.so (raises if it is missing; with require_gpu, also if no
    CUDA device is visible)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise ImportError(f"{SO} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(SO)
        P, I, D, SZ, U64P = C.c_void_p, C.c_int, C.c_double, C.c_size_t, C.POINTER(C.c_uint64)
        L.lopc_compress_bound.argtypes = [I, U64P, I]
        L.lopc_compress_bound.restype = SZ
        L.lopc_compress_workspace_bytes.argtypes = [I, U64P, I, I]
        L.lopc_compress_workspace_bytes.restype = SZ
        L.lopc_decompress_workspace_bytes.argtypes = [SZ, SZ, I]
        L.lopc_decompress_workspace_bytes.restype = SZ
        L.lopc_compress.argtypes = [P, I, U64P, I, D, P, C.POINTER(SZ)]
        L.lopc_compress_ex.argtypes = [P, I, U64P, I, D, P, C.POINTER(SZ), P, SZ, P]
        L.lopc_decompress.argtypes = [P, SZ, P, SZ]
        L.lopc_decompress_ex.argtypes = [P, SZ, P, SZ, P, SZ, P]
        L.lopc_repair_ex.argtypes = [P, I, U64P, I, D, P, P, P, SZ, P]
        L.lopc_stream_info.argtypes = [P, SZ, C.POINTER(I), U64P, C.POINTER(I), C.POINTER(D), U64P,
                                       C.POINTER(C.c_uint32)]
        L.lopc_last_stats.argtypes = [C.POINTER(Stats)]
        L.lopc_set_timing.argtypes = [I]
        L.lopc_set_timing.restype = None
        L.lopc_strerror.restype = C.c_char_p
        L.lopc_last_error_string.restype = C.c_char_p
        for f in ("lopc_compress", "lopc_compress_ex", "lopc_decompress", "lopc_decompress_ex", "lopc_repair_ex",
                  "lopc_stream_info", "lopc_last_stats", "lopc_abi_version"):
            getattr(L, f).restype = I
        _lib = L
    if require_gpu and not torch.cuda.is_available():
        raise RuntimeError("liblopc needs a CUDA GPU (B200); there is no CPU fallback")
    return _lib


_dims_cache: dict = {}


def _dims(shape):
    key = tuple(int(v) for v in shape)
    d = _dims_cache.get(key)
    if d is None:
        d = (C.c_uint64 * 3)(*(list(key) + [0] * (3 - len(key))))
        _dims_cache[key] = d
    return d


class _on_device:
    """torch.cuda.device(dev) only when dev is not already current (the
    context switch costs host time on every call)."""

    __slots__ = ("ctx",)

    def __init__(self, dev):
        self.ctx = torch.cuda.device(dev) if dev.index is not None and dev.index != torch.cuda.current_device() else None

    def __enter__(self):
        if self.ctx is not None:
            self.ctx.__enter__()

    def __exit__(self, *a):
        if self.ctx is not None:
            self.ctx.__exit__(*a)


_size_cache: dict = {}


def _cached_size(fn_name: str, *args) -> int:
    key = (fn_name,) + tuple(int(a) if not isinstance(a, C.Array) else tuple(a) for a in args)
    v = _size_cache.get(key)
    if v is None:
        v = int(getattr(load(False), fn_name)(*args))
        _size_cache[key] = v
    return v


def _dtype_code(dt) -> int:
    if dt == torch.float32:
        return F32
    if dt == torch.float64:
        return F64
    raise TypeError(f"LOPC compresses float32/float64 grids, got {dt}")


def _check(rc: int, what: str):
    if rc != 0:
        raise LopcError(rc, what, load(False).lopc_last_error_string().decode())


_ws = threading.local()  # one workspace per (host thread, device): calls of two threads never share one


def _workspace(nbytes: int, device) -> torch.Tensor:
    key = torch.device(device).index if torch.device(device).type == "cuda" else torch.cuda.current_device()
    d = getattr(_ws, "d", None)
    if d is None:
        d = _ws.d = {}
    t = d.get(key)
    if t is None or t.numel() < nbytes:
        t = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=f"cuda:{key}")
        d[key] = t
    return t


def _stream(device=None):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def compress_bound(shape, dtype) -> int:
    return int(load(False).lopc_compress_bound(len(shape), _dims(shape), _dtype_code(dtype)))


def compress(x: torch.Tensor, eps: float, out: torch.Tensor | None = None) -> torch.Tensor:
    """lopc_compress_ex on x (2D/3D float32/float64, device or host memory).
    Returns a uint8 tensor view of exactly the stream bytes (on ``out``'s
    device/host memory if given, else on x's device; host x -> host out)."""
    L = load()
    if x.dim() not in (2, 3):
        raise ValueError("x must be 2D or 3D")
    x = x.contiguous()
    dev = x.device if x.is_cuda else torch.device("cuda", torch.cuda.current_device())
    if out is None:
        out = torch.empty(compress_bound(x.shape, x.dtype), dtype=torch.uint8, device=x.device)
    host_io = int((not x.is_cuda) or (not out.is_cuda))
    need = _cached_size("lopc_compress_workspace_bytes", x.dim(), _dims(x.shape), _dtype_code(x.dtype), host_io)
    ws = _workspace(need, dev)
    nbytes = C.c_size_t(out.numel())
    with _on_device(dev):
        rc = L.lopc_compress_ex(C.c_void_p(x.data_ptr()), x.dim(), _dims(x.shape), _dtype_code(x.dtype),
                                float(eps), C.c_void_p(out.data_ptr()), C.byref(nbytes),
                                C.c_void_p(ws.data_ptr()), ws.numel(), _stream(dev))
    _check(rc, "lopc_compress")
    return out[: nbytes.value]


def stream_info(stream: torch.Tensor) -> dict:
    hdr = stream[:64].cpu().numpy().tobytes() if stream.numel() >= 64 else bytes(stream.cpu().numpy())
    buf = C.create_string_buffer(hdr, len(hdr))
    nd, dt, e = C.c_int(), C.c_int(), C.c_double()
    d3 = (C.c_uint64 * 3)()
    n, c = C.c_uint64(), C.c_uint32()
    rc = load(False).lopc_stream_info(buf, len(hdr), C.byref(nd), d3, C.byref(dt), C.byref(e), C.byref(n), C.byref(c))
    _check(rc, "lopc_stream_info")
    dims = tuple(int(v) for v in d3)
    shape = dims[1:] if nd.value == 2 else dims
    return {"ndims": nd.value, "shape": shape, "dtype": torch.float32 if dt.value == 0 else torch.float64,
            "eps": e.value, "n": n.value, "chunks": c.value}


def decompress(stream: torch.Tensor, out: torch.Tensor | None = None, info: dict | None = None) -> torch.Tensor:
    """lopc_decompress_ex.  ``stream`` may live on the device or the host; the
    result is allocated on the stream's device (or on ``out``)."""
    L = load()
    stream = stream.contiguous()
    if out is None:
        info = info or stream_info(stream)
        dev = stream.device if stream.is_cuda else torch.device("cuda", torch.cuda.current_device())
        out = torch.empty(info["shape"], dtype=info["dtype"], device=dev)
    dev = out.device if out.is_cuda else (stream.device if stream.is_cuda else
                                          torch.device("cuda", torch.cuda.current_device()))
    host_io = int((not stream.is_cuda) or (not out.is_cuda))
    nb = out.numel() * out.element_size()
    need = _cached_size("lopc_decompress_workspace_bytes", stream.numel(), nb, host_io)
    ws = _workspace(need, dev)
    with _on_device(dev):
        rc = L.lopc_decompress_ex(C.c_void_p(stream.data_ptr()), stream.numel(), C.c_void_p(out.data_ptr()), nb,
                                  C.c_void_p(ws.data_ptr()), ws.numel(), _stream(dev))
    _check(rc, "lopc_decompress")
    return out


def repair(x: torch.Tensor, eps: float):
    """Steps a1-a3 only: returns (flags u16 as int16, subbins u32 as int32),
    both device tensors shaped like x."""
    L = load()
    x = x.contiguous()
    flags = torch.empty(x.shape, dtype=torch.int16, device=x.device)
    s = torch.empty(x.shape, dtype=torch.int32, device=x.device)
    need = L.lopc_compress_workspace_bytes(x.dim(), _dims(x.shape), _dtype_code(x.dtype), 0)
    ws = _workspace(need, x.device)
    with torch.cuda.device(x.device):
        rc = L.lopc_repair_ex(C.c_void_p(x.data_ptr()), x.dim(), _dims(x.shape), _dtype_code(x.dtype), float(eps),
                              C.c_void_p(flags.data_ptr()), C.c_void_p(s.data_ptr()), C.c_void_p(ws.data_ptr()),
                              ws.numel(), _stream(x.device))
    _check(rc, "lopc_repair_ex")
    return flags, s


def set_timing(on=True):
    load(False).lopc_set_timing(int(on) if not isinstance(on, bool) else (1 if on else 0))


def set_repair_engine(engine: int):
    """0: tile fixpoints over alternating shifted tilings (default; falls back
    to 2 when a subbin exceeds 8 planes); 1: the paper's point worklist (f2);
    2: r1's dense tile pass + point worklist tail (u32 subbins)."""
    L = load(False)
    L.lopc_set_repair_engine.argtypes = [C.c_int]
    L.lopc_set_repair_engine.restype = C.c_int
    _check(L.lopc_set_repair_engine(int(engine)), "lopc_set_repair_engine")


def set_decoder(decoder: int):
    """1: one CTA per chunk (default); 2: 2-CTA clusters."""
    L = load(False)
    L.lopc_set_decoder.argtypes = [C.c_int]
    L.lopc_set_decoder.restype = C.c_int
    _check(L.lopc_set_decoder(int(decoder)), "lopc_set_decoder")


def set_index64(force: bool):
    """Force the int64 index builds of k_quant_flags / k_sweep (test switch)."""
    L = load(False)
    L.lopc_set_index64.argtypes = [C.c_int]
    L.lopc_set_index64.restype = C.c_int
    _check(L.lopc_set_index64(int(bool(force))), "lopc_set_index64")
    _size_cache.clear()  # workspace sizes depend on the index width


def last_stats() -> dict:
    st = Stats()
    load(False).lopc_last_stats(C.byref(st))
    d = {name: getattr(st, name) for name, _ in Stats._fields_}
    d["pass_items"] = [int(v) for v in st.pass_items]
    d["phase_cycles"] = [int(v) for v in st.phase_cycles]
    d["pass_us"] = [float(v) for v in st.pass_us]
    return d


# ---- multi-GPU slab mode (include/lopc.h) --------------------
def _slab_syms(L):
    if getattr(L, "_slab_ready", False):
        return L
    P, I, D, SZ, U64, U64P = C.c_void_p, C.c_int, C.c_double, C.c_size_t, C.c_uint64, C.POINTER(C.c_uint64)
    L.lopc_comm_unique_id.argtypes = [P]
    L.lopc_comm_create.argtypes = [C.POINTER(P), I, I, P]
    L.lopc_comm_destroy.argtypes = [P]
    L.lopc_slab_partition.argtypes = [I, U64P, I, I, U64P]
    L.lopc_slab_info.argtypes = [I, U64P, I, U64, U64, I, I, U64P]
    L.lopc_slab_workspace_bytes.argtypes = [I, U64P, I, U64, U64]
    L.lopc_slab_workspace_bytes.restype = SZ
    L.lopc_slab_bound.argtypes = [I, U64P, I, U64, U64]
    L.lopc_slab_bound.restype = SZ
    L.lopc_write_header.argtypes = [P, I, U64P, I, D, U64]
    L.lopc_compress_slab.argtypes = [P, P, I, U64P, I, D, U64, U64, P, C.POINTER(SZ), U64P, U64P, P, SZ, P]
    L.lopc_decompress_slab_workspace_bytes.argtypes = [U64]
    L.lopc_decompress_slab_workspace_bytes.restype = SZ
    L.lopc_decompress_slab.argtypes = [P, P, SZ, U64, U64, P, SZ, P, SZ, P]
    L.lopc_compress_slabs_local.argtypes = [P, I, U64P, I, D, I, U64P, P, C.POINTER(SZ)]
    for f in ("lopc_comm_unique_id", "lopc_comm_create", "lopc_comm_destroy", "lopc_slab_partition", "lopc_slab_info",
              "lopc_write_header", "lopc_compress_slab", "lopc_decompress_slab", "lopc_compress_slabs_local"):
        getattr(L, f).restype = I
    L._slab_ready = True
    return L


def slab_partition(shape, dtype, world: int) -> list[int]:
    """Chunk-aligned, chunk-balanced range bounds (world+1 entries)."""
    L = _slab_syms(load(False))
    b = (C.c_uint64 * (world + 1))()
    _check(L.lopc_slab_partition(len(shape), _dims(shape), _dtype_code(dtype), world, b), "lopc_slab_partition")
    return [int(v) for v in b]


def slab_info(shape, dtype, e_begin: int, e_end: int, has_lo: bool, has_hi: bool) -> dict:
    L = _slab_syms(load(False))
    v = (C.c_uint64 * 8)()
    _check(L.lopc_slab_info(len(shape), _dims(shape), _dtype_code(dtype), e_begin, e_end, int(has_lo), int(has_hi), v),
           "lopc_slab_info")
    keys = ("box_begin", "box_points", "halo", "ghosts_lo", "ghosts_hi", "send_lo", "send_hi", "chunks")
    return dict(zip(keys, (int(t) for t in v)))


def slab_bound(shape, dtype, e_begin: int, e_end: int) -> int:
    L = _slab_syms(load(False))
    return int(L.lopc_slab_bound(len(shape), _dims(shape), _dtype_code(dtype), e_begin, e_end))


def write_header(shape, dtype, eps: float, total_bytes: int) -> bytes:
    L = _slab_syms(load(False))
    h = C.create_string_buffer(64)
    _check(L.lopc_write_header(h, len(shape), _dims(shape), _dtype_code(dtype), float(eps), total_bytes),
           "lopc_write_header")
    return h.raw


def comm_unique_id() -> bytes:
    L = _slab_syms(load())
    b = C.create_string_buffer(128)
    _check(L.lopc_comm_unique_id(b), "lopc_comm_unique_id")
    return b.raw


class Comm:
    """NCCL communicator of the slab mode (one rank per GPU/process)."""

    def __init__(self, world: int, rank: int, uid: bytes):
        L = _slab_syms(load())
        self.world, self.rank = world, rank
        self.h = C.c_void_p()
        buf = C.create_string_buffer(uid, 128)
        _check(L.lopc_comm_create(C.byref(self.h), world, rank, buf), "lopc_comm_create")

    def close(self):
        if self.h:
            load(False).lopc_comm_destroy(self.h)
            self.h = C.c_void_p()


def compress_slab(comm, x_slab: torch.Tensor, shape, eps: float, e_begin: int, e_end: int, out=None):
    """lopc_compress_slab: x_slab = the rank's values [e_begin, e_end) of the
    global grid `shape` (device).  Returns (out_local view, payload_offset,
    total_bytes)."""
    L = _slab_syms(load())
    x_slab = x_slab.contiguous()
    dt = _dtype_code(x_slab.dtype)
    cap = L.lopc_slab_bound(len(shape), _dims(shape), dt, e_begin, e_end)
    if out is None:
        out = torch.empty(cap, dtype=torch.uint8, device=x_slab.device)
    need = L.lopc_slab_workspace_bytes(len(shape), _dims(shape), dt, e_begin, e_end)
    ws = _workspace(need, x_slab.device)
    nb = C.c_size_t(out.numel())
    po, tot = C.c_uint64(), C.c_uint64()
    with torch.cuda.device(x_slab.device):
        rc = L.lopc_compress_slab(comm.h if comm is not None else None, C.c_void_p(x_slab.data_ptr()), len(shape),
                                  _dims(shape), dt, float(eps), e_begin, e_end, C.c_void_p(out.data_ptr()),
                                  C.byref(nb), C.byref(po), C.byref(tot), C.c_void_p(ws.data_ptr()), ws.numel(),
                                  _stream(x_slab.device))
    _check(rc, "lopc_compress_slab")
    return out[: nb.value], int(po.value), int(tot.value)


def decompress_slab(header: bytes, local: torch.Tensor, e_begin: int, e_end: int, dtype, out=None) -> torch.Tensor:
    L = _slab_syms(load())
    W = 16384 // (4 if dtype == torch.float32 else 8)
    if out is None:
        out = torch.empty(e_end - e_begin, dtype=dtype, device=local.device)
    cl = (e_end - e_begin + W - 1) // W
    ws = _workspace(L.lopc_decompress_slab_workspace_bytes(cl), local.device)
    hb = C.create_string_buffer(header, 64)
    with torch.cuda.device(local.device):
        rc = L.lopc_decompress_slab(hb, C.c_void_p(local.data_ptr()), local.numel(), e_begin, e_end,
                                    C.c_void_p(out.data_ptr()), out.numel() * out.element_size(),
                                    C.c_void_p(ws.data_ptr()), ws.numel(), _stream(local.device))
    _check(rc, "lopc_decompress_slab")
    return out


def compress_slabs_local(x: torch.Tensor, eps: float, bounds) -> torch.Tensor:
    """Test hook: the slab algorithm over len(bounds)-1 ranges on one device."""
    L = _slab_syms(load())
    x = x.contiguous()
    cap = compress_bound(x.shape, x.dtype)
    out = torch.empty(cap, dtype=torch.uint8, device=x.device)
    b = (C.c_uint64 * len(bounds))(*bounds)
    nb = C.c_size_t(cap)
    with torch.cuda.device(x.device):
        rc = L.lopc_compress_slabs_local(C.c_void_p(x.data_ptr()), x.dim(), _dims(x.shape), _dtype_code(x.dtype),
                                         float(eps), len(bounds) - 1, b, C.c_void_p(out.data_ptr()), C.byref(nb))
    _check(rc, "lopc_compress_slabs_local")
    return out[: nb.value]


# ---- row a0 / f1: NOA eps on the device -------------------------------------
def _noa_syms(L):
    if getattr(L, "_noa_ready", False):
        return L
    P, I, D, SZ, U64P = C.c_void_p, C.c_int, C.c_double, C.c_size_t, C.POINTER(C.c_uint64)
    L.lopc_value_range.argtypes = [P, I, U64P, I, C.POINTER(D), C.POINTER(D), U64P, P, SZ, P]
    L.lopc_value_range.restype = I
    L.lopc_noa_eps.argtypes = [D, D, C.c_uint64, D]
    L.lopc_noa_eps.restype = D
    L.lopc_compress_noa.argtypes = [P, I, U64P, I, D, P, C.POINTER(SZ), C.POINTER(D), P, SZ, P]
    L.lopc_compress_noa.restype = I
    L._noa_ready = True
    return L


def value_range(x: torch.Tensor):
    """(min, max, finite count) of a device tensor, one fused read (k_value_range)."""
    L = _noa_syms(load())
    x = x.contiguous()
    ws = _workspace(256, x.device)
    lo, hi, n = C.c_double(), C.c_double(), C.c_uint64()
    with torch.cuda.device(x.device):
        rc = L.lopc_value_range(C.c_void_p(x.data_ptr()), x.dim(), _dims(x.shape), _dtype_code(x.dtype),
                                C.byref(lo), C.byref(hi), C.byref(n), C.c_void_p(ws.data_ptr()), ws.numel(),
                                _stream(x.device))
    _check(rc, "lopc_value_range")
    return lo.value, hi.value, int(n.value)


def noa_eps(vmin: float, vmax: float, n_finite: int, rel: float) -> float:
    return float(_noa_syms(load(False)).lopc_noa_eps(vmin, vmax, n_finite, rel))


def compress_noa(x: torch.Tensor, rel: float, out: torch.Tensor | None = None):
    """lopc_compress_noa: eps = rel * (max - min) found on the device, then
    compress.  Returns (stream view, eps)."""
    L = _noa_syms(load())
    x = x.contiguous()
    if not x.is_cuda:
        raise ValueError("compress_noa takes a device tensor")
    cap = compress_bound(x.shape, x.dtype)
    if out is None:
        out = torch.empty(cap, dtype=torch.uint8, device=x.device)
    need = max(256, L.lopc_compress_workspace_bytes(x.dim(), _dims(x.shape), _dtype_code(x.dtype), 0))
    ws = _workspace(need, x.device)
    nb = C.c_size_t(out.numel())
    e = C.c_double()
    with torch.cuda.device(x.device):
        rc = L.lopc_compress_noa(C.c_void_p(x.data_ptr()), x.dim(), _dims(x.shape), _dtype_code(x.dtype), float(rel),
                                 C.c_void_p(out.data_ptr()), C.byref(nb), C.byref(e), C.c_void_p(ws.data_ptr()),
                                 ws.numel(), _stream(x.device))
    _check(rc, "lopc_compress_noa")
    return out[: nb.value], e.value


# ---- k_check: order / bound / error statistics -------------------------------
class CheckResult(C.Structure):
    _fields_ = [("order_violations", C.c_uint64), ("bound_violations", C.c_uint64), ("n_regular", C.c_uint64),
                ("max_abs_err", C.c_double), ("sum_sq_err", C.c_double)]


def check(x: torch.Tensor, y: torch.Tensor, eps: float) -> dict:
    """lopc_check on two device arrays of the same grid; adds mse and PSNR
    (20 log10(range) - 10 log10(mse), range over the finite values of x)."""
    import math

    L = _noa_syms(load())
    if not getattr(L, "_check_ready", False):
        L.lopc_check.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_uint64), C.c_int, C.c_double,
                                 C.POINTER(CheckResult), C.c_void_p, C.c_size_t, C.c_void_p]
        L.lopc_check.restype = C.c_int
        L._check_ready = True
    x, y = x.contiguous(), y.contiguous()
    if x.shape != y.shape or x.dtype != y.dtype:
        raise ValueError("x and y must have the same shape and dtype")
    ws = _workspace(256, x.device)
    r = CheckResult()
    with torch.cuda.device(x.device):
        rc = L.lopc_check(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), x.dim(), _dims(x.shape),
                          _dtype_code(x.dtype), float(eps), C.byref(r), C.c_void_p(ws.data_ptr()), ws.numel(),
                          _stream(x.device))
    _check(rc, "lopc_check")
    d = {n: getattr(r, n) for n, _ in CheckResult._fields_}
    lo, hi, _ = value_range(x)
    d["mse"] = d["sum_sq_err"] / d["n_regular"] if d["n_regular"] else 0.0
    d["psnr_db"] = (20 * math.log10(hi - lo) - 10 * math.log10(d["mse"])) if d["mse"] > 0 and hi > lo else None
    return d


class CriticalResult(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("false_positives", "false_negatives", "false_types", "pair_mismatches",
                                          "critical_x", "critical_y")]


def critical_points(x: torch.Tensor, y: torch.Tensor) -> dict:
    """lopc_critical_points: Table III FP/FN/FT of y against x (device arrays)."""
    L = load()
    if not getattr(L, "_crit_ready", False):
        L.lopc_critical_points.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_uint64), C.c_int,
                                           C.POINTER(CriticalResult), C.c_void_p, C.c_size_t, C.c_void_p]
        L.lopc_critical_points.restype = C.c_int
        L._crit_ready = True
    x, y = x.contiguous(), y.contiguous()
    ws = _workspace(256, x.device)
    r = CriticalResult()
    with torch.cuda.device(x.device):
        rc = L.lopc_critical_points(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), x.dim(), _dims(x.shape),
                                    _dtype_code(x.dtype), C.byref(r), C.c_void_p(ws.data_ptr()), ws.numel(),
                                    _stream(x.device))
    _check(rc, "lopc_critical_points")
    return {n: int(getattr(r, n)) for n, _ in CriticalResult._fields_}
