// lopc_api.cu — host orchestration behind include/lopc.h (liblopc.so).
//
// compress:   [H2D stage] -> k_quant_flags -> k_sweep (cooperative, device-
//             side termination) -> k_encode (look-back placement, header) ->
//             one D2H read of the status block -> [D2H stage]
// decompress: [H2D stage] -> k_decode (persistent, header validated on the
//             device) -> one D2H read of the status block -> [D2H stage]
//
// Scratch comes only from the caller's workspace; nothing is allocated inside
// the *_ex calls.  See DESIGN.md §7 for the HBM layout.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/lopc.h"
#include "lopc_codec.cuh"
#include "lopc_repair.cuh"
#include "lopc_tiles.cuh"
#include "lopc_noa.cuh"
#include "lopc_check.cuh"

using namespace lopc;

namespace {

// Concurrency (calls on different streams or workspaces are
// independent): everything a call writes on the host side is per thread —
// the error text, the stats, the pinned status slot, the side streams and
// events, the timing events, the plain calls' workspace pool — and keyed by
// device.  Only configuration (lopc_set_timing / lopc_set_repair_engine) and
// the once-initialised TMA entry point are process-wide.
thread_local char g_errmsg[512] = "";
thread_local lopc_stats g_stats{};
int g_timing = 0;
int g_engine = 0;  // lopc_set_repair_engine
constexpr int kMaxDev = 64;

int set_cuda_error(cudaError_t e, const char* where) {
  snprintf(g_errmsg, sizeof(g_errmsg), "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
  return LOPC_E_CUDA;
}

#define CK(call)                                      \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return set_cuda_error(e_, #call); \
  } while (0)

struct Shape {
  int ndims, dtype, k;
  uint64_t d0, d1, d2, n, C;
};

int make_shape(int ndims, const uint64_t* dims, int dtype, Shape& s) {
  if (dtype != LOPC_F32 && dtype != LOPC_F64) return LOPC_E_ARG;
  if (!dims) return LOPC_E_ARG;
  if (ndims != 2 && ndims != 3) return LOPC_E_SHAPE;
  const uint64_t lim = 1ull << 40;
  s.ndims = ndims;
  s.dtype = dtype;
  s.k = dtype == LOPC_F32 ? 4 : 8;
  if (ndims == 2) {
    s.d0 = 1;
    s.d1 = dims[0];
    s.d2 = dims[1];
  } else {
    s.d0 = dims[0];
    s.d1 = dims[1];
    s.d2 = dims[2];
  }
  if (s.d0 > lim || s.d1 > lim || s.d2 > lim) return LOPC_E_SHAPE;
  if (s.d0 && s.d1 && (s.d0 * s.d1 > lim || s.d0 * s.d1 * s.d2 > lim)) return LOPC_E_SHAPE;
  s.n = s.d0 * s.d1 * s.d2;
  const uint64_t W = kChunkBytes / s.k;
  s.C = (s.n + W - 1) / W;
  return LOPC_OK;
}

int check_eps(double eps) {
  if (!(eps >= std::ldexp(1.0, -900) && eps <= std::ldexp(1.0, 1000))) return LOPC_E_ARG;
  return LOPC_OK;
}

inline size_t al(size_t v) { return (v + 255) & ~size_t(255); }

// RN32(1/eps) for the f32 quantizer fast path; NaN disables it outside
// 2^-120 < eps < 2^120.
float inv32_of(double eps) {
  if (!(eps > std::ldexp(1.0, -120) && eps < std::ldexp(1.0, 120))) return std::nanf("");
  return (float)(1.0 / eps);
}

int g_force_i64 = 0;  // lopc_set_index64: test switch for the int64 index builds on small grids
bool use_i32(const Shape& sh) { return !g_force_i64 && sh.n < (1ull << 31) - (1ull << 24); }

struct CLayout {
  size_t ctr, bitmap, state, act0, act1, cesc, zero_end, plist, flags, s, sp, list0, list1, stage, sizes, off, stage_in,
      stage_out, total;
  uint64_t bmw, nseg;
  int ntz, nty, ntx;
  uint64_t ntiles;
  uint32_t tnt[2][3];  // k_tiles: tiles per axis of tiling 0 / 1
  uint64_t tn[2];
};

CLayout compress_layout(const Shape& s, bool host_in, bool host_out) {
  CLayout L{};
  if (s.ndims == 3) {
    L.ntz = (int)((s.d0 + Geo<3>::TZ - 1) / Geo<3>::TZ);
    L.nty = (int)((s.d1 + Geo<3>::TY - 1) / Geo<3>::TY);
    L.ntx = (int)((s.d2 + Geo<3>::TX - 1) / Geo<3>::TX);
  } else {
    L.ntz = 1;
    L.nty = (int)((s.d1 + Geo<2>::TY - 1) / Geo<2>::TY);
    L.ntx = (int)((s.d2 + Geo<2>::TX - 1) / Geo<2>::TX);
  }
  L.ntiles = s.n ? (uint64_t)L.ntz * L.nty * L.ntx : 0;
  {
    using T3 = TG<3>;
    using T2 = TG<2>;
    const uint64_t TZ = s.ndims == 3 ? T3::TZ : 1, TY = s.ndims == 3 ? T3::TY : T2::TY;
    const uint64_t SZ = s.ndims == 3 ? T3::SZ : 0, SY = s.ndims == 3 ? T3::SY : T2::SY;
    L.tnt[0][0] = (uint32_t)((s.d0 + TZ - 1) / TZ);
    L.tnt[0][1] = (uint32_t)((s.d1 + TY - 1) / TY);
    L.tnt[1][0] = (uint32_t)((s.d0 + SZ + TZ - 1) / TZ);
    L.tnt[1][1] = (uint32_t)((s.d1 + SY + TY - 1) / TY);
    L.tnt[0][2] = L.tnt[1][2] = (uint32_t)((s.d2 + 31) / 32);
    for (int t = 0; t < 2; ++t) L.tn[t] = s.n ? (uint64_t)L.tnt[t][0] * L.tnt[t][1] * L.tnt[t][2] : 0;
  }
  size_t o = 0;
  L.ctr = o;
  o += al(sizeof(Counters));
  L.bmw = (s.n + 31) / 32;
  L.bitmap = o;
  o += al(2 * 4 * L.bmw);
  L.state = o;
  o += al(8 * (s.C / kScanTile + 1));
  L.act0 = o;
  o += al(4 * L.tn[0]);
  L.act1 = o;
  o += al(4 * L.tn[1]);
  L.cesc = o;  // one bit per chunk: it holds an escape (k_quant_flags -> the subbin encoder)
  o += al(4 * ((s.C + 31) / 32));
  L.zero_end = o;
  L.plist = o;
  o += al(2 * (use_i32(s) ? 4 : 8) * s.n);  // worklist entries: the index width the kernels will use
  L.nseg = (s.d2 + 31) / 32;
  L.flags = o;
  o += al(4ull * s.d0 * s.d1 * L.nseg * (s.ndims == 3 ? Geo<3>::SW : Geo<2>::SW));
  L.s = o;
  o += al(4 * s.n);
  L.sp = o;  // subbin planes (k_tiles): 8 words per 32-point segment
  o += al(4ull * kSP * s.d0 * s.d1 * L.nseg);
  L.list0 = o;
  o += al(4 * L.tn[0]);
  L.list1 = o;
  o += al(4 * L.tn[1]);
  L.stage = o;
  o += al(2ull * kChunkBytes * s.C);
  L.sizes = o;
  o += al(8 * s.C);
  L.off = o;
  o += al(8 * s.C);
  L.stage_in = o;
  if (host_in) o += al(s.k * s.n);
  L.stage_out = o;
  if (host_out) o += al(kHdrBytes + 8 * s.C + 2ull * kChunkBytes * s.C);
  L.total = o;
  return L;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

#ifndef LOPC_PIPE_RANGES
#define LOPC_PIPE_RANGES 8
#endif
constexpr int kPipeRanges = LOPC_PIPE_RANGES;  // host-I/O decompress pipeline depth (4 in r1)

struct DevInfo {
  int dev = -1, sms = 0;
  cudaStream_t side = nullptr;           // bin-stream encode runs here, beside the repair
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t side2 = nullptr;            // host-I/O decompress: D2H of decoded ranges
  cudaEvent_t ev_in[kPipeRanges] = {}, ev_dec[kPipeRanges] = {}, ev_out = nullptr;
  int occ_sweep2 = 0, occ_sweep3 = 0, occ_sweep2w = 0, occ_sweep3w = 0, occ_decode = 0, occ_tiles2 = 0, occ_tiles3 = 0;
  int occ_decode1 = 0;
  bool attrs = false;
};
// One per (host thread, device): created on the thread's first call on that
// device, never re-created (no leak on device switches).
thread_local DevInfo tl_dev[kMaxDev];

int dev_info(DevInfo*& out) {
  int dev;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) return LOPC_E_ARG;
  DevInfo& g_dev = tl_dev[dev];
  if (!g_dev.attrs) {
    g_dev = DevInfo{};
    g_dev.dev = dev;
    CK(cudaStreamCreateWithFlags(&g_dev.side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&g_dev.ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g_dev.ev_join, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&g_dev.side2, cudaStreamNonBlocking));
    for (int i = 0; i < kPipeRanges; ++i) {
      CK(cudaEventCreateWithFlags(&g_dev.ev_in[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&g_dev.ev_dec[i], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&g_dev.ev_out, cudaEventDisableTiming));
    CK(cudaDeviceGetAttribute(&g_dev.sms, cudaDevAttrMultiProcessorCount, dev));
    const int smem = (int)sizeof(EncSmem), dsmem = (int)sizeof(DecSmem);
    CK(cudaFuncSetAttribute(k_encode<float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_encode<float, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_encode<double, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_encode<double, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem));
    CK(cudaFuncSetAttribute(k_decode1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DecSmem2)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_dev.occ_decode1, k_decode1, kCodecThreads, sizeof(DecSmem2)));
#define QRA(TT, ND)                                                                                      \
  CK(cudaFuncSetAttribute(k_quant_flags<TT, ND, int32_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                          (int)quant_flags_smem<TT, ND, false>()));                                        \
  CK(cudaFuncSetAttribute(k_quant_flags<TT, ND, int64_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                          (int)quant_flags_smem<TT, ND, false>()));                                        \
  CK(cudaFuncSetAttribute(k_quant_flags<TT, ND, int32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                          (int)quant_flags_smem<TT, ND, true>()));                                         \
  CK(cudaFuncSetAttribute(k_quant_flags<TT, ND, int64_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                          (int)quant_flags_smem<TT, ND, true>()));
    QRA(float, 3) QRA(float, 2) QRA(double, 3) QRA(double, 2)
#undef QRA
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_dev.occ_sweep2, k_sweep<2, int32_t>, kSweepThreads, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_dev.occ_sweep3, k_sweep<3, int32_t>, kSweepThreads, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_dev.occ_sweep2w, k_sweep<2, int64_t>, kSweepThreads, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_dev.occ_sweep3w, k_sweep<3, int64_t>, kSweepThreads, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_dev.occ_tiles2, k_tiles<2>, kTileThreads, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_dev.occ_tiles3, k_tiles<3>, kTileThreads, 0));
    {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(2 * 148 * 8, 1, 1);
      cfg.blockDim = dim3(kCodecThreads, 1, 1);
      cfg.dynamicSmemBytes = dsmem;
      CK(cudaOccupancyMaxActiveClusters(&g_dev.occ_decode, k_decode, &cfg));  // whole GPU, clusters
    }
    g_dev.attrs = true;
  }
  out = &g_dev;
  return LOPC_OK;
}

// a8: k_decode1 (one CTA per chunk, both streams; the default) or k_decode
// (2-CTA clusters; LOPC_DECODER=2), persistent over `chunks` chunks.
int g_decoder = -1;  // lopc_set_decoder; -1: LOPC_DECODER from the environment, else 1
int launch_decode(const DevInfo* di, const DecodeArgs& da, uint64_t chunks, cudaStream_t st) {
  if (g_decoder < 0) g_decoder = getenv("LOPC_DECODER") ? atoi(getenv("LOPC_DECODER")) : 1;
  if (g_decoder == 2) {
    unsigned grid = 2u * (unsigned)(di->occ_decode > 0 ? di->occ_decode : 1);
    if (grid > 2 * chunks) grid = (unsigned)(2 * chunks);
    if (grid < 2) grid = 2;
    k_decode<<<grid, kCodecThreads, sizeof(DecSmem), st>>>(da);
  } else {
    uint64_t grid = (uint64_t)(di->occ_decode1 > 0 ? di->occ_decode1 : 1) * (uint64_t)di->sms;
    if (grid > chunks) grid = chunks;
    if (grid < 1) grid = 1;
    k_decode1<<<(unsigned)grid, kCodecThreads, sizeof(DecSmem2), st>>>(da);
  }
  CK(cudaGetLastError());
  return LOPC_OK;
}

// Pinned status slot for the single D2H read per call: one per host thread
// (a call blocks its thread until the slot has been read, so calls of
// different threads never share one).
thread_local Counters* tl_host_ctr = nullptr;
int host_ctr(Counters*& h) {
  if (!tl_host_ctr) CK(cudaMallocHost(&tl_host_ctr, sizeof(Counters)));
  h = tl_host_ctr;
  return LOPC_OK;
}

// Per-call CUDA-event marks (lopc_set_timing).  The events are created once
// per (thread, device) and reused, so timing adds no allocation to the call.
thread_local cudaEvent_t g_ev_all[kMaxDev][8] = {};
struct Timer {
  cudaEvent_t* ev = nullptr;
  int n = 0;
  bool on = false;
  cudaStream_t st = nullptr;
  int init(cudaStream_t s) {
    st = s;
    on = g_timing != 0;
    if (!on) return LOPC_OK;
    int dev;
    CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDev) return LOPC_E_ARG;
    ev = g_ev_all[dev];
    if (!ev[0])
      for (int i = 0; i < 8; ++i) CK(cudaEventCreate(&ev[i]));
    return LOPC_OK;
  }
  void mark() {
    if (on && n < 8) cudaEventRecord(ev[n++], st);
  }
  float ms(int a, int b) {
    float v = 0;
    if (on && b < n) cudaEventElapsedTime(&v, ev[a], ev[b]);
    return v;
  }
};

int map_err(uint32_t e) {
  if (e & kErrVersion) return LOPC_E_VERSION;
  if (e & kErrCorrupt) return LOPC_E_CORRUPT;
  if (e & kErrNoSpace) return LOPC_E_NOSPACE;
  if (e & (kErrBound | kErrOverflow | kErrPassCap)) return LOPC_E_INTERNAL;
  return LOPC_OK;
}

void write_header_host(uint8_t* h, const Shape& s, double eps, uint64_t total) {
  memset(h, 0, kHdrBytes);
  memcpy(h, "LOPC", 4);
  uint16_t ver = 1;
  memcpy(h + 4, &ver, 2);
  h[6] = (uint8_t)s.dtype;
  h[7] = (uint8_t)s.ndims;
  memcpy(h + 8, &s.d0, 8);
  memcpy(h + 16, &s.d1, 8);
  memcpy(h + 24, &s.d2, 8);
  memcpy(h + 32, &eps, 8);
  memcpy(h + 40, &s.n, 8);
  uint32_t cb = kChunkBytes, C = (uint32_t)s.C;
  memcpy(h + 48, &cb, 4);
  memcpy(h + 52, &C, 4);
  memcpy(h + 56, &total, 8);
}

RepairArgs make_repair_args(const Shape& sh, const void* x, double eps, uint8_t* ws, const CLayout& L) {
  RepairArgs ra{};
  ra.x = x;
  ra.flags = reinterpret_cast<uint32_t*>(ws + L.flags);
  ra.nseg = (int64_t)L.nseg;
  ra.s = reinterpret_cast<uint32_t*>(ws + L.s);
  ra.plist = ws + L.plist;
  ra.bitmap = reinterpret_cast<uint32_t*>(ws + L.bitmap);
  ra.cap = sh.n;
  ra.bmw = L.bmw;
  ra.ctr = reinterpret_cast<Counters*>(ws + L.ctr);
  ra.eps = eps;
  ra.inv = 1.0 / eps;
  ra.inv32 = inv32_of(eps);
  ra.d0 = (int64_t)sh.d0;
  ra.d1 = (int64_t)sh.d1;
  ra.d2 = (int64_t)sh.d2;
  ra.ntz = L.ntz;
  ra.nty = L.nty;
  ra.ntx = L.ntx;
  ra.ntiles = (int64_t)L.ntiles;
  ra.max_passes = 1 << 20;
  ra.own_lo = 0;
  ra.own_hi = (int64_t)sh.n;
  ra.skip_dense = 0;
  ra.prof = g_timing >= 2;
  ra.engine = 0;
  ra.cesc = reinterpret_cast<uint32_t*>(ws + L.cesc);
  ra.chunk_shift = sh.k == 4 ? 12 : 11;  // log2 of the elements per 16 KiB chunk
  return ra;
}


// TMA tensor map of x for the halo-box loads of k_quant_flags (driver entry
// point fetched at run time: no libcuda link dependency).  Returns false when
// TMA does not apply (unaligned base, rows not a multiple of 16 bytes).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode_tiled = nullptr;
std::once_flag g_encode_once;
int g_use_tma = 1;  // LOPC_NO_TMA=1 in the environment disables (tests cover both paths)

bool make_halo_map(const Shape& sh, const void* x, CUtensorMap* m) {
  std::call_once(g_encode_once, [] {
    const char* env = getenv("LOPC_NO_TMA");
    if (env && env[0] == '1') g_use_tma = 0;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_tiled = reinterpret_cast<EncodeTiledFn>(fn);
  });
  if (!g_use_tma || (uintptr_t)x % 16 || (sh.d2 * sh.k) % 16) return false;
  if (sh.d0 > (1ull << 31) || sh.d1 > (1ull << 31) || sh.d2 > (1ull << 31)) return false;
  if (!g_encode_tiled) return false;
  const CUtensorMapDataType dt = sh.k == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  CUresult r;
  if (sh.ndims == 3) {
    const cuuint64_t gd[3] = {sh.d2, sh.d1, sh.d0}, gs[2] = {sh.d2 * sh.k, sh.d1 * sh.d2 * sh.k};
    const cuuint32_t box[3] = {sh.k == 4 ? 40u : 36u, (cuuint32_t)Geo<3>::HY, (cuuint32_t)Geo<3>::HZ}, es[3] = {1, 1, 1};
    r = g_encode_tiled(m, dt, 3, const_cast<void*>(x), gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t gd[2] = {sh.d2, sh.d1}, gs[1] = {sh.d2 * sh.k};
    const cuuint32_t box[2] = {sh.k == 4 ? 40u : 36u, (cuuint32_t)Geo<2>::HY}, es[2] = {1, 1};
    r = g_encode_tiled(m, dt, 2, const_cast<void*>(x), gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS;
}

// a1 + a2: k_quant_flags over the tile grid (TMA halo loads when possible).
int launch_quant_flags(const Shape& sh, const RepairArgs& ra, const CLayout& L, cudaStream_t st) {
  const dim3 tgrid((unsigned)L.ntx, (unsigned)L.nty, (unsigned)L.ntz);
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  const bool tma = make_halo_map(sh, ra.x, &tm);
#define QR(TT, ND, IX)                                                                                          \
  do {                                                                                                          \
    if (tma)                                                                                                    \
      k_quant_flags<TT, ND, IX, true><<<tgrid, kRepairThreads, quant_flags_smem<TT, ND, true>(), st>>>(ra, tm);   \
    else                                                                                                        \
      k_quant_flags<TT, ND, IX, false><<<tgrid, kRepairThreads, quant_flags_smem<TT, ND, false>(), st>>>(ra, tm); \
  } while (0)
  if (use_i32(sh)) {
    if (sh.dtype == LOPC_F32) {
      if (sh.ndims == 3) QR(float, 3, int32_t); else QR(float, 2, int32_t);
    } else {
      if (sh.ndims == 3) QR(double, 3, int32_t); else QR(double, 2, int32_t);
    }
  } else {
    if (sh.dtype == LOPC_F32) {
      if (sh.ndims == 3) QR(float, 3, int64_t); else QR(float, 2, int64_t);
    } else {
      if (sh.ndims == 3) QR(double, 3, int64_t); else QR(double, 2, int64_t);
    }
  }
#undef QR
  CK(cudaGetLastError());
  g_stats.tma = tma ? 1 : 0;
  return LOPC_OK;
}

// a3: one cooperative k_sweep launch (dense pass unless ra.skip_dense).
int launch_sweep(const Shape& sh, RepairArgs& ra, const CLayout& L, cudaStream_t st) {
  DevInfo* di;
  int rc = dev_info(di);
  if (rc) return rc;
  const bool i32 = use_i32(sh);
  int occ = sh.ndims == 3 ? (i32 ? di->occ_sweep3 : di->occ_sweep3w) : (i32 ? di->occ_sweep2 : di->occ_sweep2w);
  uint64_t grid = (uint64_t)occ * di->sms;
  if (grid > L.ntiles) grid = L.ntiles;
  if (grid < 1) grid = 1;
  void* kargs[] = {&ra};
#define SW(ND, IX) \
  CK(cudaLaunchCooperativeKernel((void*)k_sweep<ND, IX>, dim3((unsigned)grid), dim3(kSweepThreads), kargs, 0, st))
  if (i32) {
    if (sh.ndims == 3) SW(3, int32_t); else SW(2, int32_t);
  } else {
    if (sh.ndims == 3) SW(3, int64_t); else SW(2, int64_t);
  }
#undef SW
  return LOPC_OK;
}

// a3 on the tile engine: one cooperative k_tiles launch (tile fixpoints over
// alternating shifted tilings, subbin planes), then the planes widened to one
// u32 per point for the encoder.
TileArgs make_tile_args(const Shape& sh, const RepairArgs& ra, uint8_t* ws, const CLayout& L) {
  TileArgs ta{};
  ta.flags = ra.flags;
  ta.sp = reinterpret_cast<uint32_t*>(ws + L.sp);
  ta.act[0] = reinterpret_cast<uint32_t*>(ws + L.act0);
  ta.act[1] = reinterpret_cast<uint32_t*>(ws + L.act1);
  ta.list[0] = reinterpret_cast<uint32_t*>(ws + L.list0);
  ta.list[1] = reinterpret_cast<uint32_t*>(ws + L.list1);
  ta.ctr = ra.ctr;
  ta.d0 = (int64_t)sh.d0;
  ta.d1 = (int64_t)sh.d1;
  ta.d2 = (int64_t)sh.d2;
  ta.nseg = (int64_t)L.nseg;
  memcpy(ta.nt, L.tnt, sizeof(ta.nt));
  ta.ntiles[0] = (uint32_t)L.tn[0];
  ta.ntiles[1] = (uint32_t)L.tn[1];
  ta.max_passes = 1 << 20;
  ta.prof = g_timing >= 2;
  ta.q0 = 1;
  return ta;
}

int launch_tiles(const Shape& sh, const RepairArgs& ra, uint8_t* ws, const CLayout& L, cudaStream_t st, bool widen,
                 int q0 = 1) {
  DevInfo* di;
  int rc = dev_info(di);
  if (rc) return rc;
  TileArgs ta = make_tile_args(sh, ra, ws, L);
  ta.q0 = q0;
  const int occ = sh.ndims == 3 ? di->occ_tiles3 : di->occ_tiles2;
  uint64_t grid = (uint64_t)occ * di->sms;
  const uint64_t need = (L.tn[1] + kTileWarps - 1) / kTileWarps;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  void* kargs[] = {&ta};
  if (sh.ndims == 3)
    CK(cudaLaunchCooperativeKernel((void*)k_tiles<3>, dim3((unsigned)grid), dim3(kTileThreads), kargs, 0, st));
  else
    CK(cudaLaunchCooperativeKernel((void*)k_tiles<2>, dim3((unsigned)grid), dim3(kTileThreads), kargs, 0, st));
  CK(cudaGetLastError());
  if (!widen) return LOPC_OK;  // compress: the encoder reads the planes
  uint64_t g2 = (sh.d0 * sh.d1 * L.nseg * 32 + 255) / 256;
  if (g2 > (uint64_t)di->sms * 16) g2 = (uint64_t)di->sms * 16;
  if (sh.ndims == 3)
    k_planes_to_s<3><<<(unsigned)g2, 256, 0, st>>>(ta.sp, ra.s, ta.d0, ta.d1, ta.d2, ta.nseg);
  else
    k_planes_to_s<2><<<(unsigned)g2, 256, 0, st>>>(ta.sp, ra.s, ta.d0, ta.d1, ta.d2, ta.nseg);
  CK(cudaGetLastError());
  return LOPC_OK;
}

// Repair engines: 0 = tile fixpoints (default; lopc_tiles.cuh), 1 = the
// paper's point worklist (f2), 2 = r1's dense tile pass + point worklist
// (k_sweep, u32 subbins; also the fallback when a subbin exceeds 8 planes).
enum { kEngTiles = 0, kEngPaper = 1, kEngSweep = 2 };
constexpr int kRetryU32 = 1;  // internal: re-run the repair on kEngSweep

// Steps a1-a3 (quantize, flags, repair to the fixpoint) on device input.
int run_repair(const Shape& sh, const void* x, double eps, uint8_t* ws, const CLayout& L, cudaStream_t st, Timer& tm,
               int engine, bool widen) {
  RepairArgs ra = make_repair_args(sh, x, eps, ws, L);
  ra.engine = engine == kEngPaper ? 1 : 0;
  int rc = launch_quant_flags(sh, ra, L, st);
  if (rc) return rc;
  if (ra.engine) CK(cudaMemsetAsync(ra.s, 0, 4 * sh.n, st));  // the worklist engine starts from s = 0
  tm.mark();
  if (engine == kEngTiles)
    rc = launch_tiles(sh, ra, ws, L, st, widen);
  else
    rc = launch_sweep(sh, ra, L, st);
  if (rc) return rc;
  tm.mark();
  return LOPC_OK;
}

// Workspace of the plain calls: one pool per (host thread, device), grown on
// demand.  The plain calls run on the legacy default stream and block until
// done, so a thread's pool is never in use by two calls at once.
thread_local void* tl_pool[kMaxDev] = {};
thread_local size_t tl_pool_size[kMaxDev] = {};
int workspace_for(size_t need, void*& ws, size_t& ws_bytes) {
  int dev;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) return LOPC_E_ARG;
  void*& pool = tl_pool[dev];
  if (pool && tl_pool_size[dev] < need) {
    CK(cudaDeviceSynchronize());  // the legacy stream's last use of the old pool
    cudaFree(pool);
    pool = nullptr;
    tl_pool_size[dev] = 0;
  }
  if (!pool) {
    size_t sz = need < (1u << 20) ? (1u << 20) : need;
    CK(cudaMalloc(&pool, sz));
    tl_pool_size[dev] = sz;
  }
  ws = pool;
  ws_bytes = tl_pool_size[dev];
  return LOPC_OK;
}

}  // namespace

extern "C" {

int lopc_abi_version(void) { return LOPC_ABI_VERSION; }

const char* lopc_strerror(int code) {
  switch (code) {
    case LOPC_OK: return "ok";
    case LOPC_E_ARG: return "invalid argument";
    case LOPC_E_SHAPE: return "invalid shape";
    case LOPC_E_NOSPACE: return "output or workspace too small";
    case LOPC_E_CORRUPT: return "corrupt stream";
    case LOPC_E_VERSION: return "unsupported stream version";
    case LOPC_E_CUDA: return "CUDA error";
    case LOPC_E_NCCL: return "NCCL error";
    case LOPC_E_INTERNAL: return "internal self-check failed";
    default: return "unknown error";
  }
}

const char* lopc_last_error_string(void) { return g_errmsg; }

void lopc_set_timing(int enable) { g_timing = enable; }

int lopc_set_decoder(int decoder) {
  if (decoder != 1 && decoder != 2) return LOPC_E_ARG;
  g_decoder = decoder;
  return LOPC_OK;
}

int lopc_set_index64(int force) {
  g_force_i64 = force != 0;
  return LOPC_OK;
}

int lopc_set_repair_engine(int engine) {
  if (engine < 0 || engine > 2) return LOPC_E_ARG;
  g_engine = engine;
  return LOPC_OK;
}

int lopc_last_stats(lopc_stats* out) {
  if (!out) return LOPC_E_ARG;
  *out = g_stats;
  return LOPC_OK;
}

size_t lopc_compress_bound(int ndims, const uint64_t* dims, int dtype) {
  Shape s;
  if (make_shape(ndims, dims, dtype, s)) return 0;
  return kHdrBytes + 8 * s.C + 2ull * kChunkBytes * s.C;
}

size_t lopc_compress_workspace_bytes(int ndims, const uint64_t* dims, int dtype, int host_io) {
  Shape s;
  if (make_shape(ndims, dims, dtype, s)) return 0;
  return compress_layout(s, host_io != 0, host_io != 0).total;
}

size_t lopc_decompress_workspace_bytes(size_t in_bytes, size_t out_bytes, int host_io) {
  size_t cmax = in_bytes > kHdrBytes ? (in_bytes - kHdrBytes) / 16 + 1 : 1;
  size_t t = al(sizeof(Counters)) + al(8 * (cmax / kScanTile + 1)) + al(8 * cmax);
  if (host_io) t += al(in_bytes) + al(out_bytes);
  return t;
}

int lopc_stream_info(const void* host_hdr, size_t n, int* ndims, uint64_t* dims3, int* dtype, double* eps,
                     uint64_t* n_elems, uint32_t* n_chunks) {
  if (!host_hdr) return LOPC_E_ARG;
  if (n < kHdrBytes) return LOPC_E_CORRUPT;
  const uint8_t* h = static_cast<const uint8_t*>(host_hdr);
  if (memcmp(h, "LOPC", 4) != 0) return LOPC_E_CORRUPT;
  uint16_t ver;
  memcpy(&ver, h + 4, 2);
  if (ver != 1) return LOPC_E_VERSION;
  int dt = h[6], nd = h[7];
  if (dt > 1 || (nd != 2 && nd != 3)) return LOPC_E_CORRUPT;
  uint64_t d[3], nn;
  double e;
  uint32_t C;
  memcpy(d, h + 8, 24);
  memcpy(&e, h + 32, 8);
  memcpy(&nn, h + 40, 8);
  memcpy(&C, h + 52, 4);
  if (nd == 2 && d[0] != 1) return LOPC_E_CORRUPT;
  if (ndims) *ndims = nd;
  if (dims3) memcpy(dims3, d, 24);
  if (dtype) *dtype = dt;
  if (eps) *eps = e;
  if (n_elems) *n_elems = nn;
  if (n_chunks) *n_chunks = C;
  return LOPC_OK;
}

}  // extern "C"

namespace {
int compress_impl(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, void* out,
                  size_t* out_bytes, void* workspace, size_t workspace_bytes, void* stream, int engine) {
  if (!out_bytes) return LOPC_E_ARG;
  Shape sh;
  int rc = make_shape(ndims, dims, dtype, sh);
  if (rc) return rc;
  if (!out || (!in && sh.n)) return LOPC_E_ARG;
  if ((rc = check_eps(eps))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool host_in = !is_device_ptr(in), host_out = !is_device_ptr(out);
  const size_t cap = *out_bytes;
  g_stats = lopc_stats{};
  g_stats.n_elems = sh.n;
  g_stats.n_chunks = sh.C;
  if (sh.n == 0) {
    if (cap < kHdrBytes) {
      *out_bytes = kHdrBytes;
      return LOPC_E_NOSPACE;
    }
    uint8_t h[kHdrBytes];
    write_header_host(h, sh, eps, kHdrBytes);
    if (host_out)
      memcpy(out, h, kHdrBytes);
    else {
      CK(cudaMemcpyAsync(out, h, kHdrBytes, cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
    }
    *out_bytes = kHdrBytes;
    g_stats.total_bytes = kHdrBytes;
    return LOPC_OK;
  }
  const CLayout L = compress_layout(sh, host_in, host_out);
  if (L.nty > 65535 || L.ntz > 65535) return LOPC_E_SHAPE;  // tile launch grid limit
  if (!workspace || workspace_bytes < L.total) return LOPC_E_NOSPACE;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  g_stats.n_tiles = L.ntiles;
  Counters* hc;
  if ((rc = host_ctr(hc))) return rc;
  DevInfo* di;
  if ((rc = dev_info(di))) return rc;
  Timer tm;
  if ((rc = tm.init(st))) return rc;
  tm.mark();  // 0
  const void* x = in;
  if (host_in) {
    CK(cudaMemcpyAsync(ws + L.stage_in, in, sh.k * sh.n, cudaMemcpyHostToDevice, st));
    x = ws + L.stage_in;
  }
  tm.mark();  // 1
  CK(cudaMemsetAsync(ws, 0, L.zero_end, st));
  tm.mark();  // 2
  uint8_t* dst = host_out ? ws + L.stage_out : static_cast<uint8_t*>(out);
  Counters* dctr = reinterpret_cast<Counters*>(ws + L.ctr);
  EncodeArgs ea{};
  ea.x = x;
  ea.s = reinterpret_cast<const uint32_t*>(ws + L.s);
  ea.stage = ws + L.stage;
  ea.sizes = reinterpret_cast<uint32_t*>(ws + L.sizes);
  ea.ctr = dctr;
  ea.eps = eps;
  ea.inv = 1.0 / eps;
  ea.inv32 = inv32_of(eps);
  ea.n = sh.n;
  ea.C = (uint32_t)sh.C;
  ea.ndims = sh.ndims;
  ea.vec = ((uintptr_t)x % 16 == 0) && ((uintptr_t)ea.s % 16 == 0);
  ea.prof = g_timing >= 2;
  ea.d0 = sh.d0;
  ea.d1 = sh.d1;
  ea.d2 = sh.d2;
  set_escape_limits(ea, sh.dtype == LOPC_F64, eps);
  const size_t smem = sizeof(EncSmem);
  // Stream order: repair, bin-stream encode, subbin-stream encode.  (r1
  // measured the bin encode beside the repair on a side stream: slower, the
  // repair fills the SMs; with subbin planes the bin CTAs also run a4, which
  // needs the repaired subbins.)
  if ((rc = run_repair(sh, x, eps, ws, L, st, tm, engine, false))) return rc;  // marks 3, 4
  if (engine == kEngTiles) {  // the encoder reads the subbin planes and, in chunks with escapes, the flags' escape words
    ea.sp = reinterpret_cast<const uint32_t*>(ws + L.sp);
    ea.flags = reinterpret_cast<const uint32_t*>(ws + L.flags);
    ea.nseg = (int64_t)L.nseg;
    ea.sw = sh.ndims == 3 ? Geo<3>::SW : Geo<2>::SW;
    ea.cesc = reinterpret_cast<const uint32_t*>(ws + L.cesc);
  }
  // The two roles are independent (both read only x / the repaired
  // subbins): the subbin grid runs on the side stream beside the bin grid
  // (their tails overlap: cfg2 encode 0.239 -> 0.225 ms; cfg3 within 1 %).
  // One interleaved grid of both roles was measured much slower (cfg3 1.15
  // -> 2.0 ms: two large role bodies in one kernel, sharing the SMs' caches).
  // LOPC_ENC_SERIAL=1: the two grids one after the other on `st`.
  static const bool enc_serial = getenv("LOPC_ENC_SERIAL") && atoi(getenv("LOPC_ENC_SERIAL")) == 1;
  if (enc_serial) {
    launch_encode(ea, sh.dtype == LOPC_F64, 1, (unsigned)sh.C, smem, st);
    launch_encode(ea, sh.dtype == LOPC_F64, 2, (unsigned)sh.C, smem, st);
  } else {
    CK(cudaEventRecord(di->ev_fork, st));
    CK(cudaStreamWaitEvent(di->side, di->ev_fork, 0));
    launch_encode(ea, sh.dtype == LOPC_F64, 2, (unsigned)sh.C, smem, di->side);
    launch_encode(ea, sh.dtype == LOPC_F64, 1, (unsigned)sh.C, smem, st);
    CK(cudaGetLastError());
    CK(cudaEventRecord(di->ev_join, di->side));
    CK(cudaStreamWaitEvent(st, di->ev_join, 0));
  }
  CK(cudaGetLastError());
  tm.mark();  // 5
  ScanArgs sa{};
  sa.sizes = ea.sizes;
  sa.C = (uint32_t)sh.C;
  sa.off = reinterpret_cast<uint64_t*>(ws + L.off);
  sa.state = reinterpret_cast<uint64_t*>(ws + L.state);
  sa.ctr = dctr;
  sa.base = kHdrBytes + 8 * sh.C;
  k_chunk_scan<<<(unsigned)((sh.C + kScanTile - 1) / kScanTile), kScanThreads, 0, st>>>(sa);
  CK(cudaGetLastError());
  PlaceArgs pa{};
  pa.stage = ws + L.stage;
  pa.sizes = ea.sizes;
  pa.off = sa.off;
  pa.out = dst;
  pa.table = dst + kHdrBytes;
  pa.header = 1;
  pa.out_cap = host_out ? (kHdrBytes + 8 * sh.C + 2ull * kChunkBytes * sh.C) : cap;
  pa.ctr = dctr;
  pa.C = (uint32_t)sh.C;
  pa.dtype = sh.dtype;
  pa.ndims = sh.ndims;
  pa.d0 = sh.d0;
  pa.d1 = sh.d1;
  pa.d2 = sh.d2;
  pa.n = sh.n;
  pa.eps = eps;
  {
    uint64_t pg = (sh.C + 7) / 8;
    const uint64_t pmax = (uint64_t)di->sms * 8;
    if (pg > pmax) pg = pmax;
    k_place<<<(unsigned)pg, 256, 0, st>>>(pa);
  }
  CK(cudaGetLastError());
  tm.mark();  // 6
  CK(cudaMemcpyAsync(hc, ws + L.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const uint64_t total = hc->total_bytes;
  g_stats.sweep_passes = hc->passes;
  g_stats.worklist_points = hc->worklist_points;
  g_stats.inner_iters = hc->inner_iters;
  g_stats.escapes = hc->escapes;
  g_stats.bin_bytes = hc->bin_bytes;
  g_stats.sub_bytes = hc->sub_bytes;
  g_stats.total_bytes = total;
  g_stats.max_subbin = hc->max_s;
  g_stats.raised = hc->raised;
  for (int i = 0; i < 16; ++i) g_stats.pass_items[i] = hc->pass_items[i];
  for (int i = 0; i < 16; ++i) g_stats.phase_cycles[i] = hc->phase[i];
  for (int i = 0; i < 16; ++i) g_stats.pass_us[i] = (float)(hc->pass_ns[i] * 1e-3);
  if (g_timing >= 2)  // diagnostic: k_tiles visit counters (tile engine) / k_sweep dense-pass cycles in phase_cycles[8..11]
    for (int i = 0; i < 4; ++i) g_stats.phase_cycles[8 + i] = hc->dense_cycles[i];
  uint32_t err = hc->err;
  if (err & kErrPlanes) return kRetryU32;  // a subbin above 8 planes: the caller re-runs on the u32 engine
  if (hc->passes >= (unsigned long long)(1 << 20) &&
      (engine == kEngTiles ? hc->tl_count[(hc->passes + 1) % 3] : hc->list_count[(hc->passes + 1) % 3]) != 0)
    err |= kErrPassCap;
  if ((rc = map_err(err & ~kErrNoSpace))) return rc;
  if (total > cap) {
    *out_bytes = total;
    return LOPC_E_NOSPACE;
  }
  if (host_out) {
    CK(cudaMemcpyAsync(out, dst, total, cudaMemcpyDeviceToHost, st));
  }
  tm.mark();  // 7
  CK(cudaStreamSynchronize(st));
  *out_bytes = total;
  g_stats.launches = tm.on ? 5 : 6;
  if (tm.on) {
    g_stats.timing_valid = 1;
    g_stats.ms_h2d = tm.ms(0, 1);
    g_stats.ms_quant_repair = tm.ms(2, 3);
    g_stats.ms_sweep = tm.ms(3, 4);
    g_stats.ms_encode = tm.ms(4, 5);
    g_stats.ms_place = tm.ms(5, 6);
    g_stats.ms_d2h = tm.ms(6, 7);
    g_stats.ms_total = tm.ms(0, 7);
  }
  return LOPC_OK;
}

}  // namespace

extern "C" {

int lopc_compress_ex(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, void* out,
                     size_t* out_bytes, void* workspace, size_t workspace_bytes, void* stream) {
  const size_t cap = out_bytes ? *out_bytes : 0;
  int rc = compress_impl(in, ndims, dims, dtype, eps, out, out_bytes, workspace, workspace_bytes, stream, g_engine);
  if (rc == kRetryU32) {  // the tile engine's 8 subbin planes overflowed: the u32 engine, same result
    *out_bytes = cap;
    rc = compress_impl(in, ndims, dims, dtype, eps, out, out_bytes, workspace, workspace_bytes, stream, kEngSweep);
  }
  return rc;
}

int lopc_compress(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, void* out,
                  size_t* out_bytes) {
  size_t need = lopc_compress_workspace_bytes(ndims, dims, dtype, 1);
  if (need == 0) {
    Shape s;
    int rc = make_shape(ndims, dims, dtype, s);
    return rc ? rc : LOPC_E_ARG;
  }
  void* ws;
  size_t wsb;
  int rc = workspace_for(need, ws, wsb);
  if (rc) return rc;
  return lopc_compress_ex(in, ndims, dims, dtype, eps, out, out_bytes, ws, wsb, nullptr);
}

int lopc_repair_ex(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, uint16_t* flags_out,
                   uint32_t* subbins_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!in) return LOPC_E_ARG;
  Shape sh;
  int rc = make_shape(ndims, dims, dtype, sh);
  if (rc) return rc;
  if ((rc = check_eps(eps))) return rc;
  if (sh.n == 0) return LOPC_OK;
  if (!is_device_ptr(in)) return LOPC_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const CLayout L = compress_layout(sh, false, false);
  if (L.nty > 65535 || L.ntz > 65535) return LOPC_E_SHAPE;
  if (!workspace || workspace_bytes < L.total) return LOPC_E_NOSPACE;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  Counters* hc;
  if ((rc = host_ctr(hc))) return rc;
  Timer tm;
  for (int engine = g_engine;;) {
    CK(cudaMemsetAsync(ws, 0, L.zero_end, st));
    if ((rc = run_repair(sh, in, eps, ws, L, st, tm, engine, true))) return rc;
    CK(cudaMemcpyAsync(hc, ws + L.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!(hc->err & kErrPlanes)) break;
    engine = kEngSweep;  // a subbin above 8 planes: the u32 engine
  }
  if (subbins_out) CK(cudaMemcpyAsync(subbins_out, ws + L.s, 4 * sh.n, cudaMemcpyDeviceToDevice, st));
  if (flags_out) {
    const uint32_t* fw = reinterpret_cast<const uint32_t*>(ws + L.flags);
    if (sh.ndims == 3)
      k_unpack_flags<3><<<1024, 256, 0, st>>>(fw, flags_out, sh.d0, sh.d1, sh.d2, (int64_t)L.nseg);
    else
      k_unpack_flags<2><<<1024, 256, 0, st>>>(fw, flags_out, sh.d0, sh.d1, sh.d2, (int64_t)L.nseg);
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(st));
  g_stats = lopc_stats{};
  g_stats.n_elems = sh.n;
  g_stats.n_tiles = L.ntiles;
  g_stats.sweep_passes = hc->passes;
  g_stats.worklist_points = hc->worklist_points;
  g_stats.inner_iters = hc->inner_iters;
  g_stats.max_subbin = hc->max_s;
  g_stats.raised = hc->raised;
  for (int i = 0; i < 16; ++i) g_stats.pass_items[i] = hc->pass_items[i];
  return map_err(hc->err);
}

// Host side of parse_header (k_decode) plus the size-table checks of
// k_chunk_scan's validating mode, on a stream in host memory; fills the
// payload offsets.  false: not a valid stream (the caller takes the device
// path, which reports the precise error).
static bool host_stream_plan(const uint8_t* in, size_t in_bytes, size_t out_cap, Hdr& h,
                             std::vector<uint64_t>& off) {
  if (in_bytes < kHdrBytes) return false;
  uint32_t h32[16];
  uint64_t h64[8];
  memcpy(h32, in, 64);
  memcpy(h64, in, 64);
  if (h32[0] != 0x43504f4cu || (h32[1] & 0xffffu) != 1u) return false;
  h = Hdr{};
  h.dtype = (h32[1] >> 16) & 0xff;
  h.ndims = (h32[1] >> 24) & 0xff;
  if (h.dtype > 1 || (h.ndims != 2 && h.ndims != 3)) return false;
  h.d0 = h64[1];
  h.d1 = h64[2];
  h.d2 = h64[3];
  if (h.ndims == 2 && h.d0 != 1) return false;
  const uint64_t lim = 1ull << 40;
  if (h.d0 > lim || h.d1 > lim || h.d2 > lim || h.d0 * h.d1 > lim) return false;
  h.n = h64[5];
  if (h.d0 * h.d1 * h.d2 != h.n || h.n > lim || h.n == 0) return false;
  memcpy(&h.eps, in + 32, 8);
  if (!(h.eps >= 0x1p-900 && h.eps <= 0x1p1000)) return false;
  if (h32[12] != kChunkBytes) return false;
  const uint64_t W = kChunkBytes / (h.dtype ? 8u : 4u);
  h.C = h32[13];
  if ((uint64_t)h.C != (h.n + W - 1) / W || h64[7] != in_bytes) return false;
  if ((uint64_t)kHdrBytes + 8ull * h.C > in_bytes || h.n * (h.dtype ? 8u : 4u) > out_cap) return false;
  const uint8_t* tab = in + kHdrBytes;
  off.resize(h.C);
  uint64_t o = kHdrBytes + 8ull * h.C;
  for (uint32_t c = 0; c < h.C; ++c) {
    uint32_t bs, ss;
    memcpy(&bs, tab + 8ull * c, 4);
    memcpy(&ss, tab + 8ull * c + 4, 4);
    if (!(bs >= 4 && bs <= kChunkBytes && (bs & 3u) == 0 && ss >= 4 && ss <= kChunkBytes && (ss & 3u) == 0))
      return false;
    off[c] = o;
    o += bs + ss;
  }
  if (o != in_bytes) return false;
  h.ok = true;
  h.err = 0;
  return true;
}

int lopc_decompress_ex(const void* in, size_t in_bytes, void* out, size_t out_capacity, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (!in) return LOPC_E_ARG;
  if (!out && out_capacity) return LOPC_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool host_in = !is_device_ptr(in), host_out = !is_device_ptr(out);
  const size_t cmax = in_bytes > kHdrBytes ? (in_bytes - kHdrBytes) / 16 + 1 : 1;
  const size_t ntile = cmax / kScanTile + 1;
  size_t o_ctr = 0, o_state = al(sizeof(Counters)), o_off = o_state + al(8 * ntile), o_in = o_off + al(8 * cmax);
  size_t o_out = o_in + (host_in ? al(in_bytes) : 0);
  size_t need = o_out + (host_out ? al(out_capacity) : 0);
  if (!workspace || workspace_bytes < need) return LOPC_E_NOSPACE;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  int rc;
  Counters* hc;
  if ((rc = host_ctr(hc))) return rc;
  DevInfo* di;
  if ((rc = dev_info(di))) return rc;
  Timer tm;
  if ((rc = tm.init(st))) return rc;
  g_stats = lopc_stats{};
  // Host stream -> host values, per-kernel timing off: a pipeline of up to
  // kPipeRanges chunk ranges — H2D of range i's payloads (stream st), k_decode of range i
  // (side stream, after its H2D), D2H of its values (second side stream,
  // after its decode) — so the PCIe copies overlap the decode.  Offsets come
  // from the host copy of the size table (validated as k_chunk_scan would).
  Hdr hh;
  std::vector<uint64_t> hoff;
  if (host_in && host_out && !tm.on && host_stream_plan(static_cast<const uint8_t*>(in), in_bytes, out_capacity, hh, hoff)) {
    const uint8_t* hin = static_cast<const uint8_t*>(in);
    uint8_t* dsrc = ws + o_in;
    uint64_t* doff = reinterpret_cast<uint64_t*>(ws + o_off);
    const uint32_t C = hh.C;
    const uint64_t k = hh.dtype ? 8 : 4, W = kChunkBytes / k;
    CK(cudaMemsetAsync(ws + o_ctr, 0, sizeof(Counters), st));
    CK(cudaMemcpyAsync(dsrc, hin, kHdrBytes + 8ull * C, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(doff, hoff.data(), 8ull * C, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(di->ev_fork, st));
    CK(cudaStreamWaitEvent(di->side, di->ev_fork, 0));
    CK(cudaStreamWaitEvent(di->side2, di->ev_fork, 0));
    const int K = C < (uint32_t)kPipeRanges ? (int)C : kPipeRanges;
    for (int i = 0; i < K; ++i) {
      const uint64_t cb = (uint64_t)C * i / K, ce = (uint64_t)C * (i + 1) / K;
      const uint64_t b0 = hoff[cb], b1 = ce == C ? in_bytes : hoff[ce];
      CK(cudaMemcpyAsync(dsrc + b0, hin + b0, b1 - b0, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(di->ev_in[i], st));
      CK(cudaStreamWaitEvent(di->side, di->ev_in[i], 0));
      DecodeArgs da{};
      da.in = dsrc;
      da.in_bytes = in_bytes;
      da.out = ws + o_out;
      da.out_cap = out_capacity;
      da.off = doff + cb;
      da.table = reinterpret_cast<const uint32_t*>(dsrc + kHdrBytes) + 2 * cb;
      da.base = dsrc;
      da.c_begin = cb;
      da.c_count = ce - cb;
      da.state_cap = C;
      da.ctr = reinterpret_cast<Counters*>(ws + o_ctr);
      da.slab = 1;
      da.given = hh;
      if ((rc = launch_decode(di, da, ce - cb, di->side))) return rc;
      CK(cudaEventRecord(di->ev_dec[i], di->side));
      CK(cudaStreamWaitEvent(di->side2, di->ev_dec[i], 0));
      const uint64_t e0 = cb * W, e1 = ce * W < hh.n ? ce * W : hh.n;
      CK(cudaMemcpyAsync(static_cast<uint8_t*>(out) + e0 * k, ws + o_out + e0 * k, (e1 - e0) * k,
                         cudaMemcpyDeviceToHost, di->side2));
    }
    CK(cudaEventRecord(di->ev_out, di->side2));
    CK(cudaStreamWaitEvent(st, di->ev_out, 0));
    CK(cudaMemcpyAsync(hc, ws + o_ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int i = 0; i < 16; ++i) g_stats.phase_cycles[i] = hc->phase[i];
    if ((rc = map_err(hc->err))) return rc;
    g_stats.launches = (uint32_t)K;
    return LOPC_OK;
  }
  tm.mark();  // 0
  const uint8_t* src = static_cast<const uint8_t*>(in);
  if (host_in) {
    CK(cudaMemcpyAsync(ws + o_in, in, in_bytes, cudaMemcpyHostToDevice, st));
    src = ws + o_in;
  }
  tm.mark();  // 1
  CK(cudaMemsetAsync(ws, 0, o_off, st));
  ScanArgs sa{};
  sa.in = src;
  sa.in_bytes = in_bytes;
  sa.off = reinterpret_cast<uint64_t*>(ws + o_off);
  sa.state = reinterpret_cast<uint64_t*>(ws + o_state);
  sa.ctr = reinterpret_cast<Counters*>(ws + o_ctr);
  sa.validate = 1;
  sa.expect_total = in_bytes;
  k_chunk_scan<<<(unsigned)ntile, kScanThreads, 0, st>>>(sa);
  CK(cudaGetLastError());
  tm.mark();  // 2
  DecodeArgs da{};
  da.in = src;
  da.in_bytes = in_bytes;
  da.out = host_out ? (void*)(ws + o_out) : out;
  da.out_cap = out_capacity;
  da.off = sa.off;
  da.table = reinterpret_cast<const uint32_t*>(src + kHdrBytes);
  da.base = src;
  da.c_begin = 0;
  da.state_cap = cmax;
  da.prof = g_timing >= 2;
  da.ctr = reinterpret_cast<Counters*>(ws + o_ctr);
  if ((rc = launch_decode(di, da, cmax, st))) return rc;
  tm.mark();  // 3
  CK(cudaMemcpyAsync(hc, ws + o_ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int i = 0; i < 16; ++i) g_stats.phase_cycles[i] = hc->phase[i];
  if ((rc = map_err(hc->err))) return rc;
  if (host_out) {
    // N * k from the (validated) header
    uint64_t nk = 0;
    uint8_t h[kHdrBytes];
    if (host_in)
      memcpy(h, in, kHdrBytes);
    else
      CK(cudaMemcpy(h, in, kHdrBytes, cudaMemcpyDeviceToHost));
    uint64_t n;
    memcpy(&n, h + 40, 8);
    nk = n * (h[6] ? 8 : 4);
    CK(cudaMemcpyAsync(out, ws + o_out, nk, cudaMemcpyDeviceToHost, st));
  }
  tm.mark();  // 4
  CK(cudaStreamSynchronize(st));
  g_stats.launches = 2;
  if (tm.on) {
    g_stats.timing_valid = 1;
    g_stats.ms_h2d = tm.ms(0, 1);
    g_stats.ms_place = tm.ms(1, 2);
    g_stats.ms_decode = tm.ms(2, 3);
    g_stats.ms_d2h = tm.ms(3, 4);
    g_stats.ms_total = tm.ms(0, 4);
  }
  return LOPC_OK;
}

int lopc_decompress(const void* in, size_t in_bytes, void* out, size_t out_capacity) {
  size_t need = lopc_decompress_workspace_bytes(in_bytes, out_capacity, 1);
  void* ws;
  size_t wsb;
  int rc = workspace_for(need, ws, wsb);
  if (rc) return rc;
  return lopc_decompress_ex(in, in_bytes, out, out_capacity, ws, wsb, nullptr);
}

}  // extern "C"


// ---- row a0 / NEXT f1: NOA eps on the device -------------------------------
namespace {
double host_value_of_key(long long k, int dtype) {
  if (dtype == LOPC_F32) {
    const uint32_t b = k >= 0 ? (uint32_t)k : (0x80000000u | (uint32_t)(-k));
    float f;
    memcpy(&f, &b, 4);
    return (double)f;
  }
  const uint64_t b = k >= 0 ? (uint64_t)k : (0x8000000000000000ull | (uint64_t)(-k));
  double d;
  memcpy(&d, &b, 8);
  return d;
}
}  // namespace

extern "C" {

int lopc_value_range(const void* in, int ndims, const uint64_t* dims, int dtype, double* vmin, double* vmax,
                     uint64_t* n_finite, void* workspace, size_t workspace_bytes, void* stream) {
  Shape sh;
  int rc = make_shape(ndims, dims, dtype, sh);
  if (rc) return rc;
  if ((!in && sh.n) || !workspace || workspace_bytes < sizeof(RangeOut)) return !workspace ? LOPC_E_ARG : LOPC_E_NOSPACE;
  if (sh.n && !is_device_ptr(in)) return LOPC_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  RangeOut h{LLONG_MAX, LLONG_MIN, 0};
  RangeOut* d = static_cast<RangeOut*>(workspace);
  CK(cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  if (sh.n) {
    DevInfo* di;
    if ((rc = dev_info(di))) return rc;
    uint64_t grid = (sh.n / 4 + 255) / 256;
    const uint64_t gmax = (uint64_t)di->sms * 8;
    if (grid > gmax) grid = gmax;
    if (grid < 1) grid = 1;
    if (sh.dtype == LOPC_F32)
      k_value_range<float><<<(unsigned)grid, 256, 0, st>>>(static_cast<const float*>(in), sh.n, d);
    else
      k_value_range<double><<<(unsigned)grid, 256, 0, st>>>(static_cast<const double*>(in), sh.n, d);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (n_finite) *n_finite = h.n_finite;
  if (vmin) *vmin = h.n_finite ? host_value_of_key(h.kmin, dtype) : 0.0;
  if (vmax) *vmax = h.n_finite ? host_value_of_key(h.kmax, dtype) : 0.0;
  return LOPC_OK;
}

double lopc_noa_eps(double vmin, double vmax, uint64_t n_finite, double rel) {
  if (!n_finite) return rel;
  const double r = vmax - vmin;
  return r > 0 ? rel * r : rel;
}

int lopc_compress_noa(const void* in, int ndims, const uint64_t* dims, int dtype, double rel, void* out,
                      size_t* out_bytes, double* eps_used, void* workspace, size_t workspace_bytes, void* stream) {
  double lo = 0, hi = 0;
  uint64_t nf = 0;
  int rc = lopc_value_range(in, ndims, dims, dtype, &lo, &hi, &nf, workspace, workspace_bytes, stream);
  if (rc) return rc;
  const double eps = lopc_noa_eps(lo, hi, nf, rel);
  if (eps_used) *eps_used = eps;
  return lopc_compress_ex(in, ndims, dims, dtype, eps, out, out_bytes, workspace, workspace_bytes, stream);
}

}  // extern "C"


// ---- k_check: order / bound / error statistics on the device ---------------
extern "C" int lopc_check(const void* x, const void* y, int ndims, const uint64_t* dims, int dtype, double eps,
                          lopc_check_result* res, void* workspace, size_t workspace_bytes, void* stream) {
  Shape sh;
  int rc = make_shape(ndims, dims, dtype, sh);
  if (rc) return rc;
  if (!res || !workspace) return LOPC_E_ARG;
  if ((rc = check_eps(eps))) return rc;
  if (workspace_bytes < sizeof(CheckOut)) return LOPC_E_NOSPACE;
  if (sh.n && (!is_device_ptr(x) || !is_device_ptr(y))) return LOPC_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CheckOut* d = static_cast<CheckOut*>(workspace);
  CK(cudaMemsetAsync(d, 0, sizeof(CheckOut), st));
  if (sh.n) {
    DevInfo* di;
    if ((rc = dev_info(di))) return rc;
    uint64_t grid = (sh.n + 255) / 256;
    if (grid > (uint64_t)di->sms * 8) grid = (uint64_t)di->sms * 8;
    const float i32 = inv32_of(eps);
    const double inv = 1.0 / eps;
#define KC(TT, ND)                                                                                             \
  k_check<TT, ND><<<(unsigned)grid, 256, 0, st>>>(static_cast<const TT*>(x), static_cast<const TT*>(y),       \
                                                   (int64_t)sh.d0, (int64_t)sh.d1, (int64_t)sh.d2, eps, inv, i32, d)
    if (sh.dtype == LOPC_F32) {
      if (sh.ndims == 3) KC(float, 3); else KC(float, 2);
    } else {
      if (sh.ndims == 3) KC(double, 3); else KC(double, 2);
    }
#undef KC
    CK(cudaGetLastError());
  }
  CheckOut h;
  CK(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  res->order_violations = h.order_bad;
  res->bound_violations = h.bound_bad;
  res->n_regular = h.n_regular;
  memcpy(&res->max_abs_err, &h.max_err_bits, 8);
  res->sum_sq_err = h.sum_sq;
  return LOPC_OK;
}


// ---- k_critical: critical-point preservation (Table III) on the device -----
namespace {
// Link adjacency of the Freudenthal star: slots i, j are joined iff their
// offsets differ by a star offset (then {p, p+o_i, p+o_j} is a triangle).
LinkAdj link_adj(int ndims) {
  LinkAdj L{};
  const int D = ndims == 3 ? 7 : 3;
  int o[14][3];
  for (int j = 0; j < 2 * D; ++j) {
    const int e = (j < D ? j : j - D) + 1, sg = j < D ? 1 : -1;
    o[j][0] = ndims == 3 ? sg * ((e >> 2) & 1) : 0;
    o[j][1] = sg * ((e >> 1) & 1);
    o[j][2] = sg * (e & 1);
  }
  for (int i = 0; i < 2 * D; ++i)
    for (int j = 0; j < 2 * D; ++j) {
      if (i == j) continue;
      bool pos = true, neg = true, nz = false;
      for (int c = 0; c < 3; ++c) {
        const int d = o[j][c] - o[i][c];
        pos = pos && (d == 0 || d == 1);
        neg = neg && (d == 0 || d == -1);
        nz = nz || d != 0;
      }
      if (nz && (pos || neg)) L.adj[i] |= (uint16_t)(1u << j);
    }
  return L;
}
}  // namespace

extern "C" int lopc_critical_points(const void* x, const void* y, int ndims, const uint64_t* dims, int dtype,
                                    lopc_critical_result* res, void* workspace, size_t workspace_bytes, void* stream) {
  Shape sh;
  int rc = make_shape(ndims, dims, dtype, sh);
  if (rc) return rc;
  if (!res || !workspace) return LOPC_E_ARG;
  if (workspace_bytes < sizeof(CritOut)) return LOPC_E_NOSPACE;
  if (sh.n && (!is_device_ptr(x) || !is_device_ptr(y))) return LOPC_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CritOut* d = static_cast<CritOut*>(workspace);
  CK(cudaMemsetAsync(d, 0, sizeof(CritOut), st));
  if (sh.n) {
    DevInfo* di;
    if ((rc = dev_info(di))) return rc;
    uint64_t grid = (sh.n + 255) / 256;
    if (grid > (uint64_t)di->sms * 8) grid = (uint64_t)di->sms * 8;
    const LinkAdj L = link_adj(sh.ndims);
#define KR(TT, ND)                                                                                          \
  k_critical<TT, ND><<<(unsigned)grid, 256, 0, st>>>(static_cast<const TT*>(x), static_cast<const TT*>(y), \
                                                      (int64_t)sh.d0, (int64_t)sh.d1, (int64_t)sh.d2, L, d)
    if (sh.dtype == LOPC_F32) {
      if (sh.ndims == 3) KR(float, 3); else KR(float, 2);
    } else {
      if (sh.ndims == 3) KR(double, 3); else KR(double, 2);
    }
#undef KR
    CK(cudaGetLastError());
  }
  CritOut h;
  CK(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  res->false_positives = h.fp;
  res->false_negatives = h.fn;
  res->false_types = h.ft;
  res->pair_mismatches = h.pair_bad;
  res->critical_x = h.crit_x;
  res->critical_y = h.crit_y;
  return LOPC_OK;
}

#include "lopc_slab.cuh"
