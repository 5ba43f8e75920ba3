// lopc_repair.cuh — quantize + flags + local-order repair.
//
// PAPER.md Alg. 1 computes bins, zero subbins and per-point flags;
// Alg. 2 raises subbins until no violation remains.  The result
// is the unique least fixpoint of s(p) = max(0, max_{n->p} s(n) + w) over the
// same-bin arcs n -> p (n precedes p in the SoS order, w = [idx n > idx p]);
// any monotone relaxation schedule reaches it (reading G14).  The schedule
// here is B200-shaped, not the paper's point worklist:
//
//   k_quant_flags   one CTA per 2048-point tile (3D 8x8x32, 2D 64x32) with a
//                   one-cell halo of (value key, exact bin) pairs in shared
//                   memory; a neighbour n is a same-bin predecessor of p iff
//                   bin(n) = bin(p) and key(n) < key(p) (+e slots; <= for -e
//                   slots, the SoS tie rule G4).
//                   Flags are stored as bit planes: for every 32-point x-row
//                   segment, word j holds star slot j of its 32 points (one
//                   warp ballot per slot).
//   k_sweep         one persistent cooperative kernel.
//     pass 1        dense, one warp per tile, bit-parallel: the level sets
//                   Lev_L = {p : s(p) >= L} of the tile-local fixpoint (halo
//                   held at 0) satisfy
//                     Lev_L = mu X. OR_{+e j} F_j & Lev_{L-1}(p + e_j)
//                                 | OR_{-e j} F_j & X(p - e_j),
//                   computed 32 points per word: the -e closure is a Jacobi
//                   loop over rows with a carry-lookahead fill along x.  s is
//                   the number of non-empty levels.  A point with s > 0 on
//                   the tile border enqueues the out-of-tile points it feeds.
//     passes >= 2   sparse, point-level: the paper's own worklist schedule
//                   (Alg. 2 with the dual worklists of P:220, atomicMax P:218)
//                   on the remaining tail; a raised point enqueues its
//                   successors.  Grid-wide barrier between passes; stop when
//                   a worklist is empty.  No host round trip per pass.
//
// Every value ever written is <= the least fixpoint (lower bounds relaxed by
// monotone max), and when the worklist empties every point satisfies the
// Bellman equation, so the result is the least fixpoint, independent of
// scheduling.
#pragma once
#include <cooperative_groups.h>
#include <cuda.h>  // CUtensorMap (TMA halo loads)

#include <type_traits>

#include "lopc_device.cuh"

namespace lopc {

template <int NDIM>
struct Geo;
template <>
struct Geo<3> {
  static constexpr int TZ = 8, TY = 8, TX = 32;
  static constexpr int HZ = TZ + 2, HY = TY + 2, HX = TX + 2;
  static constexpr int ZH = 1;
  static constexpr int D = 7;   // +e offsets (G2)
  static constexpr int SW = 16; // words per 32-point flag segment (14 slots, word 14 = escapes)
};
template <>
struct Geo<2> {
  static constexpr int TZ = 1, TY = 64, TX = 32;
  static constexpr int HZ = 1, HY = TY + 2, HX = TX + 2;
  static constexpr int ZH = 0;
  static constexpr int D = 3;
  static constexpr int SW = 8;  // 6 slots, word 6 = escapes
};

#ifndef LOPC_SWEEP_CTAS
#define LOPC_SWEEP_CTAS 3  // k_sweep CTAs per SM (register budget 85; 4 and 5 measured slower)
#endif
#ifndef LOPC_QF_CESC_LATE
#define LOPC_QF_CESC_LATE 1  // k_quant_flags marks the chunks with escapes after its row loop (not in the store path)
#endif
#ifndef LOPC_QF_CTAS64
#define LOPC_QF_CTAS64 3  // k_quant_flags CTAs (of 512) per SM for f64 (4: 32 registers, 9.29 -> 9.42 ms on cfg5)
#endif
#ifndef LOPC_QF_CTAS
#define LOPC_QF_CTAS 4  // k_quant_flags CTAs (of 512) per SM for f32 (32 registers, no spills: 0.180 -> 0.172 ms on cfg2); f64 keeps 3
#endif
#ifndef LOPC_SUBS_CTAS
#define LOPC_SUBS_CTAS 6  // k_encode<T, 2> (subbin stream) CTAs per SM: 40 registers (r2: with the planes-mode subbin role 1.4-1.8 % faster than 5)
#endif
#ifndef LOPC_CODEC_CTAS
#define LOPC_CODEC_CTAS 6  // k_encode / k_decode CTAs per SM (register budget 40; 4 and 5 measured slower)
#endif
constexpr int kRepairThreads = 512;
constexpr int kSweepThreads = 256;
constexpr int kSweepWarps = kSweepThreads / 32;
constexpr int kPassHist = 16;
constexpr int kLevelPlanes = 8;  // dense-pass levels per tile before handing over to the worklist
#ifndef LOPC_SMALL_LIST
#define LOPC_SMALL_LIST 256
#endif
constexpr unsigned long long kSmallList = LOPC_SMALL_LIST;  // sparse passes this short run on block 0 alone
#ifndef LOPC_CHASE
#define LOPC_CHASE 8
#endif
#ifndef LOPC_CHASE_BUDGET
#define LOPC_CHASE_BUDGET 12
#endif
#ifndef LOPC_CHASE_MAX_PASS
#define LOPC_CHASE_MAX_PASS 2  // chase only in the first sparse pass (cfg3 sweep 5.26 -> 4.99 ms, cfg2 unchanged)
#endif
#ifndef LOPC_CHASE_MAX_LOG2
#define LOPC_CHASE_MAX_LOG2 18
#endif
constexpr int kChase = LOPC_CHASE;                // depth-first successor stack per lane in the sparse passes
constexpr int kChaseBudget = LOPC_CHASE_BUDGET;   // chased evaluations per list point
constexpr unsigned long long kChaseMaxList = 1ull << LOPC_CHASE_MAX_LOG2;  // chase only when the pass list is at most this long
constexpr int kMaxLevel = (1 << kLevelPlanes) - 1;

// Star slot j (G2): j < D is +e, j >= D is -e, with e = (j mod D) + 1 read
// as bits (dz, dy, dx) in 3D and (dy, dx) in 2D: 3D order (0,0,1) (0,1,0)
// (0,1,1) (1,0,0) (1,0,1) (1,1,0) (1,1,1); 2D (0,1) (1,0) (1,1).
template <int NDIM>
__host__ __device__ __forceinline__ constexpr int slot_dz(int j) {
  return NDIM == 2 ? 0 : (j < Geo<NDIM>::D ? 1 : -1) * ((((j % Geo<NDIM>::D) + 1) >> 2) & 1);
}
template <int NDIM>
__host__ __device__ __forceinline__ constexpr int slot_dy(int j) {
  return (j < Geo<NDIM>::D ? 1 : -1) * ((((j % Geo<NDIM>::D) + 1) >> 1) & 1);
}
template <int NDIM>
__host__ __device__ __forceinline__ constexpr int slot_dx(int j) {
  return (j < Geo<NDIM>::D ? 1 : -1) * (((j % Geo<NDIM>::D) + 1) & 1);
}
template <int NDIM>
__host__ __device__ __forceinline__ constexpr int slot_hoff(int j) {
  using G = Geo<NDIM>;
  return slot_dz<NDIM>(j) * G::HY * G::HX + slot_dy<NDIM>(j) * G::HX + slot_dx<NDIM>(j);
}
template <int NDIM>
__host__ __device__ __forceinline__ constexpr int slot_opp(int j) {
  return j < Geo<NDIM>::D ? j + Geo<NDIM>::D : j - Geo<NDIM>::D;
}

struct Counters {
  uint32_t ticket2;  // k_chunk_scan tiles
  uint32_t tile_ticket;  // k_sweep dense pass: dynamic tile assignment
  uint32_t pad0;
  uint32_t ticket;
  uint32_t err;  // kErr* bits
  uint32_t max_s;
  uint32_t pad[2];
  unsigned long long escapes;
  unsigned long long total_bytes;
  unsigned long long passes;
  unsigned long long worklist_points;
  unsigned long long bin_bytes;
  unsigned long long sub_bytes;
  unsigned long long inner_iters;
  unsigned long long raised;
  unsigned long long list_count[3];  // point worklists (rotating)
  uint32_t pass_items[kPassHist];    // [1] tiles of the dense pass, [q>1] worklist points of pass q
  unsigned long long phase[16];      // diagnostic: SM cycles per codec phase (lopc_set_timing(2))
  unsigned long long ghost_changed;  // slab mode: ghosts raised by the last k_ghost_inject
  unsigned long long pass_ns[kPassHist];  // diagnostic (prof): k_sweep pass end times, ns after the launch
  unsigned long long dense_cycles[4];     // diagnostic (prof): dense pass load / levels / s write / border, per warp
  uint32_t tl_count[3];   // k_tiles: active-tile list lengths (rotating by pass)
  uint32_t tl_ticket[3];  // k_tiles: per-pass tile tickets (rotating)
};

// Diagnostic phase clock: thread 0 of a block adds the cycles since the last
// mark to ctr->phase[i] (only when enabled; all threads are past a barrier).
struct PhaseClock {
  long long t;
  bool on;
  __device__ __forceinline__ void start(bool enable) {
    on = enable && threadIdx.x == 0;
    if (on) t = clock64();
  }
  __device__ __forceinline__ void mark(Counters* c, int i) {
    if (on) {
      const long long n = clock64();
      atomicAdd(&c->phase[i], (unsigned long long)(n - t));
      t = n;
    }
  }
};

enum : uint32_t {
  kErrBound = 1u,
  kErrCorrupt = 2u,
  kErrNoSpace = 4u,
  kErrOverflow = 8u,
  kErrPassCap = 16u,
  kErrVersion = 32u,
  kErrPlanes = 64u,  // k_tiles: a subbin above kMaxPlaneLevel (the host reruns with the u32 engine)
};

struct RepairArgs {
  const void* x;
  uint32_t* flags;    // bit-plane flags: segment (z, y, xs) at ((z*d1 + y)*nseg + xs)*SW
  uint32_t* s;
  void* plist;        // 2 x cap point indices (Idx-sized), worklists of passes >= 2
  uint32_t* bitmap;   // 2 x bmw words: per-point "already enqueued" bits, self-clearing
  uint64_t cap;       // entries per worklist (= N)
  uint64_t bmw;       // words per bitmap
  Counters* ctr;
  double eps, inv;
  float inv32;         // RN32(1/eps) for the f32 fast path, NaN = off
  int64_t d0, d1, d2;  // z, y, x extents (2D: d0 = 1)
  int64_t nseg;        // 32-point segments per x-row
  int ntz, nty, ntx;
  int64_t ntiles;
  int max_passes;
  int64_t own_lo, own_hi;  // points with incoming arcs: [own_lo, own_hi) (slab mode; else [0, N))
  int skip_dense;          // k_sweep: start with the sparse passes (slab rounds >= 2)
  int prof;                // diagnostic: k_sweep pass times (ns) into ctr->phase[14..15]
  int engine;              // 0: dense tile pass + worklist tail; 1: the paper's point worklist from pass 1 (f2)
  uint32_t* cesc;          // k_quant_flags: bit c set when chunk c holds an escape (box chunks in slab mode: unused)
  int chunk_shift;         // log2 of the elements per chunk
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Enqueue point q for pass `pass` if `valid` (dedup by the pass's bitmap).
// Warp-collective (all 32 lanes call it together): one list-counter atomic
// per warp instead of one per point.
template <typename Idx>
__device__ __forceinline__ void enqueue_warp(const RepairArgs& a, Idx q, bool valid, int pass) {
  using UIdx = typename std::make_unsigned<Idx>::type;
  bool fresh = false;
  if (valid) {
    const uint32_t bit = 1u << ((uint32_t)q & 31u);
    const uint32_t old = atomicOr(&a.bitmap[(size_t)(pass & 1) * a.bmw + ((UIdx)q >> 5)], bit);
    fresh = !(old & bit);
  }
  const uint32_t m = __ballot_sync(0xffffffffu, fresh);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&a.ctr->list_count[pass % 3], (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (fresh) static_cast<UIdx*>(a.plist)[(size_t)(pass & 1) * a.cap + base + __popc(m & ((1u << lane) - 1u))] = (UIdx)q;
}

template <int NDIM, typename Idx>
__device__ __forceinline__ Idx slot_goff(int j, Idx plane, Idx d2) {
  return (Idx)slot_dz<NDIM>(j) * plane + (Idx)slot_dy<NDIM>(j) * d2 + (Idx)slot_dx<NDIM>(j);
}

// Successors of point p: the slots j whose neighbour q = p + off(j) has an
// arc from p (q's flag slot opp(j) is set).  All flag loads are independent.
template <int NDIM, typename Idx>
__device__ __forceinline__ uint32_t succ_cand(const RepairArgs& a, bool active, Idx z, Idx y, Idx x) {
  using G = Geo<NDIM>;
  constexpr int D = G::D;
  constexpr int SW = G::SW;
  const Idx d0 = (Idx)a.d0, d1 = (Idx)a.d1, d2 = (Idx)a.d2;
  const size_t nseg = (size_t)a.nseg;
  uint32_t w[2 * D];
  uint32_t inb = 0;
#pragma unroll
  for (int j = 0; j < 2 * D; ++j) {
    const Idx qx = x + slot_dx<NDIM>(j), qy = y + slot_dy<NDIM>(j), qz = z + slot_dz<NDIM>(j);
    const bool v = active && qx >= 0 && qx < d2 && qy >= 0 && qy < d1 && qz >= 0 && qz < d0;
    w[j] = v ? __ldg(a.flags + ((size_t)(qz * d1 + qy) * nseg + (size_t)(qx >> 5)) * SW + slot_opp<NDIM>(j)) : 0u;
    inb |= (uint32_t)v << j;
  }
  uint32_t cand = 0;
#pragma unroll
  for (int j = 0; j < 2 * D; ++j) {
    const uint32_t qx = (uint32_t)(x + slot_dx<NDIM>(j));
    cand |= (((w[j] >> (qx & 31u)) & 1u) & (inb >> j)) << j;
  }
  return cand;
}

// Enqueue the points p + off(j), j in `mask`, for pass `pass`: all bitmap
// atomics are issued before any result is used, and the warp reserves its
// list slots with one atomicAdd (warp-collective: all 32 lanes call).
template <int NDIM, typename Idx>
__device__ __forceinline__ void enqueue_mask(const RepairArgs& a, Idx p, uint32_t mask, int pass) {
  using UIdx = typename std::make_unsigned<Idx>::type;
  constexpr int D = Geo<NDIM>::D;
  const Idx d2 = (Idx)a.d2, plane = (Idx)a.d1 * d2;
  uint32_t old[2 * D];
#pragma unroll
  for (int j = 0; j < 2 * D; ++j) {
    old[j] = 0;
    if ((mask >> j) & 1u) {
      const Idx q = p + slot_goff<NDIM, Idx>(j, plane, d2);
      old[j] = atomicOr(&a.bitmap[(size_t)(pass & 1) * a.bmw + ((UIdx)q >> 5)], 1u << ((uint32_t)q & 31u));
    }
  }
  uint32_t fresh = 0;
#pragma unroll
  for (int j = 0; j < 2 * D; ++j) {
    const Idx q = p + slot_goff<NDIM, Idx>(j, plane, d2);
    fresh |= (((mask >> j) & 1u) & ((~old[j] >> ((uint32_t)q & 31u)) & 1u)) << j;
  }
  const int lane = threadIdx.x & 31;
  const uint32_t c = __popc(fresh);
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  if (!tot) return;
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(&a.ctr->list_count[pass % 3], (unsigned long long)tot);
  base = __shfl_sync(0xffffffffu, base, 31) + (incl - c);
  UIdx* L = static_cast<UIdx*>(a.plist) + (size_t)(pass & 1) * a.cap;
  for (uint32_t m = fresh; m; m &= m - 1) {
    const int j = __ffs(m) - 1;
    L[base++] = (UIdx)(p + slot_goff<NDIM, Idx>(j, plane, d2));
  }
}

// Rows of the halo box handled per warp, and elements per lane per row.
template <int NDIM>
struct HaloRows {
  static constexpr int R = Geo<NDIM>::HZ * Geo<NDIM>::HY;
  static constexpr int RPW = (R + kRepairThreads / 32 - 1) / (kRepairThreads / 32);
  static constexpr int EPL = (Geo<NDIM>::HX + 31) / 32;
};

template <typename T>
__device__ __forceinline__ T value_of_key(typename VT<T>::I k);
template <>
__device__ __forceinline__ float value_of_key<float>(int32_t k) {
  return __uint_as_float(bits_of_key32(k));
}
template <>
__device__ __forceinline__ double value_of_key<double>(int64_t k) {
  return __longlong_as_double((long long)bits_of_key64(k));
}

// Load a (HZ x HY x HX) halo box of words starting at grid coordinate
// (z0 - ZH, y0 - 1, x0 - 1) into registers, one warp per row; every load is
// issued before any use.  Out-of-grid elements read as `fill`.
template <int NDIM, typename W, typename Idx>
struct HaloLoad {
  using HR = HaloRows<NDIM>;
  W v[HR::RPW][HR::EPL];
  bool ok[HR::RPW][HR::EPL];
  __device__ __forceinline__ void load(const W* __restrict__ base, Idx z0, Idx y0, Idx x0, Idx d0, Idx d1, Idx d2,
                                       bool interior, W fill) {
    using G = Geo<NDIM>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Idx plane = d1 * d2;
    const W* org = base + ((z0 - G::ZH) * plane + (y0 - 1) * d2 + (x0 - 1));
#pragma unroll
    for (int i = 0; i < HR::RPW; ++i) {
      const int r = warp + i * (kRepairThreads / 32);
      const int hz = r / G::HY, hy = r % G::HY;
      const W* row = org + ((Idx)hz * plane + (Idx)hy * d2);
      bool rowok = r < HR::R;
      if (!interior) {
        const Idx gz = z0 + hz - G::ZH, gy = y0 + hy - 1;
        rowok = rowok && gz >= 0 && gz < d0 && gy >= 0 && gy < d1;
      }
#pragma unroll
      for (int e = 0; e < HR::EPL; ++e) {
        const int hx = lane + 32 * e;
        bool o = rowok && hx < G::HX;
        if (!interior) {
          const Idx gx = x0 + hx - 1;
          o = o && gx >= 0 && gx < d2;
        }
        ok[i][e] = o;
        v[i][e] = o ? __ldg(row + hx) : fill;
      }
    }
  }
};

template <int NDIM, typename Idx>
__device__ __forceinline__ bool tile_interior(Idx z0, Idx y0, Idx x0, Idx d0, Idx d1, Idx d2) {
  using G = Geo<NDIM>;
  return z0 - G::ZH >= 0 && z0 + G::TZ + G::ZH <= d0 && y0 >= 1 && y0 + G::TY + 1 <= d1 && x0 >= 1 &&
         x0 + G::TX + 1 <= d2;
}

// ---------------------------------------------------------------------------
// k_quant_flags: a1 (exact bins of the tile's points) + a2 (flags).
//
// Same-bin test without the neighbour's bin: keys (ord) are monotone in x and
// bins are key intervals [key(lo(b)), key(lo(b+1))), so for a regular p with
// bin b_p and any neighbour n,
//   n ~> p  <=>  key(lo(b_p)) <= key_n < key_p        (+e slot: n has larger idx)
//   n ~> p  <=>  key(lo(b_p)) <= key_n <= key_p       (-e slot: n wins ties, G4)
// (key_n in [lo(b_p), x_p] puts n in bin b_p, hence regular; NaN and
// out-of-grid neighbours carry a key below every lo key; an escaped p gets
// lo key = max, so it has no incoming arcs, O8).  Halo points therefore need
// only their key; only the tile's own points are quantized.
// ---------------------------------------------------------------------------
// Halo box layout in shared memory.  Plain load: row stride HX (34), column
// 0 = x0 - 1.  TMA load: the box must start on a 16-byte boundary in x (and
// its inner extent be a multiple of 16 B), so it starts at x0 - 16/k:
// column XO = 16/k - 1 holds x0 - 1, stride 40 (f32) / 36 (f64).
template <typename T, int NDIM, bool TMA>
__host__ __device__ constexpr int halo_stride() {
  return TMA ? (sizeof(T) == 4 ? 40 : 36) : Geo<NDIM>::HX;
}
template <typename T, bool TMA>
__host__ __device__ constexpr int halo_xoff() {
  return TMA ? 16 / (int)sizeof(T) - 1 : 0;
}

template <typename T, int NDIM, bool TMA = false>
constexpr size_t quant_flags_smem() {
  using G = Geo<NDIM>;
  return (size_t)G::HZ * G::HY * halo_stride<T, NDIM, TMA>() * sizeof(typename VT<T>::I) + 128;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <typename T, int NDIM, typename Idx, bool TMA>
__global__ void __launch_bounds__(kRepairThreads, sizeof(T) == 4 ? LOPC_QF_CTAS : LOPC_QF_CTAS64) k_quant_flags(RepairArgs a, const __grid_constant__ CUtensorMap tmap) {
  using G = Geo<NDIM>;
  using I = typename VT<T>::I;
  using U = typename VT<T>::U;
  using HR = HaloRows<NDIM>;
  constexpr int HXS = halo_stride<T, NDIM, TMA>();
  constexpr int XO = halo_xoff<T, TMA>();
  constexpr int TP = G::TZ * G::TY * G::TX;
  constexpr int PPT = TP / kRepairThreads;
  constexpr int D = G::D;
  constexpr int NB = G::HZ * G::HY * HXS;  // halo box elements
  constexpr I kLow = (I)VT<T>::kSentinel;                                    // NaN / outside the grid
  constexpr I kHigh = (I)(((typename std::make_unsigned<I>::type)kLow) - 1u);  // max: escaped p

  extern __shared__ __align__(128) uint8_t qf_smem[];
  I* K = reinterpret_cast<I*>(qf_smem);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = blockIdx.x, ty = blockIdx.y, tz = blockIdx.z;  // 3D launch grid: no index division
  const Idx d0 = (Idx)a.d0, d1 = (Idx)a.d1, d2 = (Idx)a.d2;
  const Idx z0 = (Idx)tz * G::TZ, y0 = (Idx)ty * G::TY, x0 = (Idx)tx * G::TX;
  const bool interior = tile_interior<NDIM, Idx>(z0, y0, x0, d0, d1, d2);

  // TMA needs non-negative box coordinates: the first tile row / column /
  // plane (halo start at -1) takes the plain load.
  bool via_tma = false;
  if constexpr (TMA) via_tma = x0 >= 16 / (int)sizeof(T) && y0 >= 1 && z0 >= G::ZH;
  if (via_tma) {
    // halo box (z0-ZH.., y0-1.., x0-1..) by one TMA tile load; out-of-grid
    // elements arrive as 0 and are marked below
    uint64_t* bar = reinterpret_cast<uint64_t*>(qf_smem + (size_t)NB * sizeof(U));
    const uint32_t sb = smem_u32(bar);
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"((uint32_t)(NB * sizeof(U)))
                   : "memory");
      const int cx = (int)x0 - 1 - XO, cy = (int)y0 - 1, cz = (int)z0 - G::ZH;
      if constexpr (NDIM == 3)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                smem_u32(qf_smem)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(cx), "r"(cy), "r"(cz), "r"(sb)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(qf_smem)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(cx), "r"(cy), "r"(sb)
            : "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(sb)
                   : "memory");
    // raw bits -> keys in place, 16 bytes per step (EV elements); a row of
    // the box is HXS / EV vectors, so the row test is once per vector
    // (the plain-load instantiation never takes this path: EV = 1 there)
    constexpr int EV = HXS % (16 / (int)sizeof(U)) == 0 ? 16 / (int)sizeof(U) : 1, VPR = HXS / EV;
    struct alignas(EV * sizeof(U)) Vec {
      U e[EV];
    };
    Vec* v4 = reinterpret_cast<Vec*>(qf_smem);
    for (int i4 = tid; i4 < NB / EV; i4 += kRepairThreads) {
      Vec v = v4[i4];
      U* u = v.e;
      bool rowok = true;
      int hx0 = 0;
      if (!interior) {
        const int row = i4 / VPR, hz = row / G::HY, hy = row % G::HY;
        hx0 = (i4 % VPR) * EV;
        const Idx gz = z0 + hz - G::ZH, gy = y0 + hy - 1;
        rowok = gz >= 0 && gz < d0 && gy >= 0 && gy < d1;
      }
#pragma unroll
      for (int e = 0; e < EV; ++e) {
        bool ok = (u[e] & ~VT<T>::kSignBit) <= VT<T>::kInfBits;  // not NaN
        if (!interior) {
          const Idx gx = x0 + (hx0 + e) - 1 - XO;
          ok = ok && rowok && gx >= 0 && gx < d2;
        }
        u[e] = (U)(ok ? (I)key_of(u[e]) : kLow);
      }
      v4[i4] = v;
    }
  } else {
    // halo: keys only
    HaloLoad<NDIM, U, Idx> L;
    L.load(static_cast<const U*>(a.x), z0, y0, x0, d0, d1, d2, interior, (U)0);
#pragma unroll
    for (int i = 0; i < HR::RPW; ++i) {
      const int r = warp + i * (kRepairThreads / 32);
#pragma unroll
      for (int e = 0; e < HR::EPL; ++e) {
        const int hx = lane + 32 * e;
        if (r < HR::R && hx < G::HX) {
          const U u = L.v[i][e];
          const bool nan = (u & ~VT<T>::kSignBit) > VT<T>::kInfBits;
          K[r * HXS + hx + XO] = (L.ok[i][e] && !nan) ? (I)key_of(u) : kLow;
        }
      }
    }
  }
  __syncthreads();

  // a1 + a2 (Alg. 1 loop 2): warp w, step k handles tile row (w + 16k): lane = x.
  // Flags leave as one ballot per slot (bit plane); lane 0 stores the segment.
#if LOPC_QF_CESC_LATE
  uint32_t escrows = 0;  // bit k: row step k stored a segment with escapes (marked after the loop)
#endif
#ifndef LOPC_QF_UNROLL
#define LOPC_QF_UNROLL 1  // the row loop rolled: 0.856 -> 0.832 ms on cfg3 (unroll 2: 0.842)
#endif
  constexpr int kQfUnroll = LOPC_QF_UNROLL;
#pragma unroll kQfUnroll
  for (int k = 0; k < PPT; ++k) {
    const int row = warp + k * (kRepairThreads / 32);
    const int lz = row / G::TY, ly = row % G::TY;
    const int h = ((lz + G::ZH) * G::HY + (ly + 1)) * HXS + (lane + 1 + XO);
    const I kp = K[h];
    I lok = kHigh;
    if (kp != kLow) {
      const T xp = value_of_key<T>(kp);
      I b;
      bool reg = qtry(xp, a.inv32, a.inv, b);
      if (!reg) {  // rare: near a half-integer, huge bins, +-Inf (exact path, out of line)
        const int64_t r = quantize_slow<T>(xp, a.eps, a.inv);
        reg = r != kEscape;
        b = (I)r;
      }
      if (reg) lok = lo_key<T>((int64_t)b, a.eps);
    }
    uint32_t wv[G::SW];  // the ballots are warp-uniform: lane 0 stores the segment
#pragma unroll
    for (int j = 0; j < G::SW; ++j) wv[j] = 0;
    // lok <= kn < kp (+e) / <= kp (-e) as one unsigned range test per slot:
    // (kn - lok) mod 2^w < span; span = 0 for an escaped / NaN p (no arcs)
    using UI = typename std::make_unsigned<I>::type;
    const UI span = lok <= kp ? (UI)((UI)kp - (UI)lok) : (UI)0;
    const UI spanle = lok <= kp ? (UI)(span + 1u) : (UI)0;
#pragma unroll
    for (int j = 0; j < 2 * D; ++j) {
      const I kn = K[h + slot_dz<NDIM>(j) * G::HY * HXS + slot_dy<NDIM>(j) * HXS + slot_dx<NDIM>(j)];
      const bool arc = (UI)((UI)kn - (UI)lok) < (j < D ? span : spanle);
      wv[j] = __ballot_sync(0xffffffffu, arc);
    }
    const Idx gz = z0 + lz, gy = y0 + ly;
    // word SW-2 (otherwise padding): escape bits (non-regular in-grid points:
    // NaN, +-Inf, |b| > BINMAX), read by the subbin encoder in planes mode
    // instead of x.  (A separate bitmap of one u32 per segment was measured:
    // the extra scattered 4-byte stores cost k_quant_flags 9 % on cfg3, more
    // than the encoder's sector reads of this word save.)
    wv[G::SW - 2] = __ballot_sync(0xffffffffu, lok == kHigh && gz < d0 && gy < d1 && x0 + lane < d2);
#if LOPC_QF_CESC_LATE
    escrows |= (uint32_t)(wv[G::SW - 2] != 0u) << k;
#endif
    if (lane == 0 && gz < d0 && gy < d1) {
      const Idx rb = (gz * d1 + gy) * d2 + x0;
#if !LOPC_QF_CESC_LATE
      if (wv[G::SW - 2]) {  // the chunk(s) of this segment's escapes (rare): the subbin encoder reads their escape words
        const uint32_t e = wv[G::SW - 2];
        const uint64_t c0 = (uint64_t)(rb + (Idx)(__ffs(e) - 1)) >> a.chunk_shift;
        const uint64_t c1 = (uint64_t)(rb + (Idx)(31 - __clz(e))) >> a.chunk_shift;
        atomicOr(&a.cesc[c0 >> 5], 1u << (c0 & 31));
        if (c1 != c0) atomicOr(&a.cesc[c1 >> 5], 1u << (c1 & 31));
      }
#endif
      if (rb < (Idx)a.own_lo || rb + 32 > (Idx)a.own_hi) {
        // slab mode: points outside the owned range get no incoming arcs
        const Idx lo_rel = (Idx)a.own_lo - rb, hi_rel = (Idx)a.own_hi - rb;
        uint32_t own = 0xffffffffu;
        if (lo_rel > 0) own = lo_rel >= 32 ? 0u : own << (uint32_t)lo_rel;
        if (hi_rel < 32) own &= hi_rel <= 0 ? 0u : (0xffffffffu >> (uint32_t)(32 - hi_rel));
#pragma unroll
        for (int j = 0; j < G::SW; ++j) wv[j] &= own;
      }
      uint4* dst = reinterpret_cast<uint4*>(a.flags + ((size_t)(gz * d1 + gy) * (size_t)a.nseg + (size_t)tx) * G::SW);
#pragma unroll
      for (int q = 0; q < G::SW / 4; ++q) dst[q] = make_uint4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
    }
  }
#if LOPC_QF_CESC_LATE
  if (lane == 0 && escrows) {  // rare: the chunks of the row segments with escapes (first and last point: a superset)
    for (int k = 0; k < PPT; ++k) {
      if (!((escrows >> k) & 1u)) continue;
      const int row = warp + k * (kRepairThreads / 32);
      const Idx gz = z0 + row / G::TY, gy = y0 + row % G::TY;
      const Idx rb = (gz * d1 + gy) * d2 + x0;
      const Idx re = rb + (x0 + 32 <= d2 ? 31 : d2 - 1 - x0);
      const uint64_t c0 = (uint64_t)rb >> a.chunk_shift, c1 = (uint64_t)re >> a.chunk_shift;
      atomicOr(&a.cesc[c0 >> 5], 1u << (c0 & 31));
      if (c1 != c0) atomicOr(&a.cesc[c1 >> 5], 1u << (c1 & 31));
    }
  }
#endif
}

// ---------------------------------------------------------------------------
// k_sweep
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t xshift(uint32_t v, int dx) {
  // value of the neighbour at x + dx, placed at bit x
  return dx > 0 ? (v >> 1) : (dx < 0 ? (v << 1) : v);
}

// Carry-lookahead fill along x: bit x is set if seed x is, or if mask bit x
// is set and bit x-1 of the result is (the -x slot, weight 0).
__device__ __forceinline__ uint32_t xfill(uint32_t g, uint32_t p) {
  g |= p & (g << 1);
  p &= p << 1;
  g |= p & (g << 2);
  p &= p << 2;
  g |= p & (g << 4);
  p &= p << 4;
  g |= p & (g << 8);
  p &= p << 8;
  g |= p & (g << 16);
  return g;
}

// flags of one point from its bit-plane segment
template <int NDIM>
__device__ __forceinline__ uint32_t point_flags(const uint32_t* seg, uint32_t bit) {
  constexpr int SW = Geo<NDIM>::SW;
  const uint4* s4 = reinterpret_cast<const uint4*>(seg);
  uint32_t f = 0;
#pragma unroll
  for (int q = 0; q < SW / 4; ++q) {
    const uint4 w = __ldg(s4 + q);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (4 * q + i < 2 * Geo<NDIM>::D) f |= ((ws[i] >> bit) & 1u) << (4 * q + i);
  }
  return f;
}

struct SweepSmem {
  uint32_t cur[kSweepWarps][64];   // level rows being closed
  uint32_t prev[kSweepWarps][64];  // Lev_{L-1} rows
};

template <int NDIM, typename Idx>
__global__ void __launch_bounds__(kSweepThreads, LOPC_SWEEP_CTAS) k_sweep(RepairArgs a) {
  namespace cg = cooperative_groups;
  using G = Geo<NDIM>;
  using UIdx = typename std::make_unsigned<Idx>::type;
  constexpr int D = G::D;
  constexpr int SW = G::SW;
  constexpr int JX = D;  // the -x slot (0,0,-1): weight 0, closed by xfill

  __shared__ SweepSmem S;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* cur = S.cur[warp];
  uint32_t* prv = S.prev[warp];
  unsigned long long my_levels = 0;
  unsigned my_raised = 0;
  uint32_t my_max = 0;
  const Idx d0 = (Idx)a.d0, d1 = (Idx)a.d1, d2 = (Idx)a.d2;
  const Idx plane = d1 * d2;
  const size_t nseg = (size_t)a.nseg;
  const uint32_t ntx = (uint32_t)a.ntx, ntxy = (uint32_t)a.ntx * (uint32_t)a.nty;

  const uint64_t t_start = (a.prof && tid == 0 && blockIdx.x == 0) ? gtimer() : 0;
  // ---- pass 1: dense, one warp per tile, bit-parallel levels -----------------
  const uint32_t gwarp = blockIdx.x * kSweepWarps + warp, nwarps = gridDim.x * kSweepWarps;
  const uint32_t ntl = (a.skip_dense || a.engine) ? 0u : (uint32_t)a.ntiles;
  uint32_t tile = 0;
  if (lane == 0) tile = atomicAdd(&a.ctr->tile_ticket, 1u);
  tile = __shfl_sync(0xffffffffu, tile, 0);
  for (; tile < ntl;) {
    const uint32_t tz = tile / ntxy, rem = tile - tz * ntxy;
    const uint32_t ty = rem / ntx, tx = rem - ty * ntx;
    const Idx z0 = (Idx)tz * G::TZ, y0 = (Idx)ty * G::TY, x0 = (Idx)tx * G::TX;
    const uint32_t vmask = x0 + 32 <= d2 ? 0xffffffffu : ((1u << (uint32_t)(d2 - x0)) - 1u);
    // own rows rr = lane + 32*i: (lz, ly)
    uint32_t F[2][2 * D];
    int lz[2], ly[2];
    bool rin[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int rr = lane + 32 * i;
      lz[i] = rr / G::TY;
      ly[i] = rr % G::TY;
      rin[i] = z0 + lz[i] < d0 && y0 + ly[i] < d1;
      const uint4* seg = reinterpret_cast<const uint4*>(
          a.flags + ((size_t)((z0 + lz[i]) * d1 + (y0 + ly[i])) * nseg + tx) * SW);
#pragma unroll
      for (int q = 0; q < SW / 4; ++q) {
        const uint4 w = rin[i] ? __ldg(seg + q) : make_uint4(0, 0, 0, 0);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * q + t < 2 * D) F[i][4 * q + t] = ws[t];
      }
    }
    long long tc0 = a.prof ? clock64() : 0;
    uint32_t cnt[2][kLevelPlanes];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int b = 0; b < kLevelPlanes; ++b) cnt[i][b] = 0;
    uint32_t lev1[2] = {0, 0}, X[2] = {0, 0};
    int L = 1;
    for (;; ++L) {
      uint32_t P[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint32_t pv = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          if (L == 1) {
            pv |= F[i][j];  // from any predecessor (s >= 0) through a w = 1 arc
          } else {
            const int nz = lz[i] + slot_dz<NDIM>(j), ny = ly[i] + slot_dy<NDIM>(j);
            const uint32_t v = (nz < G::TZ && ny < G::TY) ? prv[nz * G::TY + ny] : 0u;
            pv |= F[i][j] & xshift(v, slot_dx<NDIM>(j));
          }
        }
        P[i] = pv;
        X[i] = xfill(pv, F[i][JX]);
      }
      // -e closure across rows (weight 0), Jacobi until stable
      for (;;) {
        cur[lane] = X[0];
        cur[lane + 32] = X[1];
        __syncwarp();
        uint32_t Y[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          uint32_t y = P[i];
#pragma unroll
          for (int j = D + 1; j < 2 * D; ++j) {
            const int nz = lz[i] + slot_dz<NDIM>(j), ny = ly[i] + slot_dy<NDIM>(j);
            const uint32_t v = (nz >= 0 && ny >= 0) ? cur[nz * G::TY + ny] : 0u;
            y |= F[i][j] & xshift(v, slot_dx<NDIM>(j));
          }
          Y[i] = xfill(y, F[i][JX]);
        }
        const bool ch = (Y[0] != X[0]) || (Y[1] != X[1]);
        X[0] = Y[0];
        X[1] = Y[1];
        __syncwarp();
        if (!__any_sync(0xffffffffu, ch)) break;
      }
      if (!__any_sync(0xffffffffu, (X[0] | X[1]) != 0)) break;  // Lev_L empty: done
      if (L == 1) {
        lev1[0] = X[0];
        lev1[1] = X[1];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {  // bit-sliced count += Lev_L
        uint32_t carry = X[i];
#pragma unroll
        for (int b = 0; b < kLevelPlanes; ++b) {
          const uint32_t t = cnt[i][b] & carry;
          cnt[i][b] ^= carry;
          carry = t;
        }
      }
      prv[lane] = X[0];
      prv[lane + 32] = X[1];
      __syncwarp();
      if (L == kMaxLevel) break;  // hand the rest to the worklist
    }
    long long tc1 = a.prof ? clock64() : 0;
    const bool capped = L == kMaxLevel;
    const int top = capped ? kMaxLevel : L - 1;  // highest non-empty level
    const int nplanes = 32 - __clz(top | 1);
    my_levels += (unsigned long long)L;
    my_max = top > (int)my_max ? (uint32_t)top : my_max;
    // write s row by row (lane = x)
    for (int r = 0; r < 64; ++r) {
      const int i = r >> 5, src = r & 31;
      uint32_t sv = 0;
#pragma unroll
      for (int b = 0; b < kLevelPlanes; ++b) {
        if (b < nplanes) {
          const uint32_t pl = __shfl_sync(0xffffffffu, i ? cnt[1][b] : cnt[0][b], src);
          sv |= ((pl >> lane) & 1u) << b;
        }
      }
      const int rz = r / G::TY, ry = r % G::TY;
      const Idx gz = z0 + rz, gy = y0 + ry, gx = x0 + lane;
      if (gz < d0 && gy < d1 && gx < d2) __stcg(&a.s[(gz * d1 + gy) * d2 + gx], sv);
    }
    long long tc2 = a.prof ? clock64() : 0;
    // border points with s > 0 feed out-of-tile points that assumed s = 0
    // (all lanes stay converged: the enqueues are warp-collective)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint32_t lv = rin[i] ? lev1[i] & vmask : 0u;
      my_raised += __popc(lv);
      if (capped) {  // unfinished: continue point-wise from the top level
        uint32_t c = rin[i] ? X[i] & vmask : 0u;
        while (__any_sync(0xffffffffu, c != 0)) {
          const int x = c ? __ffs(c) - 1 : 0;
          enqueue_warp<Idx>(a, ((z0 + lz[i]) * d1 + (y0 + ly[i])) * d2 + x0 + x, c != 0, 2);
          c &= c - 1;
        }
      }
      if (!__any_sync(0xffffffffu, lv != 0)) continue;
      // all neighbour flag words first (independent loads, one latency), then
      // the feeds and their enqueues
      uint32_t win[2 * D], wed[2 * D];
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        const int dz = slot_dz<NDIM>(j), dy = slot_dy<NDIM>(j), dx = slot_dx<NDIM>(j);
        const int tlz = lz[i] + dz, tly = ly[i] + dy;
        const bool row_in = tlz >= 0 && tlz < G::TZ && tly >= 0 && tly < G::TY;
        const Idx gz = z0 + tlz, gy = y0 + tly;
        const bool gin = gz >= 0 && gz < d0 && gy >= 0 && gy < d1;
        const uint32_t cand = !gin ? 0u : (row_in ? (lv & (dx > 0 ? 0x80000000u : (dx < 0 ? 1u : 0u))) : lv);
        const uint32_t* rowf = a.flags + ((size_t)(gin ? gz * d1 + gy : 0) * nseg) * SW + slot_opp<NDIM>(j);
        const uint32_t inseg = cand & (dx > 0 ? 0x7fffffffu : (dx < 0 ? 0xfffffffeu : 0xffffffffu));
        win[j] = inseg ? __ldg(rowf + (size_t)tx * SW) : 0u;
        wed[j] = 0;
        if (dx > 0 && (cand >> 31) && x0 + 32 < d2) wed[j] = __ldg(rowf + (size_t)(tx + 1) * SW);
        if (dx < 0 && (cand & 1u) && tx > 0) wed[j] = __ldg(rowf + (size_t)(tx - 1) * SW);
      }
      // feeds of all slots; each slot's candidates are consecutive points of
      // one row, so their dedup bits lie in <= 2 bitmap words: <= 2 atomics
      // per slot, all issued before any result is used, then one list
      // reservation for the whole warp
      uint32_t fresh[2 * D];
      Idx fbase[2 * D];
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        const int dz = slot_dz<NDIM>(j), dy = slot_dy<NDIM>(j), dx = slot_dx<NDIM>(j);
        const int tlz = lz[i] + dz, tly = ly[i] + dy;
        const bool row_in = tlz >= 0 && tlz < G::TZ && tly >= 0 && tly < G::TY;
        const Idx gz = z0 + tlz, gy = y0 + tly;
        const bool gin = gz >= 0 && gz < d0 && gy >= 0 && gy < d1;
        const uint32_t cand = !gin ? 0u : (row_in ? (lv & (dx > 0 ? 0x80000000u : (dx < 0 ? 1u : 0u))) : lv);
        const uint32_t inseg = cand & (dx > 0 ? 0x7fffffffu : (dx < 0 ? 0xfffffffeu : 0xffffffffu));
        uint32_t feed = inseg & xshift(win[j], dx);
        if (dx > 0 && (cand >> 31) && (wed[j] & 1u)) feed |= 0x80000000u;
        if (dx < 0 && (cand & 1u) && (wed[j] >> 31)) feed |= 1u;
        Idx base = gin ? (gz * d1 + gy) * d2 + x0 + dx : 0;  // point of feed bit 0
        if (base < 0) {  // only row 0, x0 = 0, dx = -1: feed bit 0 is clear there
          feed >>= 1;
          base += 1;
        }
        fbase[j] = base;
        fresh[j] = feed;
        if (feed) {
          const uint32_t sh = (uint32_t)base & 31u;
          uint32_t* bw = a.bitmap + ((UIdx)base >> 5);
          const uint32_t m0 = feed << sh, m1 = sh ? feed >> (32u - sh) : 0u;
          const uint32_t o0 = m0 ? atomicOr(bw, m0) : 0u;
          const uint32_t o1 = m1 ? atomicOr(bw + 1, m1) : 0u;
          fresh[j] = ((~o0 & m0) >> sh) | (sh ? ((~o1 & m1) << (32u - sh)) : 0u);
        }
      }
      uint32_t c = 0;
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) c += __popc(fresh[j]);
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
      if (wtot) {
        unsigned long long pos = 0;
        if (lane == 31) pos = atomicAdd(&a.ctr->list_count[2], (unsigned long long)wtot);
        pos = __shfl_sync(0xffffffffu, pos, 31) + (incl - c);
        UIdx* Lst = static_cast<UIdx*>(a.plist);  // pass 2 list: (2 & 1) * cap = 0
#pragma unroll
        for (int j = 0; j < 2 * D; ++j)
          for (uint32_t m = fresh[j]; m; m &= m - 1) Lst[pos++] = (UIdx)(fbase[j] + (__ffs(m) - 1));
      }
    }
    if (a.prof && lane == 0) {
      const long long tc3 = clock64();
      atomicAdd(&a.ctr->dense_cycles[1], (unsigned long long)(tc1 - tc0));
      atomicAdd(&a.ctr->dense_cycles[2], (unsigned long long)(tc2 - tc1));
      atomicAdd(&a.ctr->dense_cycles[3], (unsigned long long)(tc3 - tc2));
    }
    if (lane == 0) tile = atomicAdd(&a.ctr->tile_ticket, 1u);
    tile = __shfl_sync(0xffffffffu, tile, 0);
  }
  if (tid == 0 && blockIdx.x == 0 && !a.skip_dense && !a.engine) a.ctr->pass_items[1] = (uint32_t)a.ntiles;
  grid.sync();
  const uint64_t t_dense = (a.prof && tid == 0 && blockIdx.x == 0) ? gtimer() : 0;
  if (a.prof && tid == 0 && blockIdx.x == 0) a.ctr->pass_ns[1] = t_dense - t_start;

  // ---- passes >= 2: sparse, point-level ------------------------------------
  // Whole grid while the list is long; once it is short, block 0 finishes
  // alone with block barriers (no grid-wide barrier per pass).
  // engine 1 (the paper's schedule): pass 1 visits every point
  // (s = 0 everywhere), later passes the points whose inputs rose.
  int q = (a.engine && !a.skip_dense) ? 1 : 2;
  bool small = false;
  for (; q <= a.max_passes; ++q) {
    const unsigned long long n =
        q == 1 ? (unsigned long long)a.cap : *(volatile unsigned long long*)&a.ctr->list_count[q % 3];
    if (n == 0) break;
    if (!small && n <= kSmallList) {
      small = true;
      if (blockIdx.x != 0) break;
    }
    const UIdx* Lq = static_cast<const UIdx*>(a.plist) + (size_t)(q & 1) * a.cap;
    const unsigned long long wbase = small ? (unsigned long long)warp * 32 : (unsigned long long)gwarp * 32;
    const unsigned long long wstep = small ? (unsigned long long)kSweepThreads : (unsigned long long)nwarps * 32;
    for (unsigned long long ib = wbase; ib < n; ib += wstep) {
      const unsigned long long i = ib + lane;
      // Each lane evaluates its list point, then chases the successors of
      // every point it raises depth-first (Gauss-Seidel within the pass);
      // what does not fit the small stack goes to the next pass's list.
      Idx cur = 0;
      bool have = i < n;
      if (have) {
        if (q == 1) {
          cur = (Idx)i;
        } else {
          cur = (Idx)__ldcg(&Lq[i]);
          const uint32_t bit = 1u << ((uint32_t)cur & 31u);
          atomicAnd(&a.bitmap[(size_t)(q & 1) * a.bmw + ((UIdx)cur >> 5)], ~bit);
        }
      }
      Idx stk[kChase];
      int sp = 0;
      // long lists: plain passes (no redundant chases); chasing only in the
      // early sparse passes (late passes of long-chain fields chase into
      // each other's work)
      int budget = (n <= kChaseMaxList && q <= LOPC_CHASE_MAX_PASS) ? kChaseBudget : 0;
      while (__any_sync(0xffffffffu, have)) {
        Idx z = 0, y = 0, x = 0;
        uint32_t best = 0;
        bool raised = false;
        if (have) {
          z = cur / plane;
          const Idx r2 = cur - z * plane;
          y = r2 / d2;
          x = r2 - y * d2;
          uint32_t fl = point_flags<NDIM>(a.flags + ((size_t)(z * d1 + y) * nseg + (size_t)(x >> 5)) * SW,
                                          (uint32_t)x & 31u);
          while (fl) {
            const int j = __ffs(fl) - 1;
            fl &= fl - 1;
            const int e = (j < D ? j : j - D) + 1;
            const Idx off = (NDIM == 3 ? (Idx)(e >> 2) * plane : (Idx)0) + (Idx)((e >> 1) & 1) * d2 + (Idx)(e & 1);
            const uint32_t v = j < D ? __ldcg(&a.s[cur + off]) + 1u : __ldcg(&a.s[cur - off]);
            best = v > best ? v : best;
          }
          if (best > __ldcg(&a.s[cur])) {
            const uint32_t old = atomicMax(&a.s[cur], best);
            raised = old < best;
          }
        }
        if (raised) {
          ++my_raised;
          my_max = best > my_max ? best : my_max;
        }
        uint32_t over = 0;
        if (__any_sync(0xffffffffu, raised)) {
          const uint32_t cand = succ_cand<NDIM, Idx>(a, raised, z, y, x);
          for (uint32_t m = cand; m; m &= m - 1) {
            const int j = __ffs(m) - 1;
            if (sp < kChase && budget > 0) {
              stk[sp++] = cur + slot_goff<NDIM, Idx>(j, plane, d2);
              --budget;
            } else {
              over |= 1u << j;
            }
          }
          if (__any_sync(0xffffffffu, over != 0)) enqueue_mask<NDIM, Idx>(a, cur, over, q + 1);
        }
        have = sp > 0;
        if (have) cur = stk[--sp];
      }
    }
    if (tid == 0 && blockIdx.x == 0) {
      a.ctr->list_count[(q + 2) % 3] = 0;
      if (q < kPassHist) a.ctr->pass_items[q] = (uint32_t)n;
      a.ctr->worklist_points += n;
      if (a.prof && q < kPassHist) a.ctr->pass_ns[q] = gtimer() - t_start;
    }
    if (small) {
      __threadfence();  // the next pass reads the lists and s through L2
      __syncthreads();
    } else {
      grid.sync();
    }
  }
  if (tid == 0 && blockIdx.x == 0) {
    a.ctr->passes = (unsigned long long)(q - 1);
    if (a.prof) {
      a.ctr->phase[14] += t_dense - t_start;
      a.ctr->phase[15] += gtimer() - t_dense;
    }
  }
  my_raised = __reduce_add_sync(0xffffffffu, my_raised);
  my_max = __reduce_max_sync(0xffffffffu, my_max);
  const unsigned lv32 = __reduce_add_sync(0xffffffffu, (unsigned)my_levels);
  if (lane == 0 && lv32) atomicAdd(&a.ctr->inner_iters, (unsigned long long)lv32 / 32ull);
  if (lane == 0 && my_raised) atomicAdd(&a.ctr->raised, (unsigned long long)my_raised);
  if (lane == 0 && my_max) atomicMax(&a.ctr->max_s, my_max);
}

// Slab mode: ghost points (box points owned by a neighbour
// rank) have no incoming arcs here; their subbins arrive from the owner after
// each repair round.  A ghost whose value rose is written and its successors
// (points with an arc from it) are enqueued for the next sparse pass (pass 2
// of the next k_sweep launch, skip_dense).  ctr->raised counts the ghosts that
// changed (the round's termination term, summed over ranks).
template <int NDIM, typename Idx>
__global__ void __launch_bounds__(256) k_ghost_inject(RepairArgs a, const uint32_t* __restrict__ recv, int64_t g0,
                                                      int64_t count) {
  const int lane = threadIdx.x & 31;
  const Idx d1 = (Idx)a.d1, d2 = (Idx)a.d2, plane = d1 * d2;
  unsigned changed = 0;
  const int64_t wstep = (int64_t)gridDim.x * blockDim.x;
  for (int64_t ib = (int64_t)(blockIdx.x * blockDim.x + (threadIdx.x & ~31)); ib < count; ib += wstep) {
    const int64_t i = ib + lane;
    bool up = false;
    Idx p = 0, z = 0, y = 0, x = 0;
    if (i < count) {
      p = (Idx)(g0 + i);
      const uint32_t v = __ldg(&recv[i]);
      if (v > a.s[p]) {
        a.s[p] = v;
        up = true;
        ++changed;
      }
      z = p / plane;
      const Idx r2 = p - z * plane;
      y = r2 / d2;
      x = r2 - y * d2;
    }
    if (!__any_sync(0xffffffffu, up)) continue;
    enqueue_mask<NDIM, Idx>(a, p, succ_cand<NDIM, Idx>(a, up, z, y, x), 2);
  }
  changed = __reduce_add_sync(0xffffffffu, changed);
  if (lane == 0 && changed) atomicAdd(&a.ctr->ghost_changed, (unsigned long long)changed);
}

// Debug/parity: bit-plane flags -> one u16 per point.
template <int NDIM>
__global__ void k_unpack_flags(const uint32_t* flags, uint16_t* out, int64_t d0, int64_t d1, int64_t d2,
                               int64_t nseg) {
  const int64_t n = d0 * d1 * d2;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = p / (d1 * d2), r = p - z * d1 * d2, y = r / d2, x = r - y * d2;
    const uint32_t* seg = flags + ((z * d1 + y) * nseg + (x >> 5)) * Geo<NDIM>::SW;
    uint32_t f = 0;
    for (int j = 0; j < 2 * Geo<NDIM>::D; ++j) f |= ((seg[j] >> (x & 31)) & 1u) << j;
    out[p] = (uint16_t)f;
  }
}

}  // namespace lopc
