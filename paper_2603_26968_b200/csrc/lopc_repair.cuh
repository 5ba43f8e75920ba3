// lopc_repair.cuh — quantize + flags + local-order repair.
//
// PAPER.md Alg. 1 computes bins, zero subbins and per-point flags;
// Alg. 2 raises subbins until no violation remains.  The result
// is the unique least fixpoint of s(p) = max(0, max_{n->p} s(n) + w) over the
// same-bin arcs n -> p (n precedes p in the SoS order, w = [idx n > idx p]);
// any monotone relaxation schedule reaches it (reading G14).  The schedule
// here is B200-shaped, not the paper's point worklist:
//
//   k_quant_repair  one CTA per 3D tile (8x8x32, 2D: 32x64) with a one-cell
//                   halo in shared memory: exact bins of tile+halo, flags of
//                   the tile (u16 in 3D / u8 in 2D), relaxation inside the
//                   tile to local convergence with the halo held at 0 (a lower
//                   bound), write flags + s.  Tiles whose boundary subbins are
//                   > 0 and feed a neighbour tile enlist that tile.
//   k_sweep         one persistent cooperative kernel: pass q processes the
//                   active-tile list q (halo s re-read from global), relaxes
//                   each tile to local convergence, writes raised subbins and
//                   enlists the neighbour tiles its raised boundary points
//                   feed; grid-wide barrier; stop when a list is empty.  No
//                   host round trip per sweep.
//
// Every value ever written is <= the least fixpoint (lower bounds relaxed by
// monotone max), and on exit every tile was last processed with its current
// halo and is locally stable, so the Bellman equation holds everywhere: the
// result is the least fixpoint, independent of scheduling.
#pragma once
#include <cooperative_groups.h>

#include "lopc_device.cuh"

namespace lopc {

template <int NDIM>
struct Geo;
template <>
struct Geo<3> {
  static constexpr int TZ = 8, TY = 8, TX = 32;
  static constexpr int HZ = TZ + 2, HY = TY + 2, HX = TX + 2;
  static constexpr int D = 7;  // +e offsets (G2)
  using Flag = uint16_t;
};
template <>
struct Geo<2> {
  static constexpr int TZ = 1, TY = 32, TX = 64;
  static constexpr int HZ = 1, HY = TY + 2, HX = TX + 2;
  static constexpr int D = 3;
  using Flag = uint8_t;
};

constexpr int kRepairThreads = 512;

// Star slot j (G2): j < D is +e_j, j >= D is -e_{j-D}.  3D order (dz,dy,dx):
// (0,0,1) (0,1,0) (0,1,1) (1,0,0) (1,0,1) (1,1,0) (1,1,1); 2D (dy,dx):
// (0,1) (1,0) (1,1).
template <int NDIM>
__host__ __device__ constexpr int slot_dz(int j) {
  return NDIM == 2 ? 0 : (j % 7 >= 3 ? (j < 7 ? 1 : -1) : 0);
}
template <int NDIM>
__host__ __device__ constexpr int slot_dy(int j) {
  return NDIM == 2 ? ((j % 3) >= 1 ? (j < 3 ? 1 : -1) : 0)
                   : (((j % 7) == 1 || (j % 7) == 2 || (j % 7) == 5 || (j % 7) == 6) ? (j < 7 ? 1 : -1) : 0);
}
template <int NDIM>
__host__ __device__ constexpr int slot_dx(int j) {
  return NDIM == 2 ? ((j % 3) != 1 ? (j < 3 ? 1 : -1) : 0)
                   : (((j % 7) == 0 || (j % 7) == 2 || (j % 7) == 4 || (j % 7) == 6) ? (j < 7 ? 1 : -1) : 0);
}
template <int NDIM>
__host__ __device__ constexpr int slot_hoff(int j) {
  using G = Geo<NDIM>;
  return slot_dz<NDIM>(j) * G::HY * G::HX + slot_dy<NDIM>(j) * G::HX + slot_dx<NDIM>(j);
}

struct Counters {
  uint32_t list_count[3];
  uint32_t ticket;
  uint32_t err;  // bit 0 bound self-check, 1 corrupt, 2 nospace, 3 subbin overflow, 4 pass cap
  uint32_t max_s;
  uint32_t pad[2];
  unsigned long long escapes;
  unsigned long long total_bytes;
  unsigned long long passes;
  unsigned long long tiles_processed;
  unsigned long long bin_bytes;
  unsigned long long sub_bytes;
  unsigned long long inner_iters;
  unsigned long long pad2;
};

enum : uint32_t {
  kErrBound = 1u,
  kErrCorrupt = 2u,
  kErrNoSpace = 4u,
  kErrOverflow = 8u,
  kErrPassCap = 16u,
  kErrVersion = 32u,
};

struct RepairArgs {
  const void* x;
  void* flags;
  uint32_t* s;
  uint32_t* stamp;   // per tile: last pass it was enlisted for
  uint32_t* lists;   // 3 x ntiles
  Counters* ctr;
  double eps, inv;
  int64_t d0, d1, d2;  // z, y, x extents (2D: d0 = 1)
  int ntz, nty, ntx;
  int64_t ntiles;
  int max_inner;
  int max_passes;
};

__device__ __forceinline__ void enlist(const RepairArgs& a, uint32_t tile, uint32_t q) {
  uint32_t old = atomicMax(&a.stamp[tile], q);
  if (old < q) {
    uint32_t slot = atomicAdd(&a.ctr->list_count[q % 3], 1u);
    a.lists[(size_t)(q % 3) * a.ntiles + slot] = tile;
  }
}

// Enlist the neighbour tiles recorded as bits (dz+1)*9 + (dy+1)*3 + (dx+1).
__device__ __forceinline__ void enlist_dirs(const RepairArgs& a, uint32_t dirs, int tz, int ty, int tx, uint32_t q) {
  int t = threadIdx.x;
  if (t < 27 && ((dirs >> t) & 1u)) {
    int nz = tz + t / 9 - 1, ny = ty + (t / 3) % 3 - 1, nx = tx + t % 3 - 1;
    if (nz >= 0 && ny >= 0 && nx >= 0 && nz < a.ntz && ny < a.nty && nx < a.ntx)
      enlist(a, (uint32_t)(((int64_t)nz * a.nty + ny) * a.ntx + nx), q);
  }
}

template <int NDIM>
__device__ __forceinline__ int dir_of_halo(int hz, int hy, int hx) {
  using G = Geo<NDIM>;
  int dz = NDIM == 2 ? 0 : (hz == 0 ? -1 : (hz == G::HZ - 1 ? 1 : 0));
  int dy = hy == 0 ? -1 : (hy == G::HY - 1 ? 1 : 0);
  int dx = hx == 0 ? -1 : (hx == G::HX - 1 ? 1 : 0);
  return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
}

// Relax the tile's points to local convergence in shared memory.  Each thread
// owns PPT points (flags in registers).  Returns the number of inner
// iterations; *capped set if the cap was hit while still changing.
template <int NDIM, int PPT>
__device__ __forceinline__ int relax_tile(uint32_t* ss, const uint32_t (&f)[PPT], const int (&h)[PPT], int max_inner,
                                          bool* capped) {
  constexpr int D = Geo<NDIM>::D;
  int it = 0;
  for (;;) {
    int changed = 0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      uint32_t m = f[k];
      if (m == 0) continue;
      uint32_t cur = ss[h[k]];
      uint32_t best = cur;
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        if (m & (1u << j)) {
          uint32_t v = ss[h[k] + slot_hoff<NDIM>(j)] + (j < D ? 1u : 0u);
          best = v > best ? v : best;
        }
      }
      if (best > cur) {
        ss[h[k]] = best;
        changed = 1;
      }
    }
    ++it;
    int any = __syncthreads_or(changed);
    if (!any) {
      *capped = false;
      return it;
    }
    if (it >= max_inner) {
      *capped = true;
      return it;
    }
  }
}

template <typename T, int NDIM>
constexpr size_t quant_repair_smem() {
  using G = Geo<NDIM>;
  return (size_t)G::HZ * G::HY * G::HX * (2 * sizeof(typename VT<T>::I) + 4) + 16;
}

// ---------------------------------------------------------------------------
// k_quant_repair: a1 + a2 + the first (tile-local) relaxation.
// ---------------------------------------------------------------------------
template <typename T, int NDIM>
__global__ void __launch_bounds__(kRepairThreads, 2) k_quant_repair(RepairArgs a) {
  using G = Geo<NDIM>;
  using I = typename VT<T>::I;
  using U = typename VT<T>::U;
  using Flag = typename G::Flag;
  constexpr int HP = G::HZ * G::HY * G::HX;
  constexpr int TP = G::TZ * G::TY * G::TX;
  constexpr int PPT = TP / kRepairThreads;
  constexpr int D = G::D;
  constexpr int ZH = NDIM == 3 ? 1 : 0;  // halo depth in z

  extern __shared__ __align__(16) uint8_t qr_smem[];
  I* sbin = reinterpret_cast<I*>(qr_smem);
  I* skey = sbin + HP;
  uint32_t* ss = reinterpret_cast<uint32_t*>(skey + HP);
  uint32_t& sdirs = ss[HP];

  const int64_t tile = blockIdx.x;
  const int tx = (int)(tile % a.ntx), ty = (int)((tile / a.ntx) % a.nty), tz = (int)(tile / ((int64_t)a.ntx * a.nty));
  const int64_t z0 = (int64_t)tz * G::TZ, y0 = (int64_t)ty * G::TY, x0 = (int64_t)tx * G::TX;
  const T* X = static_cast<const T*>(a.x);
  const I kNone = (I)VT<T>::kSentinel;  // escaped or outside the grid

  if (threadIdx.x == 0) sdirs = 0;
  for (int hi = threadIdx.x; hi < HP; hi += kRepairThreads) {
    int hx = hi % G::HX, hy = (hi / G::HX) % G::HY, hz = hi / (G::HX * G::HY);
    int64_t gz = z0 + hz - ZH, gy = y0 + hy - 1, gx = x0 + hx - 1;
    I b = kNone, k = 0;
    if (gz >= 0 && gy >= 0 && gx >= 0 && gz < a.d0 && gy < a.d1 && gx < a.d2) {
      T v = X[(gz * a.d1 + gy) * a.d2 + gx];
      I q;
      if (quantize<T>(v, a.eps, a.inv, q)) {
        b = q;
        k = (I)key_of((U)as_bits(v));
      }
    }
    sbin[hi] = b;
    skey[hi] = k;
    ss[hi] = 0;
  }
  __syncthreads();

  uint32_t f[PPT];
  int h[PPT];
  bool inb[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    int lp = threadIdx.x + k * kRepairThreads;
    int lx = lp % G::TX, ly = (lp / G::TX) % G::TY, lz = lp / (G::TX * G::TY);
    h[k] = ((lz + ZH) * G::HY + (ly + 1)) * G::HX + (lx + 1);
    inb[k] = (z0 + lz < a.d0) && (y0 + ly < a.d1) && (x0 + lx < a.d2);
    uint32_t m = 0;
    I bp = sbin[h[k]];
    if (bp != kNone) {
      I kp = skey[h[k]];
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        int hn = h[k] + slot_hoff<NDIM>(j);
        // arc n -> p: same bin and n precedes p in SoS order.  A +e neighbour
        // has the larger index, so it precedes p only with a smaller key; a -e
        // neighbour precedes p on ties too (G4).
        if (sbin[hn] == bp && (j < D ? skey[hn] < kp : skey[hn] <= kp)) m |= 1u << j;
      }
    }
    f[k] = m;
  }

  bool capped = false;
  int iters = relax_tile<NDIM, PPT>(ss, f, h, a.max_inner, &capped);

  // write flags and s; find boundary points with s > 0 that feed a neighbour
  Flag* F = static_cast<Flag*>(a.flags);
  uint32_t my_dirs = 0;
  uint32_t my_max = 0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    if (!inb[k]) continue;
    int lp = threadIdx.x + k * kRepairThreads;
    int lx = lp % G::TX, ly = (lp / G::TX) % G::TY, lz = lp / (G::TX * G::TY);
    int64_t gi = ((z0 + lz) * a.d1 + (y0 + ly)) * a.d2 + (x0 + lx);
    uint32_t sv = ss[h[k]];
    F[gi] = (Flag)f[k];
    a.s[gi] = sv;
    my_max = sv > my_max ? sv : my_max;
    bool border = lx == 0 || lx == G::TX - 1 || ly == 0 || ly == G::TY - 1 ||
                  (NDIM == 3 && (lz == 0 || lz == G::TZ - 1));
    if (sv > 0 && border) {
      I bp = sbin[h[k]], kp = skey[h[k]];
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) {
        int hn = h[k] + slot_hoff<NDIM>(j);
        int hx = hn % G::HX, hy = (hn / G::HX) % G::HY, hz = hn / (G::HX * G::HY);
        bool outside = hx == 0 || hx == G::HX - 1 || hy == 0 || hy == G::HY - 1 ||
                       (NDIM == 3 && (hz == 0 || hz == G::HZ - 1));
        // arc p -> n (p precedes n): the neighbour tile assumed s(p) = 0
        if (outside && sbin[hn] == bp && (j < D ? kp <= skey[hn] : kp < skey[hn]))
          my_dirs |= 1u << dir_of_halo<NDIM>(hz, hy, hx);
      }
    }
  }
  if (my_dirs) atomicOr(&sdirs, my_dirs);
  // warp-reduce max subbin for stats
  for (int o = 16; o > 0; o >>= 1) {
    uint32_t v = __shfl_xor_sync(0xffffffffu, my_max, o);
    my_max = v > my_max ? v : my_max;
  }
  if ((threadIdx.x & 31) == 0 && my_max) atomicMax(&a.ctr->max_s, my_max);
  __syncthreads();
  uint32_t dirs = sdirs;
  if (capped) dirs |= 1u << 13;  // self
  enlist_dirs(a, dirs, tz, ty, tx, 1u);
  if (threadIdx.x == 0) atomicAdd(&a.ctr->inner_iters, (unsigned long long)iters);
}

// ---------------------------------------------------------------------------
// k_sweep: persistent passes over active tiles (cooperative launch).
// ---------------------------------------------------------------------------
template <int NDIM>
__global__ void __launch_bounds__(kRepairThreads, 2) k_sweep(RepairArgs a) {
  namespace cg = cooperative_groups;
  using G = Geo<NDIM>;
  using Flag = typename G::Flag;
  constexpr int HP = G::HZ * G::HY * G::HX;
  constexpr int TP = G::TZ * G::TY * G::TX;
  constexpr int PPT = TP / kRepairThreads;
  constexpr int D = G::D;
  constexpr int ZH = NDIM == 3 ? 1 : 0;

  __shared__ uint32_t ss[HP];
  __shared__ Flag sf[HP];
  __shared__ uint8_t sraised[TP];
  __shared__ uint32_t sdirs;
  __shared__ uint32_t sn;

  cg::grid_group grid = cg::this_grid();
  const Flag* F = static_cast<const Flag*>(a.flags);

  for (int q = 1; q <= a.max_passes; ++q) {
    if (threadIdx.x == 0) sn = *(volatile uint32_t*)&a.ctr->list_count[q % 3];
    __syncthreads();
    const uint32_t n = sn;
    if (n == 0) break;
    const uint32_t* L = a.lists + (size_t)(q % 3) * a.ntiles;
    unsigned long long my_iters = 0;
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
      const uint32_t tile = __ldcg(&L[i]);
      const int tx = (int)(tile % a.ntx), ty = (int)((tile / a.ntx) % a.nty),
                tz = (int)(tile / ((int64_t)a.ntx * a.nty));
      const int64_t z0 = (int64_t)tz * G::TZ, y0 = (int64_t)ty * G::TY, x0 = (int64_t)tx * G::TX;
      if (threadIdx.x == 0) sdirs = 0;
      for (int hi = threadIdx.x; hi < HP; hi += kRepairThreads) {
        int hx = hi % G::HX, hy = (hi / G::HX) % G::HY, hz = hi / (G::HX * G::HY);
        int64_t gz = z0 + hz - ZH, gy = y0 + hy - 1, gx = x0 + hx - 1;
        uint32_t sv = 0;
        Flag fv = 0;
        if (gz >= 0 && gy >= 0 && gx >= 0 && gz < a.d0 && gy < a.d1 && gx < a.d2) {
          int64_t gi = (gz * a.d1 + gy) * a.d2 + gx;
          sv = __ldcg(&a.s[gi]);
          fv = F[gi];
        }
        ss[hi] = sv;
        sf[hi] = fv;
      }
      __syncthreads();
      uint32_t f[PPT], s_old[PPT];
      int h[PPT];
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        int lp = threadIdx.x + k * kRepairThreads;
        int lx = lp % G::TX, ly = (lp / G::TX) % G::TY, lz = lp / (G::TX * G::TY);
        h[k] = ((lz + ZH) * G::HY + (ly + 1)) * G::HX + (lx + 1);
        f[k] = sf[h[k]];
        s_old[k] = ss[h[k]];
      }
      bool capped = false;
      my_iters += relax_tile<NDIM, PPT>(ss, f, h, a.max_inner, &capped);
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        int lp = threadIdx.x + k * kRepairThreads;
        uint32_t sv = ss[h[k]];
        bool raised = sv != s_old[k];
        sraised[lp] = raised;
        if (raised) {
          int lx = lp % G::TX, ly = (lp / G::TX) % G::TY, lz = lp / (G::TX * G::TY);
          int64_t gi = ((z0 + lz) * a.d1 + (y0 + ly)) * a.d2 + (x0 + lx);
          __stcg(&a.s[gi], sv);
        }
      }
      __syncthreads();
      // a halo point n fed (through its flags) by a raised tile point must
      // be re-relaxed: enlist its tile for the next pass.
      uint32_t my_dirs = 0;
      for (int hi = threadIdx.x; hi < HP; hi += kRepairThreads) {
        int hx = hi % G::HX, hy = (hi / G::HX) % G::HY, hz = hi / (G::HX * G::HY);
        bool outside = hx == 0 || hx == G::HX - 1 || hy == 0 || hy == G::HY - 1 ||
                       (NDIM == 3 && (hz == 0 || hz == G::HZ - 1));
        uint32_t m = sf[hi];
        if (!outside || m == 0) continue;
        bool hit = false;
#pragma unroll
        for (int j = 0; j < 2 * D; ++j) {
          if (m & (1u << j)) {
            int hp = hi + slot_hoff<NDIM>(j);
            int px = hp % G::HX, py = (hp / G::HX) % G::HY, pz = hp / (G::HX * G::HY);
            bool inside = px >= 1 && px <= G::TX && py >= 1 && py <= G::TY &&
                          (NDIM == 2 || (pz >= 1 && pz <= G::TZ));
            if (inside && sraised[((pz - ZH) * G::TY + (py - 1)) * G::TX + (px - 1)]) hit = true;
          }
        }
        if (hit) my_dirs |= 1u << dir_of_halo<NDIM>(hz, hy, hx);
      }
      if (my_dirs) atomicOr(&sdirs, my_dirs);
      __syncthreads();
      uint32_t dirs = sdirs;
      if (capped) dirs |= 1u << 13;
      enlist_dirs(a, dirs, tz, ty, tx, (uint32_t)q + 1u);
      __syncthreads();  // smem reuse by the next tile
    }
    if (threadIdx.x == 0) {
      if (my_iters) atomicAdd(&a.ctr->inner_iters, my_iters);
      if (blockIdx.x == 0) {
        a.ctr->list_count[(q + 2) % 3] = 0;
        a.ctr->passes = (unsigned long long)q;
        a.ctr->tiles_processed += n;
      }
    }
    grid.sync();
  }
}

}  // namespace lopc
