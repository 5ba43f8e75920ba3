// lopc_tiles.cuh — the repair (Alg. 2) as exact
// tile fixpoints re-run over alternating, half-shifted tilings.
//
// The least fixpoint s(p) = max(0, max_{n->p} s(n) + w) (O9; w = [idx n >
// idx p]) is computed tile by tile: a tile computes the exact fixpoint
// of its own points with the values outside it held fixed (its one-cell halo)
// and its current values as lower bounds (seeds).  Any such step only raises
// values towards the least fixpoint (every value written is a lower bound of
// it), so any schedule that re-runs every tile whose inputs changed reaches it
// (reading G14).  The schedule is B200-shaped, not the paper's point worklist
// (P:218-220):
//
//   pass 1        every tile of tiling 0 (8x8x32 in 3D, 64x32 in 2D: one
//                 warp each), halo and seeds 0 (the r1 dense pass).
//   pass q >= 2   the ACTIVE tiles of tiling (q-1) mod 2.  Tiling 1 is
//                 tiling 0 shifted by half a tile in z and y (x stays
//                 32-aligned so a tile row is one flag / plane segment): a
//                 chain that crosses a tile border in one tiling runs inside
//                 a tile of the other (overlapping-domain / alternating
//                 Schwarz relaxation).  A tile of pass q+1 is active iff one
//                 of its points has a star neighbour that changed in pass q;
//                 pass q builds that list (per-tile mark words + an
//                 append-only list) and processes its own list in reverse
//                 build order, so consecutive passes sweep in opposite
//                 directions (values written earlier in the pass are read
//                 live: Gauss-Seidel across the tiles of one pass).
//   stop          when a pass changes nothing.  Then every point was
//                 evaluated after the last change of each of its neighbours,
//                 so every Bellman equation holds: the least fixpoint.
//
// Inside a tile the fixpoint is computed bit-parallel on level sets
// Lev_L = {p : s(p) >= L} (one u32 per 32-point row, one row per lane):
//   Lev_L = mu X. Seed_L | OR_{+e j} F_j & Lev_{L-1}(p + e_j)
//                        | OR_{-e j} F_j & X(p - e_j),
// where rows outside the tile are the halo's fixed level sets [s_h >= L].
// The -e slots (w = 0) close within a level: a carry-lookahead fill along x
// (the -x slot) and a Jacobi loop across rows; the +e slots (w = 1) feed the
// next level.  s is the number of non-empty levels, kept bit-sliced.
//
// Subbins live in HBM as bit planes with the flags' segmentation: for every
// 32-point x-segment of a row, 8 u32 words (word b = bit b of the 32 subbins).
// Tiles read and write them without transposes; 8 planes hold s <= 255 (a
// tile reaching level kMaxPlaneLevel raises kErrPlanes and the host re-runs
// the repair on the u32 engine of lopc_repair.cuh).
#pragma once
#include <cooperative_groups.h>

#include "lopc_repair.cuh"

namespace lopc {

constexpr int kSP = 8;                 // subbin planes per segment
constexpr int kMaxPlaneLevel = 255;    // Lev_255 non-empty -> kErrPlanes
constexpr int kTileThreads = 256;
constexpr int kTileWarps = kTileThreads / 32;
#ifndef LOPC_TILE_CTAS
#define LOPC_TILE_CTAS 3
#endif

template <int NDIM>
struct TBox {
  using G = Geo<NDIM>;
  static constexpr int BY = G::TY + 2;                 // box rows along y (halo included)
  static constexpr int NB = (G::TZ + 2 * G::ZH) * BY;  // box rows
  static constexpr int NH = NDIM == 3 ? 34 : 2;        // halo rows the star reaches
  static constexpr int SZ = NDIM == 3 ? G::TZ / 2 : 0; // tiling 1 shift (z, y)
  static constexpr int SY = G::TY / 2;
  __host__ __device__ static constexpr int idx(int bz, int by) { return (bz + G::ZH) * BY + (by + 1); }
  // halo row h -> box coordinates (bz, by): the rows a star offset of a tile
  // row reaches: z0-1 plane (y0-1 .. y0+TY-1), z0+TZ plane (y0 .. y0+TY),
  // y0-1 and y0+TY rows of every tile plane
  __host__ __device__ static void halo(int h, int& bz, int& by) {
    if (NDIM == 2) {
      bz = 0;
      by = h == 0 ? -1 : G::TY;
      return;
    }
    if (h < 9) {
      bz = -1;
      by = h - 1;
    } else if (h < 18) {
      bz = G::TZ;
      by = h - 9;
    } else if (h < 26) {
      bz = h - 18;
      by = -1;
    } else {
      bz = h - 26;
      by = G::TY;
    }
  }
};

struct TileArgs {
  const uint32_t* flags;  // bit-plane flags (k_quant_flags), SW words per segment
  uint32_t* sp;           // subbin planes, kSP words per segment
  uint32_t* act[2];       // per-tile mark words of tiling 0 / 1
  uint32_t* list[2];      // active-tile lists of tiling 0 / 1
  Counters* ctr;
  int64_t d0, d1, d2, nseg;
  uint32_t nt[2][3];      // tiles per axis (z, y, x) of tiling 0 / 1
  uint32_t ntiles[2];
  int max_passes;
  int prof;
};

struct TileWarpSmem {
  uint32_t lv[2][TBox<3>::NB];  // level words of the box rows, [L & 1]
  uint8_t ed[2][TBox<3>::NB];   // edge level bits: bit 0 = x0-1, bit 1 = x0+32
  uint32_t hp[TBox<3>::NH][kSP];
  uint8_t he[TBox<3>::NH][2];   // halo rows' edge subbins (x0-1, x0+32)
};

// s >= L on bit-sliced planes (L uniform across the warp)
__device__ __forceinline__ uint32_t planes_ge(const uint32_t (&p)[kSP], uint32_t L) {
  uint32_t ge = 0, eq = 0xffffffffu;
#pragma unroll
  for (int b = kSP - 1; b >= 0; --b) {
    if ((L >> b) & 1u)
      eq &= p[b];
    else
      ge |= eq & p[b];
  }
  return ge | eq;
}

// One row's subbin planes (x-aligned segment tx) and the subbins of its x
// halo points x0-1, x0+32 (bits 31 / 0 of the neighbouring segments).
// L2 loads: other tiles write planes during the pass.
__device__ __forceinline__ void load_sp_row(const TileArgs& a, int64_t gz, int64_t gy, int64_t tx, uint32_t (&p)[kSP],
                                            uint32_t& eL, uint32_t& eR) {
#pragma unroll
  for (int b = 0; b < kSP; ++b) p[b] = 0;
  eL = eR = 0;
  if (gz < 0 || gz >= a.d0 || gy < 0 || gy >= a.d1) return;
  const uint4* r4 = reinterpret_cast<const uint4*>(a.sp + ((size_t)(gz * a.d1 + gy) * (size_t)a.nseg + (size_t)tx) * kSP);
  const uint4 c0 = __ldcg(r4), c1 = __ldcg(r4 + 1);
  p[0] = c0.x, p[1] = c0.y, p[2] = c0.z, p[3] = c0.w, p[4] = c1.x, p[5] = c1.y, p[6] = c1.z, p[7] = c1.w;
  if (tx > 0) {
    const uint4 l0 = __ldcg(r4 - 2), l1 = __ldcg(r4 - 1);
    eL = (l0.x >> 31) | ((l0.y >> 31) << 1) | ((l0.z >> 31) << 2) | ((l0.w >> 31) << 3) | ((l1.x >> 31) << 4) |
         ((l1.y >> 31) << 5) | ((l1.z >> 31) << 6) | ((l1.w >> 31) << 7);
  }
  if (tx + 1 < a.nseg) {
    const uint4 q0 = __ldcg(r4 + 2), q1 = __ldcg(r4 + 3);
    eR = (q0.x & 1u) | ((q0.y & 1u) << 1) | ((q0.z & 1u) << 2) | ((q0.w & 1u) << 3) | ((q1.x & 1u) << 4) |
         ((q1.y & 1u) << 5) | ((q1.z & 1u) << 6) | ((q1.w & 1u) << 7);
  }
}

// Exact fixpoint of one tile (one warp).  SEEDED: current subbins are lower
// bounds and the halo holds the neighbours' current subbins; otherwise both
// are 0 (pass 1).  Writes changed rows, marks the tiles of the other tiling
// that hold a star neighbour of a changed point, returns the number of
// changed points (lane-summed by the caller).
template <int NDIM, bool SEEDED>
__device__ __forceinline__ uint32_t tile_fix(const TileArgs& a, int tiling, uint32_t tz, uint32_t ty, uint32_t tx,
                                             TileWarpSmem& W, int next_pass, uint32_t& my_max) {
  using G = Geo<NDIM>;
  using B = TBox<NDIM>;
  constexpr int D = G::D;
  constexpr int SW = G::SW;
  constexpr int JX = D;  // the -x slot (0,0,-1): weight 0, closed by xfill
  const int lane = threadIdx.x & 31;
  const int64_t d0 = a.d0, d1 = a.d1, d2 = a.d2;
  const size_t nseg = (size_t)a.nseg;
  const int64_t z0 = (int64_t)tz * G::TZ - (tiling ? B::SZ : 0);
  const int64_t y0 = (int64_t)ty * G::TY - (tiling ? B::SY : 0);
  const int64_t x0 = (int64_t)tx * G::TX;
  const uint32_t vmask = x0 + 32 <= d2 ? 0xffffffffu : ((1u << (uint32_t)(d2 - x0)) - 1u);

  // own rows rr = lane + 32 i: flags, seeds, edge subbins
  uint32_t F[2][2 * D];
  uint32_t sp[2][kSP];
  uint32_t eL[2], eR[2];
  int lz[2], ly[2], bi[2];
  bool rin[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int rr = lane + 32 * i;
    lz[i] = rr / G::TY;
    ly[i] = rr % G::TY;
    bi[i] = B::idx(lz[i], ly[i]);
    const int64_t gz = z0 + lz[i], gy = y0 + ly[i];
    rin[i] = gz >= 0 && gz < d0 && gy >= 0 && gy < d1;
    const uint4* seg = reinterpret_cast<const uint4*>(a.flags + ((size_t)(rin[i] ? gz * d1 + gy : 0) * nseg + tx) * SW);
#pragma unroll
    for (int q = 0; q < SW / 4; ++q) {
      const uint4 w = rin[i] ? __ldg(seg + q) : make_uint4(0, 0, 0, 0);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (4 * q + t < 2 * D) F[i][4 * q + t] = ws[t];
    }
    if (SEEDED) {
      load_sp_row(a, gz, gy, (int64_t)tx, sp[i], eL[i], eR[i]);
    } else {
#pragma unroll
      for (int b = 0; b < kSP; ++b) sp[i][b] = 0;
      eL[i] = eR[i] = 0;
    }
  }
  // halo rows: planes and edge subbins to shared memory
  if (SEEDED) {
    for (int h = lane; h < B::NH; h += 32) {
      int bz, by;
      B::halo(h, bz, by);
      uint32_t p[kSP], l, r;
      load_sp_row(a, z0 + bz, y0 + by, (int64_t)tx, p, l, r);
#pragma unroll
      for (int b = 0; b < kSP; ++b) W.hp[h][b] = p[b];
      W.he[h][0] = (uint8_t)l;
      W.he[h][1] = (uint8_t)r;
    }
  }
  // level words of the box: halo rows hold 0 (pass 1) or their level sets
  for (int t = lane; t < B::NB; t += 32) {
    W.lv[0][t] = 0;
    W.lv[1][t] = 0;
    W.ed[0][t] = 0;
    W.ed[1][t] = 0;
  }
  __syncwarp();

  uint32_t cnt[2][kSP];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int b = 0; b < kSP; ++b) cnt[i][b] = 0;
  uint32_t X[2] = {0, 0};
  int L = 1;
  for (;; ++L) {
    uint32_t* cur = W.lv[L & 1];
    const uint32_t* prv = W.lv[(L - 1) & 1];
    uint8_t* cE = W.ed[L & 1];
    const uint8_t* pE = W.ed[(L - 1) & 1];
    if (SEEDED) {  // the halo's level sets at L (prv holds L - 1 from the last level)
      for (int h = lane; h < B::NH; h += 32) {
        int bz, by;
        B::halo(h, bz, by);
        uint32_t p[kSP];
#pragma unroll
        for (int b = 0; b < kSP; ++b) p[b] = W.hp[h][b];
        const int t = B::idx(bz, by);
        cur[t] = planes_ge(p, (uint32_t)L);
        cE[t] = (uint8_t)(((uint32_t)W.he[h][0] >= (uint32_t)L) | (((uint32_t)W.he[h][1] >= (uint32_t)L) << 1));
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) cE[bi[i]] = (uint8_t)((eL[i] >= (uint32_t)L) | ((eR[i] >= (uint32_t)L) << 1));
      __syncwarp();
    }
    uint32_t P[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      uint32_t pv = SEEDED ? planes_ge(sp[i], (uint32_t)L) : 0u;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (L == 1) {
          pv |= F[i][j];  // from any predecessor (s >= 0) through a w = 1 arc
        } else {
          const int t = B::idx(lz[i] + slot_dz<NDIM>(j), ly[i] + slot_dy<NDIM>(j));
          uint32_t v = prv[t];
          if (slot_dx<NDIM>(j) > 0) v = (v >> 1) | (SEEDED ? ((uint32_t)(pE[t] >> 1) << 31) : 0u);
          pv |= F[i][j] & v;
        }
      }
      if (SEEDED) pv |= F[i][JX] & (uint32_t)(cE[bi[i]] & 1u);  // -x neighbour x0-1 (halo) at level L
      P[i] = pv;
      X[i] = xfill(pv, F[i][JX]);
    }
    // -e closure across rows (weight 0), Jacobi until stable
    for (;;) {
      cur[bi[0]] = X[0];
      cur[bi[1]] = X[1];
      __syncwarp();
      uint32_t Y[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint32_t y = P[i];
#pragma unroll
        for (int j = D + 1; j < 2 * D; ++j) {
          const int t = B::idx(lz[i] + slot_dz<NDIM>(j), ly[i] + slot_dy<NDIM>(j));
          uint32_t v = cur[t];
          if (slot_dx<NDIM>(j) < 0) v = (v << 1) | (SEEDED ? (uint32_t)(cE[t] & 1u) : 0u);
          y |= F[i][j] & v;
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
    if (L == kMaxPlaneLevel) {  // s would not fit 8 planes: the host re-runs on the u32 engine
      if (lane == 0) atomicOr(&a.ctr->err, kErrPlanes);
      break;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {  // bit-sliced count += Lev_L
      uint32_t carry = X[i];
#pragma unroll
      for (int b = 0; b < kSP; ++b) {
        const uint32_t t = cnt[i][b] & carry;
        cnt[i][b] ^= carry;
        carry = t;
      }
    }
  }
  const uint32_t top = (uint32_t)(L - 1);
  my_max = top > my_max ? top : my_max;

  // changed points, write-back, marks for the next pass
  uint32_t nch = 0, zy_mask = 0, xs = 0;
  const int nt = tiling ^ 1;
  const int64_t nz0 = z0 - 1 + (nt ? B::SZ : 0), ny0 = y0 - 1 + (nt ? B::SY : 0);
  const int64_t tzb = nz0 >= 0 ? nz0 / G::TZ : -1, tyb = ny0 >= 0 ? ny0 / G::TY : -1;  // next-tiling tile of (z0-1, y0-1)
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    uint32_t ch = 0;
#pragma unroll
    for (int b = 0; b < kSP; ++b) ch |= cnt[i][b] ^ sp[i][b];
    ch &= rin[i] ? vmask : 0u;
    const int64_t gz = z0 + lz[i], gy = y0 + ly[i];
    if (SEEDED ? ch != 0u : rin[i]) {  // pass 1 writes every row (no memset of the planes)
      uint4* dst = reinterpret_cast<uint4*>(a.sp + ((size_t)(gz * d1 + gy) * nseg + tx) * kSP);
      __stcg(dst, make_uint4(cnt[i][0] & vmask, cnt[i][1] & vmask, cnt[i][2] & vmask, cnt[i][3] & vmask));
      __stcg(dst + 1, make_uint4(cnt[i][4] & vmask, cnt[i][5] & vmask, cnt[i][6] & vmask, cnt[i][7] & vmask));
    }
    if (!ch) continue;
    nch += __popc(ch);
    // next-tiling tiles of the rows z-1..z+1, y-1..y+1 relative to (tzb, tyb)
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz) {
      if (NDIM == 2 && dz) continue;
      const int64_t z = gz + dz;
      if (z < 0 || z >= d0) continue;
      const int rz = (int)((z + (nt ? B::SZ : 0)) / G::TZ - tzb);
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy) {
        const int64_t y = gy + dy;
        if (y < 0 || y >= d1) continue;
        const int ry = (int)((y + (nt ? B::SY : 0)) / G::TY - tyb);
        zy_mask |= 1u << (rz * 3 + ry);
      }
    }
    xs |= 2u | (ch & 1u) | ((ch >> 31) << 2);  // bit 0: tx-1, 1: tx, 2: tx+1
  }
  zy_mask = __reduce_or_sync(0xffffffffu, zy_mask);
  xs = __reduce_or_sync(0xffffffffu, xs);
  if (zy_mask) {
    // lane k < 27 handles (rz, ry, rx) = k: mark, and append the fresh ones
    const int rz = lane / 9, ry = (lane / 3) % 3, rx = lane % 3;
    bool fresh = false;
    uint32_t id = 0;
    if (lane < 27 && ((zy_mask >> (rz * 3 + ry)) & 1u) && ((xs >> rx) & 1u)) {
      const int64_t ntz = tzb + rz, nty = tyb + ry, ntx = (int64_t)tx + rx - 1;
      if (ntz >= 0 && ntz < a.nt[nt][0] && nty >= 0 && nty < a.nt[nt][1] && ntx >= 0 && ntx < a.nt[nt][2]) {
        id = (uint32_t)((ntz * a.nt[nt][1] + nty) * a.nt[nt][2] + ntx);
        fresh = atomicOr(&a.act[nt][id], 1u) == 0u;
      }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, fresh);
    if (m) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&a.ctr->tl_count[next_pass % 3], (uint32_t)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (fresh) a.list[nt][base + __popc(m & ((1u << lane) - 1u))] = id;
    }
  }
  return nch;
}

template <int NDIM>
__global__ void __launch_bounds__(kTileThreads, LOPC_TILE_CTAS) k_tiles(TileArgs a) {
  namespace cg = cooperative_groups;
  using G = Geo<NDIM>;
  __shared__ TileWarpSmem S[kTileWarps];
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TileWarpSmem& W = S[warp];
  uint32_t my_max = 0;
  unsigned long long my_changed = 0;
  const uint64_t t_start = (a.prof && tid == 0 && blockIdx.x == 0) ? gtimer() : 0;
  int q = 1;
  for (; q <= a.max_passes; ++q) {
    const int tiling = (q - 1) & 1;
    const uint32_t n = q == 1 ? a.ntiles[0] : *(volatile uint32_t*)&a.ctr->tl_count[q % 3];
    if (n == 0) break;
    const uint32_t ntx = a.nt[tiling][2], ntxy = a.nt[tiling][1] * ntx;
    for (;;) {
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(&a.ctr->tl_ticket[q % 3], 1u);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= n) break;
      uint32_t id;
      if (q == 1) {
        id = t;
      } else {
        id = __ldcg(&a.list[tiling][n - 1 - t]);  // reverse build order: alternate sweep direction
        if (lane == 0) a.act[tiling][id] = 0u;     // may be marked again for pass q + 2
      }
      const uint32_t tz = id / ntxy, rem = id - tz * ntxy, ty = rem / ntx, tx = rem - ty * ntx;
      uint32_t c = q == 1 ? tile_fix<NDIM, false>(a, tiling, tz, ty, tx, W, q + 1, my_max)
                          : tile_fix<NDIM, true>(a, tiling, tz, ty, tx, W, q + 1, my_max);
      my_changed += c;
    }
    if (tid == 0 && blockIdx.x == 0) {
      a.ctr->tl_count[(q + 2) % 3] = 0;
      a.ctr->tl_ticket[(q + 2) % 3] = 0;
      if (q < kPassHist) a.ctr->pass_items[q] = n;
      a.ctr->worklist_points += n;  // tiles processed
      if (a.prof && q < kPassHist) a.ctr->pass_ns[q] = gtimer() - t_start;
    }
    __threadfence();
    grid.sync();
  }
  if (tid == 0 && blockIdx.x == 0) a.ctr->passes = (unsigned long long)(q - 1);
  const unsigned cw = __reduce_add_sync(0xffffffffu, (unsigned)my_changed);
  my_max = __reduce_max_sync(0xffffffffu, my_max);
  if (lane == 0 && cw) atomicAdd(&a.ctr->raised, (unsigned long long)cw);
  if (lane == 0 && my_max) atomicMax(&a.ctr->max_s, my_max);
  (void)G::TZ;
}

// Subbin planes -> one u32 per point (the encoder's input, and repair_ex).
template <int NDIM>
__global__ void __launch_bounds__(256) k_planes_to_s(const uint32_t* __restrict__ sp, uint32_t* __restrict__ s,
                                                     int64_t d0, int64_t d1, int64_t d2, int64_t nseg) {
  const int lane = threadIdx.x & 31;
  const int64_t nrowseg = d0 * d1 * nseg;
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < nrowseg;
       g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = g / nseg, sg = g - row * nseg;
    const int64_t x = sg * 32 + lane;
    const uint4* p4 = reinterpret_cast<const uint4*>(sp + (size_t)g * kSP);
    const uint4 a0 = __ldg(p4), a1 = __ldg(p4 + 1);
    const uint32_t w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < kSP; ++b) v |= ((w[b] >> lane) & 1u) << b;
    if (x < d2) __stcs(&s[row * d2 + x], v);
  }
}

}  // namespace lopc
