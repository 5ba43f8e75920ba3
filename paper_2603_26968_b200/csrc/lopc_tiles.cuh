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
//   pass 1        every tile of tiling 0 (4x8x32 in 3D, 32x32 in 2D: one
//                 warp each, lane = row), halo and seeds 0.
//   pass q >= 2   the ACTIVE tiles of tiling (q-1) mod 2.  Tiling 1 is
//                 tiling 0 shifted by half a tile in z and y (x stays
//                 32-aligned so a tile row is one flag / plane segment): a
//                 chain that crosses a tile border in one tiling runs inside
//                 a tile of the other (overlapping-domain / alternating
//                 Schwarz relaxation).  A tile of pass q+1 is active iff one
//                 of its points is an out-of-tile star neighbour of a point
//                 that changed in pass q (successors inside the changed
//                 point's own tile are satisfied by that tile's fixpoint);
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

// Tile geometry of the repair: 32 rows of 32 points, one row per lane
// (3D 4 x 8 x 32, 2D 32 x 32); the box adds the one-cell halo in z and y.
template <int NDIM>
struct TG {
  static constexpr int TZ = NDIM == 3 ? 4 : 1, TY = NDIM == 3 ? 8 : 32, ZH = NDIM == 3 ? 1 : 0;
  static constexpr int D = NDIM == 3 ? 7 : 3;          // +e offsets (G2)
  static constexpr int SW = NDIM == 3 ? 16 : 8;        // flag words per segment (Geo<NDIM>::SW)
  static constexpr int BY = TY + 2;                    // box rows along y
  static constexpr int NB = (TZ + 2 * ZH) * BY;        // box rows
  static constexpr int NH = NDIM == 3 ? 2 * (TY + 1) + 2 * TZ : 2;  // halo rows a star offset reaches (26 / 2)
  static constexpr int SZ = TZ / 2, SY = TY / 2;       // tiling 1 shift (z, y)
  __host__ __device__ static constexpr int idx(int bz, int by) { return (bz + ZH) * BY + (by + 1); }
  // halo row h -> box coordinates: the z0-1 plane (y0-1 .. y0+TY-1), the
  // z0+TZ plane (y0 .. y0+TY), then the y0-1 and y0+TY rows of every plane
  __host__ __device__ static void halo(int h, int& bz, int& by) {
    if (NDIM == 2) {
      bz = 0;
      by = h == 0 ? -1 : TY;
      return;
    }
    if (h <= TY) {
      bz = -1;
      by = h - 1;
    } else if (h <= 2 * TY + 1) {
      bz = TZ;
      by = h - (TY + 1);
    } else if (h < 2 * TY + 2 + TZ) {
      bz = h - (2 * TY + 2);
      by = -1;
    } else {
      bz = h - (2 * TY + 2 + TZ);
      by = TY;
    }
  }
};
static_assert(TG<3>::TZ * TG<3>::TY == 32 && TG<2>::TY == 32, "one tile row per lane");
static_assert(TG<3>::NH <= 32, "one halo row per lane");

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
  int q0;  // first pass: 1 (all tiles of tiling 0, unseeded), or 2 (slab rounds: the list of tiling 1 built by k_ghost_inject_tiles)
};

struct TileWarpSmem {
  uint32_t lv[2][TG<3>::NB];  // level words of the box rows, [L & 1]
  uint8_t ed[2][TG<3>::NB];   // edge level bits: bit 0 = x0-1, bit 1 = x0+32
  uint32_t hp[kSP][32];       // halo row planes, [plane][lane] (register relief)
  uint8_t hidx[32];           // box row of lane's halo row (kept here: re-deriving it per level costs ~20 instructions)
};

// s >= L on bit-sliced planes, branch-free: no borrow out of s - L
template <int NP>
__device__ __forceinline__ uint32_t planes_ge(const uint32_t (&p)[NP], uint32_t L) {
  uint32_t borrow = 0;
#pragma unroll
  for (int b = 0; b < NP; ++b) {
    const uint32_t l = 0u - ((L >> b) & 1u);  // bit b of L as a mask
    // borrow' = (~p & l) | (~(p ^ l) & borrow)
    borrow = (~p[b] & l) | (~(p[b] ^ l) & borrow);
  }
  // values < 2^NP: L >= 2^NP is above all of them
  return (L >> NP) ? 0u : ~borrow;
}

// One row's subbin planes (x-aligned segment tx) and the subbins of its x
// halo points x0-1, x0+32 (bits 31 / 0 of the neighbouring segments).
// L2 loads: other tiles write planes during the pass.
__device__ __forceinline__ void load_sp_row(const TileArgs& a, bool in, int64_t gz, int64_t gy, int64_t tx,
                                            uint32_t (&p)[kSP], uint32_t& eL, uint32_t& eR) {
#pragma unroll
  for (int b = 0; b < kSP; ++b) p[b] = 0;
  eL = eR = 0;
  if (!in || gz < 0 || gz >= a.d0 || gy < 0 || gy >= a.d1) return;
  const uint4* r4 = reinterpret_cast<const uint4*>(a.sp + ((size_t)(gz * a.d1 + gy) * (size_t)a.nseg + (size_t)tx) * kSP);
  const bool hl = tx > 0, hr = tx + 1 < a.nseg;
  const uint4 c0 = __ldcg(r4), c1 = __ldcg(r4 + 1);
  const uint4 l0 = hl ? __ldcg(r4 - 2) : make_uint4(0, 0, 0, 0), l1 = hl ? __ldcg(r4 - 1) : make_uint4(0, 0, 0, 0);
  const uint4 q0 = hr ? __ldcg(r4 + 2) : make_uint4(0, 0, 0, 0), q1 = hr ? __ldcg(r4 + 3) : make_uint4(0, 0, 0, 0);
  p[0] = c0.x, p[1] = c0.y, p[2] = c0.z, p[3] = c0.w, p[4] = c1.x, p[5] = c1.y, p[6] = c1.z, p[7] = c1.w;
  eL = (l0.x >> 31) | ((l0.y >> 31) << 1) | ((l0.z >> 31) << 2) | ((l0.w >> 31) << 3) | ((l1.x >> 31) << 4) |
       ((l1.y >> 31) << 5) | ((l1.z >> 31) << 6) | ((l1.w >> 31) << 7);
  eR = (q0.x & 1u) | ((q0.y & 1u) << 1) | ((q0.z & 1u) << 2) | ((q0.w & 1u) << 3) | ((q1.x & 1u) << 4) |
       ((q1.y & 1u) << 5) | ((q1.z & 1u) << 6) | ((q1.w & 1u) << 7);
}

// The level loop of one tile on NP bit planes: cnt = the new subbins (planes
// >= NP zero).  Returns L = 1 + the highest non-empty level, or -1 when a
// level reaches 2^NP - 1 (the count would not fit NP planes).
//
// L0 (seeded passes): no constraint of this tile is violated below level L0
// (every change since its points were last evaluated raised a point from a
// value >= L0 - 1, so only levels >= L0 of its successors can have moved):
// Lev_L = Seed_L for L < L0, and the loop starts at L0 from Seed_{L0-1}.
// first_new: the lowest level where Lev_L != Seed_L (0: nothing changed) —
// the level hint this visit passes on with its marks.
template <int NDIM, bool SEEDED, int NP>
__device__ __forceinline__ int tile_levels(const uint32_t (&F)[2 * TG<NDIM>::D], const uint32_t (&sp)[kSP], uint32_t eL,
                                           uint32_t eR, uint32_t hL, uint32_t hR, int bi, int hbi, int lz, int ly,
                                           TileWarpSmem& W, uint32_t (&cnt)[kSP], int L0, int& first_new) {
  using G = TG<NDIM>;
  constexpr int D = G::D;
  constexpr int JX = D;  // the -x slot (0,0,-1): weight 0, closed by xfill
  const int lane = threadIdx.x & 31;
  (void)lz;
  (void)ly;
  // level words of the box: Lev_0 = every point (s >= 0: the flags mask the
  // arcs, so all-ones serves), the other buffer 0 (pass 1's halo stays 0)
  const int Ls = SEEDED ? L0 : 1;
  for (int t = lane; t < G::NB; t += 32) {
    W.lv[0][t] = 0xffffffffu;
    W.lv[1][t] = 0;
    W.ed[0][t] = 3;
    W.ed[1][t] = 0;
  }
  __syncwarp();
  uint32_t spn[NP];
#pragma unroll
  for (int b = 0; b < NP; ++b) spn[b] = sp[b];
#pragma unroll
  for (int b = 0; b < kSP; ++b) cnt[b] = 0;
  first_new = 0;
  if (SEEDED && L0 > 1) {
    // start from Seed_{L0-1}: level words and edge bits of the tile and halo
    // rows at L0 - 1, and the counts min(seed, L0 - 1)
    const uint32_t Lb = (uint32_t)(L0 - 1);
    uint32_t* prv = W.lv[Lb & 1];
    uint8_t* pE = W.ed[Lb & 1];
    if (lane < G::NH) {
      uint32_t hp[NP];
#pragma unroll
      for (int b = 0; b < NP; ++b) hp[b] = W.hp[b][lane];
      const int hb = W.hidx[lane];
      prv[hb] = planes_ge<NP>(hp, Lb);
      pE[hb] = (uint8_t)((hL >= Lb) | ((hR >= Lb) << 1));
    }
    const uint32_t m = planes_ge<NP>(spn, Lb);
    prv[bi] = m;
    pE[bi] = (uint8_t)((eL >= Lb) | ((eR >= Lb) << 1));
#pragma unroll
    for (int b = 0; b < NP; ++b) cnt[b] = (m & (0u - ((Lb >> b) & 1u))) | (~m & spn[b]);
    __syncwarp();
  }
  uint32_t X = 0;
  int L = Ls;
  for (;; ++L) {
    uint32_t* cur = W.lv[L & 1];
    const uint32_t* prv = W.lv[(L - 1) & 1];
    uint8_t* cE = W.ed[L & 1];
    const uint8_t* pE = W.ed[(L - 1) & 1];
    if (SEEDED) {  // the halo's level sets at L (prv holds L - 1 from the last level)
      if (lane < G::NH) {
        uint32_t hp[NP];
#pragma unroll
        for (int b = 0; b < NP; ++b) hp[b] = W.hp[b][lane];
        const int hb = W.hidx[lane];
        cur[hb] = planes_ge<NP>(hp, (uint32_t)L);
        cE[hb] = (uint8_t)((hL >= (uint32_t)L) | ((hR >= (uint32_t)L) << 1));
      }
      cE[bi] = (uint8_t)((eL >= (uint32_t)L) | ((eR >= (uint32_t)L) << 1));
      __syncwarp();
    }
    const uint32_t seedL = SEEDED ? planes_ge<NP>(spn, (uint32_t)L) : 0u;
    uint32_t pv = seedL;
#pragma unroll
    for (int j = 0; j < D; ++j) {  // +e slots: w = 1 arcs from Lev_{L-1}
      const int t = bi + slot_dz<NDIM>(j) * G::BY + slot_dy<NDIM>(j);
      uint32_t v = prv[t];
      if (slot_dx<NDIM>(j) > 0) v = (v >> 1) | ((uint32_t)(pE[t] >> 1) << 31);
      pv |= F[j] & v;
    }
    if (SEEDED) pv |= F[JX] & (uint32_t)(cE[bi] & 1u);  // -x neighbour x0-1 (halo) at level L
    if (!SEEDED && L == 1) {  // pass 1: the halo is 0 at every level >= 1 (the Lev_0 buffer is reused for L = 2)
      __syncwarp();
      for (int t = lane; t < G::NB; t += 32) {
        W.lv[0][t] = 0;
        W.ed[0][t] = 0;
      }
    }
    const uint32_t P = pv;
    X = xfill(pv, F[JX]);
    // -e closure across rows (weight 0), Jacobi until stable
    for (;;) {
      cur[bi] = X;
      __syncwarp();
      uint32_t y = P;
#pragma unroll
      for (int j = D + 1; j < 2 * D; ++j) {
        const int t = bi + slot_dz<NDIM>(j) * G::BY + slot_dy<NDIM>(j);
        uint32_t v = cur[t];
        if (slot_dx<NDIM>(j) < 0) v = (v << 1) | (SEEDED ? (uint32_t)(cE[t] & 1u) : 0u);
        y |= F[j] & v;
      }
      const uint32_t Y = xfill(y, F[JX]);
      const bool ch = Y != X;
      X = Y;
      __syncwarp();
      if (!__any_sync(0xffffffffu, ch)) break;
    }
    if (!__any_sync(0xffffffffu, X != 0)) break;  // Lev_L empty: done
    if (SEEDED && first_new == 0 && __any_sync(0xffffffffu, X != seedL)) first_new = L;
    if (L == (1 << NP) - 1) return -1;            // the count would not fit NP planes
    uint32_t carry = X;  // bit-sliced count += Lev_L
#pragma unroll
    for (int b = 0; b < NP; ++b) {
      const uint32_t t = cnt[b] & carry;
      cnt[b] ^= carry;
      carry = t;
    }
  }
  return L;
}

// Exact fixpoint of one tile (one warp, lane = tile row).  SEEDED: current
// subbins are lower bounds and the halo holds the neighbours' current
// subbins; otherwise both are 0 (pass 1).  Writes changed rows, marks the
// tiles of the other tiling that hold a star neighbour of a changed point,
// returns this lane's number of changed points.
template <int NDIM, bool SEEDED>
__device__ __forceinline__ uint32_t tile_fix(const TileArgs& a, int tiling, uint32_t tz, uint32_t ty, uint32_t tx,
                                             TileWarpSmem& W, int next_pass, uint32_t& my_max, uint32_t* mark) {
  using G = TG<NDIM>;
  constexpr int D = G::D;
  constexpr int SW = G::SW;
  const int lane = threadIdx.x & 31;
  const int64_t d0 = a.d0, d1 = a.d1, d2 = a.d2;
  const size_t nseg = (size_t)a.nseg;
  const int64_t z0 = (int64_t)tz * G::TZ - (tiling ? G::SZ : 0);
  const int64_t y0 = (int64_t)ty * G::TY - (tiling ? G::SY : 0);
  const int64_t x0 = (int64_t)tx * 32;
  const uint32_t vmask = x0 + 32 <= d2 ? 0xffffffffu : ((1u << (uint32_t)(d2 - x0)) - 1u);

  // own row: flags, seeds, edge subbins
  const int lz = lane / G::TY, ly = lane % G::TY, bi = G::idx(lz, ly);
  const int64_t gz = z0 + lz, gy = y0 + ly;
  const bool rin = gz >= 0 && gz < d0 && gy >= 0 && gy < d1;
  // this tile's mark word (seeded passes): 256 - the lowest level that may
  // have moved (all marks for this pass were made in the previous one),
  // loaded beside the row loads; reset so the tile can be marked again for
  // the pass after next
  const uint32_t mw = (SEEDED && mark) ? __ldcg(mark) : 0u;
  uint32_t F[2 * D];
  {
    const uint4* seg = reinterpret_cast<const uint4*>(a.flags + ((size_t)(rin ? gz * d1 + gy : 0) * nseg + tx) * SW);
#pragma unroll
    for (int q = 0; q < SW / 4; ++q) {
      const uint4 w = rin ? __ldg(seg + q) : make_uint4(0, 0, 0, 0);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (4 * q + t < 2 * D) F[4 * q + t] = ws[t];
    }
  }
  uint32_t sp[kSP], eL = 0, eR = 0;
  // halo row of this lane (lane < NH): planes (to shared memory) and edge subbins
  uint32_t hL = 0, hR = 0;
  int hbi = 0;
  if (SEEDED) {
    load_sp_row(a, true, gz, gy, (int64_t)tx, sp, eL, eR);
    int hz, hy;
    G::halo(lane < G::NH ? lane : 0, hz, hy);
    hbi = G::idx(hz, hy);
    uint32_t hp[kSP];
    load_sp_row(a, lane < G::NH, z0 + hz, y0 + hy, (int64_t)tx, hp, hL, hR);
#pragma unroll
    for (int b = 0; b < kSP; ++b) W.hp[b][lane] = hp[b];
    W.hidx[lane] = (uint8_t)hbi;
  } else {
#pragma unroll
    for (int b = 0; b < kSP; ++b) sp[b] = 0;
  }
  // the level sets on NP planes: NP = 4 when every seed and halo subbin is
  // below 16 (the usual tile), re-run on 8 planes if a level reaches 16
  uint32_t cnt[kSP];
  uint32_t big = 0;
#pragma unroll
  for (int b = 4; b < kSP; ++b) big |= sp[b] | (SEEDED && lane < G::NH ? W.hp[b][lane] : 0u);
  big |= (eL | eR | hL | hR) >> 4;
  const int lmin = mw ? 256 - (int)mw : 1;
  if (SEEDED && mark && lane == 0) *mark = 0u;
  int L = 0, first_new = 0;
  if (!__any_sync(0xffffffffu, big != 0))
    L = tile_levels<NDIM, SEEDED, 4>(F, sp, eL, eR, hL, hR, bi, hbi, lz, ly, W, cnt, lmin, first_new);
  if (L <= 0) {
    L = tile_levels<NDIM, SEEDED, kSP>(F, sp, eL, eR, hL, hR, bi, hbi, lz, ly, W, cnt, lmin, first_new);
    if (L < 0) {  // s would not fit 8 planes: the host re-runs on the u32 engine
      if (lane == 0) atomicOr(&a.ctr->err, kErrPlanes);
      L = kMaxPlaneLevel;
    }
  }
  const uint32_t top = (uint32_t)(L - 1);
  my_max = top > my_max ? top : my_max;
  if (SEEDED && a.prof && lane == 0) {  // diagnostic (lopc_set_timing(2)): seeded visits, visits with a change,
    atomicAdd(&a.ctr->dense_cycles[0], 1ull);  // levels run, levels below the first changed one
    if (first_new) atomicAdd(&a.ctr->dense_cycles[1], 1ull);
    atomicAdd(&a.ctr->dense_cycles[2], (unsigned long long)(L - lmin + 1));
    atomicAdd(&a.ctr->dense_cycles[3], (unsigned long long)(first_new ? first_new - lmin : L - lmin + 1));
  }

  // changed points, write-back, marks for the next pass
  uint32_t ch = 0;
#pragma unroll
  for (int b = 0; b < kSP; ++b) ch |= cnt[b] ^ sp[b];
  ch &= rin ? vmask : 0u;
  if (SEEDED ? ch != 0u : rin) {  // pass 1 writes every row (no memset of the planes)
    uint4* dst = reinterpret_cast<uint4*>(a.sp + ((size_t)(gz * d1 + gy) * nseg + tx) * kSP);
    __stcg(dst, make_uint4(cnt[0] & vmask, cnt[1] & vmask, cnt[2] & vmask, cnt[3] & vmask));
    __stcg(dst + 1, make_uint4(cnt[4] & vmask, cnt[5] & vmask, cnt[6] & vmask, cnt[7] & vmask));
  }
  const int nt = tiling ^ 1;
  const int64_t nz0 = z0 - 1 + (nt ? G::SZ : 0), ny0 = y0 - 1 + (nt ? G::SY : 0);
  const int64_t tzb = nz0 >= 0 ? nz0 / G::TZ : -1, tyb = ny0 >= 0 ? ny0 / G::TY : -1;  // next-tiling tile of (z0-1, y0-1)
  // Only successors OUTSIDE this tile can have become unsatisfied (inside,
  // the tile's fixpoint already accounts for every change): mark the
  // next-tiling tiles holding the out-of-tile star neighbours of changed
  // points.  m27 bit (rz * 9 + ry * 3 + rx): tile (tzb + rz, tyb + ry, tx + rx - 1).
  uint32_t m27 = 0;
  if (ch) {
#pragma unroll
    for (int j = 0; j < 2 * D; ++j) {
      const int dz = slot_dz<NDIM>(j), dy = slot_dy<NDIM>(j), dx = slot_dx<NDIM>(j);
      const int nz = lz + dz, ny = ly + dy;
      const bool row_out = nz < 0 || nz >= G::TZ || ny < 0 || ny >= G::TY;
      // a changed p can only feed q = p + e_j if q -> p is not an arc: within
      // a bin the arcs follow one total order (G4), so F_j(p) (the arc q -> p)
      // rules p -> q out
      const uint32_t cj = ch & ~F[j];
      uint32_t xm;
      if (row_out)
        xm = dx == 0 ? (cj ? 2u : 0u)
                     : dx > 0 ? (((cj & 0x7fffffffu) ? 2u : 0u) | ((cj >> 31) << 2))
                              : (((cj & 0xfffffffeu) ? 2u : 0u) | (cj & 1u));
      else
        xm = dx > 0 ? ((cj >> 31) << 2) : dx < 0 ? (cj & 1u) : 0u;
      const int64_t z = gz + dz, y = gy + dy;
      if (!xm || z < 0 || z >= d0 || y < 0 || y >= d1) continue;
      const int rz = (int)((z + (nt ? G::SZ : 0)) / G::TZ - tzb);
      const int ry = (int)((y + (nt ? G::SY : 0)) / G::TY - tyb);
      m27 |= xm << (rz * 9 + ry * 3);
    }
  }
  m27 = __reduce_or_sync(0xffffffffu, m27);
  if (m27) {
    // lane k < 27 marks tile k of the 3x3x3 neighbourhood; the fresh ones are appended
    const int rz = lane / 9, ry = (lane / 3) % 3, rx = lane % 3;
    bool fresh = false;
    uint32_t id = 0;
    // (selects, not a.x[nt]: a runtime index into the parameter struct
    // would copy it to local memory)
    const uint32_t nz = nt ? a.nt[1][0] : a.nt[0][0], ny = nt ? a.nt[1][1] : a.nt[0][1], nx = a.nt[0][2];
    uint32_t* act = nt ? a.act[1] : a.act[0];
    uint32_t* lst = nt ? a.list[1] : a.list[0];
    if (lane < 27 && ((m27 >> lane) & 1u)) {
      const int64_t mtz = tzb + rz, mty = tyb + ry, mtx = (int64_t)tx + rx - 1;
      if (mtz >= 0 && mtz < nz && mty >= 0 && mty < ny && mtx >= 0 && mtx < nx) {
        id = (uint32_t)((mtz * ny + mty) * nx + mtx);
        // mark word 256 - (lowest level that may have moved): the next visit
        // starts there (pass 1 changes everything from level 1)
        fresh = atomicMax(&act[id], 256u - (uint32_t)(SEEDED ? first_new : 1)) == 0u;
      }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, fresh);
    if (m) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&a.ctr->tl_count[next_pass % 3], (uint32_t)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (fresh) lst[base + __popc(m & ((1u << lane) - 1u))] = id;
    }
  }
  return (uint32_t)__popc(ch);
}

template <int NDIM>
__global__ void __launch_bounds__(kTileThreads, LOPC_TILE_CTAS) k_tiles(TileArgs a) {
  namespace cg = cooperative_groups;
  __shared__ TileWarpSmem S[kTileWarps];
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TileWarpSmem& W = S[warp];
  uint32_t my_max = 0;
  unsigned long long my_changed = 0;
  const uint64_t t_start = (a.prof && tid == 0 && blockIdx.x == 0) ? gtimer() : 0;
  int q = a.q0;
  for (; q <= a.max_passes; ++q) {
    const int tiling = (q - 1) & 1;
    const uint32_t n = q == 1 ? a.ntiles[0] : *(volatile uint32_t*)&a.ctr->tl_count[q % 3];
    if (n == 0) break;
    const uint32_t ntx = a.nt[0][2], ntxy = (tiling ? a.nt[1][1] : a.nt[0][1]) * ntx;
    const uint32_t* lst = tiling ? a.list[1] : a.list[0];
    uint32_t* act = tiling ? a.act[1] : a.act[0];
    // pass 1: static round-robin over all tiles (uniform work); later
    // passes: dynamic tickets over the active list, the next ticket fetched
    // while the current tile runs (its atomic round trip off the critical path)
    const uint32_t gw = blockIdx.x * kTileWarps + warp, nw = gridDim.x * kTileWarps;
    uint32_t tnext = gw;
    if (q > 1 && lane == 0) tnext = atomicAdd(&a.ctr->tl_ticket[q % 3], 1u);
    for (uint32_t k = 0;; ++k) {
      uint32_t t = q > 1 ? __shfl_sync(0xffffffffu, tnext, 0) : gw + k * nw;
      if (t >= n) break;
      if (q > 1 && lane == 0) tnext = atomicAdd(&a.ctr->tl_ticket[q % 3], 1u);
      const uint32_t id = q == 1 ? t : __ldcg(&lst[n - 1 - t]);  // reverse build order: alternate sweep direction
      const uint32_t tz = id / ntxy, rem = id - tz * ntxy, ty = rem / ntx, tx = rem - ty * ntx;
      my_changed += q == 1 ? tile_fix<NDIM, false>(a, tiling, tz, ty, tx, W, q + 1, my_max, nullptr)
                           : tile_fix<NDIM, true>(a, tiling, tz, ty, tx, W, q + 1, my_max, act + id);
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
}

// Subbin planes -> u32 for the linear range [start, start + count) of the
// plane grid (slab mode: the boundary points a halo exchange sends).
__global__ void __launch_bounds__(256) k_planes_range(const uint32_t* __restrict__ sp, uint32_t* __restrict__ s,
                                                      int64_t d2, int64_t nseg, int64_t start, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = start + i, row = p / d2, x = p - row * d2;
    const uint32_t* w = sp + ((size_t)row * (size_t)nseg + (size_t)(x >> 5)) * kSP;
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < kSP; ++b) v |= ((__ldg(w + b) >> (x & 31)) & 1u) << b;
    s[p] = v;
  }
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

// Slab mode on the tile engine: ghost points (box points
// owned by a neighbour rank) have no incoming arcs here, so no tile ever
// changes them; their subbins arrive from the owner after each round.  A
// ghost whose value rose gets its plane bits rewritten (one thread per
// point, each bit owned by one thread: per-bit atomics, no lost updates
// between the points of one segment) and marks the tiles of tiling 1 that
// hold its star neighbours, with the level hint old + 1 (its level sets
// changed from level old + 1 up), for the seeded first pass (q0 = 2) of the
// next k_tiles launch.  ctr->ghost_changed counts the raised ghosts (the
// round's termination term, summed over ranks).
template <int NDIM>
__global__ void __launch_bounds__(256) k_ghost_inject_tiles(TileArgs a, const uint32_t* __restrict__ recv, int64_t g0,
                                                            int64_t count) {
  using G = TG<NDIM>;
  const int lane = threadIdx.x & 31;
  const int64_t d0 = a.d0, d1 = a.d1, d2 = a.d2, plane = d1 * d2;
  unsigned changed = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = g0 + i;
    const int64_t z = p / plane, r2 = p - z * plane, y = r2 / d2, x = r2 - y * d2;
    uint32_t* w = a.sp + ((size_t)(z * d1 + y) * (size_t)a.nseg + (size_t)(x >> 5)) * kSP;
    const uint32_t bit = 1u << (x & 31);
    uint32_t old = 0;
#pragma unroll
    for (int b = 0; b < kSP; ++b) old |= ((__ldcg(w + b) & bit) ? 1u : 0u) << b;
    const uint32_t v = __ldg(&recv[i]);
    if (v <= old) continue;
    ++changed;
    if (v > (uint32_t)kMaxPlaneLevel) {  // does not fit 8 planes: the caller re-runs on the u32 engine
      atomicOr(&a.ctr->err, kErrPlanes);
      continue;
    }
#pragma unroll
    for (int b = 0; b < kSP; ++b) {
      const uint32_t nb = (v >> b) & 1u, ob = (old >> b) & 1u;
      if (nb && !ob) atomicOr(w + b, bit);
      if (!nb && ob) atomicAnd(w + b, ~bit);
    }
    // tiles of tiling 1 holding a star neighbour (the 3x3x3 box around p, clipped)
    const uint32_t mw = 256u - (old + 1u);
    const int64_t sz = G::SZ, sy = G::SY;
    const uint32_t ntz = a.nt[1][0], nty = a.nt[1][1], ntx = a.nt[1][2];
    const int64_t tz0 = (z - (NDIM == 3 ? 1 : 0) + sz) / G::TZ, tz1 = (z + (NDIM == 3 ? 1 : 0) + sz) / G::TZ;
    const int64_t ty0 = (y - 1 + sy) / G::TY, ty1 = (y + 1 + sy) / G::TY;
    const int64_t tx0 = (x > 0 ? x - 1 : 0) >> 5, tx1 = (x + 1 < d2 ? x + 1 : x) >> 5;
    for (int64_t tz = tz0; tz <= tz1; ++tz)
      for (int64_t ty = ty0; ty <= ty1; ++ty)
        for (int64_t tx = tx0; tx <= tx1; ++tx) {
          if (tz < 0 || tz >= ntz || ty < 0 || ty >= nty) continue;
          const uint32_t id = (uint32_t)((tz * nty + ty) * ntx + tx);
          if (atomicMax(&a.act[1][id], mw) == 0u) {
            const uint32_t slot = atomicAdd(&a.ctr->tl_count[2], 1u);
            a.list[1][slot] = id;
          }
        }
  }
  (void)d0;
  changed = __reduce_add_sync(0xffffffffu, changed);
  if (lane == 0 && changed) atomicAdd(&a.ctr->ghost_changed, (unsigned long long)changed);
}

}  // namespace lopc
