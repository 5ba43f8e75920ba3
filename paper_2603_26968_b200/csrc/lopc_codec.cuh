// lopc_codec.cuh — chunked lossless coding and decoding.
//
// Bins: "the lossless portion of PFPL" (readings G17-G19):
//   DIFFNB_k -> BIT_k -> RZE_1.
// Subbins: the LC pipelines BIT_4 RZE_4 RZE_1 / BIT_8 RZE_8 RZE_1.
// k_encode<T, 1> encodes the bins and k_encode<T, 2> the subbins of one
// 16 KiB chunk per CTA, into the chunk's 32 KiB staging slot; then
// k_chunk_scan (decoupled look-back over the size table: the exclusive prefix
// of bin_size + sub_size, a7) and k_place copy every payload to its final
// place (so the stream bytes move twice: a per-chunk look-back inside the
// encoder was measured slower).  With the tile engine the
// subbin CTAs read the repaired subbins as bit planes and the escape bits of
// the flags, not x; the bound self-check a4 runs in the bin CTAs.  Stream
// format: DESIGN.md §4.
//
// Word buffers in shared memory use an XOR swizzle so that the 32x32 bit
// transposes of BIT_k run bank-conflict-free.  u32 words (f32): the 16-byte
// chunk index within a 32-word group is XORed with the group's low 3 bits,
//   w ^ (((w >> 5) & 7) << 2),
// so 4-word aligned runs stay contiguous and in order (every access of 4+
// consecutive words is one 128-bit LDS/STS) and a quarter-warp reading the
// same chunk of 8 consecutive groups hits 8 distinct bank quads.  u64 words
// (f64): word w lives at (w & ~31) | ((w ^ (w >> 5)) & 31) (scalar accesses).
#pragma once
#include "lopc_device.cuh"
#include "lopc_repair.cuh"

namespace lopc {

constexpr int kCodecThreads = 256;

template <typename U>
__device__ __forceinline__ int swz(int w) {
  if constexpr (sizeof(U) == 4)
    return w ^ (((w >> 5) & 7) << 2);
  else
    return (w & ~31) | ((w ^ (w >> 5)) & 31);
}

// ---------------------------------------------------------------------------
// Block-wide exclusive scan (sum) over NT threads.
// ---------------------------------------------------------------------------
template <typename V, int NT = kCodecThreads>
__device__ __forceinline__ V block_scan_excl(V v, V* wsum, V* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  V x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    V y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    V t = lane < NW ? wsum[lane] : V(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      V y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < NW) wsum[lane] = t;
  }
  __syncthreads();
  V base = w ? wsum[w - 1] : V(0);
  *total = wsum[NW - 1];
  __syncthreads();
  return base + x - v;
}

// Two u64 exclusive scans in one pass (the same three block barriers);
// wsum needs 2 * NT/32 entries.
template <int NT = kCodecThreads>
__device__ __forceinline__ void block_scan_excl2(unsigned long long& a, unsigned long long& b, unsigned long long* wsum,
                                                 unsigned long long& ta, unsigned long long& tb) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long x = a, y = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long xo = __shfl_up_sync(0xffffffffu, x, o), yo = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) {
      x += xo;
      y += yo;
    }
  }
  if (lane == 31) {
    wsum[w] = x;
    wsum[NW + w] = y;
  }
  __syncthreads();
  if (w == 0) {
    unsigned long long t = lane < NW ? wsum[lane] : 0ull, u = lane < NW ? wsum[NW + lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long to = __shfl_up_sync(0xffffffffu, t, o), uo = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) {
        t += to;
        u += uo;
      }
    }
    if (lane < NW) {
      wsum[lane] = t;
      wsum[NW + lane] = u;
    }
  }
  __syncthreads();
  const unsigned long long ba = w ? wsum[w - 1] : 0ull, bb = w ? wsum[NW + w - 1] : 0ull;
  ta = wsum[NW - 1];
  tb = wsum[2 * NW - 1];
  __syncthreads();
  a = ba + x - a;
  b = bb + y - b;
}

// OR-combine `v` over aligned groups of `lanes` lanes.
__device__ __forceinline__ uint32_t group_or(uint32_t v, int lanes) {
  for (int o = 1; o < lanes; o <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// RZE_g (Fig. 2; format DESIGN.md §4), block-parallel.
//
// A "unit" is 16 words of g bytes: it owns exactly bytes 2u and 2u+1 of the
// first bitmap B0, so a thread with one unit knows its two B0 bytes, the B1
// bits at those positions (B0[t] != B0[t-1]) and hence its K0 bytes; one
// packed block scan gives every unit its K0 rank and its data rank.  B0 is
// never materialised.  The small upper levels (B1 -> B2 -> B3: <= 272 bytes)
// run on one warp with warp scans.
// ---------------------------------------------------------------------------
struct RzeScratch {
  uint32_t b1[72];   // B1, <= 272 bytes
  uint32_t b2[12];   // B2, <= 34 bytes
  uint32_t b3[4];    // B3, <= 5 bytes
  uint32_t pre1[72]; // decode: exclusive popcount prefix of B1 words
  uint8_t k1[288];   // K1
  uint8_t k2[48];    // K2
  uint32_t wsum[32];
  unsigned long long wsum64[32];  // (block_scan_excl2 uses 2 * 8 entries)
  uint32_t info[8];
  uint32_t ud[256];  // g = 4 / 8: per unit, non-zero word mask | data rank << 16
};

__device__ __forceinline__ int rze_sizes(uint32_t n, uint32_t* sz) {
  int top = 0;
  sz[0] = (n + 7) / 8;
  while (sz[top] > 8) {
    sz[top + 1] = (sz[top] + 7) / 8;
    ++top;
  }
  return top;
}

// 4 bits: which bytes of w are non-zero
__device__ __forceinline__ uint32_t nz4(uint32_t w) {
  const uint32_t t = (((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) & 0x80808080u;
  return (((t >> 7) * 0x00204081u) >> 21) & 0xfu;
}

// non-zero-word mask of 8 words of g bytes starting at p (16-byte aligned)
__device__ __forceinline__ uint32_t nz_words8(const uint8_t* p, int g) {
  if (g == 1) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    return nz4(v.x) | (nz4(v.y) << 4);
  }
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint32_t m = 0;
  if (g == 4) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint4 v = q[k];
      m |= ((uint32_t)(v.x != 0) | ((uint32_t)(v.y != 0) << 1) | ((uint32_t)(v.z != 0) << 2) |
            ((uint32_t)(v.w != 0) << 3)) << (4 * k);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 v = q[k];
      m |= ((uint32_t)((v.x | v.y) != 0) | ((uint32_t)((v.z | v.w) != 0) << 1)) << (2 * k);
    }
  }
  return m;
}

// Bits of an 8-bit (byte_mask) or 32-bit (word_mask) group starting at bit
// `start` that lie below `size`.
__device__ __forceinline__ uint32_t byte_mask(uint32_t size, uint32_t start) {
  return start >= size ? 0u : (size - start >= 8 ? 0xffu : (1u << (size - start)) - 1u);
}
__device__ __forceinline__ uint32_t word_mask(uint32_t size, uint32_t start) {
  return start >= size ? 0u : (size - start >= 32 ? 0xffffffffu : (1u << (size - start)) - 1u);
}

// Exclusive prefix over the warp of popc(bits) for 8-bit per-lane groups, by
// eight independent ballots (no dependent shuffle chain); tot = the total.
__device__ __forceinline__ uint32_t warp_prefix8(uint32_t bits, uint32_t& tot) {
  const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;
  uint32_t ex = 0;
  tot = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t b = __ballot_sync(0xffffffffu, (bits >> k) & 1u);
    ex += __popc(b & lt);
    tot += __popc(b);
  }
  return ex;
}

// one warp: next bitmap level.  bi: si bytes; writes B_{i+1} bytes to bn and
// K_i (bytes of bi whose B_{i+1} bit is set) to kb; returns |K_i|.
__device__ __forceinline__ uint32_t level_up_warp(const uint8_t* bi, uint32_t si, uint8_t* bn, uint8_t* kb) {
  const int lane = threadIdx.x & 31;
  uint32_t kcount = 0;
  for (uint32_t base = 0; base < si; base += 256) {
    const uint32_t t0 = base + 8 * lane;
    uint32_t bits = 0;
    if (t0 < si) {
      uint32_t prev = t0 ? bi[t0 - 1] : 0u;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (t0 + k < si) {
          const uint32_t cur = bi[t0 + k];
          bits |= (uint32_t)(cur != prev) << k;
          prev = cur;
        }
      }
      bn[t0 / 8] = (uint8_t)bits;
    }
    uint32_t tot;
    uint32_t pos = kcount + warp_prefix8(bits, tot);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if ((bits >> k) & 1u) kb[pos++] = bi[t0 + k];
    kcount += tot;
  }
  return kcount;
}

#ifndef LOPC_ENC_PF
#define LOPC_ENC_PF 1
#endif
#ifndef LOPC_DEC_PF
#define LOPC_DEC_PF 1  // k_decode1: the next chunk's payload prefetched into 0 nothing, 1 L1, 2 L2
#endif
__device__ __forceinline__ void pf_l1_bytes(const void* p) {
#if LOPC_DEC_PF == 1
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#elif LOPC_DEC_PF == 2
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#else
  (void)p;
#endif
}

// Byte i of a decoder input: shared memory, or (GIN) the payload in global
// memory read through L1 (the caller bounds i by the payload length).
template <bool GIN>
__device__ __forceinline__ uint32_t rd8(const uint8_t* p, uint32_t i) {
  if constexpr (GIN)
    return (uint32_t)__ldg(p + i);
  else
    return (uint32_t)p[i];
}

// One bitmap level down, in registers: lane l holds the 8 bits of level i+1
// that select level-i bytes 8l..8l+7 (`bits`, masked to the level size) and
// gets those bytes back: byte k = K_i[r - 1], r = the set bits at or before
// it counting from kcount (0 when r = 0), i.e. B_i[t] is the last K byte
// selected at or before t.  kcount += this block's |K_i|.  klim: bytes
// readable at kin (a corrupt payload may announce more K bytes than it holds;
// with GIN those reads must not leave the payload).
template <bool GIN>
__device__ __forceinline__ unsigned long long level_down_reg(uint32_t bits, const uint8_t* kin, uint32_t klim,
                                                             uint32_t& kcount) {
  uint32_t tot;
  uint32_t r = kcount + warp_prefix8(bits, tot);
  unsigned long long v = 0ull;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    r += (bits >> k) & 1u;
    v |= (unsigned long long)(r && r - 1 < klim ? rd8<GIN>(kin, r - 1) : 0u) << (8 * k);
  }
  kcount += tot;
  return v;
}

// RZE_g encode of `in` (shared, 16-byte aligned, L bytes, zero up to the next
// multiple of 16g) into `out` (shared, any alignment).  Returns the encoded
// length; `out` is written only if that length <= limit.
//
// Only the first L_act bytes (a multiple of 16g, block-uniform) may be
// non-zero: the bytes past them are taken as zero without being read (the
// caller knows which bit planes are all zero), so only the units up to the
// first all-zero one are visited.  L_act = L reads everything.
__device__ uint32_t rze_enc(const uint8_t* in, uint32_t L, int g, uint8_t* out, uint32_t limit, RzeScratch& R,
                            uint32_t L_act) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t n = L / (uint32_t)g;
  uint32_t sz[6];
  const int top = rze_sizes(n, sz);
  const uint32_t units = (n + 15) / 16, ub = 16u * (uint32_t)g;
  // units >= uact are all zero; unit uact still carries a B1 bit (B0 falls to 0)
  const uint32_t uact = top == 0 ? units : min(units, L_act / ub);
  const uint32_t uvis = min(units, uact + 1);
  constexpr int MAXIT = 5;  // units per thread: <= 1088 units / 256 threads
  uint32_t mk[MAXIT], rk[MAXIT];
  uint32_t running = 0;
  const int iters = (int)((uvis + kCodecThreads - 1) / kCodecThreads);
  if (top >= 1)  // B1 words past the visited units are zero
    for (uint32_t t = (uint32_t)iters * (kCodecThreads / 16) + tid; t < (units + 15) / 16; t += kCodecThreads) R.b1[t] = 0;
  // All units' masks first, then ONE pass of two u64 block scans: the data
  // counts (13 bits per iteration 0-3, <= 4096; 12 bits for iteration 4,
  // units >= 1024: <= 1024) and the K0 counts (10 bits per iteration, <= 512).
  unsigned long long pd = 0, pkc = 0;
#pragma unroll
  for (int it = 0; it < MAXIT; ++it) {
    mk[it] = 0;
    if (it >= iters) continue;
    const uint32_t u = (uint32_t)(it * kCodecThreads + tid);
    uint32_t m = 0, prevb = 0;
    if (u < uvis) {
      const uint8_t* p = in + u * ub;
      if (u < uact) m = nz_words8(p, g) | (nz_words8(p + 8 * g, g) << 8);
      prevb = u ? nz_words8(p - 8 * g, g) : 0u;
    }
    const uint32_t lo = m & 0xffu, hi = m >> 8;
    uint32_t b1 = 0;
    if (top >= 1 && u < uvis) b1 = (uint32_t)(lo != prevb) | ((uint32_t)(hi != lo && 2 * u + 1 < sz[0]) << 1);
    pd += (unsigned long long)__popc(m) << (13 * it);
    pkc += (unsigned long long)__popc(b1) << (10 * it);
    mk[it] = m | (b1 << 16);
    if (top >= 1) {
      const uint32_t w = group_or(b1 << (2 * (u & 15)), 16);
      if ((lane & 15) == 0 && u < units) R.b1[u >> 4] = w;  // zero past uvis
    }
  }
  unsigned long long td, tk;
  block_scan_excl2(pd, pkc, R.wsum64, td, tk);
#pragma unroll
  for (int it = 0; it < MAXIT; ++it) {
    if (it >= iters) break;
    const uint32_t field = it < 4 ? 0x1fffu : 0xfffu;
    const uint32_t ex = (uint32_t)((pd >> (13 * it)) & field) | ((uint32_t)((pkc >> (10 * it)) & 0x3ffu) << 20);
    rk[it] = running + ex;
    running += (uint32_t)((td >> (13 * it)) & field) | ((uint32_t)((tk >> (10 * it)) & 0x3ffu) << 20);
  }
  const uint32_t ndata = running & 0xfffffu, nk0 = running >> 20;
  __syncthreads();
  if (tid < 32) {
    uint32_t k2n = 0, k1n = 0;
    const uint8_t* b1 = reinterpret_cast<const uint8_t*>(R.b1);
    const uint8_t* b2 = reinterpret_cast<const uint8_t*>(R.b2);
    if (top >= 2) k1n = level_up_warp(b1, sz[1], reinterpret_cast<uint8_t*>(R.b2), R.k1);
    __syncwarp();
    if (top >= 3) k2n = level_up_warp(b2, sz[2], reinterpret_cast<uint8_t*>(R.b3), R.k2);
    __syncwarp();
    uint32_t o = sz[top];
    const uint32_t o2 = o;
    if (top >= 3) o += k2n;
    const uint32_t o1 = o;
    if (top >= 2) o += k1n;
    const uint32_t koff = o;
    const uint32_t doff = koff + nk0;
    const uint32_t total = doff + (uint32_t)g * ndata;
    if (total <= limit && top >= 1) {
      const uint8_t* bt = top == 1 ? b1 : (top == 2 ? b2 : reinterpret_cast<const uint8_t*>(R.b3));
      if ((uint32_t)lane < sz[top]) out[lane] = bt[lane];
      if (top >= 3)
        for (uint32_t t = lane; t < k2n; t += 32) out[o2 + t] = R.k2[t];
      if (top >= 2)
        for (uint32_t t = lane; t < k1n; t += 32) out[o1 + t] = R.k1[t];
    }
    if (lane == 0) {
      R.info[0] = koff;
      R.info[1] = doff;
      R.info[2] = total;
    }
  }
  __syncthreads();
  const uint32_t koff = R.info[0], doff = R.info[1], total = R.info[2];
  if (total <= limit) {
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      if (it >= iters) break;
      const uint32_t u = (uint32_t)(it * kCodecThreads + tid);
      const bool valid = u < uvis;
      const uint32_t m = valid ? mk[it] & 0xffffu : 0u, b1 = mk[it] >> 16;
      const uint32_t dr = rk[it] & 0xfffffu;
      if (valid) {
        const uint32_t kr = rk[it] >> 20;
        if (top == 0) {  // B0 itself is the top level (<= 8 bytes)
          if (2 * u < sz[0]) out[2 * u] = (uint8_t)(m & 0xffu);
          if (2 * u + 1 < sz[0]) out[2 * u + 1] = (uint8_t)(m >> 8);
        } else {
          uint32_t k = koff + kr;
          if (b1 & 1u) out[k++] = (uint8_t)(m & 0xffu);
          if (b1 & 2u) out[k] = (uint8_t)(m >> 8);
        }
      }
      uint8_t* d = out + doff;
      if (g == 1) {
        if (valid) {
          const uint4 v = *reinterpret_cast<const uint4*>(in + u * ub);
          const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
          uint32_t r = dr;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if ((m >> j) & 1u) d[r++] = (uint8_t)(w4[j >> 2] >> (8 * (j & 3)));
          }
        }
      } else if (valid) {
        R.ud[u] = m | (dr << 16);  // g = 4 / 8: units <= 256, data ranks < 2^13
      }
    }
  }
  if (g != 1) {
    // g = 4 / 8: the non-zero words of the visited units are scattered one
    // u32 per thread step over the whole block (the units with data cluster
    // in the first bit planes; one unit per warp at a time left most warps
    // idle at the closing barrier)
    __syncthreads();
    if (total <= limit) {
      const int uwl = g == 4 ? 0 : 1;  // log2(u32 per word)
      const uint32_t pu = 16u << uwl;   // u32 per unit
      const uint32_t* in32 = reinterpret_cast<const uint32_t*>(in);
      uint8_t* d = out + doff;
      for (uint32_t q = tid; q < uvis * pu; q += kCodecThreads) {
        const uint32_t e = R.ud[q >> (4 + uwl)], m = e & 0xffffu, j = (q & (pu - 1u)) >> uwl;
        if ((m >> j) & 1u) {
          const uint32_t w = in32[q];
          uint8_t* o = d + (size_t)((e >> 16) + __popc(m & ((1u << j) - 1u))) * g + 4 * (q & (uint32_t)((1 << uwl) - 1));
          o[0] = (uint8_t)w;
          o[1] = (uint8_t)(w >> 8);
          o[2] = (uint8_t)(w >> 16);
          o[3] = (uint8_t)(w >> 24);
        }
      }
    }
  }
  __syncthreads();
  return total;
}

// RZE_g decode: `in` (shared, any alignment) holds in_len payload bytes;
// reconstructs L bytes into `out` (shared, 16-byte aligned, room for L
// rounded up to 16g).  Returns the payload bytes consumed, or 0xffffffff if
// the payload is too short for what its bitmaps announce (corrupt).
//
// align = 0: all L bytes are written.  align > 0 (a multiple of 16g): B0 is
// zero past its last change when the last K0 byte is 0, so the units past
// it are all zero; only the bytes up to the next multiple of `align` after
// them are written (the rest of `out` is left as it was) and *act returns
// that length — the caller's bit planes past *act are zero.
//
// GIN: `in` is the payload in global memory (g = 1 only); every read stays
// below in_len, whatever the payload announces.
template <bool GIN = false>
__device__ uint32_t rze_dec(const uint8_t* in, uint32_t in_len, uint32_t L, int g, uint8_t* out, RzeScratch& R,
                            uint32_t align, uint32_t* act) {
  const int tid = threadIdx.x;
  const uint32_t n = L / (uint32_t)g;
  uint32_t sz[6];
  const int top = rze_sizes(n, sz);
  const uint32_t units = (n + 15) / 16, ub = 16u * (uint32_t)g;
  if (tid < 32) {
    // warp 0: the bitmap levels above B0, in registers (lane l holds the
    // bytes 8l..8l+7 of a level; every prefix count is eight ballots, not a
    // dependent shuffle chain), then the B1 words and their popcount prefix
    const int lane = tid;
    bool ok = sz[top] <= in_len;
    uint32_t pos = sz[top];
    uint32_t uact = units;
    if (ok && top >= 1) {
      unsigned long long b1v[2] = {0ull, 0ull};  // B1 bytes 8l.. (block 0) and 256 + 8l.. (block 1: sz1 > 256)
      if (top == 1) {
        if (lane == 0)
          for (uint32_t k = 0; k < sz[1]; ++k) b1v[0] |= (unsigned long long)rd8<GIN>(in, k) << (8 * k);
      } else {
        unsigned long long b2v = 0ull;  // B2 bytes 8l..8l+7
        if (top == 2) {
          if (lane == 0)
            for (uint32_t k = 0; k < sz[2]; ++k) b2v |= (unsigned long long)rd8<GIN>(in, k) << (8 * k);
        } else {  // top == 3: B2 from B3 (the top bytes) and K2
          const uint32_t bits = ((uint32_t)lane < sz[3] ? rd8<GIN>(in, lane) : 0u) & byte_mask(sz[2], 8u * lane);
          uint32_t k2n = 0;
          b2v = level_down_reg<GIN>(bits, in + pos, in_len - pos, k2n);
          pos += k2n;
          ok = ok && pos <= in_len;
        }
        if (ok) {
          uint32_t k1n = 0;
#pragma unroll
          for (int blk = 0; blk < 2; ++blk) {
            if (blk == 1 && sz[1] <= 256) break;
            const uint32_t bi = 32u * blk + lane;  // the B2 byte that selects B1 bytes 8 bi .. 8 bi + 7
            const unsigned long long src = __shfl_sync(0xffffffffu, b2v, (int)(bi >> 3));
            const uint32_t bits = (uint32_t)(src >> (8 * (bi & 7))) & byte_mask(sz[1], 8u * bi);
            b1v[blk] = level_down_reg<GIN>(bits, in + pos, in_len - pos, k1n);
          }
          pos += k1n;
          ok = ok && pos <= in_len;
        }
      }
      // B1 words 2 (32 blk + l), +1 (bits < sz0 only), their exclusive
      // popcount prefix, and the last set bit
      const uint32_t nw1 = (sz[0] + 31) / 32;
      uint32_t carry = 0;
      int last = -1;
#pragma unroll
      for (int blk = 0; blk < 2; ++blk) {
        if (blk == 1 && nw1 <= 64) break;
        const uint32_t w = 2u * (32u * blk + lane);
        const uint32_t w0 = (uint32_t)b1v[blk] & word_mask(sz[0], 32u * w);
        const uint32_t w1 = (uint32_t)(b1v[blk] >> 32) & word_mask(sz[0], 32u * (w + 1));
        const uint32_t c = __popc(w0) + __popc(w1);
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const uint32_t ex = carry + incl - c;
        if (w < nw1) {
          R.b1[w] = w0;
          R.pre1[w] = ex;
        }
        if (w + 1 < nw1) {
          R.b1[w + 1] = w1;
          R.pre1[w + 1] = ex + __popc(w0);
        }
        if (w1)
          last = (int)(32 * (w + 1)) + 31 - __clz(w1);
        else if (w0)
          last = (int)(32 * w) + 31 - __clz(w0);
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      last = __reduce_max_sync(0xffffffffu, last);
      const uint32_t koff = pos;
      pos += carry;  // |K0|
      ok = ok && pos <= in_len;
      // B0[t] = B0[last] for t >= last; when that byte is 0, units >= ceil(last / 2) are zero
      if (ok && align) uact = last < 0 ? 0u : (rd8<GIN>(in, pos - 1) == 0 ? ((uint32_t)last + 1) / 2 : units);
      if (lane == 0) R.info[0] = koff;
    }
    if (lane == 0) {
      R.info[1] = top == 0 ? sz[0] : pos;
      R.info[2] = ok;
      R.info[3] = uact;
    }
  }
  __syncthreads();
  if (!R.info[2]) {
    __syncthreads();
    return 0xffffffffu;
  }
  const uint32_t koff = R.info[0], doff = R.info[1], uact = R.info[3];
  // bytes written: the active units, then zeros up to the alignment
  const uint32_t wend = align ? min(units * ub, (uact * ub + align - 1) / align * align) : units * ub;
  for (uint32_t t = uact * ub / 16 + tid; t < wend / 16; t += kCodecThreads)
    reinterpret_cast<uint4*>(out)[t] = make_uint4(0, 0, 0, 0);
  if (act) *act = wend;
  constexpr int MAXIT = 5;
  const int iters = (int)((uact + kCodecThreads - 1) / kCodecThreads);
  // All units' masks first, then ONE block scan of the per-iteration data
  // counts packed into a u64 (13 bits for each of iterations 0-3: <= 4096;
  // 12 bits for iteration 4, which covers units 1024..1087: <= 1024), instead
  // of one scan (three block barriers) per 256 units.
  uint32_t mm[MAXIT];
  unsigned long long pk = 0;
#pragma unroll
  for (int it = 0; it < MAXIT; ++it) {
    mm[it] = 0;
    if (it >= iters) continue;
    const uint32_t u = (uint32_t)(it * kCodecThreads + tid);
    uint32_t m = 0;
    if (u < uact) {
      uint32_t lo, hi;
      const uint32_t t0 = 2 * u, t1 = 2 * u + 1;
      if (top == 0) {
        lo = t0 < sz[0] && t0 < in_len ? rd8<GIN>(in, t0) : 0u;
        hi = t1 < sz[0] && t1 < in_len ? rd8<GIN>(in, t1) : 0u;
      } else {
        const uint32_t w0 = R.b1[t0 >> 5];
        const uint32_t r0 = R.pre1[t0 >> 5] + __popc(w0 & ((2u << (t0 & 31)) - 1u));
        const uint32_t r1 = r0 + ((w0 >> (t1 & 31)) & 1u);  // t0, t1 share a B1 word
        lo = r0 ? rd8<GIN>(in, koff + r0 - 1) : 0u;
        hi = t1 < sz[0] ? (r1 ? rd8<GIN>(in, koff + r1 - 1) : 0u) : 0u;
      }
      m = lo | (hi << 8);
      if (16 * u + 16 > n) m &= (1u << (n - 16 * u)) - 1u;
    }
    mm[it] = m;
    pk += (unsigned long long)__popc(m) << (13 * it);
  }
  unsigned long long ptot;
  const unsigned long long pex = block_scan_excl<unsigned long long>(pk, R.wsum64, &ptot);
  const uint32_t running_all = (uint32_t)((ptot & 0x1fff) + ((ptot >> 13) & 0x1fff) + ((ptot >> 26) & 0x1fff) +
                                          ((ptot >> 39) & 0x1fff) + (ptot >> 52));
  const bool bad = doff + (uint32_t)g * running_all > in_len;  // block-uniform
  uint32_t running = 0;
#pragma unroll
  for (int it = 0; it < MAXIT; ++it) {
    if (it >= iters) break;
    const uint32_t u = (uint32_t)(it * kCodecThreads + tid);
    const uint32_t m = mm[it];
    const uint32_t field = it < 4 ? 0x1fffu : 0xfffu;
    uint32_t dr = running + (uint32_t)((pex >> (13 * it)) & field);
    running += (uint32_t)((ptot >> (13 * it)) & field);
    if (!bad && g == 1 && u < uact) {
      const uint8_t* src = in + doff;
      uint8_t* dst = out + u * ub;
      uint32_t w4[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if ((m >> j) & 1u) w4[j >> 2] |= rd8<GIN>(src, dr++) << (8 * (j & 3));
      *reinterpret_cast<uint4*>(dst) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    } else if (!bad && g != 1 && u < uact) {
      R.ud[u] = m | (dr << 16);  // g = 4 / 8: units <= 256, data ranks < 2^13
    }
  }
  if (!GIN && g != 1) {
    // g = 4 / 8: the active units' words are rebuilt 16 bytes per thread
    // step over the whole block (the units with data cluster in the first
    // bit planes; one unit per warp at a time left most warps idle at the
    // closing barrier)
    __syncthreads();
    if (!bad) {
      const int uwl = g == 4 ? 0 : 1;      // log2(u32 per word)
      const uint32_t q4 = 4u << uwl;       // 16-byte vectors per unit
      const uint8_t* src = in + doff;
      uint4* out4 = reinterpret_cast<uint4*>(out);
      for (uint32_t q = tid; q < uact * q4; q += kCodecThreads) {
        const uint32_t e = R.ud[q >> (2 + uwl)], m = e & 0xffffu, dr = e >> 16;
        const uint32_t o = (q & (q4 - 1u)) * 4u;  // first u32 of the vector within its unit
        uint32_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t j = (o + k) >> uwl, hh = (o + k) & (uint32_t)((1 << uwl) - 1);
          v[k] = 0;
          if ((m >> j) & 1u) {  // unaligned 4 bytes: two aligned words and a funnel shift
            const uintptr_t ad = reinterpret_cast<uintptr_t>(src) + (uintptr_t)(dr + __popc(m & ((1u << j) - 1u))) * g + 4 * hh;
            const uint32_t* w = reinterpret_cast<const uint32_t*>(ad & ~(uintptr_t)3);
            v[k] = __funnelshift_r(w[0], w[1], (uint32_t)(ad & 3) * 8u);
          }
        }
        out4[q] = make_uint4(v[0], v[1], v[2], v[3]);
      }
    }
  }
  __syncthreads();
  return bad ? 0xffffffffu : doff + (uint32_t)g * running;
}

// ---------------------------------------------------------------------------
// 32x32 bit-matrix transpose in registers: on return A[j] bit i = old A[i] bit j.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void transpose32(uint32_t (&A)[32]) {
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
    const uint32_t m = j == 16 ? 0x0000ffffu : j == 8 ? 0x00ff00ffu : j == 4 ? 0x0f0f0f0fu : j == 2 ? 0x33333333u : 0x55555555u;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if ((k & j) == 0) {
        uint32_t t = ((A[k] >> j) ^ A[k + j]) & m;
        A[k + j] ^= t;
        A[k] ^= t << j;
      }
    }
  }
}

template <typename U>
__host__ __device__ constexpr U nb_mask() {
  return (U)0xAAAAAAAAAAAAAAAAull;
}

// In-place BIT_k (G20) on one shared buffer (words swizzled -> planes
// linear): every (group, 32-bit half) item is staged in registers, then the
// block synchronises, then the results are stored.  With DIFF, word i is
// first replaced by NB(w[i] - w[i-1]) (DIFFNB_k, G18/G19), on the fly.
// Returns P (block-uniform): planes >= P are all zero.  Only planes < P are
// stored (rze_enc never reads past P planes: its L_act).  *pm is a zeroed
// shared word.  All threads must call.
template <typename U, bool DIFF>
__device__ __forceinline__ int bit_forward_inplace(uint8_t* buf, int W, unsigned long long* pm) {
  const int groups = W / 32, items = groups * (int)(sizeof(U) / 4);
  const int t = threadIdx.x, g = t % groups, half = t / groups;
  const U* words = reinterpret_cast<const U*>(buf);
  uint32_t A[32];
  uint32_t orv = 0;
  if (t < items) {
    if constexpr (sizeof(U) == 4) {  // 8 conflict-free 128-bit loads (swz<u32>)
      const uint4* w4 = reinterpret_cast<const uint4*>(buf);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 v = w4[8 * g + (j ^ (g & 7))];
        A[4 * j] = v.x, A[4 * j + 1] = v.y, A[4 * j + 2] = v.z, A[4 * j + 3] = v.w;
      }
      if (DIFF) {
        U prev = g ? words[swz<U>(32 * g - 1)] : (U)0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const U cur = A[i];
          A[i] = (uint32_t)(((U)(cur - prev) + nb_mask<U>()) ^ nb_mask<U>());
          prev = cur;
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) orv |= A[i];
    } else {  // (f64: the high-half items usually see all-zero words)
      U prev = (DIFF && g) ? words[swz<U>(32 * g - 1)] : (U)0;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        U w = words[swz<U>(32 * g + i)];
        if (DIFF) {
          const U cur = w;
          w = (U)(((U)(cur - prev) + nb_mask<U>()) ^ nb_mask<U>());
          prev = cur;
        }
        A[i] = (uint32_t)(w >> (32 * half));
        orv |= A[i];
      }
    }
    if (sizeof(U) == 4 || orv) transpose32(A);  // f64: all-zero high halves are their own transpose
  }
  // warps lie within one half (groups is a multiple of 32)
  orv = __reduce_or_sync(0xffffffffu, orv);
  if ((t & 31) == 0 && orv) atomicOr(pm, (unsigned long long)orv << (32 * (t < items ? half : 0)));
  __syncthreads();
  const unsigned long long m = *pm;
  const int P = m ? 64 - __clzll((long long)m) : 0;
  if (t < items) {
    uint32_t* planes = reinterpret_cast<uint32_t*>(buf);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (32 * half + j >= P) break;
      planes[(32 * half + j) * groups + g] = A[j];
    }
  }
  __syncthreads();
  return P;
}

// BIT_k of words whose planes >= P are zero, P <= 8 (the usual subbin
// chunk: subbins are small): warp w transposes the groups [GPW w, GPW w + GPW)
// with one warp ballot per (group, plane); lane k keeps the planes of group
// GPW w + k, so the plane stores are conflict-free.  In place, all threads.
template <typename U, int P>
__device__ __forceinline__ void bit_forward_ballot_p(uint8_t* buf, int W) {
  constexpr int NW = kCodecThreads / 32;
  const int groups = W / 32, gpw = groups / NW;  // 16 (f32) / 8 (f64)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const U* words = reinterpret_cast<const U*>(buf);
  uint32_t m[P > 0 ? P : 1];
#pragma unroll
  for (int j = 0; j < P; ++j) m[j] = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (k < gpw) {
      const uint32_t w = (uint32_t)words[swz<U>(32 * (gpw * warp + k) + lane)];
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const uint32_t v = __ballot_sync(0xffffffffu, (w & (1u << j)) != 0u);
        m[j] = lane == k ? v : m[j];
      }
    }
  }
  __syncthreads();
  uint32_t* planes = reinterpret_cast<uint32_t*>(buf);
  if (lane < gpw) {
#pragma unroll
    for (int j = 0; j < P; ++j) planes[j * groups + gpw * warp + lane] = m[j];
  }
  __syncthreads();
}

template <typename U>
__device__ __forceinline__ void bit_forward_ballot(uint8_t* buf, int W, int P) {
  switch (P) {
    case 0: bit_forward_ballot_p<U, 0>(buf, W); break;
    case 1: bit_forward_ballot_p<U, 1>(buf, W); break;
    case 2: bit_forward_ballot_p<U, 2>(buf, W); break;
    case 3: bit_forward_ballot_p<U, 3>(buf, W); break;
    case 4: bit_forward_ballot_p<U, 4>(buf, W); break;
    case 5: bit_forward_ballot_p<U, 5>(buf, W); break;
    case 6: bit_forward_ballot_p<U, 6>(buf, W); break;
    case 7: bit_forward_ballot_p<U, 7>(buf, W); break;
    default: bit_forward_ballot_p<U, 8>(buf, W); break;
  }
}

// Inverse BIT_k: planes (linear, `pb`) -> words (swizzled, `wb`); planes >= P
// are zero and not read.  INPLACE (pb == wb): all loads, barrier, all
// stores; out of place there is no barrier between them, so the 32 staged
// words are not live across one.
// All threads must call.
template <typename U, bool INPLACE>
__device__ __forceinline__ void bit_inverse_inplace(const uint8_t* pb, uint8_t* wb, int W, int P) {
  const int groups = W / 32, items = groups * (int)(sizeof(U) / 4);
  const int t = threadIdx.x, g = t % groups, half = t / groups;
  uint32_t A[32];
  if (t < items) {
    const uint32_t* planes = reinterpret_cast<const uint32_t*>(pb);
#pragma unroll
    for (int j = 0; j < 32; ++j) A[j] = 32 * half + j < P ? planes[(32 * half + j) * groups + g] : 0u;
    if (sizeof(U) == 4 || 32 * half < P) transpose32(A);  // f64 high half with no planes: zeros
  }
  if (INPLACE) __syncthreads();
  if (t < items) {
    if constexpr (sizeof(U) == 4) {  // 8 conflict-free 128-bit stores (swz<u32>)
      uint4* w4 = reinterpret_cast<uint4*>(wb);
#pragma unroll
      for (int j = 0; j < 8; ++j) w4[8 * g + (j ^ (g & 7))] = make_uint4(A[4 * j], A[4 * j + 1], A[4 * j + 2], A[4 * j + 3]);
    } else {
      uint32_t* w32 = reinterpret_cast<uint32_t*>(wb);
#pragma unroll
      for (int i = 0; i < 32; ++i) w32[swz<U>(32 * g + i) * 2 + half] = A[i];
    }
  }
  __syncthreads();
}

// The same for P <= 3 (the usual subbin chunk) without transposes: lane l of
// warp w builds word 32 g + l of its groups g from bit l of the P plane words
// (broadcast loads).  All threads must call.
template <typename U, int P, bool INPLACE>
__device__ __forceinline__ void bit_inverse_small_p(const uint8_t* pb, uint8_t* wb, int W) {
  constexpr int NW = kCodecThreads / 32;
  const int groups = W / 32, gpw = groups / NW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* planes = reinterpret_cast<const uint32_t*>(pb);
  uint32_t wv[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    wv[k] = 0;
    if (k < gpw) {
      const int g = gpw * warp + k;
#pragma unroll
      for (int j = 0; j < P; ++j) wv[k] |= ((planes[j * groups + g] >> lane) << j) & (1u << j);
    }
  }
  if (INPLACE) __syncthreads();
  U* words = reinterpret_cast<U*>(wb);
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (k < gpw) words[swz<U>(32 * (gpw * warp + k) + lane)] = (U)wv[k];
  __syncthreads();
}

template <typename U, bool INPLACE>
__device__ __forceinline__ void bit_inverse_planes(const uint8_t* pb, uint8_t* wb, int W, int P) {
  switch (P) {
    case 0: bit_inverse_small_p<U, 0, INPLACE>(pb, wb, W); break;
    case 1: bit_inverse_small_p<U, 1, INPLACE>(pb, wb, W); break;
    case 2: bit_inverse_small_p<U, 2, INPLACE>(pb, wb, W); break;
    case 3: bit_inverse_small_p<U, 3, INPLACE>(pb, wb, W); break;
    default: bit_inverse_inplace<U, INPLACE>(pb, wb, W, P); break;
  }
}

// ---------------------------------------------------------------------------
// k_encode
// ---------------------------------------------------------------------------
struct EncodeArgs {
  const uint32_t* cesc;  // planes mode: bit c set when chunk c holds an escape (from k_quant_flags); null = read every escape word
  uint64_t sp_off;       // planes mode: plane-grid index of element 0 (slab mode: the owned range's offset in the box)
  const void* x;
  const uint32_t* s;
  uint8_t* stage;    // C x 32 KiB staging slots (workspace)
  uint32_t* sizes;   // 2C: (bin_size, sub_size)
  Counters* ctr;
  double eps, inv;
  uint64_t n;
  uint32_t C;
  int ndims;
  int vec;  // x and s are 16-byte aligned: vector loads allowed
  float inv32;  // RN32(1/eps) for the f32 fast path, NaN = off
  int prof;     // diagnostic phase clocks
  uint64_t d0, d1, d2;
  double xlim;   // |x| < xlim proves x regular (finite, |b| <= BINMAX): the subbin CTAs' escape test
  float xlim32;  // the same bound as a float (f32 data)
  // Subbin planes (tile engine, lopc_tiles.cuh): 8 u32 per 32-point x-segment
  // (word b = bit b of the segment's 32 subbins); null: u32 subbins in s.
  // With planes, the escape bits come from word sw - 2 of each flag segment
  // (k_quant_flags) and the bound self-check a4 runs in the bin
  // CTAs, which hold x and the bins already: the subbin CTAs read no x.
  const uint32_t* sp;
  const uint32_t* flags;  // flag segments: word sw - 2 holds the escape bits (k_quant_flags)
  int64_t nseg;
  int sw;
};

// Subbin planes b0 .. b0+NPL-1 (and, with ESC, the escape bits) of the 32
// linear elements starting at row `row`, column x (bits past n are 0): one
// x-segment when rows are whole segments (d2 a multiple of 32), else up to
// three segment pieces across a row end.  `left` = n - (linear index of the
// first element).
template <int NPL>
__device__ __forceinline__ void gather_group(const EncodeArgs& a, uint64_t row, uint32_t x, uint64_t left, int b0,
                                             bool want_esc, uint32_t (&pl)[NPL], uint32_t& esc) {
#pragma unroll
  for (int b = 0; b < NPL; ++b) pl[b] = 0;
  esc = 0;
  const uint32_t d2 = (uint32_t)a.d2;
  if ((d2 & 31) == 0) {
    // rows are whole segments: the group IS segment (row * nseg + x / 32)
    if (left == 0) return;
    const size_t rs = (size_t)row * (size_t)a.nseg + (x >> 5);
    if constexpr (NPL == 4) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.sp + rs * 8 + b0));
      pl[0] = v.x, pl[1] = v.y, pl[2] = v.z, pl[3] = v.w;
    } else {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(a.sp + rs * 8 + b0));
      pl[0] = v.x, pl[1] = v.y;
    }
    if (want_esc) esc = __ldg(a.flags + rs * (size_t)a.sw + (a.sw - 2));
    return;  // (n is a multiple of 32 here: no partial group)
  }
  if (d2 >= 32) {
    // at most three pieces (the rest of a segment, the row's end, the next
    // row's start): every load is issued before any is used
    uint32_t o[3], bit[3], m[3];
    size_t rs[3];
    bool on[3];
    uint32_t oo = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      on[k] = oo < 32 && left > 0;
      const uint32_t sg = x >> 5, bt = x & 31;
      uint32_t take = 32 - bt < 32 - oo ? 32 - bt : 32 - oo;
      if (d2 - x < take) take = d2 - x;
      if (left < take) take = (uint32_t)left;
      if (!on[k]) take = 0;
      o[k] = oo;
      bit[k] = bt;
      m[k] = take >= 32 ? 0xffffffffu : ((1u << take) - 1u);
      rs[k] = (size_t)row * (size_t)a.nseg + sg;
      oo += take;
      left -= take;
      x += take;
      if (x == d2) {
        x = 0;
        ++row;
      }
    }
    uint32_t w[3][NPL], e[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      e[k] = 0;
#pragma unroll
      for (int b = 0; b < NPL; ++b) w[k][b] = 0;
      if (on[k]) {
        if constexpr (NPL == 4) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.sp + rs[k] * 8 + b0));
          w[k][0] = v.x, w[k][1] = v.y, w[k][2] = v.z, w[k][3] = v.w;
        } else {
          static_assert(NPL == 2, "2 or 4 planes per thread");
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(a.sp + rs[k] * 8 + b0));
          w[k][0] = v.x, w[k][1] = v.y;
        }
        if (want_esc) e[k] = __ldg(a.flags + rs[k] * (size_t)a.sw + (a.sw - 2));
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
      for (int b = 0; b < NPL; ++b) pl[b] |= ((w[k][b] >> bit[k]) & m[k]) << o[k];
      esc |= ((e[k] >> bit[k]) & m[k]) << o[k];
    }
    return;
  }
  for (uint32_t o = 0; o < 32 && left > 0;) {  // rows shorter than a segment: one piece per row
    const uint32_t seg = x >> 5, bit = x & 31;
    uint32_t take = 32 - bit < 32 - o ? 32 - bit : 32 - o;
    if (d2 - x < take) take = d2 - x;
    if (left < take) take = (uint32_t)left;
    const uint32_t m = take >= 32 ? 0xffffffffu : ((1u << take) - 1u);
    const size_t rs = (size_t)row * (size_t)a.nseg + seg;
    uint32_t w[NPL];
    if constexpr (NPL == 4) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.sp + rs * 8 + b0));
      w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
    } else {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(a.sp + rs * 8 + b0));
      w[0] = v.x, w[1] = v.y;
    }
#pragma unroll
    for (int b = 0; b < NPL; ++b) pl[b] |= ((w[b] >> bit) & m) << o;
    if (want_esc) esc |= ((__ldg(a.flags + rs * (size_t)a.sw + (a.sw - 2)) >> bit) & m) << o;
    o += take;
    left -= take;
    x += take;
    if (x == d2) {
      x = 0;
      ++row;
    }
  }
}

// One element's subbin from the planes (the raw-fallback rebuild; rare).
__device__ __forceinline__ uint32_t subbin_at(const EncodeArgs& a, uint64_t i) {
  const uint64_t row = i / a.d2, x = i - row * a.d2;
  const uint32_t* p = a.sp + ((size_t)row * (size_t)a.nseg + (x >> 5)) * 8;
  uint32_t v = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) v |= ((__ldg(p + b) >> (x & 31)) & 1u) << b;
  return v;
}

// xlim = 2^30 eps (f32 data) / 2^49 eps (f64): |x| below it gives |x/eps| < 2^30
// (2^49), so |b| <= 2^30 < BINMAX = 2^31 - 2 (|b| <= 2^49 < 2^50), and x is
// finite.  xlim32 rounds 2^30 eps down to a float (FLT_MAX if larger; 0 if it
// underflows, which only sends every point to the exact test).
inline void set_escape_limits(EncodeArgs& ea, bool f64, double eps) {
  ea.xlim = ldexp(eps, f64 ? 49 : 30);
  const double l = ldexp(eps, 30);
  float f = l >= 3.4028234663852886e38 ? 3.4028234663852886e38f : (float)l;
  if ((double)f > l) f = nextafterf(f, 0.0f);
  ea.xlim32 = f;
}

__device__ __forceinline__ bool surely_regular(float x, const EncodeArgs& a) { return fabsf(x) < a.xlim32; }
__device__ __forceinline__ bool surely_regular(double x, const EncodeArgs& a) { return fabs(x) < a.xlim; }


constexpr uint64_t kFlagAgg = 1ull << 62, kFlagIncl = 2ull << 62, kValMask = (1ull << 62) - 1;

// Decoupled look-back, one warp: publish this chunk's aggregate, then sum the
// predecessors 32 at a time (lane i looks at chunk c-1-i) until the nearest
// inclusive prefix is found; publish the inclusive prefix.  Returns the
// exclusive prefix in every lane.  Forward progress: chunk ids come from a
// ticket in scheduling order, so every predecessor is already running.
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* state, uint32_t c, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (c == 0) {
    if (lane == 0) st_release_u64(&state[0], kFlagIncl | agg);
    return 0;
  }
  if (lane == 0) st_release_u64(&state[c], kFlagAgg | agg);
  uint64_t excl = 0;
  int64_t base = (int64_t)c - 1;
  for (;;) {
    const int64_t i = base - lane;
    const uint64_t v = i >= 0 ? ld_acquire_u64(&state[i]) : kFlagIncl;
    const uint32_t incl = __ballot_sync(0xffffffffu, (v >> 62) == 2);
    const uint32_t none = __ballot_sync(0xffffffffu, (v >> 62) == 0);
    const int first = incl ? __ffs(incl) - 1 : 31;
    const uint32_t need = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
    if (none & need) continue;  // a predecessor has not published yet
    uint64_t part = lane <= first ? (v & kValMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    excl += part;
    if (incl) break;
    base -= 32;
  }
  if (lane == 0) st_release_u64(&state[c], kFlagIncl | (excl + agg));
  return excl;
}

__device__ __forceinline__ uint32_t pad4(uint32_t v) { return (v + 3u) & ~3u; }

// One CTA per (chunk, stream): k_encode<T, 1> encodes the bins of chunk
// blockIdx.x, k_encode<T, 2> its subbins.
struct EncSmem {
  alignas(16) uint8_t Wd[kChunkBytes + 64];  // words -> planes (in place) -> [subbins] payload
  alignas(16) uint8_t O[17408 + 128];        // [bins] payload | [subbins] a4 queue, RZE_k output
  RzeScratch R;
  unsigned long long pm[2];                  // OR of the words (subbins) / plane mask of BIT
  uint32_t misc[4];
  unsigned long long row0;                   // planes mode: (row, x) of the chunk's first element
  uint32_t x0;
};

template <typename T, int ROLE>
__device__ __forceinline__ void encode_chunk_role(const EncodeArgs& a, const uint32_t c, uint8_t* smem_raw) {
  using U = typename VT<T>::U;
  using I = typename VT<T>::I;
  constexpr bool SUBS = ROLE == 2;
  constexpr int K = VT<T>::K;
  constexpr int W = kChunkBytes / K;
  constexpr int PER = W / kCodecThreads;  // words per thread (16 f32, 8 f64)
  constexpr int PB = W / 8;               // bytes per bit plane
  EncSmem& sm = *reinterpret_cast<EncSmem*>(smem_raw);
  U* WD = reinterpret_cast<U*>(sm.Wd);
  uint16_t* Q = reinterpret_cast<uint16_t*>(sm.O);
  const int tid = threadIdx.x, lane = tid & 31;
  PhaseClock pc;
  pc.start(a.prof);
  if (tid == 0) {
    sm.misc[0] = 0;  // a4 queue length
    sm.pm[0] = 0;
    sm.pm[1] = 0;
  }
  const uint64_t e0 = (uint64_t)c * W;
  const uint32_t cnt = (uint32_t)min((uint64_t)W, a.n - e0);
  const T* X = static_cast<const T*>(a.x) + e0;
#if LOPC_ENC_PF
  // f64 bin role: the chunk's x requested from DRAM now (into L2, no
  // registers), so its loads after the plane gather hit L2 (cfg5 encode
  // 12.51 -> 12.25 ms; for f32 it measured 1 % slower, so not there)
  if (!SUBS && sizeof(T) == 8 && (uint32_t)tid < (uint32_t)(cnt * sizeof(T) + 127) / 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(X) + 128 * tid));
#endif
  const uint32_t* S = a.s + e0;
  constexpr int G = W / 32;  // 32-element groups of the chunk
  uint32_t* PL = reinterpret_cast<uint32_t*>(sm.O);  // planes mode: [b * G + g] subbin planes, [8G + g] escapes
  if (tid == 0) {
    sm.misc[1] = 0;  // OR over the chunk of the plane-nonzero masks
    sm.misc[2] = 0;  // any escape in the chunk
    if (a.sp) {      // (row, x) of the chunk's first element: one 64-bit division per CTA
      sm.row0 = (e0 + a.sp_off) / a.d2;
      sm.x0 = (uint32_t)(e0 + a.sp_off - sm.row0 * a.d2);
    }
  }
  __syncthreads();
  if (a.sp) {  // gather the chunk's subbin planes and escape bits (both roles)
    // all threads: group g = tid mod G, planes [b0, b0 + NPL) (f32: 2 x 4
    // planes, f64: 4 x 2 planes per group); the first thread of a group
    // also takes its escape bits.  The group's (row, x): one 64-bit division
    // per CTA, then 32-bit steps (rows of d2 < 2^32 points).
    constexpr int NPL = 8 * G / kCodecThreads;
    const int g = tid % G, b0 = (tid / G) * NPL;
    const uint64_t r0 = sm.row0;
    const uint32_t xg = sm.x0 + 32u * (uint32_t)g, d2 = (uint32_t)a.d2;
    const uint32_t dr = xg / d2;
    const uint64_t i0 = e0 + 32ull * g;
    uint32_t pl[NPL], esc;
    // (the escape words only in chunks that hold an escape: k_quant_flags
    // marks them; a 32-byte sector per segment otherwise.  No chunk bits
    // (slab mode): every chunk reads them)
    const bool esc_chunk = !a.cesc || ((a.cesc[c >> 5] >> (c & 31)) & 1u);
    gather_group<NPL>(a, r0 + dr, xg - dr * d2, i0 < a.n ? a.n - i0 : 0, b0, SUBS && b0 == 0 && esc_chunk, pl, esc);
    uint32_t nzp = 0;
#pragma unroll
    for (int b = 0; b < NPL; ++b) {
      PL[(b0 + b) * G + g] = pl[b];
      nzp |= (uint32_t)(pl[b] != 0u) << (b0 + b);
    }
    if (b0 == 0) PL[8 * G + g] = esc;
    nzp = __reduce_or_sync(0xffffffffu, nzp);
    const uint32_t ae = __reduce_or_sync(0xffffffffu, esc);
    if (lane == 0) {
      if (nzp) atomicOr(&sm.misc[1], nzp);
      if (ae) atomicOr(&sm.misc[2], 1u);
    }
    __syncthreads();
    pc.mark(a.ctr, 0);
  }

  // --- a1: re-quantize; bin words (ROLE 1) or subbin words + a4 queue (ROLE 2).
  // Thread slot k = 4v + q holds element 4 (v * NT + tid) + q.  Elements past
  // the chunk's end load as x = 0, s = 0, whose words are 0 (b(0) = 0), the
  // zero padding of G23.
  constexpr int NV = PER / 2;  // two halves of PER slots (register budget)
  uint32_t qmask = 0, nesc = 0, bad4 = 0;
  const uint32_t pmk = sm.misc[1];
  const int npl = pmk ? 32 - __clz(pmk) : 0;  // planes mode: non-zero subbin planes of the chunk
  U orw = 0;
#pragma unroll 1
  for (int hh = 0; hh < ((SUBS && a.sp) ? 0 : 2); ++hh) {
    T xs[NV];
    uint32_t ss[NV];
    if (a.vec && cnt == (uint32_t)W) {
#pragma unroll
      for (int v = 0; v < NV / 4; ++v) {
        const int i0 = 4 * ((hh * (NV / 4) + v) * kCodecThreads + tid);
        if constexpr (sizeof(T) == 4) {
          const float4 xv = __ldg(reinterpret_cast<const float4*>(X + i0));
          xs[4 * v] = xv.x, xs[4 * v + 1] = xv.y, xs[4 * v + 2] = xv.z, xs[4 * v + 3] = xv.w;
        } else {
          const double2 x0 = __ldg(reinterpret_cast<const double2*>(X + i0));
          const double2 x1 = __ldg(reinterpret_cast<const double2*>(X + i0 + 2));
          xs[4 * v] = x0.x, xs[4 * v + 1] = x0.y, xs[4 * v + 2] = x1.x, xs[4 * v + 3] = x1.y;
        }
        if constexpr (SUBS) {
          const uint4 sv = __ldg(reinterpret_cast<const uint4*>(S + i0));
          ss[4 * v] = sv.x, ss[4 * v + 1] = sv.y, ss[4 * v + 2] = sv.z, ss[4 * v + 3] = sv.w;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int i = 4 * ((hh * (NV / 4) + (k >> 2)) * kCodecThreads + tid) + (k & 3);
        const bool in = (uint32_t)i < cnt;
        xs[k] = in ? X[i] : (T)0;
        if constexpr (SUBS) ss[k] = in ? S[i] : 0u;
      }
    }
#pragma unroll
    for (int v = 0; v < NV / 4; ++v) {
      U wv[4];
      if constexpr (!SUBS) {  // fast attempt, rare exact fix-up (near a half-integer, escapes, huge bins)
        I bb[4];
        uint32_t slow = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) slow |= (uint32_t)!qtry(xs[4 * v + q], a.inv32, a.inv, bb[q]) << q;
#pragma unroll
        for (int q = 0; q < 4; ++q) wv[q] = (U)bb[q];
        if (slow) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if ((slow >> q) & 1u) {
              const int64_t r = quantize_slow<T>(xs[4 * v + q], a.eps, a.inv);
              nesc += r == kEscape;
              wv[q] = r == kEscape ? VT<T>::kSentinel : (U)(I)r;
            }
          }
        }
        if (a.sp && npl) {
          // a4 (planes mode), here where x and the bins are in registers:
          // key(lo(b)) + s <= key(x) for the elements with s > 0 (proof (i),
          // S:151-159).  The 4 subbins as bytes of s4: plane b's nibble of
          // the 4 elements spread to bit b of each byte (bit q -> bit 8q by
          // one multiply: q + 7q, no carries).
          const int e4 = 4 * ((hh * (NV / 4) + v) * kCodecThreads + tid);
          const uint32_t g = (uint32_t)e4 >> 5, sh = (uint32_t)e4 & 31u;
          uint32_t s4 = 0;
          for (int b = 0; b < npl; ++b) s4 |= ((((PL[b * G + g] >> sh) & 0xfu) * 0x00204081u) & 0x01010101u) << b;
          if (s4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t sq = (s4 >> (8 * q)) & 0xffu;
              if (sq) {
                if (wv[q] == VT<T>::kSentinel)
                  bad4 = 1;  // an escaped point has no arcs, so no subbin
                else if ((int64_t)lo_key<T>((int64_t)(I)wv[q], a.eps) + (int64_t)sq >
                         (int64_t)key_of((U)as_bits(xs[4 * v + q])))
                  bad4 = 1;
              }
            }
          }
        }
      } else {  // escape test only: |x| < xlim proves the point regular
        uint32_t slow = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          slow |= (uint32_t)!surely_regular(xs[4 * v + q], a) << q;
          wv[q] = (U)ss[4 * v + q];
        }
        if (slow) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (((slow >> q) & 1u) && quantize_slow<T>(xs[4 * v + q], a.eps, a.inv) == kEscape) {
              wv[q] = (U)as_bits(xs[4 * v + q]);
              ss[4 * v + q] = 0;  // not queued for a4
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          qmask |= (uint32_t)(ss[4 * v + q] != 0) << (hh * NV + 4 * v + q);
          orw |= wv[q];
        }
      }
      const int i4 = 4 * ((hh * (NV / 4) + v) * kCodecThreads + tid);
      if constexpr (sizeof(U) == 4) {
        *reinterpret_cast<uint4*>(&WD[swz<U>(i4)]) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) WD[swz<U>(i4 + q)] = wv[q];
      }
    }
  }
  if constexpr (SUBS) {  // a4 queue: one warp scan per thread-mask; OR of the words
    const uint32_t nq = __popc(qmask);
    uint32_t incl = nq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t base = 0;
    if (lane == 31 && incl) base = atomicAdd(&sm.misc[0], incl);
    base = __shfl_sync(0xffffffffu, base, 31) + incl - nq;
    for (uint32_t m = qmask; m; m &= m - 1) {
      const int k = __ffs(m) - 1;
      Q[base++] = (uint16_t)(4 * ((k >> 2) * kCodecThreads + tid) + (k & 3));
    }
    const uint32_t olo = __reduce_or_sync(0xffffffffu, (uint32_t)orw);
    const uint32_t ohi = sizeof(U) == 8 ? __reduce_or_sync(0xffffffffu, (uint32_t)((uint64_t)orw >> 32)) : 0u;
    if (lane == 0 && (olo | ohi)) atomicOr(&sm.pm[0], ((unsigned long long)ohi << 32) | olo);
  } else {
    const uint32_t esc = __reduce_add_sync(0xffffffffu, nesc);
    if (lane == 0 && esc) atomicAdd(&a.ctr->escapes, (unsigned long long)esc);
    if (__any_sync(0xffffffffu, bad4) && lane == 0) atomicOr(&a.ctr->err, kErrBound);
  }
  if (SUBS && a.sp && sm.misc[2]) {
    // planes mode, a chunk with escapes: words = subbins from the planes,
    // raw bits of x at the escapes (the only x this CTA reads)
    for (int i = tid; i < W; i += kCodecThreads) {
      const int g = i >> 5, bit = i & 31;
      uint32_t sv = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) sv |= ((PL[b * G + g] >> bit) & 1u) << b;
      const U w = ((PL[8 * G + g] >> bit) & 1u) ? (U)as_bits(X[i]) : (U)sv;
      WD[swz<U>(i)] = w;
      orw |= w;
    }
    const uint32_t olo = __reduce_or_sync(0xffffffffu, (uint32_t)orw);
    const uint32_t ohi = sizeof(U) == 8 ? __reduce_or_sync(0xffffffffu, (uint32_t)((uint64_t)orw >> 32)) : 0u;
    if (lane == 0 && (olo | ohi)) atomicOr(&sm.pm[0], ((unsigned long long)ohi << 32) | olo);
  }
  __syncthreads();
  pc.mark(a.ctr, 1);


  uint32_t size;
  if constexpr (SUBS) {
    // --- a4: bound self-check of the queued points: key(lo(b)) + s <= key(x)
    const uint32_t nq = sm.misc[0];
    uint32_t bad = 0;
    for (uint32_t q = tid; q < nq; q += kCodecThreads) {
      const int i = Q[q];
      const T x = X[i];
      I b = 0;
      if (!qtry(x, a.inv32, a.inv, b)) b = (I)quantize_slow<T>(x, a.eps, a.inv);
      const uint32_t sq = (uint32_t)WD[swz<U>(i)];
      if ((int64_t)lo_key<T>((int64_t)b, a.eps) + (int64_t)sq > (int64_t)key_of((U)as_bits(x))) bad = 1;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&a.ctr->err, kErrBound);
    pc.mark(a.ctr, 2);
    // --- a6: subbins: BIT_k -> RZE_k -> RZE_1 ----------------------
    int P;
    if (a.sp && !sm.misc[2]) {
      // planes mode without escapes: BIT_k of the subbin words IS the
      // gathered planes (planes >= 8 are zero): copy the P non-zero ones
      const uint32_t pmk = sm.misc[1];
      P = pmk ? 32 - __clz(pmk) : 0;
      uint32_t* planes = reinterpret_cast<uint32_t*>(sm.Wd);
      for (int t = tid; t < P * G; t += kCodecThreads) planes[t] = PL[t];
      __syncthreads();
    } else {
      const unsigned long long ow = sm.pm[0];
      P = ow ? 64 - __clzll((long long)ow) : 0;
      if (P <= 8)
        bit_forward_ballot<U>(sm.Wd, W, P);
      else
        P = bit_forward_inplace<U, false>(sm.Wd, W, &sm.pm[1]);
    }
    pc.mark(a.ctr, 3);
    const uint32_t l1 = rze_enc(sm.Wd, kChunkBytes, K, sm.O, 0xffffffffu, sm.R, (uint32_t)P * PB);
    for (uint32_t t = l1 + tid; t < ((l1 + 15) & ~15u) + 16; t += kCodecThreads) sm.O[t] = 0;
    __syncthreads();
    pc.mark(a.ctr, 5);
    const uint32_t l2 = rze_enc(sm.O, l1, 1, sm.Wd + 2, kChunkBytes - 6, sm.R, (l1 + 15) & ~15u);
    size = l2 <= kChunkBytes - 6 ? pad4(2 + l2) : kChunkBytes;
    if (size < kChunkBytes) {
      if (tid == 0) {
        sm.Wd[0] = (uint8_t)(l1 & 0xffu);
        sm.Wd[1] = (uint8_t)(l1 >> 8);
      }
      if ((uint32_t)tid < size - 2 - l2) sm.Wd[2 + l2 + tid] = 0;
    }
    pc.mark(a.ctr, 6);
  } else {
    // --- a5: bins: DIFFNB_k -> BIT_k -> RZE_1 -------------------
    const int P = bit_forward_inplace<U, true>(sm.Wd, W, &sm.pm[1]);
    pc.mark(a.ctr, 3);
    const uint32_t l = rze_enc(sm.Wd, kChunkBytes, 1, sm.O, kChunkBytes - 4, sm.R, (uint32_t)P * PB);
    size = l <= kChunkBytes - 4 ? pad4(l) : kChunkBytes;
    if (size < kChunkBytes && (uint32_t)tid < size - l) sm.O[l + tid] = 0;
    pc.mark(a.ctr, 4);
  }
  __syncthreads();

  // --- a7 (part 1): the payload goes to this chunk's staging slot (bins at
  // +0, subbins at +16 KiB); k_chunk_scan + k_place put it in the stream.
  if (tid == 0) {
    a.sizes[2 * c + (SUBS ? 1 : 0)] = size;
    atomicAdd(SUBS ? &a.ctr->sub_bytes : &a.ctr->bin_bytes, (unsigned long long)size);
  }
  uint32_t* dst = reinterpret_cast<uint32_t*>(a.stage + (size_t)c * 2 * kChunkBytes + (SUBS ? kChunkBytes : 0));
  if (size == kChunkBytes) {
    // raw fallback (G23): rebuild the words (the buffer now holds planes)
    for (int i = tid; i < W; i += kCodecThreads) {
      U w = 0;
      if ((uint32_t)i < cnt) {
        I b;
        if (quantize_fast<T>(X[i], a.inv32, a.eps, a.inv, b))
          w = SUBS ? (U)(a.sp ? subbin_at(a, a.sp_off + e0 + (uint64_t)i) : S[i]) : (U)b;
        else
          w = SUBS ? (U)as_bits(X[i]) : VT<T>::kSentinel;
      }
#pragma unroll
      for (int h = 0; h < K / 4; ++h) dst[i * (K / 4) + h] = (uint32_t)(w >> (32 * h));
    }
  } else {
    const uint4* src = reinterpret_cast<const uint4*>(SUBS ? sm.Wd : sm.O);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (uint32_t i = tid; i < (size + 15) / 16; i += kCodecThreads) d4[i] = src[i];
  }
  __syncthreads();
  pc.mark(a.ctr, 7);
}

template <typename T, int ROLE>
__global__ void __launch_bounds__(kCodecThreads, ROLE == 2 ? LOPC_SUBS_CTAS : LOPC_CODEC_CTAS) k_encode(EncodeArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  encode_chunk_role<T, ROLE>(a, blockIdx.x, smem_raw);
}

// Host: one k_encode grid of C CTAs for one stream (role 1 bins, 2 subbins).
inline void launch_encode(const EncodeArgs& ea, bool f64, int role, unsigned C, size_t smem, cudaStream_t st) {
  if (C == 0) return;
  if (!f64)
    (role == 1 ? k_encode<float, 1> : k_encode<float, 2>)<<<C, kCodecThreads, smem, st>>>(ea);
  else
    (role == 1 ? k_encode<double, 1> : k_encode<double, 2>)<<<C, kCodecThreads, smem, st>>>(ea);
}

// ---------------------------------------------------------------------------
// k_chunk_scan: a7 (part 2), the one prefix sum of the stream format: chunk
// payload offsets = exclusive scan of (bin_size + sub_size).  Decoupled
// look-back over tiles of 2048 chunks (each tile's aggregate is available at
// once, so the look-back never waits long).  In decode mode the sizes come
// from the stream's table and are validated.
// ---------------------------------------------------------------------------
#ifndef LOPC_SCAN_THREADS
#define LOPC_SCAN_THREADS 512
#endif
#ifndef LOPC_SCAN_PER
#define LOPC_SCAN_PER 4
#endif
constexpr int kScanThreads = LOPC_SCAN_THREADS;
constexpr int kScanPer = LOPC_SCAN_PER;
constexpr int kScanTile = kScanThreads * kScanPer;

struct ScanArgs {
  const uint32_t* sizes;  // 2C u32: (bin_size, sub_size) pairs (encode mode)
  const uint8_t* in;      // decode mode: the stream (C and the table come from it)
  uint64_t in_bytes;
  uint32_t C;             // encode mode
  uint64_t* off;          // out: C payload offsets
  uint64_t* state;        // per-tile look-back state (zeroed)
  Counters* ctr;
  int validate;           // decode: check 4 <= size <= 16384, size % 4 == 0
  uint64_t expect_total;  // decode: the stream length
  uint64_t base;          // sizes mode: offset of the first payload (64 + 8C, or 0 / 8C in slab mode)
};

__global__ void __launch_bounds__(kScanThreads) k_chunk_scan(ScanArgs a) {
  __shared__ unsigned long long wsum[32];
  __shared__ unsigned long long excl_s;
  __shared__ uint32_t tile_s;
  __shared__ uint32_t C_s;
  const int tid = threadIdx.x;
  if (tid == 0) {
    tile_s = atomicAdd(&a.ctr->ticket2, 1u);
    uint32_t C = a.C;
    if (a.in) {  // decode: C from the header, bounded by the stream length
      C = 0;
      if (a.in_bytes >= kHdrBytes && reinterpret_cast<const uint32_t*>(a.in)[0] == 0x43504f4cu) {
        C = reinterpret_cast<const uint32_t*>(a.in)[13];
        if ((uint64_t)kHdrBytes + 8ull * C > a.in_bytes) C = 0;
      }
    }
    C_s = C;
  }
  __syncthreads();
  const uint32_t tile = tile_s, C = C_s;
  if ((uint64_t)tile * kScanTile >= C) return;  // beyond the last tile: nobody waits on it
  const uint32_t* sizes = a.in ? reinterpret_cast<const uint32_t*>(a.in + kHdrBytes) : a.sizes;
  const uint64_t base = a.in ? (uint64_t)kHdrBytes + 8ull * C : a.base;
  const uint32_t c0 = tile * kScanTile + tid * kScanPer;
  unsigned long long v[kScanPer];
  unsigned long long run = 0;
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    v[k] = 0;
    const uint32_t c = c0 + k;
    if (c < C) {
      const uint32_t bs = sizes[2 * c], ss = sizes[2 * c + 1];
      if (a.validate && !(bs >= 4 && bs <= kChunkBytes && (bs & 3u) == 0 && ss >= 4 && ss <= kChunkBytes &&
                          (ss & 3u) == 0))
        bad = true;
      v[k] = (unsigned long long)bs + ss;
    }
    run += v[k];
  }
  if (bad) atomicOr(&a.ctr->err, kErrCorrupt);
  unsigned long long tot;
  const unsigned long long ex = block_scan_excl<unsigned long long, kScanThreads>(run, wsum, &tot);
  if (tid < 32) {
    const uint64_t e = lookback_warp(a.state, tile, tot);
    if (tid == 0) excl_s = e;
  }
  __syncthreads();
  unsigned long long o = base + excl_s + ex;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const uint32_t c = c0 + k;
    if (c < C) {
      a.off[c] = o;
      o += v[k];
      if (c == C - 1) {
        a.ctr->total_bytes = o;
        if (a.validate && o != a.expect_total) atomicOr(&a.ctr->err, kErrCorrupt);
      }
    }
  }
}

// k_place: a7 (part 3) — move each staged chunk to its offset, write the
// size table and the header.  One warp per chunk.
struct PlaceArgs {
  const uint8_t* stage;
  const uint32_t* sizes;
  const uint64_t* off;
  uint8_t* out;          // payload c goes to out + off[c]
  uint8_t* table;        // size-table entry c goes to table + 8c
  int header;            // write the 64-byte header at out (whole-stream mode)
  uint64_t out_cap;
  Counters* ctr;
  uint32_t C;
  int dtype, ndims;
  uint64_t d0, d1, d2, n;
  double eps;
};

// one warp copies n words (4-byte aligned destination): 128-bit loads from
// the 16-byte aligned staging slot, four of them in flight per lane, words
// stored one by one (the stream offset is only 4-byte aligned)
__device__ __forceinline__ void place_words(const uint32_t* src, uint32_t* dst, uint32_t n, int lane) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  const uint32_t n4 = n / 4;
  for (uint32_t b = 0; b < n4; b += 128) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = b + 32 * k + lane;
      v[k] = i < n4 ? __ldcs(&s4[i]) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = b + 32 * k + lane;
      if (i < n4) {
        dst[4 * i] = v[k].x;
        dst[4 * i + 1] = v[k].y;
        dst[4 * i + 2] = v[k].z;
        dst[4 * i + 3] = v[k].w;
      }
    }
  }
  for (uint32_t i = 4 * n4 + lane; i < n; i += 32) dst[i] = __ldcs(&src[i]);
}

__global__ void __launch_bounds__(256) k_place(PlaceArgs a) {
  const int lane = threadIdx.x & 31;
  const uint64_t total = a.ctr->total_bytes;
  if (total > a.out_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&a.ctr->err, kErrNoSpace);
    return;
  }
  const uint32_t nw = gridDim.x * (blockDim.x / 32);
  for (uint32_t c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); c < a.C; c += nw) {
    const uint32_t bs = a.sizes[2 * c], ss = a.sizes[2 * c + 1];
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.stage + (size_t)c * 2 * kChunkBytes);
    uint32_t* dst = reinterpret_cast<uint32_t*>(a.out + a.off[c]);
    place_words(src, dst, bs / 4, lane);
    place_words(src + kChunkBytes / 4, dst + bs / 4, ss / 4, lane);
    if (lane == 0) {
      uint32_t* tab = reinterpret_cast<uint32_t*>(a.table + 8ull * c);
      tab[0] = bs;
      tab[1] = ss;
    }
    if (a.header && c == 0 && lane == 0) {
      uint32_t* h32 = reinterpret_cast<uint32_t*>(a.out);
      uint64_t* h64 = reinterpret_cast<uint64_t*>(a.out);
      h32[0] = 0x43504f4cu;  // "LOPC"
      h32[1] = 1u | ((uint32_t)a.dtype << 16) | ((uint32_t)a.ndims << 24);
      h64[1] = a.d0;
      h64[2] = a.d1;
      h64[3] = a.d2;
      h64[4] = (uint64_t)__double_as_longlong(a.eps);
      h64[5] = a.n;
      h32[12] = kChunkBytes;
      h32[13] = a.C;
      h64[7] = total;
    }
  }
}

// ---------------------------------------------------------------------------
// k_decode (persistent; dtype from the stream header)
// ---------------------------------------------------------------------------
struct Hdr {
  int dtype, ndims;
  uint64_t d0, d1, d2, n;
  double eps;
  uint32_t C;
  bool ok;
  uint32_t err;
};

struct DecodeArgs {
  const uint8_t* in;    // whole-stream mode: the stream (header validated on the device)
  uint64_t in_bytes;
  void* out;            // chunk c (global index) decodes to out + c W
  uint64_t out_cap;
  const uint64_t* off;  // payload offsets of the chunks [c_begin, c_begin + c_count), from k_chunk_scan
  const uint32_t* table;  // their (bin, sub) size pairs
  const uint8_t* base;  // payload of local chunk l at base + off[l]
  uint64_t c_begin, c_count;
  uint64_t state_cap;   // chunk entries available in the workspace
  Counters* ctr;
  int prof;             // diagnostic phase clocks
  int slab;             // slab mode: header given (host-validated), no whole-stream checks
  Hdr given;
};

__device__ __forceinline__ Hdr parse_header(const DecodeArgs& a) {
  if (a.slab) return a.given;
  Hdr h{};
  h.ok = false;
  h.err = kErrCorrupt;
  if (a.in_bytes < kHdrBytes) return h;
  const uint32_t* h32 = reinterpret_cast<const uint32_t*>(a.in);
  const uint64_t* h64 = reinterpret_cast<const uint64_t*>(a.in);
  if (h32[0] != 0x43504f4cu) return h;
  if ((h32[1] & 0xffffu) != 1u) {
    h.err = kErrVersion;
    return h;
  }
  h.dtype = (h32[1] >> 16) & 0xff;
  h.ndims = (h32[1] >> 24) & 0xff;
  if (h.dtype > 1 || (h.ndims != 2 && h.ndims != 3)) return h;
  h.d0 = h64[1];
  h.d1 = h64[2];
  h.d2 = h64[3];
  if (h.ndims == 2 && h.d0 != 1) return h;
  const uint64_t lim = 1ull << 40;
  if (h.d0 > lim || h.d1 > lim || h.d2 > lim || h.d0 * h.d1 > lim) return h;
  h.n = h64[5];
  if (h.d0 * h.d1 * h.d2 != h.n || h.n > lim) return h;
  h.eps = __longlong_as_double((long long)h64[4]);
  if (!(h.eps >= 0x1p-900 && h.eps <= 0x1p1000)) return h;
  if (h32[12] != kChunkBytes) return h;
  const uint64_t W = kChunkBytes / (h.dtype ? 8u : 4u);
  h.C = h32[13];
  if ((uint64_t)h.C != (h.n + W - 1) / W) return h;
  if (h64[7] != a.in_bytes) return h;
  if ((uint64_t)kHdrBytes + 8ull * h.C > a.in_bytes) return h;
  if ((uint64_t)h.C > a.state_cap) return h;
  if (h.n * (h.dtype ? 8u : 4u) > a.out_cap) {
    h.err = kErrNoSpace;
    return h;
  }
  h.ok = true;
  h.err = 0;
  return h;
}

// One CTA per (chunk, stream), the two CTAs of a chunk form a 2-CTA cluster:
// rank 0 decodes the bins, rank 1 the subbins, each into its own shared
// memory; after a cluster barrier each CTA reconstructs half of the chunk,
// reading the partner's words through distributed shared memory.
struct DecSmem {
  alignas(16) uint8_t Wd[kChunkBytes + 64];  // payload (subbins) -> planes -> words (swizzled)
  alignas(16) uint8_t O[17408 + 128];        // payload (bins) | RZE_1^-1 output (subbins)
  RzeScratch R;
  uint32_t bad, ticket;
  int tmin, tmax;  // bin range of the half being reconstructed (f32 lo-key table)
};

// Copy `len` payload bytes (global, 4-aligned) into shared memory and zero
// the next 64 bytes.
__device__ __forceinline__ void load_payload(const uint8_t* g, uint32_t len, uint8_t* s) {
  const uint32_t* g32 = reinterpret_cast<const uint32_t*>(g);
  uint32_t* s32 = reinterpret_cast<uint32_t*>(s);
  for (uint32_t i = threadIdx.x; i < len / 4; i += kCodecThreads) s32[i] = __ldg(&g32[i]);
  if (threadIdx.x < 16) s32[len / 4 + threadIdx.x] = 0;
}

template <typename T>
__device__ __noinline__ void decode_stream(const DecodeArgs& a, const uint8_t* p, uint32_t size, bool subs, DecSmem& sm,
                                           uint8_t* BX, uint8_t* BY) {
  using U = typename VT<T>::U;
  constexpr int K = VT<T>::K;
  constexpr int W = kChunkBytes / K;
  constexpr int PER = W / kCodecThreads;
  // Buffers: bins: payload BX -> planes BY -> words BX (out of place; the
  // payload is dead once RZE^-1 has produced the planes); subbins: payload
  // BX -> RZE_1^-1 output BY -> planes BX -> words BX (in place).  The
  // 2-CTA decode passes (O, Wd) for bins and (Wd, O) for subbins.
  U* WD = reinterpret_cast<U*>(BX);
  const int tid = threadIdx.x;
  bool bad = false;
  PhaseClock pc;
  pc.start(a.prof);
  if (size == kChunkBytes) {  // raw words
    const U* g = reinterpret_cast<const U*>(p);
    for (int i = tid; i < W; i += kCodecThreads) WD[swz<U>(i)] = g[i];
    __syncthreads();
    pc.mark(a.ctr, subs ? 10 : 9);
    return;
  }
  constexpr uint32_t PB = W / 8;  // bytes per bit plane
  uint32_t act = kChunkBytes;     // planes past act / PB are zero (and not written)
  if (!subs) {
    load_payload(p, size, BX);
    __syncthreads();
    const uint32_t used = rze_dec(BX, size, kChunkBytes, 1, BY, sm.R, PB, &act);
    if (used == 0xffffffffu || pad4(used) != size) bad = true;
  } else {
    load_payload(p, size, BX);
    __syncthreads();
    const uint32_t l1 = (uint32_t)BX[0] | ((uint32_t)BX[1] << 8);
    const uint32_t l1max = kChunkBytes + kChunkBytes / K / 8 + 64 + 8;
    if (l1 > l1max || size < 2) bad = true;
    if (!bad) {
      const uint32_t used = rze_dec(BX + 2, size - 2, l1, 1, BY, sm.R, 0, nullptr);
      if (used == 0xffffffffu || pad4(2 + used) != size) bad = true;
    }
    if (!bad) {
      const uint32_t used2 = rze_dec(BY, l1, kChunkBytes, K, BX, sm.R, PB, &act);
      if (used2 != l1) bad = true;
    }
  }
  pc.mark(a.ctr, subs ? 10 : 9);
  if (bad) {  // uniform across the block (rze_dec results are block-wide)
    if (tid == 0) {
      sm.bad = 1;
      atomicOr(&a.ctr->err, kErrCorrupt);
    }
    __syncthreads();
    return;
  }
  if (subs)
    bit_inverse_planes<U, true>(BX, BX, W, (int)(act / PB));
  else
    bit_inverse_planes<U, false>(BY, BX, W, (int)(act / PB));
  pc.mark(a.ctr, 11);
  if (!subs) {  // NB^-1 + prefix sum (thread owns PER consecutive words)
    U d[PER];
    U run = 0;
#pragma unroll
    for (int v = 0; v < PER; ++v) {
      U u;
      if constexpr (sizeof(U) == 4) {
        if (v % 4 == 0) {
          const uint4 q = *reinterpret_cast<const uint4*>(&WD[swz<U>(tid * PER + v)]);
          d[v] = q.x, d[v + 1] = q.y, d[v + 2] = q.z, d[v + 3] = q.w;
        }
        u = d[v];
      } else {
        u = WD[swz<U>(tid * PER + v)];
      }
      d[v] = (U)((u ^ nb_mask<U>()) - nb_mask<U>());
      run += d[v];
    }
    U tot, ex;
    if constexpr (sizeof(U) == 4)
      ex = block_scan_excl<uint32_t>(run, sm.R.wsum, &tot);
    else
      ex = (U)block_scan_excl<unsigned long long>((unsigned long long)run, sm.R.wsum64,
                                                   reinterpret_cast<unsigned long long*>(&tot));
    U acc = ex;
#pragma unroll
    for (int v = 0; v < PER; ++v) {
      acc += d[v];
      d[v] = acc;
    }
#pragma unroll
    for (int v = 0; v < PER; ++v) {
      if constexpr (sizeof(U) == 4) {
        if (v % 4 == 0)
          *reinterpret_cast<uint4*>(&WD[swz<U>(tid * PER + v)]) = make_uint4(d[v], d[v + 1], d[v + 2], d[v + 3]);
      } else {
        WD[swz<U>(tid * PER + v)] = d[v];
      }
    }
    __syncthreads();
    pc.mark(a.ctr, 12);
  }
}

// a8: x^ = value with key(lo(b)) + s, or the raw escape (G10), for the
// half `r` of chunk c; WB/WS point at the two CTAs' word buffers (DSMEM).
// Thread t owns PER consecutive elements: lo(b) is computed only when the
// bin changes from the thread's previous element (bins are locally
// repetitive), and the values leave as 16-byte stores.
template <typename T, typename SM>
__device__ __forceinline__ void reconstruct_half(const DecodeArgs& a, const Hdr& h, uint32_t c, int r, const uint8_t* wb,
                                                 int wb_off, const uint8_t* ws, int ws_off, SM& sm,
                                                 int32_t* tab) {
  using U = typename VT<T>::U;
  using I = typename VT<T>::I;
  constexpr int W = kChunkBytes / VT<T>::K;
  constexpr int PER = W / kCodecThreads / 2;  // 8 (f32) / 4 (f64)
  const U* WB = reinterpret_cast<const U*>(wb);
  const U* SW = reinterpret_cast<const U*>(ws);
  const uint64_t e0 = (uint64_t)c * W;
  const uint32_t cnt = (uint32_t)min((uint64_t)W, h.n - e0);
  const int i0 = r * (W / 2) + threadIdx.x * PER;
  U bwv[PER], swv[PER];
#pragma unroll
  for (int v = 0; v < PER; ++v) {
    if constexpr (sizeof(U) == 4) {  // 4-word runs are contiguous (swz<u32>)
      if (v % 4 == 0) {
        const uint4 b = *reinterpret_cast<const uint4*>(&WB[swz<U>(i0 + v - wb_off)]);
        const uint4 q = *reinterpret_cast<const uint4*>(&SW[swz<U>(i0 + v - ws_off)]);
        bwv[v] = b.x, bwv[v + 1] = b.y, bwv[v + 2] = b.z, bwv[v + 3] = b.w;
        swv[v] = q.x, swv[v + 1] = q.y, swv[v + 2] = q.z, swv[v + 3] = q.w;
      }
    } else {
      bwv[v] = WB[swz<U>(i0 + v - wb_off)];
      swv[v] = SW[swz<U>(i0 + v - ws_off)];
    }
  }
  U out[PER];
  if constexpr (sizeof(U) == 4) {
    // f32: key(lo(b)) for every bin of the half in a shared table when the
    // half's bin range is small (the usual case: bins are locally smooth),
    // else per element; the same lo_key32_nb either way
    constexpr int kTab = 2048;  // entries at `tab` (8 KiB after the copied half)
    int lmin = INT_MAX, lmax = INT_MIN;
#pragma unroll
    for (int v = 0; v < PER; ++v)
      if (bwv[v] != VT<T>::kSentinel) {
        lmin = min(lmin, (int)bwv[v]);
        lmax = max(lmax, (int)bwv[v]);
      }
    lmin = __reduce_min_sync(0xffffffffu, lmin);
    lmax = __reduce_max_sync(0xffffffffu, lmax);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&sm.tmin, lmin);
      atomicMax(&sm.tmax, lmax);
    }
    __syncthreads();
    const int tmin = sm.tmin;
    const int64_t R = (int64_t)sm.tmax - (int64_t)tmin + 1;
    const bool use_tab = R > 0 && R <= kTab;
    if (use_tab) {
      for (int k = threadIdx.x; k < (int)R; k += kCodecThreads) tab[k] = lo_key32_nb(tmin + k, h.eps);
      __syncthreads();
    }
#pragma unroll
    for (int v = 0; v < PER; ++v) {
      const U bw = bwv[v];
      const bool esc = bw == VT<T>::kSentinel;
      const int32_t lk = use_tab ? tab[esc ? 0 : (int)bw - tmin] : lo_key32_nb((int32_t)bw, h.eps);
      const uint32_t k = (uint32_t)lk + (uint32_t)swv[v];  // wraps only for escapes
      out[v] = esc ? swv[v] : ((int32_t)k >= 0 ? k : (0x80000000u | (0u - k)));
    }
  } else {
#pragma unroll
    for (int v = 0; v < PER; ++v) {  // branch-free: lo(b) per element
      const U bw = bwv[v];
      const U bits = bits_of_key64(lo_key<T>((int64_t)(I)bw, h.eps) + (int64_t)swv[v]);
      out[v] = bw == VT<T>::kSentinel ? swv[v] : bits;
    }
  }
  T* O = static_cast<T*>(a.out) + e0 + i0;
  if ((uint32_t)i0 + PER <= cnt && ((uintptr_t)O & 15) == 0) {
#pragma unroll
    for (int v = 0; v < PER; v += 16 / (int)sizeof(T)) {
      if constexpr (sizeof(T) == 4)
        __stcs(reinterpret_cast<uint4*>(O + v), make_uint4(out[v], out[v + 1], out[v + 2], out[v + 3]));
      else
        __stcs(reinterpret_cast<ulonglong2*>(O + v), make_ulonglong2(out[v], out[v + 1]));
    }
  } else {
#pragma unroll
    for (int v = 0; v < PER; ++v)
      if ((uint32_t)(i0 + v) < cnt) reinterpret_cast<U*>(O)[v] = out[v];
  }
}

__device__ __forceinline__ bool h32_err(const DecodeArgs& a) {
  return (*(volatile uint32_t*)&a.ctr->err) & (kErrCorrupt | kErrVersion | kErrNoSpace);
}

// Persistent: 2-CTA cluster k decodes chunks k, k + clusters, ... (static
// round-robin: no ticket, so no cluster barrier at the top of the loop).
// Per chunk: [decode own stream] -> cluster barrier (release/acquire: the
// partner's words are complete) -> copy the partner's half -> relaxed
// cluster barrier (both copies done; only execution order is needed, so the
// outstanding output stores are not waited for) -> reconstruct from local smem.
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kCodecThreads, LOPC_CODEC_CTAS) k_decode(DecodeArgs a) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  DecSmem& sm = *reinterpret_cast<DecSmem*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  const int r = (int)cl.block_rank();
  // every exit below is taken by both CTAs of the cluster (same header, same
  // flag word, same chunk sequence) so the cluster barriers stay matched
  const Hdr h = parse_header(a);
  if (!h.ok) {
    if (blockIdx.x == 0 && tid == 0) atomicOr(&a.ctr->err, h.err);
    return;
  }
  if (h32_err(a)) return;  // k_chunk_scan flagged the table
  const uint64_t ncnk = a.slab ? a.c_count : (uint64_t)h.C;
  const DecSmem* s0 = cl.map_shared_rank(&sm, 0);
  const DecSmem* s1 = cl.map_shared_rank(&sm, 1);
  if (tid == 0) sm.bad = 0;  // sticky: a corrupt chunk fails the whole call
  cl.sync();                 // both flags initialised
  const uint64_t nclu = gridDim.x / 2;
  for (uint64_t l = blockIdx.x / 2; l < ncnk; l += nclu) {
    __syncthreads();  // this CTA's previous reconstruct is done with its smem
    if (tid == 0) {
      sm.tmin = INT_MAX;
      sm.tmax = INT_MIN;
    }
    const uint32_t sz = a.table[2 * l + r];
    const uint8_t* p = a.base + a.off[l] + (r ? a.table[2 * l] : 0u);
    if (h.dtype == 0)
      decode_stream<float>(a, p, sz, r != 0, sm, r ? sm.Wd : sm.O, r ? sm.O : sm.Wd);
    else
      decode_stream<double>(a, p, sz, r != 0, sm, r ? sm.Wd : sm.O, r ? sm.O : sm.Wd);
    cl.sync();  // release/acquire: the partner's words are complete
    const uint64_t c = a.c_begin + l;
    const bool ok = !s0->bad && !s1->bad;
    // the partner's words of this CTA's half, copied once into local smem
    // with 16-byte DSMEM loads: rank 0 (bin words in its sm.O) takes the
    // subbin half 0 into its sm.Wd (planes, dead); rank 1 (subbin words in its
    // sm.Wd) takes the bin half 1 into its sm.O (RZE_1 output, dead)
    constexpr int HB = kChunkBytes / 2;
    if (ok) {
      const uint4* rem = reinterpret_cast<const uint4*>(r ? s0->O + HB : s1->Wd);
      uint4* loc = reinterpret_cast<uint4*>(r ? sm.O : sm.Wd);
      for (int t = tid; t < HB / 16; t += kCodecThreads) loc[t] = rem[t];
    }
    cluster_sync_relaxed();  // both copies done: the partner may overwrite its words next
    __syncthreads();         // the local copy is visible to the whole CTA
    if (ok) {
      const int half_w = h.dtype == 0 ? 2048 : 1024;  // W / 2
      // bins in sm.O (rank 1: the copied half, offset W/2), subbins in sm.Wd;
      // the f32 lo-key table in the free 8 KiB after this CTA's copied half
      int32_t* tab = reinterpret_cast<int32_t*>((r ? sm.O : sm.Wd) + HB);
      if (h.dtype == 0)
        reconstruct_half<float>(a, h, (uint32_t)c, r, sm.O, r ? half_w : 0, sm.Wd, 0, sm, tab);
      else
        reconstruct_half<double>(a, h, (uint32_t)c, r, sm.O, r ? half_w : 0, sm.Wd, 0, sm, tab);
    }
  }
  cl.sync();  // no CTA leaves while its partner may still read its flags
}

// Single-CTA decode (the default; the 2-CTA cluster k_decode above is the
// alternative, lopc_set_decoder(2)).  One CTA decodes both streams of a chunk
// and reconstructs it from its own shared memory: no cluster barriers, no
// DSMEM copy.  The payloads are read where they lie (global memory, through
// L1; the next chunk's payload is prefetched into L1 while this one
// decodes), so only two 16 KiB buffers are needed and 6 CTAs fit an SM:
//   subbins: payload -> RZE_1^-1 -> C -> RZE_k^-1 -> planes A -> words A
//   bins:    payload -> RZE_1^-1 -> planes C -> words C -> NB^-1 + prefix sum
//   x^:      from the words in C (bins) and A (subbins); the f32 lo-key
//            table of a half overwrites that half's bin words once every
//            thread holds its elements (reconstruct_half).
// Persistent: CTA b decodes chunks b, b + gridDim.x, ...
#ifndef LOPC_DEC1_CTAS
#define LOPC_DEC1_CTAS 6
#endif
struct DecSmem2 {
  alignas(16) uint8_t A[kChunkBytes + 64];  // subbins: planes -> words
  alignas(16) uint8_t C[17408 + 128];       // subbins: RZE_1^-1 output; bins: planes -> words
  RzeScratch R;
  uint32_t bad;
  int tmin, tmax;
};

// Raw chunk stream (size == kChunkBytes): the words as they are, swizzled.
template <typename U>
__device__ __forceinline__ void raw_words(const uint8_t* p, uint8_t* buf) {
  constexpr int W = kChunkBytes / (int)sizeof(U);
  const U* g = reinterpret_cast<const U*>(p);
  U* wd = reinterpret_cast<U*>(buf);
  for (int i = threadIdx.x; i < W; i += kCodecThreads) wd[swz<U>(i)] = g[i];
}

// Both streams of one chunk into words (bins in C, subbins in A).  Returns
// false (block-uniform) for a corrupt payload.
template <typename T>
__device__ __noinline__ bool decode_chunk_g(const uint8_t* p, uint32_t bs, uint32_t ss, DecSmem2& sm) {
  using U = typename VT<T>::U;
  constexpr int K = VT<T>::K;
  constexpr int W = kChunkBytes / K;
  constexpr int PER = W / kCodecThreads;
  constexpr uint32_t PB = W / 8;  // bytes per bit plane
  const int tid = threadIdx.x;
  const uint8_t* ps = p + bs;
  // subbins
  if (ss == kChunkBytes) {
    raw_words<U>(ps, sm.A);
  } else {
    if (ss < 2) return false;
    const uint32_t l1 = (uint32_t)__ldg(ps) | ((uint32_t)__ldg(ps + 1) << 8);
    if (l1 > kChunkBytes + kChunkBytes / K / 8 + 64 + 8) return false;
    const uint32_t used = rze_dec<true>(ps + 2, ss - 2, l1, 1, sm.C, sm.R, 0, nullptr);
    if (used == 0xffffffffu || pad4(2 + used) != ss) return false;
    uint32_t act = kChunkBytes;
    const uint32_t used2 = rze_dec<false>(sm.C, l1, kChunkBytes, K, sm.A, sm.R, PB, &act);
    if (used2 != l1) return false;
    bit_inverse_planes<U, true>(sm.A, sm.A, W, (int)(act / PB));
  }
  // bins
  if (bs == kChunkBytes) {
    raw_words<U>(p, sm.C);
    __syncthreads();
    return true;
  }
  uint32_t act = kChunkBytes;
  const uint32_t used = rze_dec<true>(p, bs, kChunkBytes, 1, sm.C, sm.R, PB, &act);
  if (used == 0xffffffffu || pad4(used) != bs) return false;
  bit_inverse_planes<U, true>(sm.C, sm.C, W, (int)(act / PB));
  // NB^-1 + prefix sum (thread owns PER consecutive words)
  U* WD = reinterpret_cast<U*>(sm.C);
  U d[PER];
  U run = 0;
#pragma unroll
  for (int v = 0; v < PER; ++v) {
    U u;
    if constexpr (sizeof(U) == 4) {
      if (v % 4 == 0) {
        const uint4 q = *reinterpret_cast<const uint4*>(&WD[swz<U>(tid * PER + v)]);
        d[v] = q.x, d[v + 1] = q.y, d[v + 2] = q.z, d[v + 3] = q.w;
      }
      u = d[v];
    } else {
      u = WD[swz<U>(tid * PER + v)];
    }
    d[v] = (U)((u ^ nb_mask<U>()) - nb_mask<U>());
    run += d[v];
  }
  U tot, ex;
  if constexpr (sizeof(U) == 4)
    ex = block_scan_excl<uint32_t>(run, sm.R.wsum, &tot);
  else
    ex = (U)block_scan_excl<unsigned long long>((unsigned long long)run, sm.R.wsum64,
                                                 reinterpret_cast<unsigned long long*>(&tot));
  U acc = ex;
#pragma unroll
  for (int v = 0; v < PER; ++v) {
    acc += d[v];
    d[v] = acc;
  }
#pragma unroll
  for (int v = 0; v < PER; ++v) {
    if constexpr (sizeof(U) == 4) {
      if (v % 4 == 0)
        *reinterpret_cast<uint4*>(&WD[swz<U>(tid * PER + v)]) = make_uint4(d[v], d[v + 1], d[v + 2], d[v + 3]);
    } else {
      WD[swz<U>(tid * PER + v)] = d[v];
    }
  }
  __syncthreads();
  return true;
}

__global__ void __launch_bounds__(kCodecThreads, LOPC_DEC1_CTAS) k_decode1(DecodeArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  DecSmem2& sm = *reinterpret_cast<DecSmem2*>(smem_raw);
  const int tid = threadIdx.x;
  const Hdr h = parse_header(a);
  if (!h.ok) {
    if (blockIdx.x == 0 && tid == 0) atomicOr(&a.ctr->err, h.err);
    return;
  }
  if (h32_err(a)) return;  // k_chunk_scan flagged the table
  const uint64_t ncnk = a.slab ? a.c_count : (uint64_t)h.C;
  for (uint64_t l = blockIdx.x; l < ncnk; l += gridDim.x) {
    const uint32_t bs = a.table[2 * l], ss = a.table[2 * l + 1];
    const uint8_t* p = a.base + a.off[l];
    {  // the next chunk's payload into L1 while this one decodes
      const uint64_t ln = l + gridDim.x;
      if (ln < ncnk) {
        const uint8_t* pn = a.base + a.off[ln];
        const uint32_t len = a.table[2 * ln] + a.table[2 * ln + 1];
        const uintptr_t b0 = reinterpret_cast<uintptr_t>(pn) & ~(uintptr_t)127;
        const uint32_t lines = (uint32_t)((reinterpret_cast<uintptr_t>(pn) + len + 127 - b0) >> 7);
        for (uint32_t k = tid; k < lines; k += kCodecThreads) pf_l1_bytes(reinterpret_cast<const void*>(b0 + 128 * (uintptr_t)k));
      }
    }
    __syncthreads();  // the previous chunk's reconstruct is done with the buffers
    const bool ok = h.dtype == 0 ? decode_chunk_g<float>(p, bs, ss, sm) : decode_chunk_g<double>(p, bs, ss, sm);
    if (!ok) {  // block-uniform
      if (tid == 0) atomicOr(&a.ctr->err, kErrCorrupt);
      return;
    }
    const uint64_t c = a.c_begin + l;
    for (int r = 0; r < 2; ++r) {
      if (tid == 0) {
        sm.tmin = INT_MAX;
        sm.tmax = INT_MIN;
      }
      __syncthreads();
      // the f32 lo-key table of half r over half r's bin words in C (loaded
      // into registers before reconstruct_half's first barrier)
      if (h.dtype == 0)
        reconstruct_half<float>(a, h, (uint32_t)c, r, sm.C, 0, sm.A, 0, sm,
                                reinterpret_cast<int32_t*>(sm.C + r * (kChunkBytes / 2)));
      else
        reconstruct_half<double>(a, h, (uint32_t)c, r, sm.C, 0, sm.A, 0, sm,
                                 reinterpret_cast<int32_t*>(sm.C + r * (kChunkBytes / 2)));
      __syncthreads();
    }
  }
}

}  // namespace lopc
