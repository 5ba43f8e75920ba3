// lopc_codec.cuh — chunked lossless coding and decoding.
//
// Bins: "the lossless portion of PFPL" (readings G17-G19):
//   DIFFNB_k -> BIT_k -> RZE_1.
// Subbins: the LC pipelines BIT_4 RZE_4 RZE_1 / BIT_8 RZE_8 RZE_1.
// One CTA encodes one 16 KiB chunk of both streams; the chunk's
// payload offset is the exclusive prefix of (bin_size + sub_size) over the
// previous chunks, found by a decoupled look-back (a7), so every payload is
// written once, at its final place.  Stream format: DESIGN.md §4.
//
// Word buffers in shared memory use an XOR swizzle so that the 32x32 bit
// transposes of BIT_k run bank-conflict-free: word w lives at
//   (w & ~31) | ((w ^ (w >> 5)) & 31).
#pragma once
#include "lopc_device.cuh"
#include "lopc_repair.cuh"

namespace lopc {

constexpr int kCodecThreads = 512;

__device__ __forceinline__ int swz(int w) { return (w & ~31) | ((w ^ (w >> 5)) & 31); }

// ---------------------------------------------------------------------------
// Block-wide exclusive scan (sum) over kCodecThreads threads.
// ---------------------------------------------------------------------------
template <typename V>
__device__ __forceinline__ V block_scan_excl(V v, V* wsum, V* total) {
  constexpr int NW = kCodecThreads / 32;
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

// OR-combine `v` over aligned groups of `lanes` lanes.
__device__ __forceinline__ uint32_t group_or(uint32_t v, int lanes) {
  for (int o = 1; o < lanes; o <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Non-zero-word bits of 16 bytes for word width g (16/g bits, LSB = first word).
__device__ __forceinline__ uint32_t nz16(uint4 v, int g) {
  if (g == 1) {
    uint32_t r = 0;
    uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t t = (((w4[i] & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w4[i]) & 0x80808080u;
      uint32_t n = ((t >> 7) & 1u) | ((t >> 14) & 2u) | ((t >> 21) & 4u) | ((t >> 28) & 8u);
      r |= n << (4 * i);
    }
    return r;
  }
  if (g == 4) return (v.x != 0) | ((v.y != 0) << 1) | ((v.z != 0) << 2) | ((v.w != 0) << 3);
  return ((v.x | v.y) != 0) | (((v.z | v.w) != 0) << 1);
}

// RZE level sizes: sz[0] = ceil(n/8); while sz[i] > 8: sz[i+1] = ceil(sz[i]/8).
__device__ __forceinline__ int rze_levels(uint32_t n, uint32_t* sz) {
  int top = 0;
  sz[0] = (n + 7) / 8;
  while (sz[top] > 8) {
    sz[top + 1] = (sz[top] + 7) / 8;
    ++top;
  }
  return top;
}

struct RzeSmem {
  uint32_t bm0[768];  // up to 24576 input words
  uint32_t bm1[96];
  uint32_t bm2[16];
  uint32_t bm3[4];
  uint8_t kb0[3072];
  uint8_t kb1[384];
  uint8_t kb2[64];
  uint32_t wsum[32];
  unsigned long long wsum64[32];
};

__device__ __forceinline__ uint32_t* rze_bm(RzeSmem& r, int i) {
  return i == 0 ? r.bm0 : (i == 1 ? r.bm1 : (i == 2 ? r.bm2 : r.bm3));
}
__device__ __forceinline__ uint8_t* rze_kb(RzeSmem& r, int i) { return i == 0 ? r.kb0 : (i == 1 ? r.kb1 : r.kb2); }

// RZE_g encode of `in` (shared, 16-byte aligned, L bytes; the bytes up to the
// next multiple of 16 must be zero) into `out` (shared).  Returns the encoded
// length; `out` is written only if that length <= out_limit.
__device__ uint32_t rze_encode(const uint8_t* in, uint32_t L, int g, uint8_t* out, uint32_t out_limit, RzeSmem& r) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t n = L / (uint32_t)g;
  const int b = 16 / g;          // bits per thread per 16 bytes
  const int lpw = 32 / b;        // lanes per bitmap word
  const uint32_t L16 = (L + 15) & ~15u;
  const int iters = (int)((L16 + kCodecThreads * 16 - 1) / (kCodecThreads * 16));
  uint32_t masks[3] = {0, 0, 0}, ranks[3] = {0, 0, 0};
  uint32_t running = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t T = (uint32_t)(it * kCodecThreads + tid);
    const uint32_t off = T * 16;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (off < L16) v = *reinterpret_cast<const uint4*>(in + off);
    uint32_t m = nz16(v, g);
    uint32_t tot;
    uint32_t ex = block_scan_excl<uint32_t>((uint32_t)__popc(m), r.wsum, &tot);
    masks[it] = m;
    ranks[it] = running + ex;
    running += tot;
    uint32_t word = group_or(m << ((T * b) & 31), lpw);
    if ((lane % lpw) == 0) r.bm0[(T * b) >> 5] = word;
  }
  __syncthreads();
  const uint32_t ndata = running;
  uint32_t sz[6], ksz[6];
  int top = 0;
  sz[0] = (n + 7) / 8;
  while (sz[top] > 8) {
    sz[top + 1] = (sz[top] + 7) / 8;
    const uint32_t* bi = rze_bm(r, top);
    const uint8_t* bb = reinterpret_cast<const uint8_t*>(bi);
    uint32_t* bn = rze_bm(r, top + 1);
    uint8_t* kb = rze_kb(r, top);
    const uint32_t nw = (sz[top] + 3) / 4;
    uint32_t krun = 0;
    for (uint32_t base = 0; base < nw; base += kCodecThreads) {
      const uint32_t w = base + tid;
      uint32_t m4 = 0;
      uint32_t cur = 0;
      if (w < nw) {
        cur = bi[w];
        uint32_t prev = w ? (uint32_t)bb[4 * w - 1] : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t byte = (cur >> (8 * j)) & 0xffu;
          if (4 * w + j < sz[top] && byte != prev) m4 |= 1u << j;
          prev = byte;
        }
      }
      uint32_t tot;
      uint32_t ex = block_scan_excl<uint32_t>((uint32_t)__popc(m4), r.wsum, &tot);
      uint32_t k = krun + ex;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (m4 & (1u << j)) kb[k++] = (uint8_t)(cur >> (8 * j));
      krun += tot;
      uint32_t word = group_or(m4 << ((w * 4) & 31), 8);
      if ((lane & 7) == 0 && w < ((nw + 7) & ~7u)) bn[w >> 3] = word;
    }
    __syncthreads();
    ksz[top] = krun;
    ++top;
  }
  uint32_t total = sz[top] + (uint32_t)g * ndata;
  for (int i = 0; i < top; ++i) total += ksz[i];
  if (total <= out_limit) {
    const uint8_t* bt = reinterpret_cast<const uint8_t*>(rze_bm(r, top));
    if ((uint32_t)tid < sz[top]) out[tid] = bt[tid];
    uint32_t off = sz[top];
    for (int i = top - 1; i >= 0; --i) {
      const uint8_t* kb = rze_kb(r, i);
      for (uint32_t t = tid; t < ksz[i]; t += kCodecThreads) out[off + t] = kb[t];
      off += ksz[i];
    }
    for (int it = 0; it < iters; ++it) {
      const uint32_t T = (uint32_t)(it * kCodecThreads + tid);
      uint32_t m = masks[it];
      uint32_t k = ranks[it];
      while (m) {
        int j = __ffs(m) - 1;
        m &= m - 1;
        const uint8_t* src = in + T * 16 + j * g;
        uint8_t* dst = out + off + k * g;
        for (int q = 0; q < g; ++q) dst[q] = src[q];
        ++k;
      }
    }
  }
  __syncthreads();
  return total;
}

// RZE_g decode: `in` (shared) holds in_len payload bytes; reconstructs L bytes
// into `out` (shared, 16-byte aligned, room for L rounded up to 16).  Returns
// the number of payload bytes consumed, or 0xffffffff if the payload is too
// short for its bitmaps (corrupt).
__device__ uint32_t rze_decode(const uint8_t* in, uint32_t in_len, uint32_t L, int g, uint8_t* out, RzeSmem& r) {
  const int tid = threadIdx.x;
  const uint32_t n = L / (uint32_t)g;
  uint32_t sz[6];
  const int top = rze_levels(n, sz);
  if (sz[top] > in_len) return 0xffffffffu;
  {
    uint8_t* bt = reinterpret_cast<uint8_t*>(rze_bm(r, top));
    if ((uint32_t)tid < ((sz[top] + 3) & ~3u)) bt[tid] = (uint32_t)tid < sz[top] ? in[tid] : 0;
  }
  __syncthreads();
  uint32_t pos = sz[top];
  for (int i = top - 1; i >= 0; --i) {
    const uint32_t* bn = rze_bm(r, i + 1);
    uint32_t* bi = rze_bm(r, i);
    const uint32_t nw = (sz[i] + 3) / 4;
    uint32_t krun = 0;
    for (uint32_t base = 0; base < nw; base += kCodecThreads) {
      const uint32_t w = base + tid;
      uint32_t m4 = 0;
      if (w < nw) {
        m4 = (bn[w >> 3] >> ((w & 7) * 4)) & 0xfu;
        uint32_t valid = sz[i] - 4 * w;  // >= 1
        if (valid < 4) m4 &= (1u << valid) - 1u;
      }
      uint32_t tot;
      uint32_t ex = block_scan_excl<uint32_t>((uint32_t)__popc(m4), r.wsum, &tot);
      if (pos + krun + tot > in_len) return 0xffffffffu;  // block-uniform
      if (w < nw) {
        uint32_t k = krun + ex;  // selected positions before this word
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (m4 & (1u << j)) ++k;
          uint32_t byte = k ? (uint32_t)in[pos + k - 1] : 0u;
          if (4 * w + j >= sz[i]) byte = 0;
          word |= byte << (8 * j);
        }
        bi[w] = word;
      }
      krun += tot;
    }
    __syncthreads();
    pos += krun;
  }
  // words
  const int b = 16 / g;
  const uint32_t L16 = (L + 15) & ~15u;
  const int iters = (int)((L16 + kCodecThreads * 16 - 1) / (kCodecThreads * 16));
  uint32_t running = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t T = (uint32_t)(it * kCodecThreads + tid);
    uint32_t m = 0;
    if (T * 16 < L16) {
      m = (r.bm0[(T * b) >> 5] >> ((T * b) & 31)) & ((1u << b) - 1u);
      uint32_t first = T * (uint32_t)b;
      if (first >= n)
        m = 0;
      else if (n - first < (uint32_t)b)
        m &= (1u << (n - first)) - 1u;
    }
    uint32_t tot;
    uint32_t ex = block_scan_excl<uint32_t>((uint32_t)__popc(m), r.wsum, &tot);
    if (pos + (uint32_t)g * (running + tot) > in_len) return 0xffffffffu;
    if (T * 16 < L16) {
      uint32_t k = running + ex;
      uint8_t tmp[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) tmp[q] = 0;
      for (int j = 0; j < b; ++j) {
        if (m & (1u << j)) {
          for (int q = 0; q < g; ++q) tmp[j * g + q] = in[pos + k * g + q];
          ++k;
        }
      }
      uint4 v;
      v.x = tmp[0] | (tmp[1] << 8) | (tmp[2] << 16) | ((uint32_t)tmp[3] << 24);
      v.y = tmp[4] | (tmp[5] << 8) | (tmp[6] << 16) | ((uint32_t)tmp[7] << 24);
      v.z = tmp[8] | (tmp[9] << 8) | (tmp[10] << 16) | ((uint32_t)tmp[11] << 24);
      v.w = tmp[12] | (tmp[13] << 8) | (tmp[14] << 16) | ((uint32_t)tmp[15] << 24);
      *reinterpret_cast<uint4*>(out + T * 16) = v;
    }
    running += tot;
  }
  __syncthreads();
  return pos + (uint32_t)g * running;
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

// BIT_k (G20): words (swizzled shared) -> 8k planes of W bits (linear bytes).
template <typename U>
__device__ __forceinline__ void bit_forward(const U* words, uint32_t* planes, int W) {
  const int groups = W / 32;
  for (int g = threadIdx.x; g < groups; g += kCodecThreads) {
#pragma unroll
    for (int half = 0; half < (int)sizeof(U) / 4; ++half) {
      uint32_t A[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) A[i] = (uint32_t)(words[swz(32 * g + i)] >> (32 * half));
      transpose32(A);
#pragma unroll
      for (int j = 0; j < 32; ++j) planes[(32 * half + j) * groups + g] = A[j];
    }
  }
}

template <typename U>
__device__ __forceinline__ void bit_inverse(const uint32_t* planes, U* words, int W) {
  const int groups = W / 32;
  for (int g = threadIdx.x; g < groups; g += kCodecThreads) {
#pragma unroll
    for (int half = 0; half < (int)sizeof(U) / 4; ++half) {
      uint32_t A[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) A[j] = planes[(32 * half + j) * groups + g];
      transpose32(A);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (half == 0)
          words[swz(32 * g + i)] = (U)A[i];
        else
          words[swz(32 * g + i)] |= (U)A[i] << (32 * half);
      }
    }
  }
}

template <typename U>
__host__ __device__ constexpr U nb_mask() {
  return (U)0xAAAAAAAAAAAAAAAAull;
}

// ---------------------------------------------------------------------------
// k_encode
// ---------------------------------------------------------------------------
struct EncodeArgs {
  const void* x;
  const uint32_t* s;
  uint8_t* out;
  uint64_t out_cap;
  uint64_t* state;  // look-back state per chunk
  Counters* ctr;
  double eps, inv;
  uint64_t n;
  uint32_t C;
  int ndims;
  int vec;  // x and s are 16-byte aligned: vector loads allowed
  uint64_t d0, d1, d2;
};

struct CodecSmem {
  alignas(16) uint8_t wb[kChunkBytes];      // bin words (swizzled)
  alignas(16) uint8_t ws[kChunkBytes];      // subbin words (swizzled)
  alignas(16) uint8_t z[17408];             // DIFFNB words / RZE_k output
  alignas(16) uint8_t sh[kChunkBytes];      // bit planes
  alignas(16) uint8_t ob[kChunkBytes + 16]; // bin payload
  alignas(16) uint8_t os[kChunkBytes + 16]; // subbin payload
  RzeSmem r;
  uint32_t misc[8];
  unsigned long long misc64[4];
};

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

template <typename T>
__global__ void __launch_bounds__(kCodecThreads, 2) k_encode(EncodeArgs a) {
  using U = typename VT<T>::U;
  using I = typename VT<T>::I;
  constexpr int K = VT<T>::K;
  constexpr int W = kChunkBytes / K;
  constexpr int PER = W / kCodecThreads;  // words per thread (8 f32, 4 f64)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CodecSmem& sm = *reinterpret_cast<CodecSmem*>(smem_raw);
  U* WB = reinterpret_cast<U*>(sm.wb);
  U* WS = reinterpret_cast<U*>(sm.ws);
  U* Z = reinterpret_cast<U*>(sm.z);
  const int tid = threadIdx.x;

  if (tid == 0) sm.misc[0] = atomicAdd(&a.ctr->ticket, 1u);
  __syncthreads();
  const uint32_t c = sm.misc[0];
  const uint64_t e0 = (uint64_t)c * W;
  const uint32_t cnt = (uint32_t)min((uint64_t)W, a.n - e0);
  const T* X = static_cast<const T*>(a.x) + e0;
  const uint32_t* S = a.s + e0;

  // --- a1 + a4: re-quantize, words, bound self-check ---------------------
  // each thread owns PER/4 runs of 4 consecutive words, loaded as 16-byte vectors
  uint32_t esc = 0, bad = 0;
#pragma unroll
  for (int v = 0; v < PER / 4; ++v) {
    const int i0 = 4 * (v * kCodecThreads + tid);
    T xs[4];
    uint32_t ss[4];
    if (a.vec && (uint32_t)i0 + 3 < cnt) {
      if constexpr (sizeof(T) == 4) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(X + i0));
        xs[0] = xv.x, xs[1] = xv.y, xs[2] = xv.z, xs[3] = xv.w;
      } else {
        const double2 x0 = __ldg(reinterpret_cast<const double2*>(X + i0));
        const double2 x1 = __ldg(reinterpret_cast<const double2*>(X + i0 + 2));
        xs[0] = x0.x, xs[1] = x0.y, xs[2] = x1.x, xs[3] = x1.y;
      }
      const uint4 sv = __ldg(reinterpret_cast<const uint4*>(S + i0));
      ss[0] = sv.x, ss[1] = sv.y, ss[2] = sv.z, ss[3] = sv.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool in = (uint32_t)(i0 + q) < cnt;
        xs[q] = in ? X[i0 + q] : (T)0;
        ss[q] = in ? S[i0 + q] : 0u;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q;
      U bw = 0, sw = 0;
      if ((uint32_t)i < cnt) {
        const T x = xs[q];
        const uint32_t sq = ss[q];
        I b;
        if (quantize<T>(x, a.eps, a.inv, b)) {
          bw = (U)b;
          sw = (U)sq;
          if (sq != 0) {
            // x^ = value with key(lo(b)) + s must not exceed x (a4)
            const T lo = lo_t<T>((int64_t)b, a.eps);
            if ((int64_t)key_of((U)as_bits(lo)) + (int64_t)sq > (int64_t)key_of((U)as_bits(x))) bad = 1;
          }
        } else {
          bw = VT<T>::kSentinel;
          sw = (U)as_bits(x);
          ++esc;
        }
      }
      WB[swz(i)] = bw;
      WS[swz(i)] = sw;
    }
  }
  if (bad) atomicOr(&a.ctr->err, kErrBound);
  esc = __reduce_add_sync(0xffffffffu, esc);
  if ((tid & 31) == 0 && esc) atomicAdd(&a.ctr->escapes, (unsigned long long)esc);
  __syncthreads();

  // --- a5: bins: DIFFNB_k -> BIT_k -> RZE_1 -----------------------------------
#pragma unroll
  for (int v = 0; v < PER; ++v) {
    const int i = v * kCodecThreads + tid;
    U cur = WB[swz(i)];
    U prev = i ? WB[swz(i - 1)] : (U)0;
    U d = cur - prev;
    Z[swz(i)] = (U)((d + nb_mask<U>()) ^ nb_mask<U>());
  }
  __syncthreads();
  bit_forward<U>(Z, reinterpret_cast<uint32_t*>(sm.sh), W);
  __syncthreads();
  const uint32_t blen = rze_encode(sm.sh, kChunkBytes, 1, sm.ob, kChunkBytes - 4, sm.r);
  const uint32_t bsize = blen <= kChunkBytes - 4 ? pad4(blen) : kChunkBytes;
  if (bsize < kChunkBytes && (uint32_t)tid < bsize - blen) sm.ob[blen + tid] = 0;

  // --- a6: subbins: BIT_k -> RZE_k -> RZE_1 ----------------------------------
  bit_forward<U>(WS, reinterpret_cast<uint32_t*>(sm.sh), W);
  __syncthreads();
  const uint32_t l1 = rze_encode(sm.sh, kChunkBytes, K, sm.z, 0xffffffffu, sm.r);
  if ((uint32_t)tid < 16) sm.z[l1 + tid] = 0;  // zero tail for the next stage's 16-byte reads
  __syncthreads();
  const uint32_t l2 = rze_encode(sm.z, l1, 1, sm.os + 2, kChunkBytes - 6, sm.r);
  const uint32_t ssize = l2 <= kChunkBytes - 6 ? pad4(2 + l2) : kChunkBytes;
  if (ssize < kChunkBytes) {
    if (tid == 0) {
      sm.os[0] = (uint8_t)(l1 & 0xffu);
      sm.os[1] = (uint8_t)(l1 >> 8);
    }
    if ((uint32_t)tid < ssize - 2 - l2) sm.os[2 + l2 + tid] = 0;
  }

  // --- a7: placement by decoupled look-back -----------------------------------
  if (tid < 32) {
    const uint64_t excl = lookback_warp(a.state, c, (uint64_t)bsize + ssize);
    if (tid == 0) sm.misc64[0] = excl;
  }
  __syncthreads();
  const uint64_t base = (uint64_t)kHdrBytes + 8ull * a.C + sm.misc64[0];
  const uint64_t end = base + bsize + ssize;
  const bool fits = end <= a.out_cap;
  if (tid == 0) {
    if (!fits) atomicOr(&a.ctr->err, kErrNoSpace);
    if ((uint64_t)kHdrBytes + 8ull * (c + 1) <= a.out_cap) {
      uint32_t* tab = reinterpret_cast<uint32_t*>(a.out + kHdrBytes + 8ull * c);
      tab[0] = bsize;
      tab[1] = ssize;
    }
    atomicAdd(&a.ctr->bin_bytes, (unsigned long long)bsize);
    atomicAdd(&a.ctr->sub_bytes, (unsigned long long)ssize);
    if (c == a.C - 1) {
      a.ctr->total_bytes = end;
      if (a.out_cap >= kHdrBytes) {
        uint32_t* h32 = reinterpret_cast<uint32_t*>(a.out);
        uint64_t* h64 = reinterpret_cast<uint64_t*>(a.out);
        h32[0] = 0x43504f4cu;  // "LOPC"
        h32[1] = 1u | ((uint32_t)(K == 4 ? 0 : 1) << 16) | ((uint32_t)a.ndims << 24);
        h64[1] = a.d0;
        h64[2] = a.d1;
        h64[3] = a.d2;
        h64[4] = (uint64_t)__double_as_longlong(a.eps);
        h64[5] = a.n;
        h32[12] = kChunkBytes;
        h32[13] = a.C;
        h64[7] = end;
      }
    }
  }
  if (!fits) return;
  uint32_t* dst = reinterpret_cast<uint32_t*>(a.out + base);
  if (bsize == kChunkBytes) {
    for (int i = tid; i < W; i += kCodecThreads) {
      U w = WB[swz(i)];
#pragma unroll
      for (int h = 0; h < K / 4; ++h) dst[i * (K / 4) + h] = (uint32_t)(w >> (32 * h));
    }
  } else {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(sm.ob);
    for (uint32_t i = tid; i < bsize / 4; i += kCodecThreads) dst[i] = src[i];
  }
  dst += bsize / 4;
  if (ssize == kChunkBytes) {
    for (int i = tid; i < W; i += kCodecThreads) {
      U w = WS[swz(i)];
#pragma unroll
      for (int h = 0; h < K / 4; ++h) dst[i * (K / 4) + h] = (uint32_t)(w >> (32 * h));
    }
  } else {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(sm.os);
    for (uint32_t i = tid; i < ssize / 4; i += kCodecThreads) dst[i] = src[i];
  }
}

// ---------------------------------------------------------------------------
// k_decode (persistent; dtype from the stream header)
// ---------------------------------------------------------------------------
struct DecodeArgs {
  const uint8_t* in;
  uint64_t in_bytes;
  void* out;
  uint64_t out_cap;
  uint64_t* state;
  uint64_t state_cap;  // entries available
  Counters* ctr;
};

struct Hdr {
  int dtype, ndims;
  uint64_t d0, d1, d2, n;
  double eps;
  uint32_t C;
  bool ok;
  uint32_t err;
};

__device__ __forceinline__ Hdr parse_header(const DecodeArgs& a) {
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

// Copy `len` payload bytes (global, 4-aligned) into shared memory and zero
// the next 16 bytes.
__device__ __forceinline__ void load_payload(const uint8_t* g, uint32_t len, uint8_t* s) {
  const uint32_t* g32 = reinterpret_cast<const uint32_t*>(g);
  uint32_t* s32 = reinterpret_cast<uint32_t*>(s);
  for (uint32_t i = threadIdx.x; i < len / 4; i += kCodecThreads) s32[i] = __ldg(&g32[i]);
  if (threadIdx.x < 4) s32[len / 4 + threadIdx.x] = 0;
}

template <typename T>
__device__ void decode_chunk(const DecodeArgs& a, const Hdr& h, uint32_t c, uint64_t off, uint32_t bsz, uint32_t ssz,
                             CodecSmem& sm) {
  using U = typename VT<T>::U;
  using I = typename VT<T>::I;
  constexpr int K = VT<T>::K;
  constexpr int W = kChunkBytes / K;
  constexpr int PER = W / kCodecThreads;
  U* WB = reinterpret_cast<U*>(sm.wb);
  U* WS = reinterpret_cast<U*>(sm.ws);
  const int tid = threadIdx.x;
  const uint8_t* pb = a.in + off;
  bool bad = false;

  // bins
  if (bsz == kChunkBytes) {
    const U* g = reinterpret_cast<const U*>(pb);
    for (int i = tid; i < W; i += kCodecThreads) WB[swz(i)] = g[i];
  } else {
    load_payload(pb, bsz, sm.ob);
    __syncthreads();
    uint32_t used = rze_decode(sm.ob, bsz, kChunkBytes, 1, sm.sh, sm.r);
    if (used == 0xffffffffu || pad4(used) != bsz) bad = true;
    if (!bad) {
      bit_inverse<U>(reinterpret_cast<const uint32_t*>(sm.sh), reinterpret_cast<U*>(sm.z), W);
      __syncthreads();
      // inverse negabinary + prefix sum (thread owns PER consecutive words)
      const U* Z = reinterpret_cast<const U*>(sm.z);
      U d[PER];
      U run = 0;
#pragma unroll
      for (int v = 0; v < PER; ++v) {
        U u = Z[swz(tid * PER + v)];
        d[v] = (U)((u ^ nb_mask<U>()) - nb_mask<U>());
        run += d[v];
      }
      U tot;
      U ex;
      if constexpr (sizeof(U) == 4)
        ex = block_scan_excl<uint32_t>(run, sm.r.wsum, &tot);
      else
        ex = (U)block_scan_excl<unsigned long long>((unsigned long long)run, sm.r.wsum64,
                                                     reinterpret_cast<unsigned long long*>(&tot));
      U acc = ex;
#pragma unroll
      for (int v = 0; v < PER; ++v) {
        acc += d[v];
        WB[swz(tid * PER + v)] = acc;
      }
    }
  }
  // subbins
  const uint8_t* ps = pb + bsz;
  if (!bad) {
    if (ssz == kChunkBytes) {
      const U* g = reinterpret_cast<const U*>(ps);
      for (int i = tid; i < W; i += kCodecThreads) WS[swz(i)] = g[i];
    } else {
      load_payload(ps, ssz, sm.os);
      __syncthreads();
      const uint32_t l1 = (uint32_t)sm.os[0] | ((uint32_t)sm.os[1] << 8);
      const uint32_t l1max = kChunkBytes + kChunkBytes / K / 8 + 64 + 8;
      if (l1 > l1max) bad = true;
      if (!bad) {
        uint32_t used = rze_decode(sm.os + 2, ssz - 2, l1, 1, sm.z, sm.r);
        if (used == 0xffffffffu || pad4(2 + used) != ssz) bad = true;
      }
      if (!bad) {
        if (tid < 16) sm.z[l1 + tid] = 0;
        __syncthreads();
        uint32_t used2 = rze_decode(sm.z, l1, kChunkBytes, K, sm.sh, sm.r);
        if (used2 != l1) bad = true;
      }
      if (!bad) {
        bit_inverse<U>(reinterpret_cast<const uint32_t*>(sm.sh), WS, W);
      }
    }
  }
  if (bad) {
    if (tid == 0) atomicOr(&a.ctr->err, kErrCorrupt);
    __syncthreads();
    return;
  }
  __syncthreads();
  // a8: x^ = value with key(lo(b)) + s, or the raw escape (G10)
  const uint64_t e0 = (uint64_t)c * W;
  const uint32_t cnt = (uint32_t)min((uint64_t)W, h.n - e0);
  T* O = static_cast<T*>(a.out) + e0;
#pragma unroll
  for (int v = 0; v < PER; ++v) {
    const int i = v * kCodecThreads + tid;
    if ((uint32_t)i < cnt) {
      U bw = WB[swz(i)], sw = WS[swz(i)];
      U bits;
      if (bw == VT<T>::kSentinel) {
        bits = sw;
      } else {
        int64_t b = (int64_t)(I)bw;
        T lo = lo_t<T>(b, h.eps);
        int64_t k = (int64_t)key_of((U)as_bits(lo)) + (int64_t)sw;
        if constexpr (sizeof(U) == 4)
          bits = bits_of_key32(k);
        else
          bits = bits_of_key64(k);
      }
      if constexpr (sizeof(U) == 4)
        O[i] = __uint_as_float(bits);
      else
        O[i] = __longlong_as_double((long long)bits);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kCodecThreads, 2) k_decode(DecodeArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  CodecSmem& sm = *reinterpret_cast<CodecSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const Hdr h = parse_header(a);
  if (!h.ok) {
    if (blockIdx.x == 0 && tid == 0) atomicOr(&a.ctr->err, h.err);
    return;
  }
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(a.in + kHdrBytes);
  for (;;) {
    if (tid < 32) {
      uint32_t c = 0;
      if (tid == 0) c = atomicAdd(&a.ctr->ticket, 1u);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (tid == 0) sm.misc[0] = c;
      if (c < h.C) {
        const uint32_t bs = tab[2 * c], ss = tab[2 * c + 1];
        bool ok = bs >= 4 && bs <= kChunkBytes && (bs & 3u) == 0 && ss >= 4 && ss <= kChunkBytes && (ss & 3u) == 0;
        const uint64_t agg = ok ? (uint64_t)bs + ss : (1ull << 40);  // poison keeps later offsets out of range
        const uint64_t excl = lookback_warp(a.state, c, agg);
        const uint64_t off = (uint64_t)kHdrBytes + 8ull * h.C + excl;
        if (!ok || off + bs + ss > a.in_bytes) ok = false;
        if (c == h.C - 1 && off + bs + ss != a.in_bytes) ok = false;
        if (tid == 0) {
          if (!ok) atomicOr(&a.ctr->err, kErrCorrupt);
          sm.misc[1] = ok;
          sm.misc[2] = bs;
          sm.misc[3] = ss;
          sm.misc64[0] = off;
        }
      }
    }
    __syncthreads();
    const uint32_t c = sm.misc[0];
    if (c >= h.C) break;
    if (sm.misc[1]) {
      if (h.dtype == 0)
        decode_chunk<float>(a, h, c, sm.misc64[0], sm.misc[2], sm.misc[3], sm);
      else
        decode_chunk<double>(a, h, c, sm.misc64[0], sm.misc[2], sm.misc[3], sm);
    }
    __syncthreads();
  }
}

}  // namespace lopc
