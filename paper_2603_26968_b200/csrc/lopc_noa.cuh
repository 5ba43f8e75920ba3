// lopc_noa.cuh — SURVEY §8(f) f1 / row a0 on the device: the NOA error bound
// eps = rel * (max - min) over the finite values ("NOA"), from one
// fused min/max read of x.  Included by lopc_api.cu.
#pragma once

namespace lopc {

// min / max as order-preserving keys (key_of): one atomicMin/atomicMax per
// block.  Non-finite values (NaN, +-Inf) are skipped; n_finite counts the rest.
struct RangeOut {
  long long kmin, kmax;
  unsigned long long n_finite;
};

template <typename T>
__global__ void __launch_bounds__(256) k_value_range(const T* __restrict__ x, uint64_t n, RangeOut* out) {
  using U = typename VT<T>::U;
  using I = typename VT<T>::I;
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  unsigned long long cnt = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (sizeof(T) == 4) {
    const uint64_t n4 = n / 4;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const bool vec = ((uintptr_t)x & 15) == 0;
    if (vec) {
      for (uint64_t j = i; j < n4; j += stride) {
        const float4 v = __ldcs(x4 + j);
        const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const U u = __float_as_uint(vs[q]);
          if ((u & 0x7f800000u) != 0x7f800000u) {
            const long long kk = key_of(u);
            lo = kk < lo ? kk : lo;
            hi = kk > hi ? kk : hi;
            ++cnt;
          }
        }
      }
      i = n4 * 4 + i;
    }
  }
  for (; i < n; i += stride) {
    const U u = (U)as_bits(x[i]);
    if ((u & VT<T>::kInfBits) != VT<T>::kInfBits) {
      const long long kk = (long long)(I)key_of(u);
      lo = kk < lo ? kk : lo;
      hi = kk > hi ? kk : hi;
      ++cnt;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  __shared__ long long slo[8], shi[8];
  __shared__ unsigned long long sc[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    slo[w] = lo;
    shi[w] = hi;
    sc[w] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      lo = min(lo, slo[k]);
      hi = max(hi, shi[k]);
      cnt += sc[k];
    }
    if (cnt) {
      atomicMin(&out->kmin, lo);
      atomicMax(&out->kmax, hi);
      atomicAdd(&out->n_finite, cnt);
    }
  }
}

}  // namespace lopc
