// lopc_device.cuh — device primitives of the LOPC hot path (sm_100a).
//
// Product code.  Shares nothing with the CPU reference implementation: the two are
// written independently from PAPER.md and DESIGN.md §3-§4 and compared only
// through their outputs.
//
// Compiled with -fmad=false: no FMA contraction anywhere; __fma_rn is used
// explicitly only for the TwoProduct error term of lo().
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace lopc {

constexpr uint32_t kChunkBytes = 16384;  // "16kB chunks" (G22)
constexpr uint32_t kHdrBytes = 64;

// Value-type traits: word width k, bin/ord integer types, escape sentinel
// (G10), BINMAX (G8).
template <typename T>
struct VT;
template <>
struct VT<float> {
  using U = uint32_t;  // raw bits / stream word
  using I = int32_t;   // bin and ord
  static constexpr int K = 4;
  static constexpr U kSentinel = 0x80000000u;
  static constexpr U kSignBit = 0x80000000u;
  static constexpr U kInfBits = 0x7f800000u;
  static constexpr double kBinMax = 2147483646.0;
};
template <>
struct VT<double> {
  using U = uint64_t;
  using I = int64_t;
  static constexpr int K = 8;
  static constexpr U kSentinel = 0x8000000000000000ull;
  static constexpr U kSignBit = 0x8000000000000000ull;
  static constexpr U kInfBits = 0x7ff0000000000000ull;
  static constexpr double kBinMax = 1125899906842624.0;
};

__host__ __device__ __forceinline__ uint32_t as_bits(float v) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(v);
#else
  uint32_t u;
  __builtin_memcpy(&u, &v, 4);
  return u;
#endif
}
__host__ __device__ __forceinline__ uint64_t as_bits(double v) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(v);
#else
  uint64_t u;
  __builtin_memcpy(&u, &v, 8);
  return u;
#endif
}

// SoS value key: monotone map of the bit pattern to an integer,
// -0.0 and +0.0 both map to 0 (G13).
__device__ __forceinline__ int32_t key_of(uint32_t u) {
  int32_t i = (int32_t)u;
  return i >= 0 ? i : -(int32_t)(u & 0x7fffffffu);
}
__device__ __forceinline__ int64_t key_of(uint64_t u) {
  int64_t i = (int64_t)u;
  return i >= 0 ? i : -(int64_t)(u & 0x7fffffffffffffffull);
}
__device__ __forceinline__ uint32_t bits_of_key32(int64_t o) {
  return o >= 0 ? (uint32_t)o : (0x80000000u | (uint32_t)(-o));
}
__device__ __forceinline__ uint64_t bits_of_key64(int64_t o) {
  return o >= 0 ? (uint64_t)o : (0x8000000000000000ull | (uint64_t)(-o));
}

// 1.5 * 2^52: adding it rounds a double of magnitude < 2^51 to an integer
// held in the low mantissa bits (no F2I/I2F conversions needed).
constexpr double kMagic = 6755399441055744.0;

__device__ __forceinline__ double i64_to_f64_exact(int64_t b) {
  // exact for |b| < 2^51
  return __longlong_as_double(__double_as_longlong(kMagic) + b) - kMagic;
}

// lo(b): the smallest dtype value >= (b - 1/2) * eps, exactly ("subbin 0
// decodes to the lowest representable value within the bin"; G7).
// a = b - 1/2 is exact; a*eps = p + e exactly with e = fma(a, eps, -p).
__device__ __forceinline__ float lo_f32(int64_t b, double eps) {
  double a = i64_to_f64_exact(b) - 0.5;
  double p = __dmul_rn(a, eps);
  double e = __fma_rn(a, eps, -p);
  float f = __double2float_ru(p);  // smallest float >= p
  if (e > 0.0 && (double)f == p) f = __uint_as_float(bits_of_key32((int64_t)key_of(__float_as_uint(f)) + 1));
  return f;
}
__device__ __forceinline__ double lo_f64(int64_t b, double eps) {
  double a = i64_to_f64_exact(b) - 0.5;
  double p = __dmul_rn(a, eps);
  double e = __fma_rn(a, eps, -p);
  if (e > 0.0) p = __longlong_as_double((long long)bits_of_key64(key_of((uint64_t)__double_as_longlong(p)) + 1));
  return p;
}
template <typename T>
__device__ __forceinline__ T lo_t(int64_t b, double eps);
template <>
__device__ __forceinline__ float lo_t<float>(int64_t b, double eps) { return lo_f32(b, eps); }
template <>
__device__ __forceinline__ double lo_t<double>(int64_t b, double eps) { return lo_f64(b, eps); }

// key(lo(b)) directly (the only form the kernels need): the same rounding as
// lo_f32 / lo_f64, with the rare exact-product check off the common path.
__device__ __forceinline__ int32_t lo_key32(int64_t b, double eps) {
  const double a = i64_to_f64_exact(b) - 0.5;
  const double p = __dmul_rn(a, eps);
  const float f = __double2float_ru(p);
  int32_t k = key_of(__float_as_uint(f));
  if ((double)f == p && __fma_rn(a, eps, -p) > 0.0) k += 1;  // p exact in f32 but below a*eps
  return k;
}
// lo_key32 without branches, for a regular f32 bin (|b| < 2^31; any b gives
// some value, so the caller may select it away for escapes).  The key stays
// in int32: |key(lo(b)) + s| < 2^31 for a regular point (its decoded value is
// a finite float).
__device__ __forceinline__ int32_t lo_key32_nb(int32_t b, double eps) {
  const double a = __dadd_rn(i64_to_f64_exact(b), -0.5);
  const double p = __dmul_rn(a, eps);
  const float f = __double2float_ru(p);
  const uint32_t u = __float_as_uint(f);
  const int32_t k = (int32_t)u >= 0 ? (int32_t)u : -(int32_t)(u & 0x7fffffffu);
  return k + (int32_t)(((double)f == p) & (__fma_rn(a, eps, -p) > 0.0));
}
__device__ __forceinline__ int64_t lo_key64(int64_t b, double eps) {
  const double a = i64_to_f64_exact(b) - 0.5;
  const double p = __dmul_rn(a, eps);
  return key_of((uint64_t)__double_as_longlong(p)) + (__fma_rn(a, eps, -p) > 0.0 ? 1 : 0);
}
template <typename T>
__device__ __forceinline__ typename VT<T>::I lo_key(int64_t b, double eps);
template <>
__device__ __forceinline__ int32_t lo_key<float>(int64_t b, double eps) { return lo_key32(b, eps); }
template <>
__device__ __forceinline__ int64_t lo_key<double>(int64_t b, double eps) { return lo_key64(b, eps); }

// Exact bin b = floor(x/eps + 1/2) (P:114 with reading G6) and the
// double-check of the north star: returns false (escape) for non-finite x or
// |b| > BINMAX (G8/G9).
//
// t = RN(x * RN(1/eps)) differs from x/eps by less than |t| 2^-51.  If t is
// farther than that from a half-integer, b = rint(t) is proven exact;
// otherwise b is fixed up by the exact interval test lo(b) <= x < lo(b+1)
// (one step suffices: |t - x/eps| < 1/4 whenever |t| <= 2^51).
template <typename T>
__device__ __forceinline__ bool quantize(T x, double eps, double inv, typename VT<T>::I& bout) {
  using I = typename VT<T>::I;
  double xd = (double)x;
  double t = xd * inv;
  // NaN/Inf fail the compare; |t| > 2 BINMAX certainly means |b| > BINMAX
  if (!(fabs(t) <= 2.0 * VT<T>::kBinMax)) return false;
  double tm = t + kMagic;
  int64_t r = __double_as_longlong(tm) - __double_as_longlong(kMagic);
  double rd = tm - kMagic;
  double d = fabs(t - rd);
  double margin = 0.5 - fabs(t) * 0x1p-50 - 0x1p-60;
  if (!(d < margin)) {
    if (xd < (double)lo_t<T>(r, eps))
      r -= 1;
    else if (xd >= (double)lo_t<T>(r + 1, eps))
      r += 1;
  }
  if (r > (int64_t)VT<T>::kBinMax || r < -(int64_t)VT<T>::kBinMax) return false;
  bout = (I)r;
  return true;
}

// f32 data: a float fast path in front of the exact double path.
// inv32 = RN32(1/eps) (0 disables the fast path; the host sets it only for
// 2^-120 < eps < 2^120).  t = RN32(x * inv32) differs from x/eps by less than
// |t| 2^-22; if t is farther than |t| 2^-21 from a half-integer and |t| <
// 2^22, b = rint(t) is exact.  Otherwise the exact double path decides.
__device__ __forceinline__ bool quantize_f32(float x, float inv32, double eps, double inv, int32_t& bout) {
  const float t = __fmul_rn(x, inv32);
  const float at = fabsf(t);
  if (at < 4194304.0f) {
    const float tm = __fadd_rn(t, 12582912.0f);  // 1.5 * 2^23: rint for |t| < 2^22
    const float r = __fsub_rn(tm, 12582912.0f);
    const float margin = __fsub_rn(0.5f, __fmul_rn(at, 0x1p-21f));
    if (fabsf(__fsub_rn(t, r)) < margin) {
      bout = (int32_t)(__float_as_uint(tm) - __float_as_uint(12582912.0f));
      return true;
    }
  }
  return quantize<float>(x, eps, inv, bout);
}

template <typename T>
__device__ __forceinline__ bool quantize_fast(T x, float inv32, double eps, double inv, typename VT<T>::I& b);
template <>
__device__ __forceinline__ bool quantize_fast<float>(float x, float inv32, double eps, double inv, int32_t& b) {
  return quantize_f32(x, inv32, eps, inv, b);
}
template <>
__device__ __forceinline__ bool quantize_fast<double>(double x, float, double eps, double inv, int64_t& b) {
  return quantize<double>(x, eps, inv, b);
}

// Split form of quantize for the codec's bulk loops: qtry_* is the
// branch-free fast attempt (returns true when it decides b, which then is the
// exact bin, in range); quantize_slow is the exact path out of line (returns
// kEscape for an escape).
constexpr int64_t kEscape = INT64_MIN;

__device__ __forceinline__ bool qtry(float x, float inv32, double, int32_t& b) {
  const float t = __fmul_rn(x, inv32);
  const float at = fabsf(t);
  const float tm = __fadd_rn(t, 12582912.0f);
  const float r = __fsub_rn(tm, 12582912.0f);
  const float margin = __fsub_rn(0.5f, __fmul_rn(at, 0x1p-21f));
  b = (int32_t)(__float_as_uint(tm) - __float_as_uint(12582912.0f));
  return (at < 4194304.0f) & (fabsf(__fsub_rn(t, r)) < margin);
}
__device__ __forceinline__ bool qtry(double x, float, double inv, int64_t& b) {
  const double t = x * inv;
  const double at = fabs(t);
  const double tm = t + kMagic;
  const double rd = tm - kMagic;
  const double margin = 0.5 - at * 0x1p-50 - 0x1p-60;
  b = __double_as_longlong(tm) - __double_as_longlong(kMagic);
  return (at <= (double)(VT<double>::kBinMax - 1)) & (fabs(t - rd) < margin);
}
template <typename T>
__device__ __noinline__ int64_t quantize_slow(T x, double eps, double inv) {
  typename VT<T>::I b;
  return quantize<T>(x, eps, inv, b) ? (int64_t)b : kEscape;
}

// ---- memory-model helpers ------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

}  // namespace lopc
