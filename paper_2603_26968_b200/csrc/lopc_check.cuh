// lopc_check.cuh — the device-side checker of SURVEY §8(d.1) ("order
// violations ... counted by k_check") and the error
// statistics of NEXT f3 (max |x - x^|, sum of squares for PSNR).
// Semantics are those of O13: an order violation is a star edge {p, p+e}
// (each edge once) with finite, non-NaN x at both ends whose SoS order
// (ord, then index) differs between x and x^; a bound violation is an escaped
// point not kept bit-exactly, or a regular point without 0 <= x - x^ <= eps
// in exact arithmetic.  Included by lopc_api.cu.
#pragma once

namespace lopc {

struct CheckOut {
  unsigned long long order_bad, bound_bad, n_regular;
  unsigned long long max_err_bits;  // max |x - x^| over regular points, as double bits (>= 0: monotone)
  double sum_sq;
};

template <typename T, int NDIM>
__global__ void __launch_bounds__(256) k_check(const T* __restrict__ x, const T* __restrict__ y, int64_t d0, int64_t d1,
                                               int64_t d2, double eps, double inv, float inv32, CheckOut* out) {
  using U = typename VT<T>::U;
  using I = typename VT<T>::I;
  constexpr int D = Geo<NDIM>::D;
  const int64_t plane = d1 * d2, n = d0 * plane;
  unsigned long long obad = 0, bbad = 0, nreg = 0;
  double mx = 0.0, ss = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const T xp = x[p], yp = y[p];
    const U bx = (U)as_bits(xp), by = (U)as_bits(yp);
    // bound (exact: TwoSum of the difference)
    I b;
    if (!quantize_fast<T>(xp, inv32, eps, inv, b)) {
      bbad += bx != by;
    } else {
      ++nreg;
      const double a = (double)xp, c = (double)yp;
      if (!(c <= a)) {
        ++bbad;
      } else {
        const double dd = a - c, bb = dd - a, err = (a - (dd - bb)) + (-c - bb);
        if (!(dd < eps || (dd == eps && err <= 0))) ++bbad;
        mx = dd > mx ? dd : mx;
        ss += dd * dd;
      }
    }
    // order on the +e star edges of p
    if (xp != xp) continue;  // NaN: no order (G11)
    const int64_t z = p / plane, r2 = p - z * plane, yy = r2 / d2, xx = r2 - yy * d2;
    const I kxp = (I)key_of(bx), kyp = (I)key_of(by);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int e = j + 1;
      const int dz = NDIM == 3 ? (e >> 2) & 1 : 0, dy = (e >> 1) & 1, dx = e & 1;
      if (z + dz >= d0 || yy + dy >= d1 || xx + dx >= d2) continue;
      const int64_t q = p + dz * plane + dy * d2 + dx;
      const T xq = x[q], yq = y[q];
      if (xq != xq) continue;
      const bool lx = kxp <= (I)key_of((U)as_bits(xq));  // p < q: ties order p first
      const bool ly = kyp <= (I)key_of((U)as_bits(yq));
      obad += (yp != yp || yq != yq || lx != ly);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    obad += __shfl_xor_sync(0xffffffffu, obad, o);
    bbad += __shfl_xor_sync(0xffffffffu, bbad, o);
    nreg += __shfl_xor_sync(0xffffffffu, nreg, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (obad) atomicAdd(&out->order_bad, obad);
    if (bbad) atomicAdd(&out->bound_bad, bbad);
    if (nreg) atomicAdd(&out->n_regular, nreg);
    atomicMax(&out->max_err_bits, (unsigned long long)__double_as_longlong(mx));
    atomicAdd(&out->sum_sq, ss);
  }
}

}  // namespace lopc

namespace lopc {

// ---------------------------------------------------------------------------
// k_critical: PL critical points of x and x^ under SoS (G5: an empty
// lower link is a minimum) on the Kuhn/Freudenthal triangulation, and the
// Table III comparison: false positives / negatives / types, plus the
// stronger (#lower, #upper link components) mismatch count (G27).  The link
// of p is its star neighbours joined by the link edges (adj: for each slot,
// the slots whose offsets differ by a star offset = the triangles through p,
// 6 edges in 2D, 36 in 3D); out-of-grid and NaN neighbours drop out.
// ---------------------------------------------------------------------------
struct CritOut {
  unsigned long long fp, fn, ft, pair_bad, crit_x, crit_y;
};
struct LinkAdj {
  uint16_t adj[14];
};

__device__ __forceinline__ int link_components(uint32_t m, const LinkAdj& L) {
  int c = 0;
  while (m) {
    uint32_t comp = m & (0u - m), prev = 0;
    while (comp != prev) {
      prev = comp;
      uint32_t g = comp;
      for (uint32_t t = comp; t; t &= t - 1) g |= L.adj[__ffs(t) - 1];
      comp = g & m;
    }
    m &= ~comp;
    ++c;
  }
  return c;
}

// type: 0 regular, 1 min, 2 max, 3 saddle
__device__ __forceinline__ int crit_type(int nl, int nu) {
  return nl == 0 ? 1 : (nu == 0 ? 2 : ((nl == 1 && nu == 1) ? 0 : 3));
}

template <typename T, int NDIM>
__global__ void __launch_bounds__(256) k_critical(const T* __restrict__ x, const T* __restrict__ y, int64_t d0,
                                                  int64_t d1, int64_t d2, LinkAdj L, CritOut* out) {
  constexpr int D = Geo<NDIM>::D;
  const int64_t plane = d1 * d2, n = d0 * plane;
  unsigned long long fp = 0, fn = 0, ft = 0, pb = 0, cx = 0, cy = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const T xp = x[p], yp = y[p];
    if (xp != xp) continue;
    const int64_t z = p / plane, r2 = p - z * plane, yy = r2 / d2, xx = r2 - yy * d2;
    uint32_t in = 0, lx = 0, ly = 0;
#pragma unroll
    for (int j = 0; j < 2 * D; ++j) {
      const int e = (j < D ? j : j - D) + 1, sg = j < D ? 1 : -1;
      const int dz = NDIM == 3 ? sg * ((e >> 2) & 1) : 0, dy = sg * ((e >> 1) & 1), dx = sg * (e & 1);
      const int64_t qz = z + dz, qy = yy + dy, qx = xx + dx;
      if (qz < 0 || qz >= d0 || qy < 0 || qy >= d1 || qx < 0 || qx >= d2) continue;
      const int64_t q = p + dz * plane + dy * d2 + dx;
      const T xq = x[q], yq = y[q];
      if (xq != xq) continue;
      in |= 1u << j;
      // SoS: q below p iff smaller value, or equal value and smaller index
      lx |= (uint32_t)(xq < xp || (xq == xp && q < p)) << j;
      ly |= (uint32_t)(yq < yp || (yq == yp && q < p)) << j;
    }
    const int nlx = link_components(lx, L), nux = link_components(in & ~lx, L);
    const int nly = link_components(ly, L), nuy = link_components(in & ~ly, L);
    const int tx = crit_type(nlx, nux), ty = crit_type(nly, nuy);
    cx += tx != 0;
    cy += ty != 0;
    fp += tx == 0 && ty != 0;
    fn += tx != 0 && ty == 0;
    ft += tx != 0 && ty != 0 && tx != ty;
    pb += nlx != nly || nux != nuy;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    fp += __shfl_xor_sync(0xffffffffu, fp, o);
    fn += __shfl_xor_sync(0xffffffffu, fn, o);
    ft += __shfl_xor_sync(0xffffffffu, ft, o);
    pb += __shfl_xor_sync(0xffffffffu, pb, o);
    cx += __shfl_xor_sync(0xffffffffu, cx, o);
    cy += __shfl_xor_sync(0xffffffffu, cy, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (fp) atomicAdd(&out->fp, fp);
    if (fn) atomicAdd(&out->fn, fn);
    if (ft) atomicAdd(&out->ft, ft);
    if (pb) atomicAdd(&out->pair_bad, pb);
    if (cx) atomicAdd(&out->crit_x, cx);
    if (cy) atomicAdd(&out->crit_y, cy);
  }
}

}  // namespace lopc
