// Diagnostic: minimal TMA tile load through a __grid_constant__ CUtensorMap
// (variants), to check the descriptor path used by k_quant_flags.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int cx, int cy) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 36 * 66 * 4);
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(bar), sd = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb) : "memory");
    if (MODE == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(36 * 66 * 4) : "memory");
    if (MODE <= 1)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(sd),
                   "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(cx), "r"(cy), "r"(sb) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(sd),
                   "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(cx), "r"(cy), "r"(sb) : "memory");
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(sb) : "memory");
  for (int i = threadIdx.x; i < 36 * 66; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main(int argc, char** argv) {
  const int MODE = argc > 1 ? atoi(argv[1]) : 0, SHAPE = argc > 2 ? atoi(argv[2]) : 0, CX = argc > 3 ? atoi(argv[3]) : -1;
  const int BOXX = argc > 4 ? atoi(argv[4]) : 36, BOXY = argc > 5 ? atoi(argv[5]) : 66;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)fn;
  printf("entry %p q=%d\n", fn, (int)q);
  for (int shape = SHAPE; shape <= SHAPE; ++shape) {
    const int d1 = shape ? 500 : 3, d2 = shape ? 500 : 4;
    std::vector<float> h(d1 * d2);
    for (int i = 0; i < d1 * d2; ++i) h[i] = (float)i;
    float* x;
    cudaMalloc(&x, h.size() * 4);
    cudaMemcpy(x, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap m;
    const cuuint64_t gd[2] = {(cuuint64_t)d2, (cuuint64_t)d1}, gs[1] = {(cuuint64_t)d2 * 4};
    const cuuint32_t box[2] = {(cuuint32_t)BOXX, (cuuint32_t)BOXY}, es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("shape %d encode %d\n", shape, (int)r);
    float* out;
    cudaMalloc(&out, 36 * 66 * 4);
    const size_t smem = 36 * 66 * 4 + 64;
    for (int mode = MODE; mode <= MODE; ++mode) {
      cudaMemset(out, 0xff, 36 * 66 * 4);
      if (mode == 0) k<0><<<1, 128, smem>>>(m, out, CX, CX);
      if (mode == 1) k<1><<<1, 128, smem>>>(m, out, CX, CX);
      if (mode == 2) k<2><<<1, 128, smem>>>(m, out, CX, CX);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> o(36 * 66);
      cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost);
      printf("  mode %d: %s  o[0]=%g o[37]=%g o[38]=%g\n", mode, cudaGetErrorString(e), o[0], o[37], o[38]);
      if (e != cudaSuccess) return 1;
    }
    cudaFree(x);
    cudaFree(out);
  }
  return 0;
}
