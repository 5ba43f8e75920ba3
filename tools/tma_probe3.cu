// Diagnostic: minimal 3D TMA tile load through a __grid_constant__ CUtensorMap.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
constexpr int BX = 36, BY = 10, BZ = 10;

__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int cx, int cy, int cz) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BX * BY * BZ * 4);
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(bar), sd = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(BX * BY * BZ * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sd),
                 "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(cx), "r"(cy), "r"(cz), "r"(sb) : "memory");
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(sb) : "memory");
  for (int i = threadIdx.x; i < BX * BY * BZ; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main(int argc, char** argv) {
  const int cx = atoi(argv[1]), cy = atoi(argv[2]), cz = atoi(argv[3]);
  const int d0 = 100, d1 = 500, d2 = 500;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)fn;
  std::vector<float> h((size_t)d0 * d1 * d2);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 1000003);
  float* x;
  cudaMalloc(&x, h.size() * 4);
  cudaMemcpy(x, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  const cuuint64_t gd[3] = {(cuuint64_t)d2, (cuuint64_t)d1, (cuuint64_t)d0}, gs[2] = {(cuuint64_t)d2 * 4, (cuuint64_t)d1 * d2 * 4};
  const cuuint32_t box[3] = {BX, BY, BZ}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  float* out;
  cudaMalloc(&out, BX * BY * BZ * 4);
  k<<<1, 128, BX * BY * BZ * 4 + 64>>>(m, out, cx, cy, cz);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> o(BX * BY * BZ);
  cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost);
  const size_t g = ((size_t)cz * d1 + cy) * d2 + cx;
  printf("enc %d coords (%d,%d,%d): %s o[0]=%g expect %g; o[BX*BY+1]=%g expect %g\n", (int)r, cx, cy, cz,
         cudaGetErrorString(e), o[0], h[g], o[BX * BY + 1], h[g + (size_t)d1 * d2 + 1]);
  return 0;
}
