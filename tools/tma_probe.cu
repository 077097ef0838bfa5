// Dev probe: 3-D TMA tile load with negative start coordinates (zero fill).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1611_06565_b200/csrc/tma.hpp"
using namespace wino;

__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int bytes, int c0, int c1) {
  extern __shared__ __align__(128) float S[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(S);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(sb), "l"(&tm), "r"(c0), "r"(c1), "r"(0), "r"(mb) : "memory");
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(mb) : "memory");
  }
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = S[i];
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  const int W = 56, H = 56, BC = 4;
  float* x; float* o;
  cudaMalloc(&x, W * H * BC * 4); cudaMalloc(&o, 1 << 20);
  float* hx = new float[W * H * BC];
  for (int i = 0; i < W * H * BC; ++i) hx[i] = (float)(i % 1000) + 1;
  cudaMemcpy(x, hx, W * H * BC * 4, cudaMemcpyHostToDevice);
  int cases[][4] = {{60, 58, -1, -1}, {60, 58, 0, 0}, {8, 8, 0, 0}, {8, 8, -1, -1}, {64, 58, -1, -1}, {60, 58, -4, -1}, {64, 64, 0, 0}, {32, 58, 0, 0}, {60, 32, 0, 0}, {60, 16, 0, 0}};
  {
    auto& cs = cases[which];
    CUtensorMap tm;
    cuuint64_t dims[3] = {W, H, BC}, strides[2] = {W * 4, W * H * 4};
    cuuint32_t box[3] = {(cuuint32_t)cs[0], (cuuint32_t)cs[1], 1}, es[3] = {1, 1, 1};
    CUresult r = get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int bytes = cs[0] * cs[1] * 4;
    k<<<1, 128, bytes>>>(tm, o, bytes, cs[2], cs[3]);
    cudaError_t e = cudaDeviceSynchronize();
    float h[4] = {0, 0, 0, 0};
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("box %dx%d start (%d,%d): encode=%d err=%s first=%g %g %g %g\n", cs[0], cs[1], cs[2], cs[3], (int)r,
           cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
