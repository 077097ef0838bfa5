// Dev probe: 3-D TMA tile load {128 t, 8 c, 1 p} (no swizzle) of a [P][C][T] float tensor whose
// innermost start coordinate is not a multiple of 4 elements (the direct-axis fold's tap shift).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_off_probe tools/tma_off_probe.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1611_06565_b200/csrc/tma.hpp"
using namespace wino;

__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int bytes, int c0, int c1, int c2) {
  extern __shared__ __align__(128) float S[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(S);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(sb), "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(mb) : "memory");
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(mb) : "memory");
  }
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = S[i];
}

int main() {
  const int T = 1024, C = 16, P = 2;
  float *x, *o;
  cudaMalloc(&x, (size_t)T * C * P * 4); cudaMalloc(&o, 1 << 20);
  float* hx = new float[T * C * P];
  for (int i = 0; i < T * C * P; ++i) hx[i] = (float)i;
  cudaMemcpy(x, hx, (size_t)T * C * P * 4, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[3] = {T, C, P}, strides[2] = {T * 4, (cuuint64_t)T * C * 4};
  cuuint32_t box[3] = {128, 8, 1}, es[3] = {1, 1, 1};
  CUresult r = get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int bytes = 128 * 8 * 4;
  float* h = new float[128 * 8];
  int bad = 0;
  const int starts[] = {0, 1, 2, 3, 5, 129, 897, 1023};
  for (int s : starts) {
    k<<<1, 128, bytes>>>(tm, o, bytes, s, 8, 1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("start %d: encode=%d err=%s\n", s, (int)r, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, o, bytes, cudaMemcpyDeviceToHost);
    int wrong = 0;
    for (int c = 0; c < 8; ++c)
      for (int t = 0; t < 128; ++t) {
        const float want = s + t < T ? (float)((1 * C + 8 + c) * T + s + t) : 0.f;
        if (h[c * 128 + t] != want) ++wrong;
      }
    printf("start %d: encode=%d ok, wrong=%d (first %g %g)\n", s, (int)r, wrong, h[0], h[1]);
    bad += wrong;
  }
  printf(bad ? "FAIL\n" : "PASS: unaligned innermost start coordinates load correctly\n");
  return bad != 0;
}
