// f16_probe.cu -- dev probe of tcgen05.mma.kind::f16 with A in TMEM (TS mode,
// packed fp16 pairs written by tcgen05.st) and B MN-major in shared memory
// loaded by TMA with 128-byte swizzle: checks the descriptor / layout
// conventions against a CPU product before they are used in a kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1611_06565_b200/csrc f16_probe.cu -o f16_probe
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"
#include "tma.hpp"

using namespace wino::tc;

constexpr int KT = 32;   // K of the test (2 MMAs of K=16)

__device__ __forceinline__ uint64_t sdesc16(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

template <int N>
__global__ void k_probe(const __grid_constant__ CUtensorMap tmB, const __half* __restrict__ A, float* __restrict__ D,
                        uint32_t lbo, uint32_t sbo, uint32_t layout, uint32_t kstep_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sb = (smem_u32(smem) + 1023u) & ~1023u;
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(smem_u32(&bar[0]), 1);
      mbar_init(smem_u32(&bar[1]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&holder)),
                 "r"(256u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  // B via TMA: boxes {64 N, KT K} at N offsets 0, 64, ... -> smem + gq * KT * 128
  if (threadIdx.x == 0) {
    mbar_expect_tx(smem_u32(&bar[0]), (uint32_t)(N * KT * 2));
    for (int gq = 0; gq < N / 64; ++gq) tma_load_3d(sb + gq * KT * 128, &tmB, gq * 64, 0, 0, smem_u32(&bar[0]));
  }
  // A into TMEM columns [128, 128 + KT/2): lane = row, column j holds (A[r][2j], A[r][2j+1])
  {
    const int row = warp * 32 + lane;
    uint32_t w[8];
    for (int c0 = 0; c0 < KT / 2; c0 += 8) {
      for (int j = 0; j < 8; ++j) {
        const __half lo = A[row * KT + 2 * (c0 + j)], hi = A[row * KT + 2 * (c0 + j) + 1];
        w[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      tmem_st8(tm + ((uint32_t)(warp * 32) << 16) + 128 + c0, w);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    mbar_wait(smem_u32(&bar[0]), 0);
    tc_fence_after();
    // kind::f16: D f32 (bit 4), A = B = f16 (0), A K-major (TMEM), B MN-major (bit 16)
    constexpr uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (elect_one()) {
      for (int k = 0; k < KT / 16; ++k) {
        const uint64_t bd = sdesc16(sb + k * kstep_bytes, lbo, sbo, layout);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
            "r"(tm + 128 + 8 * k), "l"(bd), "r"(idesc), "r"(k > 0 ? 1u : 0u)
            : "memory");
      }
      tc_commit(smem_u32(&bar[1]));
    }
    __syncwarp();
  }
  mbar_wait(smem_u32(&bar[1]), 0);
  tc_fence_after();
  {
    const int row = warp * 32 + lane;
    for (int cb = 0; cb < N; cb += 32) {
      uint32_t r[32];
      tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + cb, r);
      for (int j = 0; j < 32; ++j) D[row * N + cb + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256u) : "memory");
  }
}

template <int N>
int run(uint32_t lbo, uint32_t sbo, uint32_t layout, uint32_t kstep) {
  std::vector<__half> hA(128 * KT), hB(KT * N);
  std::vector<float> fA(128 * KT), fB(KT * N);
  srand(1);
  for (int i = 0; i < 128 * KT; ++i) { float v = (rand() % 17) - 8; hA[i] = __float2half(v); fA[i] = v; }
  for (int i = 0; i < KT * N; ++i) { float v = (rand() % 13) - 6; hB[i] = __float2half(v); fB[i] = v; }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  // B [K][N] row-major (N contiguous): TMA dims (N, K, 1), box {64, KT, 1}, 128B swizzle
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)KT, 1};
  cuuint64_t strides[2] = {(cuuint64_t)N * 2, (cuuint64_t)N * 2 * KT};
  cuuint32_t box[3] = {64, (cuuint32_t)KT, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult cr = wino::get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, dB, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
  cudaFuncSetAttribute(k_probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_probe<N><<<1, 128, 64 * 1024>>>(tm, dA, dD, lbo, sbo, layout, kstep);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> D(128 * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      float ref = 0;
      for (int k = 0; k < KT; ++k) ref += fA[i * KT + k] * fB[k * N + j];
      if (D[i * N + j] != ref) ++bad;
    }
  printf("N=%d lbo=%u sbo=%u layout=%u kstep=%u: %s, %d / %d wrong (D[0]=%g D[1]=%g)\n", N, lbo, sbo, layout, kstep,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), bad, 128 * N, D[0], D[1]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad;
}

int main() {
  // candidates: layout 2 = SWIZZLE_128B; LBO = distance between 64-element
  // groups along N (KT * 128 B); SBO = 8 K-rows (1024 B); next K=16 step at
  // +16 rows (2048 B)
  run<64>(KT * 128, 1024, 2, 2048);
  run<128>(KT * 128, 1024, 2, 2048);
  run<64>(1024, KT * 128, 2, 2048);
  run<128>(1024, KT * 128, 2, 2048);
  return 0;
}
