// mma_pair_bench.cu -- dev microbenchmark: cycles per tcgen05.mma.cta_group::2
// (M = 256 over a CTA pair) for kind::tf32 (K = 8) and kind::f16 (K = 16),
// A in TMEM (TS) or shared memory (SS), one thread issuing an unrolled stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1611_06565_b200/csrc mma_pair_bench.cu -o mma_pair_bench
#include <cstdio>

#include "tc_common.cuh"

using namespace wino::tc;

template <int N, bool F16, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_pair(unsigned long long* out, int L) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  const uint32_t sb = smem_u32(smem);
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      mbar_init(smem_u32(&bar), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&holder)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tm = holder;
  constexpr uint32_t idesc = F16 ? ((1u << 4) | (TS ? 0u : (1u << 15)) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
                                    ((uint32_t)(256 >> 4) << 24))
                                 : ((1u << 4) | (2u << 7) | (2u << 10) | (TS ? 0u : (1u << 15)) | (1u << 16) |
                                    ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24));
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0 && rank == 0) {
    const uint64_t db = sdesc(sb + 32768, 16u * 128u, 512u);
    const uint64_t da = sdesc(sb, 16u * 128u, 512u);
    const uint32_t a_t = tm + 256;
    __syncwarp();
    t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < L; i += 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if constexpr (F16) {
            if constexpr (TS)
              asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(tm), "r"(a_t), "l"(db),
                           "r"(idesc) : "memory");
            else
              asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tm), "l"(da), "l"(db),
                           "r"(idesc) : "memory");
          } else {
            if constexpr (TS)
              asm volatile("tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(tm), "r"(a_t), "l"(db),
                           "r"(idesc) : "memory");
            else
              asm volatile("tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tm), "l"(da), "l"(db),
                           "r"(idesc) : "memory");
          }
        }
      }
      tc2_commit_mc(smem_u32(&bar));
    }
    __syncwarp();
  }
  if (warp == 0) {
    mbar_wait(smem_u32(&bar), 0);
    t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[blockIdx.x / 2] = t1 - t0;
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512u) : "memory");
  }
}

template <int N, bool F16, bool TS>
void run(int L) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 128);
  auto k = k_pair<N, F16, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  k<<<2, 128, 48 * 1024>>>(d, L);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("pair %s %s N=%3d: %6.1f cycles/MMA %s\n", F16 ? "f16 " : "tf32", TS ? "TS" : "SS", N, (double)h / L,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  const int L = 3008;
  run<128, false, true>(L);
  run<128, true, true>(L);
  run<128, false, false>(L);
  run<128, true, false>(L);
  run<256, false, true>(L);
  run<256, true, true>(L);
  run<64, true, true>(L);
  return 0;
}
