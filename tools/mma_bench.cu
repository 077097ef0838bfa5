// mma_bench.cu -- dev microbenchmark: issue rate of tcgen05.mma.kind::tf32
// (M = 128, K = 8) from one thread, per N and A-operand source (TMEM "TS" or
// shared memory "SS"), one accumulator chain vs alternating accumulators.
// Prints cycles per MMA (clock64 around L MMAs + commit + wait) on one SM
// and on all SMs at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1611_06565_b200/csrc mma_bench.cu -o mma_bench
#include <cstdio>
#include <cstdlib>

#include "tc_common.cuh"

using namespace wino::tc;

__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int N, bool TS, bool F16 = false>
__global__ void __launch_bounds__(128, 1) k_mma_rate(unsigned long long* out, int L, int nacc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const uint32_t sb = smem_u32(smem);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      mbar_init(smem_u32(&bar), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&holder)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  if (warp == 0) {
    constexpr uint32_t idesc = F16 ? ((1u << 4) | (TS ? 0u : (1u << 15)) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
                                      ((uint32_t)(128 >> 4) << 24))
                                   : TS ? idesc_tf32_ts<N>() : idesc_tf32<N>();
    const uint64_t db = sdesc(sb + 32768, 8u * 128u, 512u);   // B: 8 K-rows x N (MN-major)
    const uint64_t da = sdesc(sb, 8u * 128u, 512u);           // A (SS mode)
    const uint32_t a_t = tm + 256;                            // A columns in TMEM (TS mode)
    unsigned long long t0 = 0, t1 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      __syncwarp();
      t0 = clock64();
      if (elect_one()) {
        if (nacc == 0) {   // unrolled by 16, constant operands (issue cost only)
          for (int i = 0; i < L; i += 16) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if constexpr (F16) {
                if constexpr (TS) mma_f16_ts(tm, a_t, db, idesc, 1u);
                else mma_f16_ss(tm, da, db, idesc, 1u);
              } else {
                if constexpr (TS) tc_mma_tf32_ts(tm, a_t, db, idesc, 1u);
                else tc_mma_tf32(tm, da, db, idesc, 1u);
              }
            }
          }
        } else {
          for (int i = 0; i < L; ++i) {
            const uint32_t d = tm + (uint32_t)((i % nacc) * N);
            if constexpr (TS) tc_mma_tf32_ts(d, a_t, db, idesc, i >= nacc ? 1u : 0u);
            else tc_mma_tf32(d, da, db, idesc, i >= nacc ? 1u : 0u);
          }
        }
        tc_commit(smem_u32(&bar));
      }
      __syncwarp();
      mbar_wait(smem_u32(&bar), (uint32_t)rep);
      t1 = clock64();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512u) : "memory");
  }
}

template <int N, bool TS, bool F16 = false>
void run(int grid, int L, int nacc) {
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  auto k = k_mma_rate<N, TS, F16>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<grid, 128, 64 * 1024>>>(d, L, nacc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  double mx = 0, sum = 0;
  for (int i = 0; i < grid; ++i) { sum += h[i]; if (h[i] > mx) mx = h[i]; }
  printf("%s%s N=%3d grid=%3d nacc=%d L=%d: %6.1f cycles/MMA (mean), %6.1f (max)  %s\n", F16 ? "f16 " : "tf32 ",
         TS ? "TS" : "SS", N, grid, nacc,
         L, sum / grid / L, mx / L, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  const int L = 3008;
  run<128, true, true>(1, L, 0);
  run<128, false, true>(1, L, 0);
  run<256, true, true>(1, L, 0);
  run<64, true, true>(1, L, 0);
  for (int grid : {1}) {
    for (int nacc : {0}) {
      run<32, true>(grid, L, nacc);
      run<64, true>(grid, L, nacc);
      run<128, true>(grid, L, nacc);
      run<32, false>(grid, L, nacc);
      run<64, false>(grid, L, nacc);
      run<128, false>(grid, L, nacc);
      run<256, true>(grid, L, nacc);
      run<256, false>(grid, L, nacc);
    }
  }
  return 0;
}
