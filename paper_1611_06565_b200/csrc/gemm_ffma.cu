// gemm_ffma.cu -- stage a3 on the CUDA cores (fp32 FMA), gemm_mode FFMA.
// The per-point GEMM of Eq. (5), M_xi = V_xi U_xi, with a
// 64 (tiles) x 64 (kernels) block tile and 16-channel smem chunks.  Each
// thread owns 4 x 4 outputs laid out so that a warp's stores to M[xi][k][t]
// cover consecutive t (coalesced).  Accumulation order: c ascending.
#include "kernels.h"

namespace wino {

__global__ void __launch_bounds__(256)
k_gemm_ffma(const float* __restrict__ V, const float* __restrict__ U, float* __restrict__ Mo, int64_t T,
            int64_t T_s, int C, int K, int K_s) {
  __shared__ float Vs[16][64];
  __shared__ float Us[16][64];
  const int xi = blockIdx.z;
  const int64_t t0 = (int64_t)blockIdx.x * 64;
  const int k0 = blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float* Vp = V + (int64_t)xi * C * T_s;
  const float* Up = U + (int64_t)xi * C * K_s;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int c0 = 0; c0 < C; c0 += 16) {
    for (int l = threadIdx.x; l < 1024; l += 256) {
      const int cc = l >> 6, tt = l & 63;
      Vs[cc][tt] = (c0 + cc < C && t0 + tt < T_s) ? Vp[(int64_t)(c0 + cc) * T_s + t0 + tt] : 0.f;
      Us[cc][tt] = (c0 + cc < C && k0 + tt < K_s) ? Up[(int64_t)(c0 + cc) * K_s + k0 + tt] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Vs[cc][tx + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Us[cc][ty + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = k0 + ty + 16 * j;
    if (k >= K) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t t = t0 + tx + 16 * i;
      if (t < T) Mo[((int64_t)xi * K + k) * T_s + t] = acc[i][j];
    }
  }
}

cudaError_t launch_gemm_ffma(const float* V, const float* U32, float* Mo, int P, int64_t T, int64_t T_s, int C,
                             int K, int K_s, cudaStream_t s) {
  dim3 grid((unsigned)((T + 63) / 64), (unsigned)((K + 63) / 64), (unsigned)P);
  k_gemm_ffma<<<grid, 256, 0, s>>>(V, U32, Mo, T, T_s, C, K, K_s);
  return cudaGetLastError();
}

}  // namespace wino
