// xform_out.cu -- host dispatch of stage a4 and stage a1, the filter
// transform:  U_xi[c][k] = (g[k, c] x_1 G ... x_N G)_xi  (Eq. (4),
// PAPER.md:160-164; cached transformed kernels PAPER.md:178).
#include <cstdlib>

#include "kernels.h"
#include "tma.hpp"
#include "xform_out.cuh"

namespace wino {

// ------------------------------------------------------------------ a1
// One thread per (xi, c, k) (k fastest -> coalesced U writes):
//   U_xi[c][k] = sum_p prod_n G_n[xi_n][p_n] g[k, c, p]   (G_n per axis)
// in fp64, rounded once to fp32, then split for 3xTF32:
//   hi = rna_tf32(u), lo = rna_tf32(u - hi)     (reading #7).
__global__ void __launch_bounds__(256)
k_filter_xform(const float* __restrict__ g, float* __restrict__ Uhi, float* __restrict__ Ulo,
               float* __restrict__ U32, const __grid_constant__ FParams fp) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;  // c * K_s + k
  const int64_t xi = blockIdx.y;
  if (i >= (int64_t)fp.C * fp.K_s) return;
  const int k = (int)(i % fp.K_s);
  const int c = (int)(i / fp.K_s);
  const int64_t at = xi * ((int64_t)fp.C * fp.K_s) + i;
  float u = 0.f;
  if (k < fp.K) {
    int rN = 1;
    for (int n = 0; n < fp.N; ++n) rN *= fp.r[n];
    const float* gk = g + ((int64_t)k * fp.C + c) * rN;
    int xd[kMaxN];
    int64_t q = xi;
    for (int n = fp.N - 1; n >= 0; --n) { xd[n] = (int)(q % fp.a[n]); q /= fp.a[n]; }
    double acc = 0.0;
    for (int p = 0; p < rN; ++p) {
      double w = 1.0;
      int pq = p;
      for (int n = fp.N - 1; n >= 0; --n) { w *= fp.G[n][xd[n]][pq % fp.r[n]]; pq /= fp.r[n]; }
      if (w != 0.0) acc = fma(w, (double)__ldg(gk + p), acc);
    }
    u = (float)acc;
  }
  const float hi = tf32_rna(u);
  if (Uhi) Uhi[at] = hi;
  if (Ulo) Ulo[at] = tf32_rna(u - hi);
  if (U32) U32[at] = u;
}

bool xform_supported(int N, int alpha, int m, int spec) {
  if (N < 1 || N > 4) return false;
  const bool n4ok = alpha <= 4;
  if (spec != kSpecRuntime) {
    if (!((alpha == 4 && m == 2) || (alpha == 6 && m == 4))) return false;
    return N < 4 || n4ok;
  }
  switch (alpha * 16 + m) {
    case 4 * 16 + 2: case 4 * 16 + 3: case 6 * 16 + 4: case 8 * 16 + 5: case 8 * 16 + 4:
    case 8 * 16 + 3: case 5 * 16 + 3: case 6 * 16 + 3:
      return N < 4 || n4ok;
    default: return false;
  }
}

cudaError_t launch_output_xform(int N, int alpha, int m, int spec, const float* Mx, float* y, const KGeom& g,
                                const XfParams& xp, const CUtensorMap* tmM, cudaStream_t s) {
  if (spec != kSpecRuntime) return launch_output_const(N, alpha, m, spec, Mx, y, g, xp, tmM, s);
  return launch_output_run(N, alpha, m, Mx, y, g, xp, tmM, s);
}

// TMA map of M [P][K][T_s] as (t, k, xi) with the output kernel's box
// {128, 1, alpha^(N-1)}; false if a TMA rule is broken (plain kernel then).
bool encode_output_map(CUtensorMap* tm, const float* Mx, int64_t T_s, int K, int64_t P, int A1) {
  EncodeTiledFn enc = get_encode();
  if (!enc || A1 > 256 || ((uintptr_t)Mx & 15) || (T_s % 128)) return false;
  cuuint64_t dims[3] = {(cuuint64_t)T_s, (cuuint64_t)K, (cuuint64_t)P};
  cuuint64_t strides[2] = {(cuuint64_t)T_s * 4, (cuuint64_t)T_s * K * 4};
  cuuint32_t box[3] = {128, 1, (cuuint32_t)A1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(Mx), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Blocked form of the same sum: a CTA owns (c, 64 kernels k); the weights
// W[xi][p] = prod_n G_n[xi_n][p_n] (fp64) and the 64 kernels' taps g[k][c][:]
// are staged in shared memory once, then U[xi][c][k] = sum_p W[xi][p] g[k,c,p]
// with lanes = consecutive k (coalesced U stores, W broadcast).  Same fp64
// products and summation order (p ascending) as k_filter_xform: identical bits.
constexpr int kFiltKB = 64;
__global__ void __launch_bounds__(256)
k_filter_xform_blk(const float* __restrict__ g, float* __restrict__ Uhi, float* __restrict__ Ulo,
                   float* __restrict__ U32, const __grid_constant__ FParams fp, int rN) {
  extern __shared__ double fsm[];
  double* W = fsm;                              // [P][rN]
  float* gs = reinterpret_cast<float*>(W + fp.P * rN);  // [kFiltKB][rN]
  const int c = blockIdx.x;
  const int k0 = blockIdx.y * kFiltKB;
  const int P = (int)fp.P;
  for (int i = threadIdx.x; i < P * rN; i += blockDim.x) {
    const int xi = i / rN, p = i - xi * rN;
    int q = xi, pq = p;
    double w = 1.0;
    for (int n = fp.N - 1; n >= 0; --n) {
      w *= fp.G[n][q % fp.a[n]][pq % fp.r[n]];
      q /= fp.a[n];
      pq /= fp.r[n];
    }
    W[i] = w;
  }
  for (int i = threadIdx.x; i < kFiltKB * rN; i += blockDim.x) {
    const int kl = i / rN, p = i - kl * rN;
    const int k = k0 + kl;
    gs[i] = k < fp.K ? __ldg(g + ((int64_t)k * fp.C + c) * rN + p) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P * kFiltKB; i += blockDim.x) {
    const int xi = i / kFiltKB, kl = i - xi * kFiltKB;
    const int k = k0 + kl;
    if (k >= fp.K_s) continue;
    float u = 0.f;
    if (k < fp.K) {
      const double* wr = W + xi * rN;
      const float* gr = gs + kl * rN;
      double acc = 0.0;
      for (int p = 0; p < rN; ++p)
        if (wr[p] != 0.0) acc = fma(wr[p], (double)gr[p], acc);
      u = (float)acc;
    }
    const int64_t at = ((int64_t)xi * fp.C + c) * fp.K_s + k;
    const float hi = tf32_rna(u);
    if (Uhi) Uhi[at] = hi;
    if (Ulo) Ulo[at] = tf32_rna(u - hi);
    if (U32) U32[at] = u;
  }
}

// a1 for the filter-side fold (kernels.h, UFoldTab): one thread per
// (xo, (q, c), (o, k)), (o, k) fastest:
//   U'[xo][q*C + c][o*K + k] = A^T_F[o][q] * sum_p prod_n G_n[xi_n][p_n] g[k, c, p],  xi = xo*Q + q
// in fp64 (the sum as k_filter_xform), rounded once to fp32, then split.
__global__ void __launch_bounds__(256)
k_filter_ufold(const float* __restrict__ g, float* __restrict__ Uhi, float* __restrict__ Ulo,
               float* __restrict__ U32, const __grid_constant__ FParams fp, const __grid_constant__ UFoldTab uf) {
  const int64_t gC = (int64_t)uf.Q * fp.C;
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;   // (q*C + c) * K_s' + (o*K + k)
  const int64_t xo = blockIdx.y;
  if (i >= gC * fp.K_s) return;
  const int ok = (int)(i % fp.K_s);
  const int qc = (int)(i / fp.K_s);
  const int q = qc / fp.C, c = qc - q * fp.C;
  const int o = ok / fp.K, k = ok - o * fp.K;
  float u = 0.f;
  const double cf = o < uf.MO ? uf.coef[q][o] : 0.0;
  if (cf != 0.0) {
    int rN = 1;
    for (int n = 0; n < fp.N; ++n) rN *= fp.r[n];
    const float* gk = g + ((int64_t)k * fp.C + c) * rN;
    int xd[kMaxN];
    int64_t qq = xo * uf.Q + q;
    for (int n = fp.N - 1; n >= 0; --n) { xd[n] = (int)(qq % fp.a[n]); qq /= fp.a[n]; }
    double acc = 0.0;
    for (int p = 0; p < rN; ++p) {
      double w = 1.0;
      int pq = p;
      for (int n = fp.N - 1; n >= 0; --n) {
        // direct-axis fold: the last axis keeps the raw tap j - o (q = j)
        if (uf.direct && n == fp.N - 1) w *= (pq % fp.r[n] == q - o) ? 1.0 : 0.0;
        else w *= fp.G[n][xd[n]][pq % fp.r[n]];
        pq /= fp.r[n];
      }
      if (w != 0.0) acc = fma(w, (double)__ldg(gk + p), acc);
    }
    u = (float)(cf * acc);
  }
  const int64_t at = xo * gC * fp.K_s + i;
  const float hi = tf32_rna(u);
  if (Uhi) Uhi[at] = hi;
  if (Ulo) Ulo[at] = tf32_rna(u - hi);
  if (U32) U32[at] = u;
}

cudaError_t launch_filter_ufold(const float* g, float* Uhi, float* Ulo, float* U32, const FParams& fp,
                                const UFoldTab& uf, cudaStream_t s) {
  if (uf.Q < 1 || uf.MO < 1 || fp.P % uf.Q) return cudaErrorInvalidValue;
  const int64_t n = (int64_t)uf.Q * fp.C * fp.K_s;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)(fp.P / uf.Q));
  k_filter_ufold<<<grid, 256, 0, s>>>(g, Uhi, Ulo, U32, fp, uf);
  return cudaGetLastError();
}

cudaError_t launch_filter_xform(const float* g, float* Uhi, float* Ulo, float* U32, const FParams& fp,
                                cudaStream_t s) {
  int rN = 1;
  for (int n = 0; n < fp.N; ++n) rN *= fp.r[n];
  const size_t smem = (size_t)fp.P * rN * 8 + (size_t)kFiltKB * rN * 4;
  const char* ev = getenv("WINO_FILTER_BLK");  // 0: the per-output kernel (tests compare both)
  if ((!ev || atoi(ev) != 0) && smem <= 100 * 1024 && fp.C <= 65535) {
    if (smem > 46 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_filter_xform_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    dim3 grid((unsigned)fp.C, (unsigned)((fp.K_s + kFiltKB - 1) / kFiltKB));
    k_filter_xform_blk<<<grid, 256, smem, s>>>(g, Uhi, Ulo, U32, fp, rN);
    return cudaGetLastError();
  }
  const int64_t n = (int64_t)fp.C * fp.K_s;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)fp.P);
  k_filter_xform<<<grid, 256, 0, s>>>(g, Uhi, Ulo, U32, fp);
  return cudaGetLastError();
}

}  // namespace wino
