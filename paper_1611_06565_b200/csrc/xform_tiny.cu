// xform_tiny.cu -- the whole forward of a tiny layer in one kernel (SURVEY
// 8(f) NEXT-3: batch-1 / few-channel layers such as BASELINE.json c1, where
// three launches and their fill / drain dominate): per block of TB tiles
//   phase A: V[xi][c][t] = (d(b, c, t) x_1 B^T .. x_N B^T)_xi   -> shared memory
//   phase B: M[xi][k][t] = sum_c V[xi][c][t] U[xi][c][k]         (fp32 FMA)
//            y tile       = M x_1 A^T .. x_N A^T, cropped, + bias, ReLU
// (Eq. (4)-(5)).  U = U_hi + U_lo of the plan's
// 3xTF32 filter buffer (|U - (U_hi + U_lo)| <= 2^-22 |U|, DESIGN.md reading
// #7).  One thread per (tile, channel) item with the alpha^N window in
// registers (alpha^N <= 64); the plan uses it only for tiny layers.
#include "kernels.h"
#include "xform_common.cuh"

namespace wino {
namespace {

template <int N, int A, int M, class Tab>
__global__ void __launch_bounds__(128)
k_tiny(const float* __restrict__ x, const float* __restrict__ Uhi, const float* __restrict__ Ulo,
       float* __restrict__ y, const __grid_constant__ KGeom g, const __grid_constant__ XfParams xp, int K_s, int TB,
       int64_t T) {
  constexpr int P = ipow(A, N);
  extern __shared__ float Vs[];  // [P][C][TB], then Us [P][C][K]
  const int64_t t0 = (int64_t)blockIdx.x * TB;
  const int C = g.C, K = g.K;
  float* Us = Vs + P * C * TB;
  // U = U_hi + U_lo staged once per block (coalesced; its loads overlap phase A's)
  for (int i = threadIdx.x; i < P * C * K; i += blockDim.x) {
    const int k = i % K, pc = i / K;
    Us[i] = __ldg(Uhi + (int64_t)pc * K_s + k) + __ldg(Ulo + (int64_t)pc * K_s + k);
  }
  // ---- phase A: one item per (tile, channel): window in registers, B^T per axis
  for (int it = threadIdx.x; it < TB * C; it += blockDim.x) {
    const int tl = it % TB, c = it / TB;
    const int64_t t = t0 + tl;
    float w[P];
    if (t < T) {
      int rem = (int)t, tn[N];
#pragma unroll
      for (int n = N - 1; n >= 0; --n) {
        tn[n] = rem % g.tiles[n];
        rem /= g.tiles[n];
      }
      const float* xb = x + ((int64_t)rem * C + c) * g.in_vol;
#pragma unroll
      for (int xi = 0; xi < P; ++xi) {
        bool ok = true;
        int64_t off = 0;
#pragma unroll
        for (int n = 0; n < N; ++n) {
          const int d = (xi / ipow(A, N - 1 - n)) % A;
          const int64_t pos = (int64_t)tn[n] * M - g.pad[n] + d;
          ok = ok && pos >= 0 && pos < g.in[n];
          off += pos * g.in_stride[n];
        }
        w[xi] = ok ? __ldg(xb + off) : 0.f;
      }
      all_axes<A, N, A, A, BTget<Tab>>(w, xp);
    } else {
#pragma unroll
      for (int xi = 0; xi < P; ++xi) w[xi] = 0.f;
    }
#pragma unroll
    for (int xi = 0; xi < P; ++xi) Vs[(xi * C + c) * TB + tl] = w[xi];
  }
  __syncthreads();
  // ---- phase B: one item per (tile, output channel)
  for (int it = threadIdx.x; it < TB * K; it += blockDim.x) {
    const int tl = it % TB, k = it / TB;
    const int64_t t = t0 + tl;
    if (t >= T) continue;
    float w[P];
#pragma unroll
    for (int xi = 0; xi < P; ++xi) {
      float acc = 0.f;
      const float* vrow = Vs + xi * C * TB + tl;
      const float* urow = Us + xi * C * K + k;
      for (int c = 0; c < C; ++c) acc = fmaf(vrow[c * TB], urow[c * K], acc);
      w[xi] = acc;
    }
    all_axes<A, N, M, M, ATget<Tab>>(w, xp);  // entry digits_to_base(o, N, M, A) holds output o
    int rem = (int)t, tn[N];
#pragma unroll
    for (int n = N - 1; n >= 0; --n) {
      tn[n] = rem % g.tiles[n];
      rem /= g.tiles[n];
    }
    float* yb = y + ((int64_t)rem * K + k) * g.out_vol;
    const float bk = g.bias ? __ldg(g.bias + k) : 0.f;
#pragma unroll
    for (int o = 0; o < ipow(M, N); ++o) {
      bool ok = true;
      int64_t off = 0;
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const int d = (o / ipow(M, N - 1 - n)) % M;
        const int64_t pos = (int64_t)tn[n] * M + d;
        ok = ok && pos < g.out[n];
        off += pos * g.out_stride[n];
      }
      if (!ok) continue;
      float v = w[digits_to_base(o, N, M, A)];
      if (g.bias || g.act) {
        v += bk;
        if (g.act == 1) v = fmaxf(v, 0.f);
      }
      yb[off] = v;
    }
  }
}

template <int N, int A, int M, class Tab>
cudaError_t launch_t(const float* x, const float* Uhi, const float* Ulo, float* y, const KGeom& g, const XfParams& xp,
                     int K_s, int TB, int smem, int64_t T, cudaStream_t s) {
  if constexpr (ipow(A, N) > 64) {
    return cudaErrorNotSupported;
  } else {
    const unsigned grid = (unsigned)((T + TB - 1) / TB);
    k_tiny<N, A, M, Tab><<<grid, 128, smem, s>>>(x, Uhi, Ulo, y, g, xp, K_s, TB, T);
    return cudaGetLastError();
  }
}

template <int A, int M, class Tab>
cudaError_t launch_byN(int N, const float* x, const float* Uhi, const float* Ulo, float* y, const KGeom& g,
                       const XfParams& xp, int K_s, int TB, int smem, int64_t T, cudaStream_t s) {
  switch (N) {
    case 1: return launch_t<1, A, M, Tab>(x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    case 2: return launch_t<2, A, M, Tab>(x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    case 3: return launch_t<3, A, M, Tab>(x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

// Tiles per block and shared memory (V block + staged U) of the tiny kernel;
// false if it does not apply.
bool tiny_shape(int N, int a, int C, int K, int64_t P, int* TB, int* smem) {
  if (P > 64 || N > 3 || a > kMaxA || P * C * K > 8192) return false;
  int tb = 32;
  while (tb > 1 && (int64_t)P * C * tb * 4 > 12 * 1024) tb /= 2;
  if ((int64_t)P * C * tb * 4 > 12 * 1024) return false;
  *TB = tb;
  *smem = (int)((P * C * tb + P * C * K) * 4);
  return true;
}

bool tiny_supported(int N, int a, int m) {
  if (N < 1 || N > 3) return false;
  switch (a * 16 + m) {
    case 4 * 16 + 2: case 4 * 16 + 3: case 5 * 16 + 3: case 6 * 16 + 3: case 6 * 16 + 4:
    case 8 * 16 + 3: case 8 * 16 + 4: case 8 * 16 + 5:
      return ipow(a, N) <= 64;
    default: return false;
  }
}

cudaError_t launch_tiny(const float* x, const float* Uhi, const float* Ulo, float* y, const KGeom& g,
                        const XfParams& xp, int N, int a, int m, int spec, int P, int K_s, int64_t T, cudaStream_t s) {
  int TB, smem;
  if (!tiny_shape(N, a, g.C, g.K, P, &TB, &smem)) return cudaErrorNotSupported;
  if (spec == kSpecDefault) {
    if (a == 4 && m == 2) return launch_byN<4, 2, ConstTab<2, 3, kPsDefault>>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    if (a == 6 && m == 4) return launch_byN<6, 4, ConstTab<4, 3, kPsDefault>>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
  }
  switch (a * 16 + m) {
    case 4 * 16 + 2: return launch_byN<4, 2, RunTab>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    case 4 * 16 + 3: return launch_byN<4, 3, RunTab>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    case 5 * 16 + 3: return launch_byN<5, 3, RunTab>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    case 6 * 16 + 3: return launch_byN<6, 3, RunTab>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    case 6 * 16 + 4: return launch_byN<6, 4, RunTab>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    case 8 * 16 + 3: return launch_byN<8, 3, RunTab>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    case 8 * 16 + 4: return launch_byN<8, 4, RunTab>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    case 8 * 16 + 5: return launch_byN<8, 5, RunTab>(N, x, Uhi, Ulo, y, g, xp, K_s, TB, smem, T, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace wino
