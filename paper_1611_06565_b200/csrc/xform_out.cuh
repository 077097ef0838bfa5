// xform_out.cuh -- stage a4, the output transform + scatter of the N-D
// Winograd layer (kernel template; instantiated by xform_out_const.cu and
// xform_out_run.cu):
//
//   y tile(b, k, t) = M[.][k][t] x_1 A^T ... x_N A^T, cropped to `out`
// (Eq. (4); stitching of overlapping tiles PAPER.md:221).
#pragma once
#include "kernels.h"
#include "xform_common.cuh"

namespace wino {
namespace out_detail {

// ------------------------------------------------------------------ a4
// One thread per (tile t, output channel k): read M[xi][k][t] for all xi,
// apply A^T along every axis (alpha -> m), crop to `out` and scatter into y.
template <int N, int A, int M, class Tab>
__global__ void __launch_bounds__(128)
k_output_xform(const float* __restrict__ Mx, float* __restrict__ y, const __grid_constant__ KGeom g,
               const __grid_constant__ XfParams xp) {
  constexpr int A1 = ipow(A, N - 1);
  constexpr int M1 = ipow(M, N - 1);
  constexpr int MN = ipow(M, N);
  pdl_wait();      // M comes from the GEMM
  pdl_trigger();
  const int64_t t = g.t_beg + (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int k = blockIdx.y;
  if (t >= g.T) return;
  const int64_t pstride = (int64_t)g.K * g.T_s;
  // running pointer over the alpha^N points (one 64-bit add per load instead
  // of a 64-bit multiply-add per point offset)
  const float* src = Mx + (int64_t)k * g.T_s + (t - g.t0);
  float o[MN];
#pragma unroll
  for (int j = 0; j < MN; ++j) o[j] = 0.f;
#pragma unroll
  for (int x1 = 0; x1 < A; ++x1) {
    float v[A1];
#pragma unroll
    for (int j = 0; j < A1; ++j) {
      v[j] = __ldg(src);
      src += pstride;
    }
    all_axes<A, N - 1, M, M, ATget<Tab>>(v, xp);
#pragma unroll
    for (int o1 = 0; o1 < M; ++o1) {
      if (!ATget<Tab>::nz(xp, o1, x1)) continue;
      const float av = ATget<Tab>::v(xp, o1, x1);
#pragma unroll
      for (int rr = 0; rr < M1; ++rr)
        o[o1 * M1 + rr] = fmaf(av, v[digits_to_base(rr, N - 1, M, A)], o[o1 * M1 + rr]);
    }
  }
  // Eq. (2) epilogue in the spatial domain: d' = f(b + conv)
  if (g.bias || g.act) {
    const float bk = g.bias ? __ldg(g.bias + k) : 0.f;
#pragma unroll
    for (int j = 0; j < MN; ++j) {
      const float v = o[j] + bk;
      o[j] = g.act == 1 ? fmaxf(v, 0.f) : v;
    }
  }
  // scatter: tile t -> (b, t_1..t_N) (32-bit: T < 2^31 is enforced at plan
  // creation); outputs past `out` are discarded
  int rem = (int)t;
  int gi[N];
#pragma unroll
  for (int n = N - 1; n >= 0; --n) {
    gi[n] = rem % g.tiles[n];
    rem /= g.tiles[n];
  }
  float* yb = y + ((int64_t)rem * g.K + k) * g.out_vol;
  const int lastpos = gi[N - 1] * M;
  const bool full_last = lastpos + M <= g.out[N - 1];
#pragma unroll
  for (int rr = 0; rr < M1; ++rr) {  // each output row along the last axis
    bool ok = true;
    int64_t off = lastpos;
#pragma unroll
    for (int ax = 0; ax < N - 1; ++ax) {
      const int d = (rr / ipow(M, N - 2 - ax)) % M;
      const int pos = gi[ax] * M + d;
      ok = ok && (pos < (int)g.out[ax]);
      off += (int64_t)pos * g.out_stride[ax];
    }
    if (!ok) continue;
    float* dst = yb + off;
    const int ob = rr * M;  // o index of (row, last = 0); last axis fastest
    if constexpr (M == 4) {
      if (full_last && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        *reinterpret_cast<float4*>(dst) = make_float4(o[ob], o[ob + 1], o[ob + 2], o[ob + 3]);
        continue;
      }
    } else if constexpr (M == 2) {
      if (full_last && ((reinterpret_cast<uintptr_t>(dst) & 7) == 0)) {
        *reinterpret_cast<float2*>(dst) = make_float2(o[ob], o[ob + 1]);
        continue;
      }
    }
#pragma unroll
    for (int l = 0; l < M; ++l)
      if (lastpos + l < g.out[N - 1]) dst[l] = o[ob + l];
  }
}

template <int N, int A, int M, class Tab>
cudaError_t launch_out(const float* Mx, float* y, const KGeom& g, const XfParams& xp, cudaStream_t s) {
  dim3 grid((unsigned)((g.T - g.t_beg + 127) / 128), (unsigned)g.K);
  return launch_pdl(k_output_xform<N, A, M, Tab>, grid, dim3(128), 0, s, Mx, y, g, xp);
}

template <int A, int M, class Tab>
cudaError_t launch_out_byN(int N, const float* Mx, float* y, const KGeom& g, const XfParams& xp, cudaStream_t s) {
  switch (N) {
    case 1: return launch_out<1, A, M, Tab>(Mx, y, g, xp, s);
    case 2: return launch_out<2, A, M, Tab>(Mx, y, g, xp, s);
    case 3: return launch_out<3, A, M, Tab>(Mx, y, g, xp, s);
    case 4:
      if constexpr (ipow(A, 3) <= 64) return launch_out<4, A, M, Tab>(Mx, y, g, xp, s);
      else return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
}

}  // namespace out_detail

cudaError_t launch_output_const(int N, int alpha, int m, int spec, const float* Mx, float* y, const KGeom& g,
                                const XfParams& xp, cudaStream_t s);
cudaError_t launch_output_run(int N, int alpha, int m, const float* Mx, float* y, const KGeom& g,
                              const XfParams& xp, cudaStream_t s);

}  // namespace wino
