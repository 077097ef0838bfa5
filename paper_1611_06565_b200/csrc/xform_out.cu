// xform_out.cu -- stage a4 (output transform + scatter) and stage a1
// (filter transform) of the N-D Winograd layer on sm_100a.
//
//   y tile(b, k, t) = M[.][k][t] x_1 A^T ... x_N A^T, cropped to `out`
//   U_xi[c][k]      = (g[k, c] x_1 G ... x_N G)_xi
// (Eq. (4); stitching PAPER.md:221; cached transformed
// kernels PAPER.md:178).
#include "kernels.h"
#include "xform_common.cuh"

namespace wino {

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
  const int64_t t = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int k = blockIdx.y;
  if (t >= g.T) return;
  const int64_t pstride = (int64_t)g.K * g.T_s;
  const float* src = Mx + (int64_t)k * g.T_s + t;
  float o[MN];
#pragma unroll
  for (int j = 0; j < MN; ++j) o[j] = 0.f;
#pragma unroll
  for (int x1 = 0; x1 < A; ++x1) {
    float v[A1];
#pragma unroll
    for (int j = 0; j < A1; ++j) v[j] = __ldg(src + (x1 * A1 + j) * pstride);
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
  // scatter: tile t -> (b, t_1..t_N); outputs past `out` are discarded
  int64_t rem = t;
  int gi[N];
#pragma unroll
  for (int n = N - 1; n >= 0; --n) {
    gi[n] = (int)(rem % g.tiles[n]);
    rem /= g.tiles[n];
  }
  float* yb = y + (rem * g.K + k) * g.out_vol;
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
      ok = ok && (pos < g.out[ax]);
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

// ------------------------------------------------------------------ a1
// One thread per (xi, c, k) (k fastest -> coalesced U writes):
//   U_xi[c][k] = sum_p prod_n G[xi_n][p_n] g[k, c, p]
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
    for (int n = 0; n < fp.N; ++n) rN *= fp.r;
    const float* gk = g + ((int64_t)k * fp.C + c) * rN;
    int xd[kMaxN];
    int64_t q = xi;
    for (int n = fp.N - 1; n >= 0; --n) { xd[n] = (int)(q % fp.a); q /= fp.a; }
    double acc = 0.0;
    for (int p = 0; p < rN; ++p) {
      double w = 1.0;
      int pq = p;
      for (int n = fp.N - 1; n >= 0; --n) { w *= fp.G[xd[n]][pq % fp.r]; pq /= fp.r; }
      if (w != 0.0) acc = fma(w, (double)__ldg(gk + p), acc);
    }
    u = (float)acc;
  }
  const float hi = tf32_rna(u);
  if (Uhi) Uhi[at] = hi;
  if (Ulo) Ulo[at] = tf32_rna(u - hi);
  if (U32) U32[at] = u;
}

// ------------------------------------------------------------------ dispatch
namespace {

template <int N, int A, int M, class Tab>
cudaError_t launch_out(const float* Mx, float* y, const KGeom& g, const XfParams& xp, cudaStream_t s) {
  dim3 grid((unsigned)((g.T + 127) / 128), (unsigned)g.K);
  k_output_xform<N, A, M, Tab><<<grid, 128, 0, s>>>(Mx, y, g, xp);
  return cudaGetLastError();
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

}  // namespace

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
                                const XfParams& xp, cudaStream_t s) {
  if (spec == kSpecDefault) {
    if (alpha == 4 && m == 2) return launch_out_byN<4, 2, ConstTab<2, 3, kPsDefault>>(N, Mx, y, g, xp, s);
    if (alpha == 6 && m == 4) return launch_out_byN<6, 4, ConstTab<4, 3, kPsDefault>>(N, Mx, y, g, xp, s);
  } else if (spec == kSpecSeq) {
    if (alpha == 4 && m == 2) return launch_out_byN<4, 2, ConstTab<2, 3, kPsSeq>>(N, Mx, y, g, xp, s);
    if (alpha == 6 && m == 4) return launch_out_byN<6, 4, ConstTab<4, 3, kPsSeq>>(N, Mx, y, g, xp, s);
  } else {
    switch (alpha * 16 + m) {
      case 4 * 16 + 2: return launch_out_byN<4, 2, RunTab>(N, Mx, y, g, xp, s);
      case 4 * 16 + 3: return launch_out_byN<4, 3, RunTab>(N, Mx, y, g, xp, s);
      case 5 * 16 + 3: return launch_out_byN<5, 3, RunTab>(N, Mx, y, g, xp, s);
      case 6 * 16 + 3: return launch_out_byN<6, 3, RunTab>(N, Mx, y, g, xp, s);
      case 6 * 16 + 4: return launch_out_byN<6, 4, RunTab>(N, Mx, y, g, xp, s);
      case 8 * 16 + 3: return launch_out_byN<8, 3, RunTab>(N, Mx, y, g, xp, s);
      case 8 * 16 + 4: return launch_out_byN<8, 4, RunTab>(N, Mx, y, g, xp, s);
      case 8 * 16 + 5: return launch_out_byN<8, 5, RunTab>(N, Mx, y, g, xp, s);
      default: break;
    }
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_filter_xform(const float* g, float* Uhi, float* Ulo, float* U32, const FParams& fp,
                                cudaStream_t s) {
  const int64_t n = (int64_t)fp.C * fp.K_s;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)fp.P);
  k_filter_xform<<<grid, 256, 0, s>>>(g, Uhi, Ulo, U32, fp);
  return cudaGetLastError();
}

}  // namespace wino
