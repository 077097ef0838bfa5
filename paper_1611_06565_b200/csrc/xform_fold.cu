// xform_fold.cu -- stage a4 after the folded GEMM (gemm_fold.cu): the
// output transform of the N - F outer axes.
//
// W[xo][o][k][t] already carries x_n A^T for the F innermost axes (o < m^F);
// per (tile t, output channel k) the alpha^(N-F) m^F values of W are
// transformed along axes 0 .. N-F-1 (alpha -> m each; Eq. (4)),
// giving the m^N output tile, which is cropped to `out` and scattered into y
// exactly as by k_output_xform (store_tile: bias / ReLU of Eq. (2) included).
#include "xform_out.cuh"

namespace wino {
namespace fold_detail {

using out_detail::store_tile;

// Transform axis AX (extent A -> M) of a register tensor laid out row-major as
// [M]^AX x [A] x [A]^(NA-1-AX) x [M]^NI  ->  [M]^(AX+1) x [A]^(NA-1-AX) x [M]^NI.
template <int A, int M, int NA, int NI, int AX, class Get>
__device__ __forceinline__ void fold_pass(const float* in, float* out, const XfParams& p) {
  constexpr int outer = ipow(M, AX);
  constexpr int inner = ipow(A, NA - 1 - AX) * ipow(M, NI);
#pragma unroll
  for (int o = 0; o < outer; ++o) {
#pragma unroll
    for (int s = 0; s < inner; ++s) {
#pragma unroll
      for (int x = 0; x < M; ++x) {
        float acc = 0.f;
        bool first = true;
#pragma unroll
        for (int i = 0; i < A; ++i) {
          if (Get::nz(p, x, i)) {
            const float v = in[(o * A + i) * inner + s];
            acc = first ? Get::v(p, x, i) * v : fmaf(Get::v(p, x, i), v, acc);
            first = false;
          }
        }
        out[(o * M + x) * inner + s] = acc;
      }
    }
  }
}

template <int A, int M, int NA, int NI, class Get, int AX = 0>
__device__ __forceinline__ void fold_axes(const float* v, float* res, const XfParams& p) {
  if constexpr (AX + 1 == NA) {
    fold_pass<A, M, NA, NI, AX, Get>(v, res, p);
  } else {
    float t[ipow(M, AX + 1) * ipow(A, NA - 1 - AX) * ipow(M, NI)];
    fold_pass<A, M, NA, NI, AX, Get>(v, t, p);
    fold_axes<A, M, NA, NI, Get, AX + 1>(t, res, p);
  }
}

// One thread per (t, k), 128 tiles per block, blockIdx.y = k.
template <int N, int A, int M, int F, class Tab>
__global__ void __launch_bounds__(128)
k_output_fold(const float* __restrict__ W, float* __restrict__ y, const __grid_constant__ KGeom g,
              const __grid_constant__ XfParams xp) {
  constexpr int NA = N - F;
  constexpr int PW = ipow(A, NA) * ipow(M, F);   // W planes
  constexpr int MN = ipow(M, N);
  pdl_wait();      // W comes from the folded GEMM
  pdl_trigger();
  // the GEMM has consumed max|V| (3xFP16 scaling): clear it for the next forward
  if (g.vmax_reset && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *g.vmax_reset = 0u;
  const int64_t t = g.t_beg + (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int k = blockIdx.y;
  if (t >= g.T) return;
  const int64_t pstride = (int64_t)g.K * g.T_s;
  const float* src = W + (int64_t)k * g.T_s + (t - g.t0);
  float v[PW];
#pragma unroll
  for (int j = 0; j < PW; ++j) {
    v[j] = __ldg(src);
    src += pstride;
  }
  float o[MN];
  fold_axes<A, M, NA, F, ATget<Tab>>(v, o, xp);
  store_tile<N, M>(o, y, g, t, k);
}

template <int N, int A, int M, int F, class Tab>
cudaError_t launch_fold(const float* W, float* y, const KGeom& g, const XfParams& xp, cudaStream_t s) {
  dim3 grid((unsigned)((g.T - g.t_beg + 127) / 128), (unsigned)g.K);
  return launch_pdl(k_output_fold<N, A, M, F, Tab>, grid, dim3(128), 0, s, W, y, g, xp);
}

}  // namespace fold_detail

// Instantiated: F(2^N, 3^N) with the default points {0, 1, -1, inf}, N = 3
// (F = 1, 2) and N = 4 (F = 2, 3); F(4^2, 3^2) with the default alpha = 6
// points, F = 1.
bool output_fold_supported(int N, int alpha, int m, int F, int spec) {
  if (spec != kSpecDefault) return false;
  if (alpha == 4 && m == 2) return (N == 3 && (F == 1 || F == 2)) || (N == 4 && (F == 2 || F == 3));
  if (alpha == 6 && m == 4) return N == 2 && F == 1;
  return false;
}

cudaError_t launch_output_fold(int N, int alpha, int m, int F, int spec, const float* W, float* y, const KGeom& g,
                               const XfParams& xp, cudaStream_t s) {
  using namespace fold_detail;
  if (!output_fold_supported(N, alpha, m, F, spec)) return cudaErrorNotSupported;
  if (alpha == 4) {
    using T = ConstTab<2, 3, kPsDefault>;
    if (N == 3 && F == 1) return launch_fold<3, 4, 2, 1, T>(W, y, g, xp, s);
    if (N == 3 && F == 2) return launch_fold<3, 4, 2, 2, T>(W, y, g, xp, s);
    if (N == 4 && F == 2) return launch_fold<4, 4, 2, 2, T>(W, y, g, xp, s);
    if (N == 4 && F == 3) return launch_fold<4, 4, 2, 3, T>(W, y, g, xp, s);
  } else {
    return launch_fold<2, 6, 4, 1, ConstTab<4, 3, kPsDefault>>(W, y, g, xp, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace wino
