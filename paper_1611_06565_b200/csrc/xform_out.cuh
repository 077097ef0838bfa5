// xform_out.cuh -- stage a4, the output transform + scatter of the N-D
// Winograd layer (kernel template; instantiated by xform_out_const.cu,
// xform_out_run.cu and xform_mixed.cu): a plain kernel with per-thread loads
// of M, and a TMA-ring kernel for alpha^(N-1) >= 32 (k_output_xform_tma);
// axis 0's transform is a template parameter (per-axis plans):
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

// Axis-0 transform of a plan (alpha_0 = A, tile step M, table Tab); equal to
// the other axes' except for per-axis plans with a distinct axis 0 (NEXT-2).
template <int A0_, int M0_, class Tab0_>
struct OAx0 {
  static constexpr int A = A0_;
  static constexpr int M = M0_;
  using Tab = Tab0_;
};

// Accumulate axis-0 group x1 (the alpha^(N-1) values v of M[xi][k][t] with
// xi_0 = x1) into the output tile o (M_0 x M^(N-1)): A^T along axes 1..N-1
// in registers, then o += A_0^T[:, x1] (x) v along axis 0.
template <int N, int A, int M, class Tab, class Ax>
__device__ __forceinline__ void accum_group(float (&o)[Ax::M * ipow(M, N - 1)], float (&v)[ipow(A, N - 1)], int x1,
                                            const XfParams& xp) {
  constexpr int M1 = ipow(M, N - 1);
  using Get0 = ATget<typename Ax::Tab>;
  all_axes<A, N - 1, M, M, ATget<Tab>>(v, xp);
#pragma unroll
  for (int o1 = 0; o1 < Ax::M; ++o1) {
    if (!Get0::nz(xp, o1, x1)) continue;
    const float av = Get0::v(xp, o1, x1);
#pragma unroll
    for (int rr = 0; rr < M1; ++rr)
      o[o1 * M1 + rr] = fmaf(av, v[digits_to_base(rr, N - 1, M, A)], o[o1 * M1 + rr]);
  }
}

template <int N, int M, int M0 = M>
__device__ __forceinline__ void store_tile(float (&o)[M0 * ipow(M, N - 1)], float* __restrict__ y, const KGeom& g,
                                           int64_t t, int k) {
  constexpr int M1 = M0 * ipow(M, N - 2);   // output rows along the last axis (N >= 2)
  constexpr int MN = M0 * ipow(M, N - 1);
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
  constexpr int ML = N == 1 ? M0 : M;  // tile length along the last axis
  const int lastpos = gi[N - 1] * ML;
  const bool full_last = lastpos + ML <= g.out[N - 1];
#pragma unroll
  for (int rr = 0; rr < (N == 1 ? 1 : M1); ++rr) {  // each output row along the last axis
    bool ok = true;
    int64_t off = lastpos;
#pragma unroll
    for (int ax = 0; ax < N - 1; ++ax) {
      // row digits: axis 0 has radix M0, the others M
      const int d = ax == 0 ? rr / ipow(M, N - 2) : (rr / ipow(M, N - 2 - ax)) % M;
      const int pos = gi[ax] * (ax == 0 ? M0 : M) + d;
      ok = ok && (pos < (int)g.out[ax]);
      off += (int64_t)pos * g.out_stride[ax];
    }
    if (!ok) continue;
    float* dst = yb + off;
    const int ob = rr * ML;  // o index of (row, last = 0); last axis fastest
    if constexpr (ML == 4) {
      if (full_last && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        *reinterpret_cast<float4*>(dst) = make_float4(o[ob], o[ob + 1], o[ob + 2], o[ob + 3]);
        continue;
      }
    } else if constexpr (ML == 2) {
      if (full_last && ((reinterpret_cast<uintptr_t>(dst) & 7) == 0)) {
        *reinterpret_cast<float2*>(dst) = make_float2(o[ob], o[ob + 1]);
        continue;
      }
    }
#pragma unroll
    for (int l = 0; l < ML; ++l)
      if (lastpos + l < g.out[N - 1]) dst[l] = o[ob + l];
  }
}

template <int N, int A, int M, class Tab, class Ax = OAx0<A, M, Tab>>
__global__ void __launch_bounds__(128)
k_output_xform(const float* __restrict__ Mx, float* __restrict__ y, const __grid_constant__ KGeom g,
               const __grid_constant__ XfParams xp) {
  constexpr int A1 = ipow(A, N - 1);
  constexpr int MN = Ax::M * ipow(M, N - 1);
  pdl_wait();      // M comes from the GEMM
  pdl_trigger();
  // the GEMM has consumed max|V| (3xFP16 scaling): clear it for the next forward
  if (g.vmax_reset && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *g.vmax_reset = 0u;
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
  for (int x1 = 0; x1 < Ax::A; ++x1) {
    float v[A1];
#pragma unroll
    for (int j = 0; j < A1; ++j) {
      v[j] = __ldg(src);
      src += pstride;
    }
    accum_group<N, A, M, Tab, Ax>(o, v, x1, xp);
  }
  store_tile<N, M, Ax::M>(o, y, g, t, k);
}

// TMA-fed variant (persistent): a CTA of 128 threads walks units (t-block of
// 128 tiles, k), consecutive units = adjacent t-blocks of one k.  Each unit
// is alpha groups (one per xi_0) of alpha^(N-1) x 128 floats of M, loaded by
// one TMA box {128 t, 1 k, alpha^(N-1) xi} into a ring of `ns` stages that
// runs ns - 1 groups ahead (across unit boundaries); threads read their
// column (conflict-free) and accumulate as above.  Keeps tens of KB of M in
// flight per SM without the per-thread load latency of the plain kernel.
template <int N, int A, int M, class Tab, class Ax = OAx0<A, M, Tab>>
__global__ void __launch_bounds__(128)
k_output_xform_tma(float* __restrict__ y, const __grid_constant__ KGeom g, const __grid_constant__ XfParams xp,
                   const __grid_constant__ CUtensorMap tmM, int ns) {
  constexpr int A1 = ipow(A, N - 1);
  constexpr int MN = Ax::M * ipow(M, N - 1);
  constexpr int A0 = Ax::A;
  constexpr uint32_t kStageBytes = A1 * 128 * 4;
  extern __shared__ __align__(128) float S[];
  __shared__ __align__(8) uint64_t full[kMaxOutStages];
  const int nblk = (int)((g.T - g.t_beg + 127) / 128);
  const int64_t nunits = (int64_t)nblk * g.K;
  const uint32_t fb0 = (uint32_t)__cvta_generic_to_shared(&full[0]);
  const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(S);
  // group q of this CTA: its (q / A0)-th unit, xi_0 = q % A0
  auto issue = [&](int64_t q, int st) {
    const int64_t u = blockIdx.x + (q / A0) * gridDim.x;
    if (u >= nunits) return;
    const int k = (int)(u / nblk), tb = (int)(u - (int64_t)k * nblk);
    const int tc = (int)(g.t_beg - g.t0) + tb * 128;
    const uint32_t bar = fb0 + 8u * st;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kStageBytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(sb0 + st * kStageBytes), "l"(&tmM), "r"(tc), "r"(k), "r"((int)(q % A0) * A1), "r"(bar)
        : "memory");
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < ns; ++st) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fb0 + 8u * st) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();      // M comes from the GEMM
  pdl_trigger();
  if (g.vmax_reset && blockIdx.x == 0 && threadIdx.x == 0) *g.vmax_reset = 0u;   // (see k_output_xform)
  if (threadIdx.x == 0)
    for (int st = 0; st < ns; ++st) issue(st, st);
  int64_t q = 0;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int k = (int)(u / nblk), tb = (int)(u - (int64_t)k * nblk);
    const int64_t t = g.t_beg + (int64_t)tb * 128 + threadIdx.x;
    float o[MN];
#pragma unroll
    for (int j = 0; j < MN; ++j) o[j] = 0.f;
#pragma unroll
    for (int x1 = 0; x1 < A0; ++x1, ++q) {
      const int st = (int)(q % ns);
      const uint32_t par = (uint32_t)((q / ns) & 1);
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(fb0 + 8u * st), "r"(par)
            : "memory");
      }
      float v[A1];
      const float* col = S + st * (A1 * 128) + threadIdx.x;
#pragma unroll
      for (int j = 0; j < A1; ++j) v[j] = col[j * 128];
      __syncthreads();  // every thread has read stage st: refill it ns groups ahead
      if (threadIdx.x == 0) issue(q + ns, st);
      accum_group<N, A, M, Tab, Ax>(o, v, x1, xp);
    }
    if (t < g.T) store_tile<N, M, Ax::M>(o, y, g, t, k);
  }
}

// Stages of the TMA-fed kernel: 2..kMaxOutStages groups of A1 x 128 floats
// within ~64 KB; 0 = plain kernel.  Measured (ncu, isolated kernels): the TMA
// ring wins when a thread has many points to load (c5, A1 = 64: 55.7 -> 49.5
// us) and loses when the groups are small (c2, A1 = 6: 28 -> 32 us; c3,
// A1 = 16: 0.55 -> 0.65 ms), where the per-group barrier and refill cost
// more than the plain loads' latency: TMA for A1 >= 32.
template <int N, int A>
constexpr int out_stages() {
  constexpr int A1 = ipow(A, N - 1);
  constexpr int bytes = A1 * 128 * 4;
  constexpr int n = (64 * 1024) / bytes;
  return (A1 < 32 || A1 > 256) ? 0 : n >= kMaxOutStages ? kMaxOutStages : n >= 2 ? n : 0;
}

template <int N, int A, int M, class Tab, class Ax = OAx0<A, M, Tab>>
cudaError_t launch_out(const float* Mx, float* y, const KGeom& g, const XfParams& xp, const CUtensorMap* tmM,
                       cudaStream_t s) {
  constexpr int ns = out_stages<N, A>();
  if constexpr (ns > 0) {
    if (tmM) {
      auto kern = k_output_xform_tma<N, A, M, Tab, Ax>;
      constexpr int smem = ns * ipow(A, N - 1) * 128 * 4;
      // per-device cache: the shared-memory opt-in is a per-context attribute
      static int grid_per_sm_dev[kMaxDevices] = {}, sms_dev[kMaxDevices] = {};
      int dev = 0;
      if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
      int& grid_per_sm = grid_per_sm_dev[dev];
      int& sms = sms_dev[dev];
      if (!grid_per_sm) {
        if (smem > 46 * 1024) {
          cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          if (e != cudaSuccess) return e;
        }
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&grid_per_sm, kern, 128, smem) != cudaSuccess ||
            grid_per_sm < 1)
          grid_per_sm = 1;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
          sms = 148;
      }
      const int64_t nunits = ((g.T - g.t_beg + 127) / 128) * (int64_t)g.K;
      int64_t grid = (int64_t)grid_per_sm * sms;
      if (grid > nunits) grid = nunits;
      return launch_pdl(kern, dim3((unsigned)grid), dim3(128), smem, s, y, g, xp, *tmM, ns);
    }
  }
  dim3 grid((unsigned)((g.T - g.t_beg + 127) / 128), (unsigned)g.K);
  return launch_pdl(k_output_xform<N, A, M, Tab, Ax>, grid, dim3(128), 0, s, Mx, y, g, xp);
}

template <int A, int M, class Tab>
cudaError_t launch_out_byN(int N, const float* Mx, float* y, const KGeom& g, const XfParams& xp,
                           const CUtensorMap* tmM, cudaStream_t s) {
  switch (N) {
    case 1: return launch_out<1, A, M, Tab>(Mx, y, g, xp, tmM, s);
    case 2: return launch_out<2, A, M, Tab>(Mx, y, g, xp, tmM, s);
    case 3: return launch_out<3, A, M, Tab>(Mx, y, g, xp, tmM, s);
    case 4:
      if constexpr (ipow(A, 3) <= 64) return launch_out<4, A, M, Tab>(Mx, y, g, xp, tmM, s);
      else return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
}

}  // namespace out_detail

cudaError_t launch_output_const(int N, int alpha, int m, int spec, const float* Mx, float* y, const KGeom& g,
                                const XfParams& xp, const CUtensorMap* tmM, cudaStream_t s);
cudaError_t launch_output_run(int N, int alpha, int m, const float* Mx, float* y, const KGeom& g,
                              const XfParams& xp, const CUtensorMap* tmM, cudaStream_t s);

}  // namespace wino
