// xform_in.cuh -- stage a2, the input-tile (data) transform of the N-D
// Winograd layer on sm_100a (kernel template; instantiated by
// xform_in_const.cu for the compile-time tables, xform_in_run(8).cu for
// run-time tables and xform_mixed.cu for per-axis plans):
//
//   V_xi[c][t] = (d(b, c, t) x_1 B_1^T x_2 ... x_N B_N^T)_xi        (Eq. (4))
//
// where d(b, c, t) is the window of x starting at t_n*m_n - P_n, zero
// outside the input (readings #2, #10).
//
// Design: the stage is HBM-bound (x read once, V written
// once, V = (alpha/m)^N x larger than x).  A slab is one (b, c) plane's input
// under tiles [a, a+bt0) of axis 0 and all tiles of the other axes (a
// contiguous run of t); a CTA owns g.npl consecutive slabs of one channel and
//   1. stages them into shared memory: one TMA box load per slab whose
//      out-of-bounds fill supplies the zero padding (kTma), or coalesced
//      4-byte cp.async (fallback for shapes that break a TMA rule); each
//      thread waits only for the slabs of its own work items,
//   2. pools the work items of all its slabs: N <= 2: one item per tile, the
//      whole window in registers; N = 3, alpha >= 6: the axis-0 pass in
//      shared memory (in place for one-tile-deep slabs), then one item per
//      (xi_0, tile), xi_0 outermost; other N >= 3: one item per (xi_0, tile)
//      with the axis-0 combination h = sum_i B^T[xi_0][i] slab_row(i)
//      (compile-time xi_0: zero entries skipped); r = 1 on the other axes:
//      one item per pixel column; window rows are read with 64/128-bit
//      shared loads,
//   3. writes V[xi][c][t]; lanes hold consecutive t, so every warp store is
//      one coalesced 128-byte line.
// Axis 0's transform (alpha_0, m_0, table) is a template parameter, equal to
// the other axes' except for per-axis plans.
//
// TMA requires the innermost start coordinate to be 16-byte aligned
// (measured: a start of -1 float faults, -4 works), so the TMA slab starts
// D = (-P_last) mod 4 columns early and the window reads are shifted by the
// compile-time D.
#pragma once
#include "kernels.h"
#include "xform_common.cuh"

namespace wino {
namespace in_detail {

__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}

// Read slab columns [Q, END) of a row whose base p is aligned to CAP floats,
// with the widest aligned vector loads.
template <int CAP, int Q, int END>
__device__ __forceinline__ void load_seg(const float* p, float* r) {
  if constexpr (Q < END) {
    constexpr int W = (CAP >= 4 && Q % 4 == 0 && Q + 4 <= END) ? 4
                      : (CAP >= 2 && Q % 2 == 0 && Q + 2 <= END) ? 2 : 1;
    if constexpr (W == 4) {
      const float4 v = *reinterpret_cast<const float4*>(p + Q);
      r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
    } else if constexpr (W == 2) {
      const float2 v = *reinterpret_cast<const float2*>(p + Q);
      r[0] = v.x; r[1] = v.y;
    } else {
      r[0] = p[Q];
    }
    load_seg<CAP, Q + W, END>(p, r + W);
  }
}

// A window values of one row: columns [D, D + A) of base p (p aligned to m floats).
template <int A, int M, int D>
__device__ __forceinline__ void load_row(const float* p, float* r) {
  constexpr int cap = M % 4 == 0 ? 4 : M % 2 == 0 ? 2 : 1;
  load_seg<cap, D, D + A>(p, r);
}

// A window values of one 16-byte aligned row with ceil(A/4) 128-bit loads
// (the tail load reads up to 3 floats past the window; the caller keeps them
// inside the row).  Lanes whose rows start at consecutive 16-byte groups then
// hit 8 distinct bank groups per quarter warp on every load.
template <int A>
__device__ __forceinline__ void load_row_wide(const float* p, float* r) {
#pragma unroll
  for (int q = 0; q < (A + 3) / 4; ++q) {
    const float4 v = *reinterpret_cast<const float4*>(p + 4 * q);
    if (4 * q + 0 < A) r[4 * q + 0] = v.x;
    if (4 * q + 1 < A) r[4 * q + 1] = v.y;
    if (4 * q + 2 < A) r[4 * q + 2] = v.z;
    if (4 * q + 3 < A) r[4 * q + 3] = v.w;
  }
}

// Axis-0 transform of a plan: F(M0, .) with alpha_0 = A0 and table Tab0.
// Equal to the other axes' (A, M, Tab) for the usual single-(m, r) plans; a
// different one for the per-axis plans with a distinct axis 0 (e.g. F(2,3)
// along time and F(4,3) along space, NEXT-2, Eq. (4)).
template <int A0_, int M0_, class Tab0_>
struct Ax0 {
  static constexpr int A = A0_;
  static constexpr int M = M0_;
  using Tab = Tab0_;
};

// dev probe (g.trace): %globaltimer of CTA event ev
__device__ __forceinline__ void in_trace(const KGeom& g, int ev) {
  if (g.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g.trace[(size_t)blockIdx.x * 8 + ev] = t;
    if (ev == 1) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      g.trace[(size_t)blockIdx.x * 8] = sm;
    }
  }
}

// V store flavour (dev A/B builds, tools/build_variant.sh): 0 plain (default),
// 1 st.cs (streaming), 2 st.cg, 3 st.wt
#ifndef WINO_VPUT_MODE
#define WINO_VPUT_MODE 0
#endif
__device__ __forceinline__ void vput(float* p, float v, float& vm) {
  (void)vm;
#if WINO_VPUT_MODE == 1
  __stcs(p, v);
#elif WINO_VPUT_MODE == 2
  __stcg(p, v);
#elif WINO_VPUT_MODE == 3
  __stwt(p, v);
#else
  *p = v;
#endif
}
// max|V| of the stored values for the 3xFP16 GEMM's scale (g.vmax set): one
// uniform test per work item, the FMNMX only in such plans (a per-store max
// in every plan cost c2's input transform ~4%)
template <int NV>
__device__ __forceinline__ void vtrack(const KGeom& g, const float* h, float& vm) {
  if (g.vmax) {
#pragma unroll
    for (int j = 0; j < NV; ++j) vm = fmaxf(vm, fabsf(h[j]));
  }
}

// One work item: axis-0 output point X0 of one tile whose window starts at
// slab offset `base` (+ D columns); writes alpha^(N-1) values of V.  Y0 >= 0:
// also the mirrored point Y0 (B^T[Y0][i] = (-1)^i B^T[X0][i]) from the same
// slab-row loads: the even- and odd-i0 partial sums e, o give X0 = e + o and
// Y0 = e - o (half the shared-memory reads of two separate items).
template <int N, int A, int M, class Tab, int D, int X0, class Ax, int Y0 = -1>
__device__ __forceinline__ void in_work(const float* __restrict__ S, int base, const KGeom& g,
                                        const XfParams& xp, float* __restrict__ vout, int64_t pstride, float& vm) {
  using Get = BTget<Tab>;
  using Get0 = BTget<typename Ax::Tab>;
  if constexpr (N == 1) {
    float h[A];
    load_row<A, M, D>(S + base, h);
    all_axes<A, 1, A, A, Get>(h, xp);
#pragma unroll
    for (int j = 0; j < A; ++j) vput(vout + j * pstride, h[j], vm);
    vtrack<A>(g, h, vm);
  } else if constexpr (N == 2 && Ax::A == A && Ax::M == M) {
    // the whole alpha x alpha window in registers: every window row is read
    // once (no per-xi_0 re-reads), both axes transformed in place
    float h[A * A];
#pragma unroll
    for (int i0 = 0; i0 < A; ++i0) load_row<A, M, D>(S + base + i0 * g.sst[0], h + i0 * A);
    all_axes<A, 2, A, A, Get>(h, xp);
#pragma unroll
    for (int j = 0; j < A * A; ++j) vput(vout + j * pstride, h[j], vm);
    vtrack<A * A>(g, h, vm);
  } else if constexpr (Y0 >= 0) {
    constexpr int NL = N - 1;
    constexpr int P1 = ipow(A, NL);
    constexpr int ROWS = ipow(A, NL - 1);
    float e[P1], o[P1];
#pragma unroll
    for (int j = 0; j < P1; ++j) { e[j] = 0.f; o[j] = 0.f; }
    bool fe = true, fo = true;
    sfor<0, Ax::A>([&](auto I0) {
      constexpr int i0 = decltype(I0)::value;
      constexpr float bv = Get0::cv(X0, i0);
      if constexpr (bv != 0.f) {
        float* h = (i0 & 1) ? o : e;
        const bool first = (i0 & 1) ? fo : fe;
#pragma unroll
        for (int rw = 0; rw < ROWS; ++rw) {
          int off = base + i0 * g.sst[0];
#pragma unroll
          for (int ax = 1; ax < N - 1; ++ax) off += ((rw / ipow(A, N - 2 - ax)) % A) * g.sst[ax];
          float r[A];
          load_row<A, M, D>(S + off, r);
#pragma unroll
          for (int i = 0; i < A; ++i) h[rw * A + i] = first ? bv * r[i] : fmaf(bv, r[i], h[rw * A + i]);
        }
        if (i0 & 1) fo = false; else fe = false;
      }
    });
#pragma unroll
    for (int j = 0; j < P1; ++j) {
      const float t = e[j];
      e[j] = t + o[j];
      o[j] = t - o[j];
    }
    all_axes<A, NL, A, A, Get>(e, xp);
#pragma unroll
    for (int j = 0; j < P1; ++j) vput(vout + (X0 * P1 + j) * pstride, e[j], vm);
    vtrack<P1>(g, e, vm);
    all_axes<A, NL, A, A, Get>(o, xp);
#pragma unroll
    for (int j = 0; j < P1; ++j) vput(vout + (Y0 * P1 + j) * pstride, o[j], vm);
    vtrack<P1>(g, o, vm);
  } else {
    constexpr int NL = N - 1;            // axes handled in registers
    constexpr int P1 = ipow(A, NL);      // values per work item
    constexpr int ROWS = ipow(A, NL - 1);
    float h[P1];
#pragma unroll
    for (int j = 0; j < P1; ++j) h[j] = 0.f;
    bool first = true;
#pragma unroll
    for (int i0 = 0; i0 < Ax::A; ++i0) {
      if (!Get0::nz(xp, X0, i0)) continue;
      const float bv = Get0::v(xp, X0, i0);
#pragma unroll
      for (int rw = 0; rw < ROWS; ++rw) {
        int off = base + i0 * g.sst[0];
        // row rw enumerates (i_1 .. i_{N-2}) with i_{N-2} fastest
#pragma unroll
        for (int ax = 1; ax < N - 1; ++ax) off += ((rw / ipow(A, N - 2 - ax)) % A) * g.sst[ax];
        float r[A];
        load_row<A, M, D>(S + off, r);
#pragma unroll
        for (int i = 0; i < A; ++i) h[rw * A + i] = first ? bv * r[i] : fmaf(bv, r[i], h[rw * A + i]);
      }
      first = false;
    }
    all_axes<A, NL, A, A, Get>(h, xp);
#pragma unroll
    for (int j = 0; j < P1; ++j) vput(vout + (X0 * P1 + j) * pstride, h[j], vm);
    vtrack<P1>(g, h, vm);
  }
}

template <int N, int A, int M, class Tab, int D, class Ax, int X0 = 0>
__device__ __forceinline__ void in_dispatch(int xi0, const float* S, int base, const KGeom& g, const XfParams& xp,
                                            float* vout, int64_t pstride, float& vm) {
  if constexpr (X0 < Ax::A) {
    if (xi0 == X0) in_work<N, A, M, Tab, D, X0, Ax>(S, base, g, xp, vout, pstride, vm);
    else in_dispatch<N, A, M, Tab, D, Ax, X0 + 1>(xi0, S, base, g, xp, vout, pstride, vm);
  }
}

// Axis-0 work-item kinds of the combination path (N >= 3, or a distinct axis
// 0): with a constant table, one kind per output point that is not the
// mirror of an earlier one (xform_common.cuh mirror_any); a kind with a
// mirror writes both points.  Run tables: one kind per point.  Only where a
// pair item's two register sets stay small (2 alpha^(N-1) <= 32: F(2^3,3^3)
// measured 0.339 -> 0.322 ms on c3's input; F(2^4,3^4) with 2 x 64 values
// per item was slower, c5 61 -> 70 us).
template <int N, int A, class Ax>
constexpr bool in_pairs() { return 2 * ipow(A, N - 1) <= 32; }
template <int N, int A, class Ax>
constexpr int in_kinds() { return in_pairs<N, A, Ax>() ? mirror_kinds<BTget<typename Ax::Tab>, Ax::A>() : Ax::A; }

template <int N, int A, int M, class Tab, int D, class Ax, int K = 0>
__device__ __forceinline__ void in_dispatch_kind(int kind, const float* S, int base, const KGeom& g,
                                                 const XfParams& xp, float* vout, int64_t pstride, float& vm) {
  if constexpr (K < in_kinds<N, A, Ax>()) {
    if (kind == K) {
      using Get0 = BTget<typename Ax::Tab>;
      constexpr bool pairs = in_pairs<N, A, Ax>();
      constexpr int x0 = pairs ? kind_point<Get0, Ax::A>(K) : K;
      constexpr int y0 = pairs ? mirror_any<Get0, Ax::A>(x0) : -1;
      in_work<N, A, M, Tab, D, x0, Ax, y0>(S, base, g, xp, vout, pstride, vm);
    } else {
      in_dispatch_kind<N, A, M, Tab, D, Ax, K + 1>(kind, S, base, g, xp, vout, pstride, vm);
    }
  }
}

__device__ __forceinline__ void tma_load_slab(uint32_t dst, const CUtensorMap* tm, const int* co, uint32_t bar,
                                              int rank) {
  switch (rank) {
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
          "l"(tm), "r"(co[0]), "r"(co[1]), "r"(co[2]), "r"(bar)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
          "l"(tm), "r"(co[0]), "r"(co[1]), "r"(co[2]), "r"(co[3]), "r"(bar)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
          "l"(tm), "r"(co[0]), "r"(co[1]), "r"(co[2]), "r"(co[3]), "r"(co[4]), "r"(bar)
          : "memory");
      break;
  }
}

// Load plane (b, box, c)'s slab with cp.async (fallback path, D == 0).
template <int N, int A, int M>
__device__ __forceinline__ void load_slab_cpasync(float* S, const float* __restrict__ x, const KGeom& g, int b,
                                                  int a0, int nt0, int c, int o1) {
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(S);
    const int e0 = nt0 * M + (A - M);
    const float* __restrict__ xb = x + ((int64_t)b * g.C + c) * g.in_vol;
    int rows = N == 1 ? 1 : e0;
#pragma unroll
    for (int ax = 1; ax < N - 1; ++ax) rows *= g.e[ax];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    // last axis: extent and global start of the slab row
    const int eL = N == 1 ? e0 : g.e[N - 1];
    const int64_t startL = (N == 1 ? (int64_t)a0 * M : 0) - g.pad[N - 1];
    const int64_t inL = g.in[N - 1];
    const int cols = N == 1 ? (e0 + 3) / 4 * 4 : g.pitch;
    for (int row = warp; row < rows; row += nwarps) {
      // decode row -> slab coordinates (i_0 .. i_{N-2}); global = start + i
      int rem = row;
      bool ok = true;
      int64_t goff = 0;
      int soff = 0;
#pragma unroll
      for (int ax = N - 2; ax >= 0; --ax) {
        const int ext = ax == 0 ? e0 : g.e[ax];
        const int i = ax == 0 ? rem : rem % ext;
        rem = ax == 0 ? 0 : rem / ext;
        const int64_t p = (ax == 0 ? (int64_t)a0 * M : ax == 1 ? (int64_t)o1 : 0) - g.pad[ax] + i;
        ok = ok && p >= 0 && p < g.in[ax];
        goff += p * g.in_stride[ax];
        soff += i * g.sst[ax];
      }
      const float* src = xb + goff + startL;
      float* drow = S + soff;
      // columns [lo, hi) are copied, the rest are zero
      const int lo = ok ? (int)max((int64_t)0, -startL) : cols;
      const int hi = ok ? (int)min((int64_t)eL, inL - startL) : cols;
      const uint32_t dst = sbase + 4u * (uint32_t)soff;
      for (int col = lane; col < cols; col += 32) {
        if (col >= lo && col < hi) cp_async4(dst + 4u * col, src + col);
        else drow[col] = 0.f;
      }
    }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// L2 prefetch of the box issue_slab_tma would load (no shared-memory destination, no barrier).
template <int N, int M, int D>
__device__ __forceinline__ void prefetch_slab_tma(const CUtensorMap* tm, const KGeom& g, int b, int a0, int c, int o1) {
  int co[5];
  co[0] = -g.pad[N - 1] - D;
#pragma unroll
  for (int ax = 0; ax < N - 1; ++ax) co[N - 1 - ax] = (ax == 0 ? a0 * M : ax == 1 ? o1 : 0) - g.pad[ax];
  co[N] = b * g.C + c;
  if constexpr (N == 2)
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(tm), "r"(co[0]), "r"(co[1]),
                 "r"(co[2]) : "memory");
  else if constexpr (N == 3)
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(tm), "r"(co[0]),
                 "r"(co[1]), "r"(co[2]), "r"(co[3]) : "memory");
  else
    asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(tm), "r"(co[0]),
                 "r"(co[1]), "r"(co[2]), "r"(co[3]), "r"(co[4]) : "memory");
}

// Issue the TMA box of plane (b, box, c) into slab S (thread 0 only).
template <int N, int M, int D>
__device__ __forceinline__ void issue_slab_tma(float* S, const CUtensorMap* tm, const KGeom& g, int b, int a0, int c,
                                               int o1, uint32_t bar) {
  int co[5];
  co[0] = -g.pad[N - 1] - D;
#pragma unroll
  for (int ax = 0; ax < N - 1; ++ax) co[N - 1 - ax] = (ax == 0 ? a0 * M : ax == 1 ? o1 : 0) - g.pad[ax];
  co[N] = b * g.C + c;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(g.slab_bytes) : "memory");
  tma_load_slab((uint32_t)__cvta_generic_to_shared(S), tm, co, bar, N + 1);
}

// One staged plane of a CTA's group (the CTA owns npl consecutive work items
// w0 .. w0+npl-1: consecutive slabs of one channel, i.e. one contiguous run
// of t per (xi, c) in V).
struct PlaneInfo {
  int b, a0, nt0, c;
  int a1;   // first axis-1 tile of the slab (banded slabs; 0 otherwise)
};

// Transform the CTA's npl staged planes: slab p at S0 + p * slab_f -> V rows
// of its tiles.  Work items of all planes form one pool, so every round of
// the block keeps all warps busy and the V stores of neighbouring planes
// (adjacent t) are issued together.
template <int N, int A, int M, class Tab, int D, class Ax>
__device__ __forceinline__ void transform_planes(float* __restrict__ S0, int slab_f, float* __restrict__ H,
                                                 float* __restrict__ V, const KGeom& g, const XfParams& xp,
                                                 const PlaneInfo* pl, int npl, uint32_t mb0, float& vm) {
  const int64_t pstride = (int64_t)g.C * g.T_s;
  // slab p's TMA box has landed once its mbarrier completes phase 0; every
  // thread waits only for the slabs of its own items, in order, so work on
  // the first slab starts while the next ones are still in flight
  int landed = -1;
  auto ensure = [&](int p) {
    if (mb0 == 0u) return;
    while (landed < p) {
      ++landed;
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n\t}"
            : "=r"(done)
            : "r"(mb0 + 8u * landed)
            : "memory");
      }
    }
  };
  auto vbase = [&](int p) -> float* {
    return V + (int64_t)pl[p].c * g.T_s +
           ((int64_t)pl[p].b * g.Tps + (int64_t)pl[p].a0 * g.R + (int64_t)pl[p].a1 * g.R1 - g.t0);
  };
  // ---- a5 direct-axis fold (xform_dfold.cu): the outer axes 0 and 1 only.
  // One warp item per (plane, t_0, t_1): lane i owns the slab-column pair
  // (2i, 2i+1) of the zero-padded row (i <= tiles_2), transforms its two
  // alpha x alpha (i_0, i_1) windows and writes the S = g.df_S slots row * S
  // + i of its row per (xo, parity) plane of Z (slots past tiles_2 get zeros);
  // the warps of a block hold consecutive t_1, i.e. one contiguous run of
  // slots per plane.  S = 32: every warp store is one full 128-byte line.
  // Measured on c3: storing only the 29 data lanes of a 32-slot row left a
  // partial sector in every line, which L2 completed from DRAM (+0.23 GB
  // read, 0.46 instead of 0.20 ms); rows packed at S = 29 (116-byte stores
  // whose sectors complete in L2, 9% fewer GEMM rows) took 0.245 ms and the
  // GEMM 0.53 instead of 0.505 ms.
  if constexpr (N == 3 && A == 4 && M == 2 && Ax::A == 4 && Ax::M == 2) {
    if (g.dfold) {
      using Get = BTget<Tab>;
      const int tl1 = g.tiles[1], tl2 = g.tiles[2];
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
      const int64_t zstride = (int64_t)g.C * g.Tz;
      const int per = g.bt0 * tl1;               // warp items of a full-depth slab
      const int sst0 = g.sst[0], sst1 = g.sst[1];
      for (int u = warp; u < npl * per; u += nwarps) {
        const int p = u / per, w = u - p * per;
        const int t0l = w / tl1, t1 = w - t0l * tl1;
        if (t0l >= pl[p].nt0) continue;
        ensure(p);
        const bool act = lane <= tl2;
        const float* sp = S0 + p * slab_f + t0l * M * sst0 + t1 * M * sst1 + (act ? 2 * lane : 0) + D;
        float he[A * A], ho[A * A];
#pragma unroll
        for (int i0 = 0; i0 < A; ++i0) {
#pragma unroll
          for (int i1 = 0; i1 < A; ++i1) {
            he[i0 * A + i1] = act ? sp[i0 * sst0 + i1 * sst1] : 0.f;
            ho[i0 * A + i1] = act ? sp[i0 * sst0 + i1 * sst1 + 1] : 0.f;
          }
        }
        all_axes<A, 2, A, A, Get>(he, xp);
        all_axes<A, 2, A, A, Get>(ho, xp);
        float* zp = V + (int64_t)pl[p].c * g.Tz +
                    (((int64_t)pl[p].b * g.tiles[0] + pl[p].a0 + t0l) * tl1 + t1) * g.df_S + lane;
        if (lane < g.df_S) {
#pragma unroll
          for (int q = 0; q < A * A; ++q) {
            vput(zp + (2 * q) * zstride, he[q], vm);
            vput(zp + (2 * q + 1) * zstride, ho[q], vm);
          }
        }
        vtrack<A * A>(g, he, vm);
        vtrack<A * A>(g, ho, vm);
      }
      return;
    }
  }
  // ---- N = 3, alpha >= 6: the axis-0 pass materialised in shared memory
  if constexpr (N == 3 && A >= 6) {
    using Get = BTget<Tab>;
    using Get0 = BTget<typename Ax::Tab>;   // axis 0: alpha_0 = Ax::A, step Ax::M
    constexpr int A0 = Ax::A, M0 = Ax::M;
    const int e1 = g.e[1], e2 = g.e[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int tl1 = g.bt1, tl2 = g.tiles[2];   // slab-local tiles (axis 1 banded or whole)
    if (g.hinplace) {
      // bt0 = 1: phase 1 rewrites every slab column (y, x) with its alpha
      // axis-0 outputs, shifted D columns left (column x + D -> x) so that
      // the phase-2 window rows are 16-byte aligned (128/64-bit loads, fewer
      // bank conflicts).  A row belongs to one warp and is walked in
      // increasing x, and within a warp every lane's loads precede the
      // stores, so each source value is read before its slot is overwritten
      // (lanes = consecutive x, conflict-free)
      // (alpha_0 = 1, F(1,1): the axis-0 pass is the identity and is skipped;
      // phase 2 then reads the slab rows at their D offset)
      if constexpr (A0 > 1) {
      // rows r = p * e1 + y walked with (p, y) stepped incrementally (a
      // run-time division per row was a fifth of this pass's instructions)
      int p = 0, y = warp;
      while (y >= e1) { y -= e1; ++p; }
      if (g.trace && threadIdx.x == 0) { ensure(npl - 1); in_trace(g, 2); }
      if (g.in_flags & 8) {   // (dev probe, in_flags & 8: staging only -- wait for the slabs, no transform)
        ensure(npl - 1);
        return;
      }
      if (e2 <= 32 && !(g.in_flags & 2)) {
        // one pass per row: two rows per iteration (their loads issued
        // together), one warp sync between a row pair's reads and its shifted
        // writes; rows are private to the warp, so no sync between pairs
        const int sst0 = g.sst[0], sst1 = g.sst[1], nrows = npl * e1;
        const bool act = lane < e2;
        for (int r = warp; r < nrows; r += 2 * nwarps) {
          int p2 = p, y2 = y + nwarps;
          while (y2 >= e1) { y2 -= e1; ++p2; }
          const bool two = r + nwarps < nrows;
          ensure(two ? p2 : p);
          float* c1 = S0 + p * slab_f + y * sst1 + lane;
          float* c2 = S0 + p2 * slab_f + y2 * sst1 + lane;
          float v1[A0], v2[A0];
          if (act) {
#pragma unroll
            for (int i = 0; i < A0; ++i) v1[i] = c1[D + i * sst0];
            if (two) {
#pragma unroll
              for (int i = 0; i < A0; ++i) v2[i] = c2[D + i * sst0];
            }
          }
          __syncwarp();  // all reads of the pair before any shifted write
          if (act) {
            float w[A0];
            xform_line<A0, A0, Get0>(v1, w, xp);
#pragma unroll
            for (int x0 = 0; x0 < A0; ++x0) c1[x0 * sst0] = w[x0];
            if (two) {
              xform_line<A0, A0, Get0>(v2, w, xp);
#pragma unroll
              for (int x0 = 0; x0 < A0; ++x0) c2[x0 * sst0] = w[x0];
            }
          }
          p = p2;
          y = y2 + nwarps;
          while (y >= e1) { y -= e1; ++p; }
        }
      } else
      for (int r = warp; r < npl * e1; r += nwarps) {
        if (g.in_flags & 2) { p = r / e1; y = r - p * e1; }   // dev A/B: the plain division
        ensure(p);
        float* row = S0 + p * slab_f + y * g.sst[1];
        for (int xb = 0; xb < e2; xb += 32) {  // every lane runs every pass (warp-wide sync below)
          const int xh = xb + lane;
          const bool act = xh < e2;
          float v[A0];
#pragma unroll
          for (int i = 0; i < A0; ++i) v[i] = act ? row[xh + D + i * g.sst[0]] : 0.f;
          __syncwarp();  // all reads of this pass before any shifted write
          if (act) {
            float w[A0];
            xform_line<A0, A0, Get0>(v, w, xp);
#pragma unroll
            for (int x0 = 0; x0 < A0; ++x0) row[xh + x0 * g.sst[0]] = w[x0];
          }
          __syncwarp();  // writes of this pass before the next pass's reads
        }
        y += nwarps;
        while (y >= e1) { y -= e1; ++p; }
      }
      }
      __syncthreads();
      in_trace(g, 3);
      // phase 2: one work item per (xi_0, plane, t1, t2) on plane xi_0 of its
      // slab; xi_0 outermost, so a round of the block writes long runs of t
      // (npl planes are adjacent in t) into each of the alpha^2 planes of V
      // it touches (measured: the V store pattern bounds this kernel).
      // g.in_pad8: t2 runs over 8 slots per row (m = 4: window starts 16 bytes
      // apart, so the 8 lanes of a quarter warp read 8 distinct bank groups;
      // slots >= tl2 idle) -- no shared-memory bank conflicts
      if (g.in_align) {
        // line-aligned items: the CTA's planes are one contiguous run of t in
        // every V plane; item v of a xi_0 group is tile v - lead of that run,
        // lead = (run start) mod 32, so a warp's 32 lanes store one 128-byte
        // aligned line (the run's first and last lines are shared with the
        // neighbouring CTAs).  Planes of one channel only (same V row).
        const int Rt = tl1 * tl2, ntile = npl * Rt;
        const int lead = (int)((vbase(0) - V) & 31);
        const int NR = (lead + ntile + 31) & ~31;
        const bool onerow = pl[0].c == pl[npl - 1].c;
        if (onerow) {
          for (int u = threadIdx.x; u < A0 * NR; u += blockDim.x) {
            const int xi0 = u / NR, tau = u - xi0 * NR - lead;
            if (tau < 0 || tau >= ntile) continue;
            const int p = tau / Rt, rem = tau - p * Rt;
            const int t1 = rem / tl2, t2 = rem - t1 * tl2;
            const float* hp0 = S0 + p * slab_f + xi0 * g.sst[0] + t1 * M * g.sst[1] + t2 * M;
            float h[A * A];
            if constexpr (A0 == 1) ensure(p);
            constexpr int DS = A0 > 1 ? 0 : D;
            // (two 128-bit loads per row instead of 128 + 64 bits: no change, c4 input 0.185 ms either way)
#pragma unroll
            for (int i1 = 0; i1 < A; ++i1) load_row<A, M, DS>(hp0 + i1 * g.sst[1], h + i1 * A);
            all_axes<A, 2, A, A, Get>(h, xp);
            float* vo = vbase(p) + rem + (int64_t)xi0 * (A * A) * pstride;
#pragma unroll
            for (int j = 0; j < A * A; ++j) vput(vo + j * pstride, h[j], vm);
            vtrack<A * A>(g, h, vm);
          }
          return;
        }
      }
      const int tl2p = g.in_pad8 ? (tl2 + 7) / 8 * 8 : tl2;
      const int R = tl1 * tl2p, nrun = npl * R;
      // item u = ((xi0 * npl + p) * tl1 + t1) * tl2 + t2, stepped by the block
      // size with mixed-radix carries (three run-time divisions per item
      // otherwise); the step's digits are computed once
      const int ustep = blockDim.x;
      const int st2 = ustep % tl2p, st1 = (ustep / tl2p) % tl1, stp = (ustep / R) % npl, sxi = ustep / nrun;
      int xi0, p, t1, t2;
      {
        const int u0 = threadIdx.x;
        xi0 = u0 / nrun;
        p = (u0 / R) % npl;
        t1 = (u0 / tl2p) % tl1;
        t2 = u0 % tl2p;
      }
      for (int u = threadIdx.x; u < A0 * nrun; u += ustep) {
        if (g.in_flags & 1) {   // dev A/B: the plain divisions
          xi0 = u / nrun;
          p = (u / R) % npl;
          t1 = (u / tl2p) % tl1;
          t2 = u % tl2p;
        }
        if (t2 < tl2) {
          const int tl = t1 * tl2 + t2;
          const float* hp0 = S0 + p * slab_f + xi0 * g.sst[0] + t1 * M * g.sst[1] + t2 * M;
          float h[A * A];
          if constexpr (A0 == 1) ensure(p);
          constexpr int DS = A0 > 1 ? 0 : D;  // shifted by phase 1, else at the TMA offset
          if constexpr (DS == 0 && M % 4 == 0) {
            if (g.in_pad8) {
#pragma unroll
              for (int i1 = 0; i1 < A; ++i1) load_row_wide<A>(hp0 + i1 * g.sst[1], h + i1 * A);
            } else {
#pragma unroll
              for (int i1 = 0; i1 < A; ++i1) load_row<A, M, DS>(hp0 + i1 * g.sst[1], h + i1 * A);
            }
          } else {
#pragma unroll
            for (int i1 = 0; i1 < A; ++i1) load_row<A, M, DS>(hp0 + i1 * g.sst[1], h + i1 * A);
          }
          all_axes<A, 2, A, A, Get>(h, xp);
          float* vo = vbase(p) + tl + (int64_t)xi0 * (A * A) * pstride;
          if (!(g.in_flags & 4)) {   // (dev probe, in_flags & 4: no V stores; results invalid)
#pragma unroll
            for (int j = 0; j < A * A; ++j) vput(vo + j * pstride, h[j], vm);
          }
          vtrack<A * A>(g, h, vm);
        }
        // next item: add the step digit by digit (t2 fastest)
        t2 += st2;
        int cy = t2 >= tl2p;
        t2 -= cy ? tl2p : 0;
        t1 += st1 + cy;
        cy = t1 >= tl1;
        t1 -= cy ? tl1 : 0;
        p += stp + cy;
        cy = p >= npl;
        p -= cy ? npl : 0;
        xi0 += sxi + cy;
      }
      return;
    }
    // separate H buffer (npl = 1): H = [t0][xi_0][y][x], window rows 16-byte aligned
    ensure(0);
    const PlaneInfo& q = pl[0];
    const int hp = g.hpitch, nt0 = q.nt0;
    // phase 1: one thread per (t0, y, x) column: alpha values along axis 0
    // (conflict-free scalar LDS, lanes = consecutive x) -> alpha xi_0 outputs
    for (int r = warp; r < nt0 * e1; r += nwarps) {
      const int y = r % e1, t0l = r / e1;
      for (int xh = lane; xh < e2; xh += 32) {
        const float* col = S0 + t0l * M0 * g.sst[0] + y * g.sst[1] + xh + D;
        float v[A0];
#pragma unroll
        for (int i = 0; i < A0; ++i) v[i] = col[i * g.sst[0]];
        float* hrow = H + (t0l * A0 * e1 + y) * hp + xh;
        float w[A0];
        xform_line<A0, A0, Get0>(v, w, xp);
#pragma unroll
        for (int x0 = 0; x0 < A0; ++x0) hrow[x0 * e1 * hp] = w[x0];
      }
    }
    __syncthreads();
    // phase 2: one work item per (t0, xi_0, t1, t2): the alpha x alpha window
    // of plane (t0, xi_0) in registers, axes 1 and 2 transformed in place
    float* __restrict__ vb = vbase(0);
    for (int w = threadIdx.x; w < nt0 * A0 * tl1 * tl2; w += blockDim.x) {
      const int t2 = w % tl2;
      int r = w / tl2;
      const int t1 = r % tl1;
      r /= tl1;
      const int xi0 = r % A0, t0l = r / A0;
      const float* hp0 = H + ((t0l * A0 + xi0) * e1 + t1 * M) * hp + t2 * M;
      float h[A * A];
#pragma unroll
      for (int i1 = 0; i1 < A; ++i1) load_row<A, M, 0>(hp0 + i1 * hp, h + i1 * A);
      all_axes<A, 2, A, A, Get>(h, xp);
      float* vo = vb + (t0l * tl1 + t1) * tl2 + t2 + (int64_t)xi0 * (A * A) * pstride;
#pragma unroll
      for (int j = 0; j < A * A; ++j) vput(vo + j * pstride, h[j], vm);
      vtrack<A * A>(g, h, vm);
    }
  } else if constexpr (A == 1 && M == 1 && N >= 2) {
    // ---- r = 1 on every axis but 0 (3x1x1-type kernels): a tile is one
    // pixel column; one work item per (plane, depth tile, pixel) reads the
    // alpha_0 values along axis 0 (lanes = consecutive pixels: conflict-free
    // loads, coalesced stores) and writes all alpha_0 points
    using Get0 = BTget<typename Ax::Tab>;
    constexpr int A0 = Ax::A, M0 = Ax::M;
    const int R = g.Rs, nper = g.bt0 * R;
    for (int u = threadIdx.x; u < npl * nper; u += blockDim.x) {
      const int p = u / nper;
      const int w = u - p * nper;
      const int t0l = w / R, rr = w - t0l * R;
      if (t0l >= pl[p].nt0) continue;
      ensure(p);
      int rem = rr, off = t0l * M0 * g.sst[0];
#pragma unroll
      for (int ax = N - 1; ax >= 1; --ax) {
        const int ext = ax == 1 ? g.bt1 : g.tiles[ax];
        const int ti = rem % ext;
        rem /= ext;
        off += ti * g.sst[ax];
      }
      const float* col = S0 + p * slab_f + off + D;
      float v[A0];
#pragma unroll
      for (int i = 0; i < A0; ++i) v[i] = col[i * g.sst[0]];
      float* vo = vbase(p) + w;
#pragma unroll
      for (int x0 = 0; x0 < A0; ++x0) {
        float acc = 0.f;
        bool first = true;
#pragma unroll
        for (int i = 0; i < A0; ++i) {
          if (Get0::nz(xp, x0, i)) {
            acc = first ? Get0::v(xp, x0, i) * v[i] : fmaf(Get0::v(xp, x0, i), v[i], acc);
            first = false;
          }
        }
        vput(vo + x0 * pstride, acc, vm);
        if (g.vmax) vm = fmaxf(vm, fabsf(acc));
      }
    }
  } else {
    // ---- work items (plane, xi_0, tile), tile fastest
    // work items per tile: one per xi_0 when N >= 3 or when axis 0 has its
    // own transform (N = 2 per-axis plans); one whole tile otherwise
    constexpr bool kComb = N >= 3 || Ax::A != A || Ax::M != M;   // axis-0 combination items
    constexpr int NX = kComb ? in_kinds<N, A, Ax>() : 1;
    if (npl == 1) {
      // one plane: no plane index to decode (the common case for large slabs)
      ensure(0);
      const int ntile = pl[0].nt0 * g.Rs;
      float* __restrict__ vb = vbase(0);
      // g.in_align: item w of a xi_0 group is tile w - lead, lead = (the plane's
      // first V row) mod 32, so a warp's lanes store one 128-byte aligned line
      // (g.in_align >= 2 only: measured neutral on c5 and slower on c3's V path, 0.328 -> 0.335 ms)
      const int lead = g.in_align >= 2 ? (int)((vb - V) & 31) : 0;
      const int NR = g.in_align >= 2 ? ((lead + ntile + 31) & ~31) : ntile;
      for (int w = threadIdx.x; w < NX * NR; w += blockDim.x) {
        const int xi0 = w / NR;
        const int tl = w - xi0 * NR - lead;
        if (tl < 0 || tl >= ntile) continue;
        int rem = tl, base = 0;
#pragma unroll
        for (int ax = N - 1; ax >= 1; --ax) {
          const int ext = ax == 1 ? g.bt1 : g.tiles[ax];
          const int ti = rem % ext;
          rem /= ext;
          base += ti * M * g.sst[ax];
        }
        base += rem * Ax::M * g.sst[0];
        if constexpr (kComb) in_dispatch_kind<N, A, M, Tab, D, Ax>(xi0, S0, base, g, xp, vb + tl, pstride, vm);
        else in_dispatch<N, A, M, Tab, D, Ax>(xi0, S0, base, g, xp, vb + tl, pstride, vm);
      }
      return;
    }
    const int ntile = g.bt0 * g.Rs;           // tiles of a full-depth slab
    const int nper = NX * ntile;
    // g.in_align, full-depth planes of one channel (one contiguous run of t in
    // every V plane): pooled line-aligned items -- item v of a xi_0 group is
    // tile v - lead of the run, lead = (run start) mod 32, so a warp's lanes
    // store one 128-byte aligned line.  Otherwise items (plane, xi_0, tile).
    // (g.in_align >= 2 only: measured slower on c2, input 33.1 -> 34.5 us)
    const bool pooled = g.in_align >= 2 && pl[0].c == pl[npl - 1].c && pl[npl - 1].nt0 == g.bt0;
    const int nrun = npl * ntile;
    const int lead = pooled ? (int)((vbase(0) - V) & 31) : 0;
    const int NR = (lead + nrun + 31) & ~31;
    const int total = pooled ? NX * NR : npl * nper;
    for (int u = threadIdx.x; u < total; u += blockDim.x) {
      int p, xi0, tl;
      if (pooled) {
        xi0 = u / NR;
        const int tau = u - xi0 * NR - lead;
        if (tau < 0 || tau >= nrun) continue;
        p = tau / ntile;
        tl = tau - p * ntile;
      } else {
        p = u / nper;
        const int w = u - p * nper;
        xi0 = w / ntile;
        tl = w - xi0 * ntile;
        if (tl >= pl[p].nt0 * g.Rs) continue;   // last axis-0 box of a sample is shorter
      }
      ensure(p);
      // local tile -> slab offset of its window
      int rem = tl, base = 0;
#pragma unroll
      for (int ax = N - 1; ax >= 1; --ax) {
        const int ext = ax == 1 ? g.bt1 : g.tiles[ax];
        const int ti = rem % ext;
        rem /= ext;
        base += ti * M * g.sst[ax];
      }
      base += rem * Ax::M * g.sst[0];
      if constexpr (kComb)
        in_dispatch_kind<N, A, M, Tab, D, Ax>(xi0, S0 + p * slab_f, base, g, xp, vbase(p) + tl, pstride, vm);
      else
        in_dispatch<N, A, M, Tab, D, Ax>(xi0, S0 + p * slab_f, base, g, xp, vbase(p) + tl, pstride, vm);
    }
  }
}

// A CTA owns npl = g.npl consecutive work items w (one (b, c) plane slab =
// tiles [a0, a0 + bt0) of axis 0 each; consecutive w are consecutive slabs of
// the same channel).  kTma (N >= 2): each slab is one TMA box starting D
// columns left of -P_last, all npl boxes issued at once; !kTma: cp.async
// fallback, D == 0.
// Block-size bound: 512 for the N = 3, alpha >= 6 (H mode) instantiations,
// whose four-slab CTAs run 384 threads (plan_input_planes); 256 elsewhere,
// which keeps the other instantiations at <= 48 registers (measured: the
// 512 bound raises them to 64 and costs c2 32.7 -> 34.5 us).
template <int N, int A>
constexpr int in_max_threads() { return (N == 3 && A >= 6) ? 512 : 256; }

template <int N, int A, int M, class Tab, int D, bool kTma, class Ax = Ax0<A, M, Tab>>
__global__ void __launch_bounds__(in_max_threads<N, A>())
k_input_xform(const float* __restrict__ x, float* __restrict__ V, const __grid_constant__ KGeom g,
              const __grid_constant__ XfParams xp, const __grid_constant__ CUtensorMap tm, int nslab) {
  extern __shared__ __align__(128) float smem_f[];
  __shared__ __align__(8) uint64_t bar[kMaxPlanes];
  __shared__ PlaneInfo pl[kMaxPlanes];
  const int slab_f = g.slot_bytes / 4;  // slot stride: 128-byte aligned TMA destinations
  float* H = smem_f + g.npl * slab_f;
  const int nwork = nslab * g.C;
  const int w0 = blockIdx.x * g.npl;
  const int npl = min(g.npl, nwork - w0);
  // slab indices of one launch fit 32 bits (nwork is an int): unsigned
  // divisions here -- the int64 ones, five plane decodes in a row on thread
  // 0 ahead of the TMA issue, held the whole block at the first barrier
  // (ncu: 18% of the c4 kernel's warp samples on that barrier)
  auto plane = [&](int w) {
    PlaneInfo q;
    const unsigned slab = (unsigned)(g.s_beg + (unsigned)w % (unsigned)nslab);   // ((b * nbox0 + box0) * nbox1 + box1)
    q.c = (int)((unsigned)w / (unsigned)nslab);
    const unsigned s0 = slab / (unsigned)g.nbox1;
    q.a1 = (int)(slab - s0 * (unsigned)g.nbox1) * g.bt1;
    q.b = (int)(s0 / (unsigned)g.nbox0);
    const int box = (int)(s0 - (unsigned)q.b * (unsigned)g.nbox0);
    q.a0 = box * g.bt0;
    q.nt0 = min(g.bt0, g.tiles[0] - q.a0);
    return q;
  };
  PlaneInfo mine{};
  if (threadIdx.x < npl) {
    mine = plane(w0 + threadIdx.x);
    pl[threadIdx.x] = mine;
  }
  pdl_wait();      // x may come from the preceding kernel; V is read by the previous GEMM
  pdl_trigger();
  in_trace(g, 1);
  if constexpr (kTma) {
    static_assert(N >= 2, "TMA slab path needs N >= 2");
    const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
    // lane 0 initialises the slab barriers, then lane p (< npl <= 8, all in
    // warp 0) issues slab p's box
    if (threadIdx.x == 0) {
      for (int p = 0; p < npl; ++p) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8u * p) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) __syncwarp();
    if (threadIdx.x < npl) {
      const int p = threadIdx.x;
      issue_slab_tma<N, Ax::M, D>(smem_f + p * slab_f, &tm, g, mine.b, mine.a0, mine.c, mine.a1 * M, mb0 + 8u * p);
    }
    // the slabs of the CTA that will follow this one on its SM: under the
    // layer's write traffic a DRAM read takes microseconds, an L2 hit does not
    if (g.in_prefetch > 0 && threadIdx.x < g.npl) {
      const long long wn = (long long)w0 + (long long)g.in_prefetch * g.npl + threadIdx.x;
      if (wn < nwork) {
        const PlaneInfo q = plane((int)wn);
        prefetch_slab_tma<N, Ax::M, D>(&tm, g, q.b, q.a0, q.c, q.a1 * M);
      }
    }
    __syncthreads();
  } else {
    static_assert(D == 0, "the cp.async slab path is unshifted");
    __syncthreads();
    for (int p = 0; p < npl; ++p)
      load_slab_cpasync<N, Ax::A, Ax::M>(smem_f + p * slab_f, x, g, pl[p].b, pl[p].a0, pl[p].nt0, pl[p].c,
                                         pl[p].a1 * M);
    __syncthreads();
  }
  float vm = 0.f;
  transform_planes<N, A, M, Tab, D, Ax>(smem_f, slab_f, H, V, g, xp, pl, npl,
                                    kTma ? (uint32_t)__cvta_generic_to_shared(&bar[0]) : 0u, vm);
  if (g.trace) {
    __syncthreads();
    in_trace(g, 4);
  }
  // max|V| of the whole launch (the 3xFP16 GEMM's scale): block reduction,
  // one atomicMax per CTA (non-negative floats order as their bit patterns)
  if (g.vmax) {
    __shared__ float wmax[32];
    for (int o = 16; o; o >>= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = vm;
    __syncthreads();
    if (threadIdx.x < 32) {
      vm = threadIdx.x < (blockDim.x >> 5) ? wmax[threadIdx.x] : 0.f;
      for (int o = 16; o; o >>= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, o));
      if (threadIdx.x == 0) atomicMax(g.vmax, __float_as_uint(vm));
    }
  }
}

template <class K>
inline cudaError_t set_smem(K kern, int bytes) {
  // the opt-in limit covers dynamic + static shared memory (barriers, plane table)
  if (bytes <= 46 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <class K>
inline cudaError_t launch_in_kern(K kern, const float* x, float* V, const KGeom& g, const XfParams& xp,
                                  const CUtensorMap& tm, int nslab, cudaStream_t s) {
  cudaError_t e;
  if ((e = set_smem(kern, g.smem_bytes)) != cudaSuccess) return e;
  const long long nwork = (long long)nslab * g.C;
  const long long grid = (nwork + g.npl - 1) / g.npl;
  return launch_pdl(kern, dim3((unsigned)grid), dim3(g.in_threads), g.smem_bytes, s, x, V, g, xp, tm, nslab);
}

// Launch one (N, alpha, m, table) instantiation over slabs [g.s_beg,
// g.s_beg + nslab).  tm != NULL selects the TMA slab (g.dL is its column
// shift, 0 or 3); kAllowTma = false compiles only the fallback (run-time tables).
template <int N, int A, int M, class Tab, bool kAllowTma, class Ax = Ax0<A, M, Tab>>
cudaError_t launch_in(const float* x, float* V, const KGeom& g, const XfParams& xp, const CUtensorMap* tm, int nslab,
                      cudaStream_t s) {
  if constexpr (kAllowTma && N >= 2) {
    if (tm && g.dL == 0) return launch_in_kern(k_input_xform<N, A, M, Tab, 0, true, Ax>, x, V, g, xp, *tm, nslab, s);
    if (tm && g.dL == 3) return launch_in_kern(k_input_xform<N, A, M, Tab, 3, true, Ax>, x, V, g, xp, *tm, nslab, s);
  }
  KGeom g1 = g;
  CUtensorMap dummy{};
  return launch_in_kern(k_input_xform<N, A, M, Tab, 0, false, Ax>, x, V, g1, xp, dummy, nslab, s);
}

template <int A, int M, class Tab, bool kAllowTma>
cudaError_t launch_in_byN(int N, const float* x, float* V, const KGeom& g, const XfParams& xp,
                          const CUtensorMap* tm, int nslab, cudaStream_t s) {
  switch (N) {
    case 1: return launch_in<1, A, M, Tab, kAllowTma>(x, V, g, xp, tm, nslab, s);
    case 2: return launch_in<2, A, M, Tab, kAllowTma>(x, V, g, xp, tm, nslab, s);
    case 3: return launch_in<3, A, M, Tab, kAllowTma>(x, V, g, xp, tm, nslab, s);
    case 4:
      if constexpr (ipow(A, 3) <= 64) return launch_in<4, A, M, Tab, kAllowTma>(x, V, g, xp, tm, nslab, s);
      else return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
}

}  // namespace in_detail

cudaError_t launch_input_const(int N, int alpha, int m, int spec, const float* x, float* V, const KGeom& g,
                               const XfParams& xp, const CUtensorMap* tm, int nslab, cudaStream_t s);
cudaError_t launch_input_run(int N, int alpha, int m, const float* x, float* V, const KGeom& g, const XfParams& xp,
                             const CUtensorMap* tm, int nslab, cudaStream_t s);

}  // namespace wino
