// xform_in.cu -- stage a2, the input-tile (data) transform of the N-D
// Winograd layer on sm_100a:
//
//   V_xi[c][t] = (d(b, c, t) x_1 B^T x_2 ... x_N B^T)_xi          (Eq. (4))
//
// where d(b, c, t) is the alpha^N window of x starting at t_n*m - P_n, zero
// outside the input (readings #2, #10).
//
// Design: the stage is HBM-bound (x read once, V written
// once, V = (alpha/m)^N x larger than x), so one CTA owns one (b, c) plane
// slab -- the input under tiles [a, a+bt0) of axis 0 and all tiles of the
// other axes, which is a contiguous run of t -- and
//   1. stages the slab into shared memory with coalesced 4-byte cp.async
//      (zero-fill supplies the padding, no branches in the math),
//   2. runs one work item per (xi_0, tile): the axis-0 combination
//      h = sum_i B^T[xi_0][i] slab_row(i) (compile-time xi_0, so zero
//      entries of B^T are skipped), then the remaining N-1 axes as register
//      line transforms, reading window rows with 64/128-bit shared loads,
//   3. writes the alpha^(N-1) values V[(xi_0, .)][c][t]; lanes hold
//      consecutive t, so every warp store is one coalesced 128-byte line.
#include "kernels.h"
#include "xform_common.cuh"

namespace wino {

namespace {

__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}

// Load A consecutive floats of a shared-memory row starting at p (p is
// aligned to m floats: 16 B for m % 4 == 0, 8 B for m % 2 == 0).
template <int A, int M>
__device__ __forceinline__ void load_row(const float* p, float* r) {
  if constexpr (M % 4 == 0) {
#pragma unroll
    for (int i = 0; i + 4 <= A; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(p + i);
      r[i] = v.x; r[i + 1] = v.y; r[i + 2] = v.z; r[i + 3] = v.w;
    }
    constexpr int q = A / 4 * 4;
    if constexpr (A - q >= 2) {
      const float2 v = *reinterpret_cast<const float2*>(p + q);
      r[q] = v.x; r[q + 1] = v.y;
    }
    if constexpr ((A - q) % 2 == 1) r[A - 1] = p[A - 1];
  } else if constexpr (M % 2 == 0) {
#pragma unroll
    for (int i = 0; i + 2 <= A; i += 2) {
      const float2 v = *reinterpret_cast<const float2*>(p + i);
      r[i] = v.x; r[i + 1] = v.y;
    }
    if constexpr (A % 2 == 1) r[A - 1] = p[A - 1];
  } else {
#pragma unroll
    for (int i = 0; i < A; ++i) r[i] = p[i];
  }
}

// One work item: axis-0 output point X0 of one tile whose window starts at
// slab offset `base`; writes alpha^(N-1) values of V (stride pstride per point).
template <int N, int A, int M, class Tab, int X0>
__device__ __forceinline__ void in_work(const float* __restrict__ S, int base, const KGeom& g,
                                        const XfParams& xp, float* __restrict__ vout, int64_t pstride) {
  using Get = BTget<Tab>;
  constexpr int NL = N - 1;              // axes handled in registers
  constexpr int P1 = ipow(A, NL);        // values per work item
  constexpr int ROWS = ipow(A, NL > 0 ? NL - 1 : 0);
  float h[P1];
  if constexpr (N == 1) {
    load_row<A, M>(S + base, h);
    all_axes<A, 1, A, A, Get>(h, xp);
#pragma unroll
    for (int j = 0; j < A; ++j) vout[j * pstride] = h[j];
    return;
  } else {
#pragma unroll
    for (int j = 0; j < P1; ++j) h[j] = 0.f;
    bool first = true;
#pragma unroll
    for (int i0 = 0; i0 < A; ++i0) {
      if (!Get::nz(xp, X0, i0)) continue;
      const float bv = Get::v(xp, X0, i0);
#pragma unroll
      for (int rw = 0; rw < ROWS; ++rw) {
        int off = base + i0 * g.sst[0];
        // row rw enumerates (i_1 .. i_{N-2}) with i_{N-2} fastest
#pragma unroll
        for (int ax = 1; ax < N - 1; ++ax) off += ((rw / ipow(A, N - 2 - ax)) % A) * g.sst[ax];
        float r[A];
        load_row<A, M>(S + off, r);
#pragma unroll
        for (int i = 0; i < A; ++i) h[rw * A + i] = first ? bv * r[i] : fmaf(bv, r[i], h[rw * A + i]);
      }
      first = false;
    }
    all_axes<A, NL, A, A, Get>(h, xp);
#pragma unroll
    for (int j = 0; j < P1; ++j) vout[(X0 * P1 + j) * pstride] = h[j];
  }
}

template <int N, int A, int M, class Tab, int X0 = 0>
__device__ __forceinline__ void in_dispatch(int xi0, const float* S, int base, const KGeom& g, const XfParams& xp,
                                            float* vout, int64_t pstride) {
  if constexpr (X0 < A) {
    if (xi0 == X0) in_work<N, A, M, Tab, X0>(S, base, g, xp, vout, pstride);
    else in_dispatch<N, A, M, Tab, X0 + 1>(xi0, S, base, g, xp, vout, pstride);
  }
}

template <int N, int A, int M, class Tab>
__global__ void __launch_bounds__(256)
k_input_xform(const float* __restrict__ x, float* __restrict__ V, const __grid_constant__ KGeom g,
              const __grid_constant__ XfParams xp) {
  extern __shared__ __align__(16) float S[];
  const int box = blockIdx.x, c = blockIdx.y, b = blockIdx.z;
  const int a0 = box * g.bt0;
  const int nt0 = min(g.bt0, g.tiles[0] - a0);
  const int e0 = nt0 * M + (A - M);
  const float* __restrict__ xb = x + ((int64_t)b * g.C + c) * g.in_vol;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(S);

  // ---- 1. slab -> shared memory (zero fill outside the input)
  {
    int rows = N == 1 ? 1 : e0;
#pragma unroll
    for (int ax = 1; ax < N - 1; ++ax) rows *= g.e[ax];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    // last axis: extent and global start of the slab row
    const int eL = N == 1 ? e0 : g.e[N - 1];
    const int64_t startL = (N == 1 ? (int64_t)a0 * M : 0) - g.pad[N - 1];
    const int64_t inL = g.in[N - 1];
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
        const int64_t p = (ax == 0 ? (int64_t)a0 * M : 0) - g.pad[ax] + i;
        ok = ok && p >= 0 && p < g.in[ax];
        goff += p * g.in_stride[ax];
        soff += i * g.sst[ax];
      }
      const float* src = xb + goff;
      const uint32_t dst = sbase + 4u * (uint32_t)soff;
      for (int col = lane; col < g.pitch; col += 32) {
        const int64_t p = startL + col;
        const bool v = ok && col < eL && p >= 0 && p < inL;
        cp_async4(dst + 4u * col, v ? src + p : xb, v);
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }

  // ---- 2./3. work items (xi_0, tile), tile fastest
  const int ntile = nt0 * g.R;
  constexpr int NX = N >= 2 ? A : 1;
  const int64_t pstride = (int64_t)g.C * g.T_s;
  const int64_t t0g = (int64_t)b * g.Tps + (int64_t)a0 * g.R;
  float* __restrict__ vbase = V + (int64_t)c * g.T_s + t0g;
  for (int w = threadIdx.x; w < NX * ntile; w += blockDim.x) {
    const int xi0 = w / ntile;
    const int tl = w - xi0 * ntile;
    // local tile -> slab offset of its window
    int rem = tl, base = 0;
#pragma unroll
    for (int ax = N - 1; ax >= 1; --ax) {
      const int ti = rem % g.tiles[ax];
      rem /= g.tiles[ax];
      base += ti * M * g.sst[ax];
    }
    base += rem * M * g.sst[0];
    in_dispatch<N, A, M, Tab>(xi0, S, base, g, xp, vbase + tl, pstride);
  }
}

}  // namespace

// Slab geometry of k_input_xform for a plan (fills g.bt0 .. g.slab_bytes).
// Returns false if even a one-tile-deep slab exceeds shared memory.
bool plan_input_slab(KGeom& g, int N, int alpha, int m) {
  const int halo = alpha - m;
  int inner = 1;  // floats of one axis-0 slab slice
  g.R = 1;
  for (int n = 1; n < N; ++n) g.R *= g.tiles[n];
  for (int n = N - 1; n >= 1; --n) {
    g.e[n] = g.tiles[n] * m + halo;
    if (n == N - 1) {
      g.pitch = (g.e[n] + 3) / 4 * 4;
      g.sst[n] = 1;
      inner = g.pitch;
    } else {
      g.sst[n] = inner;
      inner *= g.e[n];
    }
  }
  if (N == 1) {
    g.pitch = 0;
    inner = 1;
  }
  g.sst[0] = inner;
  const size_t kTarget = 64 * 1024, kMax = 200 * 1024;
  int bt0 = g.tiles[0];
  auto bytes = [&](int bt) {
    const int e0 = bt * m + halo;
    if (N == 1) return (size_t)((e0 + 3) / 4 * 4) * 4;
    return (size_t)e0 * inner * 4;
  };
  while (bt0 > 1 && bytes(bt0) > kTarget) bt0 = (bt0 + 1) / 2;
  if (bytes(bt0) > kMax) return false;
  g.bt0 = bt0;
  g.nbox0 = (g.tiles[0] + bt0 - 1) / bt0;
  g.e[0] = bt0 * m + halo;
  if (N == 1) {
    // the slab is one row: pitch covers e0 (the kernel's row loop sees rows = 1)
    g.pitch = (g.e[0] + 3) / 4 * 4;
  }
  g.slab_bytes = (int)bytes(bt0);
  return true;
}

namespace {

template <int N, int A, int M, class Tab>
cudaError_t launch_in(const float* x, float* V, const KGeom& g, const XfParams& xp, int B, cudaStream_t s) {
  auto kern = k_input_xform<N, A, M, Tab>;
  static int attr_set = 0;
  if (g.slab_bytes > 48 * 1024 && attr_set < g.slab_bytes) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, g.slab_bytes);
    if (e != cudaSuccess) return e;
    attr_set = g.slab_bytes;
  }
  dim3 grid((unsigned)g.nbox0, (unsigned)g.C, (unsigned)B);
  kern<<<grid, 256, g.slab_bytes, s>>>(x, V, g, xp);
  return cudaGetLastError();
}

template <int A, int M, class Tab>
cudaError_t launch_in_byN(int N, const float* x, float* V, const KGeom& g, const XfParams& xp, int B,
                          cudaStream_t s) {
  switch (N) {
    case 1: return launch_in<1, A, M, Tab>(x, V, g, xp, B, s);
    case 2: return launch_in<2, A, M, Tab>(x, V, g, xp, B, s);
    case 3: return launch_in<3, A, M, Tab>(x, V, g, xp, B, s);
    case 4:
      if constexpr (ipow(A, 3) <= 64) return launch_in<4, A, M, Tab>(x, V, g, xp, B, s);
      else return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

cudaError_t launch_input_xform(int N, int alpha, int m, int spec, const float* x, float* V, const KGeom& g,
                               const XfParams& xp, int B, cudaStream_t s) {
  if (spec == kSpecDefault) {
    if (alpha == 4 && m == 2) return launch_in_byN<4, 2, ConstTab<2, 3, kPsDefault>>(N, x, V, g, xp, B, s);
    if (alpha == 6 && m == 4) return launch_in_byN<6, 4, ConstTab<4, 3, kPsDefault>>(N, x, V, g, xp, B, s);
  } else if (spec == kSpecSeq) {
    if (alpha == 4 && m == 2) return launch_in_byN<4, 2, ConstTab<2, 3, kPsSeq>>(N, x, V, g, xp, B, s);
    if (alpha == 6 && m == 4) return launch_in_byN<6, 4, ConstTab<4, 3, kPsSeq>>(N, x, V, g, xp, B, s);
  } else {
    switch (alpha * 16 + m) {
      case 4 * 16 + 2: return launch_in_byN<4, 2, RunTab>(N, x, V, g, xp, B, s);
      case 4 * 16 + 3: return launch_in_byN<4, 3, RunTab>(N, x, V, g, xp, B, s);
      case 5 * 16 + 3: return launch_in_byN<5, 3, RunTab>(N, x, V, g, xp, B, s);
      case 6 * 16 + 3: return launch_in_byN<6, 3, RunTab>(N, x, V, g, xp, B, s);
      case 6 * 16 + 4: return launch_in_byN<6, 4, RunTab>(N, x, V, g, xp, B, s);
      case 8 * 16 + 3: return launch_in_byN<8, 3, RunTab>(N, x, V, g, xp, B, s);
      case 8 * 16 + 4: return launch_in_byN<8, 4, RunTab>(N, x, V, g, xp, B, s);
      case 8 * 16 + 5: return launch_in_byN<8, 5, RunTab>(N, x, V, g, xp, B, s);
      default: break;
    }
  }
  return cudaErrorNotSupported;
}

}  // namespace wino
