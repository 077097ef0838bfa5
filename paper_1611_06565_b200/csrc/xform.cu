// xform.cu -- stages a1 (filter), a2 (input tile) and a4 (output tile)
// transforms of the N-D Winograd layer, sm_100a.
//
// Every transform is a chain of n-mode products (Eq. (3))
// applied separably per axis (Eq. (4)).  The transform
// matrices are tiny (alpha <= 8), so per (tile, channel) the work is done in
// registers with compile-time-unrolled line transforms; zero entries of the
// matrices are skipped at compile time for the default point sets ("U is
// sparse ... traversed in the outermost loops"; "exploiting the
// sparsity of the matrices themselves").
//
// Layouts:
//   x [B][C][in...]  ->  V [P][C][T_s]   (P = alpha^N points; T fastest so the
//                                         GEMM reads V as an MN-major operand)
//   M [P][K][T_s]    ->  y [B][K][out...]
//   g [K][C][r^N]    ->  U_hi, U_lo [P][C][K_s]  (MN-major B operand)
// t (tile index) is row-major over (b, t_1, ..., t_N); a warp's 32 lanes are
// 32 consecutive tiles, so every V / M access is a coalesced 128 B line.
#include "common.cuh"
#include "kernels.h"

namespace wino {

// Coefficient getters: value and "is this entry used" (constant for ConstTab).
template <class Tab>
struct BTget {
  __device__ static __forceinline__ float v(const XfParams& p, int x, int i) { return Tab::bt(p, x, i); }
  __device__ static __forceinline__ bool nz(const XfParams& p, int x, int i) {
    if constexpr (Tab::kConst) return Tab::bt(p, x, i) != 0.f; else return true;
  }
};
template <class Tab>
struct ATget {
  __device__ static __forceinline__ float v(const XfParams& p, int x, int i) { return Tab::at(p, x, i); }
  __device__ static __forceinline__ bool nz(const XfParams& p, int x, int i) {
    if constexpr (Tab::kConst) return Tab::at(p, x, i) != 0.f; else return true;
  }
};

__host__ __device__ constexpr bool leading_ok(int o, int ax, int A, int Mr) {
  // the `ax` leading base-A digits of o (indexing axes < ax) are all < Mr
  for (int i = 0; i < ax; ++i) {
    if (o % A >= Mr) return false;
    o /= A;
  }
  return true;
}

// In-place 1-D transform of every line along axis AX of a register array of
// A^NL floats (axis 0 slowest):  v[.., X, ..] = sum_I Get(X, I) v[.., I, ..]
// for X < R.  Axes < AX hold only Mr valid entries (already reduced).  All
// loops unroll fully, so the table reads are compile-time constants for
// ConstTab and unused (zero) terms disappear.
template <int A, int NL, int AX, int R, int Mr, class Get>
__device__ __forceinline__ void line_pass(float* v, const XfParams& p) {
  constexpr int stride = ipow(A, NL - 1 - AX);
  constexpr int outer = ipow(A, AX);
#pragma unroll
  for (int o = 0; o < outer; ++o) {
    if (!leading_ok(o, AX, A, Mr)) continue;
#pragma unroll
    for (int s = 0; s < stride; ++s) {
      const int base = o * A * stride + s;
      float in[A];
#pragma unroll
      for (int i = 0; i < A; ++i) in[i] = v[base + i * stride];
#pragma unroll
      for (int x = 0; x < R; ++x) {
        float acc = 0.f;
        bool first = true;
#pragma unroll
        for (int i = 0; i < A; ++i) {
          if (Get::nz(p, x, i)) {
            acc = first ? Get::v(p, x, i) * in[i] : fmaf(Get::v(p, x, i), in[i], acc);
            first = false;
          }
        }
        v[base + x * stride] = acc;
      }
    }
  }
}

template <int A, int NL, int R, int Mr, class Get>
__device__ __forceinline__ void all_axes(float* v, const XfParams& p) {
  if constexpr (NL > 0) line_pass<A, NL, 0, R, Mr, Get>(v, p);
  if constexpr (NL > 1) line_pass<A, NL, 1, R, Mr, Get>(v, p);
  if constexpr (NL > 2) line_pass<A, NL, 2, R, Mr, Get>(v, p);
  if constexpr (NL > 3) line_pass<A, NL, 3, R, Mr, Get>(v, p);
}

// ------------------------------------------------------------------ a2
// One thread per (tile t, channel c): gather the alpha^N window of x (zero
// outside the input: reading #10), apply B^T along every axis, write the
// alpha^N transformed values V[xi][c][t].
template <int N, int A, int M, class Tab>
__global__ void __launch_bounds__(128)
k_input_xform(const float* __restrict__ x, float* __restrict__ V, const __grid_constant__ KGeom g,
              const __grid_constant__ XfParams xp) {
  constexpr int P = ipow(A, N);
  const int64_t t = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int c = blockIdx.y;
  if (t >= g.T_s) return;
  const int64_t pstride = (int64_t)g.C * g.T_s;
  float* vout = V + (int64_t)c * g.T_s + t;
  if (t >= g.T) {  // GEMM row padding: zeros
#pragma unroll 4
    for (int i = 0; i < P; ++i) vout[i * pstride] = 0.f;
    return;
  }
  int64_t rem = t;
  int gi[N];
#pragma unroll
  for (int n = N - 1; n >= 0; --n) {
    gi[n] = (int)(rem % g.tiles[n]);
    rem /= g.tiles[n];
  }
  const float* xb = x + (rem * g.C + c) * g.in_vol;
  int64_t base = 0;
  uint32_t vmask[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    const int o = gi[n] * M - g.pad[n];
    base += (int64_t)o * g.in_stride[n];
    uint32_t mk = 0;
#pragma unroll
    for (int i = 0; i < A; ++i) mk |= (uint32_t)((o + i) >= 0 && (o + i) < g.in[n]) << i;
    vmask[n] = mk;
  }
  if constexpr (P <= 64) {
    // whole window in registers, N separable passes
    float w[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      bool ok = true;
      int64_t off = base;
#pragma unroll
      for (int ax = 0; ax < N; ++ax) {
        const int d = (j / ipow(A, N - 1 - ax)) % A;
        ok = ok && ((vmask[ax] >> d) & 1u);
        off += d * g.in_stride[ax];
      }
      w[j] = ok ? __ldg(xb + off) : 0.f;
    }
    all_axes<A, N, A, A, BTget<Tab>>(w, xp);
#pragma unroll
    for (int j = 0; j < P; ++j) vout[j * pstride] = w[j];
  } else {
    // outer loop over the first-axis point xi_1; slabs re-read via L1
    constexpr int A1 = ipow(A, N - 1);
#pragma unroll
    for (int x1 = 0; x1 < A; ++x1) {
      float v[A1];
#pragma unroll
      for (int j = 0; j < A1; ++j) v[j] = 0.f;
#pragma unroll
      for (int i1 = 0; i1 < A; ++i1) {
        if (!BTget<Tab>::nz(xp, x1, i1)) continue;
        const float bv = BTget<Tab>::v(xp, x1, i1);
        const bool ok0 = (vmask[0] >> i1) & 1u;
#pragma unroll
        for (int j = 0; j < A1; ++j) {
          bool ok = ok0;
          int64_t off = base + i1 * g.in_stride[0];
#pragma unroll
          for (int ax = 1; ax < N; ++ax) {
            const int d = (j / ipow(A, N - 1 - ax)) % A;
            ok = ok && ((vmask[ax] >> d) & 1u);
            off += d * g.in_stride[ax];
          }
          const float dv = ok ? __ldg(xb + off) : 0.f;
          v[j] = fmaf(bv, dv, v[j]);
        }
      }
      all_axes<A, N - 1, A, A, BTget<Tab>>(v, xp);
#pragma unroll
      for (int j = 0; j < A1; ++j) vout[(x1 * A1 + j) * pstride] = v[j];
    }
  }
}

__host__ __device__ constexpr int digits_to_base(int rr, int ndig, int from, int to) {
  // reinterpret the ndig base-`from` digits of rr in base `to`
  int s = 0, q = rr, w = 1;
  for (int i = 0; i < ndig; ++i) {
    s += (q % from) * w;
    q /= from;
    w *= to;
  }
  return s;
}

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
// One thread per (c, k) pair (k fastest -> coalesced U writes): all alpha^N
// values U_xi = sum_p prod_n G[xi_n][p_n] g[k,c,p] in fp64, rounded once to
// fp32, then split for 3xTF32: hi = rna_tf32(u), lo = rna_tf32(u - hi).
__global__ void __launch_bounds__(256)
k_filter_xform(const float* __restrict__ g, float* __restrict__ Uhi, float* __restrict__ Ulo,
               float* __restrict__ U32, const __grid_constant__ FParams fp) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= (int64_t)fp.C * fp.K_s) return;
  const int k = (int)(i % fp.K_s);
  const int c = (int)(i / fp.K_s);
  const int64_t pst = (int64_t)fp.C * fp.K_s;
  int rN = 1;
  for (int n = 0; n < fp.N; ++n) rN *= fp.r;
  const float* gk = g + ((int64_t)k * fp.C + c) * rN;
  for (int64_t xi = 0; xi < fp.P; ++xi) {
    float u = 0.f;
    if (k < fp.K) {
      int xd[kMaxN];
      int64_t q = xi;
      for (int n = fp.N - 1; n >= 0; --n) { xd[n] = (int)(q % fp.a); q /= fp.a; }
      double acc = 0.0;
      for (int p = 0; p < rN; ++p) {
        double w = 1.0;
        int pq = p;
        for (int n = fp.N - 1; n >= 0; --n) { w *= fp.G[xd[n]][pq % fp.r]; pq /= fp.r; }
        if (w != 0.0) acc = fma(w, (double)gk[p], acc);
      }
      u = (float)acc;
    }
    const float hi = tf32_rna(u);
    if (Uhi) Uhi[xi * pst + i] = hi;
    if (Ulo) Ulo[xi * pst + i] = tf32_rna(u - hi);
    if (U32) U32[xi * pst + i] = u;
  }
}

// ------------------------------------------------------------------ dispatch
template <int N, int A, int M, class Tab>
static cudaError_t launch_pair(bool input, const float* src, float* dst, const KGeom& g,
                               const XfParams& xp, cudaStream_t s) {
  if (input) {
    dim3 grid((unsigned)((g.T_s + 127) / 128), (unsigned)g.C);
    k_input_xform<N, A, M, Tab><<<grid, 128, 0, s>>>(src, dst, g, xp);
  } else {
    dim3 grid((unsigned)((g.T + 127) / 128), (unsigned)g.K);
    k_output_xform<N, A, M, Tab><<<grid, 128, 0, s>>>(src, dst, g, xp);
  }
  return cudaGetLastError();
}

template <int A, int M, class Tab>
static cudaError_t launch_byN(int N, bool input, const float* src, float* dst, const KGeom& g,
                              const XfParams& xp, cudaStream_t s) {
  switch (N) {
    case 1: return launch_pair<1, A, M, Tab>(input, src, dst, g, xp, s);
    case 2: return launch_pair<2, A, M, Tab>(input, src, dst, g, xp, s);
    case 3: return launch_pair<3, A, M, Tab>(input, src, dst, g, xp, s);
    case 4:
      if constexpr (ipow(A, 3) <= 64) return launch_pair<4, A, M, Tab>(input, src, dst, g, xp, s);
      else return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
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

cudaError_t launch_xform(bool input, int N, int alpha, int m, int spec, const float* src, float* dst,
                         const KGeom& g, const XfParams& xp, cudaStream_t s) {
  if (spec == kSpecDefault) {
    if (alpha == 4 && m == 2) return launch_byN<4, 2, ConstTab<2, 3, kPsDefault>>(N, input, src, dst, g, xp, s);
    if (alpha == 6 && m == 4) return launch_byN<6, 4, ConstTab<4, 3, kPsDefault>>(N, input, src, dst, g, xp, s);
  } else if (spec == kSpecSeq) {
    if (alpha == 4 && m == 2) return launch_byN<4, 2, ConstTab<2, 3, kPsSeq>>(N, input, src, dst, g, xp, s);
    if (alpha == 6 && m == 4) return launch_byN<6, 4, ConstTab<4, 3, kPsSeq>>(N, input, src, dst, g, xp, s);
  } else {
    switch (alpha * 16 + m) {
      case 4 * 16 + 2: return launch_byN<4, 2, RunTab>(N, input, src, dst, g, xp, s);
      case 4 * 16 + 3: return launch_byN<4, 3, RunTab>(N, input, src, dst, g, xp, s);
      case 5 * 16 + 3: return launch_byN<5, 3, RunTab>(N, input, src, dst, g, xp, s);
      case 6 * 16 + 3: return launch_byN<6, 3, RunTab>(N, input, src, dst, g, xp, s);
      case 6 * 16 + 4: return launch_byN<6, 4, RunTab>(N, input, src, dst, g, xp, s);
      case 8 * 16 + 3: return launch_byN<8, 3, RunTab>(N, input, src, dst, g, xp, s);
      case 8 * 16 + 4: return launch_byN<8, 4, RunTab>(N, input, src, dst, g, xp, s);
      case 8 * 16 + 5: return launch_byN<8, 5, RunTab>(N, input, src, dst, g, xp, s);
      default: break;
    }
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_filter_xform(const float* g, float* Uhi, float* Ulo, float* U32, const FParams& fp,
                                cudaStream_t s) {
  const int64_t n = (int64_t)fp.C * fp.K_s;
  k_filter_xform<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, Uhi, Ulo, U32, fp);
  return cudaGetLastError();
}

}  // namespace wino
