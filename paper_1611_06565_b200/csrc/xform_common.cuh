// xform_common.cuh -- register-level separable line transforms shared by
// the input (a2) and output (a4) transform kernels.
//
// Every transform is a chain of n-mode products (Eq. (3))
// applied separably per axis (Eq. (4)).  The matrices are
// tiny (alpha <= 8): per line the work is done in registers with
// compile-time-unrolled loops; with ConstTab tables the zero entries vanish
// at compile time and +-1 entries become adds ("U is sparse ... traversed in
// the outermost loops"; "exploiting the sparsity of the
// matrices themselves").
#pragma once
#include "common.cuh"

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

}  // namespace wino
