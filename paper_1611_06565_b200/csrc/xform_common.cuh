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
  static constexpr bool kConst = Tab::kConst;
  __device__ static __forceinline__ float v(const XfParams& p, int x, int i) { return Tab::bt(p, x, i); }
  __device__ static __forceinline__ bool nz(const XfParams& p, int x, int i) {
    if constexpr (Tab::kConst) return Tab::bt(p, x, i) != 0.f; else return true;
  }
  // compile-time value (ConstTab only)
  __host__ __device__ static constexpr float cv(int x, int i) {
    if constexpr (Tab::kConst) return Tab::kTab.BT[x][i]; else return 0.f;
  }
};
template <class Tab>
struct ATget {
  static constexpr bool kConst = Tab::kConst;
  __device__ static __forceinline__ float v(const XfParams& p, int x, int i) { return Tab::at(p, x, i); }
  __device__ static __forceinline__ bool nz(const XfParams& p, int x, int i) {
    if constexpr (Tab::kConst) return Tab::at(p, x, i) != 0.f; else return true;
  }
  __host__ __device__ static constexpr float cv(int x, int i) {
    if constexpr (Tab::kConst) return Tab::kTab.AT[x][i]; else return 0.f;
  }
};

// Mirrored rows of a constant table.  Symmetric interpolation points (p, -p)
// give B^T rows in pairs related by the sign pattern (-1)^i; such a pair is
// computed from shared partial sums of the even and odd terms, e.g. F(4,3)
// with {0, +-3/2, +-2/3, inf}: 22 -> 18 operations per line.  Only the
// summation order changes (fp32 rounding, within the same tolerance; DESIGN.md
// reading #7).  (The transposed form for the mirrored columns of A^T --
// butterflies of the input pairs, 18 -> 14 operations per F(4,3) line --
// measured slower in the output transform: c4 a4 0.154 -> 0.160 ms, c2 31 ->
// 33 us; not used.)
template <class Get, int A>
__host__ __device__ constexpr int row_nnz(int x, int par) {   // par: 0 even, 1 odd, 2 all columns
  int n = 0;
  for (int i = 0; i < A; ++i)
    if ((par == 2 || (i & 1) == par) && Get::cv(x, i) != 0.f) ++n;
  return n;
}
// row y > x (< R) with cv(y, i) == (-1)^i cv(x, i), when pairing saves work; else -1
template <class Get, int A, int R>
__host__ __device__ constexpr int mirror_row(int x) {
  if (row_nnz<Get, A>(x, 0) < 1 || row_nnz<Get, A>(x, 1) < 1 || row_nnz<Get, A>(x, 2) < 3) return -1;
  for (int y = x + 1; y < R; ++y) {
    bool ok = true;
    for (int i = 0; i < A; ++i) {
      const float a = Get::cv(x, i), b = Get::cv(y, i);
      if (b != ((i & 1) ? -a : a)) ok = false;
    }
    if (ok) {
      for (int z = 0; z < x; ++z)   // y already taken by an earlier row
        if (row_nnz<Get, A>(z, 0) >= 1 && row_nnz<Get, A>(z, 1) >= 1 && row_nnz<Get, A>(z, 2) >= 3) {
          bool okz = true;
          for (int i = 0; i < A; ++i) {
            const float a = Get::cv(z, i), b = Get::cv(y, i);
            if (b != ((i & 1) ? -a : a)) okz = false;
          }
          if (okz) return -1;
        }
      return y;
    }
  }
  return -1;
}
template <class Get, int A, int R>
__host__ __device__ constexpr bool is_mirror_row(int y) {
  for (int x = 0; x < y; ++x)
    if (mirror_row<Get, A, R>(x) == y) return true;
  return false;
}
template <class Get, int A, int R>
__host__ __device__ constexpr bool has_mirror_rows() {
  for (int x = 0; x < R; ++x)
    if (mirror_row<Get, A, R>(x) >= 0) return true;
  return false;
}
// Mirrored row pairs regardless of their length (row y > x of a constant
// table with cv(y, i) == (-1)^i cv(x, i)): an a2 work item that combines the
// slab rows along axis 0 for output point x can produce y from the same row
// loads (xform_in.cuh).  -1: none, or x is itself the mirror of a row.
template <class Get, int A>
__host__ __device__ constexpr int mirror_any(int x) {
  if constexpr (!Get::kConst) {
    return -1;
  } else {
    for (int z = 0; z < x; ++z) {   // x already taken as the mirror of z
      bool ok = true;
      for (int i = 0; i < A; ++i) {
        const float a = Get::cv(z, i), b = Get::cv(x, i);
        if (b != ((i & 1) ? -a : a)) ok = false;
      }
      if (ok) return -1;
    }
    for (int y = x + 1; y < A; ++y) {
      bool ok = true, used = false;
      for (int i = 0; i < A; ++i) {
        const float a = Get::cv(x, i), b = Get::cv(y, i);
        if (b != ((i & 1) ? -a : a)) ok = false;
        if (a != 0.f) used = true;
      }
      if (ok && used) return y;
    }
    return -1;
  }
}
template <class Get, int A>
__host__ __device__ constexpr bool is_mirror_any(int y) {
  for (int x = 0; x < y; ++x)
    if (mirror_any<Get, A>(x) == y) return true;
  return false;
}
// work-item kinds along axis 0: every output point that is not the mirror of
// an earlier one (a kind with a mirror produces both points)
template <class Get, int A>
__host__ __device__ constexpr int mirror_kinds() {
  int n = 0;
  for (int x = 0; x < A; ++x)
    if (!is_mirror_any<Get, A>(x)) ++n;
  return n;
}
template <class Get, int A>
__host__ __device__ constexpr int kind_point(int k) {
  for (int x = 0; x < A; ++x)
    if (!is_mirror_any<Get, A>(x) && k-- == 0) return x;
  return -1;
}

// One line: out[x] = sum_i Get(x, i) in[i] for x < R (in and out may not
// alias).  Constant tables with mirrored rows take the shared partial sums;
// otherwise one FMA chain per output, zero terms skipped.
template <int A, int R, class Get>
__device__ __forceinline__ void xform_line(const float* in, float* out, const XfParams& p) {
  if constexpr (Get::kConst && has_mirror_rows<Get, A, R>()) {
    sfor<0, R>([&](auto X) {
      constexpr int x = decltype(X)::value;
      if constexpr (!is_mirror_row<Get, A, R>(x)) {
        constexpr int y = mirror_row<Get, A, R>(x);
        float e = 0.f, o = 0.f, acc = 0.f;
        bool fe = true, fo = true, fa = true;
        sfor<0, A>([&](auto I) {
          constexpr int i = decltype(I)::value;
          constexpr float c = Get::cv(x, i);
          if constexpr (c != 0.f) {
            if constexpr (y < 0) {
              acc = fa ? c * in[i] : fmaf(c, in[i], acc);
              fa = false;
            } else if constexpr (i & 1) {
              o = fo ? c * in[i] : fmaf(c, in[i], o);
              fo = false;
            } else {
              e = fe ? c * in[i] : fmaf(c, in[i], e);
              fe = false;
            }
          }
        });
        if constexpr (y >= 0) {
          out[x] = e + o;
          out[y] = e - o;
        } else {
          out[x] = acc;
        }
      }
    });
  } else {
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
      out[x] = acc;
    }
  }
}

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
      float in[A], out[R];
#pragma unroll
      for (int i = 0; i < A; ++i) in[i] = v[base + i * stride];
      xform_line<A, R, Get>(in, out, p);
#pragma unroll
      for (int x = 0; x < R; ++x) v[base + x * stride] = out[x];
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
