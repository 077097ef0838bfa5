// xform_mixed.cu -- fused a2 / a4 instantiations for per-axis plans whose
// axis 0 has its own F(m0, r0) while the other axes share F(m, r) (NEXT-2,
// Eq. (4)'s per-axis B_n / A_n), e.g. F(2,3) along the time
// axis of a video layer with F(4,3) along space.  Default points, N = 3.
#include "xform_in.cuh"
#include "xform_out.cuh"

namespace wino {

namespace {
using T23 = ConstTab<2, 3, kPsDefault>;
using T43 = ConstTab<4, 3, kPsDefault>;
using T11 = ConstTab<1, 1, kPsDefault>;  // r = 1 along an axis: F(1,1), the identity

// (alpha0, m0) x (alpha, m) -> index of the instantiated pair, -1 if none:
// F(2,3) x F(4,3), F(4,3) x F(2,3), and the anisotropic 1 x 3 (x 3) / 3 x 1
// (x 1) kernels of (2+1)-D video layers: F(1,1) x F(4,3) | F(2,3) and
// F(4,3) | F(2,3) x F(1,1)
int pair_index(int a0, int m0, int a, int m) {
  const int k0 = a0 == 4 && m0 == 2 ? 0 : a0 == 6 && m0 == 4 ? 1 : a0 == 1 && m0 == 1 ? 2 : -1;
  const int k = a == 4 && m == 2 ? 0 : a == 6 && m == 4 ? 1 : a == 1 && m == 1 ? 2 : -1;
  if (k0 < 0 || k < 0 || k0 == k || (k0 == 2 && k == 2)) return -1;
  return k0 * 3 + k;
}
}  // namespace

bool mixed_supported(int N, int alpha0, int m0, int alpha, int m) {
  if (N != 2 && N != 3) return false;
  return pair_index(alpha0, m0, alpha, m) >= 0;
}

cudaError_t launch_input_mixed(int N, int alpha0, int m0, int alpha, int m, const float* x, float* V, const KGeom& g,
                               const XfParams& xp, const CUtensorMap* tm, int nslab, cudaStream_t s) {
  using namespace in_detail;
  const int pi = pair_index(alpha0, m0, alpha, m);
#define WINO_MIXED_IN(NN, A, M, TAB, A0, M0, TAB0) \
  return launch_in<NN, A, M, TAB, true, Ax0<A0, M0, TAB0>>(x, V, g, xp, tm, nslab, s)
  if (N == 2) {
    switch (pi) {
      case 0 * 3 + 1: WINO_MIXED_IN(2, 6, 4, T43, 4, 2, T23);
      case 1 * 3 + 0: WINO_MIXED_IN(2, 4, 2, T23, 6, 4, T43);
      case 2 * 3 + 0: WINO_MIXED_IN(2, 4, 2, T23, 1, 1, T11);
      case 2 * 3 + 1: WINO_MIXED_IN(2, 6, 4, T43, 1, 1, T11);
      case 0 * 3 + 2: WINO_MIXED_IN(2, 1, 1, T11, 4, 2, T23);
      case 1 * 3 + 2: WINO_MIXED_IN(2, 1, 1, T11, 6, 4, T43);
      default: break;
    }
  } else if (N == 3) {
    switch (pi) {
      case 0 * 3 + 1: WINO_MIXED_IN(3, 6, 4, T43, 4, 2, T23);
      case 1 * 3 + 0: WINO_MIXED_IN(3, 4, 2, T23, 6, 4, T43);
      case 2 * 3 + 0: WINO_MIXED_IN(3, 4, 2, T23, 1, 1, T11);
      case 2 * 3 + 1: WINO_MIXED_IN(3, 6, 4, T43, 1, 1, T11);
      case 0 * 3 + 2: WINO_MIXED_IN(3, 1, 1, T11, 4, 2, T23);
      case 1 * 3 + 2: WINO_MIXED_IN(3, 1, 1, T11, 6, 4, T43);
      default: break;
    }
  }
#undef WINO_MIXED_IN
  return cudaErrorNotSupported;
}

cudaError_t launch_output_mixed(int N, int alpha0, int m0, int alpha, int m, const float* Mx, float* y,
                                const KGeom& g, const XfParams& xp, const CUtensorMap* tmM, cudaStream_t s) {
  using namespace out_detail;
  const int pi = pair_index(alpha0, m0, alpha, m);
#define WINO_MIXED_OUT(NN, A, M, TAB, A0, M0, TAB0) \
  return launch_out<NN, A, M, TAB, OAx0<A0, M0, TAB0>>(Mx, y, g, xp, tmM, s)
  if (N == 2) {
    switch (pi) {
      case 0 * 3 + 1: WINO_MIXED_OUT(2, 6, 4, T43, 4, 2, T23);
      case 1 * 3 + 0: WINO_MIXED_OUT(2, 4, 2, T23, 6, 4, T43);
      case 2 * 3 + 0: WINO_MIXED_OUT(2, 4, 2, T23, 1, 1, T11);
      case 2 * 3 + 1: WINO_MIXED_OUT(2, 6, 4, T43, 1, 1, T11);
      case 0 * 3 + 2: WINO_MIXED_OUT(2, 1, 1, T11, 4, 2, T23);
      case 1 * 3 + 2: WINO_MIXED_OUT(2, 1, 1, T11, 6, 4, T43);
      default: break;
    }
  } else if (N == 3) {
    switch (pi) {
      case 0 * 3 + 1: WINO_MIXED_OUT(3, 6, 4, T43, 4, 2, T23);
      case 1 * 3 + 0: WINO_MIXED_OUT(3, 4, 2, T23, 6, 4, T43);
      case 2 * 3 + 0: WINO_MIXED_OUT(3, 4, 2, T23, 1, 1, T11);
      case 2 * 3 + 1: WINO_MIXED_OUT(3, 6, 4, T43, 1, 1, T11);
      case 0 * 3 + 2: WINO_MIXED_OUT(3, 1, 1, T11, 4, 2, T23);
      case 1 * 3 + 2: WINO_MIXED_OUT(3, 1, 1, T11, 6, 4, T43);
      default: break;
    }
  }
#undef WINO_MIXED_OUT
  return cudaErrorNotSupported;
}

}  // namespace wino
