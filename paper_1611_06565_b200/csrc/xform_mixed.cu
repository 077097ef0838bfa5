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
}  // namespace

bool mixed_supported(int N, int alpha0, int m0, int alpha, int m) {
  if (N != 2 && N != 3) return false;
  return (alpha0 == 4 && m0 == 2 && alpha == 6 && m == 4) || (alpha0 == 6 && m0 == 4 && alpha == 4 && m == 2);
}

cudaError_t launch_input_mixed(int N, int alpha0, int m0, int alpha, int m, const float* x, float* V, const KGeom& g,
                               const XfParams& xp, const CUtensorMap* tm, int nslab, cudaStream_t s) {
  using namespace in_detail;
  if (N == 2 && alpha0 == 4 && m0 == 2 && alpha == 6 && m == 4)
    return launch_in<2, 6, 4, T43, true, Ax0<4, 2, T23>>(x, V, g, xp, tm, nslab, s);
  if (N == 2 && alpha0 == 6 && m0 == 4 && alpha == 4 && m == 2)
    return launch_in<2, 4, 2, T23, true, Ax0<6, 4, T43>>(x, V, g, xp, tm, nslab, s);
  if (N == 3 && alpha0 == 4 && m0 == 2 && alpha == 6 && m == 4)
    return launch_in<3, 6, 4, T43, true, Ax0<4, 2, T23>>(x, V, g, xp, tm, nslab, s);
  if (N == 3 && alpha0 == 6 && m0 == 4 && alpha == 4 && m == 2)
    return launch_in<3, 4, 2, T23, true, Ax0<6, 4, T43>>(x, V, g, xp, tm, nslab, s);
  return cudaErrorNotSupported;
}

cudaError_t launch_output_mixed(int N, int alpha0, int m0, int alpha, int m, const float* Mx, float* y,
                                const KGeom& g, const XfParams& xp, const CUtensorMap* tmM, cudaStream_t s) {
  using namespace out_detail;
  if (N == 2 && alpha0 == 4 && m0 == 2 && alpha == 6 && m == 4)
    return launch_out<2, 6, 4, T43, OAx0<4, 2, T23>>(Mx, y, g, xp, tmM, s);
  if (N == 2 && alpha0 == 6 && m0 == 4 && alpha == 4 && m == 2)
    return launch_out<2, 4, 2, T23, OAx0<6, 4, T43>>(Mx, y, g, xp, tmM, s);
  if (N == 3 && alpha0 == 4 && m0 == 2 && alpha == 6 && m == 4)
    return launch_out<3, 6, 4, T43, OAx0<4, 2, T23>>(Mx, y, g, xp, tmM, s);
  if (N == 3 && alpha0 == 6 && m0 == 4 && alpha == 4 && m == 2)
    return launch_out<3, 4, 2, T23, OAx0<6, 4, T43>>(Mx, y, g, xp, tmM, s);
  return cudaErrorNotSupported;
}

}  // namespace wino
