// xform_out_const.cu -- a4 instantiations for the compile-time point sets.
#include "xform_out.cuh"

namespace wino {

cudaError_t launch_output_const(int N, int alpha, int m, int spec, const float* Mx, float* y, const KGeom& g,
                                const XfParams& xp, const CUtensorMap* tmM, cudaStream_t s) {
  using namespace out_detail;
  if (spec == kSpecDefault) {
    if (alpha == 4 && m == 2) return launch_out_byN<4, 2, ConstTab<2, 3, kPsDefault>>(N, Mx, y, g, xp, tmM, s);
    if (alpha == 6 && m == 4) return launch_out_byN<6, 4, ConstTab<4, 3, kPsDefault>>(N, Mx, y, g, xp, tmM, s);
  } else if (spec == kSpecSeq) {
    if (alpha == 4 && m == 2) return launch_out_byN<4, 2, ConstTab<2, 3, kPsSeq>>(N, Mx, y, g, xp, tmM, s);
    if (alpha == 6 && m == 4) return launch_out_byN<6, 4, ConstTab<4, 3, kPsSeq>>(N, Mx, y, g, xp, tmM, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace wino
