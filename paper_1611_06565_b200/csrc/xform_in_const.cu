// xform_in_const.cu -- a2 instantiations for the compile-time (default and
// SPEC-order) point sets: zero/one entries of B^T folded, TMA slab loads.
#include "xform_in.cuh"

namespace wino {

cudaError_t launch_input_const(int N, int alpha, int m, int spec, const float* x, float* V, const KGeom& g,
                               const XfParams& xp, const CUtensorMap* tm, int nslab, cudaStream_t s) {
  using namespace in_detail;
  if (spec == kSpecDefault) {
    if (alpha == 4 && m == 2) return launch_in_byN<4, 2, ConstTab<2, 3, kPsDefault>, true>(N, x, V, g, xp, tm, nslab, s);
    if (alpha == 6 && m == 4) return launch_in_byN<6, 4, ConstTab<4, 3, kPsDefault>, true>(N, x, V, g, xp, tm, nslab, s);
  } else if (spec == kSpecSeq) {
    if (alpha == 4 && m == 2) return launch_in_byN<4, 2, ConstTab<2, 3, kPsSeq>, true>(N, x, V, g, xp, tm, nslab, s);
    if (alpha == 6 && m == 4) return launch_in_byN<6, 4, ConstTab<4, 3, kPsSeq>, true>(N, x, V, g, xp, tm, nslab, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace wino
