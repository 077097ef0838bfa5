// xform_in_run.cu -- a2 instantiations with run-time transform tables (any
// interpolation points), alpha in {4, 5}: cp.async slab loads.  alpha in
// {6, 8}: xform_in_run8.cu (alpha = 8 with TMA slabs where the shape allows).
#include "xform_in.cuh"

namespace wino {

cudaError_t launch_input_run45(int N, int alpha, int m, const float* x, float* V, const KGeom& g, const XfParams& xp,
                               const CUtensorMap* tm, int nslab, cudaStream_t s) {
  using namespace in_detail;
  switch (alpha * 16 + m) {
    case 4 * 16 + 2: return launch_in_byN<4, 2, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 4 * 16 + 3: return launch_in_byN<4, 3, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 5 * 16 + 3: return launch_in_byN<5, 3, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace wino
