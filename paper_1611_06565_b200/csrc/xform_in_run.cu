// xform_in_run.cu -- a2 instantiations with run-time transform tables (any
// interpolation points; alpha in {4, 5, 6, 8}); cp.async slab loads.
#include "xform_in.cuh"

namespace wino {

cudaError_t launch_input_run(int N, int alpha, int m, const float* x, float* V, const KGeom& g, const XfParams& xp,
                             int nslab, cudaStream_t s) {
  using namespace in_detail;
  switch (alpha * 16 + m) {
    case 4 * 16 + 2: return launch_in_byN<4, 2, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 4 * 16 + 3: return launch_in_byN<4, 3, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 5 * 16 + 3: return launch_in_byN<5, 3, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 6 * 16 + 3: return launch_in_byN<6, 3, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 6 * 16 + 4: return launch_in_byN<6, 4, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 8 * 16 + 3: return launch_in_byN<8, 3, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 8 * 16 + 4: return launch_in_byN<8, 4, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 8 * 16 + 5: return launch_in_byN<8, 5, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace wino
