// xform_out_run.cu -- a4 instantiations with run-time transform tables.
#include "xform_out.cuh"

namespace wino {

cudaError_t launch_output_run(int N, int alpha, int m, const float* Mx, float* y, const KGeom& g,
                              const XfParams& xp, const CUtensorMap* tmM, cudaStream_t s) {
  using namespace out_detail;
  switch (alpha * 16 + m) {
    case 4 * 16 + 2: return launch_out_byN<4, 2, RunTab>(N, Mx, y, g, xp, tmM, s);
    case 4 * 16 + 3: return launch_out_byN<4, 3, RunTab>(N, Mx, y, g, xp, tmM, s);
    case 5 * 16 + 3: return launch_out_byN<5, 3, RunTab>(N, Mx, y, g, xp, tmM, s);
    case 6 * 16 + 3: return launch_out_byN<6, 3, RunTab>(N, Mx, y, g, xp, tmM, s);
    case 6 * 16 + 4: return launch_out_byN<6, 4, RunTab>(N, Mx, y, g, xp, tmM, s);
    case 8 * 16 + 3: return launch_out_byN<8, 3, RunTab>(N, Mx, y, g, xp, tmM, s);
    case 8 * 16 + 4: return launch_out_byN<8, 4, RunTab>(N, Mx, y, g, xp, tmM, s);
    case 8 * 16 + 5: return launch_out_byN<8, 5, RunTab>(N, Mx, y, g, xp, tmM, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace wino
