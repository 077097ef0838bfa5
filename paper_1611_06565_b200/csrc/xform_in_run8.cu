// xform_in_run8.cu -- a2 instantiations with run-time transform tables,
// alpha in {6, 8} (split from xform_in_run.cu for parallel compilation).
#include "xform_in.cuh"

namespace wino {

cudaError_t launch_input_run45(int N, int alpha, int m, const float* x, float* V, const KGeom& g, const XfParams& xp,
                               const CUtensorMap* tm, int nslab, cudaStream_t s);

cudaError_t launch_input_run(int N, int alpha, int m, const float* x, float* V, const KGeom& g, const XfParams& xp,
                             const CUtensorMap* tm, int nslab, cudaStream_t s) {
  using namespace in_detail;
  switch (alpha * 16 + m) {
    // TMA slabs measured faster for alpha = 8 (Figure 4's F(5,4): a2 1.34 ->
    // 1.11 ms) but slower for F(3,4) (1.37 -> 1.75 ms): alpha 6 stays on cp.async
    case 6 * 16 + 3: return launch_in_byN<6, 3, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 6 * 16 + 4: return launch_in_byN<6, 4, RunTab, false>(N, x, V, g, xp, nullptr, nslab, s);
    case 8 * 16 + 3: return launch_in_byN<8, 3, RunTab, true>(N, x, V, g, xp, tm, nslab, s);
    case 8 * 16 + 4: return launch_in_byN<8, 4, RunTab, true>(N, x, V, g, xp, tm, nslab, s);
    case 8 * 16 + 5: return launch_in_byN<8, 5, RunTab, true>(N, x, V, g, xp, tm, nslab, s);
    default: return launch_input_run45(N, alpha, m, x, V, g, xp, tm, nslab, s);
  }
}

}  // namespace wino
