// xform_dfold.cu -- stage a2 of the direct-axis fold (a5; DESIGN.md reading
// #21): the input transform of the N - 1 outer axes only.
//
// For the innermost axis the layer's F(m, r) is folded into the GEMM from
// both sides: with Z the input transformed along axes 0 .. N-2 and left raw
// along the last axis,
//   W[xo][o][k][t] = sum_q A^T[o][q] sum_c V_{xo,q}[c][t] U_{xo,q}[c][k]          (Eq. (4)-(5))
//                  = sum_{j,c} Z_{xo}[c][t_outer][m t_last + j] *
//                    ( sum_q A^T[o][q] B^T[q][j] U_{xo,q}[c][k] )
// and the bracket is the outer-axes filter transform at tap j - o of the last
// axis (the F(m, r) identity), zero unless 0 <= j - o < r.
// Z is 1/alpha of V per input column instead of alpha/m per tile: half of V
// for F(2,3), written once and read once (PAPER.md:180 places the inverse
// transform over the reduced output; PAPER.md:236-243 the intensity argument
// for keeping the per-point products matrix-shaped).
//
// Layout: Z[(xo * 2 + par)][c][slot], slot = row * 32 + i, row = (b, t_0 ..
// t_{N-2}) row-major, column xp = 2 i + par of the zero-padded input row (xp
// = input column + pad), i <= tiles_last (<= 31; slots past that stay zero
// from the plan's workspace memset).  Tap j of tile t_last reads plane par =
// j & 1 at slot t_last + (j >> 1): the GEMM's A operand is a contiguous run
// of slots per tap.
//
// The a2 kernel is the fused input transform's slab kernel in its dfold mode
// (xform_in.cuh, g.dfold): the same TMA slab staging, one warp item per
// (t_0, t_1) row of tiles.  (Two register-only versions that read x straight
// from global memory -- one warp per row of tiles, and a sliding axis-1 window
// -- measured 0.46 / 0.52 ms on c3 against 0.32 ms for the V path: under the
// layer's write traffic a DRAM read takes ~5 us, which only the slab's single
// up-front bulk load hides; an L2 bulk prefetch did not help.)
#include "kernels.h"

namespace wino {
// F(2,3) with the default points, N = 3, at most 31 tiles along the last axis.
bool input_dfold_supported(int N, int alpha, int m, int spec, int tiles_last) {
  return N == 3 && alpha == 4 && m == 2 && spec == kSpecDefault && tiles_last >= 1 && tiles_last <= 31;
}

}  // namespace wino
