// kernels.h -- internal launchers (host side) of the device stages.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace wino {

enum { kSpecRuntime = 0, kSpecDefault = 1, kSpecSeq = 2 };

bool xform_supported(int N, int alpha, int m, int spec);
// alpha0 / m0: axis 0's F(m0, r0) (= alpha / m except in per-axis plans)
bool plan_input_slab(KGeom& g, int N, int alpha0, int m0, int alpha, int m, bool tma);
void plan_input_planes(KGeom& g, int64_t nwork, int num_sms);
// a2: x [B][C][in...] -> V [P][C][T_s], input slabs [g.s_beg, g.s_beg + nslab)
// (slab = b * nbox0 + box; V row = t - g.t0)
// tm: TMA map of x from encode_input_map (NULL = cp.async fallback path)
bool encode_input_map(CUtensorMap* tm, const float* x, const KGeom& g, int N, int B);
cudaError_t launch_input_xform(int N, int alpha, int m, int spec, const float* x, float* V, const KGeom& g,
                               const XfParams& xp, const CUtensorMap* tm, int nslab, cudaStream_t s);
// a4: M [P][K][T_s] -> y [B][K][out...] for tiles [g.t_beg, g.T) (M row = t - g.t0)
// tmM: TMA map of M from encode_output_map (NULL = plain per-thread loads)
bool encode_output_map(CUtensorMap* tm, const float* Mx, int64_t T_s, int K, int64_t P, int A1);
cudaError_t launch_output_xform(int N, int alpha, int m, int spec, const float* Mx, float* y, const KGeom& g,
                                const XfParams& xp, const CUtensorMap* tmM, cudaStream_t s);
// per-axis (m_n, r_n) plans (xform_nd.cu): multi-pass a2 / a4 over tiles [t_lo, t_hi)
cudaError_t launch_input_nd(const float* x, float* V, const KGeom& g, const NdParams& q, int N, int64_t P,
                            int64_t t_lo, int64_t t_hi, cudaStream_t s);
cudaError_t launch_output_nd(const float* Mx, float* W, float* y, const KGeom& g, const NdParams& q, int N,
                             int64_t t_lo, int64_t t_hi, cudaStream_t s);
// per-axis plans with a distinct axis 0 and fused kernels (xform_mixed.cu)
bool mixed_supported(int N, int alpha0, int m0, int alpha, int m);
cudaError_t launch_input_mixed(int N, int alpha0, int m0, int alpha, int m, const float* x, float* V, const KGeom& g,
                               const XfParams& xp, const CUtensorMap* tm, int nslab, cudaStream_t s);
cudaError_t launch_output_mixed(int N, int alpha0, int m0, int alpha, int m, const float* Mx, float* y,
                                const KGeom& g, const XfParams& xp, const CUtensorMap* tmM, cudaStream_t s);
// tiny layers: a2 + a3 + a4 in one kernel (xform_tiny.cu)
bool tiny_shape(int N, int a, int C, int K, int64_t P, int* TB, int* smem);
bool tiny_supported(int N, int a, int m);
cudaError_t launch_tiny(const float* x, const float* Uhi, const float* Ulo, float* y, const KGeom& g,
                        const XfParams& xp, int N, int a, int m, int spec, int P, int K_s, int64_t T, cudaStream_t s);
cudaError_t launch_filter_xform(const float* g, float* Uhi, float* Ulo, float* U32, const FParams& fp,
                                cudaStream_t s);

// a3, CUDA-core fp32 FMA: Mo[xi][k][t] = sum_c V[xi][c][t] U[xi][c][k]
cudaError_t launch_gemm_ffma(const float* V, const float* U32, float* Mo, int P, int64_t T, int64_t T_s,
                             int C, int K, int K_s, cudaStream_t s);

// a3 on tcgen05 tensor cores.
// GEMM variants (all compute the same products in the same order per output
// row -> bit-identical results; the plan times the supported ones once and
// keeps the fastest, see tc_gemm_tune).
enum { kGemmSS = 0, kGemmTS = 1, kGemmPair = 2 };
struct TcGemm {
  CUtensorMap tmA;    // V   [P][C][T_s]   (t, c, xi): 32 x kc boxes, 128B swizzle (SS mode)
  CUtensorMap tmA_ts; // V   128 x kc boxes, no swizzle (TS / pair modes: raw V ring)
  CUtensorMap tmBhi;  // U_hi [P][C][K_s]
  CUtensorMap tmBlo;  // U_lo
  int bn;             // N tile (32, 64, 128, 256)
  int bn_max;         // widest N tile for K (pick_bn)
  int kc;             // channels per pipeline stage (multiple of 8, <= 32)
  int three;          // 1: 3xTF32, 0: 1xTF32
  int num_sms;
  bool resident;      // U block kept in shared memory (SS / TS modes)
  int variant;        // kGemmSS, kGemmTS or kGemmPair
  bool can_ts, can_pair;
  int dbg;            // dev-only experiment knob (WINO_GEMM_DBG), 0 in production
  bool ready;
};
cudaError_t tc_gemm_prepare(TcGemm& tg, const float* V, const float* Uhi, const float* Ulo, int P,
                            int64_t T_s, int C, int K_s, int K, int three, int device);
// Time every supported variant on the plan's workspace (rows [0, T)) and keep
// the fastest; WINO_GEMM_VARIANT=0/1/2 forces one.  The timing launches run
// on a private non-blocking stream, which is synchronised (not the device);
// results are cached per (device, shape), so re-planning launches nothing.
// Vw: the plan's V buffer, rewritten (zeros) before each timed launch (NULL = no)
cudaError_t tc_gemm_tune(TcGemm& tg, float* Mo, int P, int64_t T, int64_t T_s, int C, int K, float* Vw);
bool ts2_supported(int bn, int kc);
int gemm_nbfast();   // unit order of the CTA-pair GEMMs (n-block fastest: 1)
cudaError_t launch_gemm_ts2(const TcGemm& tg, float* Mo, int P, int64_t t_lo, int64_t T, int64_t T_s, int C, int K,
                            cudaStream_t s);
// a3 with the 3xFP16 scaled split on kind::f16 (gemm_f16.cu), CTA pairs, BN 128
bool f16_supported(int K, int kc);
cudaError_t f16_encode_u(CUtensorMap* tm, const void* base, int64_t K_s, int C, int P, int kc);
// vres: the V-resident kernel k_gemm_f16n where it applies (f16n_applies:
// 128 < K <= 256, C <= 256); it honours zmask (bit nb*8 + c: U chunk
// (n-block nb, k-chunk c) is zero and skipped).  Same products, same order
// per output as k_gemm_f16p: bit-identical results.
bool f16n_applies(int C, int K, int kc);
// df (direct-axis fold, xform_dfold.cu; V-resident kernel only): the A operand
// is Z [P*2][cz][Tz] -- k-chunk (tap j, channels c0..) of unit (xo, 256-slot
// block) is the box of plane xo*2 + (j & 1) at slot + (j >> 1) (loaded from
// the 16-byte aligned slot, the shift applied by the converter); T counts
// slots (rows * S) and the epilogue stores slot (row, i < tl2) at tile
// row * tl2 + i of W.
constexpr int kDfoldSlots = 32;   // full 128-byte lines per row (packed rows of tl2 + 1 slots measured slower)
struct DFoldGemm {
  const CUtensorMap* tmA;   // Z as (slot, c, plane), box {132, kc, 1}, no swizzle (f16_encode_z)
  int tl2;                  // tiles along the last axis (<= 31)
  int S;                    // slots per row of tiles (kDfoldSlots)
  int cz;                   // layer channels C (a multiple of the k-chunk)
};
cudaError_t f16_encode_z(CUtensorMap* tm, const float* Z, int64_t Tz, int cz, int planes, int kc);
cudaError_t launch_gemm_f16(const TcGemm& tg, const CUtensorMap& tmBhi16, const CUtensorMap& tmBlo16, float* Mo,
                            int P, int64_t t_lo, int64_t T, int64_t T_s, int C, int K, const unsigned int* vmax,
                            const float* uscal, cudaStream_t s, int zmask = 0, bool vres = true,
                            const DFoldGemm* df = nullptr);
// U (fp32) -> scaled fp16 hi / lo halves; *uscal = 2^su (mx: scratch word)
cudaError_t launch_split16(const float* u32, int64_t n, unsigned int* mx, void* hi, void* lo, float* uscal,
                           cudaStream_t s);

// a3 with the output transform of the F innermost axes folded into the
// epilogue (gemm_fold.cu): W[xo][o][k][t] = sum_q prod_f A^T[o_f][q_f] D_{xo*Q+q}
// (Q = alpha^F points q, MO = m^F outputs o), W [P/Q * MO][K][T_s].
constexpr int kMaxFoldQ = 64, kMaxFoldMO = 4;
struct FoldTab {
  float coef[kMaxFoldQ][kMaxFoldMO];   // coef[q][o], fp32 RNE of the exact product
};
bool fold_shape(int K, int MO, int kc, int* bn, int* g);
bool fold_feasible(int bn, int kc, int C, int Q);   // the folded GEMM's pipeline fits TMEM / shared memory
cudaError_t launch_gemm_fold(const TcGemm& tg, int bn, int g, int MO, float* W, int P, int Q, int64_t t_lo,
                             int64_t T, int64_t T_s, int C, int K, const FoldTab& fold, cudaStream_t s);
// a4 after the folded GEMM: A^T along axes 0 .. N-F-1 of W (xform_fold.cu)
bool output_fold_supported(int N, int alpha, int m, int F, int spec);
cudaError_t launch_output_fold(int N, int alpha, int m, int F, int spec, const float* W, float* y, const KGeom& g,
                               const XfParams& xp, cudaStream_t s);
// a5, filter-side fold: the same W from a plain batched GEMM.  By linearity
//   W[xo][o][k][t] = sum_q A^T_F[o][q] sum_c V_{xo*Q+q}[c][t] U_{xo*Q+q}[c][k]
//                  = sum_{(q,c)} V'[xo][(q,c)][t] U'[xo][(q,c)][(o,k)],
//   U'[xo][(q,c)][(o,k)] = A^T_F[o][q] U_{xo*Q+q}[c][k],
// where V' is V itself viewed as [P/Q][Q*C][T_s]: W = V' U' is one GEMM per
// outer point xo with a Q*C-deep reduction and MO*K columns, written in W's
// layout [P/Q][MO*K][T_s].  U' is computed by the filter transform (fp64,
// one rounding), so A^T_F costs nothing per forward; the GEMM does MO x the
// multiply-adds of the unfused one (the fold's zero coefficients included).
constexpr int kMaxUFoldQ = 64, kMaxUFoldMO = 8;
struct UFoldTab {
  double coef[kMaxUFoldQ][kMaxUFoldMO];   // exact product of A^T entries, RNE to fp64
  int Q, MO;
  // direct-axis fold (F = 1, xform_dfold.cu): row (q, c) is tap j = q of the
  // raw last axis, U'[xo][(j,c)][(o,k)] = (g x_outer G)[xo][c][k][j - o]
  // (coef[j][o] = 1 for 0 <= j - o < r, else 0): the last axis takes the
  // filter tap itself instead of G
  int direct;
};
// a2 of the direct-axis fold: x -> Z [P/alpha * 2][C][Tz] by launch_input_xform
// with g.dfold set (xform_in.cuh); the shapes it takes (xform_dfold.cu)
bool input_dfold_supported(int N, int alpha, int m, int spec, int tiles_last);
// U' [P/Q][Q*C][K_s'] (K_s' >= MO*K, = fp.K_s) from g; fp.P / fp.C / fp.K are the layer's
cudaError_t launch_filter_ufold(const float* g, float* Uhi, float* Ulo, float* U32, const FParams& fp,
                                const UFoldTab& uf, cudaStream_t s);
// rows [t_lo, T) of every point (t_lo a multiple of 4)
cudaError_t launch_gemm_tc(const TcGemm& tg, float* Mo, int P, int64_t t_lo, int64_t T, int64_t T_s, int C, int K,
                           cudaStream_t s);

}  // namespace wino
