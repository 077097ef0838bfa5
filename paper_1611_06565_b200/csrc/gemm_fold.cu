// gemm_fold.cu -- stage a3 with the output transform of the F innermost axes
// folded into the GEMM epilogue ("epilogue: a4 applied to
// D_xi from TMEM"; "the inverse transform can be applied once
// over the reduced output").
//
// Transform points xi are row-major over (xi_0 .. xi_{N-1}); split
// xi = xo * Q + q with q the last F digits (Q = alpha^F).  For a tile t and
// output channel k the unfused pipeline writes M_xi[k][t] for all alpha^N
// points and a4 reduces them with A^T along every axis.  Here a work unit
// (xo, n-block, m-block) runs the Q GEMMs  D_q = V_{xo,q} U_{xo,q}  (3xTF32,
// TMEM accumulators, as k_gemm_ts) one after another, and the epilogue folds
// each D_q into m^F register accumulators per (t, k):
//
//     W[xo][o][k][t] = sum_q  A^T_F[o][q] D_q[t][k],
//     A^T_F[o][q] = prod_f A^T[o_f][q_f]           (o < MO = m^F),
//
// i.e. the n-mode products x_n A^T of the last F axes (Eq. (4)) applied to
// the accumulator before it leaves the SM.  W has (m/alpha)^F of M's size:
// the GEMM writes and a4 reads that much less (c3 F(2^3,3^3): 1/2 at F = 1,
// 1/4 at F = 2).  a4 then applies A^T along the remaining N - F axes
// (k_output_fold, xform_fold.cu).
//
// Warps: 0-7 converter (raw V -> V_hi / V_lo in TMEM, as k_gemm_ts),
// 8 .. 8+4G-1 epilogue (lane quarter w % 4, column group (w - 8) / 4: each
// thread holds one tile row t and BN/G output channels, MO x BN/G fp32
// accumulators), then the V producer, the MMA issuer and the U producer.
#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "tc_common.cuh"
#include "tma.hpp"

namespace wino {
namespace tc {

// NCV converter warps (4 or 8), 4G epilogue warps, 3 single-thread roles
template <int G, int NCV>
constexpr int fold_threads() { return 32 * (NCV + 4 * G + 3); }
constexpr int kMaxAcc = 8;      // TMEM accumulator stages
constexpr int kMaxAStage = 8;   // TMEM A (V_hi | V_lo) stages

// tcgen05.ld of CW (16 or 32) consecutive columns of this warp's 32 lanes, then wait.
template <int CW>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[CW]) {
  if constexpr (CW == 32) {
    tmem_ld32(taddr, r);
  } else {
    static_assert(CW == 16, "CW must be 16 or 32");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }
}

template <int BN, int G, int MO, int KC, int NCV>
__global__ void __launch_bounds__(fold_threads<G, NCV>(), 1)
k_gemm_fold(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
            const __grid_constant__ CUtensorMap tmBlo, float* __restrict__ W, int P, int Q, int R, int t_lo, int T,
            long long T_s, int C, int K, int nraw, int nbr, int na, int nacc, int l2hint, int dbg,
            unsigned long long* __restrict__ trace, const __grid_constant__ FoldTab fold) {
  // dev probe: clock64 timestamps of CTA 0's pipeline events (trace != NULL)
#define FTR(role, ev, idx)                                                                   \
  do {                                                                                       \
    if (trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (idx) < 256)                  \
      trace[((role) * 4 + (ev)) * 256 + (idx)] = clock64();                                  \
  } while (0)
  constexpr int CW = BN / G;                 // output channels per epilogue thread
  static_assert(CW % 16 == 0, "column group must be a multiple of 16");
  constexpr int kEpi0 = NCV, kProdV = NCV + 4 * G, kMma = kProdV + 1, kProdU = kProdV + 2;
  constexpr int NK = KC / 8;                 // K=8 MMA steps per chunk
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (sraw & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  const uint32_t sbase = sraw + pad;
  const int n_chunks = (C + KC - 1) / KC;
  const int S = R * n_chunks;                // chunks per group (R points' full C reduction)
  const uint32_t a_bytes = (uint32_t)BM * KC * 4;
  const uint32_t b_bytes = (uint32_t)BN * KC * 4;
  const uint32_t raw0 = sbase;
  const uint32_t bres = raw0 + nraw * a_bytes;          // U ring: nbr group stages of S (U_hi | U_lo) pairs
  const uint32_t bar0 = bres + 2u * S * nbr * b_bytes;
  auto rfull = [&](int s) { return bar0 + 8u * s; };
  auto rempty = [&](int s) { return bar0 + 8u * (nraw + s); };
  auto ufull = [&](int s) { return bar0 + 8u * (2 * nraw + s); };
  auto uempty = [&](int s) { return bar0 + 8u * (2 * nraw + nbr + s); };
  const uint32_t bar1 = bar0 + 8u * (2 * nraw + 2 * nbr);
  auto tfull = [&](int a) { return bar1 + 8u * a; };          // a < kMaxAcc (accumulator groups)
  auto tempty = [&](int a) { return bar1 + 8u * (kMaxAcc + a); };
  auto afull = [&](int a) { return bar1 + 8u * (2 * kMaxAcc + a); };   // a < kMaxAStage
  auto aempty = [&](int a) { return bar1 + 8u * (2 * kMaxAcc + kMaxAStage + a); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + (bar1 - sbase) + 8 * (2 * kMaxAcc + 2 * kMaxAStage));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // TMEM: nacc accumulator groups of R D's (R * BN columns each) + na A
  // stages of S chunks (V_hi | V_lo, 2 KC columns per chunk)
  const uint32_t a_col0 = (uint32_t)(nacc * R * BN);
  const uint32_t kCols = pow2_cols(nacc * R * BN + na * S * 2 * KC);

  if (warp == kMma) {
    if (lane == 0) {
      for (int s = 0; s < nraw; ++s) {
        mbar_init(rfull(s), 1);
        mbar_init(rempty(s), 32 * NCV);
      }
      for (int s = 0; s < nbr; ++s) {
        mbar_init(ufull(s), 1);
        mbar_init(uempty(s), 1);
      }
      for (int a = 0; a < nacc; ++a) {
        mbar_init(tfull(a), 1);
        mbar_init(tempty(a), 128 * G);
      }
      for (int a = 0; a < na; ++a) {
        mbar_init(afull(a), 32 * NCV);
        mbar_init(aempty(a), 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();      // V comes from the input transform; W (= M buffer) is read by the previous output transform
  pdl_trigger();

  const int n_mblk = (T - t_lo + BM - 1) / BM;
  const int n_nblk = (K + BN - 1) / BN;
  const long long per_xo = (long long)n_nblk * n_mblk;
  const long long total = (long long)(P / Q) * per_xo;
  const int ngrp = Q / R;                    // groups per unit
  // grid-strided units u -> (xo, m-block, n-block), n-block fastest: CTAs
  // running side by side share the V block of one m-block (its L2 copy
  // serves every n-block)
  auto decode = [&](long long u, int& xo, int& mb, int& nb) {
    xo = (int)(u / per_xo);
    const int rr = (int)(u - (long long)xo * per_xo);
    mb = rr / n_nblk;
    nb = rr - mb * n_nblk;
  };

  if (warp == kProdV) {
    if (lane == 0) {  // ---------------- V producer (raw ring, one box per chunk)
      int s = 0, vci = 0;
      uint32_t ph = 0;
      for (long long u = blockIdx.x; u < total; u += gridDim.x) {
        int xo, mb, nb;
        decode(u, xo, mb, nb);
        for (int q = 0; q < Q; ++q) {
          const int xi = xo * Q + q;
          for (int ch = 0; ch < n_chunks; ++ch) {
            mbar_wait(rempty(s), ph ^ 1u);
            FTR(0, 0, vci);
            ++vci;
            if (dbg & 8) {               // dev probe: no V loads
              mbar_arrive(rfull(s));
            } else {
              mbar_expect_tx(rfull(s), a_bytes);
              if (l2hint)
                tma_load_3d_hint(raw0 + s * a_bytes, &tmA, t_lo + mb * BM, ch * KC, xi, rfull(s), l2_policy(false));
              else
                tma_load_3d(raw0 + s * a_bytes, &tmA, t_lo + mb * BM, ch * KC, xi, rfull(s));
            }
            if (++s == nraw) { s = 0; ph ^= 1u; }
          }
        }
      }
    }
  } else if (warp == kProdU) {
    if (lane == 0) {  // ---------------- U producer: one ring stage per group (S chunk pairs)
      int s = 0, uci = 0;
      uint32_t ph = 0;
      for (long long u = blockIdx.x; u < total; u += gridDim.x) {
        int xo, mb, nb;
        decode(u, xo, mb, nb);
        for (int gi = 0; gi < ngrp; ++gi) {
          mbar_wait(uempty(s), ph ^ 1u);
          FTR(4, 0, uci);
          ++uci;
          const uint32_t st = bres + s * S * 2 * b_bytes;
          mbar_expect_tx(ufull(s), 2u * S * b_bytes);
          for (int r = 0; r < R; ++r) {
            const int xi = xo * Q + gi * R + r;
            for (int ch = 0; ch < n_chunks; ++ch) {
              const uint32_t sc = st + (r * n_chunks + ch) * 2 * b_bytes;
#pragma unroll
              for (int gq = 0; gq < BN / 32; ++gq) {
                tma_load_3d(sc + gq * KC * 128, &tmBhi, nb * BN + gq * 32, ch * KC, xi, ufull(s));
                tma_load_3d(sc + b_bytes + gq * KC * 128, &tmBlo, nb * BN + gq * 32, ch * KC, xi, ufull(s));
              }
            }
          }
          if (++s == nbr) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == kMma) {
    // ---------------- MMA issuer: one group (R D's, S chunks) per handshake
    constexpr uint32_t idesc = idesc_tf32_ts<BN>();
    constexpr uint32_t lbo = (uint32_t)KC * 128u;
    int as = 0, us = 0, mci = 0;
    uint32_t aph = 0, uph = 0, acc = 0, cph = 0;
    for (long long u = blockIdx.x; u < total; u += gridDim.x) {
      for (int gi = 0; gi < ngrp; ++gi) {
        mbar_wait(tempty(acc), cph ^ 1u);
        mbar_wait(afull(as), aph);
        mbar_wait(ufull(us), uph);
        FTR(2, 0, mci);
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * R * BN;
        const uint32_t a0 = tmem_base + a_col0 + as * S * 2 * KC;
        const uint32_t b0 = bres + us * S * 2 * b_bytes;
        if (elect_one()) {
          const uint64_t desc0 = sdesc(b0, lbo, 512u);
          const uint32_t bhi32 = (uint32_t)(desc0 >> 32);
          uint32_t bh = (uint32_t)desc0;               // low half of U_hi chunk c's descriptor
          int ch = 0;
          uint32_t d = d0, a_hi = a0;
          for (int c = 0; c < S; ++c) {            // chunk c = (r, ch) of the group
            if (!(dbg & 1))                        // (dbg & 1: dev probe, no MMAs)
              mma3_chunk_ts<NK>(d, a_hi, a_hi + KC, bh, bh + (b_bytes >> 4), bhi32, idesc, ch == 0);
            bh += (2 * b_bytes) >> 4;
            a_hi += 2 * KC;
            if (++ch == n_chunks) { ch = 0; d += BN; }
          }
          tc_commit(aempty(as));
          tc_commit(uempty(us));
          tc_commit(tfull(acc));
        }
        __syncwarp();
        FTR(2, 2, mci);
        ++mci;
        if (++as == na) { as = 0; aph ^= 1u; }
        if (++us == nbr) { us = 0; uph ^= 1u; }
        if (++acc == (uint32_t)nacc) { acc = 0; cph ^= 1u; }
      }
    }
  } else if (warp < NCV) {  // ---- converter (NCV warps): raw V rows -> TMEM A stage (hi / lo)
    const int qd = warp & 3, grp = warp >> 2;
    const int row = qd * 32 + lane;
    const uint32_t lane_sel = (uint32_t)(qd * 32) << 16;
    constexpr int cg0h = (KC / 8) / (NCV / 4);   // column groups of 8 per converter warp
    int rs = 0, as = 0, cci = 0;
    uint32_t rph = 0, aph = 0;
    for (long long u = blockIdx.x; u < total; u += gridDim.x) {
      for (int gi = 0; gi < ngrp; ++gi) {
        mbar_wait(aempty(as), aph ^ 1u);
        if (warp == 0) FTR(1, 1, cci);
        tc_fence_after();
        const uint32_t abase = tmem_base + lane_sel + a_col0 + as * S * 2 * KC;
        for (int c = 0; c < S; ++c) {
          mbar_wait(rfull(rs), rph);
          const float* raw = reinterpret_cast<const float*>(smem + rs * a_bytes) + row;
          const uint32_t ahi = abase + c * 2 * KC;
          if (!(dbg & 4)) {                    // (dbg & 4: dev probe, no conversion)
#pragma unroll
            for (int cgi = 0; cgi < cg0h; ++cgi) {
              const int cg = grp * cg0h + cgi;
              uint32_t hi[8], lo[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float v = raw[(cg * 8 + j) * BM];
                const uint32_t h = tf32_rna_bits(__float_as_uint(v));
                hi[j] = h;
                lo[j] = tf32_rna_bits(__float_as_uint(v - __uint_as_float(h)));
              }
              tmem_st8(ahi + cg * 8, hi);
              tmem_st8(ahi + KC + cg * 8, lo);
            }
          }
          // the raw slot is free once this thread's loads of it are done
          mbar_arrive(rempty(rs));
          if (++rs == nraw) { rs = 0; rph ^= 1u; }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(afull(as));
        if (warp == 0) FTR(1, 2, cci);
        ++cci;
        if (++as == na) { as = 0; aph ^= 1u; }
      }
    }
  } else if (warp < kEpi0 + 4 * G) {  // ---- epilogue: fold D_q into MO accumulators per (t, k)
    const int qd = warp & 3, cgp = (warp - kEpi0) >> 2;
    const uint32_t lane_sel = (uint32_t)(qd * 32) << 16;
    const uint64_t pol = l2_policy(true);   // W stays in L2 for a4 (evict-last)
    uint32_t acc = 0, aph = 0;
    int edi = 0;
    for (long long u = blockIdx.x; u < total; u += gridDim.x) {
      int xo, mb, nb;
      decode(u, xo, mb, nb);
      float z[MO][CW];
#pragma unroll
      for (int o = 0; o < MO; ++o)
#pragma unroll
        for (int j = 0; j < CW; ++j) z[o][j] = 0.f;
      for (int gi = 0; gi < ngrp; ++gi) {
        mbar_wait(tfull(acc), aph);
        if (warp == kEpi0) FTR(3, 0, edi);
        tc_fence_after();
        for (int r = 0; r < R; ++r) {
          const int q = gi * R + r;
          const uint32_t ta = tmem_base + lane_sel + (acc * R + r) * BN + cgp * CW;
          float cf[MO];
#pragma unroll
          for (int o = 0; o < MO; ++o) cf[o] = fold.coef[q][o];
          // this thread's CW columns in 16-column loads (register budget); the
          // accumulator group is released once all its D's are in registers
#pragma unroll
          for (int h = 0; h < CW / 16; ++h) {
            uint32_t rr[16];
            if (!(dbg & 2)) tmem_ld_cols<16>(ta + h * 16, rr);   // (dbg & 2: no loads / math)
            if (r == R - 1 && h == CW / 16 - 1) {
              tc_fence_before();
              mbar_arrive(tempty(acc));
            }
            if (dbg & 2) continue;
#pragma unroll
            for (int o = 0; o < MO; ++o) {
              if (cf[o] != 0.f) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  z[o][h * 16 + j] = fmaf(cf[o], __uint_as_float(rr[j]), z[o][h * 16 + j]);
              }
            }
          }
        }
        if (warp == kEpi0) FTR(3, 1, edi);
        ++edi;
        if (++acc == (uint32_t)nacc) { acc = 0; aph ^= 1u; }
      }
      // W[(xo * MO + o)][k][t]: lanes = consecutive t, one 128-byte line per (o, k)
      const int t = t_lo + mb * BM + qd * 32 + lane;
      const int k0 = nb * BN + cgp * CW;
      if (t < T && !(dbg & 16)) {       // (dbg & 16: dev probe, no W stores)
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          float* p = W + ((long long)(xo * MO + o) * K + k0) * T_s + t;
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            if (k0 + j < K) {
              if (l2hint) st_hint(p, z[o][j], pol);
              else __stcs(p, z[o][j]);
            }
            p += T_s;
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == kMma) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kCols) : "memory");
  }
#undef FTR
}

}  // namespace tc

// ---------------------------------------------------------------- host side
// Pipeline shape of one launch: R points per group (S = R * n_chunks chunks),
// na A stages and nacc accumulator groups in TMEM, nraw raw V stages and nbr
// U group stages in shared memory.
struct FoldPipe {
  int R, na, nacc, nraw, nbr;
  size_t smem;
};

static bool fold_pipe(int bn, int kc, int C, int Q, FoldPipe* fp) {
  const int n_chunks = (C + kc - 1) / kc;
  const size_t a = (size_t)tc::BM * kc * 4;
  const size_t b2 = 2ull * bn * kc * 4;
  const size_t fixed = 1024 + 1024;   // alignment pad + barriers / TMEM holder
  const size_t budget = 232448;
  // the widest group (R | Q) that leaves two A stages and two accumulator
  // groups in TMEM; fewer handshakes per D (measured: the MMA warp's per-step
  // waits and commits bound the small-N GEMM)
  int R = 0;
  for (int r = 4; r >= 1; r /= 2)
    if (Q % r == 0 && 2 * r * n_chunks * 2 * kc + 2 * r * bn <= 512) { R = r; break; }
  if (const char* ev = getenv("WINO_FOLD_R")) {       // dev knob
    const int r = atoi(ev);
    if (r >= 1 && Q % r == 0 && 2 * r * n_chunks * 2 * kc + 2 * r * bn <= 512) R = r;
  }
  if (!R) return false;
  const int S = R * n_chunks;
  int na = 2;
  int nacc = (512 - na * S * 2 * kc) / (R * bn);
  if (nacc > tc::kMaxAcc) nacc = tc::kMaxAcc;
  if (nacc < 2) return false;
  size_t left = budget - fixed;
  int nb = 3;
  while (nb > 1 && nb * S * b2 + 3 * a > left) --nb;
  if (nb * S * b2 + 2 * a > left) return false;
  left -= nb * S * b2;
  int nr = (int)(left / a);
  if (nr > 8) nr = 8;
  fp->R = R;
  fp->na = na;
  fp->nacc = nacc;
  fp->nraw = nr;
  fp->nbr = nb;
  fp->smem = budget - (left - nr * a);
  return true;
}

bool fold_feasible(int bn, int kc, int C, int Q) {
  FoldPipe fp;
  return fold_pipe(bn, kc, C, Q, &fp);
}

// (BN, G) for MO accumulators per output channel: the widest N tile whose
// per-thread accumulators (MO x BN / G) stay within 64 registers with at
// most two column groups (8 epilogue warps) and an instantiated kernel.
bool fold_shape(int K, int MO, int kc, int* bn, int* g) {
  static const int kBn[3] = {128, 64, 32};   // >= 32: the U maps load 32-column boxes
  for (int i = 0; i < 3; ++i) {
    const int b = kBn[i];
    if (b > 32 && b / 2 >= K) continue;                 // no wider than needed for K
    for (int gg = 1; gg <= 2; ++gg) {
      const int cw = b / gg;
      if (cw % 16 || MO * cw > 64) continue;
      if (!((b == 64 && gg == 2 && MO == 2) || (b == 32 && gg == 1 && MO == 2) || (b == 32 && gg == 2 && MO == 4)))
        continue;                                       // instantiated shapes (launch_gemm_fold)
      if (kc != 32 && kc != 64) continue;
      *bn = b;
      *g = gg;
      return true;
    }
  }
  return false;
}

// dev-only probe knob (results invalid when set): 1 no MMAs, 2 no epilogue
// loads / math, 4 no conversion, 8 no V loads, 16 no W stores
static int fold_dbg() {
  const char* ev = getenv("WINO_FOLD_DBG");
  return ev ? atoi(ev) : 0;
}

// dev-only pipeline trace (WINO_FOLD_TRACE=<file>): CTA 0's clock64 event
// times of the next launch; dumped by fold_trace_dump() after it completes
static unsigned long long* g_trace = nullptr;
static unsigned long long* fold_trace() {
  if (!getenv("WINO_FOLD_TRACE")) return nullptr;
  if (!g_trace && cudaMalloc(&g_trace, 5 * 4 * 256 * 8) != cudaSuccess) g_trace = nullptr;
  if (g_trace) cudaMemset(g_trace, 0, 5 * 4 * 256 * 8);
  return g_trace;
}
static void fold_trace_dump(cudaStream_t s) {
  const char* path = getenv("WINO_FOLD_TRACE");
  if (!path || !g_trace) return;
  static unsigned long long h[5 * 4 * 256];
  cudaStreamSynchronize(s);
  cudaMemcpy(h, g_trace, sizeof h, cudaMemcpyDeviceToHost);
  if (FILE* f = fopen(path, "wb")) {
    fwrite(h, sizeof h, 1, f);
    fclose(f);
  }
}

template <int BN, int G, int MO, int KC, int NCV>
static cudaError_t launch_fold_t(const TcGemm& tg, float* W, int P, int Q, int64_t t_lo, int64_t T, int64_t T_s,
                                 int C, int K, const FoldTab& fold, int l2hint, cudaStream_t s) {
  FoldPipe fp;
  if (!fold_pipe(BN, KC, C, Q, &fp)) return cudaErrorInvalidConfiguration;
  auto kern = tc::k_gemm_fold<BN, G, MO, KC, NCV>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fp.smem);
  if (e != cudaSuccess) return e;
  const long long units = (long long)(P / Q) * ((K + BN - 1) / BN) * ((T - t_lo + tc::BM - 1) / tc::BM);
  const int grid = (int)(units < tg.num_sms ? units : tg.num_sms);
  if (grid <= 0) return cudaSuccess;
  if (getenv("WINO_DEBUG"))
    fprintf(stderr, "[wino] k_gemm_fold<%d,%d,%d,%d,%d>: R %d na %d nacc %d nraw %d nbr %d smem %zu\n", BN, G, MO,
            KC, NCV, fp.R, fp.na, fp.nacc, fp.nraw, fp.nbr, fp.smem);
  const long long Ts = T_s;
  cudaError_t er = launch_pdl(kern, dim3(grid), dim3(tc::fold_threads<G, NCV>()), fp.smem, s, tg.tmA_ts, tg.tmBhi,
                              tg.tmBlo, W, P, Q, fp.R, (int)t_lo, (int)T, Ts, C, K, fp.nraw, fp.nbr, fp.na, fp.nacc,
                              l2hint, fold_dbg(), fold_trace(), fold);
  fold_trace_dump(s);
  return er;
}

cudaError_t launch_gemm_fold(const TcGemm& tg, int bn, int g, int MO, float* W, int P, int Q, int64_t t_lo,
                             int64_t T, int64_t T_s, int C, int K, const FoldTab& fold, cudaStream_t s) {
  if (!tg.ready || !tg.three) return cudaErrorNotReady;
  static int l2hint = -1;
  if (l2hint < 0) {
    const char* ev = getenv("WINO_L2_HINTS");
    l2hint = ev ? (atoi(ev) != 0) : 1;
  }
  // 4 converter warps: 128 registers per thread with 8 epilogue warps
  // (measured: 8 converter warps, 96 registers, no faster -- c5 0.1599 vs
  // 0.1587 ms, c3 F = 1 1.73 vs 2.00 ms)
#define WINO_FOLD_CASE(B, GG, O)                                                                              \
  if (bn == B && g == GG && MO == O) {                                                                        \
    if (tg.kc == 64) return launch_fold_t<B, GG, O, 64, 4>(tg, W, P, Q, t_lo, T, T_s, C, K, fold, l2hint, s);  \
    return launch_fold_t<B, GG, O, 32, 4>(tg, W, P, Q, t_lo, T, T_s, C, K, fold, l2hint, s);                   \
  }
  WINO_FOLD_CASE(64, 2, 2)
  WINO_FOLD_CASE(32, 1, 2)
  WINO_FOLD_CASE(32, 2, 4)
#undef WINO_FOLD_CASE
  return cudaErrorNotSupported;
}

}  // namespace wino
