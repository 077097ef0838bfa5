// gemm_f16.cu -- stage a3 with an fp32-accurate 3 x FP16 split on the
// kind::f16 tensor-core path (twice the TF32 rate), CTA pairs, A in TMEM.
//
// For every transform point xi, M_xi = V_xi U_xi (Eq. (5))
// with V and U scaled by powers of two and split into two fp16 parts:
//     v' = v * 2^-sv,  v' = v_hi + v_lo,  v_hi = fp16_rn(v'),  v_lo = fp16_rn(v' - v_hi)
//     u' = u * 2^-su   (same split, done once by the filter transform)
//     M  = 2^(sv + su) (v_lo u_hi + v_hi u_lo + v_hi u_hi)      fp32 accumulation
// fp16 x fp16 products are exact in fp32 and hi + lo carries 22 significant
// bits, as the RNA TF32 split of the 3xTF32 scheme does (DESIGN.md reading
// #7); the scales keep v', u' <= 2^15 (max|V| is reduced by the input
// transform, max|U| by the filter transform), so nothing overflows fp16 and
// elements below 2^-14 of the scaled range only lose absolute precision far
// under the fp32 rounding of the sums.  The kind::f16 MMA takes K = 16 per
// instruction (tf32: 8), so the three products cost what 1.5 TF32 products do.
//
// Structure as k_gemm_ts2 (gemm_ts2.cu): a unit (xi, n-block, 256-tile
// m-pair) on a cluster of two CTAs; each CTA converts its own 128 rows into
// its TMEM (packed fp16 pairs, lower k in the low half) and loads half of each
// U chunk; the leader issues tcgen05.mma.cta_group::2.kind::f16 M=256 N=BN
// K=16; commits multicast to both CTAs.  Warps: 0-3 and 11-14 converter, 4-7
// epilogue, 8 V producer, 9 MMA issuer (leader) / TMEM owner, 10 U producer.
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "tc_common.cuh"
#include "tma.hpp"

namespace wino {
namespace tc {
namespace {

// kind::f16: D f32 (bit 4), A = B = f16 (format 0), A K-major (TMEM), B
// MN-major (bit 16), M = 256 (pair), N = BN.
template <int BN>
__host__ __device__ constexpr uint32_t idesc_f16_pair() {
  return (1u << 4) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

__device__ __forceinline__ void mma2_f16_split(uint32_t d, uint32_t a_tmem, uint32_t b_lo32, uint32_t b_hi32,
                                               uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 bd;\n\tmov.b64 bd, {%2, %3};\n\tsetp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], bd, %4, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "r"(b_lo32), "r"(b_hi32), "r"(idesc), "r"(acc)
      : "memory");
}

// Shared-memory descriptor of a 16-bit MN-major operand with 128-byte
// swizzle (layout type 2): rows of 128 B = 64 elements along N, 8-row swizzle
// atoms (SBO = 1024 B) along K, LBO = distance between 64-element groups along
// N (verified on B200 by tools/f16_probe.cu).
__device__ __forceinline__ uint64_t sdesc_f16(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// 2^k as a float for |k| < 126
__device__ __forceinline__ float exp2i(int k) { return __uint_as_float((uint32_t)(127 + k) << 23); }

// scale exponent for a max magnitude m (float bits): 2^-s with m * 2^-s <= 2^15
__device__ __forceinline__ int scale_exp(uint32_t mbits) {
  if (mbits == 0u || mbits >= 0x7F800000u) return 0;   // zero (or non-finite: left as is)
  const int e = (int)(mbits >> 23) - 127;               // m < 2^(e+1)
  return e + 1 - 15;                                    // s
}

template <int BN, int KC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsTS, 1)
k_gemm_f16p(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
            const __grid_constant__ CUtensorMap tmBlo, float* __restrict__ Mo, int P, int t_lo, int T, long long T_s,
            int C, int K, int nraw, int nbr, int l2hint, const unsigned int* __restrict__ vmax,
            const float* __restrict__ uscal, int dbg, int nbfast) {
  constexpr int HN = BN / 2;  // U columns loaded by each CTA
  static_assert(HN == 64, "one 64-wide fp16 swizzle group per CTA half");
  constexpr int NKS = KC / 16;                 // K=16 MMA steps per chunk
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (sraw & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  const uint32_t sbase = sraw + pad;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n_chunks = (C + KC - 1) / KC;
  const uint32_t a_bytes = (uint32_t)BM * KC * 4;   // raw fp32 V chunk
  const uint32_t hb_bytes = (uint32_t)HN * KC * 2;  // this CTA's half of one U chunk (hi or lo), fp16
  const uint32_t raw0 = sbase;
  const uint32_t ub0 = raw0 + nraw * a_bytes;
  const uint32_t bar0 = ub0 + 2u * nbr * hb_bytes;
  auto rfull = [&](int s) { return bar0 + 8u * s; };
  auto rempty = [&](int s) { return bar0 + 8u * (nraw + s); };
  auto ufull = [&](int s) { return bar0 + 8u * (2 * nraw + s); };
  auto uempty = [&](int s) { return bar0 + 8u * (2 * nraw + nbr + s); };
  const uint32_t bar1 = bar0 + 8u * (2 * nraw + 2 * nbr);
  auto tfull = [&](int a) { return bar1 + 8u * a; };          // a < 4
  auto tempty = [&](int a) { return bar1 + 8u * (4 + a); };
  auto afull = [&](int a) { return bar1 + 8u * (8 + a); };    // a < 4
  auto aempty = [&](int a) { return bar1 + 8u * (12 + a); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + (bar1 - sbase) + 128);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // TMEM: nacc accumulators + na A stages (V_hi | V_lo packed: KC columns
  // each).  The packed fp16 stages are half the tf32 ones, which leaves room
  // for a third accumulator: the tensor work per unit halved, so the epilogue
  // (TMEM loads, M stores) needs the extra slack
  const int nacc = (512 - 2 * KC) / BN >= 3 ? 3 : 2;
  int na = (512 - nacc * BN) / KC;
  na = na > 4 ? 4 : na;
  const uint32_t kCols = pow2_cols(nacc * BN + KC * na);
  const uint32_t a_col0 = nacc * BN;

  if (warp == 9) {
    if (lane == 0) {
      for (int s = 0; s < nraw; ++s) {
        mbar_init(rfull(s), 1);
        mbar_init(rempty(s), 256);
      }
      for (int s = 0; s < nbr; ++s) {
        mbar_init(ufull(s), 1);
        mbar_init(uempty(s), 1);
      }
      for (int a = 0; a < nacc; ++a) {
        mbar_init(tfull(a), 1);
        mbar_init(tempty(a), 2);
      }
      for (int a = 0; a < na; ++a) {
        mbar_init(afull(a), 2);
        mbar_init(aempty(a), 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();      // V and max|V| come from the input transform
  pdl_trigger();
  const int sv = scale_exp(*vmax);
  const float vscale = exp2i(-sv);                  // v' = v * 2^-sv
  const float mscale = exp2i(sv) * __ldg(uscal);    // M = 2^(sv + su) * acc  (uscal = 2^su)

  const int n_mp = (T - t_lo + 2 * BM - 1) / (2 * BM);
  const int n_nblk = (K + BN - 1) / BN;
  const unsigned per_xi = (unsigned)n_nblk * (unsigned)n_mp;   // units fit 32 bits (32-bit decode)
  const unsigned total = (unsigned)P * per_xi;
  const unsigned u_beg = blockIdx.x >> 1, u_step = gridDim.x >> 1;

  if (warp == 8) {
    if (lane == 0) {  // ---------------- V producer: this CTA's 128 rows
      int s = 0;
      uint32_t ph = 0;
      for (unsigned u = u_beg; u < total; u += u_step) {
        const int xi = (int)(u / per_xi);
        const int mp = nbfast ? (int)(u % per_xi) / n_nblk : (int)(u % per_xi) % n_mp;
        const int row0 = t_lo + mp * 2 * BM + (int)rank * BM;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(rempty(s), ph ^ 1u);
          mbar_expect_tx(rfull(s), a_bytes);
          if (l2hint) tma_load_3d_hint(raw0 + s * a_bytes, &tmA, row0, ch * KC, xi, rfull(s), l2_policy(false));
          else tma_load_3d(raw0 + s * a_bytes, &tmA, row0, ch * KC, xi, rfull(s));
          if (++s == nraw) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {  // ---------------- U producer: this CTA's 64 columns (hi, lo)
      int s = 0;
      uint32_t ph = 0;
      for (unsigned u = u_beg; u < total; u += u_step) {
        const int xi = (int)(u / per_xi);
        const int nb = nbfast ? (int)(u % per_xi) % n_nblk : (int)(u % per_xi) / n_mp;
        const int col0 = nb * BN + (int)rank * HN;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(uempty(s), ph ^ 1u);
          const uint32_t st = ub0 + s * 2 * hb_bytes;
          const uint32_t lb = mapa(ufull(s), 0);
          if (leader) mbar_expect_tx(ufull(s), 4u * hb_bytes);
          tma_load_3d_pair(st, &tmBhi, col0, ch * KC, xi, lb);
          tma_load_3d_pair(st + hb_bytes, &tmBlo, col0, ch * KC, xi, lb);
          if (++s == nbr) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 9) {
    if (leader) {  // ---------------- MMA issuer (leader CTA)
      constexpr uint32_t idesc = idesc_f16_pair<BN>();
      constexpr uint32_t lbo = (uint32_t)KC * 128u;
      int as = 0, us = 0;
      uint32_t aph = 0, uph = 0, acc = 0, cph = 0;
      for (unsigned u = u_beg; u < total; u += u_step) {
        mbar_wait(tempty(acc), cph ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(afull(as), aph);
          mbar_wait(ufull(us), uph);
          tc_fence_after();
          const uint32_t b_hi = ub0 + us * 2 * hb_bytes;
          const uint64_t dh = sdesc_f16(b_hi, lbo), dl = sdesc_f16(b_hi + hb_bytes, lbo);
          const uint32_t bhi32 = (uint32_t)(dh >> 32), bh = (uint32_t)dh, bl = (uint32_t)dl;
          const uint32_t a_hi = tmem_base + a_col0 + as * KC, a_lo = a_hi + KC / 2;
          if (elect_one()) {
#pragma unroll
            for (int j = 0; j < ((dbg & 1) ? 0 : NKS); ++j) {   // K=16 step j: A columns +8j, B rows +16j (2048 B)
              mma2_f16_split(d, a_lo + 8 * j, bh + 128 * j, bhi32, idesc, (ch | j) != 0);
              mma2_f16_split(d, a_hi + 8 * j, bl + 128 * j, bhi32, idesc, 1u);
              mma2_f16_split(d, a_hi + 8 * j, bh + 128 * j, bhi32, idesc, 1u);
            }
            tc2_commit_mc(aempty(as));
            tc2_commit_mc(uempty(us));
          }
          __syncwarp();
          if (++as == na) { as = 0; aph ^= 1u; }
          if (++us == nbr) { us = 0; uph ^= 1u; }
        }
        if (elect_one()) tc2_commit_mc(tfull(acc));
        __syncwarp();
        if (++acc == (uint32_t)nacc) { acc = 0; cph ^= 1u; }
      }
    }
  } else if (warp < 4 || (warp >= 11 && warp < 15)) {  // ---- converter (8 warps): raw V row -> TMEM fp16 pairs
    const int q = warp & 3, grp = warp < 4 ? 0 : 1;
    const int row = q * 32 + lane;
    const uint32_t lane_sel = (uint32_t)(q * 32) << 16;
    constexpr int NG = KC / 16;                 // 16-channel groups per chunk
    const int g0 = grp * NG / 2, g1 = (grp + 1) * NG / 2;
    int rs = 0, as = 0;
    uint32_t rph = 0, aph = 0;
    for (unsigned u = u_beg; u < total; u += u_step) {
      for (int ch = 0; ch < n_chunks; ++ch) {
        mbar_wait(rfull(rs), rph);
        mbar_wait(aempty(as), aph ^ 1u);
        tc_fence_after();
        const float* rawp = reinterpret_cast<const float*>(smem + rs * a_bytes) + row;
        const uint32_t ahi = tmem_base + lane_sel + a_col0 + as * KC;
        for (int gg = g0; gg < ((dbg & 2) ? g0 : g1); ++gg) {
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            // channels 2j, 2j+1 -> one packed pair each for hi and lo (paired
            // conversions: cvt.rn.f16x2.f32; the lower channel in the low half)
            const float v0 = rawp[(gg * 16 + 2 * j) * BM] * vscale;
            const float v1 = rawp[(gg * 16 + 2 * j + 1) * BM] * vscale;
            const __half2 h = __floats2half2_rn(v0, v1);
            const float2 hf = __half22float2(h);
            const __half2 l = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
            hi[j] = *reinterpret_cast<const uint32_t*>(&h);
            lo[j] = *reinterpret_cast<const uint32_t*>(&l);
          }
          tmem_st8(ahi + gg * 8, hi);
          tmem_st8(ahi + KC / 2 + gg * 8, lo);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(rempty(rs));
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (threadIdx.x == 0) mbar_arrive_cluster(mapa(afull(as), 0));
        if (++rs == nraw) { rs = 0; rph ^= 1u; }
        if (++as == na) { as = 0; aph ^= 1u; }
      }
    }
  } else if (warp < 8) {  // warps 4-7 ------------------ epilogue: own 128 rows, M = 2^(sv+su) acc
    const int q = warp - 4;
    const uint32_t tempty_l[4] = {mapa(tempty(0), 0), mapa(tempty(1), 0), mapa(tempty(2), 0), mapa(tempty(3), 0)};
    const uint64_t pol = l2_policy(true);
    uint32_t acc = 0, aph = 0;
    for (unsigned u = u_beg; u < total; u += u_step) {
      const int xi = (int)(u / per_xi);
      const int rr = (int)(u % per_xi);
      const int nb = nbfast ? rr % n_nblk : rr / n_mp, mp = nbfast ? rr / n_nblk : rr % n_mp;
      mbar_wait(tfull(acc), aph);
      tc_fence_after();
      const int t = t_lo + mp * 2 * BM + (int)rank * BM + q * 32 + lane;
      float* out = Mo + ((long long)xi * K + (long long)nb * BN) * T_s + t;
      const int kr_all = K - nb * BN;
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      // 32-column blocks, the next block's TMEM load in flight while this
      // block's 32 stores issue
      uint32_t ra[32], rb[32];
      tmem_ld32_nowait(ta, ra);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int cb = 0; cb < BN / 32; ++cb) {
        uint32_t(&cur)[32] = (cb & 1) ? rb : ra;
        uint32_t(&nxt)[32] = (cb & 1) ? ra : rb;
        if (cb + 1 < BN / 32) tmem_ld32_nowait(ta + (cb + 1) * 32, nxt);
        if (t < T && !(dbg & 4)) {
          float* p = out + (long long)cb * 32 * T_s;
          const int kr = kr_all - cb * 32;
          store_m32<true>(p, cur, T_s, kr, l2hint, pol, mscale);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (threadIdx.x == 128) mbar_arrive_cluster(tempty_l[acc]);
      if (++acc == (uint32_t)nacc) { acc = 0; aph ^= 1u; }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kCols) : "memory");
  }
}

// V-resident variant for K = NB * BN with NB = 2 (k_gemm_f16n): a unit is
// (xi, m-pair) and covers every n-block.  The unit's whole converted V block
// (C / KC chunks, KC TMEM columns each) sits in TMEM next to NB accumulators
// (NB * BN + C <= 512 columns), so V is loaded and converted once per unit
// instead of once per n-block (k_gemm_f16p re-reads it through L2 and
// converts it NB times).  Chunk slot c is released for the next unit's
// conversion by the last n-block's MMA on it; accumulator nb is drained by
// the epilogue while the MMAs of the next n-block run.  zmask bit nb*8 + c:
// U chunk (nb, c) is zero by construction (filter-side fold, A^T_F[o][q] = 0
// for every column of the n-block), its U load and MMAs are skipped.
// DF (direct-axis fold, xform_dfold.cu): the A operand is Z [P*2][df_cz][Tz]
// in rows of df_S slots; k-chunk ch holds tap j = ch*KC / df_cz (df_cz a multiple of
// KC), loaded as the {BM + 4, KC} box of plane xi*2 + (j & 1) at the unit's
// 16-byte aligned first slot (TMA start coordinates must be 16-byte aligned:
// tools/tma_off_probe.cu) and read by the converter at slot + (j >> 1); T
// counts slots (df_S per row of tiles), and the epilogue stores
// slot (row, i < df_tl2) at tile row * df_tl2 + i of W.
template <int BN, int KC, int NB, bool DF = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsTS, 1)
k_gemm_f16n(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
            const __grid_constant__ CUtensorMap tmBlo, float* __restrict__ Mo, int P, int t_lo, int T, long long T_s,
            int C, int K, int nraw, int nbr, int l2hint, const unsigned int* __restrict__ vmax,
            const float* __restrict__ uscal, int zmask, int df_tl2, int df_cz, int df_S) {
  constexpr int BMR = DF ? BM + 4 : BM;   // raw-stage row pitch (slots)
  constexpr int HN = BN / 2;
  static_assert(HN == 64, "one 64-wide fp16 swizzle group per CTA half");
  constexpr int NKS = KC / 16;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (sraw & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  const uint32_t sbase = sraw + pad;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n_chunks = (C + KC - 1) / KC;            // <= (512 - NB * BN) / KC (host-checked)
  const uint32_t a_bytes = (uint32_t)BMR * KC * 4;
  const uint32_t hb_bytes = (uint32_t)HN * KC * 2;
  const uint32_t raw0 = sbase;
  const uint32_t ub0 = (raw0 + nraw * a_bytes + 1023u) & ~1023u;   // (DF: a_bytes is not a multiple of 1024)
  const uint32_t bar0 = ub0 + 2u * nbr * hb_bytes;
  auto rfull = [&](int s) { return bar0 + 8u * s; };
  auto rempty = [&](int s) { return bar0 + 8u * (nraw + s); };
  auto ufull = [&](int s) { return bar0 + 8u * (2 * nraw + s); };
  auto uempty = [&](int s) { return bar0 + 8u * (2 * nraw + nbr + s); };
  const uint32_t bar1 = bar0 + 8u * (2 * nraw + 2 * nbr);
  auto tfull = [&](int a) { return bar1 + 8u * a; };          // a < NB
  auto tempty = [&](int a) { return bar1 + 8u * (4 + a); };
  auto afull = [&](int c) { return bar1 + 8u * (8 + c); };    // c < 16 chunk slots
  auto aempty = [&](int c) { return bar1 + 8u * (24 + c); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + (bar1 - sbase) + 8 * 40);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t kCols = 512;
  const uint32_t a_col0 = NB * BN;

  if (warp == 9) {
    if (lane == 0) {
      for (int s = 0; s < nraw; ++s) {
        mbar_init(rfull(s), 1);
        mbar_init(rempty(s), 256);
      }
      for (int s = 0; s < nbr; ++s) {
        mbar_init(ufull(s), 1);
        mbar_init(uempty(s), 1);
      }
      for (int a = 0; a < NB; ++a) {
        mbar_init(tfull(a), 1);
        mbar_init(tempty(a), 2);
      }
      for (int c = 0; c < n_chunks; ++c) {
        mbar_init(afull(c), 2);
        mbar_init(aempty(c), 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();
  pdl_trigger();
  const int sv = scale_exp(*vmax);
  const float vscale = exp2i(-sv);
  const float mscale = exp2i(sv) * __ldg(uscal);

  const int n_mp = (T - t_lo + 2 * BM - 1) / (2 * BM);
  const unsigned total = (unsigned)P * (unsigned)n_mp;   // units fit 32 bits (32-bit decode)
  const unsigned u_beg = blockIdx.x >> 1, u_step = gridDim.x >> 1;
  auto skip = [&](int nb, int c) { return (zmask >> (nb * 8 + c)) & 1; };

  if (warp == 8) {
    if (lane == 0) {  // ---------------- V producer: this CTA's 128 rows, once per unit
      int s = 0;
      uint32_t ph = 0;
      for (unsigned u = u_beg; u < total; u += u_step) {
        const int xi = (int)(u / n_mp);
        const int row0 = t_lo + (int)(u % n_mp) * 2 * BM + (int)rank * BM;
        // DF: one box per (parity plane, channel chunk) -- taps j and j + 2
        // read the same box at slots + 0 / + 1 (2 * df_cz / KC loads per unit)
        const int n_loads = DF ? 2 * (df_cz / KC) : n_chunks;
        for (int ch = 0; ch < n_loads; ++ch) {
          mbar_wait(rempty(s), ph ^ 1u);
          mbar_expect_tx(rfull(s), a_bytes);
          int crow = ch * KC, plane = xi;
          if constexpr (DF) {
            const int par = crow / df_cz;
            crow -= par * df_cz;
            plane = xi * 2 + par;
          }
          if (l2hint) tma_load_3d_hint(raw0 + s * a_bytes, &tmA, row0, crow, plane, rfull(s), l2_policy(false));
          else tma_load_3d(raw0 + s * a_bytes, &tmA, row0, crow, plane, rfull(s));
          if (++s == nraw) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {  // ---------------- U producer: (n-block, chunk) pairs of the unit
      int s = 0;
      uint32_t ph = 0;
      for (unsigned u = u_beg; u < total; u += u_step) {
        const int xi = (int)(u / n_mp);
        for (int nb = 0; nb < NB; ++nb) {
          const int col0 = nb * BN + (int)rank * HN;
          for (int ch = 0; ch < n_chunks; ++ch) {
            if (skip(nb, ch)) continue;
            mbar_wait(uempty(s), ph ^ 1u);
            const uint32_t st = ub0 + s * 2 * hb_bytes;
            const uint32_t lb = mapa(ufull(s), 0);
            if (leader) mbar_expect_tx(ufull(s), 4u * hb_bytes);
            tma_load_3d_pair(st, &tmBhi, col0, ch * KC, xi, lb);
            tma_load_3d_pair(st + hb_bytes, &tmBlo, col0, ch * KC, xi, lb);
            if (++s == nbr) { s = 0; ph ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 9) {
    if (leader) {  // ---------------- MMA issuer (leader CTA)
      constexpr uint32_t idesc = idesc_f16_pair<BN>();
      constexpr uint32_t lbo = (uint32_t)KC * 128u;
      int us = 0;
      uint32_t uph = 0, uphase = 0;   // uphase: the unit's parity (A slots, accumulators)
      for (unsigned u = u_beg; u < total; u += u_step) {
        for (int nb = 0; nb < NB; ++nb) {
          mbar_wait(tempty(nb), uphase ^ 1u);
          tc_fence_after();
          const uint32_t d = tmem_base + nb * BN;
          bool first = true;
          for (int ch = 0; ch < n_chunks; ++ch) {
            const bool sk = skip(nb, ch);
            if (nb == 0) mbar_wait(afull(ch), uphase);
            if (!sk) {
              mbar_wait(ufull(us), uph);
              tc_fence_after();
              const uint32_t b_hi = ub0 + us * 2 * hb_bytes;
              const uint64_t dh = sdesc_f16(b_hi, lbo), dl = sdesc_f16(b_hi + hb_bytes, lbo);
              const uint32_t bhi32 = (uint32_t)(dh >> 32), bh = (uint32_t)dh, bl = (uint32_t)dl;
              const uint32_t a_hi = tmem_base + a_col0 + ch * KC, a_lo = a_hi + KC / 2;
              if (elect_one()) {
#pragma unroll
                for (int j = 0; j < NKS; ++j) {
                  mma2_f16_split(d, a_lo + 8 * j, bh + 128 * j, bhi32, idesc, (first && j == 0) ? 0u : 1u);
                  mma2_f16_split(d, a_hi + 8 * j, bl + 128 * j, bhi32, idesc, 1u);
                  mma2_f16_split(d, a_hi + 8 * j, bh + 128 * j, bhi32, idesc, 1u);
                }
                tc2_commit_mc(uempty(us));
              }
              __syncwarp();
              first = false;
              if (++us == nbr) { us = 0; uph ^= 1u; }
            }
            if (nb == NB - 1) {   // last reader of chunk slot ch in this unit
              if (elect_one()) tc2_commit_mc(aempty(ch));
              __syncwarp();
            }
          }
          if (elect_one()) tc2_commit_mc(tfull(nb));
          __syncwarp();
        }
        uphase ^= 1u;
      }
    }
  } else if (warp < 4 || (warp >= 11 && warp < 15)) {  // ---- converter (8 warps), each chunk once per unit
    const int q = warp & 3, grp = warp < 4 ? 0 : 1;
    const int row = q * 32 + lane;
    const uint32_t lane_sel = (uint32_t)(q * 32) << 16;
    constexpr int NG = KC / 16;
    const int g0 = grp * NG / 2, g1 = (grp + 1) * NG / 2;
    int rs = 0;
    uint32_t rph = 0, uphase = 0;
    unsigned ld0 = 0;   // DF: raw loads issued before this unit (stage of load L: (ld0 + L) % nraw)
    const int ncz = DF ? df_cz / KC : 1;
    for (unsigned u = u_beg; u < total; u += u_step) {
      for (int ch = 0; ch < n_chunks; ++ch) {
        int tap = 0;
        if constexpr (DF) {   // chunk (tap j, cc) reads load (j & 1, cc), filled once per unit
          tap = ch / ncz;
          const unsigned ld = ld0 + (unsigned)((tap & 1) * ncz + (ch - tap * ncz));
          rs = (int)(ld % (unsigned)nraw);
          rph = (ld / (unsigned)nraw) & 1u;
        }
        mbar_wait(rfull(rs), rph);
        mbar_wait(aempty(ch), uphase ^ 1u);
        tc_fence_after();
        const float* rawp = reinterpret_cast<const float*>(smem + rs * a_bytes) + row;
        if constexpr (DF) rawp += tap >> 1;   // tap j's slot shift
        const uint32_t ahi = tmem_base + lane_sel + a_col0 + ch * KC;
        for (int gg = g0; gg < g1; ++gg) {
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float v0 = rawp[(gg * 16 + 2 * j) * BMR] * vscale;
            const float v1 = rawp[(gg * 16 + 2 * j + 1) * BMR] * vscale;
            const __half2 h = __floats2half2_rn(v0, v1);
            const float2 hf = __half22float2(h);
            const __half2 l = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
            hi[j] = *reinterpret_cast<const uint32_t*>(&h);
            lo[j] = *reinterpret_cast<const uint32_t*>(&l);
          }
          tmem_st8(ahi + gg * 8, hi);
          tmem_st8(ahi + KC / 2 + gg * 8, lo);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        if constexpr (DF) {
          if (tap >= 2) mbar_arrive(rempty(rs));   // the box's second and last reader
        } else {
          mbar_arrive(rempty(rs));
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (threadIdx.x == 0) mbar_arrive_cluster(mapa(afull(ch), 0));
        if constexpr (!DF) {
          if (++rs == nraw) { rs = 0; rph ^= 1u; }
        }
      }
      if constexpr (DF) ld0 += 2u * (unsigned)ncz;
      uphase ^= 1u;
    }
  } else if (warp < 8) {  // warps 4-7 ------------------ epilogue: NB accumulators per unit
    const int q = warp - 4;
    const uint64_t pol = l2_policy(true);
    uint32_t uphase = 0;
    for (unsigned u = u_beg; u < total; u += u_step) {
      const int xi = (int)(u / n_mp);
      const int mp = (int)(u % n_mp);
      int t = t_lo + mp * 2 * BM + (int)rank * BM + q * 32 + lane;
      bool live = t < T;
      if constexpr (DF) {   // slot row * S + i -> tile row * tl2 + i; slot i = tl2 of a row only feeds the taps
        const int zr = t / df_S, zi = t - zr * df_S;
        live = live && zi < df_tl2;
        t = zr * df_tl2 + zi;
      }
      for (int nb = 0; nb < NB; ++nb) {
        mbar_wait(tfull(nb), uphase);
        tc_fence_after();
        float* out = Mo + ((long long)xi * K + (long long)nb * BN) * T_s + t;
        const int kr_all = K - nb * BN;
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + nb * BN;
        uint32_t ra[32], rb[32];
        tmem_ld32_nowait(ta, ra);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int cb = 0; cb < BN / 32; ++cb) {
          uint32_t(&cur)[32] = (cb & 1) ? rb : ra;
          uint32_t(&nxt)[32] = (cb & 1) ? ra : rb;
          if (cb + 1 < BN / 32) tmem_ld32_nowait(ta + (cb + 1) * 32, nxt);
          if (live) store_m32<true>(out + (long long)cb * 32 * T_s, cur, T_s, kr_all - cb * 32, l2hint, pol, mscale);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (threadIdx.x == 128) mbar_arrive_cluster(mapa(tempty(nb), 0));
      }
      uphase ^= 1u;
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kCols) : "memory");
  }
}

}  // namespace
}  // namespace tc

// ---------------------------------------------------------------- host side
static bool f16_smem(int kc, int* nraw, int* nbr, size_t* bytes, int raw_rows = tc::BM) {
  const size_t a = (size_t)raw_rows * kc * 4;   // (BM + 4 rows under the direct-axis fold)
  const size_t hb2 = 2ull * 64 * kc * 2;     // hi + lo halves of one chunk, fp16
  const size_t fixed = 1024 + 1024 + (raw_rows != tc::BM ? 1024 : 0);   // + the U ring's 1 KB alignment
  const size_t budget = 232448;
  size_t left = budget - fixed;
  int nb = 4;
  while (nb > 2 && nb * hb2 + 4 * a > left) --nb;
  if (nb * hb2 + 2 * a > left) return false;
  left -= nb * hb2;
  int nr = (int)(left / a);
  if (nr > 8) nr = 8;
  *nraw = nr;
  *nbr = nb;
  *bytes = budget - (left - nr * a);
  return true;
}

// fp16 U maps: [P][C][K_s] halves viewed as (k, c, xi), box {64, kc, 1}, 128-byte swizzle.
cudaError_t f16_encode_u(CUtensorMap* tm, const void* base, int64_t K_s, int C, int P, int kc) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {(cuuint64_t)K_s, (cuuint64_t)C, (cuuint64_t)P};
  cuuint64_t strides[2] = {(cuuint64_t)K_s * 2, (cuuint64_t)K_s * 2 * C};
  cuuint32_t box[3] = {64, (cuuint32_t)kc, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

bool f16_supported(int K, int kc) {
  int nr, nb;
  size_t by;
  return K > 64 && (kc == 32 || kc == 64) && f16_smem(kc, &nr, &nb, &by);
}

// dev-only probe knob (results invalid when set): 1 no MMAs, 2 no conversion, 4 no M stores
static int f16_dbg() {
  const char* ev = getenv("WINO_F16_DBG");
  return ev ? atoi(ev) : 0;
}

template <int KC>
static cudaError_t launch_f16_kc(const TcGemm& tg, const CUtensorMap& tmBhi16, const CUtensorMap& tmBlo16, float* Mo,
                                 int P, int64_t t_lo, int64_t T, int64_t T_s, int C, int K, const unsigned int* vmax,
                                 const float* uscal, cudaStream_t s) {
  constexpr int BN = 128;
  int nraw, nbr;
  size_t smem;
  if (!f16_smem(KC, &nraw, &nbr, &smem)) return cudaErrorInvalidConfiguration;
  auto kern = tc::k_gemm_f16p<BN, KC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long units = (long long)P * ((K + BN - 1) / BN) * ((T - t_lo + 2 * tc::BM - 1) / (2 * tc::BM));
  if (units >= (1LL << 31)) return cudaErrorNotSupported;   // the kernel decodes units in 32 bits
  // co-resident CTA pairs (occupancy query, as the tf32 pair kernel)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  static int max_pairs_dev[kMaxDevices][2] = {};
  int& max_pairs = max_pairs_dev[dev][KC == 64 ? 1 : 0];
  if (!max_pairs) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(tg.num_sms);
    cfg.blockDim = dim3(tc::kThreadsTS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) n = tg.num_sms / 2;
    max_pairs = n;
  }
  long long pairs = max_pairs < units ? max_pairs : units;
  if (pairs < 1) return cudaSuccess;
  static int l2hint = -1;
  if (l2hint < 0) {
    const char* ev = getenv("WINO_L2_HINTS");
    l2hint = ev ? (atoi(ev) != 0) : 1;
  }
  const long long Ts = T_s;
  return launch_pdl(kern, dim3((unsigned)(2 * pairs)), dim3(tc::kThreadsTS), smem, s, tg.tmA_ts, tmBhi16, tmBlo16, Mo,
                    P, (int)t_lo, (int)T, Ts, C, K, nraw, nbr, l2hint, vmax, uscal, f16_dbg(), gemm_nbfast());
}

// k_gemm_f16n (V block resident in TMEM across the two n-blocks)
template <int KC, bool DF>
static cudaError_t launch_f16n_kc(const TcGemm& tg, const CUtensorMap& tmBhi16, const CUtensorMap& tmBlo16,
                                  float* Mo, int P, int64_t t_lo, int64_t T, int64_t T_s, int C, int K,
                                  const unsigned int* vmax, const float* uscal, int zmask, cudaStream_t s,
                                  const DFoldGemm* df) {
  constexpr int BN = 128, NB = 2;
  int nraw, nbr;
  size_t smem;
  if (!f16_smem(KC, &nraw, &nbr, &smem, DF ? tc::BM + 4 : tc::BM)) return cudaErrorInvalidConfiguration;
  if (DF && nraw < 2 * (df->cz / KC)) return cudaErrorInvalidConfiguration;   // a unit's boxes are held together
  auto kern = tc::k_gemm_f16n<BN, KC, NB, DF>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long units = (long long)P * ((T - t_lo + 2 * tc::BM - 1) / (2 * tc::BM));
  if (units >= (1LL << 31)) return cudaErrorNotSupported;   // the kernel decodes units in 32 bits
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  static int max_pairs_dev[kMaxDevices][2] = {};
  int& max_pairs = max_pairs_dev[dev][KC == 64 ? 1 : 0];
  if (!max_pairs) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(tg.num_sms);
    cfg.blockDim = dim3(tc::kThreadsTS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) n = tg.num_sms / 2;
    max_pairs = n;
  }
  const long long pairs = max_pairs < units ? max_pairs : units;
  if (pairs < 1) return cudaSuccess;
  static int l2hint = -1;
  if (l2hint < 0) {
    const char* ev = getenv("WINO_L2_HINTS");
    l2hint = ev ? (atoi(ev) != 0) : 1;
  }
  const long long Ts = T_s;
  return launch_pdl(kern, dim3((unsigned)(2 * pairs)), dim3(tc::kThreadsTS), smem, s, DF ? *df->tmA : tg.tmA_ts, tmBhi16,
                    tmBlo16, Mo, P, (int)t_lo, (int)T, Ts, C, K, nraw, nbr, l2hint, vmax, uscal, zmask, DF ? df->tl2 : 0,
                    DF ? df->cz : 0, DF ? df->S : 1);
}

// Z of the direct-axis fold as (slot, c, plane): box {BM + 4, kc, 1}, no swizzle, zero fill past Tz
cudaError_t f16_encode_z(CUtensorMap* tm, const float* Z, int64_t Tz, int cz, int planes, int kc) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {(cuuint64_t)Tz, (cuuint64_t)cz, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)Tz * 4, (cuuint64_t)Tz * 4 * cz};
  cuuint32_t box[3] = {(cuuint32_t)tc::BM + 4, (cuuint32_t)kc, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(Z), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// The V-resident kernel applies to two 128-wide n-blocks (128 < K <= 256)
// whose converted V block fits next to both accumulators in TMEM (C <= 256).
bool f16n_applies(int C, int K, int kc) {
  const int n_chunks = (C + kc - 1) / kc;
  return K > 128 && K <= 256 && n_chunks * kc + 2 * 128 <= 512 && n_chunks <= 16;
}

cudaError_t launch_gemm_f16(const TcGemm& tg, const CUtensorMap& tmBhi16, const CUtensorMap& tmBlo16, float* Mo,
                            int P, int64_t t_lo, int64_t T, int64_t T_s, int C, int K, const unsigned int* vmax,
                            const float* uscal, cudaStream_t s, int zmask, bool vres, const DFoldGemm* df) {
  if (df) {   // direct-axis fold: the V-resident kernel only (the plan checked f16n_applies)
    if (!f16n_applies(C, K, tg.kc) || df->cz % tg.kc != 0 || t_lo != 0) return cudaErrorNotSupported;
    if (tg.kc == 64) return launch_f16n_kc<64, true>(tg, tmBhi16, tmBlo16, Mo, P, t_lo, T, T_s, C, K, vmax, uscal, zmask, s, df);
    if (tg.kc == 32) return launch_f16n_kc<32, true>(tg, tmBhi16, tmBlo16, Mo, P, t_lo, T, T_s, C, K, vmax, uscal, zmask, s, df);
    return cudaErrorNotSupported;
  }
  if (vres && f16n_applies(C, K, tg.kc)) {
    if (tg.kc == 64) return launch_f16n_kc<64, false>(tg, tmBhi16, tmBlo16, Mo, P, t_lo, T, T_s, C, K, vmax, uscal, zmask, s, nullptr);
    if (tg.kc == 32) return launch_f16n_kc<32, false>(tg, tmBhi16, tmBlo16, Mo, P, t_lo, T, T_s, C, K, vmax, uscal, zmask, s, nullptr);
  }
  if (tg.kc == 64) return launch_f16_kc<64>(tg, tmBhi16, tmBlo16, Mo, P, t_lo, T, T_s, C, K, vmax, uscal, s);
  if (tg.kc == 32) return launch_f16_kc<32>(tg, tmBhi16, tmBlo16, Mo, P, t_lo, T, T_s, C, K, vmax, uscal, s);
  return cudaErrorNotSupported;
}

// ---------------------------------------------------------------- filter split
// U (fp32, computed by the filter transform into `u32`) -> fp16 hi / lo with
// the power-of-two scale 2^-su, su from max|U| (k_absmax); uscal[0] = 2^su.
__global__ void k_absmax(const float* __restrict__ u, int64_t n, unsigned int* __restrict__ mx) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(u[i]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float wm[32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) atomicMax(mx, __float_as_uint(m));
  }
}

__global__ void k_split16(const float* __restrict__ u, int64_t n, const unsigned int* __restrict__ mx,
                          __half* __restrict__ hi, __half* __restrict__ lo, float* __restrict__ uscal) {
  const int su = tc::scale_exp(*mx);
  const float sc = tc::exp2i(-su);
  if (blockIdx.x == 0 && threadIdx.x == 0) *uscal = tc::exp2i(su);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = u[i] * sc;
    const __half h = __float2half_rn(v);
    hi[i] = h;
    lo[i] = __float2half_rn(v - __half2float(h));
  }
}

cudaError_t launch_split16(const float* u32, int64_t n, unsigned int* mx, void* hi, void* lo, float* uscal,
                           cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(mx, 0, 4, s);
  if (e != cudaSuccess) return e;
  k_absmax<<<592, 256, 0, s>>>(u32, n, mx);
  k_split16<<<592, 256, 0, s>>>(u32, n, mx, reinterpret_cast<__half*>(hi), reinterpret_cast<__half*>(lo), uscal);
  return cudaGetLastError();
}

}  // namespace wino
