// gemm_tc.cu -- stage a3 on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// For every transform point xi (Eq. (5)):
//     M_xi[t][k] = sum_c V_xi[t][c] U_xi[c][k]      ([T x C] x [C x K])
// fp32-accurate via 3xTF32 (reading #7):
//     V = V_hi + V_lo,  U = U_hi + U_lo  (hi = rna_tf32(x), lo = rna_tf32(x - hi))
//     M = V_lo U_hi + V_hi U_lo + V_hi U_hi       accumulated in fp32 in TMEM.
//
// One persistent, warp-specialised kernel (352 threads, 1 CTA per SM); a work
// unit is (xi, n-block, m-block) of 128 tiles x BN output channels.
//   warp 8      V producer: TMA of raw V chunks (fp32, 128 t x kc c) into a
//               deep raw ring (MN-major, 128 B rows, SWIZZLE_128B_BASE32B).
//   warps 0-3   converter: raw V chunk -> V_hi, V_lo in the 2-stage operand
//               ring (the tf32 rounding must be explicit: the tensor core
//               would truncate).
//   warp 10     U producer: U_hi / U_lo chunks into the operand ring, or the
//               whole U n-block once into a resident region (kRes).
//   warp 9      MMA issuer (one thread): 3 x (kc/8) tcgen05.mma.kind::tf32
//               M=128 N=BN K=8 per chunk into a double-buffered TMEM
//               accumulator; tcgen05.commit frees operand stages / publishes
//               the accumulator.
//   warps 4-7   epilogue: tcgen05.ld 32x32b.x32 -> registers -> M[xi][k][t]
//               (each warp stores 32 consecutive t per column: 128 B lines).
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "kernels.h"
#include "tc_common.cuh"
#include "tma.hpp"

namespace wino {
namespace tc {

// Work unit u = (xi, n-block, m-block), m-block fastest.  Two shared-memory
// rings decouple HBM latency from the tensor core:
//   raw ring (R stages):  V chunk [kc c][128 t] fp32, straight from TMA;
//                         deep, so >= ~50 KB of V loads stay in flight;
//   op ring  (H stages):  the MMA operands of one chunk: V_hi, V_lo (written
//                         by the converter warps) and, when U is streamed,
//                         the U_hi / U_lo chunk (TMA by the B producer).
// kRes (U-resident): CTA i owns the contiguous unit range [i U/G, (i+1) U/G)
//   and keeps the whole U_xi n-block (hi and lo, all C) in shared memory,
//   reloading it when (xi, n-block) changes.  !kRes: U chunks ride in the op
//   ring.  Warps: 0-3 converter, 4-7 epilogue, 8 V producer, 9 MMA issuer,
//   10 U producer.
template <int BN, bool kRes>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
          const __grid_constant__ CUtensorMap tmBlo, float* __restrict__ Mo, int P, int t_lo, int T, long long T_s,
          int C, int K, int kc, int three, int nraw, int nop, int nbr, int l2hint) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (sraw & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  const uint32_t sbase = sraw + pad;
  const int n_chunks = (C + kc - 1) / kc;
  const uint32_t a_bytes = (uint32_t)BM * kc * 4;   // one V chunk (raw, hi or lo)
  const uint32_t b_bytes = (uint32_t)BN * kc * 4;   // one U chunk (hi or lo)
  const uint32_t op_bytes = 2 * a_bytes;
  const uint32_t raw0 = sbase;
  const uint32_t op0 = raw0 + nraw * a_bytes;
  // U: the resident block (hi chunks then lo chunks), or a ring of nbr
  // stages each holding one chunk's U_hi and U_lo
  const uint32_t bres = op0 + nop * op_bytes;
  const uint32_t bres_bytes = kRes ? 2u * n_chunks * b_bytes : 2u * nbr * b_bytes;
  const uint32_t bar0 = bres + bres_bytes;                          // 8-byte barriers
  auto rfull = [&](int s) { return bar0 + 8u * s; };
  auto rempty = [&](int s) { return bar0 + 8u * (nraw + s); };
  auto ofull = [&](int s) { return bar0 + 8u * (2 * nraw + s); };
  auto oempty = [&](int s) { return bar0 + 8u * (2 * nraw + nop + s); };
  auto ufull = [&](int s) { return bar0 + 8u * (2 * nraw + 2 * nop + s); };
  auto uempty = [&](int s) { return bar0 + 8u * (2 * nraw + 2 * nop + nbr + s); };
  const uint32_t bar1 = bar0 + 8u * (2 * nraw + 2 * nop + 2 * nbr);
  auto tfull = [&](int a) { return bar1 + 8u * a; };
  auto tempty = [&](int a) { return bar1 + 8u * (2 + a); };
  const uint32_t bfull = bar1 + 32u;
  const uint32_t bempty = bar1 + 40u;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + (bar1 - sbase) + 48);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kCols = tmem_cols(BN);

  if (warp == 9) {
    if (lane == 0) {
      for (int s = 0; s < nraw; ++s) {
        mbar_init(rfull(s), 1);
        mbar_init(rempty(s), 1);
      }
      for (int s = 0; s < nop; ++s) {
        mbar_init(ofull(s), 1);
        mbar_init(oempty(s), 1);
      }
      for (int s = 0; s < nbr; ++s) {
        mbar_init(ufull(s), 1);
        mbar_init(uempty(s), 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(tfull(a), 1);
        mbar_init(tempty(a), 128);
      }
      mbar_init(bfull, 1);
      mbar_init(bempty, 1);
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
  pdl_wait();      // V comes from the input transform; M is read by the previous output transform
  pdl_trigger();

  const int n_mblk = (T - t_lo + BM - 1) / BM;
  const int n_nblk = (K + BN - 1) / BN;
  const long long per_xi = (long long)n_nblk * n_mblk;
  const long long total = (long long)P * per_xi;
  // this CTA's units: [u_beg, u_end) step u_step
  long long u_beg, u_end, u_step;
  if constexpr (kRes) {
    u_beg = total * blockIdx.x / gridDim.x;
    u_end = total * (blockIdx.x + 1) / gridDim.x;
    u_step = 1;
  } else {
    u_beg = blockIdx.x;
    u_end = total;
    u_step = gridDim.x;
  }

  if (warp == 8) {
    if (lane == 0) {  // ---------------- V producer (raw ring)
      int s = 0;
      uint32_t ph = 0;
      for (long long u = u_beg; u < u_end; u += u_step) {
        const int xi = (int)(u / per_xi);
        const int mb = (int)(u % per_xi) % n_mblk;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(rempty(s), ph ^ 1u);
          const uint32_t st = raw0 + s * a_bytes;
          mbar_expect_tx(rfull(s), a_bytes);
#pragma unroll
          for (int gq = 0; gq < BM / 32; ++gq)
            if (l2hint)
              tma_load_3d_hint(st + gq * kc * 128, &tmA, t_lo + mb * BM + gq * 32, ch * kc, xi, rfull(s),
                               l2_policy(false));
            else
              tma_load_3d(st + gq * kc * 128, &tmA, t_lo + mb * BM + gq * 32, ch * kc, xi, rfull(s));
          if (++s == nraw) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {  // ---------------- U producer
      if constexpr (kRes) {
        long long cur_pair = -1;
        int nload = 0;
        for (long long u = u_beg; u < u_end; ++u) {
          const long long pair = u / n_mblk;
          if (pair == cur_pair) continue;
          const int xi = (int)(u / per_xi);
          const int nb = (int)(u % per_xi) / n_mblk;
          if (nload > 0) mbar_wait(bempty, (uint32_t)((nload - 1) & 1));
          mbar_expect_tx(bfull, (three ? 2u : 1u) * n_chunks * b_bytes);
          for (int ch = 0; ch < n_chunks; ++ch)
#pragma unroll
            for (int gq = 0; gq < BN / 32; ++gq) {
              tma_load_3d(bres + ch * b_bytes + gq * kc * 128, &tmBhi, nb * BN + gq * 32, ch * kc, xi, bfull);
              if (three)
                tma_load_3d(bres + (n_chunks + ch) * b_bytes + gq * kc * 128, &tmBlo, nb * BN + gq * 32, ch * kc, xi,
                            bfull);
            }
          cur_pair = pair;
          ++nload;
        }
      } else {
        int s = 0;
        uint32_t ph = 0;
        for (long long u = u_beg; u < u_end; u += u_step) {
          const int xi = (int)(u / per_xi);
          const int nb = (int)(u % per_xi) / n_mblk;
          for (int ch = 0; ch < n_chunks; ++ch) {
            mbar_wait(uempty(s), ph ^ 1u);
            const uint32_t st = bres + s * 2 * b_bytes;
            mbar_expect_tx(ufull(s), (three ? 2u : 1u) * b_bytes);
#pragma unroll
            for (int gq = 0; gq < BN / 32; ++gq) {
              tma_load_3d(st + gq * kc * 128, &tmBhi, nb * BN + gq * 32, ch * kc, xi, ufull(s));
              if (three) tma_load_3d(st + b_bytes + gq * kc * 128, &tmBlo, nb * BN + gq * 32, ch * kc, xi, ufull(s));
            }
            if (++s == nbr) { s = 0; ph ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 9) {
    {  // ---------------- MMA issuer (warp-uniform loop, elected lane issues)
      constexpr uint32_t idesc = idesc_tf32<BN>();
      const uint32_t lbo = (uint32_t)kc * 128u;
      int s = 0, us = 0;
      uint32_t ph = 0, uph = 0, acc = 0, aph = 0;
      long long cur_pair = -1;
      int nload = 0;
      for (long long u = u_beg; u < u_end; u += u_step) {
        if constexpr (kRes) {
          const long long pair = u / n_mblk;
          if (pair != cur_pair) {
            mbar_wait(bfull, (uint32_t)(nload & 1));
            tc_fence_after();
            cur_pair = pair;
            ++nload;
          }
        }
        mbar_wait(tempty(acc), aph ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(ofull(s), ph);
          if constexpr (!kRes) mbar_wait(ufull(us), uph);
          tc_fence_after();
          const uint32_t st = op0 + s * op_bytes;
          const uint32_t b_hi = kRes ? bres + ch * b_bytes : bres + us * 2 * b_bytes;
          const uint32_t b_lo = kRes ? bres + (n_chunks + ch) * b_bytes : b_hi + b_bytes;
          // descriptors of k-step 0; k-step j is +j*1024 B = +64 in the address field
          const uint64_t dah = sdesc(st, lbo, 512u), dal = sdesc(st + a_bytes, lbo, 512u);
          const uint64_t dbh = sdesc(b_hi, lbo, 512u), dbl = sdesc(b_lo, lbo, 512u);
          const int nk = kc / 8;
          if (elect_one()) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // kc <= 64: at most 8 K=8 steps
              if (j < nk) {
                const uint32_t accum = (ch | j) != 0;
                const uint64_t o = 64ull * j;
                if (three) {
                  tc_mma_tf32(d, dal + o, dbh + o, idesc, accum);
                  tc_mma_tf32(d, dah + o, dbl + o, idesc, 1u);
                  tc_mma_tf32(d, dah + o, dbh + o, idesc, 1u);
                } else {
                  tc_mma_tf32(d, dah + o, dbh + o, idesc, accum);
                }
              }
            }
            tc_commit(oempty(s));
            if constexpr (!kRes) tc_commit(uempty(us));
          }
          __syncwarp();
          if (++s == nop) { s = 0; ph ^= 1u; }
          if constexpr (!kRes) {
            if (++us == nbr) { us = 0; uph ^= 1u; }
          }
        }
        if (elect_one()) {
          tc_commit(tfull(acc));
          // release the resident U block after its last unit
          if constexpr (kRes) {
            if (u + 1 >= u_end || (u + 1) / n_mblk != cur_pair) tc_commit(bempty);
          }
        }
        __syncwarp();
        acc ^= 1u;
        if (acc == 0) aph ^= 1u;
      }
    }
  } else if (warp < 4) {  // ---------------- converter (128 threads): raw -> hi, lo
    int rs = 0, os = 0;
    uint32_t rph = 0, oph = 0;
    const int n4 = (int)(a_bytes / 16);
    for (long long u = u_beg; u < u_end; u += u_step) {
      for (int ch = 0; ch < n_chunks; ++ch) {
        mbar_wait(rfull(rs), rph);
        mbar_wait(oempty(os), oph ^ 1u);
        const float4* araw = reinterpret_cast<const float4*>(smem + rs * a_bytes);
        float4* ahi = reinterpret_cast<float4*>(smem + (op0 - sbase) + os * op_bytes);
        float4* alo = reinterpret_cast<float4*>(smem + (op0 - sbase) + os * op_bytes + a_bytes);
#pragma unroll 4
        for (int i = threadIdx.x; i < n4; i += 128) {
          const float4 v = araw[i];
          float4 h, l;
          h.x = tf32_rna(v.x); h.y = tf32_rna(v.y); h.z = tf32_rna(v.z); h.w = tf32_rna(v.w);
          ahi[i] = h;
          if (three) {
            l.x = tf32_rna(v.x - h.x); l.y = tf32_rna(v.y - h.y);
            l.z = tf32_rna(v.z - h.z); l.w = tf32_rna(v.w - h.w);
            alo[i] = l;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 0) {
          mbar_arrive(rempty(rs));
          mbar_arrive(ofull(os));
        }
        if (++rs == nraw) { rs = 0; rph ^= 1u; }
        if (++os == nop) { os = 0; oph ^= 1u; }
      }
    }
  } else if (warp < 8) {  // warps 4-7 ------------------ epilogue
    const int q = warp - 4;
    const uint64_t pol = l2_policy(true);
    uint32_t acc = 0, aph = 0;
    for (long long u = u_beg; u < u_end; u += u_step) {
      const int xi = (int)(u / per_xi);
      const int rr = (int)(u % per_xi);
      const int nb = rr / n_mblk, mb = rr % n_mblk;
      mbar_wait(tfull(acc), aph);
      tc_fence_after();
      const int t = t_lo + mb * BM + q * 32 + lane;
      // M[xi][k][t]: this lane's column t, rows k = nb*BN + j (stride T_s)
      float* out = Mo + ((long long)xi * K + (long long)nb * BN) * T_s + t;
      const bool full_n = (nb + 1) * BN <= K;
#pragma unroll 1
      for (int cb = 0; cb < BN / 32; ++cb) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + cb * 32, r);
        if (t < T) {
          float* p = out + (long long)cb * 32 * T_s;
          // M stays in L2 for a4 (evict-last policy)
          store_m32<false>(p, r, T_s, full_n ? 32 : K - nb * BN - cb * 32, l2hint, pol, 1.f);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty(acc));
      acc ^= 1u;
      if (acc == 0) aph ^= 1u;
    }
  }
  __syncthreads();
  if (warp == 9) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kCols) : "memory");
  }
}


// TS-mode GEMM.  Same units, U handling (resident or ring) and epilogue as
// k_gemm_tc, but:
//   raw ring:   V chunk [kc c][128 t] fp32, TMA box {128, kc} without swizzle;
//   converter:  thread = tile row t (warp q owns TMEM lanes 32q..32q+31):
//               reads its kc raw values (conflict-free 4-byte LDS), splits
//               hi/lo in registers and writes them with tcgen05.st into one of
//               two TMEM A stages (columns a0 + s*2kc: hi, +kc: lo);
//   MMA:        tcgen05.mma ... [d], [a_tmem], b_desc (A from TMEM).
// TMEM columns: 2*BN accumulators + 4*kc A stages.
template <int BN, bool kRes>
__global__ void __launch_bounds__(kThreadsTS, 1)
k_gemm_ts(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
          const __grid_constant__ CUtensorMap tmBlo, float* __restrict__ Mo, int P, int t_lo, int T, long long T_s,
          int C, int K, int kc, int three, int nraw, int nbr, int dbg, int l2hint) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (sraw & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  const uint32_t sbase = sraw + pad;
  const int n_chunks = (C + kc - 1) / kc;
  const uint32_t a_bytes = (uint32_t)BM * kc * 4;
  const uint32_t b_bytes = (uint32_t)BN * kc * 4;
  const uint32_t raw0 = sbase;
  const uint32_t bres = raw0 + nraw * a_bytes;
  const uint32_t bres_bytes = kRes ? 2u * n_chunks * b_bytes : 2u * nbr * b_bytes;
  const uint32_t bar0 = bres + bres_bytes;
  auto rfull = [&](int s) { return bar0 + 8u * s; };
  auto rempty = [&](int s) { return bar0 + 8u * (nraw + s); };
  auto ufull = [&](int s) { return bar0 + 8u * (2 * nraw + s); };
  auto uempty = [&](int s) { return bar0 + 8u * (2 * nraw + nbr + s); };
  const uint32_t bar1 = bar0 + 8u * (2 * nraw + 2 * nbr);
  auto tfull = [&](int a) { return bar1 + 8u * a; };
  auto tempty = [&](int a) { return bar1 + 8u * (2 + a); };
  auto afull = [&](int a) { return bar1 + 8u * (4 + a); };   // a < 4
  auto aempty = [&](int a) { return bar1 + 8u * (8 + a); };
  const uint32_t bfull = bar1 + 96u;   // after afull(0..3) at +32, aempty(0..3) at +64
  const uint32_t bempty = bar1 + 104u;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + (bar1 - sbase) + 112);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // TMEM: 2 accumulators + na A stages (V_hi | V_lo), na in [2, 4]
  int na = (512 - 2 * BN) / (2 * kc);
  na = na > 4 ? 4 : na;
  const uint32_t kCols = pow2_cols(2 * BN + 2 * kc * na);
  const uint32_t a_col0 = 2 * BN;

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
      for (int a = 0; a < 2; ++a) {
        mbar_init(tfull(a), 1);
        mbar_init(tempty(a), 128);
      }
      for (int a = 0; a < na; ++a) {
        mbar_init(afull(a), 256);
        mbar_init(aempty(a), 1);
      }
      mbar_init(bfull, 1);
      mbar_init(bempty, 1);
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
  pdl_wait();      // V comes from the input transform; M is read by the previous output transform
  pdl_trigger();

  const int n_mblk = (T - t_lo + BM - 1) / BM;
  const int n_nblk = (K + BN - 1) / BN;
  const long long per_xi = (long long)n_nblk * n_mblk;
  const long long total = (long long)P * per_xi;
  long long u_beg, u_end, u_step;
  if constexpr (kRes) {
    u_beg = total * blockIdx.x / gridDim.x;
    u_end = total * (blockIdx.x + 1) / gridDim.x;
    u_step = 1;
  } else {
    u_beg = blockIdx.x;
    u_end = total;
    u_step = gridDim.x;
  }

  if (warp == 8) {
    if (lane == 0) {  // ---------------- V producer (raw ring, one box per chunk)
      int s = 0;
      uint32_t ph = 0;
      for (long long u = u_beg; u < u_end; u += u_step) {
        const int xi = (int)(u / per_xi);
        const int mb = (int)(u % per_xi) % n_mblk;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(rempty(s), ph ^ 1u);
          if (dbg & 16) {
            mbar_arrive(rfull(s));  // dev knob: no V loads
          } else {
            mbar_expect_tx(rfull(s), a_bytes);
            if (l2hint)
              tma_load_3d_hint(raw0 + s * a_bytes, &tmA, t_lo + mb * BM, ch * kc, xi, rfull(s), l2_policy(false));
            else
              tma_load_3d(raw0 + s * a_bytes, &tmA, t_lo + mb * BM, ch * kc, xi, rfull(s));
          }
          if (++s == nraw) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {  // ---------------- U producer
      if constexpr (kRes) {
        long long cur_pair = -1;
        int nload = 0;
        for (long long u = u_beg; u < u_end; ++u) {
          const long long pair = u / n_mblk;
          if (pair == cur_pair) continue;
          const int xi = (int)(u / per_xi);
          const int nb = (int)(u % per_xi) / n_mblk;
          if (nload > 0) mbar_wait(bempty, (uint32_t)((nload - 1) & 1));
          mbar_expect_tx(bfull, (three ? 2u : 1u) * n_chunks * b_bytes);
          for (int ch = 0; ch < n_chunks; ++ch)
#pragma unroll
            for (int gq = 0; gq < BN / 32; ++gq) {
              tma_load_3d(bres + ch * b_bytes + gq * kc * 128, &tmBhi, nb * BN + gq * 32, ch * kc, xi, bfull);
              if (three)
                tma_load_3d(bres + (n_chunks + ch) * b_bytes + gq * kc * 128, &tmBlo, nb * BN + gq * 32, ch * kc, xi,
                            bfull);
            }
          cur_pair = pair;
          ++nload;
        }
      } else {
        int s = 0;
        uint32_t ph = 0;
        for (long long u = u_beg; u < u_end; u += u_step) {
          const int xi = (int)(u / per_xi);
          const int nb = (int)(u % per_xi) / n_mblk;
          for (int ch = 0; ch < n_chunks; ++ch) {
            mbar_wait(uempty(s), ph ^ 1u);
            const uint32_t st = bres + s * 2 * b_bytes;
            if (dbg & 8) {  // dev knob: no U loads
              mbar_arrive(ufull(s));
              if (++s == nbr) { s = 0; ph ^= 1u; }
              continue;
            }
            mbar_expect_tx(ufull(s), (three ? 2u : 1u) * b_bytes);
#pragma unroll
            for (int gq = 0; gq < BN / 32; ++gq) {
              tma_load_3d(st + gq * kc * 128, &tmBhi, nb * BN + gq * 32, ch * kc, xi, ufull(s));
              if (three) tma_load_3d(st + b_bytes + gq * kc * 128, &tmBlo, nb * BN + gq * 32, ch * kc, xi, ufull(s));
            }
            if (++s == nbr) { s = 0; ph ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 9) {
    {  // ---------------- MMA issuer (warp-uniform loop, elected lane issues)
      constexpr uint32_t idesc = idesc_tf32_ts<BN>();
      const int nk = (dbg & 4) ? 0 : kc / 8;
      const uint32_t lbo = (uint32_t)kc * 128u;
      int as = 0, us = 0;
      uint32_t aph = 0, uph = 0, acc = 0, cph = 0;
      long long cur_pair = -1;
      int nload = 0;
      for (long long u = u_beg; u < u_end; u += u_step) {
        if constexpr (kRes) {
          const long long pair = u / n_mblk;
          if (pair != cur_pair) {
            mbar_wait(bfull, (uint32_t)(nload & 1));
            tc_fence_after();
            cur_pair = pair;
            ++nload;
          }
        }
        mbar_wait(tempty(acc), cph ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(afull(as), aph);
          if constexpr (!kRes) mbar_wait(ufull(us), uph);
          tc_fence_after();
          const uint32_t b_hi = kRes ? bres + ch * b_bytes : bres + us * 2 * b_bytes;
          const uint32_t b_lo = kRes ? bres + (n_chunks + ch) * b_bytes : b_hi + b_bytes;
          uint64_t dbh = sdesc(b_hi, lbo, 512u), dbl = sdesc(b_lo, lbo, 512u);
          const uint32_t a_hi = tmem_base + a_col0 + as * 2 * kc, a_lo = a_hi + kc;
          if (elect_one()) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // kc <= 64: at most 8 K=8 steps
              if (j < nk) {
                const uint32_t accum = (ch | j) != 0;
                if (three) {
                  tc_mma_tf32_ts(d, a_lo + 8 * j, dbh + 64 * j, idesc, accum);
                  tc_mma_tf32_ts(d, a_hi + 8 * j, dbl + 64 * j, idesc, 1u);
                  tc_mma_tf32_ts(d, a_hi + 8 * j, dbh + 64 * j, idesc, 1u);
                } else {
                  tc_mma_tf32_ts(d, a_hi + 8 * j, dbh + 64 * j, idesc, accum);
                }
              }
            }
            tc_commit(aempty(as));
            if constexpr (!kRes) tc_commit(uempty(us));
          }
          __syncwarp();
          if (++as == na) { as = 0; aph ^= 1u; }
          if constexpr (!kRes) {
            if (++us == nbr) { us = 0; uph ^= 1u; }
          }
        }
        if (elect_one()) {
          tc_commit(tfull(acc));
          if constexpr (kRes) {
            if (u + 1 >= u_end || (u + 1) / n_mblk != cur_pair) tc_commit(bempty);
          }
        }
        __syncwarp();
        acc ^= 1u;
        if (acc == 0) cph ^= 1u;
      }
    }
  } else if (warp < 4 || (warp >= 11 && warp < 15)) {  // ---- converter (8 warps): raw V row -> TMEM hi / lo
    // warps w and w' with w % 4 == w' % 4 own TMEM lane quarter w % 4; the
    // second group (warps 11-14) converts the upper half of each chunk's channels
    const int q = warp & 3, grp = warp < 4 ? 0 : 1;
    const int row = q * 32 + lane;
    const uint32_t lane_sel = (uint32_t)(q * 32) << 16;
    const int cg0 = grp * (kc / 8) / 2, cg1 = (grp + 1) * (kc / 8) / 2;
    int rs = 0, as = 0;
    uint32_t rph = 0, aph = 0;
    for (long long u = u_beg; u < u_end; u += u_step) {
      for (int ch = 0; ch < n_chunks; ++ch) {
        mbar_wait(rfull(rs), rph);
        mbar_wait(aempty(as), aph ^ 1u);
        tc_fence_after();
        const float* raw = reinterpret_cast<const float*>(smem + rs * a_bytes) + row;
        const uint32_t ahi = tmem_base + lane_sel + a_col0 + as * 2 * kc;
        for (int cg = cg0; cg < ((dbg & 2) ? cg0 : cg1); ++cg) {
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float v = raw[(cg * 8 + j) * BM];
            const uint32_t h = tf32_rna_bits(__float_as_uint(v));
            hi[j] = h;
            lo[j] = tf32_rna_bits(__float_as_uint(v - __uint_as_float(h)));
          }
          tmem_st8(ahi + cg * 8, hi);
          if (three) tmem_st8(ahi + kc + cg * 8, lo);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(rempty(rs));
        mbar_arrive(afull(as));
        if (++rs == nraw) { rs = 0; rph ^= 1u; }
        if (++as == na) { as = 0; aph ^= 1u; }
      }
    }
  } else if (warp < 8) {  // warps 4-7 ------------------ epilogue
    const int q = warp - 4;
    const uint64_t pol = l2_policy(true);
    uint32_t acc = 0, aph = 0;
    for (long long u = u_beg; u < u_end; u += u_step) {
      const int xi = (int)(u / per_xi);
      const int rr = (int)(u % per_xi);
      const int nb = rr / n_mblk, mb = rr % n_mblk;
      mbar_wait(tfull(acc), aph);
      tc_fence_after();
      const int t = t_lo + mb * BM + q * 32 + lane;
      float* out = Mo + ((long long)xi * K + (long long)nb * BN) * T_s + t;
      const bool full_n = (nb + 1) * BN <= K;
#pragma unroll 1
      for (int cb = 0; cb < BN / 32; ++cb) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + cb * 32, r);
        if (t < T && !(dbg & 1)) {
          float* p = out + (long long)cb * 32 * T_s;
          // M stays in L2 for a4 (evict-last policy)
          store_m32<false>(p, r, T_s, full_n ? 32 : K - nb * BN - cb * 32, l2hint, pol, 1.f);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty(acc));
      acc ^= 1u;
      if (acc == 0) aph ^= 1u;
    }
  }
  __syncthreads();
  if (warp == 9) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kCols) : "memory");
  }
}

}  // namespace tc

// ---------------------------------------------------------------- host side
// 3-D view (inner, c, xi) of a [P][C][inner_s] fp32 array; box {32, kc, 1}.
static cudaError_t encode3d(CUtensorMap* tm, const float* base, int64_t inner_s, int C, int P, int kc) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {(cuuint64_t)inner_s, (cuuint64_t)C, (cuuint64_t)P};
  cuuint64_t strides[2] = {(cuuint64_t)inner_s * 4, (cuuint64_t)inner_s * 4 * C};
  cuuint32_t box[3] = {32, (cuuint32_t)kc, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static int pick_bn(int K) {
  if (K <= 32) return 32;
  if (K <= 64) return 64;
  if (K <= 128) return 128;
  return 256;
}

// Shared-memory plan of one launch: raw ring depth, op ring depth, bytes.
// Resident mode keeps the whole U n-block (hi + lo) beside the two rings.
struct TcSmem {
  int nraw, nop, nbr;
  size_t bytes;
};
// Rings: raw V (nraw x 128*kc*4), operands V_hi/V_lo (nop = 2), and U either
// resident (all chunks) or a ring of nbr chunk stages (U_hi + U_lo).  Depth
// goes first to U (its L2 latency must hide behind <= nbr chunk MMAs), then
// to the raw V ring.
static TcSmem tc_smem(int bn, int kc, int C, bool res) {
  const int n_chunks = (C + kc - 1) / kc;
  const size_t a = (size_t)tc::BM * kc * 4;
  const size_t b2 = 2ull * bn * kc * 4;
  const size_t fixed = 1024 + 1024;
  const size_t budget = 232448;
  TcSmem t{0, 2, 0, 0};
  size_t left = budget - fixed - 2 * (2 * a);
  if (res) {
    const size_t bres = (size_t)n_chunks * b2;
    if (bres + a > left) return t;
    left -= bres;
  } else {
    int nbr = 3;
    while (nbr > 1 && nbr * b2 + 2 * a > left) --nbr;
    if (nbr * b2 + a > left) return t;
    t.nbr = nbr;
    left -= nbr * b2;
  }
  int nraw = (int)(left / a);
  if (nraw > 8) nraw = 8;
  if (const char* ev = getenv("WINO_GEMM_NRAW")) nraw = nraw < atoi(ev) ? nraw : atoi(ev);  // dev knob
  t.nraw = nraw;
  t.bytes = budget - (left - nraw * a);
  return t;
}

// TS-mode shared memory: raw V ring + U (resident or ring).
static TcSmem ts_smem(int bn, int kc, int C, bool res) {
  const int n_chunks = (C + kc - 1) / kc;
  const size_t a = (size_t)tc::BM * kc * 4;
  const size_t b2 = 2ull * bn * kc * 4;
  const size_t fixed = 1024 + 1024;
  const size_t budget = 232448;
  TcSmem t{0, 0, 0, 0};
  size_t left = budget - fixed;
  if (res) {
    const size_t bres = (size_t)n_chunks * b2;
    if (bres + 2 * a > left) return t;
    left -= bres;
  } else {
    int nbr = 4;
    if (const char* ev = getenv("WINO_GEMM_NBR")) nbr = atoi(ev);  // dev knob
    while (nbr > 1 && nbr * b2 + 3 * a > left) --nbr;
    if (nbr * b2 + 2 * a > left) return t;
    t.nbr = nbr;
    left -= nbr * b2;
  }
  int nraw = (int)(left / a);
  if (nraw > 8) nraw = 8;
  if (const char* ev = getenv("WINO_GEMM_NRAW")) nraw = nraw < atoi(ev) ? nraw : atoi(ev);  // dev knob
  t.nraw = nraw;
  t.bytes = budget - (left - nraw * a);
  return t;
}

template <int BN>
static cudaError_t set_attr(size_t smem, bool res, bool ts) {
  const cudaFuncAttribute at = cudaFuncAttributeMaxDynamicSharedMemorySize;
  if (ts) return res ? cudaFuncSetAttribute(tc::k_gemm_ts<BN, true>, at, (int)smem)
                     : cudaFuncSetAttribute(tc::k_gemm_ts<BN, false>, at, (int)smem);
  return res ? cudaFuncSetAttribute(tc::k_gemm_tc<BN, true>, at, (int)smem)
             : cudaFuncSetAttribute(tc::k_gemm_tc<BN, false>, at, (int)smem);
}

// V tensor map of the TS raw ring: box {128 t, kc c, 1}, no swizzle.
static cudaError_t encode_v_ts(CUtensorMap* tm, const float* base, int64_t T_s, int C, int P, int kc) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {(cuuint64_t)T_s, (cuuint64_t)C, (cuuint64_t)P};
  cuuint64_t strides[2] = {(cuuint64_t)T_s * 4, (cuuint64_t)T_s * 4 * C};
  cuuint32_t box[3] = {(cuuint32_t)tc::BM, (cuuint32_t)kc, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static TcSmem plan_smem(const TcGemm& tg, int C) {
  return tg.variant == kGemmTS ? ts_smem(tg.bn, tg.kc, C, tg.resident) : tc_smem(tg.bn, tg.kc, C, tg.resident);
}

// Capabilities and shared-memory attributes for N tile `bn` (tg.kc, tg.resident set).
static cudaError_t prep_bn(TcGemm& tg, int bn, int C) {
  tg.bn = bn;
  // TS mode (A in TMEM) when the accumulators and two A stages fit in TMEM;
  // CTA pairs (cta_group::2) on top of TS
  tg.can_ts = 2 * bn + 4 * tg.kc <= 512;
  tg.can_pair = tg.can_ts && ts2_supported(bn, tg.kc);
  cudaError_t e = cudaSuccess;
  for (int ts = 0; ts <= (tg.can_ts ? 1 : 0); ++ts) {
    const TcSmem sm = ts ? ts_smem(bn, tg.kc, C, tg.resident) : tc_smem(bn, tg.kc, C, tg.resident);
    if (sm.nraw < 1) {
      if (!ts) return cudaErrorInvalidConfiguration;
      tg.can_ts = tg.can_pair = false;
      break;
    }
    switch (bn) {
      case 32: e = set_attr<32>(sm.bytes, tg.resident, ts); break;
      case 64: e = set_attr<64>(sm.bytes, tg.resident, ts); break;
      case 128: e = set_attr<128>(sm.bytes, tg.resident, ts); break;
      default: e = set_attr<256>(sm.bytes, tg.resident, ts); break;
    }
    if (e != cudaSuccess) return e;
  }
  tg.variant = tg.can_ts ? kGemmTS : kGemmSS;
  return cudaSuccess;
}

cudaError_t tc_gemm_prepare(TcGemm& tg, const float* V, const float* Uhi, const float* Ulo, int P, int64_t T_s,
                            int C, int K_s, int K, int three, int device) {
  tg.ready = false;
  tg.bn_max = pick_bn(K);
  // k-chunk: 32 channels; 64 for C >= 256 (half the chunk handshakes: c4
  // 0.789 -> 0.753 ms; at C = 128 the bigger rings leave no shared memory for
  // the neighbouring kernels and the step gets slower, c2 0.102 -> 0.105 ms)
  tg.kc = C >= 256 ? 64 : C >= 32 ? 32 : ((C + 7) / 8) * 8;
  if (const char* ev = getenv("WINO_GEMM_KC")) tg.kc = atoi(ev);  // dev knob (8, 16, 32, 64)
  tg.three = three;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  tg.num_sms = sms;
  // U streamed through its ring by default: the grid-strided unit order keeps
  // the CTAs on neighbouring m-blocks (DRAM locality), measured faster than
  // the U-resident contiguous ranges; WINO_GEMM_RES=1 selects U-resident
  tg.resident = false;
  if (const char* ev = getenv("WINO_GEMM_RES")) {
    const int bn = tg.bn_max;
    const bool ts = 2 * bn + 4 * tg.kc <= 512;
    tg.resident = atoi(ev) != 0 && (ts ? ts_smem(bn, tg.kc, C, true) : tc_smem(bn, tg.kc, C, true)).nraw >= 4;
  }
  tg.dbg = 0;  // dev-only experiment knob: 1 no M stores, 2 no V split, 4 no MMAs (results invalid)
  if (const char* ev = getenv("WINO_GEMM_DBG")) tg.dbg = atoi(ev);
  cudaError_t e;
  if ((e = encode3d(&tg.tmA, V, T_s, C, P, tg.kc)) != cudaSuccess) return e;
  if ((e = encode_v_ts(&tg.tmA_ts, V, T_s, C, P, tg.kc)) != cudaSuccess) return e;
  if ((e = encode3d(&tg.tmBhi, Uhi, K_s, C, P, tg.kc)) != cudaSuccess) return e;
  if ((e = encode3d(&tg.tmBlo, Ulo ? Ulo : Uhi, K_s, C, P, tg.kc)) != cudaSuccess) return e;
  int bn = tg.bn_max;
  if (const char* ev = getenv("WINO_GEMM_BN")) {  // dev knob: smaller N tile (divides K_s)
    const int b = atoi(ev);
    if ((b == 32 || b == 64 || b == 128) && b < bn) bn = b;
  }
  if ((e = prep_bn(tg, bn, C)) != cudaSuccess) {
    // a 256-wide N tile does not fit the rings at this k-chunk: 128 only
    if (bn <= 128) return e;
    cudaGetLastError();
    tg.bn_max = bn = 128;
    if ((e = prep_bn(tg, bn, C)) != cudaSuccess) return e;
  }
  tg.ready = true;
  return cudaSuccess;
}

// L2 policies in the GEMMs (V evict-first, M evict-last); WINO_L2_HINTS=0 disables
static int gemm_l2hint() {
  static int h = -1;
  if (h < 0) {
    const char* ev = getenv("WINO_L2_HINTS");
    h = ev ? (atoi(ev) != 0) : 1;
  }
  return h;
}

template <int BN>
static cudaError_t launch_bn(const TcGemm& tg, int grid, const TcSmem& sm, cudaStream_t s, float* Mo, int P,
                             int t_lo, int T, int64_t T_s, int C, int K) {
  const dim3 gd(grid), bd(tc::kThreads), bdts(tc::kThreadsTS);
  const long long Ts = T_s;
  if (tg.variant == kGemmTS) {
    if (tg.resident)
      return launch_pdl(tc::k_gemm_ts<BN, true>, gd, bdts, sm.bytes, s, tg.tmA_ts, tg.tmBhi, tg.tmBlo, Mo, P, t_lo, T, Ts,
                        C, K, tg.kc, tg.three, sm.nraw, sm.nbr, tg.dbg, gemm_l2hint());
    return launch_pdl(tc::k_gemm_ts<BN, false>, gd, bdts, sm.bytes, s, tg.tmA_ts, tg.tmBhi, tg.tmBlo, Mo, P, t_lo, T, Ts,
                      C, K, tg.kc, tg.three, sm.nraw, sm.nbr, tg.dbg, gemm_l2hint());
  }
  if (tg.resident)
    return launch_pdl(tc::k_gemm_tc<BN, true>, gd, bd, sm.bytes, s, tg.tmA, tg.tmBhi, tg.tmBlo, Mo, P, t_lo, T, Ts,
                      C, K, tg.kc, tg.three, sm.nraw, sm.nop, sm.nbr, gemm_l2hint());
  return launch_pdl(tc::k_gemm_tc<BN, false>, gd, bd, sm.bytes, s, tg.tmA, tg.tmBhi, tg.tmBlo, Mo, P, t_lo, T, Ts,
                    C, K, tg.kc, tg.three, sm.nraw, sm.nop, sm.nbr, gemm_l2hint());
}

cudaError_t launch_gemm_tc(const TcGemm& tg, float* Mo, int P, int64_t t_lo, int64_t T, int64_t T_s, int C, int K,
                           cudaStream_t s) {
  if (!tg.ready) return cudaErrorNotReady;
  if (tg.variant == kGemmPair) return launch_gemm_ts2(tg, Mo, P, t_lo, T, T_s, C, K, s);
  const TcSmem sm = plan_smem(tg, C);
  const long long units = (long long)P * ((K + tg.bn - 1) / tg.bn) * ((T - t_lo + tc::BM - 1) / tc::BM);
  const int grid = (int)(units < tg.num_sms ? units : tg.num_sms);
  if (grid <= 0) return cudaSuccess;
  switch (tg.bn) {
    case 32: return launch_bn<32>(tg, grid, sm, s, Mo, P, (int)t_lo, (int)T, T_s, C, K);
    case 64: return launch_bn<64>(tg, grid, sm, s, Mo, P, (int)t_lo, (int)T, T_s, C, K);
    case 128: return launch_bn<128>(tg, grid, sm, s, Mo, P, (int)t_lo, (int)T, T_s, C, K);
    default: return launch_bn<256>(tg, grid, sm, s, Mo, P, (int)t_lo, (int)T, T_s, C, K);
  }
}

// Process-wide cache of tuning results, keyed by device and problem shape:
// a second plan of the same shape (tests, multi-layer nets, re-planning)
// takes the earlier choice without launching anything.
namespace {
struct TuneKey {
  int dev, P, C, K, three, kc;
  int64_t T, T_s;
  bool operator==(const TuneKey& o) const {
    return dev == o.dev && P == o.P && C == o.C && K == o.K && three == o.three && kc == o.kc && T == o.T &&
           T_s == o.T_s;
  }
};
struct TuneVal { int bn, variant; };
constexpr int kTuneCache = 64;
TuneKey g_tune_key[kTuneCache];
TuneVal g_tune_val[kTuneCache];
int g_tune_n = 0;
std::mutex g_tune_mu;
}  // namespace

cudaError_t tc_gemm_tune(TcGemm& tg, float* Mo, int P, int64_t T, int64_t T_s, int C, int K, float* Vw) {
  if (const char* ev = getenv("WINO_GEMM_VARIANT")) {
    const int v = atoi(ev);
    if ((v == kGemmTS && tg.can_ts) || (v == kGemmPair && tg.can_pair) || v == kGemmSS) tg.variant = v;
    return cudaSuccess;
  }
  if (getenv("WINO_GEMM_BN")) return cudaSuccess;  // dev knob fixes the tile and the default variant
  int dev = 0;
  cudaGetDevice(&dev);
  const TuneKey key{dev, P, C, K, tg.three, tg.kc, T, T_s};
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    for (int i = 0; i < g_tune_n; ++i)
      if (g_tune_key[i] == key) {
        cudaError_t e = prep_bn(tg, g_tune_val[i].bn, C);
        if (e == cudaSuccess) tg.variant = g_tune_val[i].variant;
        return e;
      }
  }
  // candidates: (N tile, variant); a 256-wide N tile (K > 128) is also tried
  // at 128, where TMEM has room for A stages and the CTA-pair kernel applies
  struct Cand { int bn, v; };
  Cand cand[8];
  int nc = 0;
  const int bns[2] = {tg.bn_max, 128};
  for (int ib = 0; ib < (tg.bn_max == 256 ? 2 : 1); ++ib) {
    cudaError_t e = prep_bn(tg, bns[ib], C);
    if (e != cudaSuccess) return e;
    cand[nc++] = {bns[ib], kGemmSS};
    if (tg.can_ts) cand[nc++] = {bns[ib], kGemmTS};
    if (tg.can_pair) cand[nc++] = {bns[ib], kGemmPair};
  }
  // all tuning work runs on a private non-blocking stream: it never
  // serialises with the caller's streams (or the legacy default stream),
  // and only this stream is synchronised
  cudaStream_t ts = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  // interleaved rounds (every candidate once per round, a warm-up launch
  // then two timed ones), summed per candidate: slow drift of clocks or L2
  // state between candidates does not decide the choice
  float tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int round = 0; round < 4 && e == cudaSuccess; ++round) {
    for (int i = 0; i < nc; ++i) {
      if ((e = prep_bn(tg, cand[i].bn, C)) != cudaSuccess) break;
      tg.variant = cand[i].v;
      if ((e = launch_gemm_tc(tg, Mo, P, 0, T, T_s, C, K, ts)) != cudaSuccess) break;  // warm-up
      // as in the forward, V has just been written when the GEMM starts: a
      // memset of V (zeros: the padding rows stay zero) precedes each timed launch
      float t = 0.f;
      for (int r = 0; r < 2; ++r) {
        if (Vw && (e = cudaMemsetAsync(Vw, 0, (size_t)P * C * T_s * 4, ts)) != cudaSuccess) break;
        if ((e = cudaEventRecord(e0, ts)) != cudaSuccess) break;
        if ((e = launch_gemm_tc(tg, Mo, P, 0, T, T_s, C, K, ts)) != cudaSuccess) break;
        if ((e = cudaEventRecord(e1, ts)) != cudaSuccess) break;
        if ((e = cudaEventSynchronize(e1)) != cudaSuccess) break;
        float tr = 0.f;
        cudaEventElapsedTime(&tr, e0, e1);
        t += tr;
      }
      if (e != cudaSuccess) break;
      tot[i] += t;
    }
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(ts);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (ts) cudaStreamDestroy(ts);
  if (e != cudaSuccess) return e;
  // the CTA-pair kernel is preferred within 6% of the fastest: inside the
  // three-kernel forward it overlaps its neighbours better than the timing
  // in isolation shows (measured: c3 1.84 -> 1.74 ms and c2 0.110 -> 0.104
  // ms per layer with the pair kernel though 3% / 1% slower alone; 6% keeps
  // c3's choice clear of timing noise, c3t's pair kernel is 17% slower)
  float best = 1e30f, best_eff = 1e30f;
  Cand bc = cand[0];
  for (int i = 0; i < nc; ++i) {
    if (getenv("WINO_DEBUG"))
      fprintf(stderr, "[wino] gemm candidate bn %d variant %d: %.4f ms per launch\n", cand[i].bn, cand[i].v,
              tot[i] / 8);
    const float eff = cand[i].v == kGemmPair ? tot[i] / 1.06f : tot[i];
    if (eff < best_eff) { best_eff = eff; best = tot[i]; bc = cand[i]; }
  }
  best /= 4;
  if ((e = prep_bn(tg, bc.bn, C)) != cudaSuccess) return e;
  tg.variant = bc.v;
  if (getenv("WINO_DEBUG"))
    fprintf(stderr, "[wino] gemm bn %d variant %d (%.4f ms per launch)\n", bc.bn, bc.v, best / 2);
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    const int slot = g_tune_n < kTuneCache ? g_tune_n++ : (int)(key.T % kTuneCache);
    g_tune_key[slot] = key;
    g_tune_val[slot] = {bc.bn, bc.v};
  }
  return cudaSuccess;
}

}  // namespace wino
