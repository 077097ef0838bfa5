// gemm_ts2.cu -- stage a3 with CTA-pair MMAs (tcgen05 cta_group::2), A in TMEM.
//
// Same computation as k_gemm_ts (gemm_tc.cu): for every transform point xi,
// M_xi = V_xi U_xi with 3xTF32 (V_lo U_hi + V_hi U_lo + V_hi U_hi), but a work
// unit is (xi, n-block, 256-tile m-pair) computed by a cluster of two CTAs
// on two SMs:
//   - each CTA owns 128 of the 256 rows: it streams its own V chunks (raw
//     TMA ring), splits them into V_hi / V_lo and writes them into its own
//     TMEM (A operand, lanes = its tile rows);
//   - each CTA loads HALF of every U chunk (BN/2 output channels), so the
//     pair reads U_xi from L2 once per 256 tiles instead of once per 128 --
//     the U re-read was the c2 GEMM's limiter (DESIGN.md a3);
//   - the leader CTA (rank 0) issues tcgen05.mma.cta_group::2 M=256 N=BN
//     K=8; the hardware takes A rows and B columns from both CTAs; each CTA's
//     TMEM receives the accumulator rows it owns;
//   - completion is multicast to both CTAs (tcgen05.commit.cta_group::2 ...
//     multicast::cluster); the peer signals readiness to the leader's
//     mbarriers through shared::cluster addresses (mapa), and its U TMA
//     completes on the leader's barrier (cp.async.bulk.tensor.cta_group::2).
// Warps per CTA: 0-3 and 11-14 converter, 4-7 epilogue, 8 V producer, 9 MMA
// issuer (leader) / TMEM owner, 10 U producer.
#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "tc_common.cuh"
#include "tma.hpp"

namespace wino {
namespace tc {
namespace {

// kind::tf32, D f32, A K-major (TMEM), B MN-major, M = 256 (pair), N = BN.
template <int BN>
__host__ __device__ constexpr uint32_t idesc_tf32_pair() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsTS, 1)
k_gemm_ts2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
           const __grid_constant__ CUtensorMap tmBlo, float* __restrict__ Mo, int P, int t_lo, int T, long long T_s,
           int C, int K, int kc, int three, int nraw, int nbr, int dbg, int l2hint, int nbfast) {
  constexpr int HN = BN / 2;  // U columns loaded by each CTA
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (sraw & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  const uint32_t sbase = sraw + pad;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n_chunks = (C + kc - 1) / kc;
  const uint32_t a_bytes = (uint32_t)BM * kc * 4;
  const uint32_t hb_bytes = (uint32_t)HN * kc * 4;  // this CTA's half of one U chunk (hi or lo)
  const uint32_t raw0 = sbase;
  const uint32_t ub0 = raw0 + nraw * a_bytes;
  const uint32_t bar0 = ub0 + 2u * nbr * hb_bytes;
  auto rfull = [&](int s) { return bar0 + 8u * s; };
  auto rempty = [&](int s) { return bar0 + 8u * (nraw + s); };
  auto ufull = [&](int s) { return bar0 + 8u * (2 * nraw + s); };
  auto uempty = [&](int s) { return bar0 + 8u * (2 * nraw + nbr + s); };
  const uint32_t bar1 = bar0 + 8u * (2 * nraw + 2 * nbr);
  auto tfull = [&](int a) { return bar1 + 8u * a; };
  auto tempty = [&](int a) { return bar1 + 8u * (2 + a); };
  auto afull = [&](int a) { return bar1 + 8u * (4 + a); };   // a < 4
  auto aempty = [&](int a) { return bar1 + 8u * (8 + a); };
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
        mbar_init(ufull(s), 1);    // leader: expect_tx of both halves
        mbar_init(uempty(s), 1);   // MMA commit (multicast)
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(tfull(a), 1);    // MMA commit (multicast)
        mbar_init(tempty(a), 2);   // one arrive per CTA's epilogue
      }
      for (int a = 0; a < na; ++a) {
        mbar_init(afull(a), 2);    // one arrive per CTA's converter
        mbar_init(aempty(a), 1);   // MMA commit (multicast)
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
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();
  pdl_trigger();

  const int n_mp = (T - t_lo + 2 * BM - 1) / (2 * BM);  // 256-tile m-pairs
  const int n_nblk = (K + BN - 1) / BN;
  const long long per_xi = (long long)n_nblk * n_mp;
  const long long total = (long long)P * per_xi;
  const long long u_beg = blockIdx.x >> 1, u_step = gridDim.x >> 1;

  if (warp == 8) {
    if (lane == 0) {  // ---------------- V producer: this CTA's 128 rows
      int s = 0;
      uint32_t ph = 0;
      for (long long u = u_beg; u < total; u += u_step) {
        const int xi = (int)(u / per_xi);
        const int mp = nbfast ? (int)(u % per_xi) / n_nblk : (int)(u % per_xi) % n_mp;
        const int row0 = t_lo + mp * 2 * BM + (int)rank * BM;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(rempty(s), ph ^ 1u);
          if (dbg & 16) {
            mbar_arrive(rfull(s));  // dev knob: no V loads
          } else {
            mbar_expect_tx(rfull(s), a_bytes);
            if (l2hint) tma_load_3d_hint(raw0 + s * a_bytes, &tmA, row0, ch * kc, xi, rfull(s), l2_policy(false));
            else tma_load_3d(raw0 + s * a_bytes, &tmA, row0, ch * kc, xi, rfull(s));
          }
          if (++s == nraw) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {  // ---------------- U producer: this CTA's BN/2 columns
      int s = 0;
      uint32_t ph = 0;
      const uint32_t half_tx = (three ? 2u : 1u) * hb_bytes;
      for (long long u = u_beg; u < total; u += u_step) {
        const int xi = (int)(u / per_xi);
        const int nb = nbfast ? (int)(u % per_xi) % n_nblk : (int)(u % per_xi) / n_mp;
        const int col0 = nb * BN + (int)rank * HN;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(uempty(s), ph ^ 1u);
          const uint32_t st = ub0 + s * 2 * hb_bytes;
          const uint32_t lb = mapa(ufull(s), 0);
          if (dbg & 8) {  // dev knob: no U loads
            if (leader) mbar_arrive(ufull(s));
            if (++s == nbr) { s = 0; ph ^= 1u; }
            continue;
          }
          if (leader) mbar_expect_tx(ufull(s), 2u * half_tx);
#pragma unroll
          for (int gq = 0; gq < HN / 32; ++gq) {
            tma_load_3d_pair(st + gq * kc * 128, &tmBhi, col0 + gq * 32, ch * kc, xi, lb);
            if (three) tma_load_3d_pair(st + hb_bytes + gq * kc * 128, &tmBlo, col0 + gq * 32, ch * kc, xi, lb);
          }
          if (++s == nbr) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 9) {
    if (leader) {  // ---------------- MMA issuer (leader CTA; warp-uniform loop, elected lane issues)
      constexpr uint32_t idesc = idesc_tf32_pair<BN>();
      const int nk = (dbg & 4) ? 0 : kc / 8;
      const uint32_t lbo = (uint32_t)kc * 128u;
      int as = 0, us = 0;
      uint32_t aph = 0, uph = 0, acc = 0, cph = 0;
      for (long long u = u_beg; u < total; u += u_step) {
        mbar_wait(tempty(acc), cph ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(afull(as), aph);
          mbar_wait(ufull(us), uph);
          tc_fence_after();
          const uint32_t b_hi = ub0 + us * 2 * hb_bytes;
          uint64_t dbh = sdesc(b_hi, lbo, 512u), dbl = sdesc(b_hi + hb_bytes, lbo, 512u);
          const uint32_t a_hi = tmem_base + a_col0 + as * 2 * kc, a_lo = a_hi + kc;
          if (elect_one()) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // kc <= 64: at most 8 K=8 steps
              if (j < nk) {
                const uint32_t accum = (ch | j) != 0;
                if (three) {
                  tc2_mma_tf32_ts(d, a_lo + 8 * j, dbh + 64 * j, idesc, accum);
                  tc2_mma_tf32_ts(d, a_hi + 8 * j, dbl + 64 * j, idesc, 1u);
                  tc2_mma_tf32_ts(d, a_hi + 8 * j, dbh + 64 * j, idesc, 1u);
                } else {
                  tc2_mma_tf32_ts(d, a_hi + 8 * j, dbh + 64 * j, idesc, accum);
                }
              }
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
        acc ^= 1u;
        if (acc == 0) cph ^= 1u;
      }
    }
  } else if (warp < 4 || (warp >= 11 && warp < 15)) {  // ---- converter (8 warps): raw V row -> own TMEM hi / lo
    // warps w and w' with w % 4 == w' % 4 own TMEM lane quarter w % 4; the
    // second group (warps 11-14) converts the upper half of each chunk's channels
    const int q = warp & 3, grp = warp < 4 ? 0 : 1;
    const int row = q * 32 + lane;
    const uint32_t lane_sel = (uint32_t)(q * 32) << 16;
    const int cg0 = grp * (kc / 8) / 2, cg1 = (grp + 1) * (kc / 8) / 2;
    
    int rs = 0, as = 0;
    uint32_t rph = 0, aph = 0;
    for (long long u = u_beg; u < total; u += u_step) {
      for (int ch = 0; ch < n_chunks; ++ch) {
        mbar_wait(rfull(rs), rph);
        mbar_wait(aempty(as), aph ^ 1u);
        tc_fence_after();
        const float* rawp = reinterpret_cast<const float*>(smem + rs * a_bytes) + row;
        const uint32_t ahi = tmem_base + lane_sel + a_col0 + as * 2 * kc;
        for (int cg = cg0; cg < cg1; ++cg) {
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float v = rawp[(cg * 8 + j) * BM];
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
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (threadIdx.x == 0) mbar_arrive_cluster(mapa(afull(as), 0));
        if (++rs == nraw) { rs = 0; rph ^= 1u; }
        if (++as == na) { as = 0; aph ^= 1u; }
      }
    }
  } else if (warp < 8) {  // warps 4-7 ------------------ epilogue: own 128 rows
    const int q = warp - 4;
    const uint32_t tempty_l[2] = {mapa(tempty(0), 0), mapa(tempty(1), 0)};
    const uint64_t pol = l2_policy(true);
    uint32_t acc = 0, aph = 0;
    for (long long u = u_beg; u < total; u += u_step) {
      const int xi = (int)(u / per_xi);
      const int rr = (int)(u % per_xi);
      const int nb = nbfast ? rr % n_nblk : rr / n_mp, mp = nbfast ? rr / n_nblk : rr % n_mp;
      mbar_wait(tfull(acc), aph);
      tc_fence_after();
      const int t = t_lo + mp * 2 * BM + (int)rank * BM + q * 32 + lane;
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
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (threadIdx.x == 128) mbar_arrive_cluster(tempty_l[acc]);
      acc ^= 1u;
      if (acc == 0) aph ^= 1u;
    }
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kCols) : "memory");
  }
}

}  // namespace
}  // namespace tc

// Shared memory of k_gemm_ts2: raw V ring + U half-chunk ring (nbr) + barriers.
static bool ts2_smem(int bn, int kc, int* nraw, int* nbr, size_t* bytes) {
  const size_t a = (size_t)tc::BM * kc * 4;
  const size_t hb2 = 2ull * (bn / 2) * kc * 4;
  const size_t fixed = 1024 + 1024;
  const size_t budget = 232448;
  size_t left = budget - fixed;
  // 4 U stages: measured (tools/pair_ring.sh) 6 or 8 give the same GEMM time
  // and a slower three-kernel step (c2 0.103 -> 0.109, c3 1.74 -> 1.89 ms)
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

bool ts2_supported(int bn, int kc) {
  int nr, nb;
  size_t by;
  return bn >= 64 && bn <= 256 && 2 * bn + 4 * kc <= 512 && ts2_smem(bn, kc, &nr, &nb, &by);
}

// Unit order within a point: n-block fastest (1, default: the pairs that
// share an m-pair's V run side by side, so its second n-block reads V from
// L2) or m-pair fastest (0); WINO_GEMM_NBFAST overrides (dev knob)
int gemm_nbfast() {
  static int v = -1;
  if (v < 0) {
    const char* ev = getenv("WINO_GEMM_NBFAST");
    v = ev ? (atoi(ev) != 0) : 1;
  }
  return v;
}

template <int BN>
static cudaError_t launch_ts2_bn(const TcGemm& tg, float* Mo, int P, int t_lo, int T, int64_t T_s, int C, int K,
                                 int num_sms, cudaStream_t s) {
  int nraw, nbr;
  size_t smem;
  if (!ts2_smem(BN, tg.kc, &nraw, &nbr, &smem)) return cudaErrorInvalidConfiguration;
  auto kern = tc::k_gemm_ts2<BN>;
  // per-device caches: the shared-memory opt-in is a per-context attribute
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  static size_t set_bytes_dev[kMaxDevices] = {};
  size_t& set_bytes = set_bytes_dev[dev];
  if (set_bytes != smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set_bytes = smem;
  }
  const long long units = (long long)P * ((K + BN - 1) / BN) * ((T - t_lo + 2 * tc::BM - 1) / (2 * tc::BM));
  // co-resident CTA pairs: with 1 CTA / SM not every SM can host a cluster
  // member (GPC boundaries), so size the persistent grid by the occupancy
  // query, not by num_sms / 2 (a second wave of clusters doubles the time)
  static int max_pairs_dev[kMaxDevices] = {};
  static size_t max_pairs_smem_dev[kMaxDevices] = {};
  int& max_pairs = max_pairs_dev[dev];
  size_t& max_pairs_smem = max_pairs_smem_dev[dev];
  if (max_pairs_smem != smem) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(num_sms);
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
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) n = num_sms / 2;
    max_pairs = n;
    max_pairs_smem = smem;
  }
  long long pairs = max_pairs;
  if (getenv("WINO_DEBUG"))
    fprintf(stderr, "[wino] k_gemm_ts2<%d>: max co-resident pairs %d, units %lld, nraw %d, nbr %d, smem %zu\n", BN,
            max_pairs, units, nraw, nbr, smem);
  if (pairs > units) pairs = units;
  // L2 policies: V loads evict-first (streamed once), M stores evict-last (a4
  // reads M right after).  Measured: c2 0.103 -> 0.100 ms, c3 1.747 -> 1.713
  // ms per layer (a4 33.1 -> 31.1 us on c2).  WINO_L2_HINTS=0 disables.
  static int l2hint = -1;
  if (l2hint < 0) {
    const char* ev = getenv("WINO_L2_HINTS");
    l2hint = ev ? (atoi(ev) != 0) : 1;
  }
  if (pairs < 1) return cudaSuccess;
  const long long Ts = T_s;
  return launch_pdl(kern, dim3((unsigned)(2 * pairs)), dim3(tc::kThreadsTS), smem, s, tg.tmA_ts, tg.tmBhi, tg.tmBlo, Mo, P,
                    t_lo, T, Ts, C, K, tg.kc, tg.three, nraw, nbr, tg.dbg, l2hint, gemm_nbfast());
}

cudaError_t launch_gemm_ts2(const TcGemm& tg, float* Mo, int P, int64_t t_lo, int64_t T, int64_t T_s, int C, int K,
                            cudaStream_t s) {
  switch (tg.bn) {
    case 64: return launch_ts2_bn<64>(tg, Mo, P, (int)t_lo, (int)T, T_s, C, K, tg.num_sms, s);
    case 128: return launch_ts2_bn<128>(tg, Mo, P, (int)t_lo, (int)T, T_s, C, K, tg.num_sms, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace wino
