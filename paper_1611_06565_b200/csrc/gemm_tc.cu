// gemm_tc.cu -- stage a3 on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// For every transform point xi (Eq. (5)):
//     M_xi[t][k] = sum_c V_xi[t][c] U_xi[c][k]      ([T x C] x [C x K])
// fp32-accurate via 3xTF32 (reading #7):
//     V = V_hi + V_lo,  U = U_hi + U_lo  (hi = rna_tf32(x), lo = rna_tf32(x - hi))
//     M = V_lo U_hi + V_hi U_lo + V_hi U_hi       accumulated in fp32 in TMEM.
//
// One persistent, warp-specialised kernel; a work unit is (xi, n-block, m-block)
// of 128 tiles x BN output channels; units are ordered xi-major so concurrently
// running CTAs share U_xi in L2.
//   warp 8      TMA producer: V tile (fp32, 128 x kc) + U_hi/U_lo tiles (BN x kc)
//               into a `stages`-deep smem ring, MN-major, 128B rows with
//               32-byte swizzle atoms (SWIZZLE_128B_BASE32B).
//   warps 0-3   converter: split the V tile in place into V_hi and V_lo (the
//               tf32 rounding must be explicit: the tensor core truncates).
//   warp 9      MMA issuer (one thread): 3 x (kc/8) tcgen05.mma.kind::tf32
//               M=128 N=BN K=8 per stage into a double-buffered TMEM accumulator;
//               tcgen05.commit frees the smem stage / publishes the accumulator.
//   warps 4-7   epilogue: tcgen05.ld 32x32b.x32 -> registers -> M[xi][k][t]
//               (each warp stores 32 consecutive t per column: 128 B lines).
#include <cstdio>

#include "kernels.h"
#include "tma.hpp"

namespace wino {
namespace tc {

constexpr int BM = 128;
constexpr int kThreads = 320;

// Debug dump (dev only; set through tc_set_debug): CTA 0 copies its first
// smem stage after conversion and the raw accumulator of its first unit.
__device__ float* g_dbg = nullptr;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// Shared-memory matrix descriptor for the canonical MN-major tf32 layout
// SWIZZLE_128B_BASE32B (layout type 1; fp32 MN-major operands require the
// 32-byte swizzle base): rows of 128 B = 32 MN elements, 32-byte chunks XORed
// with (row mod 4), 4 K-rows (512 B) per swizzle atom.
//   LBO = byte distance between 32-element groups along MN,
//   SBO = byte distance between 4-row atoms along K (512 when dense).
// Bits: addr>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version 1 [46,48),
// layout type [61,64).  The TMA side writes the same pattern with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
  return d;
}

// Instruction descriptor kind::tf32: D f32 (bit 4), A/B tf32 (=2 at bits 7, 10),
// A and B MN-major (bits 15, 16), N>>3 at bit 17, M>>4 at bit 24.
template <int BN>
__host__ __device__ constexpr uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

constexpr uint32_t tmem_cols(int bn) {
  return (2 * bn) <= 32 ? 32 : (2 * bn) <= 64 ? 64 : (2 * bn) <= 128 ? 128 : (2 * bn) <= 256 ? 256 : 512;
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
          const __grid_constant__ CUtensorMap tmBlo, float* __restrict__ Mo, int P, int T, long long T_s,
          int C, int K, int kc, int three, int stages) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (sraw & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  const uint32_t sbase = sraw + pad;
  const uint32_t a_bytes = (uint32_t)BM * kc * 4;
  const uint32_t b_bytes = (uint32_t)BN * kc * 4;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  const uint32_t bar0 = sbase + stages * stage_bytes;  // 8-byte barriers
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto conv = [&](int s) { return bar0 + 8u * (stages + s); };
  auto empty = [&](int s) { return bar0 + 8u * (2 * stages + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (3 * stages + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (3 * stages + 2 + a); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + stages * stage_bytes + 8 * (3 * stages + 4));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kCols = tmem_cols(BN);

  if (warp == 9) {
    if (lane == 0) {
      for (int s = 0; s < stages; ++s) {
        mbar_init(full(s), 1);
        mbar_init(conv(s), 128);
        mbar_init(empty(s), 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(tfull(a), 1);
        mbar_init(tempty(a), 128);
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

  const int n_mblk = (T + BM - 1) / BM;
  const int n_nblk = (K + BN - 1) / BN;
  const int n_chunks = (C + kc - 1) / kc;
  const long long per_xi = (long long)n_nblk * n_mblk;
  const long long total = (long long)P * per_xi;

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      const uint32_t tx = a_bytes + (three ? 2u : 1u) * b_bytes;
      for (long long u = blockIdx.x; u < total; u += gridDim.x) {
        const int xi = (int)(u / per_xi);
        const int rr = (int)(u % per_xi);
        const int nb = rr / n_mblk, mb = rr % n_mblk;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(empty(s), ph ^ 1u);
          const uint32_t st = sbase + s * stage_bytes;
          mbar_expect_tx(full(s), tx);
#pragma unroll
          for (int gq = 0; gq < BM / 32; ++gq)
            tma_load_3d(st + gq * kc * 128, &tmA, mb * BM + gq * 32, ch * kc, xi, full(s));
#pragma unroll
          for (int gq = 0; gq < BN / 32; ++gq) {
            tma_load_3d(st + 2 * a_bytes + gq * kc * 128, &tmBhi, nb * BN + gq * 32, ch * kc, xi, full(s));
            if (three)
              tma_load_3d(st + 2 * a_bytes + b_bytes + gq * kc * 128, &tmBlo, nb * BN + gq * 32, ch * kc, xi,
                          full(s));
          }
          if (++s == stages) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_tf32<BN>();
      const uint32_t lbo = (uint32_t)kc * 128u;
      int s = 0;
      uint32_t ph = 0, acc = 0, aph = 0;
      for (long long u = blockIdx.x; u < total; u += gridDim.x) {
        mbar_wait(tempty(acc), aph ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(conv(s), ph);
          tc_fence_after();
          const uint32_t st = sbase + s * stage_bytes;
          const uint32_t a_hi = st, a_lo = st + a_bytes, b_hi = st + 2 * a_bytes, b_lo = b_hi + b_bytes;
          for (int j = 0; j < kc / 8; ++j) {
            const uint32_t off = (uint32_t)j * 1024u;
            const uint32_t accum = (ch | j) != 0;
            const uint64_t dah = sdesc(a_hi + off, lbo, 512u);
            const uint64_t dbh = sdesc(b_hi + off, lbo, 512u);
            if (three) {
              tc_mma_tf32(d, sdesc(a_lo + off, lbo, 512u), dbh, idesc, accum);
              tc_mma_tf32(d, dah, sdesc(b_lo + off, lbo, 512u), idesc, 1u);
              tc_mma_tf32(d, dah, dbh, idesc, 1u);
            } else {
              tc_mma_tf32(d, dah, dbh, idesc, accum);
            }
          }
          tc_commit(empty(s));
          if (++s == stages) { s = 0; ph ^= 1u; }
        }
        tc_commit(tfull(acc));
        acc ^= 1u;
        if (acc == 0) aph ^= 1u;
      }
    }
  } else if (warp < 4) {  // ---------------- converter (128 threads)
    int s = 0;
    uint32_t ph = 0;
    const int n4 = (int)(a_bytes / 16);
    for (long long u = blockIdx.x; u < total; u += gridDim.x) {
      for (int ch = 0; ch < n_chunks; ++ch) {
        mbar_wait(full(s), ph);
        float4* araw = reinterpret_cast<float4*>(smem + s * stage_bytes);
        float4* alo = reinterpret_cast<float4*>(smem + s * stage_bytes + a_bytes);
        for (int i = threadIdx.x; i < n4; i += 128) {
          const float4 v = araw[i];
          float4 h, l;
          h.x = tf32_rna(v.x); h.y = tf32_rna(v.y); h.z = tf32_rna(v.z); h.w = tf32_rna(v.w);
          araw[i] = h;
          if (three) {
            l.x = tf32_rna(v.x - h.x); l.y = tf32_rna(v.y - h.y);
            l.z = tf32_rna(v.z - h.z); l.w = tf32_rna(v.w - h.w);
            alo[i] = l;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (g_dbg && blockIdx.x == 0 && u == blockIdx.x && ch == 0) {
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const float* sp = reinterpret_cast<const float*>(smem + s * stage_bytes);
          for (uint32_t i = threadIdx.x; i < stage_bytes / 4; i += 128) g_dbg[i] = sp[i];
        }
        mbar_arrive(conv(s));
        if (++s == stages) { s = 0; ph ^= 1u; }
      }
    }
  } else {  // warps 4-7 ------------------ epilogue
    const int q = warp - 4;
    uint32_t acc = 0, aph = 0;
    for (long long u = blockIdx.x; u < total; u += gridDim.x) {
      const int xi = (int)(u / per_xi);
      const int rr = (int)(u % per_xi);
      const int nb = rr / n_mblk, mb = rr % n_mblk;
      mbar_wait(tfull(acc), aph);
      tc_fence_after();
      const int t = mb * BM + q * 32 + lane;
      float* out = Mo + (long long)xi * K * T_s + t;
#pragma unroll 1
      for (int cb = 0; cb < BN / 32; ++cb) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + cb * 32, r);
        const int k0 = nb * BN + cb * 32;
        if (g_dbg && blockIdx.x == 0 && u == blockIdx.x) {
          for (int j = 0; j < 32; ++j) g_dbg[65536 + (q * 32 + lane) * 256 + cb * 32 + j] = __uint_as_float(r[j]);
        }
        if (t < T) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (k0 + j < K) out[(long long)(k0 + j) * T_s] = __uint_as_float(r[j]);
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
cudaError_t tc_set_debug(float* p) { return cudaMemcpyToSymbol(tc::g_dbg, &p, sizeof(p)); }

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

static size_t tc_smem_bytes(int bn, int kc, int* stages_out) {
  const size_t stage = 2ull * tc::BM * kc * 4 + 2ull * bn * kc * 4;
  const size_t budget = 232448 - 1024 - 512;
  int st = (int)(budget / stage);
  if (st > 6) st = 6;
  if (stages_out) *stages_out = st;
  return (size_t)st * stage + 1024 + 512;
}

cudaError_t tc_gemm_prepare(TcGemm& tg, const float* V, const float* Uhi, const float* Ulo, int P, int64_t T_s,
                            int C, int K_s, int K, int three, int device) {
  tg.ready = false;
  tg.bn = pick_bn(K);
  tg.kc = C >= 32 ? 32 : ((C + 7) / 8) * 8;
  tg.three = three;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  tg.num_sms = sms;
  cudaError_t e;
  if ((e = encode3d(&tg.tmA, V, T_s, C, P, tg.kc)) != cudaSuccess) return e;
  if ((e = encode3d(&tg.tmBhi, Uhi, K_s, C, P, tg.kc)) != cudaSuccess) return e;
  if ((e = encode3d(&tg.tmBlo, Ulo ? Ulo : Uhi, K_s, C, P, tg.kc)) != cudaSuccess) return e;
  int st;
  const size_t smem = tc_smem_bytes(tg.bn, tg.kc, &st);
  switch (tg.bn) {
    case 32: e = cudaFuncSetAttribute(tc::k_gemm_tc<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); break;
    case 64: e = cudaFuncSetAttribute(tc::k_gemm_tc<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); break;
    case 128: e = cudaFuncSetAttribute(tc::k_gemm_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); break;
    default: e = cudaFuncSetAttribute(tc::k_gemm_tc<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); break;
  }
  if (e != cudaSuccess) return e;
  tg.ready = true;
  return cudaSuccess;
}

cudaError_t launch_gemm_tc(const TcGemm& tg, float* Mo, int P, int64_t T, int64_t T_s, int C, int K,
                           cudaStream_t s) {
  if (!tg.ready) return cudaErrorNotReady;
  int st;
  const size_t smem = tc_smem_bytes(tg.bn, tg.kc, &st);
  const long long units = (long long)P * ((K + tg.bn - 1) / tg.bn) * ((T + tc::BM - 1) / tc::BM);
  const int grid = (int)(units < tg.num_sms ? units : tg.num_sms);
  if (grid <= 0) return cudaSuccess;
  switch (tg.bn) {
    case 32: tc::k_gemm_tc<32><<<grid, tc::kThreads, smem, s>>>(tg.tmA, tg.tmBhi, tg.tmBlo, Mo, P, (int)T, T_s, C, K, tg.kc, tg.three, st); break;
    case 64: tc::k_gemm_tc<64><<<grid, tc::kThreads, smem, s>>>(tg.tmA, tg.tmBhi, tg.tmBlo, Mo, P, (int)T, T_s, C, K, tg.kc, tg.three, st); break;
    case 128: tc::k_gemm_tc<128><<<grid, tc::kThreads, smem, s>>>(tg.tmA, tg.tmBhi, tg.tmBlo, Mo, P, (int)T, T_s, C, K, tg.kc, tg.three, st); break;
    default: tc::k_gemm_tc<256><<<grid, tc::kThreads, smem, s>>>(tg.tmA, tg.tmBhi, tg.tmBlo, Mo, P, (int)T, T_s, C, K, tg.kc, tg.three, st); break;
  }
  return cudaGetLastError();
}

}  // namespace wino
