// tc_common.cuh -- device helpers of the tcgen05 GEMM kernels (gemm_tc.cu,
// gemm_ts2.cu): mbarriers, TMA, UMMA shared-memory / instruction
// descriptors, TMEM load/store, tf32 split.  PTX forms follow the PTX ISA
// (tcgen05, cp.async.bulk.tensor, mbarrier); shapes per SURVEY V8.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace wino {
namespace tc {

constexpr int BM = 128;
constexpr int kThreads = 352;    // SS kernel: 4 converter, 4 epilogue, 3 single-thread roles
constexpr int kThreadsTS = 480;  // TS kernels: + 4 more converter warps (11-14)

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
// L2 eviction-priority policies (createpolicy) and hinted accesses: V is
// streamed once (evict-first), M is read right after by a4 (evict-last).
__device__ __forceinline__ uint64_t l2_policy(bool last) {
  uint64_t pol;
  if (last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_3d_hint(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                                 uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_hint(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
// One lane of the (fully active) warp: lane 0.  The MMA issuer runs its loop
// in the whole warp so loop state stays warp-uniform (uniform registers feed
// UTCHMMA directly); only the elected lane issues tcgen05.mma / commit.
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(p));
  return p != 0;
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

// tcgen05.ld 32x32b.x32 without the wait (the caller issues tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// One 32-row block of an accumulator column to M: p[j T_s] = scale * r[j]
// for j < kr (kr >= 32: all 32), evict-last policy `pol` when l2hint.  Full
// blocks are branch-free runs: a per-store test of kr / l2hint made the
// compiler re-materialise the policy operand at every store (R2UR pairs),
// which bounded the epilogue (measured on the 3xFP16 GEMM: c3 GEMM 1.90 ->
// 0.93 ms).
template <bool kScale>
__device__ __forceinline__ void store_m32(float* p, const uint32_t (&r)[32], long long T_s, int kr, int l2hint,
                                          uint64_t pol, float scale) {
  if (kr >= 32) {
    if (l2hint) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        st_hint(p + j * T_s, kScale ? __uint_as_float(r[j]) * scale : __uint_as_float(r[j]), pol);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) __stcs(p + j * T_s, kScale ? __uint_as_float(r[j]) * scale : __uint_as_float(r[j]));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < kr) __stcs(p + j * T_s, kScale ? __uint_as_float(r[j]) * scale : __uint_as_float(r[j]));
  }
}

constexpr uint32_t tmem_cols(int bn) {
  return (2 * bn) <= 32 ? 32 : (2 * bn) <= 64 ? 64 : (2 * bn) <= 128 ? 128 : (2 * bn) <= 256 ? 256 : 512;
}


// ---- A operand in TMEM ("TS" mode): the MMA reads only U from shared memory.
// A (V_hi / V_lo chunk, 128 rows x kc columns) lives in TMEM columns, one tile
// row t per lane; K-major by construction (a_major bit 15 = 0).
template <int BN>
__host__ __device__ constexpr uint32_t idesc_tf32_ts() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// Lean issue of one chunk's 3xTF32 MMAs in TS mode (measured, tools/mma_bench.cu:
// a kind::tf32 M=128 K=8 MMA occupies the tensor pipe N/2 cycles -- 16 at N = 32
// -- but a loop that recomputes its operands each iteration issues one only
// every ~54 cycles, so small-N GEMMs were issue-bound).  Fully unrolled over
// the NK K=8 steps; the B descriptor is passed as its two 32-bit halves (the
// start-address field sits in the low half and never carries out of it), so
// each MMA needs one 32-bit add per operand.
__device__ __forceinline__ void mma_ts_split(uint32_t d, uint32_t a_tmem, uint32_t b_lo32, uint32_t b_hi32,
                                             uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 bd;\n\tmov.b64 bd, {%2, %3};\n\tsetp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], bd, %4, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "r"(b_lo32), "r"(b_hi32), "r"(idesc), "r"(acc)
      : "memory");
}
// d += V_lo U_hi + V_hi U_lo + V_hi U_hi over NK K=8 steps; A (V_hi at a_hi,
// V_lo at a_lo) in TMEM, U_hi / U_lo descriptors (low halves bh / bl, shared
// high half bhi32); `first`: the chunk opens the accumulation (D overwritten).
template <int NK>
__device__ __forceinline__ void mma3_chunk_ts(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t bh, uint32_t bl,
                                              uint32_t bhi32, uint32_t idesc, bool first) {
#pragma unroll
  for (int j = 0; j < NK; ++j) {
    mma_ts_split(d, a_lo + 8 * j, bh + 64 * j, bhi32, idesc, (j == 0 && first) ? 0u : 1u);
    mma_ts_split(d, a_hi + 8 * j, bl + 64 * j, bhi32, idesc, 1u);
    mma_ts_split(d, a_hi + 8 * j, bh + 64 * j, bhi32, idesc, 1u);
  }
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ uint32_t tf32_rna_bits(uint32_t u) { return (u + 0x1000u) & 0xFFFFE000u; }

// ---- CTA pairs (cta_group::2, clusters of two) -------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of `addr` (own shared::cta address) in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// wait with cluster-scope acquire: for barriers the peer CTA arrives on
__device__ __forceinline__ void mbar_wait_cl(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
// Arrive on a barrier of a CTA of the cluster (cl_addr from mapa).  Default
// (.release, .cta) semantics: the data it publishes is TMEM content ordered by
// tcgen05.wait::st + tcgen05.fence::before_thread_sync, not generic memory,
// and an explicit .release.cluster costs a CTA-wide MEMBAR per arrive.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cl_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
// TMA whose complete_tx lands on a barrier of the pair's leader (cl_bar).
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                                 uint32_t cl_bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(cl_bar)
      : "memory");
}
__device__ __forceinline__ void tc2_commit_mc(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tc2_mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                                uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

constexpr uint32_t pow2_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }


}  // namespace tc
}  // namespace wino
