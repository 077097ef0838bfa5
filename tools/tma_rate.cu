// Dev probe: achieved HBM read rate of TMA / bulk-copy plane loads as a
// function of box shape (row width), CTAs per SM and slots in flight.
// Each CTA walks planes grid-strided, loading each plane (56x56 fp32, the c2
// input plane) into one of `slots` SMEM slots; no compute.
//   mode 0: 3-D tiled box {64, 58, 1} at (-4, -1, p)   (current slab load)
//   mode 1: 2-D tiled box {224, 14} on the flat view [P*14][224]
//   mode 2: 1-D cp.async.bulk of 12544 B
//   mode 3: 2-D tiled box {56, 56} at (0, 0) (no padding, same row count)
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1611_06565_b200/csrc/tma.hpp"
using namespace wino;

__device__ __forceinline__ void wait_bar(uint32_t mb, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(mb), "r"(ph) : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap tm, const float* x, int P, int mode, int slots, int slot_bytes,
                  int bytes, unsigned long long* sink) {
  // modes 5/6 (c4 geometry): plane p = (b*C + c) * 2 + depth box

  extern __shared__ __align__(128) unsigned char S[];
  __shared__ __align__(8) uint64_t bar[8];
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(S);
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) {
      uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar[i]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int it = 0;
  auto issue = [&](int p, int s) {
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t dst = sb + s * slot_bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    if (mode == 0) {
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(dst), "l"(&tm), "r"(-4), "r"(-1), "r"(p), "r"(mb) : "memory");
    } else if (mode == 1) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(dst), "l"(&tm), "r"(0), "r"(p * 14), "r"(mb) : "memory");
    } else if (mode == 5) {
      const int bc = p >> 1, d0 = (p & 1) * 4 - 1;
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(dst), "l"(&tm), "r"(-4), "r"(-1), "r"(d0), "r"(bc), "r"(mb) : "memory");
    } else if (mode == 6) {
      const int bc = p >> 1, d0 = (p & 1) * 4;  // 4..6 planes in range: copy 4 planes + 1 halo (5 x 3136 B)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(x + (size_t)bc * 6272 + (size_t)(d0 > 0 ? d0 - 1 : 0) * 784), "r"(5 * 3136), "r"(mb) : "memory");
    } else if (mode == 2) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(x + (size_t)p * 3136), "r"(12544), "r"(mb) : "memory");
    } else {
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(dst), "l"(&tm), "r"(0), "r"(0), "r"(p), "r"(mb) : "memory");
    }
  };
  // prologue: fill all slots
  int p = blockIdx.x;
  int q = p;
  for (int s = 0; s < slots && q < P; ++s, q += gridDim.x) issue(q, s);
  int s = 0;
  unsigned ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long acc = 0;
  for (; p < P; p += gridDim.x) {
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    wait_bar(mb, ph[s]);
    ph[s] ^= 1;
    acc += S[s * slot_bytes + (it & 127)];
    ++it;
    if (q < P) { issue(q, s); q += gridDim.x; }
    s = (s + 1) % slots;
  }
  if (acc == 0xFFFFFFFFull) *sink = acc;
}

int main(int argc, char** argv) {
  const int P = 32768;  // planes: 411 MB
  float* x;
  cudaMalloc(&x, (size_t)P * 3136 * 4);
  cudaMemset(x, 0, (size_t)P * 3136 * 4);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  auto enc = get_encode();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm = 148;
  for (int mode = 0; mode < 7; ++mode) {
    CUtensorMap tm{};
    int bytes;
    int Pm = P;
    double payload = 12544;
    if (mode == 4) continue;
    if (mode == 5 || mode == 6) {
      // x viewed as [BC][8][28][28] (c4 planes), 2 depth boxes per (b, c)
      const cuuint64_t BC = (cuuint64_t)P * 3136 / 6272;
      Pm = (int)(BC * 2);
      cuuint64_t dims[4] = {28, 28, 8, BC};
      cuuint64_t strides[3] = {28 * 4, 784 * 4, 6272 * 4};
      cuuint32_t box[4] = {36, 30, 6, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) { printf("enc %d\n", r); return 1; }
      bytes = mode == 5 ? 36 * 30 * 6 * 4 : 5 * 3136;
      payload = 3136.0 * 4;  // unique x bytes per box (4 of 8 depth planes)
    } else if (mode == 0 || mode == 3) {
      cuuint64_t dims[3] = {56, 56, (cuuint64_t)P};
      cuuint64_t strides[2] = {56 * 4, 56 * 56 * 4};
      cuuint32_t box[3] = {mode == 0 ? 64u : 56u, mode == 0 ? 58u : 56u, 1};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) { printf("enc %d\n", r); return 1; }
      bytes = box[0] * box[1] * 4;
    } else {
      cuuint64_t dims[2] = {224, (cuuint64_t)P * 14};
      cuuint64_t strides[1] = {224 * 4};
      cuuint32_t box[2] = {224, 14};
      cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) { printf("enc %d\n", r); return 1; }
      bytes = 12544;
    }
    const int slot_bytes = (bytes + 127) / 128 * 128;
    for (int cps : {1, 2, 3, 4}) {
      for (int slots : {1, 2, 4}) {
        const int smem = slots * slot_bytes;
        if (smem * cps > 220 * 1024) continue;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int grid = nsm * cps;
        for (int w = 0; w < 2; ++w) k<<<grid, 32, smem>>>(tm, x, Pm, mode, slots, slot_bytes, bytes, sink);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int rr = 0; rr < reps; ++rr) k<<<grid, 32, smem>>>(tm, x, Pm, mode, slots, slot_bytes, bytes, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        const double gbs = (double)Pm * payload * reps / (ms * 1e-3) / 1e9;
        printf("mode %d cta/sm %d slots %d  %.1f us/launch  %.0f GB/s (unique x) %s\n", mode, cps, slots,
               ms * 1e3 / reps, gbs, err ? cudaGetErrorString(err) : "");
      }
    }
  }
  return 0;
}
