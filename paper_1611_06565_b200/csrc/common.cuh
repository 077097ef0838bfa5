// common.cuh -- shared device/host definitions of the B200 Winograd path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>

#include <type_traits>
#include <utility>

#include "synth.hpp"

namespace wino {

constexpr int kMaxN = 4;      // spatial dims supported on the device path
constexpr int kMaxA = 8;      // alpha <= 8 on the device path
constexpr int kMaxPlanes = 8;  // input-transform slabs staged per CTA
constexpr int kMaxOutStages = 8;  // output-transform TMA ring depth
constexpr int kMaxDevices = 64;   // per-device caches of launch attributes

constexpr int ipow(int b, int e) { return e <= 0 ? 1 : b * ipow(b, e - 1); }

// Compile-time loop: f(std::integral_constant<int, i>) for i in [B, E).
template <int B, int E, class F>
__host__ __device__ __forceinline__ void sfor(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    sfor<B + 1, E>(std::forward<F>(f));
  }
}

// Geometry of one plan, passed by value (__grid_constant__) to the transform kernels.
struct KGeom {
  int64_t in[kMaxN];         // input extents
  int64_t in_stride[kMaxN];  // element strides inside one (b, c) plane
  int64_t out[kMaxN];        // output extents
  int64_t out_stride[kMaxN];
  int tiles[kMaxN];          // ceil(out / m)
  int pad[kMaxN];
  int64_t in_vol, out_vol;   // per (b, c) / (b, k) plane
  int64_t Tps;               // tiles per sample
  int64_t T;                 // end of the tile range of this launch (B * Tps unchunked)
  int64_t T_s;               // row stride of V and M (multiple of 128)
  int64_t t_beg;             // first tile of this launch (output transform)
  int64_t t0;                // V / M row of tile t is t - t0 (L2-chunked buffers)
  int64_t s_beg;             // first input slab ((b * nbox0 + box0) * nbox1 + box1) of this launch
  int C, K;
  int m;                     // output tile length (runtime copy)
  const float* bias;         // optional per-output-channel bias b[k] of Eq. (2) (NULL = none)
  int act;                   // activation f of Eq. (2): 0 identity, 1 ReLU
  // Input-transform slab (xform_in.cu, plan_input_slab): one CTA stages, for
  // one (b, c) plane, the input needed by tiles [a, a + bt0) along axis 0 and
  // every tile along axes 1..N-1 (a contiguous run of t), zero padded.
  int bt0;                   // tiles along axis 0 per CTA
  int nbox0;                 // ceil(tiles[0] / bt0)
  int e[kMaxN];              // slab extents for a full box (axis 0: bt0*m + alpha - m; axis 1: bt1*m + alpha - m)
  int pitch;                 // padded last-axis extent (multiple of 4 floats)
  int dL;                    // TMA column shift of the slab rows (0 or 3)
  int sst[kMaxN];            // slab element strides (sst[N-1] = 1)
  int R;                     // tiles per axis-0 slice: prod_{n>=1} tiles[n]
  // Axis-1 banding (N >= 3, one-tile-deep slabs whose full axis-1 extent
  // would not fit shared memory): a slab covers tiles [a1, a1 + bt1) of axis
  // 1 -- still one contiguous run of t, since axis 1 is the outermost axis
  // inside an axis-0 slice.  Unbanded: bt1 = tiles[1], nbox1 = 1.
  int bt1;                   // axis-1 tiles per slab (divides tiles[1])
  int nbox1;                 // tiles[1] / bt1
  int R1;                    // prod_{n>=2} tiles[n]: t stride of axis 1
  int Rs;                    // tiles per axis-0 slice of one slab: bt1 * R1
  int slab_bytes;            // bytes of the slab (one TMA box)
  int slot_bytes;            // slab slot stride (slab_bytes rounded up to 128)
  int hpitch;                // N = 3, alpha >= 6: row pitch of the axis-0 pass buffer H
  int hinplace;              // N = 3, alpha >= 6, bt0 = 1: the axis-0 pass overwrites the slab (no H)
  int npl;                   // slabs per CTA (consecutive work items, one TMA box each)
  int in_threads;            // block size of the input kernel (<= 256; <= 512 in H mode)
  int smem_bytes;            // dynamic shared memory of the input kernel (npl slabs + H)
  int in_flags;              // dev A/B knob of the input kernel (WINO_IN_FLAGS; 0 in production)
  int in_align;              // in-place H mode: phase-2 items laid out so that every warp stores one
                             // 128-byte aligned line of V (WINO_IN_ALIGN)
  int in_prefetch;           // > 0: each CTA prefetches into L2 the slabs of the CTA in_prefetch blocks
                             // ahead (cp.async.bulk.prefetch.tensor), WINO_IN_PREFETCH
  int in_pad8;               // in-place H mode, m = 4: phase-2 items on 8 axis-2 slots per row
                             // (slots >= tiles[2] idle) so 8 lanes read 8 distinct 16-byte bank groups
  // 3xFP16 GEMM scaling (gemm_f16.cu): a2 atomically maxes |V| into *vmax,
  // a4 resets *vmax_reset = 0 for the next forward (NULL = not used)
  unsigned int* vmax;
  unsigned int* vmax_reset;
  unsigned long long* trace;   // dev probe (WINO_IN_TRACE): per-CTA %globaltimer events of a2 (NULL in production)
  // a5 direct-axis fold (xform_dfold.cu): a2 transforms the outer axes only and
  // writes Z [P/alpha * 2][C][Tz] (32-slot rows) instead of V
  int dfold;
  int df_S;                    // slots per row of tiles (32; > tiles_last)
  int64_t Tz;                  // slot pitch of a Z plane
};

// Runtime transform tables (generic path); constant-bank resident.
struct XfParams {
  float AT[kMaxA][kMaxA];
  float BT[kMaxA][kMaxA];
};

// Tables for the filter transform (fp64), one G per axis (axis n: a[n] x r[n]).
struct FParams {
  double G[kMaxN][kMaxA][kMaxA];
  int a[kMaxN], r[kMaxN];
  int N, C, K, K_s;
  int64_t P;  // prod_n a[n]
};

// Per-axis transforms of an N-D plan with different (m_n, r_n) per axis
// (Eq. (4) indexes B_n, A_n by n; xform_nd.cu).
struct NdParams {
  float BT[kMaxN][kMaxA][kMaxA];  // axis n: a[n] x a[n]
  float AT[kMaxN][kMaxA][kMaxA];  // axis n: m[n] x a[n]
  int a[kMaxN], m[kMaxN];
};

// Table providers.  ConstTab<M, R, PS>: tables synthesised at compile time
// into a __device__ constexpr object; inside fully unrolled loops every read
// is a constant, so zero entries vanish and +-1 become FADDs.  RunTab: the
// values come from XfParams at run time (any interpolation points).
template <int M, int R, int PS>
__device__ constexpr FloatTables kDevTab = to_tables(synthesize_default(M, R, PS));

template <int M_, int R_, int PS_>
struct ConstTab {
  static constexpr bool kConst = true;
  static_assert(synthesize_default(M_, R_, PS_).err == 0, "default synthesis failed");
  // the same tables as compile-time constants (structure detection, xform_common.cuh)
  static constexpr FloatTables kTab = to_tables(synthesize_default(M_, R_, PS_));
  __device__ static __forceinline__ float bt(const XfParams&, int x, int i) { return kDevTab<M_, R_, PS_>.BT[x][i]; }
  __device__ static __forceinline__ float at(const XfParams&, int x, int i) { return kDevTab<M_, R_, PS_>.AT[x][i]; }
};
struct RunTab {
  static constexpr bool kConst = false;
  __device__ static __forceinline__ float bt(const XfParams& p, int x, int i) { return p.BT[x][i]; }
  __device__ static __forceinline__ float at(const XfParams& p, int x, int i) { return p.AT[x][i]; }
};

// tf32 round-to-nearest, ties away from zero (= cvt.rna.tf32.f32) of a finite
// fp32 value, result as an fp32 container with the low 13 bits clear.  On the
// sign-magnitude bit pattern, adding half an ulp of tf32 (0x1000) and
// truncating rounds the magnitude half-up; two integer ops instead of the
// NaN/Inf-guarded cvt sequence.
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// Programmatic dependent launch (PDL).  Kernels of the forward are launched
// with programmatic stream serialization, so a kernel may start (prologue:
// barrier init, TMEM alloc, descriptor prefetch) while its predecessor drains.
// pdl_wait() blocks until every prerequisite grid has completed and its
// memory is visible -- it must precede any access to data the predecessor
// (or anything before it) produces or consumes; it is a no-op without PDL.
// pdl_trigger() lets dependents launch once all CTAs of this grid issued it;
// each kernel issues it only after its own pdl_wait (so dependents that run
// early can rely on everything before this grid being complete).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// WINO_PDL=0 (dev knob): plain stream-ordered launches (griddepcontrol is a
// no-op without the attribute)
// WINO_PDL_MASK (dev knob): PDL only for the stages whose bit is set (1
// input transform, 2 GEMM, 4 output transform; the plan tags the stage it
// launches through pdl_stage())
inline int& pdl_cur_stage() {
  static thread_local int st = 0;
  return st;
}
inline void pdl_stage(int s) { pdl_cur_stage() = s; }
inline bool pdl_enabled() {
  static int on = -1, mask = 7;
  if (on < 0) {
    const char* ev = getenv("WINO_PDL");
    on = ev ? (atoi(ev) != 0) : 1;
    if (const char* em = getenv("WINO_PDL_MASK")) mask = atoi(em);
  }
  const int st = pdl_cur_stage();
  return on != 0 && (st == 0 || (mask >> (st - 1)) & 1);
}

// Launch `kern` with the PDL attribute on stream s (unless `pdl` is false:
// plain stream order).  Grids of more than kPdlMaxCtasPerSm CTAs per SM are
// launched without it (pdl_grid_ok): launched early behind the GEMM, c3's
// 100k-CTA output grid made the layer 5% slower (1.27 vs 1.20 ms), while the
// 6k-CTA c2 and 2k-CTA c5 output grids gain from the overlap.
constexpr int kPdlMaxCtasPerSm = 64;
inline bool pdl_grid_ok(long long ctas) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  static int sms_dev[kMaxDevices] = {};
  if (!sms_dev[dev] && cudaDeviceGetAttribute(&sms_dev[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    sms_dev[dev] = 148;
  return ctas <= (long long)kPdlMaxCtasPerSm * sms_dev[dev];
}
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() && pdl_grid_ok((long long)grid.x * grid.y * grid.z) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace wino
