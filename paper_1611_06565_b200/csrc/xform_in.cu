// xform_in.cu -- host side of stage a2: slab geometry, the TMA descriptor of
// x, and dispatch to the instantiations (xform_in_const.cu, xform_in_run.cu).
#include <cstdio>
#include <cstdlib>

#include "tma.hpp"
#include "xform_in.cuh"

namespace wino {

// Slab geometry of k_input_xform for a plan (fills g.bt0 .. g.slab_bytes).
// The box spans tiles [a, a+bt0) of axis 0 and all tiles of the other axes;
// bt0 is the largest (halving) count whose slab stays near 64 KB of shared
// memory.  With `tma` the last-axis rows start dL = (-P_last) mod 4 columns
// early (16-byte aligned TMA start).  Returns false if even a one-tile-deep
// slab exceeds 200 KB.
bool plan_input_slab(KGeom& g, int N, int alpha0, int m0, int alpha, int m, bool tma) {
  const int halo = alpha - m;      // axes >= 1
  const int halo0 = alpha0 - m0;   // axis 0 (its own F(m0, r0) in per-axis plans)
  const int pl = g.pad[N - 1];
  g.dL = (tma && N >= 2) ? ((4 - pl % 4) % 4) : 0;
  g.R = 1;
  for (int n = 1; n < N; ++n) g.R *= g.tiles[n];
  g.R1 = 1;
  for (int n = 2; n < N; ++n) g.R1 *= g.tiles[n];
  int inner = 1;  // floats of one axis-0 slab slice
  // N = 3, alpha >= 6: H = axis-0 pass of the slab, [bt0][alpha][e1][hpitch]
  const bool hmode = N == 3 && alpha >= 6;
  // slab extents of axes >= 1 for bt1 axis-1 tiles per slab
  auto layout = [&](int bt1) {
    g.bt1 = N >= 2 ? bt1 : 1;
    inner = 1;
    for (int n = N - 1; n >= 1; --n) {
      g.e[n] = (n == 1 ? bt1 : g.tiles[n]) * m + halo;
      if (n == N - 1) {
        g.pitch = (g.e[n] + g.dL + 3) / 4 * 4;
        g.sst[n] = 1;
        inner = g.pitch;
      } else {
        g.sst[n] = inner;
        inner *= g.e[n];
      }
    }
    g.sst[0] = inner;
    g.hpitch = hmode ? (g.e[2] + 3) / 4 * 4 : 0;
  };
  auto slab = [&](int bt) {
    const int e0 = bt * m0 + halo0;
    if (N == 1) return (size_t)((e0 + 3) / 4 * 4) * 4;
    return (size_t)e0 * inner * 4;
  };
  auto hbytes = [&](int bt) { return hmode ? (size_t)bt * alpha0 * g.e[1] * g.hpitch * 4 : (size_t)0; };
  layout(N >= 2 ? g.tiles[1] : 1);
  // one slab (+ H) near 64 KB (48 KB in H mode: measured c4 337 -> 288 us at bt0 = 1)
  int bt0 = g.tiles[0];
  size_t target = hmode ? 48 * 1024 : 64 * 1024;
  if (const char* ev = getenv("WINO_IN_TARGET_KB")) target = (size_t)atoi(ev) * 1024;  // dev knob
  while (bt0 > 1 && slab(bt0) + hbytes(bt0) > target) bt0 = (bt0 + 1) / 2;
  // Large planes (N >= 3): when even a one-tile-deep slab is over 100 KB,
  // band axis 1 -- the widest divisor bt1 of tiles[1] whose slab meets the
  // target, else the widest that fits at all (C3D-size 112 x 112 planes,
  // large volumes).  Slabs up to 100 KB stay unbanded (the
  // measured BASELINE configs: c3 59 KB, c5 69 KB).
  g.nbox1 = 1;
  size_t band_at = 100 * 1024;
  if (const char* ev = getenv("WINO_IN_BAND_KB")) band_at = (size_t)atoi(ev) * 1024;  // dev / test knob
  if (N >= 3 && bt0 == 1 && slab(1) + hbytes(1) > band_at) {
    const int t1 = g.tiles[1];
    int pick = 0, fit = 0;
    for (int d = t1; d >= 1; --d) {
      if (t1 % d) continue;
      layout(d);
      const size_t sz = slab(1) + (hmode ? 0 : hbytes(1));   // in-place H mode (bt0 = 1)
      if (!fit && sz + 128 <= 200 * 1024) fit = d;
      if (sz <= target) { pick = d; break; }
    }
    if (!pick) pick = fit;
    if (!pick) pick = t1;
    layout(pick);
    g.nbox1 = t1 / pick;
  }
  g.Rs = g.bt1 * g.R1;
  if (N < 2) g.Rs = g.R;
  // H mode with a one-tile-deep slab: every slab column is private to the
  // thread that transforms it along axis 0, so the pass writes its alpha
  // outputs back into the column (no H buffer; several slabs fit a CTA)
  const char* ev_inpl = getenv("WINO_IN_HINPLACE");  // dev knob: 0 keeps the separate H
  g.hinplace = (hmode && bt0 == 1 && (!ev_inpl || atoi(ev_inpl) != 0)) ? 1 : 0;
  const size_t hb = g.hinplace ? 0 : hbytes(bt0);
  if (slab(bt0) + 128 + hb > 200 * 1024) return false;
  g.bt0 = bt0;
  g.npl = 1;  // plan_input_planes() raises it
  g.nbox0 = (g.tiles[0] + bt0 - 1) / bt0;
  g.e[0] = bt0 * m0 + halo0;
  if (N == 1) g.pitch = (g.e[0] + 3) / 4 * 4;
  g.in_threads = 256;
  if (const char* ev = getenv("WINO_IN_THREADS")) {  // dev knob, clamped to the kernel's launch bound
    const int tmax = hmode ? 512 : 256;               // (in_max_threads: 512 in H mode, else 256)
    g.in_threads = (atoi(ev) + 31) / 32 * 32;
    g.in_threads = g.in_threads < 64 ? 64 : g.in_threads > tmax ? tmax : g.in_threads;
  }
  g.in_flags = 0;
  if (const char* ev = getenv("WINO_IN_FLAGS")) g.in_flags = atoi(ev);  // dev A/B knob
  // line-aligned a2 work items: 1 = in-place H mode (c4 input 0.211 -> 0.185 ms), 2 = every path
  // (dev A/B: slower on c2 / c3), 0 = off
  g.in_align = 1;
  if (const char* ev = getenv("WINO_IN_ALIGN")) g.in_align = atoi(ev);
  g.in_prefetch = 0;
  if (const char* ev = getenv("WINO_IN_PREFETCH")) g.in_prefetch = atoi(ev);
  g.in_pad8 = 0;
  g.slab_bytes = (int)slab(bt0);
  g.slot_bytes = (g.slab_bytes + 127) / 128 * 128;
  g.smem_bytes = (int)(g.slot_bytes + hb);
  return true;
}

// Slabs per CTA (g.npl) for `nwork` work items: a CTA owns consecutive slabs
// of one channel (adjacent runs of t in V) and pools their work items, xi_0
// outermost in H mode, so each round of the block stores long runs of t per
// plane of V.  Measured (B200, tools/in_sweep.sh): c2 37.1 -> 32.8 us and c4
// 0.297 -> 0.247 ms at npl = 2 -> two slabs per CTA when they fit 64 KB,
// keeping >= 4 CTAs per SM of work; in-place H mode (aligned rows) four.
// Not with a separate H buffer.
void plan_input_planes(KGeom& g, int64_t nwork, int num_sms) {
  const bool pooled = g.hinplace || g.hpitch == 0;
  int npl = 1;
  if (pooled && 2 * g.slot_bytes <= 64 * 1024 && nwork / 2 >= 4LL * num_sms) npl = 2;
  // H mode in place (aligned phase-2 rows): four one-tile-deep slabs per CTA
  // when they fit ~104 KB (c4 input 0.237 -> 0.218 ms at npl 4 vs 2)
  // (deep slabs only: a single-plane slab -- F(1,1) along axis 0 -- keeps 2)
  if (g.hinplace && g.e[0] >= 4 && 4 * g.slot_bytes <= 104 * 1024 && nwork / 4 >= 2LL * num_sms) {
    npl = 4;
    // 384 threads for the 6 x 196 pooled items of a c4 CTA (measured: input
    // 0.216 -> 0.206 ms vs 256, 0.209 at 512)
    if (!getenv("WINO_IN_THREADS")) g.in_threads = 384;
  }
  if (const char* ev = getenv("WINO_IN_NPL")) npl = atoi(ev);  // dev knob
  if (npl < 1) npl = 1;
  if (npl > kMaxPlanes) npl = kMaxPlanes;
  if (!pooled) npl = 1;
  g.npl = npl;
  // in-place H mode with m = 4: phase-2 items on 8 slots per axis-1 row
  // (conflict-free 128-bit window loads; the wide tail load of the last real
  // tile stays inside the row), block size with the fewest idle item slots
  // in the last round (WINO_IN_PAD8=0, dev knob: dense items)
  const char* ev_p8 = getenv("WINO_IN_PAD8");
  const int tl2 = g.tiles[2];
  if (g.hinplace && g.m % 4 == 0 && g.e[0] > 1 && tl2 % 8 && (tl2 - 1) * g.m + 8 <= g.pitch &&
      (!ev_p8 || atoi(ev_p8) != 0)) {
    g.in_pad8 = 1;
    if (!getenv("WINO_IN_THREADS")) {
      const int64_t items = (int64_t)g.e[0] * npl * g.bt1 * ((tl2 + 7) / 8 * 8);   // alpha_0 (bt0 = 1) x slots
      int best = g.in_threads;
      int64_t waste = (items + best - 1) / best * best - items;
      for (int t = 256; t <= 512; t += 32) {
        const int64_t w = (items + t - 1) / t * t - items;
        if (w < waste) { waste = w; best = t; }
      }
      g.in_threads = best;
    }
  }
  g.smem_bytes = npl * g.slot_bytes + (pooled ? 0 : (g.smem_bytes - g.slot_bytes));
}

// TMA descriptor of x viewed as (in_{N-1}, .., in_0, B*C) with the slab box;
// false if the shape breaks a TMA rule (16-byte strides/base, box <= 256,
// supported column shift), in which case the cp.async path runs.
bool encode_input_map(CUtensorMap* tm, const float* x, const KGeom& g, int N, int B) {
  EncodeTiledFn enc = get_encode();
  if (!enc || N < 2 || ((uintptr_t)x & 15) || !(g.dL == 0 || g.dL == 3)) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  for (int k = 0; k < N; ++k) {  // TMA dim k = spatial axis N-1-k
    const int ax = N - 1 - k;
    dims[k] = (cuuint64_t)g.in[ax];
    box[k] = (cuuint32_t)(k == 0 ? g.pitch : g.e[ax]);
    if (k > 0) strides[k - 1] = (cuuint64_t)g.in_stride[ax] * 4;
  }
  dims[N] = (cuuint64_t)B * g.C;
  box[N] = 1;
  strides[N - 1] = (cuuint64_t)g.in_vol * 4;
  for (int k = 0; k < N; ++k) {
    if (box[k] > 256 || strides[k] % 16) return false;
  }
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, N + 1, const_cast<float*>(x), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static cudaError_t launch_input_xform1(int N, int alpha, int m, int spec, const float* x, float* V, const KGeom& g,
                                       const XfParams& xp, const CUtensorMap* tm, int nslab, cudaStream_t s) {
  if (spec != kSpecRuntime) return launch_input_const(N, alpha, m, spec, x, V, g, xp, tm, nslab, s);
  return launch_input_run(N, alpha, m, x, V, g, xp, tm, nslab, s);
}

// dev probe (WINO_IN_TRACE=<file>): every a2 launch records, per CTA, its SM
// and the %globaltimer at start / slabs landed / axis-0 pass done / end
// (H mode in place), and the last launch's records are written to <file>
// (one line per CTA).  The launch is synchronised; results stay valid.
cudaError_t launch_input_xform(int N, int alpha, int m, int spec, const float* x, float* V, const KGeom& g,
                               const XfParams& xp, const CUtensorMap* tm, int nslab, cudaStream_t s) {
  const char* path = getenv("WINO_IN_TRACE");
  if (!path) return launch_input_xform1(N, alpha, m, spec, x, V, g, xp, tm, nslab, s);
  const long long grid = ((long long)nslab * g.C + g.npl - 1) / g.npl;
  const size_t bytes = (size_t)grid * 8 * sizeof(unsigned long long);
  KGeom g1 = g;
  cudaError_t e = cudaMalloc(&g1.trace, bytes);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(g1.trace, 0, bytes, s);
  e = launch_input_xform1(N, alpha, m, spec, x, V, g1, xp, tm, nslab, s);
  cudaStreamSynchronize(s);
  unsigned long long* h = (unsigned long long*)malloc(bytes);
  cudaMemcpy(h, g1.trace, bytes, cudaMemcpyDeviceToHost);
  if (FILE* f = fopen(path, "w")) {
    for (long long b = 0; b < grid; ++b)
      fprintf(f, "%llu %llu %llu %llu %llu\n", h[b * 8], h[b * 8 + 1], h[b * 8 + 2], h[b * 8 + 3], h[b * 8 + 4]);
    fclose(f);
  }
  free(h);
  cudaFree(g1.trace);
  return e;
}

}  // namespace wino
