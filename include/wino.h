/*
 * wino.h -- C ABI of libwino.so, the B200 (sm_100a) N-dimensional Winograd
 * convolution layer F(m^N, r^N) of Budden et al., "Deep Tensor Convolution on
 * Multicores" (arXiv 1611.06565).  Citations: PAPER.md:<line> of the paper
 * text; DESIGN.md "readings" for every place the paper is silent.
 *
 * What one layer computes (Eq. (2), with b = 0, f = id):
 *
 *   y[b,k,o] = sum_c sum_{p in [0,r)^N} g[k,c,p] * xt[b,c,o+p-P]
 *
 * cross-correlation (no flip, reading #1), stride 1, symmetric zero padding P
 * per axis (reading #2), out_n = in_n + 2 P_n - r + 1.  It is evaluated by the
 * N-D fast algorithm of Eq. (4), batched per transform
 * point as in Eq. (5):
 *
 *   a0 host: exact-rational Toom-Cook synthesis of A^T (m x alpha),
 *      G (alpha x r), B^T (alpha x alpha), alpha = m + r - 1, from alpha
 *      interpolation points          [plan_create]
 *   a1 U_xi = (g[k,c] x_1 G ... x_N G)_xi   (kernel transform)  [filter_transform]
 *   a2 V_xi = (tile(b,c,t) x_1 B^T ... x_N B^T)_xi  (data transform)   [forward]
 *   a3 M_xi = V_xi U_xi, a [tiles x C] x [C x K] GEMM per point xi     [forward]
 *   a4 y tile = M[.][k][t] x_1 A^T ... x_N A^T, cropped/scattered      [forward]
 *
 * Conventions for every call:
 *  - Tensor pointers are DEVICE pointers (fp32, contiguous, row-major, on the
 *    plan's device) unless the name says _host.  The caller owns x, g, y and
 *    must keep them alive until the stream work completes.
 *  - Layouts: x [B][C][in_1]..[in_N], g [K][C][r]..[r] (r^N), y [B][K][out_1]..[out_N]
 *    (torch's contiguous convNd layout; reading #11).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls are stream-ordered and do not synchronise the host unless noted.
 *  - No exception crosses the ABI.  On failure a call returns a nonzero
 *    wino_status and wino_last_error() returns a thread-local message.
 *  - Concurrency: one call at a time per plan; distinct plans
 *    are independent.
 */
#ifndef WINO_H_
#define WINO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define WINO_API __attribute__((visibility("default")))
#else
#define WINO_API
#endif

typedef struct wino_plan_s* wino_plan_t;
typedef void* wino_stream_t; /* a cudaStream_t */

typedef enum {
  WINO_OK = 0,
  WINO_ERR_ARG = 1,         /* N not in 1..4, m/r/C/K/batch < 1, NULL pointer, B > planned batch */
  WINO_ERR_SHAPE = 2,       /* kernel larger than the padded input (out_n < 1) */
  WINO_ERR_POINTS = 3,      /* point list unparsable, duplicate, >1 infinity, count != alpha */
  WINO_ERR_SYNTH = 4,       /* exact identity check failed, or rational overflow */
  WINO_ERR_STATE = 5,       /* forward before the filter transform */
  WINO_ERR_UNSUPPORTED = 6, /* alpha_n > 8, prod alpha_n > 65535, > 2^31 tiles, or an unknown fuse bit */
  WINO_ERR_CUDA = 7,        /* CUDA launch/runtime error (incl. async errors surfaced here) */
  WINO_ERR_NOMEM = 8        /* device or pinned allocation failed */
} wino_status;

/* GEMM schemes for stage a3 (all fp32-accurate except WINO_GEMM_1XTF32). */
enum {
  WINO_GEMM_AUTO = 0,   /* = WINO_GEMM_3XTF32 */
  WINO_GEMM_FFMA = 1,   /* CUDA-core fp32 FMA, smem-tiled */
  WINO_GEMM_1XTF32 = 2, /* single tf32 product: debug/accuracy experiments only */
  WINO_GEMM_3XTF32 = 3, /* tcgen05 kind::tf32, hi*hi + hi*lo + lo*hi, TMEM fp32 accumulators */
  WINO_GEMM_3XF16 = 4   /* tcgen05 kind::f16 (2x the tf32 rate): V, U scaled by powers of two
                           (max|V| from the input transform, max|U| from the filter transform)
                           and split into fp16 hi + lo; hi*hi + hi*lo + lo*hi, fp32 accumulators;
                           single-(m, r) fused plans with K > 64, k-chunk 32 or 64 */
};

/* Activation f of Eq. (2) for wino_forward_ex. */
enum { WINO_ACT_NONE = 0, WINO_ACT_RELU = 1 };

/* Fusion bitmask (plan_create_ex `fuse`). */
enum {
  WINO_FUSE_NONE = 0,
  WINO_FUSE_L2_CHUNK = 4 /* run a2->a3->a4 over tile chunks sized to stay L2-resident */
};

/* ---- plan lifetime -------------------------------------------------------
 * wino_plan_create: validate arguments, synthesise the transforms exactly for
 * the default points of alpha (reading #5), check the Eq. (1)
 * identity exactly (else WINO_ERR_SYNTH), upload fp32/fp64 constants, and
 * allocate the transformed-filter buffer U and the workspace (V, M) for up
 * to `batch` samples on the current device.
 * Device work at plan creation (none of it on the caller's streams): the
 * workspace is zeroed, and the tcgen05 GEMM variant / N tile are chosen by
 * timing the supported candidates on the plan's own workspace (about 4 rounds
 * x up to 6 candidates x 3 GEMM launches, milliseconds).  Both run on a
 * private non-blocking stream that is synchronised before returning (the
 * device and other streams are not), and the timing choice is cached per
 * (device, shape) in the process, so a second plan of the same shape
 * launches no timing kernels.  The choice never changes results: every
 * variant computes bit-identical outputs (tests/test_gpu_parity.py).  The
 * environment variable WINO_GEMM_VARIANT=0/1/2 fixes the variant without
 * timing.
 *   N        number of spatial dims, 1..4
 *   dims     N input extents in_n >= 1
 *   m, r     output-tile length S and kernel length G of F(m, r)
 *   C, K     input channels M and output channels / kernels K
 *   batch    largest batch a forward call will pass
 *   padding  N symmetric zero-pad amounts P_n >= 0 (NULL = all zero)
 * On success *plan owns all device memory it allocated. */
WINO_API wino_status wino_plan_create(wino_plan_t* plan, int N, const int64_t* dims, int m, int r,
                             int C, int K, int batch, const int* padding);

/* As above with explicit choices.
 *   points    NULL = default; else alpha comma-separated rationals in row
 *             order, e.g. "0,3/2,-3/2,2/3,-2/3,inf" (at most one "inf").
 *   gemm_mode WINO_GEMM_* (0 = 3xTF32 on tcgen05).
 *   fuse      WINO_FUSE_* bitmask (0 = three stream-ordered kernels).
 *   device    CUDA device ordinal, -1 = current.
 * Kernel selection: (N, alpha, m) with fused transform kernels (alpha, m in
 * {(4,2), (4,3), (6,4), (8,5), (8,4), (8,3), (5,3), (6,3)}, N <= 3, and N = 4
 * with alpha = 4) take them; large N >= 3 planes band the input slab along
 * axis 1 (info in_bands).  Every other F(m, r) with alpha <= 8 -- alpha = 7,
 * F(2,5), F(2,4), F(4,2), N = 4 with alpha > 4 -- and planes too large even
 * for one band run the generic multi-pass transforms (info axis_mode 2;
 * same GEMM, results equal up to rounding; `fuse` is then ignored). */
WINO_API wino_status wino_plan_create_ex(wino_plan_t* plan, int N, const int64_t* dims, int m, int r,
                                int C, int K, int batch, const int* padding, const char* points,
                                int gemm_mode, int fuse, int device);

/* Per-axis transforms F(m_1 x .. x m_N, r_1 x .. x r_N): Eq. (4) indexes A_n,
 * B_n, C_n by axis, e.g. F(2,3) along time and F(4,3)
 * along space, or anisotropic kernels r = (1,3,3).  m[0..N), r[0..N) >= 1
 * with alpha_n = m_n + r_n - 1 <= 8 and prod alpha_n <= 65535; default
 * points per alpha_n; g is [K][C][r_1]..[r_N].  Equal (m_n, r_n) on every
 * axis returns the plan of wino_plan_create_ex (fused kernels); N = 2, 3 with
 * a distinct axis 0 over equal other axes, each of F(2,3), F(4,3), F(1,1),
 * runs fused kernels with an axis-0 transform of its own (info axis_mode 1);
 * any other mix runs generic multi-pass transforms around the same GEMM
 * (axis_mode 2).  No fusion bitmask.  Errors as wino_plan_create_ex. */
WINO_API wino_status wino_plan_create_nd(wino_plan_t* plan, int N, const int64_t* dims, const int* m,
                                         const int* r, int C, int K, int batch, const int* padding,
                                         int gemm_mode, int device);

/* Frees every device/host buffer of the plan.  The caller must ensure no work
 * using the plan is still in flight (synchronise first).  NULL is a no-op. */
WINO_API wino_status wino_plan_destroy(wino_plan_t plan);

/* ---- hot path --------------------------------------------------------------
 * a1: U = g x_n G (fp64 arithmetic, one rounding to fp32, then the tf32 hi/lo
 * split), cached in the plan until the next call ("transformed kernels are
 * cached").  g: device [K][C][r^N]. */
WINO_API wino_status wino_filter_transform(wino_plan_t plan, const float* g, wino_stream_t stream);

/* a2 -> a3 -> a4 on `stream`, no host synchronisation.  x: device
 * [B][C][in...], y: device [B][K][out...], 1 <= B <= planned batch.
 * WINO_ERR_STATE if no filter transform (or mark_ready) happened. */
WINO_API wino_status wino_forward(wino_plan_t plan, const float* x, float* y, int B, wino_stream_t stream);

/* The full layer of Eq. (2), d' = f(b + conv):
 *   bias        device [K] fp32 per-output-channel bias b, or NULL (b = 0)
 *   activation  WINO_ACT_NONE (f = identity) or WINO_ACT_RELU (f = max(., 0))
 * applied in the spatial domain inside the output transform (a4), after A^T
 * (SURVEY NEXT-2); otherwise identical to wino_forward (which is
 * wino_forward_ex(plan, x, y, B, NULL, WINO_ACT_NONE, stream)). */
WINO_API wino_status wino_forward_ex(wino_plan_t plan, const float* x, float* y, int B, const float* bias,
                                     int activation, wino_stream_t stream);

/* End-to-end variant with HOST buffers x_host (B x C x in...) and y_host
 * (B x K x out...).  The batch is split into up to 8 sample chunks pipelined
 * over three streams (H2D copies, the forward on `stream`, D2H copies) into
 * plan-owned device buffers, so both copy directions overlap the compute;
 * synchronises before returning.  Host buffers should be pinned
 * (cudaHostAlloc / torch pin_memory) for full PCIe bandwidth and overlap. */
WINO_API wino_status wino_forward_host(wino_plan_t plan, const float* x_host, float* y_host, int B,
                              wino_stream_t stream);

/* ---- queries ---------------------------------------------------------------- */
/* out[0..N): output extents. */
WINO_API wino_status wino_plan_out_dims(wino_plan_t plan, int64_t* out);
/* Device bytes: workspace (V + M) and filter buffer (U_hi + U_lo). */
WINO_API wino_status wino_plan_sizes(wino_plan_t plan, size_t* workspace_bytes, size_t* filter_bytes);
/* info[0..25): N, m, r, alpha, C, K, batch, T_per_sample, T_stride, n_points
 * (alpha^N), K_stride, gemm_mode, fuse, n_blk, k_chunk, chunk_slabs (0 =
 * unchunked), gemm_variant (0 SMEM-A, 1 TMEM-A, 2 CTA-pair; -1 FFMA; chosen by
 * timing the supported variants once in plan_create), input slab depth bt0,
 * input slabs per CTA npl, axis mode (0 one F(m, r) on every axis, 1 fused
 * kernels with a distinct axis-0 F(m0, r0), 2 generic per-axis passes), tiny
 * (1: the whole forward runs in one kernel, chosen for tiny layers), launches
 * (kernel launches of one full-batch forward), in_bands (axis-1 bands of the
 * fused input transform's slab: 1 unbanded, > 1 for large N >= 3 planes, 0
 * on the generic path), fold (F > 0: the output transform of the F innermost
 * axes is folded into the GEMM, a5; 0: unfused), fold_mode (1: epilogue fold
 * of the accumulators, gemm_fold.cu; 2: filter-side fold, A^T of those axes
 * multiplied into the cached transformed filter U' at wino_filter_transform
 * time and the GEMM run as (n_points / alpha^F) GEMMs of depth alpha^F * C
 * and width m^F * K; 3: the direct-axis fold, F = 1 -- as 2, and B^T of the
 * innermost axis is folded into U' as well, so the input transform covers
 * the outer axes only (the workspace's V region then holds Z [n_points /
 * alpha * 2][C][slots], 32 slots per row of tiles of the last axis: even /
 * odd zero-padded input columns) and the GEMM computes the innermost axis as
 * a direct correlation, PAPER.md:52-56 / Eq. (4); same results within the
 * plan's tolerance; 0: none). */
WINO_API wino_status wino_plan_info(wino_plan_t plan, int64_t* info);

/* ---- multi-GPU hooks (U is computed once and NCCL-broadcast) ------------------
 * The filter buffer (U_hi then U_lo, contiguous) for an external broadcast;
 * after filling it on another rank call wino_filter_mark_ready. */
WINO_API wino_status wino_filter_buffer(wino_plan_t plan, void** dev_ptr, size_t* bytes);
WINO_API wino_status wino_filter_mark_ready(wino_plan_t plan);

/* ---- test / stage hooks --------------------------------------------------------
 * Device pointers of the unfused workspace: V [n_points][C][T_stride] and
 * M [n_points][K][T_stride] (valid after a forward with fuse == 0).  Under
 * an a5 fold (wino_plan_info fold_mode) the M region holds W
 * [n_points / alpha^F * m^F][K][T_stride]; under fold_mode 3 the V region
 * holds Z (see wino_plan_info). */
WINO_API wino_status wino_workspace(wino_plan_t plan, void** V, void** M);

/* Per-stage CUDA-event timing of forward calls (bench instrumentation).
 * enable=1 starts recording (resets accumulators); ms[0..3) receives the
 * summed milliseconds of input transform, GEMM, output transform over the
 * recorded calls and *calls their number (synchronises the recorded events). */
WINO_API wino_status wino_profile_enable(wino_plan_t plan, int enable);
WINO_API wino_status wino_profile_read(wino_plan_t plan, double* ms, int* calls);

/* Host-only exact synthesis (no device needed).  Fills, for F(m, r) with the
 * given points (NULL = default), AT (m x alpha), G (alpha x r), BT
 * (alpha x alpha) as doubles (RNE from exact rationals) and, if json != NULL,
 * a JSON document {"m","r","alpha","points","AT","G","BT"} of exact rational
 * strings (truncated to `cap` bytes, NUL-terminated). */
WINO_API wino_status wino_synthesize(int m, int r, const char* points, double* AT, double* G, double* BT,
                            char* json, size_t cap);
/* The plan's transforms, same format. */
WINO_API wino_status wino_get_transforms(wino_plan_t plan, double* AT, double* G, double* BT, char* json,
                                size_t cap);

/* Thread-local message for the last failing call on this thread ("" if none). */
WINO_API const char* wino_last_error(void);
/* Library version string. */
WINO_API const char* wino_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WINO_H_ */
