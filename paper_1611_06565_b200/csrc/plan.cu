// plan.cu -- the C ABI of include/wino.h: argument validation, geometry,
// exact transform synthesis (stage a0), device buffers, stage launches.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"
#include "synth.hpp"
#include "wino.h"

using namespace wino;

namespace {

thread_local std::string g_err;

wino_status fail(wino_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? WINO_ERR_NOMEM : WINO_ERR_CUDA,       \
                  "%s failed: %s", #expr, cudaGetErrorString(e_));                       \
  } while (0)

// ---- exact points --------------------------------------------------------
bool parse_int(const char*& s, int64_t& v) {
  while (*s == ' ') ++s;
  bool neg = false;
  if (*s == '+' || *s == '-') neg = (*s++ == '-');
  if (*s < '0' || *s > '9') return false;
  __int128 acc = 0;
  while (*s >= '0' && *s <= '9') {
    acc = acc * 10 + (*s++ - '0');
    if (acc > (__int128)INT64_MAX) return false;
  }
  v = (int64_t)(neg ? -acc : acc);
  return true;
}

// "0,3/2,-3/2,inf" -> points; returns count or -1
int parse_points(const char* spec, Point* out, int cap) {
  int n = 0;
  const char* s = spec;
  while (true) {
    while (*s == ' ') ++s;
    if (n >= cap) return -1;
    Point p;
    if (!strncmp(s, "inf", 3) || !strncmp(s, "INF", 3)) {
      p.inf = true;
      s += 3;
      if (!strncmp(s, "inity", 5)) s += 5;
    } else {
      int64_t num, den = 1;
      if (!parse_int(s, num)) return -1;
      while (*s == ' ') ++s;
      if (*s == '/') {
        ++s;
        if (!parse_int(s, den) || den == 0) return -1;
      }
      RatOps o;
      p.v = o.make(num, den);
      if (o.overflow) return -1;
    }
    out[n++] = p;
    while (*s == ' ') ++s;
    if (*s == ',') { ++s; continue; }
    if (*s == 0) break;
    return -1;
  }
  return n;
}

bool same_points(const Point* a, const Point* b, int n) {
  for (int i = 0; i < n; ++i) {
    if (a[i].inf != b[i].inf) return false;
    if (!a[i].inf && !req(a[i].v, b[i].v)) return false;
  }
  return true;
}

std::string rat_str(Rat q) {
  char buf[64];
  if (q.d == 1) snprintf(buf, sizeof buf, "%lld", (long long)q.n);
  else snprintf(buf, sizeof buf, "%lld/%lld", (long long)q.n, (long long)q.d);
  return buf;
}

std::string transforms_json(const Transforms& t) {
  std::string j = "{\"m\":" + std::to_string(t.m) + ",\"r\":" + std::to_string(t.r) +
                  ",\"alpha\":" + std::to_string(t.a) + ",\"points\":[";
  for (int k = 0; k < t.a; ++k) {
    if (k) j += ",";
    j += "\"" + (t.pts[k].inf ? std::string("inf") : rat_str(t.pts[k].v)) + "\"";
  }
  auto mat = [&](const char* name, const Rat (*M)[kMaxAlpha], int rows, int cols) {
    j += std::string("],\"") + name + "\":[";
    for (int i = 0; i < rows; ++i) {
      if (i) j += ",";
      j += "[";
      for (int c = 0; c < cols; ++c) {
        if (c) j += ",";
        j += "\"" + rat_str(M[i][c]) + "\"";
      }
      j += "]";
    }
  };
  mat("AT", t.AT, t.m, t.a);
  mat("G", t.G, t.a, t.r);
  mat("BT", t.BT, t.a, t.a);
  j += "]}";
  return j;
}

wino_status synth_checked(int m, int r, const char* points, Transforms& t, int& spec) {
  if (m < 1 || r < 1) return fail(WINO_ERR_ARG, "m and r must be >= 1 (m=%d r=%d)", m, r);
  const int a = m + r - 1;
  if (a > kMaxAlpha) return fail(WINO_ERR_UNSUPPORTED, "alpha = m + r - 1 = %d exceeds %d", a, kMaxAlpha);
  Point pts[kMaxAlpha]{};
  Point def[kMaxAlpha]{}, seq[kMaxAlpha]{};
  default_points(a, kPsDefault, def);
  const bool have_seq = default_points(a, kPsSeq, seq) == 0;
  if (points == nullptr || *points == 0) {
    for (int i = 0; i < a; ++i) pts[i] = def[i];
  } else {
    const int n = parse_points(points, pts, kMaxAlpha);
    if (n < 0) return fail(WINO_ERR_POINTS, "cannot parse points \"%s\"", points);
    if (n != a) return fail(WINO_ERR_POINTS, "need alpha = m + r - 1 = %d points, got %d", a, n);
  }
  t = synthesize(m, r, pts);
  if (t.err == 3) return fail(WINO_ERR_POINTS, "points must be distinct with at most one infinity");
  if (t.err) return fail(WINO_ERR_SYNTH, "exact synthesis/identity check failed for F(%d,%d)", m, r);
  spec = kSpecRuntime;
  if (r == 3 && (m == 2 || m == 4)) {
    if (same_points(pts, def, a)) spec = kSpecDefault;
    else if (have_seq && same_points(pts, seq, a)) spec = kSpecSeq;
  }
  return WINO_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Zero device memory at plan creation on a private non-blocking stream (no
// implicit synchronisation with the caller's streams or the legacy stream).
cudaError_t zero_private(void* ptr, size_t bytes) {
  cudaStream_t s = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(ptr, 0, bytes, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return e != cudaSuccess ? e : e2;
}

constexpr int kMaxProf = 4096;
constexpr int kHostChunks = 16;  // wino_forward_host pipeline depth

}  // namespace

struct wino_plan_s {
  int N = 0, m = 0, r = 0, a = 0, C = 0, K = 0, batch = 0, gemm_mode = 0, fuse = 0, device = 0, spec = 0;
  int64_t in[kMaxN]{}, out[kMaxN]{};
  int pad[kMaxN]{}, tiles[kMaxN]{};
  int64_t Tps = 0, T_s = 0, P = 0, K_s = 0;
  Transforms tf{};
  XfParams xp{};
  FParams fp{};
  KGeom geom{};
  float* ubuf = nullptr;  // U_hi | U_lo | (U32)
  float *Uhi = nullptr, *Ulo = nullptr, *U32 = nullptr;
  size_t filter_bytes = 0, filter_bcast_bytes = 0;
  float *V = nullptr, *M = nullptr;
  size_t ws_bytes = 0;
  float *x_dev = nullptr, *y_dev = nullptr;   // wino_forward_host staging
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t e_in[kHostChunks]{}, e_fw[kHostChunks]{}, e_start = nullptr;
  bool filter_ready = false;
  TcGemm tg{};
  CUtensorMap tm_x{};          // input-transform TMA map (cached per x pointer / B)
  CUtensorMap tm_M{};          // output-transform TMA map of M (fixed workspace)
  bool tm_M_ok = false;
  const float* tm_x_ptr = nullptr;
  int tm_x_B = 0;
  bool tm_x_ok = false;
  bool use_tma_in = true;      // env WINO_IN_TMA=0 forces the cp.async path
  // L2-chunked pipeline (fuse & WINO_FUSE_L2_CHUNK): V and M hold one chunk
  // of chunk_slabs input slabs (rows t - t_lo), sized to stay L2-resident
  bool chunked = false;
  int64_t chunk_slabs = 0;
  // per-axis (m_n, r_n) plan (wino_plan_create_nd with unequal axes):
  // generic multi-pass transforms (xform_nd.cu), scratch W for the output passes
  bool nd = false;
  // tiny layers: the whole forward in one kernel (xform_tiny.cu)
  bool tiny = false;
  // fused plan with a distinct axis 0 (F(m0, r0); xform_mixed.cu)
  bool mixed = false;
  int m0 = 0, r0 = 0, a0 = 0;
  int mn[kMaxN]{}, rn[kMaxN]{}, an[kMaxN]{};
  NdParams ndp{};
  float* W = nullptr;
  // a5: output transform of the fold_F innermost axes in the GEMM epilogue
  // (gemm_fold.cu); the M buffer then holds W [P/Q * MO][K][T_s]
  int fold_F = 0, fold_Q = 1, fold_MO = 1, fold_bn = 0, fold_g = 0;
  FoldTab fold_tab{};
  // a5 filter-side fold (kernels.h, UFoldTab): uf_F > 0 folds A^T of the
  // uf_F innermost axes into U' at filter-transform time; the GEMM is then
  // the plain batched GEMM of shape (gP, gC, gK) = (P/Q, Q*C, MO*K) writing W
  int uf_F = 0;
  UFoldTab uf_tab{};
  int64_t gP = 0;
  int gC = 0, gK = 0;
  int zmask = 0;   // U' chunks that are zero by construction (skipped by the V-resident f16 GEMM)
  // a5 direct-axis fold (xform_dfold.cu, reading #21): with uf_F = 1,
  // B^T of the last axis is folded into U' as well -- the GEMM's A operand is
  // Z (outer axes transformed, last axis raw; in the V buffer), U' holds the
  // outer-axes filter transform per tap, and the last axis is computed directly
  bool df = false;
  int64_t df_Tz = 0;          // slot pitch of a Z plane
  CUtensorMap tmA_df{};
  bool f16n = true;   // 3xFP16: the V-resident kernel where it applies (WINO_F16N=0, dev knob: k_gemm_f16p)
  // 3xFP16 GEMM (gemm_f16.cu): U as scaled fp16 halves in ubuf (hi | lo |
  // tail: uscal, umax | fp32 staging of the filter transform), vmax: max|V|
  // word (a2 maxes it, the GEMM reads it, a4 clears it)
  bool f16 = false;
  void *U16hi = nullptr, *U16lo = nullptr;
  float* uscal = nullptr;
  unsigned int* umax = nullptr;
  float* U32tmp = nullptr;
  unsigned int* vmax = nullptr;
  CUtensorMap tmBhi16{}, tmBlo16{};
  bool prof = false;
  int prof_calls = 0;
  std::vector<cudaEvent_t> ev;  // pool; prof_stage[i] tags pair (2i, 2i+1)
  std::vector<int> prof_stage;
};

extern "C" {

const char* wino_last_error(void) { return g_err.c_str(); }
const char* wino_version(void) { return "wino-nd-b200 0.1 (sm_100a)"; }

wino_status wino_synthesize(int m, int r, const char* points, double* AT, double* G, double* BT, char* json,
                            size_t cap) {
  Transforms t;
  int spec;
  wino_status st = synth_checked(m, r, points, t, spec);
  if (st) return st;
  const int a = t.a;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < a; ++j)
      if (AT) AT[i * a + j] = rat_to_f64(t.AT[i][j]);
  for (int i = 0; i < a; ++i)
    for (int j = 0; j < r; ++j)
      if (G) G[i * r + j] = rat_to_f64(t.G[i][j]);
  for (int i = 0; i < a; ++i)
    for (int j = 0; j < a; ++j)
      if (BT) BT[i * a + j] = rat_to_f64(t.BT[i][j]);
  if (json && cap) {
    const std::string s = transforms_json(t);
    const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    memcpy(json, s.data(), n);
    json[n] = 0;
  }
  return WINO_OK;
}

static wino_status create_generic(wino_plan_t* plan_out, int N, const int64_t* dims, const int* m, const int* r,
                                  const char* points, int C, int K, int batch, const int* padding, int gemm_mode,
                                  int device);

// a5 epilogue fusion (gemm_fold.cu): fold the output transform of the F
// innermost axes into the GEMM.  F from WINO_FOLD (dev knob) else the
// measured default (fold_default); kept only where the folded kernels are
// instantiated.  coef[q][o] = prod_f A^T[o_f][q_f], exact then RNE to fp32.
static int fold_default(const wino_plan_s* p) {
  // F(2^N, 3^N) with the default points, F = 2 (tools/fold_bench.sh, B200,
  // ms per layer): c5 (N = 4) 0.192 -> 0.158 (GEMM 0.092 -> 0.085, a4 0.052 ->
  // 0.019); c3 (N = 3) 1.700 -> 1.655 (GEMM 0.84 -> 1.17, a4 0.54 -> 0.19).
  // Not F = 1 on c3 (1.73: the 64-wide N tile doubles the conversions) nor
  // F(4^2, 3^2) (c2 0.100 -> 0.155: 128 channels through a 32-wide tile)
  if (p->a == 4 && p->m == 2 && p->N >= 3) return 2;
  return 0;
}

static void plan_fold(wino_plan_s* p) {
  int F = fold_default(p);
  if (const char* ev = getenv("WINO_FOLD")) F = atoi(ev);
  if (F < 1 || F >= p->N) return;
  const int a = p->a, m = p->m;
  const int Q = ipow(a, F), MO = ipow(m, F);
  if (Q > kMaxFoldQ || MO > kMaxFoldMO || !output_fold_supported(p->N, a, m, F, p->spec)) return;
  int bn = 0, g = 0;
  if (!fold_shape(p->K, MO, p->tg.kc, &bn, &g) || !fold_feasible(bn, p->tg.kc, p->C, Q)) return;
  for (int q = 0; q < Q; ++q)
    for (int o = 0; o < MO; ++o) {
      RatOps ro;
      Rat c{1, 1};
      int qq = q, oo = o;
      for (int f = 0; f < F; ++f) {   // digits, last axis fastest
        c = ro.mul(c, p->tf.AT[oo % m][qq % a]);
        qq /= a;
        oo /= m;
      }
      p->fold_tab.coef[q][o] = rat_to_f32(c);
    }
  p->fold_F = F;
  p->fold_Q = Q;
  p->fold_MO = MO;
  p->fold_bn = bn;
  p->fold_g = g;
}

// a5 filter-side fold depth F for a fused-kernel plan: WINO_UFOLD (dev knob)
// else the measured default (0: off).
static int ufold_default(int N, int a, int m, int C, int K) {
  // F(2^3, 3^3), F = 1 (tools/ufold_bench.sh, tools/f16n_ab.sh, B200, ms per
  // layer): c3 1.69 (epilogue fold F = 2, 3xTF32) -> 1.28 (GEMM 1.14 -> 0.57,
  // a4 0.19 -> 0.31).  Not F(4^2, 3^2) (c2 0.102 -> 0.133: the 4x wider GEMM
  // is tensor-bound) nor N = 4 (c5: only F >= 2 exists there, see below).
  // An explicit WINO_FOLD (the epilogue-fold dev knob) turns this default off.
  // Only where the folded GEMM (alpha C deep, m K wide) takes the 3xFP16
  // scheme (auto_gemm_mode: both >= 128), as measured.
  if (getenv("WINO_FOLD")) return 0;
  if (a == 4 && m == 2 && N == 3 && a * C >= 128 && m * K >= 128) return 1;
  return 0;
}
// F = 1 only: the fold lengthens each TMEM accumulation chain Q = alpha^F
// times (Q*C terms per accumulator), and the tensor core's fp32 accumulation
// error grows with it (measured, ragged c3-like layer, relL2 vs float64:
// unfused / epilogue fold 3.9e-7, filter-side F = 1 6.1e-7 (3xFP16) / 1.0e-6
// (3xTF32), F = 2 1.6e-6 / 2.9e-6, F(2^4,3^4) F = 3 4.2e-6 / 8.3e-6 --
// BASELINE.json's 2e-6 budget holds only at F = 1).
constexpr int kMaxUFoldF = 1;

// coef[q][o] = prod_f A^T[o_f][q_f] over the F innermost axes (last axis fastest)
static void fold_coefs(const Transforms& t, int F, UFoldTab& uf) {
  const int a = t.a, m = t.m;
  uf.Q = ipow(a, F);
  uf.MO = ipow(m, F);
  for (int q = 0; q < uf.Q; ++q)
    for (int o = 0; o < uf.MO; ++o) {
      RatOps ro;
      Rat c{1, 1};
      int qq = q, oo = o;
      for (int f = 0; f < F; ++f) {
        c = ro.mul(c, t.AT[oo % m][qq % a]);
        qq /= a;
        oo /= m;
      }
      uf.coef[q][o] = rat_to_f64(c);
    }
}

// a5 direct-axis fold on top of the filter-side fold F = 1 where it applies
// (F(2^3,3^3), V-resident 3xFP16 GEMM): default on (measured);
// WINO_DFOLD=0 (dev knob) keeps the plain filter-side fold.
// Default rule: at least 24 tiles along the last axis (Z rows are 32 slots
// wide, so fewer tiles waste GEMM rows);
// WINO_DFOLD=1 takes it wherever the kernels apply (tests), 0 never.
static bool dfold_wanted(int tiles_last) {
  const char* ev = getenv("WINO_DFOLD");
  if (ev) return atoi(ev) != 0;
  return tiles_last >= 24;
}

// Zero U' chunks of the filter-side fold: bit nb * 8 + ch is set when every
// column of n-block nb (width bn) has A^T_F[o][q] = 0 for the chunk's point q
// (chunks of kc channels, C a multiple of kc so a chunk holds one q); an
// n-block keeps at least one chunk.  WINO_UFOLD_SKIP=0 (dev knob): no skips.
static int ufold_zmask(const wino_plan_s* p, int bn) {
  const char* ev = getenv("WINO_UFOLD_SKIP");
  if (ev && atoi(ev) == 0) return 0;
  const int kc = p->tg.kc, n_chunks = p->gC / kc, nnb = (p->gK + bn - 1) / bn;
  if (n_chunks > 8 || nnb > 4) return 0;
  int mask = 0;
  for (int nb = 0; nb < nnb; ++nb) {
    int mnb = 0;
    for (int ch = 0; ch < n_chunks; ++ch) {
      const int q = ch * kc / p->C;
      bool zero = true;
      for (int col = nb * bn; col < (nb + 1) * bn && col < p->gK; ++col)
        if (p->uf_tab.coef[q][col / p->K] != 0.0) zero = false;
      if (zero) mnb |= 1 << ch;
    }
    if (mnb != (1 << n_chunks) - 1) mask |= mnb << (nb * 8);
  }
  return mask;
}

// WINO_GEMM_AUTO's scheme for a fused-kernel plan: 3xTF32 unless the 3xFP16
// split (twice the tensor rate) applies; WINO_GEMM_AUTO_MODE=3/4 overrides
// (dev knob).  See fold_default / DESIGN.md for the measurements.
static int auto_gemm_mode(int N, int a, int m, int C, int K, bool mixed, int fuse) {
  (void)N; (void)a; (void)m; (void)mixed;
  const bool f16_ok = K > 64 && C >= 32 && !(fuse & WINO_FUSE_L2_CHUNK);   // (f16_supported, checked again later)
  if (const char* ev = getenv("WINO_GEMM_AUTO_MODE")) {
    const int v = atoi(ev);
    return v == WINO_GEMM_3XF16 && f16_ok ? v : WINO_GEMM_3XTF32;
  }
  // 3xFP16 where measured faster (tools/nbfast.sh, B200, ms per layer): c4
  // (C = K = 256) 0.733 -> 0.685 (GEMM 0.369 -> 0.295: tensor-bound in
  // 3xTF32), c2 (C = K = 128) 0.1034 -> 0.1011; not c3 (C = 64: 1.73 -> 1.80,
  // the k-chunk of 32 leaves too little tensor work per handshake)
  if (f16_ok && C >= 128 && K >= 128) return WINO_GEMM_3XF16;
  return WINO_GEMM_3XTF32;
}

// WINO_ND_GENERIC=1: every plan takes the generic multi-pass transforms (dev / test knob)
static bool force_generic() {
  const char* ev = getenv("WINO_ND_GENERIC");
  return ev && atoi(ev) != 0;
}

// The fused-kernel plan: F(m, r) on axes 1..N-1 and F(m0, r0) on axis 0
// (m0 = m, r0 = r for single-(m, r) plans; a distinct axis 0 only for the
// instantiated per-axis combinations, mixed_supported()).
static wino_status create_core(wino_plan_t* plan_out, int N, const int64_t* dims, int m0, int r0, int m, int r, int C,
                               int K, int batch, const int* padding, const char* points, int gemm_mode, int fuse,
                               int device) {
  if (!plan_out) return fail(WINO_ERR_ARG, "plan pointer is NULL");
  *plan_out = nullptr;
  if (N < 1 || N > kMaxN) return fail(WINO_ERR_ARG, "N must be in 1..4 (got %d)", N);
  if (!dims) return fail(WINO_ERR_ARG, "dims is NULL");
  if (C < 1 || K < 1 || batch < 1) return fail(WINO_ERR_ARG, "C, K, batch must be >= 1");
  if (gemm_mode < 0 || gemm_mode > 4) return fail(WINO_ERR_ARG, "bad gemm_mode %d", gemm_mode);
  if (fuse & ~WINO_FUSE_L2_CHUNK) return fail(WINO_ERR_UNSUPPORTED, "fuse bitmask %d not implemented in this build", fuse);
  Transforms t, t0;
  int spec, spec0;
  wino_status st = synth_checked(m, r, points, t, spec);
  if (st) return st;
  const bool mixed = m0 != m || r0 != r;
  if (mixed) {
    st = synth_checked(m0, r0, nullptr, t0, spec0);
    if (st) return st;
  } else {
    t0 = t;
    spec0 = spec;
  }
  const int a = t.a, a0 = t0.a;
  // (mixed plans come from wino_plan_create_nd with default points on every
  // axis: exactly the compile-time tables of xform_mixed.cu)
  if (mixed && (points || fuse || !mixed_supported(N, a0, m0, a, m)))
    return fail(WINO_ERR_UNSUPPORTED, "no fused kernels for axis-0 F(%d,%d) with F(%d,%d) on N=%d", m0, r0, m, r, N);
  if (a > kMaxA || a0 > kMaxA)
    return fail(WINO_ERR_UNSUPPORTED, "alpha = %d exceeds %d on the device path", a > a0 ? a : a0, kMaxA);
  // single-(m, r) plans without fused kernels for (N, alpha, m) take the
  // generic multi-pass transforms (same GEMM, same results up to rounding)
  const int mv[kMaxN] = {m, m, m, m}, rv[kMaxN] = {r, r, r, r};
  if (!mixed && (!xform_supported(N, a, m, spec) || force_generic()))
    return create_generic(plan_out, N, dims, mv, rv, points, C, K, batch, padding, gemm_mode, device);

  wino_plan_s* p = new wino_plan_s();
  p->N = N; p->m = m; p->r = r; p->a = a; p->C = C; p->K = K; p->batch = batch;
  p->mixed = mixed;
  p->m0 = m0; p->r0 = r0; p->a0 = a0;
  {
    // a5 filter-side fold: tensor-core GEMMs only, single-(m, r) plans with
    // the folded output kernels instantiated, no L2 chunking
    int F = ufold_default(N, a, m, C, K);
    if (const char* ev = getenv("WINO_UFOLD")) F = atoi(ev);
    const bool tc_req = gemm_mode == WINO_GEMM_AUTO || gemm_mode == WINO_GEMM_3XTF32 || gemm_mode == WINO_GEMM_3XF16;
    if (F >= 1 && F <= kMaxUFoldF && F < N && tc_req && !mixed && !(fuse & WINO_FUSE_L2_CHUNK) && ipow(a, F) <= kMaxUFoldQ &&
        ipow(m, F) <= kMaxUFoldMO && output_fold_supported(N, a, m, F, spec)) {
      p->uf_F = F;
      fold_coefs(t, F, p->uf_tab);
    }
  }
  {
    const int Q = p->uf_F ? p->uf_tab.Q : 1, MO = p->uf_F ? p->uf_tab.MO : 1;
    p->gP = (int64_t)a0 * ipow(a, N - 1) / Q;
    p->gC = Q * C;
    p->gK = MO * K;
  }
  p->gemm_mode = gemm_mode == WINO_GEMM_AUTO ? auto_gemm_mode(N, a, m, p->gC, p->gK, mixed, fuse) : gemm_mode;
  p->fuse = fuse;
  p->spec = spec;
  if (const char* ev = getenv("WINO_IN_TMA")) p->use_tma_in = atoi(ev) != 0;
  p->tf = t;
  int64_t Tps = 1;
  for (int n = 0; n < N; ++n) {
    p->in[n] = dims[n];
    p->pad[n] = padding ? padding[n] : 0;
    if (dims[n] < 1 || p->pad[n] < 0) { delete p; return fail(WINO_ERR_ARG, "dims must be >= 1 and padding >= 0"); }
    const int rn = n == 0 ? r0 : r, mn = n == 0 ? m0 : m;
    p->out[n] = dims[n] + 2 * p->pad[n] - rn + 1;
    if (p->out[n] < 1) { delete p; return fail(WINO_ERR_SHAPE, "kernel %d larger than padded input %lld on axis %d", rn, (long long)(dims[n] + 2 * p->pad[n]), n); }
    p->tiles[n] = (int)((p->out[n] + mn - 1) / mn);
    Tps *= p->tiles[n];
  }
  p->Tps = Tps;
  const int64_t T = Tps * batch;
  if (T > (int64_t)INT32_MAX - 256) { delete p; return fail(WINO_ERR_UNSUPPORTED, "too many tiles (%lld)", (long long)T); }
  p->T_s = (T + 127) / 128 * 128;
  p->P = (int64_t)a0 * ipow(a, N - 1);
  p->f16 = p->gemm_mode == WINO_GEMM_3XF16;
  const bool tc = p->gemm_mode == WINO_GEMM_3XTF32 || p->gemm_mode == WINO_GEMM_1XTF32 || p->f16;
  // K stride of U (the GEMM's B operand; MO * K columns under the filter-side fold)
  const int gK = p->gK;
  const int bn = gK <= 32 ? 32 : gK <= 64 ? 64 : gK <= 128 ? 128 : 256;
  p->K_s = tc ? (gK + bn - 1) / bn * bn : (gK + 31) / 32 * 32;

  // tables
  const FloatTables ft = to_tables(t), ft0 = to_tables(t0);
  for (int i = 0; i < kMaxA; ++i)
    for (int j = 0; j < kMaxA; ++j) {
      p->xp.AT[i][j] = ft.AT[i][j];
      p->xp.BT[i][j] = ft.BT[i][j];
      for (int n = 0; n < kMaxN; ++n) p->fp.G[n][i][j] = n == 0 ? ft0.G[i][j] : ft.G[i][j];
    }
  for (int n = 0; n < kMaxN; ++n) { p->fp.a[n] = n == 0 ? a0 : a; p->fp.r[n] = n == 0 ? r0 : r; }
  p->fp.N = N; p->fp.C = C; p->fp.K = K; p->fp.K_s = (int)p->K_s; p->fp.P = p->P;

  KGeom& g = p->geom;
  int64_t sin = 1, sout = 1;
  for (int n = N - 1; n >= 0; --n) {
    g.in[n] = p->in[n]; g.out[n] = p->out[n]; g.tiles[n] = p->tiles[n]; g.pad[n] = p->pad[n];
    g.in_stride[n] = sin; g.out_stride[n] = sout;
    sin *= p->in[n]; sout *= p->out[n];
  }
  g.in_vol = sin; g.out_vol = sout; g.Tps = Tps; g.T = T; g.T_s = p->T_s; g.C = C; g.K = K; g.m = m;
  // the TMA slab needs 16-byte row strides (and a supported column shift, see encode_input_map)
  const bool tma_shape = N >= 2 && (p->in[N - 1] % 4) == 0;
  p->use_tma_in = p->use_tma_in && tma_shape;
  if (!plan_input_slab(g, N, a0, m0, a, m, p->use_tma_in)) {
    delete p;
    // even a banded one-tile-deep slab exceeds shared memory: generic passes
    if (!mixed) return create_generic(plan_out, N, dims, mv, rv, points, C, K, batch, padding, gemm_mode, device);
    return fail(WINO_ERR_UNSUPPORTED, "input slab of one axis-0 tile exceeds shared memory (inner extents too large)");
  }

  // L2 chunking: chunk_slabs input slabs per chunk, V + M of a chunk near
  // WINO_CHUNK_MB (default 48 MB, under the 126 MB L2 with x / y traffic)
  if ((fuse & WINO_FUSE_L2_CHUNK) && g.nbox1 == 1) {  // (not with axis-1 banded slabs)
    double mb = 48.0;
    if (const char* ev = getenv("WINO_CHUNK_MB")) mb = atof(ev);
    const double slab_bytes = (double)g.bt0 * g.R * p->P * (C + K) * 4.0;
    int64_t cs = (int64_t)(mb * 1048576.0 / slab_bytes);
    const int64_t nslab = (int64_t)batch * g.nbox0;
    if (cs < 1) cs = 1;
    if (cs < nslab) {
      p->chunked = true;
      p->chunk_slabs = cs;
      p->T_s = ((int64_t)cs * g.bt0 * g.R + 127) / 128 * 128;
      g.T_s = p->T_s;
    }
  }

  // device buffers
  if (device < 0) {
    if (cudaGetDevice(&device) != cudaSuccess) { delete p; return fail(WINO_ERR_CUDA, "no CUDA device"); }
  }
  p->device = device;
  DeviceGuard guard(device);
  {
    int nsm = 148;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) nsm = 148;
    const int64_t nslab_all = p->chunked ? p->chunk_slabs : (int64_t)batch * g.nbox0 * g.nbox1;
    plan_input_planes(g, nslab_all * C, nsm);
  }
  const size_t ucount = (size_t)p->gP * p->gC * p->K_s;   // U, or U' under the filter-side fold
  const int nbuf = p->gemm_mode == WINO_GEMM_FFMA ? 1 : 2;
  p->filter_bytes = ucount * 4 * nbuf + (p->f16 ? 256 : 0);
  // a5 direct-axis fold candidate (decided below, once the GEMM's k-chunk is
  // known): Z [gP * 2][C][df_Tz] shares the V region, which is sized for both
  const bool df_cand = p->uf_F == 1 && r == 3 && !p->chunked && p->gemm_mode == WINO_GEMM_3XF16 &&
                       !mixed && g.nbox1 == 1 && input_dfold_supported(N, a, m, spec, p->tiles[N - 1]) &&
                       dfold_wanted(p->tiles[N - 1]);
  size_t v_floats = (size_t)p->P * C * p->T_s;
  if (df_cand) {
    p->df_Tz = ((int64_t)batch * p->tiles[0] * p->tiles[1] * kDfoldSlots + 255) / 256 * 256;
    const size_t z_floats = (size_t)p->gP * 2 * C * p->df_Tz;
    if (z_floats > v_floats) v_floats = z_floats;
  }
  p->ws_bytes = (v_floats + (size_t)p->P * K * p->T_s) * 4;
  cudaError_t e = cudaMalloc(&p->ubuf, p->filter_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&p->V, p->ws_bytes);
  if (e == cudaSuccess && p->f16) e = cudaMalloc(&p->vmax, 256);
  if (e == cudaSuccess && p->f16) e = zero_private(p->vmax, 256);
  if (e != cudaSuccess) {
    cudaFree(p->ubuf);
    cudaFree(p->vmax);
    delete p;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? WINO_ERR_NOMEM : WINO_ERR_CUDA, "device allocation failed: %s",
                cudaGetErrorString(e));
  }
  p->M = p->V + v_floats;
  // GEMM padding rows t in [T, T_s) of V are never written: zero them once
  e = zero_private(p->V, p->ws_bytes);
  if (e != cudaSuccess) {
    cudaFree(p->ubuf);
    cudaFree(p->V);
    delete p;
    return fail(WINO_ERR_CUDA, "workspace memset failed: %s", cudaGetErrorString(e));
  }
  {
    // a4 reads M through TMA boxes unless disabled (WINO_OUT_TMA=0, dev knob)
    const char* ev = getenv("WINO_OUT_TMA");
    int64_t A1 = 1;
    for (int n = 1; n < N; ++n) A1 *= a;
    p->tm_M_ok = (!ev || atoi(ev) != 0) && encode_output_map(&p->tm_M, p->M, p->T_s, K, p->P, (int)A1);
  }
  if (p->gemm_mode == WINO_GEMM_FFMA) {
    p->U32 = p->ubuf;
  } else {
    p->Uhi = p->ubuf;
    p->Ulo = p->ubuf + ucount;
  }
  p->filter_bcast_bytes = p->filter_bytes;
  if (p->f16) {
    // [hi16 | lo16 | tail 256 B | fp32 staging]; broadcast = hi, lo and the scale
    uint8_t* b = reinterpret_cast<uint8_t*>(p->ubuf);
    p->U16hi = b;
    p->U16lo = b + ucount * 2;
    p->uscal = reinterpret_cast<float*>(b + ucount * 4);
    p->umax = reinterpret_cast<unsigned int*>(b + ucount * 4 + 4);
    p->U32tmp = reinterpret_cast<float*>(b + ucount * 4 + 256);
    p->filter_bcast_bytes = ucount * 4 + 256;
  }
  if (tc) {
    // the GEMM runs on (gP, gC, gK) = (P, C, K), or (P/Q, Q*C, MO*K) with V
    // viewed as [P/Q][Q*C][T_s] under the filter-side fold
    const int gP = (int)p->gP, gC = p->gC;
    e = tc_gemm_prepare(p->tg, p->V, p->Uhi, p->Ulo, gP, p->T_s, gC, (int)p->K_s, gK,
                        p->gemm_mode == WINO_GEMM_1XTF32 ? 0 : 1, device);
    if (e == cudaSuccess && p->f16) {
      if (p->chunked || !f16_supported(gK, p->tg.kc)) {
        wino_plan_destroy(p);
        return fail(WINO_ERR_UNSUPPORTED, "3xFP16 GEMM needs K > 64, a k-chunk of 32 or 64 (C >= 32) and no L2 chunking");
      }
      e = f16_encode_u(&p->tmBhi16, p->U16hi, p->K_s, gC, gP, p->tg.kc);
      if (e == cudaSuccess) e = f16_encode_u(&p->tmBlo16, p->U16lo, p->K_s, gC, gP, p->tg.kc);
      if (const char* ev = getenv("WINO_F16N")) p->f16n = atoi(ev) != 0;
      if (df_cand && p->f16n && C % p->tg.kc == 0 && f16n_applies(gC, gK, p->tg.kc)) {
        // direct-axis fold: Z planes of 32-slot rows in the V buffer
        if (f16_encode_z(&p->tmA_df, p->V, p->df_Tz, C, (int)p->gP * 2, p->tg.kc) == cudaSuccess) {
          p->df = true;
          p->uf_tab.direct = 1;
          for (int j = 0; j < a; ++j)
            for (int o = 0; o < m; ++o) p->uf_tab.coef[j][o] = (j - o >= 0 && j - o < r) ? 1.0 : 0.0;
        }
      }
      if (p->uf_F && p->f16n && C % p->tg.kc == 0 && f16n_applies(gC, gK, p->tg.kc)) p->zmask = ufold_zmask(p, 128);
    }
    if (e == cudaSuccess && !p->uf_F && !mixed && !p->chunked && p->gemm_mode == WINO_GEMM_3XTF32) plan_fold(p);
    if (e == cudaSuccess && !p->fold_F && !p->f16)
      e = tc_gemm_tune(p->tg, p->M, gP, p->chunked ? p->T_s : T, p->T_s, gC, gK, p->V);
    if (e != cudaSuccess) {
      wino_plan_destroy(p);
      return fail(WINO_ERR_CUDA, "tcgen05 GEMM setup failed: %s", cudaGetErrorString(e));
    }
  }
  {
    // tiny layers (e.g. c1: 8x8, 4 -> 4 channels): one launch does a2 + a3
    // + a4; fp32 FMA with U = U_hi + U_lo (3xTF32 plans only).  Opt-in
    // (WINO_TINY=1): measured on c1 in CUDA-graph replay it takes 6.65 us
    // per forward against 5.88 us for the three PDL-chained kernels.
    // Decided on per-sample sizes and K <= 64 only, so batch shards and K
    // shards of a tiny layer take the same path (reading #8)
    int TB, smem;
    const char* ev = getenv("WINO_TINY");
    p->tiny = (ev && atoi(ev) != 0) && !mixed && !p->chunked && !p->uf_F && p->gemm_mode == WINO_GEMM_3XTF32 &&
              tiny_supported(N, a, m) && tiny_shape(N, a, C, K, p->P, &TB, &smem) && p->P * Tps * (int64_t)C <= 8192 &&
              K <= 64;
  }
  *plan_out = p;
  return WINO_OK;
}

wino_status wino_plan_create_ex(wino_plan_t* plan_out, int N, const int64_t* dims, int m, int r, int C, int K,
                                int batch, const int* padding, const char* points, int gemm_mode, int fuse,
                                int device) {
  return create_core(plan_out, N, dims, m, r, m, r, C, K, batch, padding, points, gemm_mode, fuse, device);
}

wino_status wino_plan_create_nd(wino_plan_t* plan_out, int N, const int64_t* dims, const int* m, const int* r,
                                int C, int K, int batch, const int* padding, int gemm_mode, int device) {
  if (!plan_out) return fail(WINO_ERR_ARG, "plan pointer is NULL");
  *plan_out = nullptr;
  if (N < 1 || N > kMaxN) return fail(WINO_ERR_ARG, "N must be in 1..4 (got %d)", N);
  if (!dims || !m || !r) return fail(WINO_ERR_ARG, "dims, m or r is NULL");
  if (C < 1 || K < 1 || batch < 1) return fail(WINO_ERR_ARG, "C, K, batch must be >= 1");
  if (gemm_mode < 0 || gemm_mode > 4) return fail(WINO_ERR_ARG, "bad gemm_mode %d", gemm_mode);
  bool uniform = true;
  for (int n = 1; n < N; ++n) uniform = uniform && m[n] == m[0] && r[n] == r[0];
  // equal axes: the single-(m, r) plan and its fused kernels
  if (uniform) return wino_plan_create_ex(plan_out, N, dims, m[0], r[0], C, K, batch, padding, nullptr, gemm_mode, 0,
                                          device);
  // a distinct axis 0 over equal other axes with instantiated fused kernels
  // (e.g. F(2,3) along time x F(4,3) along space); WINO_ND_GENERIC=1 forces
  // the generic multi-pass path (dev / test knob)
  bool rest_equal = N >= 2;
  for (int n = 2; n < N; ++n) rest_equal = rest_equal && m[n] == m[1] && r[n] == r[1];
  if (rest_equal && !force_generic() && m[0] + r[0] - 1 <= kMaxA && m[1] + r[1] - 1 <= kMaxA &&
      mixed_supported(N, m[0] + r[0] - 1, m[0], m[1] + r[1] - 1, m[1])) {
    wino_status st =
        create_core(plan_out, N, dims, m[0], r[0], m[1], r[1], C, K, batch, padding, nullptr, gemm_mode, 0, device);
    if (st != WINO_ERR_UNSUPPORTED) return st;   // (e.g. a slab too large for the fused kernels: generic)
  }
  return create_generic(plan_out, N, dims, m, r, nullptr, C, K, batch, padding, gemm_mode, device);
}

// The generic multi-pass per-axis plan (xform_nd.cu around the same GEMM):
// any F(m_n, r_n) with alpha_n <= 8 per axis and any extents.  Also the
// fallback of single-(m, r) plans the fused kernels do not cover (alpha = 7,
// F(2,5), N = 4 with alpha > 4, slabs too large for shared memory); then
// `points` (one list for every axis) may be given.
static wino_status create_generic(wino_plan_t* plan_out, int N, const int64_t* dims, const int* m, const int* r,
                                  const char* points, int C, int K, int batch, const int* padding, int gemm_mode,
                                  int device) {
  if (gemm_mode == WINO_GEMM_3XF16)
    return fail(WINO_ERR_UNSUPPORTED, "3xFP16 GEMM only with the fused transform kernels (not the generic passes)");
  Transforms tn[kMaxN];
  int64_t P = 1;
  for (int n = 0; n < N; ++n) {
    int spec;
    wino_status st = synth_checked(m[n], r[n], points, tn[n], spec);
    if (st) return st;
    if (tn[n].a > kMaxA)
      return fail(WINO_ERR_UNSUPPORTED, "alpha_%d = m + r - 1 = %d exceeds %d on the device path", n, tn[n].a, kMaxA);
    P *= tn[n].a;
  }
  wino_plan_s* p = new wino_plan_s();
  p->nd = true;
  p->N = N; p->m = m[0]; p->r = r[0]; p->a = tn[0].a; p->C = C; p->K = K; p->batch = batch;
  p->gemm_mode = gemm_mode == WINO_GEMM_AUTO ? WINO_GEMM_3XTF32 : gemm_mode;
  p->spec = kSpecRuntime;
  p->use_tma_in = false;
  p->tf = tn[0];
  int64_t Tps = 1;
  for (int n = 0; n < N; ++n) {
    p->mn[n] = m[n]; p->rn[n] = r[n]; p->an[n] = tn[n].a;
    p->in[n] = dims[n];
    p->pad[n] = padding ? padding[n] : 0;
    if (dims[n] < 1 || p->pad[n] < 0) { delete p; return fail(WINO_ERR_ARG, "dims must be >= 1 and padding >= 0"); }
    p->out[n] = dims[n] + 2 * p->pad[n] - r[n] + 1;
    if (p->out[n] < 1) { delete p; return fail(WINO_ERR_SHAPE, "kernel %d larger than padded input %lld on axis %d", r[n], (long long)(dims[n] + 2 * p->pad[n]), n); }
    p->tiles[n] = (int)((p->out[n] + m[n] - 1) / m[n]);
    Tps *= p->tiles[n];
  }
  p->Tps = Tps;
  const int64_t T = Tps * batch;
  if (T > (int64_t)INT32_MAX - 256) { delete p; return fail(WINO_ERR_UNSUPPORTED, "too many tiles (%lld)", (long long)T); }
  p->T_s = (T + 127) / 128 * 128;
  p->P = P;
  p->gP = P;
  p->gC = C;
  p->gK = K;
  if (P > 65535) { delete p; return fail(WINO_ERR_UNSUPPORTED, "prod alpha_n = %lld points exceeds 65535", (long long)P); }
  const bool tc = p->gemm_mode == WINO_GEMM_3XTF32 || p->gemm_mode == WINO_GEMM_1XTF32;
  const int bn = K <= 32 ? 32 : K <= 64 ? 64 : K <= 128 ? 128 : 256;
  p->K_s = tc ? (K + bn - 1) / bn * bn : (K + 31) / 32 * 32;
  // per-axis tables: B_n^T, A_n^T (fp32, RNE from exact), G_n (fp64)
  for (int n = 0; n < kMaxN; ++n) {
    const FloatTables ft = to_tables(tn[n < N ? n : 0]);
    for (int i = 0; i < kMaxA; ++i)
      for (int j = 0; j < kMaxA; ++j) {
        p->ndp.BT[n][i][j] = ft.BT[i][j];
        p->ndp.AT[n][i][j] = ft.AT[i][j];
        p->fp.G[n][i][j] = ft.G[i][j];
      }
    p->ndp.a[n] = n < N ? tn[n].a : 1;
    p->ndp.m[n] = n < N ? m[n] : 1;
    p->fp.a[n] = n < N ? tn[n].a : 1;
    p->fp.r[n] = n < N ? r[n] : 1;
  }
  p->fp.N = N; p->fp.C = C; p->fp.K = K; p->fp.K_s = (int)p->K_s; p->fp.P = P;
  KGeom& g = p->geom;
  int64_t sin = 1, sout = 1;
  for (int n = N - 1; n >= 0; --n) {
    g.in[n] = p->in[n]; g.out[n] = p->out[n]; g.tiles[n] = p->tiles[n]; g.pad[n] = p->pad[n];
    g.in_stride[n] = sin; g.out_stride[n] = sout;
    sin *= p->in[n]; sout *= p->out[n];
  }
  g.in_vol = sin; g.out_vol = sout; g.Tps = Tps; g.T = T; g.T_s = p->T_s; g.C = C; g.K = K; g.m = m[0];
  if (device < 0) {
    if (cudaGetDevice(&device) != cudaSuccess) { delete p; return fail(WINO_ERR_CUDA, "no CUDA device"); }
  }
  p->device = device;
  DeviceGuard guard(device);
  const size_t ucount = (size_t)P * C * p->K_s;
  const int nbuf = p->gemm_mode == WINO_GEMM_FFMA ? 1 : 2;
  p->filter_bytes = ucount * 4 * nbuf;
  p->ws_bytes = ((size_t)P * C * p->T_s + (size_t)P * K * p->T_s) * 4;
  cudaError_t e = cudaMalloc(&p->ubuf, p->filter_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&p->V, p->ws_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&p->W, (size_t)P * K * p->T_s * 4);
  if (e == cudaSuccess) e = zero_private(p->V, p->ws_bytes);
  if (e != cudaSuccess) {
    wino_plan_destroy(p);
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? WINO_ERR_NOMEM : WINO_ERR_CUDA, "device allocation failed: %s",
                cudaGetErrorString(e));
  }
  p->M = p->V + (size_t)P * C * p->T_s;
  if (p->gemm_mode == WINO_GEMM_FFMA) {
    p->U32 = p->ubuf;
  } else {
    p->Uhi = p->ubuf;
    p->Ulo = p->ubuf + ucount;
  }
  p->filter_bcast_bytes = p->filter_bytes;
  if (tc) {
    e = tc_gemm_prepare(p->tg, p->V, p->Uhi, p->Ulo, (int)P, p->T_s, C, (int)p->K_s, K,
                        p->gemm_mode == WINO_GEMM_3XTF32 ? 1 : 0, device);
    if (e == cudaSuccess) e = tc_gemm_tune(p->tg, p->M, (int)P, T, p->T_s, C, K, p->V);
    if (e != cudaSuccess) {
      wino_plan_destroy(p);
      return fail(WINO_ERR_CUDA, "tcgen05 GEMM setup failed: %s", cudaGetErrorString(e));
    }
  }
  *plan_out = p;
  return WINO_OK;
}

wino_status wino_plan_create(wino_plan_t* plan, int N, const int64_t* dims, int m, int r, int C, int K, int batch,
                             const int* padding) {
  return wino_plan_create_ex(plan, N, dims, m, r, C, K, batch, padding, nullptr, WINO_GEMM_AUTO, 0, -1);
}

wino_status wino_plan_destroy(wino_plan_t p) {
  if (!p) return WINO_OK;
  DeviceGuard guard(p->device);
  cudaFree(p->ubuf);
  cudaFree(p->V);
  cudaFree(p->x_dev);
  cudaFree(p->y_dev);
  cudaFree(p->W);
  cudaFree(p->vmax);
  for (cudaEvent_t e : p->ev) cudaEventDestroy(e);
  if (p->s_in) {
    for (int i = 0; i < kHostChunks; ++i) {
      cudaEventDestroy(p->e_in[i]);
      cudaEventDestroy(p->e_fw[i]);
    }
    cudaEventDestroy(p->e_start);
    cudaStreamDestroy(p->s_in);
    cudaStreamDestroy(p->s_out);
  }
  delete p;
  return WINO_OK;
}

wino_status wino_filter_transform(wino_plan_t p, const float* g, wino_stream_t stream) {
  if (!p || !g) return fail(WINO_ERR_ARG, "NULL plan or filter pointer");
  DeviceGuard guard(p->device);
  CUDA_TRY(cudaGetLastError());
  if (p->f16) {
    // fp32 U (one rounding from fp64) into the staging area, then the scaled fp16 split
    if (p->uf_F) CUDA_TRY(launch_filter_ufold(g, nullptr, nullptr, p->U32tmp, p->fp, p->uf_tab, (cudaStream_t)stream));
    else CUDA_TRY(launch_filter_xform(g, nullptr, nullptr, p->U32tmp, p->fp, (cudaStream_t)stream));
    CUDA_TRY(launch_split16(p->U32tmp, p->gP * p->gC * p->K_s, p->umax, p->U16hi, p->U16lo, p->uscal,
                            (cudaStream_t)stream));
  } else if (p->uf_F) {
    CUDA_TRY(launch_filter_ufold(g, p->Uhi, p->Ulo, p->U32, p->fp, p->uf_tab, (cudaStream_t)stream));
  } else {
    CUDA_TRY(launch_filter_xform(g, p->Uhi, p->Ulo, p->U32, p->fp, (cudaStream_t)stream));
  }
  p->filter_ready = true;
  return WINO_OK;
}

// First tile of input slab s (flattened (b * nbox0 + box0) * nbox1 + box1).
static int64_t slab_tile(const KGeom& g, int64_t s) {
  const int64_t s0 = s / g.nbox1, box1 = s % g.nbox1;
  const int64_t b = s0 / g.nbox0, box = s0 % g.nbox0;
  const int64_t a0 = box * g.bt0 < g.tiles[0] ? box * g.bt0 : g.tiles[0];
  return b * g.Tps + a0 * g.R + box1 * g.bt1 * g.R1;
}

// Stage timing (wino_profile_*): a start/end event pair around one launch.
struct ProfScope {
  wino_plan_t p;
  cudaStream_t s;
  int stage;
  cudaEvent_t b = nullptr, e = nullptr;
  cudaError_t begin() {
    const size_t i = p->prof_stage.size();
    while (p->ev.size() < 2 * (i + 1)) {
      cudaEvent_t ev;
      cudaError_t r = cudaEventCreate(&ev);
      if (r != cudaSuccess) return r;
      p->ev.push_back(ev);
    }
    b = p->ev[2 * i];
    e = p->ev[2 * i + 1];
    p->prof_stage.push_back(stage);
    return cudaEventRecord(b, s);
  }
  cudaError_t end() { return cudaEventRecord(e, s); }
};

static wino_status forward_impl(wino_plan_t p, const float* x, float* y, int B, cudaStream_t s,
                                const float* bias = nullptr, int act = 0) {
  KGeom g = p->geom;
  g.bias = bias;
  g.act = act;
  const bool rec = p->prof && p->prof_calls < kMaxProf;
  if (p->tiny) {
    ProfScope pt{p, s, 1};
    if (rec) CUDA_TRY(pt.begin());
    CUDA_TRY(launch_tiny(x, p->Uhi, p->Ulo, y, g, p->xp, p->N, p->a, p->m, p->spec, (int)p->P, (int)p->K_s,
                         (int64_t)B * p->Tps, s));
    if (rec) CUDA_TRY(pt.end());
    if (rec) ++p->prof_calls;
    return WINO_OK;
  }
  if (p->nd) {
    // per-axis plan: generic multi-pass transforms around the same GEMM
    const int64_t T = (int64_t)B * p->Tps;
    g.T = T;
    g.t0 = 0;
    g.t_beg = 0;
    ProfScope ps{p, s, 0};
    if (rec) CUDA_TRY(ps.begin());
    CUDA_TRY(launch_input_nd(x, p->V, g, p->ndp, p->N, p->P, 0, T, s));
    if (rec) CUDA_TRY(ps.end());
    ProfScope pg{p, s, 1};
    if (rec) CUDA_TRY(pg.begin());
    if (p->gemm_mode == WINO_GEMM_FFMA) {
      CUDA_TRY(launch_gemm_ffma(p->V, p->U32, p->M, (int)p->P, T, p->T_s, p->C, p->K, (int)p->K_s, s));
    } else {
      CUDA_TRY(launch_gemm_tc(p->tg, p->M, (int)p->P, 0, T, p->T_s, p->C, p->K, s));
    }
    if (rec) CUDA_TRY(pg.end());
    ProfScope po{p, s, 2};
    if (rec) CUDA_TRY(po.begin());
    CUDA_TRY(launch_output_nd(p->M, p->W, y, g, p->ndp, p->N, 0, T, s));
    if (rec) CUDA_TRY(po.end());
    if (rec) ++p->prof_calls;
    return WINO_OK;
  }
  if (p->f16) {
    g.vmax = p->vmax;
    g.vmax_reset = p->vmax;
  }
  // TMA map of x, re-encoded when the input pointer or batch changes
  if (p->use_tma_in && (x != p->tm_x_ptr || B != p->tm_x_B)) {
    p->tm_x_ok = encode_input_map(&p->tm_x, x, g, p->N, B);
    p->tm_x_ptr = x;
    p->tm_x_B = B;
  }
  const CUtensorMap* tm = p->use_tma_in && p->tm_x_ok ? &p->tm_x : nullptr;
  const int64_t nslab = (int64_t)B * g.nbox0 * g.nbox1;
  const int64_t step = p->chunked ? p->chunk_slabs : nslab;
  for (int64_t s0 = 0; s0 < nslab; s0 += step) {
    const int64_t s1 = s0 + step < nslab ? s0 + step : nslab;
    const int64_t t_lo = slab_tile(g, s0), t_hi = slab_tile(g, s1);
    g.s_beg = s0;
    g.dfold = p->df ? 1 : 0;   // a2 writes Z (outer axes only) into the V region
    g.Tz = p->df_Tz;
    g.df_S = kDfoldSlots;
    g.t0 = p->chunked ? t_lo : 0;
    g.t_beg = t_lo;
    g.T = t_hi;
    ProfScope ps{p, s, 0};
    if (rec) CUDA_TRY(ps.begin());
    pdl_stage(1);
    if (p->mixed) {
      CUDA_TRY(launch_input_mixed(p->N, p->a0, p->m0, p->a, p->m, x, p->V, g, p->xp, tm, (int)(s1 - s0), s));
    } else {
      CUDA_TRY(launch_input_xform(p->N, p->a, p->m, p->spec, x, p->V, g, p->xp, tm, (int)(s1 - s0), s));
    }
    if (rec) CUDA_TRY(ps.end());
    ProfScope pg{p, s, 1};
    if (rec) CUDA_TRY(pg.begin());
    pdl_stage(2);
    if (p->df) {
      // the GEMM's rows are Z's slots: 32 per (b, t_0, t_1) row of tiles
      const DFoldGemm dg{&p->tmA_df, p->tiles[p->N - 1], kDfoldSlots, p->C};
      const int64_t slots = (int64_t)B * p->tiles[0] * p->tiles[1] * kDfoldSlots;
      CUDA_TRY(launch_gemm_f16(p->tg, p->tmBhi16, p->tmBlo16, p->M, (int)p->gP, 0, slots, p->T_s, p->gC, p->gK,
                               p->vmax, p->uscal, s, p->zmask, true, &dg));
    } else if (p->f16) {
      CUDA_TRY(launch_gemm_f16(p->tg, p->tmBhi16, p->tmBlo16, p->M, (int)p->gP, t_lo - g.t0, t_hi - g.t0, p->T_s,
                               p->gC, p->gK, p->vmax, p->uscal, s, p->zmask, p->f16n));
    } else if (p->fold_F) {
      CUDA_TRY(launch_gemm_fold(p->tg, p->fold_bn, p->fold_g, p->fold_MO, p->M, (int)p->P, p->fold_Q, t_lo - g.t0,
                                t_hi - g.t0, p->T_s, p->C, p->K, p->fold_tab, s));
    } else if (p->gemm_mode == WINO_GEMM_FFMA) {
      CUDA_TRY(launch_gemm_ffma(p->V, p->U32, p->M, (int)p->P, t_hi - g.t0, p->T_s, p->C, p->K, (int)p->K_s, s));
    } else {
      CUDA_TRY(launch_gemm_tc(p->tg, p->M, (int)p->gP, t_lo - g.t0, t_hi - g.t0, p->T_s, p->gC, p->gK, s));
    }
    if (rec) CUDA_TRY(pg.end());
    ProfScope po{p, s, 2};
    if (rec) CUDA_TRY(po.begin());
    pdl_stage(3);
    if (p->fold_F || p->uf_F) {
      CUDA_TRY(launch_output_fold(p->N, p->a, p->m, p->fold_F + p->uf_F, p->spec, p->M, y, g, p->xp, s));
    } else if (p->mixed) {
      CUDA_TRY(launch_output_mixed(p->N, p->a0, p->m0, p->a, p->m, p->M, y, g, p->xp,
                                   p->tm_M_ok ? &p->tm_M : nullptr, s));
    } else {
      CUDA_TRY(launch_output_xform(p->N, p->a, p->m, p->spec, p->M, y, g, p->xp, p->tm_M_ok ? &p->tm_M : nullptr, s));
    }
    if (rec) CUDA_TRY(po.end());
    pdl_stage(0);
  }
  if (rec) ++p->prof_calls;
  return WINO_OK;
}

wino_status wino_forward_ex(wino_plan_t p, const float* x, float* y, int B, const float* bias, int activation,
                            wino_stream_t stream) {
  if (!p || !x || !y) return fail(WINO_ERR_ARG, "NULL plan, x or y");
  if (B < 1 || B > p->batch) return fail(WINO_ERR_ARG, "B=%d outside 1..%d (planned batch)", B, p->batch);
  if (activation != WINO_ACT_NONE && activation != WINO_ACT_RELU)
    return fail(WINO_ERR_ARG, "unknown activation %d", activation);
  if (!p->filter_ready) return fail(WINO_ERR_STATE, "forward before wino_filter_transform / mark_ready");
  DeviceGuard guard(p->device);
  CUDA_TRY(cudaGetLastError());
  return forward_impl(p, x, y, B, (cudaStream_t)stream, bias, activation);
}

wino_status wino_forward(wino_plan_t p, const float* x, float* y, int B, wino_stream_t stream) {
  return wino_forward_ex(p, x, y, B, nullptr, WINO_ACT_NONE, stream);
}

// Host-buffer forward: the batch is split into sample chunks and pipelined
// over three streams -- H2D copies (s_in), the forward kernels (the caller's
// stream), D2H copies (s_out) -- so PCIe traffic in both directions overlaps
// the compute and each other.  Chunks share the plan workspace, so their
// forwards stay ordered on the compute stream.  Synchronises before return.
wino_status wino_forward_host(wino_plan_t p, const float* x_host, float* y_host, int B, wino_stream_t stream) {
  if (!p || !x_host || !y_host) return fail(WINO_ERR_ARG, "NULL plan, x_host or y_host");
  if (B < 1 || B > p->batch) return fail(WINO_ERR_ARG, "B=%d outside 1..%d (planned batch)", B, p->batch);
  if (!p->filter_ready) return fail(WINO_ERR_STATE, "forward before wino_filter_transform / mark_ready");
  DeviceGuard guard(p->device);
  const size_t xs = (size_t)p->C * p->geom.in_vol;   // floats per sample
  const size_t ys = (size_t)p->K * p->geom.out_vol;
  if (!p->x_dev) CUDA_TRY(cudaMalloc(&p->x_dev, (size_t)p->batch * xs * 4));
  if (!p->y_dev) CUDA_TRY(cudaMalloc(&p->y_dev, (size_t)p->batch * ys * 4));
  if (!p->s_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
    for (int i = 0; i < kHostChunks; ++i) {
      CUDA_TRY(cudaEventCreateWithFlags(&p->e_in[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&p->e_fw[i], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventCreateWithFlags(&p->e_start, cudaEventDisableTiming));
  }
  cudaStream_t s = (cudaStream_t)stream;
  // 8 chunks (measured best or within 3% of best on c2-c5, tools/e2e_probe.py);
  // WINO_HOST_CHUNKS overrides
  int nch = 8;
  if (const char* ev = getenv("WINO_HOST_CHUNKS")) nch = atoi(ev);
  if (nch < 1) nch = 1;
  if (nch > kHostChunks) nch = kHostChunks;
  if (nch > B) nch = B;
  // the copy streams start after everything already queued on the caller's stream
  CUDA_TRY(cudaEventRecord(p->e_start, s));
  CUDA_TRY(cudaStreamWaitEvent(p->s_in, p->e_start, 0));
  CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->e_start, 0));
  for (int i = 0; i < nch; ++i) {
    const int b0 = (int)((int64_t)B * i / nch), b1 = (int)((int64_t)B * (i + 1) / nch);
    const size_t nb = (size_t)(b1 - b0);
    CUDA_TRY(cudaMemcpyAsync(p->x_dev + b0 * xs, x_host + b0 * xs, nb * xs * 4, cudaMemcpyHostToDevice, p->s_in));
    CUDA_TRY(cudaEventRecord(p->e_in[i], p->s_in));
    CUDA_TRY(cudaStreamWaitEvent(s, p->e_in[i], 0));
    wino_status st = forward_impl(p, p->x_dev + b0 * xs, p->y_dev + b0 * ys, (int)nb, s);
    if (st) return st;
    CUDA_TRY(cudaEventRecord(p->e_fw[i], s));
    CUDA_TRY(cudaStreamWaitEvent(p->s_out, p->e_fw[i], 0));
    CUDA_TRY(cudaMemcpyAsync(y_host + b0 * ys, p->y_dev + b0 * ys, nb * ys * 4, cudaMemcpyDeviceToHost, p->s_out));
  }
  CUDA_TRY(cudaStreamSynchronize(p->s_out));
  CUDA_TRY(cudaStreamSynchronize(s));
  return WINO_OK;
}

wino_status wino_plan_out_dims(wino_plan_t p, int64_t* out) {
  if (!p || !out) return fail(WINO_ERR_ARG, "NULL argument");
  for (int n = 0; n < p->N; ++n) out[n] = p->out[n];
  return WINO_OK;
}

wino_status wino_plan_sizes(wino_plan_t p, size_t* ws, size_t* fb) {
  if (!p) return fail(WINO_ERR_ARG, "NULL plan");
  if (ws) *ws = p->ws_bytes;
  if (fb) *fb = p->filter_bytes;
  return WINO_OK;
}

wino_status wino_plan_info(wino_plan_t p, int64_t* info) {
  if (!p || !info) return fail(WINO_ERR_ARG, "NULL argument");
  // kernel launches of one full-batch forward
  int64_t launches = 3;
  if (p->tiny) launches = 1;
  else if (p->chunked) launches = 3 * (((int64_t)p->batch * p->geom.nbox0 + p->chunk_slabs - 1) / p->chunk_slabs);
  const int64_t v[25] = {p->N, p->m, p->r, p->a, p->C, p->K, p->batch, p->Tps, p->T_s, p->P, p->K_s,
                         p->gemm_mode, p->fuse, p->tg.bn, p->tg.kc, p->chunked ? p->chunk_slabs : 0,
                         p->gemm_mode == WINO_GEMM_FFMA ? -1 : p->tg.variant, p->geom.bt0,
                         p->geom.npl, p->nd ? 2 : p->mixed ? 1 : 0, p->tiny ? 1 : 0, launches,
                         p->nd ? 0 : p->geom.nbox1, p->fold_F + p->uf_F,
                         p->df ? 3 : p->uf_F ? 2 : p->fold_F ? 1 : 0};
  memcpy(info, v, sizeof v);
  return WINO_OK;
}

wino_status wino_filter_buffer(wino_plan_t p, void** dev_ptr, size_t* bytes) {
  if (!p || !dev_ptr || !bytes) return fail(WINO_ERR_ARG, "NULL argument");
  *dev_ptr = p->ubuf;
  *bytes = p->filter_bcast_bytes;
  return WINO_OK;
}

wino_status wino_filter_mark_ready(wino_plan_t p) {
  if (!p) return fail(WINO_ERR_ARG, "NULL plan");
  p->filter_ready = true;
  return WINO_OK;
}

wino_status wino_workspace(wino_plan_t p, void** V, void** M) {
  if (!p) return fail(WINO_ERR_ARG, "NULL plan");
  if (V) *V = p->V;
  if (M) *M = p->M;
  return WINO_OK;
}

wino_status wino_profile_enable(wino_plan_t p, int enable) {
  if (!p) return fail(WINO_ERR_ARG, "NULL plan");
  p->prof = enable != 0;
  p->prof_calls = 0;
  p->prof_stage.clear();
  return WINO_OK;
}

wino_status wino_profile_read(wino_plan_t p, double* ms, int* calls) {
  if (!p) return fail(WINO_ERR_ARG, "NULL plan");
  DeviceGuard guard(p->device);
  double acc[3] = {0, 0, 0};
  for (size_t i = 0; i < p->prof_stage.size(); ++i) {
    CUDA_TRY(cudaEventSynchronize(p->ev[2 * i + 1]));
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, p->ev[2 * i], p->ev[2 * i + 1]));
    acc[p->prof_stage[i]] += t;
  }
  if (ms) for (int s = 0; s < 3; ++s) ms[s] = acc[s];
  if (calls) *calls = p->prof_calls;
  return WINO_OK;
}

wino_status wino_get_transforms(wino_plan_t p, double* AT, double* G, double* BT, char* json, size_t cap) {
  if (!p) return fail(WINO_ERR_ARG, "NULL plan");
  const Transforms& t = p->tf;
  const int a = t.a, m = t.m, r = t.r;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < a; ++j)
      if (AT) AT[i * a + j] = rat_to_f64(t.AT[i][j]);
  for (int i = 0; i < a; ++i)
    for (int j = 0; j < r; ++j)
      if (G) G[i * r + j] = rat_to_f64(t.G[i][j]);
  for (int i = 0; i < a; ++i)
    for (int j = 0; j < a; ++j)
      if (BT) BT[i * a + j] = rat_to_f64(t.BT[i][j]);
  if (json && cap) {
    const std::string s = transforms_json(t);
    const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    memcpy(json, s.data(), n);
    json[n] = 0;
  }
  return WINO_OK;
}

}  // extern "C"
