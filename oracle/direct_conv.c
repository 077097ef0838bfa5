/*
 * oracle/direct_conv.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain float64 direct N-D cross-correlation: the definition the Winograd
 * path must reproduce.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with paper_1611_06565_b200/ (the CUDA path).
 *
 * Definition followed (Eq. (2), with bias b = 0 and
 * f = identity; the N-D extension "by looping over additional subscripts on
 * g and d"; readings #1, #2, #3 of DESIGN.md):
 *
 *   y[b,k,o] = sum_{c=0}^{C-1} sum_{p in [0,r_1)x..x[0,r_N)}
 *                 g[k,c,p] * xt[b,c,o+p-P],      o in [0,out_1)x..x[0,out_N)
 *   out_n    = in_n + 2 P_n - r_n + 1
 *   xt       = x zero-extended outside [0,in_n)  (symmetric zero padding P_n)
 *
 * Arithmetic: every product and sum in IEEE double, in the fixed order
 * "c ascending, then p row-major".  Inputs are the fp32
 * values, promoted exactly to double.
 *
 * Layouts (row-major, last index fastest):
 *   x [B][C][in_1]..[in_N]   float
 *   g [K][C][r_1]..[r_N]     float
 *   y [B][K][out_1]..[out_N] double
 */
#include <stdint.h>
#include <stdlib.h>

#define ORACLE_MAX_N 8

static int64_t prod(const int64_t* v, int n) {
  int64_t p = 1;
  for (int i = 0; i < n; ++i) p *= v[i];
  return p;
}

/* One output element y[b,k,o] (o given as N coordinates). */
static double one_output(int N, const int64_t* in, const int64_t* r,
                         const int64_t* pad, int64_t C, const float* xb,
                         const float* gk, const int64_t* o) {
  const int64_t in_vol = prod(in, N);
  const int64_t r_vol = prod(r, N);
  double acc = 0.0;
  for (int64_t c = 0; c < C; ++c) {
    const float* xc = xb + c * in_vol;
    const float* gc = gk + c * r_vol;
    for (int64_t pf = 0; pf < r_vol; ++pf) {     /* p row-major */
      int64_t rem = pf, xoff = 0, stride = 1;
      int inside = 1;
      /* decode p (last axis fastest) and the input coordinate o+p-P */
      int64_t pc[ORACLE_MAX_N];
      for (int n = N - 1; n >= 0; --n) { pc[n] = rem % r[n]; rem /= r[n]; }
      for (int n = N - 1; n >= 0; --n) {
        int64_t i = o[n] + pc[n] - pad[n];
        if (i < 0 || i >= in[n]) { inside = 0; break; }
        xoff += i * stride;
        stride *= in[n];
      }
      if (inside) acc += (double)gc[pf] * (double)xc[xoff];
    }
  }
  return acc;
}

int oracle_out_dims(int N, const int64_t* in, const int64_t* r,
                    const int64_t* pad, int64_t* out) {
  if (N < 1 || N > ORACLE_MAX_N) return 1;
  for (int n = 0; n < N; ++n) {
    out[n] = in[n] + 2 * pad[n] - r[n] + 1;
    if (out[n] < 1) return 2;
  }
  return 0;
}

/* Full direct correlation.  Parallel over (b,k) only; each output element is
 * still the same sequential sum, so the result does not depend on threads. */
int oracle_direct_conv_f64(int N, const int64_t* in, const int64_t* r,
                           const int64_t* pad, int64_t B, int64_t C, int64_t K,
                           const float* x, const float* g, double* y) {
  int64_t out[ORACLE_MAX_N];
  int st = oracle_out_dims(N, in, r, pad, out);
  if (st) return st;
  const int64_t in_vol = prod(in, N), r_vol = prod(r, N), out_vol = prod(out, N);
  int64_t bk;
#pragma omp parallel for schedule(dynamic, 1)
  for (bk = 0; bk < B * K; ++bk) {
    const int64_t b = bk / K, k = bk % K;
    const float* xb = x + b * C * in_vol;
    const float* gk = g + k * C * r_vol;
    double* yo = y + bk * out_vol;
    int64_t o[ORACLE_MAX_N];
    for (int64_t of = 0; of < out_vol; ++of) {
      int64_t rem = of;
      for (int n = N - 1; n >= 0; --n) { o[n] = rem % out[n]; rem /= out[n]; }
      yo[of] = one_output(N, in, r, pad, C, xb, gk, o);
    }
  }
  return 0;
}

/* Selected outputs only: flat indices into y [B][K][out...].  Used for
 * full-size parity on sampled outputs. */
int oracle_direct_conv_at(int N, const int64_t* in, const int64_t* r,
                          const int64_t* pad, int64_t B, int64_t C, int64_t K,
                          const float* x, const float* g, int64_t npts,
                          const int64_t* flat_idx, double* vals) {
  int64_t out[ORACLE_MAX_N];
  int st = oracle_out_dims(N, in, r, pad, out);
  if (st) return st;
  const int64_t in_vol = prod(in, N), r_vol = prod(r, N), out_vol = prod(out, N);
  int64_t i;
  for (i = 0; i < npts; ++i)
    if (flat_idx[i] < 0 || flat_idx[i] >= B * K * out_vol) return 3;
#pragma omp parallel for schedule(dynamic, 16)
  for (i = 0; i < npts; ++i) {
    int64_t f = flat_idx[i];
    const int64_t of = f % out_vol;
    const int64_t bk = f / out_vol;
    const int64_t b = bk / K, k = bk % K;
    int64_t o[ORACLE_MAX_N], rem = of;
    for (int n = N - 1; n >= 0; --n) { o[n] = rem % out[n]; rem /= out[n]; }
    vals[i] = one_output(N, in, r, pad, C, x + b * C * in_vol,
                         g + k * C * r_vol, o);
  }
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
