// xform_nd.cu -- input and output transforms of a plan with a different
// (m_n, r_n) on every axis (NEXT-2; Eq. (4) indexes the transforms by n:
//   V = d x_1 B_1^T x_2 ... x_N B_N^T,   y tile = M x_1 A_1^T ... x_N A_N^T,
// PAPER.md:160-164).  alpha_n = m_n + r_n - 1 <= 8, N <= 4, run-time tables.
//
// Generic multi-pass design (correctness and generality first; the uniform
// (m, r) plans keep the fused single-pass kernels of xform_in / xform_out):
//   a2: extract the alpha_1 x .. x alpha_N window of every tile into
//       V[xi][c][t] (zero padding) fused with B_N^T along the last axis,
//       then one in-place pass per remaining axis n applying B_n^T;
//   a4: one pass per axis n = 0 .. N-2 applying A_n^T along xi_n (alpha_n ->
//       m_n, ping-pong between M and a scratch buffer), then the last axis'
//       pass fused with bias / ReLU (Eq. (2)) and the crop + scatter into y
//       (m_{N-1} contiguous floats per thread).
// Every pass is HBM-streaming with t fastest (coalesced 128-byte warps).
#include "kernels.h"

namespace wino {
namespace {

// t -> (b, t_0 .. t_{N-1}) (t < 2^31 checked at plan creation)
__device__ __forceinline__ int decode_tile(int t, const KGeom& g, int N, int* tn) {
  int rem = t;
  for (int n = N - 1; n >= 0; --n) {
    tn[n] = rem % g.tiles[n];
    rem /= g.tiles[n];
  }
  return rem;  // sample b
}

// V[xi][c][t] = x[b][c][t_n m_n - P_n + xi_n] (0 outside).  grid (T/256, C, P)
__global__ void __launch_bounds__(256)
k_nd_extract(const float* __restrict__ x, float* __restrict__ V, const __grid_constant__ KGeom g,
             const __grid_constant__ NdParams q, int N, int64_t t_lo, int64_t t_hi) {
  const int64_t t = t_lo + (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int c = blockIdx.y;
  const int xi = blockIdx.z;
  pdl_wait();
  pdl_trigger();
  if (t >= t_hi) return;
  int tn[kMaxN], xn[kMaxN];
  const int b = decode_tile((int)t, g, N, tn);
  int rem = xi;
  for (int n = N - 1; n >= 0; --n) {
    xn[n] = rem % q.a[n];
    rem /= q.a[n];
  }
  bool ok = true;
  int64_t off = 0;
  for (int n = 0; n < N; ++n) {
    const int64_t pos = (int64_t)tn[n] * q.m[n] - g.pad[n] + xn[n];
    ok = ok && pos >= 0 && pos < g.in[n];
    off += pos * g.in_stride[n];
  }
  const float v = ok ? __ldg(x + ((int64_t)b * g.C + c) * g.in_vol + off) : 0.f;
  V[((int64_t)xi * g.C + c) * g.T_s + (t - g.t0)] = v;
}

// Window extraction fused with the last axis' pass: one thread per (t, c,
// line = xi without its last digit) reads the alpha_{N-1} consecutive x
// values of its window row (zero outside) and writes B_{N-1}^T of them.
// grid (T/256, C, P / a_{N-1}).
__global__ void __launch_bounds__(256)
k_nd_extract_last(const float* __restrict__ x, float* __restrict__ V, const __grid_constant__ KGeom g,
                  const __grid_constant__ NdParams q, int N, int64_t t_lo, int64_t t_hi) {
  const int64_t t = t_lo + (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int c = blockIdx.y;
  const int line = blockIdx.z;
  pdl_wait();
  pdl_trigger();
  if (t >= t_hi) return;
  const int L = N - 1, aL = q.a[L];
  int tn[kMaxN], xn[kMaxN];
  const int b = decode_tile((int)t, g, N, tn);
  int rem = line;
  for (int n = L - 1; n >= 0; --n) {
    xn[n] = rem % q.a[n];
    rem /= q.a[n];
  }
  bool ok = true;
  int64_t off = 0;
  for (int n = 0; n < L; ++n) {
    const int64_t pos = (int64_t)tn[n] * q.m[n] - g.pad[n] + xn[n];
    ok = ok && pos >= 0 && pos < g.in[n];
    off += pos * g.in_stride[n];
  }
  const int64_t p0 = (int64_t)tn[L] * q.m[L] - g.pad[L];
  const float* xr = x + ((int64_t)b * g.C + c) * g.in_vol + off;
  float v[kMaxA];
#pragma unroll
  for (int i = 0; i < kMaxA; ++i) {
    const int64_t pos = p0 + i;
    v[i] = (i < aL && ok && pos >= 0 && pos < g.in[L]) ? __ldg(xr + pos) : 0.f;
  }
  const int64_t ps = (int64_t)g.C * g.T_s;
  float* vo = V + ((int64_t)line * aL * g.C + c) * g.T_s + (t - g.t0);
#pragma unroll
  for (int o = 0; o < kMaxA; ++o) {
    if (o >= aL) break;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxA; ++i)
      if (i < aL) acc = fmaf(q.BT[L][o][i], v[i], acc);
    vo[o * ps] = acc;
  }
}

// In place along axis n of V[xi][c][t]: (xi_n) <- sum_i B_n^T[xi_n][i] (i).
// grid (T/256, C, P / a_n): blockIdx.z enumerates the xi with xi_n = 0.
__global__ void __launch_bounds__(256)
k_nd_mode_in(float* __restrict__ V, const __grid_constant__ KGeom g, const __grid_constant__ NdParams q, int N,
             int n, int64_t t_lo, int64_t t_hi) {
  const int64_t t = t_lo + (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int c = blockIdx.y;
  pdl_wait();
  pdl_trigger();
  if (t >= t_hi) return;
  // xi stride of axis n, and the line's base xi (xi_n = 0)
  int stride = 1;
  for (int j = N - 1; j > n; --j) stride *= q.a[j];
  const int an = q.a[n];
  const int line = blockIdx.z;
  const int base = (line / stride) * (stride * an) + line % stride;
  const int64_t ps = (int64_t)stride * g.C * g.T_s;
  float* p0 = V + ((int64_t)base * g.C + c) * g.T_s + (t - g.t0);
  float v[kMaxA];
#pragma unroll
  for (int i = 0; i < kMaxA; ++i)
    if (i < an) v[i] = p0[i * ps];
#pragma unroll
  for (int o = 0; o < kMaxA; ++o) {
    if (o >= an) break;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxA; ++i)
      if (i < an) acc = fmaf(q.BT[n][o][i], v[i], acc);
    p0[o * ps] = acc;
  }
}

// Axis-n pass of the output transform (n >= 1): src has xi extents ein[]
// (axes > n already reduced to m), dst the same with axis n -> m_n.
// grid (T/256, K, lines = prod_{j != n} ein[j]).
__global__ void __launch_bounds__(256)
k_nd_mode_out(const float* __restrict__ src, float* __restrict__ dst, const __grid_constant__ KGeom g,
              const __grid_constant__ NdParams q, int N, int n, int4 ein_lo, int64_t t_lo, int64_t t_hi) {
  const int64_t t = t_lo + (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int k = blockIdx.y;
  pdl_wait();
  pdl_trigger();
  if (t >= t_hi) return;
  const int ein[4] = {ein_lo.x, ein_lo.y, ein_lo.z, ein_lo.w};
  int sin = 1, sout = 1;
  for (int j = N - 1; j > n; --j) {
    sin *= ein[j];
    sout *= ein[j];
  }
  const int an = ein[n], mn = q.m[n];
  const int line = blockIdx.z;
  const int hi = line / sin, lo = line % sin;
  const int bin = hi * (sin * an) + lo, bout = hi * (sout * mn) + lo;
  const int64_t pin = (int64_t)sin * g.K * g.T_s, pout = (int64_t)sout * g.K * g.T_s;
  const float* s0 = src + ((int64_t)bin * g.K + k) * g.T_s + (t - g.t0);
  float* d0 = dst + ((int64_t)bout * g.K + k) * g.T_s + (t - g.t0);
  float v[kMaxA];
#pragma unroll
  for (int i = 0; i < kMaxA; ++i)
    if (i < an) v[i] = __ldg(s0 + i * pin);
#pragma unroll
  for (int o = 0; o < kMaxA; ++o) {
    if (o >= mn) break;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxA; ++i)
      if (i < an) acc = fmaf(q.AT[n][o][i], v[i], acc);
    d0[o * pout] = acc;
  }
}

// Axis-0 pass fused with Eq. (2)'s bias / ReLU and the crop + scatter:
// src xi extents (a_0, m_1, .., m_{N-1}).  grid (T/256, K, prod_{j>=1} m_j).
__global__ void __launch_bounds__(256)
k_nd_scatter(const float* __restrict__ src, float* __restrict__ y, const __grid_constant__ KGeom g,
             const __grid_constant__ NdParams q, int N, int64_t t_lo, int64_t t_hi) {
  const int64_t t = t_lo + (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int k = blockIdx.y;
  const int orest = blockIdx.z;  // (o_1 .. o_{N-1}) row-major
  pdl_wait();
  pdl_trigger();
  if (t >= t_hi) return;
  int rest = 1;
  for (int j = 1; j < N; ++j) rest *= q.m[j];
  const int a0 = q.a[0], m0 = q.m[0];
  const int64_t p0s = (int64_t)rest * g.K * g.T_s;
  const float* s0 = src + ((int64_t)orest * g.K + k) * g.T_s + (t - g.t0);
  float v[kMaxA];
#pragma unroll
  for (int i = 0; i < kMaxA; ++i)
    if (i < a0) v[i] = __ldg(s0 + i * p0s);
  int tn[kMaxN], on[kMaxN];
  const int b = decode_tile((int)t, g, N, tn);
  int rem = orest;
  for (int j = N - 1; j >= 1; --j) {
    on[j] = rem % q.m[j];
    rem /= q.m[j];
  }
  bool ok = true;
  int64_t off = 0;
  for (int j = 1; j < N; ++j) {
    const int64_t pos = (int64_t)tn[j] * q.m[j] + on[j];
    ok = ok && pos < g.out[j];
    off += pos * g.out_stride[j];
  }
  if (!ok) return;
  const float bk = g.bias ? __ldg(g.bias + k) : 0.f;
  float* yb = y + ((int64_t)b * g.K + k) * g.out_vol + off;
#pragma unroll
  for (int o = 0; o < kMaxA; ++o) {
    if (o >= m0) break;
    const int64_t pos = (int64_t)tn[0] * m0 + o;
    if (pos >= g.out[0]) break;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxA; ++i)
      if (i < a0) acc = fmaf(q.AT[0][o][i], v[i], acc);
    if (g.bias || g.act) {
      acc += bk;
      if (g.act == 1) acc = fmaxf(acc, 0.f);
    }
    yb[pos * g.out_stride[0]] = acc;
  }
}

// Last-axis pass fused with Eq. (2)'s bias / ReLU and the crop + scatter:
// src xi extents (m_0, .., m_{N-2}, a_{N-1}); one thread per (t, k, output
// offsets o_0 .. o_{N-2}) writes m_{N-1} contiguous outputs of a y row.
// grid (T/256, K, prod_{j<N-1} m_j).
__global__ void __launch_bounds__(256)
k_nd_scatter_last(const float* __restrict__ src, float* __restrict__ y, const __grid_constant__ KGeom g,
                  const __grid_constant__ NdParams q, int N, int64_t t_lo, int64_t t_hi) {
  const int64_t t = t_lo + (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int k = blockIdx.y;
  const int orest = blockIdx.z;  // (o_0 .. o_{N-2}) row-major
  pdl_wait();
  pdl_trigger();
  if (t >= t_hi) return;
  const int L = N - 1, aL = q.a[L], mL = q.m[L];
  const int64_t pl = (int64_t)g.K * g.T_s;  // xi stride of the last axis
  const float* s0 = src + ((int64_t)orest * aL * g.K + k) * g.T_s + (t - g.t0);
  float v[kMaxA];
#pragma unroll
  for (int i = 0; i < kMaxA; ++i)
    if (i < aL) v[i] = __ldg(s0 + i * pl);
  int tn[kMaxN], on[kMaxN];
  const int b = decode_tile((int)t, g, N, tn);
  int rem = orest;
  for (int j = L - 1; j >= 0; --j) {
    on[j] = rem % q.m[j];
    rem /= q.m[j];
  }
  bool ok = true;
  int64_t off = 0;
  for (int j = 0; j < L; ++j) {
    const int64_t pos = (int64_t)tn[j] * q.m[j] + on[j];
    ok = ok && pos < g.out[j];
    off += pos * g.out_stride[j];
  }
  if (!ok) return;
  const float bk = g.bias ? __ldg(g.bias + k) : 0.f;
  float* yr = y + ((int64_t)b * g.K + k) * g.out_vol + off;
#pragma unroll
  for (int o = 0; o < kMaxA; ++o) {
    if (o >= mL) break;
    const int64_t pos = (int64_t)tn[L] * mL + o;
    if (pos >= g.out[L]) break;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxA; ++i)
      if (i < aL) acc = fmaf(q.AT[L][o][i], v[i], acc);
    if (g.bias || g.act) {
      acc += bk;
      if (g.act == 1) acc = fmaxf(acc, 0.f);
    }
    yr[pos] = acc;
  }
}

}  // namespace

cudaError_t launch_input_nd(const float* x, float* V, const KGeom& g, const NdParams& q, int N, int64_t P,
                            int64_t t_lo, int64_t t_hi, cudaStream_t s) {
  const unsigned bx = (unsigned)((t_hi - t_lo + 255) / 256);
  // extraction fused with the last axis' B^T (one V pass less, contiguous x rows)
  cudaError_t e = launch_pdl(k_nd_extract_last, dim3(bx, (unsigned)g.C, (unsigned)(P / q.a[N - 1])), dim3(256), 0,
                             s, x, V, g, q, N, t_lo, t_hi);
  for (int n = N - 2; n >= 0 && e == cudaSuccess; --n) {
    if (q.a[n] == 1 && q.BT[n][0][0] == 1.f) continue;  // r_n = m_n = 1: B_n^T = [1], nothing to do
    e = launch_pdl(k_nd_mode_in, dim3(bx, (unsigned)g.C, (unsigned)(P / q.a[n])), dim3(256), 0, s, V, g, q, N, n,
                   t_lo, t_hi);
  }
  return e;
}

cudaError_t launch_output_nd(const float* Mx, float* W, float* y, const KGeom& g, const NdParams& q, int N,
                             int64_t t_lo, int64_t t_hi, cudaStream_t s) {
  const unsigned bx = (unsigned)((t_hi - t_lo + 255) / 256);
  int ein[4] = {1, 1, 1, 1};
  for (int n = 0; n < N; ++n) ein[n] = q.a[n];
  const float* src = Mx;
  float* bufs[2] = {W, const_cast<float*>(Mx)};
  int which = 0;
  cudaError_t e = cudaSuccess;
  // axes 0 .. N-2 reduced alpha -> m in M <-> W, then the last axis fused
  // with the scatter (each thread writes m_{N-1} contiguous floats of y)
  for (int n = 0; n <= N - 2 && e == cudaSuccess; ++n) {
    if (ein[n] == 1 && q.m[n] == 1 && q.AT[n][0][0] == 1.f) continue;  // A_n^T = [1]
    int lines = 1;
    for (int j = 0; j < N; ++j)
      if (j != n) lines *= ein[j];
    float* dst = bufs[which];
    e = launch_pdl(k_nd_mode_out, dim3(bx, (unsigned)g.K, (unsigned)lines), dim3(256), 0, s, src, dst, g, q, N, n,
                   make_int4(ein[0], ein[1], ein[2], ein[3]), t_lo, t_hi);
    ein[n] = q.m[n];
    src = dst;
    which ^= 1;
  }
  if (e != cudaSuccess) return e;
  int rest = 1;
  for (int j = 0; j < N - 1; ++j) rest *= q.m[j];
  return launch_pdl(k_nd_scatter_last, dim3(bx, (unsigned)g.K, (unsigned)rest), dim3(256), 0, s, src, y, g, q, N,
                    t_lo, t_hi);
}

}  // namespace wino
