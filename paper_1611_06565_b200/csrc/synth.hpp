// synth.hpp -- exact-rational Toom-Cook synthesis of the 1-D Winograd
// transforms F(m, r) (stage a0), usable both at run time (plan_create, any
// interpolation points) and at compile time (constexpr tables that let the
// transform kernels fold zero and +-1 entries, "U is sparse",
// PAPER.md:221 "exploiting the sparsity of the matrices").
//
// Construction (the only parameter is m(x) = prod (x - p_k);
// "Cook-Toom"): with alpha = m + r - 1 points p_k (one may be infinity),
//   V_n (alpha x n) Vandermonde rows (1, p, .., p^{n-1}); infinity row (0..0,1)
//   linear convolution of a length-r kernel with length-m data:
//       s = V_alpha^{-1} [(V_r g) (.) (V_m d)]
//   its transpose is the length-alpha-tile correlation F(m, r) of Eq. (1):
//       A^T = V_m^T (m x alpha),  G = V_r (alpha x r),  B^T = V_alpha^{-T}
// followed by the diagonal rescaling of DESIGN.md reading #6 (each B^T row a
// primitive integer vector, positive factor moved into the G row).  The exact
// bilinear identity  A^T[(G g) (.) (B^T d)] = valid correlation  is checked
// on every basis pair before anything is emitted.
//
// Floats are emitted round-to-nearest-even from the exact rationals.
#pragma once
#include <stdint.h>

namespace wino {

constexpr int kMaxAlpha = 10;

using i128 = __int128;

constexpr i128 iabs(i128 v) { return v < 0 ? -v : v; }
constexpr i128 igcd(i128 a, i128 b) {
  a = iabs(a);
  b = iabs(b);
  while (b != 0) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}

struct Rat {
  int64_t n = 0, d = 1;  // d > 0, gcd(n, d) = 1
};

struct RatOps {
  bool overflow = false;
  constexpr Rat make(i128 n, i128 d) {
    if (d == 0) { overflow = true; return Rat{}; }
    if (d < 0) { n = -n; d = -d; }
    i128 g = igcd(n, d);
    if (g > 1) { n /= g; d /= g; }
    const i128 lim = (i128)INT64_MAX;
    if (n > lim || -n > lim || d > lim) { overflow = true; return Rat{}; }
    return Rat{(int64_t)n, (int64_t)d};
  }
  constexpr Rat add(Rat a, Rat b) { return make((i128)a.n * b.d + (i128)b.n * a.d, (i128)a.d * b.d); }
  constexpr Rat sub(Rat a, Rat b) { return make((i128)a.n * b.d - (i128)b.n * a.d, (i128)a.d * b.d); }
  constexpr Rat mul(Rat a, Rat b) { return make((i128)a.n * b.n, (i128)a.d * b.d); }
  constexpr Rat div(Rat a, Rat b) { return make((i128)a.n * b.d, (i128)a.d * b.n); }
};

constexpr bool req(Rat a, Rat b) { return a.n == b.n && a.d == b.d; }

struct Point {
  bool inf = false;
  Rat v{};
};

struct Transforms {
  int m = 0, r = 0, a = 0;
  Point pts[kMaxAlpha]{};
  Rat AT[kMaxAlpha][kMaxAlpha]{};  // m x alpha
  Rat G[kMaxAlpha][kMaxAlpha]{};   // alpha x r
  Rat BT[kMaxAlpha][kMaxAlpha]{};  // alpha x alpha
  int err = 0;                     // 0 ok, 3 points, 4 synth/overflow/identity
};

// Default point sequences (reading #5): alpha == 6 uses
// {0, 3/2, -3/2, 2/3, -2/3, inf} (lower fp32 error than {0,+-1,+-2,inf});
// otherwise 0, 1, -1, 2, -2, 1/2, -1/2, 3, -3, 1/3, -1/3, ... then inf.
enum PointSet { kPsDefault = 0, kPsSeq = 1, kPsAlt6 = 2 };

constexpr Point seq_point(int i) {
  // 0, 1, -1, 2, -2, 1/2, -1/2, 3, -3, 1/3, -1/3, 4, -4
  const int64_t num[] = {0, 1, -1, 2, -2, 1, -1, 3, -3, 1, -1, 4, -4};
  const int64_t den[] = {1, 1, 1, 1, 1, 2, 2, 1, 1, 3, 3, 1, 1};
  Point p;
  p.v = Rat{num[i], den[i]};
  return p;
}

constexpr int default_points(int alpha, int ps, Point* out) {
  if (alpha < 1 || alpha > kMaxAlpha) return 3;
  if (alpha == 1) { out[0] = Point{}; return 0; }
  if ((ps == kPsAlt6 || ps == kPsDefault) && alpha == 6) {
    const int64_t num[] = {0, 3, -3, 2, -2};
    const int64_t den[] = {1, 2, 2, 3, 3};
    for (int i = 0; i < 5; ++i) out[i].v = Rat{num[i], den[i]}, out[i].inf = false;
    out[5].inf = true;
    return 0;
  }
  if (ps == kPsAlt6) return 3;
  for (int i = 0; i < alpha - 1; ++i) out[i] = seq_point(i);
  out[alpha - 1].inf = true;
  return 0;
}

// Vandermonde row value p^j (infinity row = e_{n-1}).
constexpr Rat vand(RatOps& o, const Point& p, int j, int n) {
  if (p.inf) return Rat{j == n - 1 ? 1 : 0, 1};
  Rat v{1, 1};
  for (int t = 0; t < j; ++t) v = o.mul(v, p.v);
  return v;
}

constexpr bool check_identity(const Transforms& t) {
  // sum_xi AT[o][xi] G[xi][i] BT[xi][j] == [j == o + i] for all o < m, i < r, j < alpha
  RatOps o;
  for (int oo = 0; oo < t.m; ++oo)
    for (int i = 0; i < t.r; ++i)
      for (int j = 0; j < t.a; ++j) {
        Rat s{0, 1};
        for (int x = 0; x < t.a; ++x) s = o.add(s, o.mul(o.mul(t.AT[oo][x], t.G[x][i]), t.BT[x][j]));
        if (o.overflow) return false;
        if (!req(s, Rat{j == oo + i ? 1 : 0, 1})) return false;
      }
  return true;
}

constexpr Transforms synthesize(int m, int r, const Point* pts) {
  Transforms t;
  RatOps o;
  const int a = m + r - 1;
  t.m = m;
  t.r = r;
  t.a = a;
  if (m < 1 || r < 1 || a > kMaxAlpha) { t.err = 3; return t; }
  int ninf = 0;
  for (int k = 0; k < a; ++k) {
    t.pts[k] = pts[k];
    if (pts[k].inf) ++ninf;
    if (!pts[k].inf && pts[k].v.d <= 0) { t.err = 3; return t; }
    for (int l = 0; l < k; ++l)
      if (!pts[k].inf && !pts[l].inf && req(pts[k].v, pts[l].v)) { t.err = 3; return t; }
  }
  if (ninf > 1) { t.err = 3; return t; }
  // A^T = V_m^T, G = V_r
  for (int k = 0; k < a; ++k) {
    for (int j = 0; j < m; ++j) t.AT[j][k] = vand(o, pts[k], j, m);
    for (int j = 0; j < r; ++j) t.G[k][j] = vand(o, pts[k], j, r);
  }
  // B^T = (V_alpha^{-1})^T via Gauss-Jordan on [V | I]
  Rat W[kMaxAlpha][2 * kMaxAlpha]{};
  for (int k = 0; k < a; ++k)
    for (int j = 0; j < a; ++j) {
      W[k][j] = vand(o, pts[k], j, a);
      W[k][a + j] = Rat{k == j ? 1 : 0, 1};
    }
  for (int c = 0; c < a; ++c) {
    int piv = -1;
    for (int k = c; k < a; ++k)
      if (W[k][c].n != 0) { piv = k; break; }
    if (piv < 0) { t.err = 4; return t; }
    if (piv != c)
      for (int j = 0; j < 2 * a; ++j) { Rat tmp = W[c][j]; W[c][j] = W[piv][j]; W[piv][j] = tmp; }
    const Rat inv = o.div(Rat{1, 1}, W[c][c]);
    for (int j = 0; j < 2 * a; ++j) W[c][j] = o.mul(W[c][j], inv);
    for (int k = 0; k < a; ++k)
      if (k != c && W[k][c].n != 0) {
        const Rat f = W[k][c];
        for (int j = 0; j < 2 * a; ++j) W[k][j] = o.sub(W[k][j], o.mul(f, W[c][j]));
      }
  }
  for (int i = 0; i < a; ++i)
    for (int j = 0; j < a; ++j) t.BT[i][j] = W[j][a + i];  // (V^{-1})^T
  // reading #6: B^T rows -> primitive integer vectors, factor into G rows
  for (int k = 0; k < a; ++k) {
    i128 L = 1;
    for (int j = 0; j < a; ++j) L = L / igcd(L, t.BT[k][j].d) * t.BT[k][j].d;
    i128 h = 0;
    for (int j = 0; j < a; ++j) h = igcd(h, (i128)t.BT[k][j].n * (L / t.BT[k][j].d));
    if (h == 0) { t.err = 4; return t; }
    const Rat lam = o.make(h, L);  // B^T row / lam is integral, primitive
    for (int j = 0; j < a; ++j) t.BT[k][j] = o.div(t.BT[k][j], lam);
    for (int j = 0; j < r; ++j) t.G[k][j] = o.mul(t.G[k][j], lam);
  }
  if (o.overflow || !check_identity(t)) t.err = 4;
  return t;
}

// Round-to-nearest-even of the exact rational n/d to a binary float with MB
// significand bits (24: float, 53: double).
template <int MB>
constexpr double rat_to_fp(Rat q) {
  if (q.n == 0) return 0.0;
  const bool neg = q.n < 0;
  const i128 un = neg ? -(i128)q.n : (i128)q.n;
  const i128 ud = q.d;
  auto bitlen = [](i128 v) {
    int b = 0;
    while (v > 0) { v >>= 1; ++b; }
    return b;
  };
  int s = MB - 1 - (bitlen(un) - bitlen(ud));
  i128 num = 0, den = 0, qq = 0;
  for (int iter = 0; iter < 4; ++iter) {
    num = s >= 0 ? (un << s) : un;
    den = s >= 0 ? ud : (ud << (-s));
    qq = num / den;
    if (qq >= ((i128)1 << MB)) { --s; continue; }
    if (qq < ((i128)1 << (MB - 1))) { ++s; continue; }
    break;
  }
  const i128 rem = num - qq * den;
  if (2 * rem > den || (2 * rem == den && (qq & 1))) ++qq;
  double v = (double)(int64_t)qq;  // exact: qq <= 2^MB <= 2^53
  for (int i = 0; i < s; ++i) v *= 0.5;
  for (int i = 0; i < -s; ++i) v *= 2.0;
  return neg ? -v : v;
}

constexpr float rat_to_f32(Rat q) { return (float)rat_to_fp<24>(q); }  // exact narrowing
constexpr double rat_to_f64(Rat q) { return rat_to_fp<53>(q); }

// Float tables of one synthesised transform set (used by kernels).
struct FloatTables {
  int m = 0, r = 0, a = 0;
  float AT[kMaxAlpha][kMaxAlpha]{};
  float BT[kMaxAlpha][kMaxAlpha]{};
  double G[kMaxAlpha][kMaxAlpha]{};
};

constexpr FloatTables to_tables(const Transforms& t) {
  FloatTables f;
  f.m = t.m;
  f.r = t.r;
  f.a = t.a;
  for (int i = 0; i < kMaxAlpha; ++i)
    for (int j = 0; j < kMaxAlpha; ++j) {
      f.AT[i][j] = rat_to_f32(t.AT[i][j]);
      f.BT[i][j] = rat_to_f32(t.BT[i][j]);
      f.G[i][j] = rat_to_f64(t.G[i][j]);
    }
  return f;
}

constexpr Transforms synthesize_default(int m, int r, int ps) {
  Point p[kMaxAlpha]{};
  Transforms t;
  if (default_points(m + r - 1, ps, p) != 0) { t.err = 3; return t; }
  return synthesize(m, r, p);
}

}  // namespace wino
