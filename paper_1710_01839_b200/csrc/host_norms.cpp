// host_norms.cpp -- Frobenius norm / relative difference in working
// precision, on the host (reference pkg/src/mpmm/matrix.py:207-294).
//
// The reference evaluates these sequentially in DD/QD arithmetic
// (ddqd.py) as a verification utility; this is the same left-to-right
// accumulation and the same sqrt/div iterations, in C++ compiled without
// contraction, so the returned doubles equal the reference's.  It runs on
// the host because the reference's result depends on the sequential order;
// it is a checker, not part of the GEMM path.
#include <cmath>
#include <cstdint>
#include <cstring>

namespace {

struct Ctx {
  bool overflow = false;
};

constexpr double kSplitter = 134217729.0;  // eft.py:19

inline double two_sum(double a, double b, double& e) {
  double s = a + b, bb = s - a;
  e = (a - (s - bb)) + (b - bb);
  return s;
}
inline double quick_two_sum(double a, double b, double& e) {
  double s = a + b;
  e = b - (s - a);
  return s;
}
inline void split(double a, double& h, double& l) {
  double t = kSplitter * a;
  h = t - (t - a);
  l = a - h;
}
inline double two_prod(double a, double b, double& e) {
  double p = a * b, ah, al, bh, bl;
  split(a, ah, al);
  split(b, bh, bl);
  e = ((ah * bh - p) + ah * bl + al * bh) + al * bl;
  return p;
}

// ---- double-double (ddqd.py:63-133) ----
struct DD {
  double h, l;
};
inline DD chk(Ctx& c, DD x) {
  if (!std::isfinite(x.h)) c.overflow = true;
  return x;
}
DD dd_add(Ctx& c, DD x, DD y) {
  double s2, t2, e;
  double s1 = two_sum(x.h, y.h, s2);
  double t1 = two_sum(x.l, y.l, t2);
  s2 += t1;
  s1 = quick_two_sum(s1, s2, e);
  s2 = e + t2;
  DD r;
  r.h = quick_two_sum(s1, s2, r.l);
  return chk(c, r);
}
DD dd_neg(DD x) { return {-x.h, -x.l}; }
DD dd_mul(Ctx& c, DD x, DD y) {
  double e, e1, e2, r1, r2, w;
  double p = two_prod(x.h, y.h, e);
  double p1 = two_prod(x.h, y.l, e1);
  double p2 = two_prod(x.l, y.h, e2);
  double tail = (e1 + e2) + x.l * y.l;
  double s = two_sum(p1, p2, r1);
  s = two_sum(e, s, r2);
  double lo_sum = (r1 + r2) + tail;
  double hi = quick_two_sum(p, s, w);
  w += lo_sum;
  DD r;
  r.h = quick_two_sum(hi, w, r.l);
  return chk(c, r);
}
DD dd_mul_double(Ctx& c, DD x, double d) {
  double e;
  double p = two_prod(x.h, d, e);
  e += x.l * d;
  DD r;
  r.h = quick_two_sum(p, e, r.l);
  return chk(c, r);
}
DD dd_div(Ctx& c, DD x, DD y) {
  double q1 = x.h / y.h;
  DD r = dd_add(c, x, dd_neg(dd_mul_double(c, y, q1)));
  double q2 = r.h / y.h;
  r = dd_add(c, r, dd_neg(dd_mul_double(c, y, q2)));
  double q3 = r.h / y.h;
  r = dd_add(c, r, dd_neg(dd_mul_double(c, y, q3)));
  double q4 = r.h / y.h;
  double t1, t2, t3;
  double s = quick_two_sum(q3, q4, t3);
  s = quick_two_sum(q2, s, t2);
  double hi = quick_two_sum(q1, s, t1);
  double lo = t1 + (t2 + t3);
  DD out;
  out.h = quick_two_sum(hi, lo, out.l);
  return chk(c, out);
}
DD dd_sqrt(Ctx& c, DD x) {
  if (x.h == 0.0 && x.l == 0.0) return {0.0, 0.0};
  DD r{std::sqrt(x.h), 0.0};
  for (int i = 0; i < 2; ++i) {
    DD t = dd_add(c, r, dd_div(c, x, r));
    r = {t.h * 0.5, t.l * 0.5};
  }
  return r;
}

// ---- quad-double (ddqd.py:140-274) ----
struct QD {
  double v[4];
};
void renorm5(double x0, double x1, double x2, double x3, double x4, double out[4]) {
  double s = quick_two_sum(x3, x4, x4);
  s = quick_two_sum(x2, s, x3);
  s = quick_two_sum(x1, s, x2);
  s = quick_two_sum(x0, s, x1);
  double comp[4] = {0.0, 0.0, 0.0, 0.0};
  double rest[4] = {x1, x2, x3, x4};
  int k = 0;
  double acc = s;
  for (double t : rest) {
    if (k == 3) {
      acc += t;
      continue;
    }
    double e;
    acc = quick_two_sum(acc, t, e);
    if (e != 0.0) {
      comp[k++] = acc;
      acc = e;
    }
  }
  comp[k] = acc;
  std::memcpy(out, comp, sizeof comp);
}
QD compress4(const double* terms, int nterms) {
  double v[32];
  int n = 0;
  for (int i = 0; i < nterms; ++i)
    if (terms[i] != 0.0) v[n++] = terms[i];
  QD out{{0.0, 0.0, 0.0, 0.0}};
  if (n == 0) return out;
  for (int p = 0; p < 4; ++p) {
    double s = v[0];
    for (int i = 1; i < n; ++i) s = two_sum(s, v[i], v[i - 1]);
    v[n - 1] = s;
  }
  if (n <= 4) {
    double w[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < n; ++i) w[4 - n + i] = v[i];
    renorm5(w[3], w[2], w[1], w[0], 0.0, out.v);
    return out;
  }
  double tail = 0.0;
  for (int i = 0; i < n - 4; ++i) tail += v[i];
  renorm5(v[n - 1], v[n - 2], v[n - 3], v[n - 4], tail, out.v);
  return out;
}
inline QD chk(Ctx& c, QD x) {
  if (!std::isfinite(x.v[0])) c.overflow = true;
  return x;
}
QD qd_add(Ctx& c, const QD& x, const QD& y) {
  double t[8] = {x.v[0], y.v[0], x.v[1], y.v[1], x.v[2], y.v[2], x.v[3], y.v[3]};
  return chk(c, compress4(t, 8));
}
QD qd_neg(const QD& x) { return {{-x.v[0], -x.v[1], -x.v[2], -x.v[3]}}; }
QD qd_mul(Ctx& c, const QD& x, const QD& y) {
  const double* a = x.v;
  const double* b = y.v;
  double t[23];
  const int pairs[10][2] = {{0, 0}, {0, 1}, {1, 0}, {0, 2}, {1, 1},
                            {2, 0}, {0, 3}, {1, 2}, {2, 1}, {3, 0}};
  for (int q = 0; q < 10; ++q) t[2 * q] = two_prod(a[pairs[q][0]], b[pairs[q][1]], t[2 * q + 1]);
  t[20] = a[1] * b[3];
  t[21] = a[2] * b[2];
  t[22] = a[3] * b[1];
  return chk(c, compress4(t, 23));
}
QD qd_mul_double(Ctx& c, const QD& x, double d) {
  double t[7];
  t[0] = two_prod(x.v[0], d, t[1]);
  t[2] = two_prod(x.v[1], d, t[3]);
  t[4] = two_prod(x.v[2], d, t[5]);
  t[6] = x.v[3] * d;
  return chk(c, compress4(t, 7));
}
QD qd_div(Ctx& c, const QD& x, const QD& y) {
  double q[5];
  QD r = x;
  for (int i = 0; i < 4; ++i) {
    q[i] = r.v[0] / y.v[0];
    r = qd_add(c, r, qd_neg(qd_mul_double(c, y, q[i])));
  }
  q[4] = r.v[0] / y.v[0];
  QD out;
  renorm5(q[0], q[1], q[2], q[3], q[4], out.v);
  return chk(c, out);
}
bool qd_zero(const QD& x) { return x.v[0] == 0.0 && x.v[1] == 0.0 && x.v[2] == 0.0 && x.v[3] == 0.0; }
QD qd_sqrt(Ctx& c, const QD& x) {
  if (qd_zero(x)) return {{0.0, 0.0, 0.0, 0.0}};
  QD r{{std::sqrt(x.v[0]), 0.0, 0.0, 0.0}};
  for (int i = 0; i < 3; ++i) {
    QD t = qd_add(c, r, qd_div(c, x, r));
    r = {{t.v[0] * 0.5, t.v[1] * 0.5, t.v[2] * 0.5, t.v[3] * 0.5}};
  }
  return r;
}
double qd_to_float(const QD& x) { return ((x.v[3] + x.v[2]) + x.v[1]) + x.v[0]; }

}  // namespace

extern "C" {

// matrix.py:229-236 frobenius_norm.  Returns 0, 1 = overflow (RangeError),
// 2 = negative square (ValueError).
int mpmm_host_frobenius_norm(int comps, const double* x, int64_t count, double* out) {
  Ctx c;
  if (comps == 2) {
    DD acc{0.0, 0.0};
    for (int64_t i = 0; i < count; ++i) {
      DD v{x[2 * i], x[2 * i + 1]};
      acc = dd_add(c, acc, dd_mul(c, v, v));
    }
    if (acc.h < 0.0) return 2;
    DD r = dd_sqrt(c, acc);
    *out = r.h + r.l;
  } else {
    QD acc{{0.0, 0.0, 0.0, 0.0}};
    for (int64_t i = 0; i < count; ++i) {
      QD v{{x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]}};
      acc = qd_add(c, acc, qd_mul(c, v, v));
    }
    if (acc.v[0] < 0.0) return 2;
    *out = qd_to_float(qd_sqrt(c, acc));
  }
  return c.overflow ? 1 : 0;
}

// matrix.py:239-294 frobenius_rel_diff: ||X - Y||_F / ||Y||_F, or ||X||_F
// ... the reference returns ||X-Y||_F when ||Y||_F is zero (matrix.py:263-264).
int mpmm_host_frobenius_rel_diff(int comps, const double* x, const double* y, int64_t count,
                                 double* out) {
  Ctx c;
  if (comps == 2) {
    DD dsq{0.0, 0.0}, ysq{0.0, 0.0};
    for (int64_t i = 0; i < count; ++i) {
      DD xv{x[2 * i], x[2 * i + 1]}, yv{y[2 * i], y[2 * i + 1]};
      DD d = dd_add(c, xv, dd_neg(yv));
      dsq = dd_add(c, dsq, dd_mul(c, d, d));
      ysq = dd_add(c, ysq, dd_mul(c, yv, yv));
    }
    DD dn = dd_sqrt(c, dsq), yn = dd_sqrt(c, ysq);
    if (yn.h == 0.0 && yn.l == 0.0) {
      *out = dn.h + dn.l;
    } else {
      DD q = dd_div(c, dn, yn);
      *out = q.h + q.l;
    }
  } else {
    QD dsq{{0.0, 0.0, 0.0, 0.0}}, ysq{{0.0, 0.0, 0.0, 0.0}};
    for (int64_t i = 0; i < count; ++i) {
      QD xv{{x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]}};
      QD yv{{y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3]}};
      QD d = qd_add(c, xv, qd_neg(yv));
      dsq = qd_add(c, dsq, qd_mul(c, d, d));
      ysq = qd_add(c, ysq, qd_mul(c, yv, yv));
    }
    QD dn = qd_sqrt(c, dsq), yn = qd_sqrt(c, ysq);
    *out = qd_zero(yn) ? qd_to_float(dn) : qd_to_float(qd_div(c, dn, yn));
  }
  return c.overflow ? 1 : 0;
}

}  // extern "C"
