// ddqd.cuh -- double-double / quad-double device arithmetic for sm_100a.
//
// Every routine here reproduces, rounding for rounding, the operation
// sequence of the reference kernels (/root/reference/pkg/src/mpmm/
// _kernels.pyx), so the GPU results are bit-identical to the reference CPU
// results.  Two rules make that hold:
//
//  * this translation unit is compiled with -fmad=false, so nvcc never
//    contracts an a*b+c into a DFMA on its own: every multiply and add
//    rounds separately, as the reference's -ffp-contract=off build does;
//  * TwoProd uses ONE explicit DFMA for the error term (err = fma(a,b,-p))
//    instead of the reference's Veltkamp/Dekker split (_kernels.pyx:19-29).
//    Both yield the unique exact error a*b - p whenever the Dekker split is
//    exact (|a|,|b| < 2^996, no underflow of the error -- the reference's
//    own eft.py:21-24 range), so the two are bit-identical there.  This
//    removes 20 of the 87 FP64 operations of a DD multiply-add.
#pragma once

#include <cstdint>

namespace mpmm {

// eft.py:27-30 _two_sum_raw
__device__ __forceinline__ double two_sum(double a, double b, double& err) {
  double s = a + b;
  double bb = s - a;
  err = (a - (s - bb)) + (b - bb);
  return s;
}

// TwoSum through magnitude order: s = fl(a + b) and the same exact error
// as two_sum, in 3 DADD instead of 6.  With t the operand of larger
// magnitude and u the other, t - s is exact (Sterbenz) and (t - s) + u is
// the exact a + b - s (Fast2Sum, Dekker 1971), the unique value two_sum
// also returns -- so every later rounding sees the same operand.  The
// sign of a zero error matches too: two_sum's error is never -0.0, and
// (t - s) + u is -0.0 only if t - s = -0.0, i.e. t = -0.0 with s = +0.0,
// which |u| <= |t| rules out.
//
// The order test costs no FP64 pipe time: the high words of a and b
// (sign, 11 exponent bits, 20 mantissa bits), read as float32 bit patterns
// under |.|, compare like the magnitudes of the doubles whenever their
// exponent fields are below 0x7f8 (|x| < 2^1017; the reference's own
// TwoProd guard is 2^996, eft.py:21) -- one FSETP on the FP32 side plus
// four SELs on the ALU pipe.  Equal high words mean equal exponents, for
// which either order is exact (float32 subnormal patterns, i.e. doubles
// below 2^-1015, compare exactly too: no -ftz).
__device__ __forceinline__ double two_sum_ord(double a, double b, double& err) {
  double s = a + b;
  const float fa = __int_as_float(__double2hiint(a));
  const float fb = __int_as_float(__double2hiint(b));
  const bool ge = fabsf(fa) >= fabsf(fb);
  const double t = ge ? a : b;
  const double u = ge ? b : a;
  err = (t - s) + u;
  return s;
}

// Either TwoSum, chosen at compile time (both bit-identical; see above).
template <bool ORD>
__device__ __forceinline__ double two_sum_t(double a, double b, double& err) {
  if constexpr (ORD) return two_sum_ord(a, b, err);
  else return two_sum(a, b, err);
}

// eft.py:33-36 _quick_two_sum_raw
__device__ __forceinline__ double quick_two_sum(double a, double b, double& err) {
  double s = a + b;
  err = b - (s - a);
  return s;
}

// eft.py:45-49 _two_prod_raw, error term by DFMA (exact; see header).
__device__ __forceinline__ double two_prod(double a, double b, double& err) {
  double p = a * b;
  err = __fma_rn(a, b, -p);
  return p;
}

// _kernels.pyx:19-29 _two_prod verbatim: Veltkamp split by 2^27 + 1 and
// Dekker's product.  Outside the domain where its error is exact (a split
// overflows for |x| >= ~2^996 -- the NaN the reference then returns --, or
// the error falls below the subnormal floor) it differs from two_prod; the
// GEMM launches route such operands here (domain.cuh), so the reference's
// results are reproduced there too, NaN for NaN.
__device__ __forceinline__ double two_prod_dekker(double a, double b, double& err) {
  const double splitter = 134217729.0;   // 2^27 + 1
  double p = a * b;
  double t = splitter * a;
  double ahh = t - (t - a);
  double ahl = a - ahh;
  t = splitter * b;
  double bhh = t - (t - b);
  double bhl = b - bhh;
  err = ((ahh * bhh - p) + ahh * bhl + ahl * bhh) + ahl * bhl;
  return p;
}

template <bool DEKKER>
__device__ __forceinline__ double two_prod_t(double a, double b, double& err) {
  if constexpr (DEKKER) return two_prod_dekker(a, b, err);
  else return two_prod(a, b, err);
}

// ---------------------------------------------------------------------------
// double-double
// ---------------------------------------------------------------------------

// ddqd.py:63-70 dd_add == _kernels.pyx:189-204 (20 DADD; 14 when ORD)
template <bool ORD = false>
__device__ __forceinline__ void dd_add(double xh, double xl, double yh, double yl,
                                       double& hi, double& lo) {
  double s2, t2, e;
  double s1 = two_sum_t<ORD>(xh, yh, s2);
  double t1 = two_sum_t<ORD>(xl, yl, t2);
  s2 = s2 + t1;
  s1 = quick_two_sum(s1, s2, e);
  s2 = e + t2;
  hi = quick_two_sum(s1, s2, lo);
}

// ddqd.py:77-91 dd_mul, as inlined at _kernels.pyx:140-171
// (4 DMUL + 3 DFMA + 23 DADD; 17 DADD when ORD).
template <bool ORD = false, bool DEKKER = false>
__device__ __forceinline__ void dd_mul(double ah, double al, double bh, double bl,
                                       double& ph, double& pl) {
  double e, e1, e2, r1, r2, w;
  double p = two_prod_t<DEKKER>(ah, bh, e);
  double p1 = two_prod_t<DEKKER>(ah, bl, e1);
  double p2 = two_prod_t<DEKKER>(al, bh, e2);
  double tail = (e1 + e2) + al * bl;
  double s = two_sum_t<ORD>(p1, p2, r1);
  s = two_sum_t<ORD>(e, s, r2);
  double losum = (r1 + r2) + tail;
  double h = quick_two_sum(p, s, w);
  w = w + losum;
  ph = quick_two_sum(h, w, pl);
}

// One DD multiply-add, the k-loop body of _kernels.pyx:135-184:
// c <- dd_add(c, dd_mul(a, b)).  50 FP64 instructions, 53 flops; with
// ORD the four TwoSums run as two_sum_ord: 38 FP64 instructions (4 DMUL +
// 3 DFMA + 31 DADD) + 4 FSETP + 16 SEL, same bits.
// DEKKER: the reference's split TwoProd (two_prod_dekker), for operands
// outside the DFMA-exact domain.
template <bool ORD = false, bool DEKKER = false>
__device__ __forceinline__ void dd_madd(double& ch, double& cl, double ah, double al,
                                        double bh, double bl) {
  double ph, pl;
  dd_mul<ORD, DEKKER>(ah, al, bh, bl, ph, pl);
  dd_add<ORD>(ch, cl, ph, pl, ch, cl);
}

// Faithful ("fast") DD multiply-add -- NOT the reference's sequence, an
// opt-in accuracy mode that meets the north_star
// bound |c - c_exact| <= 4 l u (|A||B|)_ij, u = 2^-104, checked against the
// exact rational oracle (tests/test_gpu_fast.py).  15 FP64 instructions
// (1 DMUL + 3 DFMA + 11 DADD = 18 flops) instead of the mirror's 50:
//   p + e = ah*bh + ah*bl + al*bh to ~2^-106 (al*bl dropped, < 2^-106 |ab|),
//   (ch, cl) += (p, e) with an exact TwoSum of the high parts and one
//   rounded add of the low parts, renormalised every step.
// Per step the new error is at most ~3 * 2^-106 * (|c| + |ab|), i.e. about
// 0.2 of the bound's per-step budget 2^-102 (|A||B|)_ij.
__device__ __forceinline__ void dd_madd_fast(double& ch, double& cl, double ah, double al,
                                             double bh, double bl) {
  double p = ah * bh;
  double e = __fma_rn(ah, bh, -p);
  e = __fma_rn(ah, bl, e);
  e = __fma_rn(al, bh, e);
  double t;
  double s = two_sum(ch, p, t);
  t = t + (cl + e);
  ch = quick_two_sum(s, t, cl);
}

// ---------------------------------------------------------------------------
// quad-double
// ---------------------------------------------------------------------------

// x != 0.0 with IEEE semantics (-0.0 is zero, NaN is not), tested on the
// bit pattern so the check runs on the integer pipe instead of issuing a
// DSETP on the FP64 pipe the arithmetic is bound by.
// (The 64-bit shift form gets pattern-matched back into a DSETP by the
// compiler; splitting the register pair in PTX keeps it on the ALU.)
__device__ __forceinline__ bool nonzero(double x) {
  unsigned lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(x));
  return ((hi & 0x7fffffffu) | lo) != 0u;
}

// Conservative nonzero test on the high word only: true means x != 0
// (some exponent or top-mantissa bit is set); false means "maybe zero"
// (x = +-0, or |x| < 2^-1042 with only low-word bits), which callers send
// to their exact path.  The high word read as a float32 under != 0 is one
// FSETP, and a chain of them folds into one predicate (FSETP.AND), where
// nonzero() is LOP3 + ISETP per term -- the QD multiply-add is bound by
// register-file reads, and each ALU instruction costs one.
__device__ __forceinline__ bool hi_nonzero(double x) {
  return __int_as_float(__double2hiint(x)) != 0.0f;
}

// ---- speculative dense path (gemm.cuh gemm_tile_interior, QDSpecOps) ------
// The gates above decide, per multiply-add, whether the register-only dense
// sequences apply: 23 + 8 + 3 + 3 high-word tests, their predicate combines
// and four branches -- ~70 non-FP64 instructions per multiply-add, 3 % of
// the QD GEMM's time (profiles/r02_qd_variants.log).  The speculative path
// runs the dense sequences unconditionally and only RECORDS the tests: a
// running minimum of |high word| (read as float32) over every tested value,
// one three-input FMNMX3 per two values, no branch.  The CTA looks at the
// minimum once per k-tile (__syncthreads_or at the barrier it has anyway);
// if any tested value may have been zero, the tile is abandoned and
// recomputed from the start by the gated, exact kernel.  A tile that
// completes therefore executed exactly the operations the gates would have
// selected -- the same bits -- and a tile that does not is never stored.

// min(|a|, |b|, |c|) of three float32 bit patterns: FMNMX3 |a|,|b|,|c|
// (sm_100).  A NaN pattern (a high word of |x| >= 2^1017: never zero) is
// skipped by min; a subnormal pattern stays nonzero (no .ftz).
__device__ __forceinline__ float min3_abs(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(fabsf(a)), "f"(fabsf(b)), "f"(fabsf(c)));
  return d;
}

__device__ __forceinline__ float hi_as_float(double x) {
  return __int_as_float(__double2hiint(x));
}

// fold the high words of t[0..N) into the running minimum m: two values
// per FMNMX3 (a chain through m -- off the arithmetic's critical path)
template <int N>
__device__ __forceinline__ void fold_min_hi(float& m, const double (&t)[N]) {
#ifdef MPMM_SPEC_NO_TESTS   // experiment only: the cost of the recorded tests
  return;
#endif
#pragma unroll
  for (int i = 0; i < N; i += 2)
    m = min3_abs(m, hi_as_float(t[i]), hi_as_float(t[i + 1 < N ? i + 1 : i]));
}

// true when some folded value had a zero high word (sign ignored)
__device__ __forceinline__ bool min_hi_is_zero(float m) {
  return (__float_as_int(m) & 0x7fffffff) == 0;
}

// ddqd.py:140-172 _renorm5 == _kernels.pyx:237-271: the general case,
// branch-free: the data-dependent "if e != 0" emission becomes predicated
// selects.  In the reference's k == 3 case "acc += v" equals the s
// computed below, so the only behavioural difference of the k == 3 case is
// that nothing is emitted.
__device__ __forceinline__ void renorm5_emit(double t, double x1, double x2, double x3,
                                             double x4, double out[4]) {
  double o0 = 0.0, o1 = 0.0, o2 = 0.0, o3 = 0.0;
  double acc = t;
  int k = 0;
  const double rest[4] = {x1, x2, x3, x4};
#pragma unroll
  for (int idx = 0; idx < 4; ++idx) {
    double v = rest[idx];
    double sn = acc + v;
    double e = v - (sn - acc);
    bool emit = (k < 3) && nonzero(e);
    if (emit) {
      o0 = (k == 0) ? sn : o0;
      o1 = (k == 1) ? sn : o1;
      o2 = (k == 2) ? sn : o2;
    }
    acc = emit ? e : sn;
    k += emit ? 1 : 0;
  }
  o0 = (k == 0) ? acc : o0;
  o1 = (k == 1) ? acc : o1;
  o2 = (k == 2) ? acc : o2;
  o3 = (k == 3) ? acc : o3;
  out[0] = o0;
  out[1] = o1;
  out[2] = o2;
  out[3] = o3;
}

// _renorm5 with a fast path for the common case: the first three emission
// errors e1, e2, e3 are nonzero, so the reference emits sn1, sn2, sn3 and
// ends (k = 3) with acc = e3 + x4.  Same operations on the same operands
// as the general loop (whose fourth error is never used when k = 3), so
// the same bits; any possibly-zero error takes renorm5_emit.
__device__ __forceinline__ void renorm5(double x0, double x1, double x2, double x3,
                                        double x4, double out[4]) {
  double s, t;
  s = quick_two_sum(x3, x4, x4);
  t = quick_two_sum(x2, s, x3);
  s = quick_two_sum(x1, t, x2);
  t = quick_two_sum(x0, s, x1);
  const double sn1 = t + x1;
  const double e1 = x1 - (sn1 - t);
  const double sn2 = e1 + x2;
  const double e2 = x2 - (sn2 - e1);
  const double sn3 = e2 + x3;
  const double e3 = x3 - (sn3 - e2);
  if (__builtin_expect(hi_nonzero(e1) & hi_nonzero(e2) & hi_nonzero(e3), 1)) {
    out[0] = sn1;
    out[1] = sn2;
    out[2] = sn3;
    out[3] = e3 + x4;
  } else {
    renorm5_emit(t, x1, x2, x3, x4, out);
  }
}

// renorm5's fast path taken unconditionally, its gate (e1, e2, e3 nonzero)
// recorded in m: valid only if the caller later finds m nonzero.
__device__ __forceinline__ void renorm5_spec(double x0, double x1, double x2, double x3,
                                             double x4, double out[4], float& m, double extra) {
  double s, t;
  s = quick_two_sum(x3, x4, x4);
  t = quick_two_sum(x2, s, x3);
  s = quick_two_sum(x1, t, x2);
  t = quick_two_sum(x0, s, x1);
  const double sn1 = t + x1;
  const double e1 = x1 - (sn1 - t);
  const double sn2 = e1 + x2;
  const double e2 = x2 - (sn2 - e1);
  const double sn3 = e2 + x3;
  const double e3 = x3 - (sn3 - e2);
  const double tested[4] = {extra, e1, e2, e3};   // `extra`: a value of the caller's to test
  fold_min_hi(m, tested);
  out[0] = sn1;
  out[1] = sn2;
  out[2] = sn3;
  out[3] = e3 + x4;
}

// ddqd.py:175-193 _compress4 for N terms that are ALL nonzero (the zero
// filter is then the identity).  Fully unrolled: registers only.
//
// The four error-free vector passes are issued as a wavefront: pass p's
// step i runs in "round" i + 2p.  Step (p, i) needs v[i] from pass p-1's
// step i+1 (round i+2p-1) and pass p's own running sum from step i-1
// (round i+2p-1), and it overwrites v[i-1], which pass p-1 last read in
// round i+2p-3 and pass p+1 first reads in round i+2p+1.  Every TwoSum
// therefore sees exactly the operands of the sequential loop
// (ddqd.py:181-186) -- same bits -- while each round holds up to four
// independent TwoSums, so in-order issue is not stalled by the pass chains.
//
// ORDMASK bit p runs pass p's TwoSums as two_sum_ord (same bits, half the
// DADDs, the order test on the FP32/ALU pipes): a knob to balance the FP64
// pipe against the ALU pipe, which the QD multiply-add loads with its zero
// tests and selects.
template <int N, int ORDMASK = 0, bool SPEC = false>
__device__ __forceinline__ void compress4_dense(double (&v)[N], double out[4],
                                                float* m = nullptr, double extra = 1.0) {
  double s[4];
#pragma unroll
  for (int d = 1; d <= (N - 1) + 6; ++d) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int i = d - 2 * p;
      if (i >= 1 && i <= N - 1) {
        if (i == 1) s[p] = v[0];
        if ((ORDMASK >> p) & 1)
          s[p] = two_sum_ord(s[p], v[i], v[i - 1]);
        else
          s[p] = two_sum(s[p], v[i], v[i - 1]);
        if (i == N - 1) v[N - 1] = s[p];
      }
    }
  }
  if constexpr (N <= 4) {
    static_assert(!SPEC, "the speculative path compresses 23 and 8 terms only");
    double w[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < N; ++i) w[4 - N + i] = v[i];
    renorm5(w[3], w[2], w[1], w[0], 0.0, out);
  } else {
    double tail = 0.0;
#pragma unroll
    for (int i = 0; i < N - 4; ++i) tail += v[i];
    if constexpr (SPEC)
      renorm5_spec(v[N - 1], v[N - 2], v[N - 3], v[N - 4], tail, out, *m, extra);
    else
      renorm5(v[N - 1], v[N - 2], v[N - 3], v[N - 4], tail, out);
  }
}

// ddqd.py:175-193 _compress4, general case (some terms zero): compaction
// with a runtime count.  Rare on full-entropy data; kept out of line so the
// dense path stays in registers.
static __device__ __noinline__ void compress4_general(const double* terms, int nterms,
                                                     double* out) {
  double buf[24];
  int n = 0;
  for (int i = 0; i < nterms; ++i)
    if (terms[i] != 0.0) buf[n++] = terms[i];
  if (n == 0) {
    out[0] = out[1] = out[2] = out[3] = 0.0;
    return;
  }
  for (int p = 0; p < 4; ++p) {
    double s = buf[0];
    for (int i = 1; i < n; ++i) s = two_sum(s, buf[i], buf[i - 1]);
    buf[n - 1] = s;
  }
  if (n <= 4) {
    double w[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < n; ++i) w[4 - n + i] = buf[i];
    renorm5(w[3], w[2], w[1], w[0], 0.0, out);
    return;
  }
  double tail = 0.0;
  for (int i = 0; i < n - 4; ++i) tail += buf[i];
  renorm5(buf[n - 1], buf[n - 2], buf[n - 3], buf[n - 4], tail, out);
}

// Copy into a private array before the out-of-line call so the caller's
// term array never has its address taken (it then stays in registers).
template <int N>
__device__ __forceinline__ void compress4_slow(const double (&v)[N], double out[4]) {
  double tmp[N];
#pragma unroll
  for (int i = 0; i < N; ++i) tmp[i] = v[i];
  double o[4];
  compress4_general(tmp, N, o);
  out[0] = o[0];
  out[1] = o[1];
  out[2] = o[2];
  out[3] = o[3];
}

// _kernels.pyx:311-341 _qd_mul_add: cc += x*y, bit-identical.
// M23 / M8: ORDMASKs of the product's 23-term and the accumulate's 8-term
// compressions (see compress4_dense).
// DEKKER: the reference's split TwoProd (outside the DFMA-exact domain).
template <int M23 = 0, int M8 = 0, bool DEKKER = false>
__device__ __forceinline__ void qd_mul_add(double cc[4], const double x[4], const double y[4]) {
  double t[23];
  t[0] = two_prod_t<DEKKER>(x[0], y[0], t[1]);
  t[2] = two_prod_t<DEKKER>(x[0], y[1], t[3]);
  t[4] = two_prod_t<DEKKER>(x[1], y[0], t[5]);
  t[6] = two_prod_t<DEKKER>(x[0], y[2], t[7]);
  t[8] = two_prod_t<DEKKER>(x[1], y[1], t[9]);
  t[10] = two_prod_t<DEKKER>(x[2], y[0], t[11]);
  t[12] = two_prod_t<DEKKER>(x[0], y[3], t[13]);
  t[14] = two_prod_t<DEKKER>(x[1], y[2], t[15]);
  t[16] = two_prod_t<DEKKER>(x[2], y[1], t[17]);
  t[18] = two_prod_t<DEKKER>(x[3], y[0], t[19]);
  t[20] = x[1] * y[3];
  t[21] = x[2] * y[2];
  t[22] = x[3] * y[1];
  // dense gate: every high word nonzero => every term nonzero (a false
  // negative only costs the exact compaction path, same bits)
  bool dense = true;
#pragma unroll
  for (int i = 0; i < 23; ++i) dense &= hi_nonzero(t[i]);
  double prod[4];
  if (dense) {
    compress4_dense<23, M23>(t, prod);
  } else {
    compress4_slow<23>(t, prod);
  }
  double add[8] = {cc[0], prod[0], cc[1], prod[1], cc[2], prod[2], cc[3], prod[3]};
  bool cz = !nonzero(cc[0]) & !nonzero(cc[1]) & !nonzero(cc[2]) & !nonzero(cc[3]);
  bool pd = hi_nonzero(prod[0]) & hi_nonzero(prod[1]) & hi_nonzero(prod[2]) &
            hi_nonzero(prod[3]);
  bool cd = hi_nonzero(cc[0]) & hi_nonzero(cc[1]) & hi_nonzero(cc[2]) & hi_nonzero(cc[3]);
  if (cd & pd) {
    compress4_dense<8, M8>(add, cc);
  } else if (cz & pd) {
    // filtered term list is exactly prod[0..3] (k = 0 of every product)
    double p4[4] = {prod[0], prod[1], prod[2], prod[3]};
    compress4_dense<4>(p4, cc);
  } else {
    compress4_slow<8>(add, cc);
  }
}

// _qd_mul_add with every gate of qd_mul_add assumed to pass -- the all-dense
// 23-term and 8-term compressions and both renorm5 fast paths -- and the
// gates' tests folded into m instead of branched on (see above).  The
// result is the reference's exactly when m stays nonzero.
//
// Which values are folded (18 per multiply-add instead of the gates' 37):
//  * NOT the 13 products: a launch of the DFMA kernels runs inside the EFT
//    domain (domain.cuh: exponents of nonzero operand components sum to
//    >= -900), where two limbs with nonzero high words have a normal
//    product -- and the operand limbs are folded once per staged k-tile
//    element by the thread that copied it (qd_spec_stage), not once per use;
//  * the 10 TwoProd errors;
//  * of the 8-term gate's cc[0..3], prod[0..3] only cc[3] and prod[3]: the
//    other six are the sums sn1..sn3 of a renorm5 fast path, and sn_i with a
//    zero high word is zero or subnormal, hence an exact sum, hence e_i = 0
//    -- already folded by that renorm5_spec.  (The caller folds all of
//    cc[0..3] once after its gated first step: qd_spec_seed.)
//  * both renorm5 gates (e1, e2, e3).
__device__ __forceinline__ void qd_mul_add_spec(double cc[4], const double x[4],
                                                const double y[4], float& m) {
  double t[23];
  t[0] = two_prod(x[0], y[0], t[1]);
  t[2] = two_prod(x[0], y[1], t[3]);
  t[4] = two_prod(x[1], y[0], t[5]);
  t[6] = two_prod(x[0], y[2], t[7]);
  t[8] = two_prod(x[1], y[1], t[9]);
  t[10] = two_prod(x[2], y[0], t[11]);
  t[12] = two_prod(x[0], y[3], t[13]);
  t[14] = two_prod(x[1], y[2], t[15]);
  t[16] = two_prod(x[2], y[1], t[17]);
  t[18] = two_prod(x[3], y[0], t[19]);
  t[20] = x[1] * y[3];
  t[21] = x[2] * y[2];
  t[22] = x[3] * y[1];
  const double tested[10] = {t[1], t[3], t[5], t[7], t[9], t[11], t[13], t[15], t[17], t[19]};
  fold_min_hi(m, tested);
  double prod[4];
  const double c3 = cc[3];
  compress4_dense<23, 0, true>(t, prod, &m, c3);       // + the incoming cc[3]
  double add[8] = {cc[0], prod[0], cc[1], prod[1], cc[2], prod[2], cc[3], prod[3]};
  const double p3 = prod[3];
  compress4_dense<8, 0, true>(add, cc, &m, p3);        // + this step's prod[3]
}

// one staged 16-byte chunk (two operand limbs), by the thread that copied it
__device__ __forceinline__ void qd_spec_stage(double2 v, float& m) {
  m = min3_abs(m, hi_as_float(v.x), hi_as_float(v.y));
}

// all four accumulator limbs, once, after a gated step (see above)
__device__ __forceinline__ void qd_spec_seed(const double cc[4], float& m) {
  const double c[4] = {cc[0], cc[1], cc[2], cc[3]};
  fold_min_hi(m, c);
}

// qd_ewise_add / qd_ewise_sub body (_kernels.pyx:407-452)
__device__ __forceinline__ void qd_add(const double x[4], const double y[4], double out[4]) {
  double add[8] = {x[0], y[0], x[1], y[1], x[2], y[2], x[3], y[3]};
  bool dense = true;
#pragma unroll
  for (int i = 0; i < 8; ++i) dense &= nonzero(add[i]);
  if (dense) {
    compress4_dense<8>(add, out);
  } else {
    compress4_slow<8>(add, out);
  }
}

}  // namespace mpmm
