// domain.cuh -- where the DFMA TwoProd equals the reference's Dekker TwoProd.
//
// The reference's kernels form every TwoProd error with Veltkamp's split
// and Dekker's product (_kernels.pyx:19-29); the mirror kernels use one
// DFMA (ddqd.cuh two_prod).  Both give the unique exact error a*b - fl(a*b)
// when, for every TwoProd operand pair (x from A, y from B):
//   * no split overflows: |x|, |y| < 2^995 (2^27+1 times them stays finite;
//     the reference's own guard is 2^996, eft.py:19-21);
//   * the product does not overflow: |x y| < 2^1001;
//   * the error is representable: e(x) + e(y) >= -900, far above the
//     -970 below which Dekker's partial products or the error itself fall
//     under the subnormal floor (eft.py:22-24);
//   * every operand is finite.
// Outside that domain the reference returns something else -- typically
// NaN from an overflowed split, which its caller reports as RangeError
// (multiply.py:124-127) -- and only the Dekker sequence reproduces it.
//
// A scan of the launch's operands (domain.cu) reduces, per operand, the
// largest biased exponent, the smallest biased exponent of a nonzero
// component and a non-finite flag into six words in HBM; every mirror GEMM
// launch carries a DomainGate and its CTAs read the words on entry: the DFMA
// kernel runs when the operands are inside the domain, the Dekker kernel
// (same tiles, two_prod_dekker) when they are not, and the other launch
// returns at once.  No host synchronisation; results are the reference's
// bits everywhere.
//
// Margins: a Strassen leaf multiplies sums of operand quadrants.  Sums of
// doubles that are all multiples of 2^q stay multiples of 2^q, so no
// nonzero leaf component is below 2^(emin - 52) -- margin_lo = 52 -- and
// each level at most doubles a magnitude -- margin_hi = depth + 1.
#pragma once

#include <cstdint>

namespace mpmm {

// words[0..2]: A's max biased exponent, 2047 - min nonzero biased exponent
// (0 when A is all zero), non-finite flag; words[3..5] the same for B.
constexpr int kDomainWords = 6;

struct DomainGate {
  const int* words = nullptr;   // null: the launch runs unconditionally
  int margin_lo = 0;            // exponent slack below (Strassen sums)
  int margin_hi = 0;            // exponent slack above (Strassen sums)
  int want_unsafe = 0;          // 0: run inside the domain; 1: run outside it
};

__host__ __device__ __forceinline__ bool domain_unsafe(const int* w, int margin_lo,
                                                       int margin_hi) {
  if (w[2] | w[5]) return true;
  const int max_a = w[0] - 1023 + margin_hi, max_b = w[3] - 1023 + margin_hi;
  if (max_a >= 995 || max_b >= 995 || max_a + max_b >= 1000) return true;
  if (w[1] == 0 || w[4] == 0) return false;   // an all-zero operand: every product is 0
  const int min_a = (2047 - w[1]) - 1023 - margin_lo;
  const int min_b = (2047 - w[4]) - 1023 - margin_lo;
  return min_a + min_b < -900;
}

#ifdef __CUDACC__
// True when this launch should not run (uniform per launch).
__device__ __forceinline__ bool gate_skip(const DomainGate& g) {
  if (g.words == nullptr) return false;
  int w[kDomainWords];
#pragma unroll
  for (int i = 0; i < kDomainWords; ++i) w[i] = __ldcg(g.words + i);
  return domain_unsafe(w, g.margin_lo, g.margin_hi) != (g.want_unsafe != 0);
}
#endif

}  // namespace mpmm
