// verify.cu -- exact componentwise check of a DD/QD product on the GPU.
//
// For each sampled output (i, j) this computes, EXACTLY,
//     d_ij = c_ij - sum_k a_ik * b_kj
// where every operand is the unevaluated sum of its 2 (DD) or 4 (QD)
// doubles: each component product x*y is split error-free into p + e
// (p = x*y, e = fma(x, y, -p)) and every p, e and component of c is added
// into a Kulisch-style fixed-point superaccumulator covering 2^-1100 ..
// 2^1100 (69 base-2^32 digits held in int64 for carry headroom).  It also
// sums S_ij = sum_k |a_ik| |b_kj| in double (relative error < l * 2^-52,
// covered by a 2^-40 inflation) and reports
//     ratio_ij = |d_ij| / (4 * l * 2^-u_exp * S_ij)
// i.e. the north_star bound |c - c_exact| <= 4 l u (|A||B|)_ij holds iff
// ratio <= 1 (u_exp = 104 for DD, 209 for QD).  This is SURVEY.md s8f-3's
// "superaccumulator exact-dot kernel": it makes exact verification of
// whole 1024^2 results, and of large samples at 8192^2, practical.
//
// One warp per sampled output: lanes split k, each lane keeps its own
// accumulator, the warp then sums the digit vectors with shuffles.
// A TwoProd whose error could underflow (|p| < 2^-960) is not exact; such
// samples report NaN instead of a ratio.
#include <cmath>
#include <cstdint>

#include "kernels.h"

namespace mpmm {

namespace {

constexpr int kDigits = 69;      // 69 * 32 = 2208 bits
constexpr int kOffset = 1100;    // bit 0 of digit 0 has weight 2^-1100

__device__ __forceinline__ void acc_add(int64_t* acc, double d, bool negate) {
  if (d == 0.0) return;
  unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(d));
  bool neg = (bits >> 63) != 0;
  if (negate) neg = !neg;
  int be = static_cast<int>((bits >> 52) & 0x7ff);
  unsigned long long man = bits & ((1ull << 52) - 1);
  int e2;
  if (be == 0) {
    e2 = -1074;               // subnormal: value = man * 2^-1074
  } else {
    man |= (1ull << 52);
    e2 = be - 1075;           // value = man * 2^(be - 1075)
  }
  int off = e2 + kOffset;     // >= 26
  int q = off >> 5, r = off & 31;
  unsigned __int128 w = static_cast<unsigned __int128>(man) << r;
  int64_t d0 = static_cast<int64_t>(static_cast<uint32_t>(w));
  int64_t d1 = static_cast<int64_t>(static_cast<uint32_t>(w >> 32));
  int64_t d2 = static_cast<int64_t>(static_cast<uint32_t>(w >> 64));
  if (neg) {
    d0 = -d0;
    d1 = -d1;
    d2 = -d2;
  }
  acc[q] += d0;
  if (q + 1 < kDigits) acc[q + 1] += d1;
  if (q + 2 < kDigits) acc[q + 2] += d2;
}

// Carry-propagate the (signed) digits and return |value| as a double.
__device__ double acc_magnitude(int64_t* acc) {
  int64_t carry = 0;
  for (int q = 0; q < kDigits; ++q) {
    int64_t v = acc[q] + carry;
    carry = v >> 32;                         // arithmetic shift: floor division
    acc[q] = v - (carry << 32);              // now in [0, 2^32)
  }
  // value = (carry * 2^(32*kDigits) + X) * 2^-kOffset with X = sum acc[q] 2^(32q);
  // |value| < 2^1024 guarantees carry in {0, -1}.  For carry = -1 the
  // magnitude is the two's complement 2^(32*kDigits) - X.
  if (carry < 0) {
    int64_t c = 1;
    for (int q = 0; q < kDigits; ++q) {
      int64_t v = (0xffffffffll - acc[q]) + c;
      c = v >> 32;
      acc[q] = v & 0xffffffffll;
    }
  }
  double v = 0.0;
  for (int q = kDigits - 1; q >= 0; --q)
    if (acc[q] != 0) v += ldexp(static_cast<double>(acc[q]), 32 * q - kOffset);
  return v;
}

template <int V>
__global__ void __launch_bounds__(128)
exact_check_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                   int64_t ldb, const double* __restrict__ C, int64_t ldc, int l,
                   const int64_t* __restrict__ idx_i, const int64_t* __restrict__ idx_j,
                   int64_t count, int u_exp, double* __restrict__ ratio) {
  constexpr int K = 2 * V;   // components per element
  const int lane = threadIdx.x & 31;
  const int64_t s = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (s >= count) return;
  const int64_t i = idx_i[s], j = idx_j[s];
  int64_t acc[kDigits];
#pragma unroll
  for (int q = 0; q < kDigits; ++q) acc[q] = 0;
  double absum = 0.0;
  bool inexact = false;
  for (int k = lane; k < l; k += 32) {
    const double* a = A + (i * lda + k) * K;
    const double* b = B + (static_cast<int64_t>(k) * ldb + j) * K;
    double x[K], y[K];
#pragma unroll
    for (int t = 0; t < K; ++t) {
      x[t] = a[t];
      y[t] = b[t];
    }
#pragma unroll
    for (int s1 = 0; s1 < K; ++s1)
#pragma unroll
      for (int s2 = 0; s2 < K; ++s2) {
        double p = x[s1] * y[s2];
        double e = __fma_rn(x[s1], y[s2], -p);
        if (p != 0.0 && fabs(p) < 0x1p-960) inexact = true;
        if (!isfinite(p)) inexact = true;
        acc_add(acc, p, true);
        acc_add(acc, e, true);
        absum += fabs(p);
      }
  }
  if (lane == 0) {
#pragma unroll
    for (int t = 0; t < K; ++t) acc_add(acc, C[(i * ldc + j) * K + t], false);
  }
  // warp reduction of the digit vectors and flags
  for (int q = 0; q < kDigits; ++q) {
    int64_t v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    acc[q] = v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) absum += __shfl_down_sync(0xffffffffu, absum, o);
  inexact = __any_sync(0xffffffffu, inexact);
  if (lane != 0) return;
  double d = acc_magnitude(acc);
  double bound = 4.0 * l * ldexp(1.0, -u_exp) * absum * (1.0 + 0x1p-40);
  double r;
  if (inexact) {
    r = NAN;
  } else if (d == 0.0) {
    r = 0.0;
  } else if (bound == 0.0) {
    r = INFINITY;
  } else {
    r = d / bound;
  }
  ratio[s] = r;
}

}  // namespace

cudaError_t exact_check_launch(int comps, int l, const double* A, int64_t lda, const double* B,
                               int64_t ldb, const double* C, int64_t ldc, const int64_t* idx_i,
                               const int64_t* idx_j, int64_t count, int u_exp, double* ratio,
                               cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  int64_t blocks = (count * 32 + 127) / 128;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  if (comps == 2)
    exact_check_kernel<1><<<(unsigned)blocks, 128, 0, stream>>>(A, lda, B, ldb, C, ldc, l, idx_i,
                                                                idx_j, count, u_exp, ratio);
  else
    exact_check_kernel<2><<<(unsigned)blocks, 128, 0, stream>>>(A, lda, B, ldb, C, ldc, l, idx_i,
                                                                idx_j, count, u_exp, ratio);
  return cudaGetLastError();
}

}  // namespace mpmm
