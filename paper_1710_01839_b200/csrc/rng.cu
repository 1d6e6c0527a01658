// rng.cu -- device-side seeded inputs, bitwise equal to the numpy spec.
//
// SURVEY.md s8d defines the BASELINE inputs with numpy.random.default_rng
// (PCG64, XSL-RR 128/64 output) and SURVEY s8f-3 asks for the same matrices
// generated on the GPU.  numpy's Generator.uniform(-1, 1) consumes one
// 64-bit draw per double: u = (x >> 11) * 2^-53, value = -1 + 2 u.  Draw k
// of a stream is the output of the LCG state after k+1 steps, so every
// thread jumps straight to its first draw (O(log k) 128-bit LCG
// composition) and then steps sequentially through a contiguous chunk.
//
// The element assembly repeats the numpy operation order exactly:
//   DD: lo = (hi * 2^-53) * f; (hi, lo) = TwoSum(hi, lo)
//   QD: x_i = (x0 * 2^(-53 i)) * u_i, then the reference's _compress4 of
//       (x0, x1, x2, x3) (ddqd.py:175-193; ddqd.cuh compress4 paths).
#include <cstdint>

#include "ddqd.cuh"
#include "kernels.h"

namespace mpmm {

namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
  return (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
}

// state after `delta` LCG steps (pcg_advance_lcg_128)
__device__ u128 lcg_advance(u128 state, u128 delta, u128 mult, u128 plus) {
  u128 acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= mult;
      acc_plus = acc_plus * mult + plus;
    }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  uint64_t x = static_cast<uint64_t>(s >> 64) ^ static_cast<uint64_t>(s);
  unsigned rot = static_cast<unsigned>(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr int kChunk = 64;

__global__ void uniform_kernel(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                               uint64_t first, int64_t count, double* __restrict__ out) {
  const int64_t e0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kChunk;
  if (e0 >= count) return;
  const u128 mult = pcg_mult();
  const u128 inc = (static_cast<u128>(i_hi) << 64) | i_lo;
  u128 s = (static_cast<u128>(s_hi) << 64) | s_lo;
  // draw e (global index first + e) is the output after first + e + 1 steps
  s = lcg_advance(s, static_cast<u128>(first + e0), mult, inc);
  const int64_t e1 = e0 + kChunk < count ? e0 + kChunk : count;
  for (int64_t e = e0; e < e1; ++e) {
    s = s * mult + inc;
    double u = static_cast<double>(xsl_rr(s) >> 11) * (1.0 / 9007199254740992.0);
    out[e] = -1.0 + 2.0 * u;
  }
}

__global__ void dd_assemble_kernel(const double* __restrict__ hi, const double* __restrict__ f,
                                   int64_t count, double2* __restrict__ out) {
  int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= count) return;
  double h = hi[e];
  double lo = (h * 0x1p-53) * f[e];
  double err;
  double s = two_sum(h, lo, err);
  out[e] = make_double2(s, err);
}

__global__ void qd_assemble_kernel(const double* __restrict__ x0, const double* __restrict__ u,
                                   int64_t count, double2* __restrict__ out) {
  int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= count) return;
  double v[4];
  v[0] = x0[e];
  v[1] = (v[0] * 0x1p-53) * u[e];
  v[2] = (v[0] * 0x1p-106) * u[count + e];
  v[3] = (v[0] * 0x1p-159) * u[2 * count + e];
  double r[4];
  if (nonzero(v[0]) & nonzero(v[1]) & nonzero(v[2]) & nonzero(v[3])) {
    compress4_dense<4>(v, r);
  } else {
    compress4_general(v, 4, r);
  }
  out[2 * e] = make_double2(r[0], r[1]);
  out[2 * e + 1] = make_double2(r[2], r[3]);
}

}  // namespace

cudaError_t uniform_launch(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                           uint64_t first, int64_t count, double* out, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  int64_t threads = (count + kChunk - 1) / kChunk;
  int64_t blocks = (threads + 255) / 256;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  uniform_kernel<<<(unsigned)blocks, 256, 0, stream>>>(s_hi, s_lo, i_hi, i_lo, first, count, out);
  return cudaGetLastError();
}

cudaError_t assemble_launch(int comps, const double* draws, int64_t count, double* out,
                            cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  if (comps == 2)
    dd_assemble_kernel<<<(unsigned)blocks, 256, 0, stream>>>(draws, draws + count, count,
                                                             reinterpret_cast<double2*>(out));
  else
    qd_assemble_kernel<<<(unsigned)blocks, 256, 0, stream>>>(draws, draws + count, count,
                                                             reinterpret_cast<double2*>(out));
  return cudaGetLastError();
}

}  // namespace mpmm
