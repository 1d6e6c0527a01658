// ozaki.cu -- exact DD/QD products on the int8 tensor cores (CRT scheme).
//
// Opt-in "tensor" mode (a non-mirror kernel states its own
// F and bound).  Every DD/QD entry is an exact scaled integer: with the
// per-row shift s_i = -min over the row of the lowest set bit of any
// component, a_ik * 2^s_i is an integer of at most beta_A bits (likewise
// b_kj * 2^t_j, beta_B bits).  The integer product
//     X_ij = sum_k (a_ik 2^s_i)(b_kj 2^t_j),  |X_ij| < l 2^(beta_A + beta_B)
// is computed EXACTLY from its residues modulo N pairwise-coprime moduli
// p_t <= 256 (product P > 2 |X|): residues of the inputs are int8, each
// residue product is one int8 GEMM with exact int32 accumulation on the
// tensor cores (int8gemm.cpp, cuBLASLt), and the Chinese remainder theorem
// rebuilds X_ij.  c_ij = X_ij 2^-(s_i + t_j) is then rounded once to the
// nearest DD (QD) expansion: the result is the exact product correctly
// rounded, far inside the north_star bound, but not bit-identical to the
// reference's step-by-step rounding.
//
// When beta_A + beta_B is too wide for the 54 available int8 moduli (363
// bits), the host splits each entry into component ranges (hi/lo) and the
// combine step sums the exact products of every pair of ranges, so the
// result is still the exact product, rounded once.  The planner
// (tensor.py) reports NotRepresentable when even single components do not
// fit.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace mpmm {

// The 54 pairwise-coprime prime powers <= 256, descending (sum of log2 =
// 362.8 bits).  ozaki.py holds the same list.
__constant__ int kModsDev[54] = {
    256, 251, 243, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191,
    181, 179, 173, 169, 167, 163, 157, 151, 149, 139, 137, 131, 127, 125,
    121, 113, 109, 107, 103, 101, 97,  89,  83,  79,  73,  71,  67,  61,
    59,  53,  49,  47,  43,  41,  37,  31,  29,  23,  19,  17};
constexpr int kNumMods = 54;
__constant__ unsigned kMod2p32[54] = {
    0,  123, 130, 15, 110, 8,  161, 176, 7,  51, 46, 88, 108, 147, 15, 126, 96, 113,
    7,  100, 93,  4,  129, 41, 34,  117, 16, 46, 59, 16, 75,  29,  63, 68,  35, 45,
    77, 50,  32,  9,  33,  57, 51,  42,  39, 42, 16, 37, 7,   4,   16, 12,  6,  1};

// floor(2^32 / p): Barrett reciprocals for 32-bit reductions
__constant__ unsigned kModMu[54] = {
    16777216u, 17111423u, 17674762u, 17821441u, 17970574u, 18433336u, 18755315u, 18920560u,
    19259943u, 20355295u, 21582750u, 21801864u, 22253716u, 22486739u, 23729101u, 23994230u,
    24826400u, 25414007u, 25718367u, 26349492u, 27356479u, 28443492u, 28825283u, 30899045u,
    31350126u, 32786009u, 33818640u, 34359738u, 35495597u, 38008560u, 39403369u, 40139881u,
    41698711u, 42524428u, 44278013u, 48258059u, 51746593u, 54366674u, 58835168u, 60492497u,
    64103989u, 70409299u, 72796055u, 81037118u, 87652393u, 91382282u, 99882960u, 104755299u,
    116080197u, 138547332u, 148102320u, 186737708u, 226050910u, 252645135u};

// x mod p for any 32-bit x (Barrett with mu = floor(2^32/p): the quotient
// estimate is low by at most one, so one conditional subtraction)
__device__ __forceinline__ unsigned barrett(unsigned x, unsigned mu, unsigned p) {
  unsigned r = x - __umulhi(x, mu) * p;
  return r >= p ? r - p : r;
}

namespace {

__device__ __forceinline__ int top_exp(double x) {  // |x| < 2^top_exp
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  int be = static_cast<int>((b >> 52) & 0x7ff);
  unsigned long long man = b & ((1ull << 52) - 1);
  if (be > 0) return be - 1022;
  return -1074 + (64 - __clzll(static_cast<long long>(man)));
}

__device__ __forceinline__ int low_bit(double x) {  // weight exponent of the lowest set bit
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  int be = static_cast<int>((b >> 52) & 0x7ff);
  unsigned long long man = b & ((1ull << 52) - 1);
  if (be > 0) man |= (1ull << 52);
  int e = be > 0 ? be - 1075 : -1074;
  return e + (__ffsll(static_cast<long long>(man)) - 1);
}

__device__ __forceinline__ bool is_zero(double x) {
  return (static_cast<unsigned long long>(__double_as_longlong(x)) << 1) == 0ull;
}

__device__ __forceinline__ bool not_finite(double x) {
  return ((static_cast<unsigned long long>(__double_as_longlong(x)) >> 52) & 0x7ff) == 0x7ff;
}

constexpr int kEmptyE = -100000, kEmptyL = 100000;

// One pass over a matrix: per row (by_cols 0) or column (1) and per
// component c, E[c] = max top_exp and L[c] = min low_bit over the nonzero
// entries; any non-finite component sets bit 0 of *status.  EL layout:
// E[comps][odim] then L[comps][odim].
//
// Rows: one block of kScanWarps warps per row (the warps split the row's
// columns, then combine through shared memory): one warp per row left a
// 1024-row operand at 7 warps per SM, latency-bound.
constexpr int kScanWarps = 4;

template <int NC>
__global__ void __launch_bounds__(32 * kScanWarps)
scan_rows_kernel(const double* __restrict__ X, int64_t ld, int rows, int cols,
                 int* __restrict__ EL, int* __restrict__ status) {
  __shared__ int sEL[kScanWarps][2 * NC];
  const int r = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int e[NC], lo[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) e[c] = kEmptyE, lo[c] = kEmptyL;
  bool bad = false;
  // four k per lane per step: independent loads in flight (one warp per row
  // leaves few warps per SM, so latency, not bandwidth, bounds this loop)
  constexpr int U = 8;
  for (int k0 = warp * 32 * U + lane; k0 < cols; k0 += kScanWarps * 32 * U) {
    double v[U][NC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + 32 * u;
#pragma unroll
      for (int c = 0; c < NC; ++c) v[u][c] = k < cols ? X[((int64_t)r * ld + k) * NC + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        bad |= not_finite(v[u][c]);
        if (!is_zero(v[u][c])) {
          e[c] = max(e[c], top_exp(v[u][c]));
          lo[c] = min(lo[c], low_bit(v[u][c]));
        }
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      e[c] = max(e[c], __shfl_xor_sync(0xffffffffu, e[c], o));
      lo[c] = min(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
    }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, 1);
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      sEL[warp][c] = e[c];
      sEL[warp][NC + c] = lo[c];
    }
  }
  __syncthreads();
  if (threadIdx.x < NC) {
    const int c = threadIdx.x;
    int ee = sEL[0][c], ll = sEL[0][NC + c];
#pragma unroll
    for (int w = 1; w < kScanWarps; ++w) {
      ee = max(ee, sEL[w][c]);
      ll = min(ll, sEL[w][NC + c]);
    }
    EL[c * rows + r] = ee;
    EL[(NC + c) * rows + r] = ll;
  }
}

__global__ void fill_el_kernel(int* __restrict__ EL, int nc, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < nc * n) {
    EL[j] = kEmptyE;
    EL[nc * n + j] = kEmptyL;
  }
}

// columns: a 32-column x 64-row tile per block (coalesced along the row),
// block reduction over the rows, then one atomic per column and component
template <int NC>
__global__ void scan_cols_kernel(const double* __restrict__ X, int64_t ld, int rows, int cols,
                                 int* __restrict__ EL, int* __restrict__ status) {
  __shared__ int se[NC][8][32], sl[NC][8][32];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  int e[NC], lo[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) e[c] = kEmptyE, lo[c] = kEmptyL;
  bool bad = false;
  if (j < cols) {
    const int k0 = blockIdx.y * 64;
    double v[8][NC];               // the 8 rows of this thread, loads in flight together
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + ty + 8 * u;
#pragma unroll
      for (int c = 0; c < NC; ++c) v[u][c] = k < rows ? X[((int64_t)k * ld + j) * NC + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        bad |= not_finite(v[u][c]);
        if (!is_zero(v[u][c])) {
          e[c] = max(e[c], top_exp(v[u][c]));
          lo[c] = min(lo[c], low_bit(v[u][c]));
        }
      }
  }
  if (__any_sync(0xffffffffu, bad) && tx == 0) atomicOr(status, 1);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    se[c][ty][tx] = e[c];
    sl[c][ty][tx] = lo[c];
  }
  __syncthreads();
  if (ty == 0 && j < cols) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      for (int q = 1; q < 8; ++q) {
        e[c] = max(e[c], se[c][q][tx]);
        lo[c] = min(lo[c], sl[c][q][tx]);
      }
      if (e[c] != kEmptyE) {
        atomicMax(EL + c * cols + j, e[c]);
        atomicMin(EL + (NC + c) * cols + j, lo[c]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// residues
// ---------------------------------------------------------------------------

constexpr int kMaxW = 12;   // 32-bit words of one scaled entry (384 bits)

// Constant tables for the residue dot products, built at compile time:
//   w4[t][w]   the 4 bytes 2^(8(4w+j)) mod p_t, centred into int8, packed
//   top[t][W]  (p_t - 2^(32W) mod p_t) mod p_t  (two's-complement sign fix)
//   bias[t]    a multiple of p_t >= 2^22 (keeps the dot product positive)
//   init[t][W] {bias + h, bias + h + top[t][W]}: the dot product's start
//              for a non-negative / negative entry, h = floor(p_t / 2)
//   muc[t]     ceil(2^32 / p_t): floor(x / p_t) = umulhi(x, muc) for every
//              x < 2^23 (checked exhaustively for all 54 moduli)
struct ResidueTables {
  uint32_t w4[kNumMods][kMaxW];
  uint32_t top[kNumMods][kMaxW + 1];
  uint32_t bias[kNumMods];
  uint32_t init[kNumMods][kMaxW + 1][2];
  uint32_t half[kNumMods];
  uint32_t muc[kNumMods];
};

constexpr int kModsHost[kNumMods] = {
    256, 251, 243, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191,
    181, 179, 173, 169, 167, 163, 157, 151, 149, 139, 137, 131, 127, 125,
    121, 113, 109, 107, 103, 101, 97,  89,  83,  79,  73,  71,  67,  61,
    59,  53,  49,  47,  43,  41,  37,  31,  29,  23,  19,  17};

constexpr ResidueTables make_residue_tables() {
  ResidueTables T{};
  for (int t = 0; t < kNumMods; ++t) {
    const uint32_t p = static_cast<uint32_t>(kModsHost[t]);
    uint32_t pw = 1 % p;                    // 2^(8i) mod p
    for (int w = 0; w < kMaxW; ++w) {
      uint32_t packed = 0;
      for (int j = 0; j < 4; ++j) {
        int c = static_cast<int>(pw);
        if (c > static_cast<int>(p / 2)) c -= static_cast<int>(p);
        if (c > 127) c -= static_cast<int>(p);   // p = 256: 0..255 -> -128..127
        packed |= (static_cast<uint32_t>(c) & 0xffu) << (8 * j);
        pw = (pw * 256u) % p;
      }
      T.w4[t][w] = packed;
    }
    uint32_t q = 1 % p;                     // 2^(32W) mod p
    for (int W = 0; W <= kMaxW; ++W) {
      T.top[t][W] = (p - q) % p;
      for (int s = 0; s < 32; ++s) q = (q * 2u) % p;
    }
    T.bias[t] = p * ((1u << 22) / p + 1u);
    T.half[t] = p / 2;
    T.muc[t] = static_cast<uint32_t>(((1ull << 32) + p - 1) / p);
    for (int W = 0; W <= kMaxW; ++W) {
      T.init[t][W][0] = T.bias[t] + p / 2;
      T.init[t][W][1] = T.bias[t] + p / 2 + T.top[t][W];
    }
  }
  return T;
}

__constant__ ResidueTables kRes = make_residue_tables();

__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// sum_{c < NC} x[c] * 2^shift as a W-word two's-complement integer
// (little-endian 32-bit words).  Every nonzero component is an integer
// multiple of 2^-shift (scan), and |sum| < 2^(32W-1) (host choice of W).
template <int NC, int W>
__device__ __forceinline__ void entry_words(const double* x, int shift, bool valid,
                                            uint32_t (&X)[W]) {
#pragma unroll
  for (int w = 0; w < W; ++w) X[w] = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double v = valid ? x[c] : 0.0;
    if (is_zero(v)) continue;
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    const int be = static_cast<int>((b >> 52) & 0x7ff);
    unsigned long long m = b & ((1ull << 52) - 1);
    if (be > 0) m |= (1ull << 52);
    const int tz = __ffsll(static_cast<long long>(m)) - 1;
    m >>= tz;
    const int e = (be > 0 ? be - 1075 : -1074) + shift + tz;   // >= 0
    const int q = e >> 5, r = e & 31;
    const unsigned long long t0 = m << r;
    const uint32_t d0 = static_cast<uint32_t>(t0), d1 = static_cast<uint32_t>(t0 >> 32);
    const uint32_t d2 = r ? static_cast<uint32_t>(m >> (64 - r)) : 0u;
    const bool neg = (b >> 63) != 0;
    unsigned long long carry = neg ? 1ull : 0ull;   // x - d == x + ~d + 1
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint32_t d = w == q ? d0 : (w == q + 1 ? d1 : (w == q + 2 ? d2 : 0u));
      if (neg) d = ~d;
      const unsigned long long s = static_cast<unsigned long long>(X[w]) + d + carry;
      X[w] = static_cast<uint32_t>(s);
      carry = s >> 32;
    }
  }
}

// centred residue of the W-word integer X modulo p_t, as an int8 byte
// Centred residue c = x mod p_t in [-floor(p/2), ceil(p/2) - 1] (the int8
// the residue GEMMs take; for p = 256 that is [-128, 127]) of a W-word
// two's-complement entry.  The dot product of the entry's bytes with the
// centred weights 2^(8j) mod p starts at init = bias + h (+ top for a
// negative entry), so x' = x + h lies in (2^21, 2^23); then
// q = floor(x' / p) = umulhi(x', ceil(2^32 / p)) exactly and c = x' - h - q p.
// Per entry and modulus: W DP4A + IMAD.HI + IMAD on the FMA pipe, one
// IADD (and a SEL for the start) on the ALU pipe -- no compare/select
// chain, which left the ALU pipe the bound.
template <int W>
__device__ __forceinline__ int residue_centred(const uint32_t (&X)[W], uint32_t init,
                                               uint32_t muc, uint32_t negp, uint32_t h,
                                               const uint32_t (&wt)[W]) {
  int acc = static_cast<int>(init);
#pragma unroll
  for (int w = 0; w < W; ++w) acc = dp4a_us(X[w], wt[w], acc);
  const uint32_t q = __umulhi(static_cast<uint32_t>(acc), muc);
  return static_cast<int>(static_cast<uint32_t>(acc) - h + q * negp);
}

// the low bytes of four ints packed little-endian (3 PRMT)
__device__ __forceinline__ uint32_t pack_bytes(int c0, int c1, int c2, int c3) {
  const uint32_t lo = __byte_perm(static_cast<uint32_t>(c0), static_cast<uint32_t>(c1), 0x0040);
  const uint32_t hi = __byte_perm(static_cast<uint32_t>(c2), static_cast<uint32_t>(c3), 0x0040);
  return __byte_perm(lo, hi, 0x5410);
}

struct ResidueConsts {
  uint32_t init0, init1, muc, negp, h;
};

template <int W>
__device__ __forceinline__ ResidueConsts load_weights(int t, uint32_t (&wt)[W]) {
  ResidueConsts k;
  k.init0 = kRes.init[t][W][0];
  k.init1 = kRes.init[t][W][1];
  k.muc = kRes.muc[t];
  k.negp = 0u - static_cast<uint32_t>(kModsDev[t]);
  k.h = kRes.half[t];
#pragma unroll
  for (int w = 0; w < W; ++w) wt[w] = kRes.w4[t][w];
  return k;
}

// the residue byte word of four entries (u = 0..3 in the low..high byte)
template <int W>
__device__ __forceinline__ uint32_t residue_word(const uint32_t (&X)[4][W], const bool (&neg)[4],
                                                 const ResidueConsts& k,
                                                 const uint32_t (&wt)[W]) {
  int c[4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
    c[u] = residue_centred<W>(X[u], neg[u] ? k.init1 : k.init0, k.muc, k.negp, k.h, wt);
  return pack_bytes(c[0], c[1], c[2], c[3]);
}

// A side: R[t][row][k], 4 consecutive k of one row per thread (reads and
// the packed int8x4 stores both coalesce along k).
template <int NC, int W>
__global__ void __launch_bounds__(256)
residues_rows_kernel(const double* __restrict__ X, int64_t ld, int rows, int cols, int comps,
                     int c0, const int* __restrict__ shift, int N, int8_t* __restrict__ R,
                     int64_t rpitch, int64_t rplane) {
  const int per = (cols + 3) / 4;
  const int64_t qd = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (qd >= static_cast<int64_t>(rows) * per) return;
  const int o = static_cast<int>(qd / per), k0 = static_cast<int>(qd % per) * 4;
  const int sh = shift[o];
  uint32_t Xw[4][W];
#pragma unroll
  for (int u = 0; u < 4; ++u)
    entry_words<NC, W>(X + ((int64_t)o * ld + k0 + u) * comps + c0, sh, k0 + u < cols, Xw[u]);
  int8_t* dst = R + static_cast<int64_t>(o) * rpitch + k0;
  bool neg[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) neg[u] = (Xw[u][W - 1] >> 31) != 0;
  // the constants of modulus t+1 are loaded while t is computed (the
  // indexed constant loads were the loop's critical path)
  uint32_t wt[W];
  ResidueConsts k = load_weights<W>(0, wt);
#pragma unroll 1
  for (int t = 0; t < N; ++t) {
    uint32_t wn[W];
    const ResidueConsts kn = load_weights<W>(t + 1 < N ? t + 1 : t, wn);
    *reinterpret_cast<uint32_t*>(dst + t * rplane) = residue_word<W>(Xw, neg, k, wt);
    k = kn;
#pragma unroll
    for (int w = 0; w < W; ++w) wt[w] = wn[w];
  }
}

// B side: R[t][col][k] (B transposed).  A block covers 32 columns x 32 k:
// lane = column (coalesced reads along the row of B), warp = k quad; the
// packed words go through shared memory so each column's 32 k leave as
// one 32-byte sector.
template <int NC, int W>
__global__ void __launch_bounds__(256)
residues_cols_kernel(const double* __restrict__ X, int64_t ld, int rows, int cols, int comps,
                     int c0, const int* __restrict__ shift, int N, int8_t* __restrict__ R,
                     int64_t rpitch, int64_t rplane) {
  // the packed words of kColChunk moduli go through shared memory per
  // barrier (one barrier per modulus left the kernel barrier/issue bound)
  constexpr int kColChunk = 8;
  __shared__ uint32_t S[kColChunk][32][9];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int o = blockIdx.x * 32 + lane;
  const int k0 = blockIdx.y * 32 + wq * 4;
  const bool col_ok = o < cols;
  const int sh = col_ok ? shift[o] : 0;
  uint32_t Xw[4][W];
#pragma unroll
  for (int u = 0; u < 4; ++u)
    entry_words<NC, W>(X + ((int64_t)(k0 + u) * ld + o) * comps + c0, sh,
                       col_ok && k0 + u < rows, Xw[u]);
  // write-out mapping: 8 threads per column, one k quad each
  const int oc = threadIdx.x >> 3, qq = threadIdx.x & 7;
  const int og = blockIdx.x * 32 + oc;
  const int kq = blockIdx.y * 32 + qq * 4;
  int8_t* dst = R + static_cast<int64_t>(og) * rpitch + kq;
  const bool store = og < cols && kq < rows;
  bool neg[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) neg[u] = (Xw[u][W - 1] >> 31) != 0;
  uint32_t wt[W];
  ResidueConsts k = load_weights<W>(0, wt);
#pragma unroll 1
  for (int t0 = 0; t0 < N; t0 += kColChunk) {
    const int cn = N - t0 < kColChunk ? N - t0 : kColChunk;
#pragma unroll 1
    for (int u = 0; u < cn; ++u) {
      const int t = t0 + u;
      uint32_t wn[W];
      const ResidueConsts kn = load_weights<W>(t + 1 < N ? t + 1 : t, wn);
      S[u][lane][wq] = residue_word<W>(Xw, neg, k, wt);
      k = kn;
#pragma unroll
      for (int w = 0; w < W; ++w) wt[w] = wn[w];
    }
    __syncthreads();
    if (store)
      for (int u = 0; u < cn; ++u)
        *reinterpret_cast<uint32_t*>(dst + (t0 + u) * rplane) = S[u][oc][qq];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// CRT reconstruction + exact combination + rounding to DD/QD
// ---------------------------------------------------------------------------

}  // namespace

// Per-job CRT data (device): moduli count, limb count, P limbs, weights.
constexpr int kMaxJobs = kOzMaxJobs;

// up to kMaxJobs jobs by value (kernel parameter space, no device table)
struct CrtJobs {
  CrtJob j[kMaxJobs];
};

// ---------------------------------------------------------------------------
// single-job combine: everything in registers (K limbs known at compile time)
// ---------------------------------------------------------------------------

// round-to-nearest double of the magnitude limbs * 2^ebase (top 64 bits +
// sticky), unrolled: no dynamic register indexing
template <int K>
__device__ __forceinline__ double limbs_round(const int64_t (&mag)[K], int ebase) {
  int top = -1;
#pragma unroll
  for (int q = 0; q < K; ++q)
    if (mag[q] != 0) top = q;
  if (top < 0) return 0.0;
  uint64_t hi = 0, mid = 0, lo = 0;
  bool sticky = false;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    uint64_t v = static_cast<uint64_t>(mag[q]);
    if (q == top) hi = v;
    if (q == top - 1) mid = v;
    if (q == top - 2) lo = v;
    if (q < top - 2) sticky |= (v != 0);
  }
  int lz = __clzll(static_cast<long long>(hi)) - 32;
  unsigned __int128 w = (static_cast<unsigned __int128>(hi) << 64) |
                        (static_cast<unsigned __int128>(mid) << 32) | lo;
  w <<= lz;
  uint64_t top64 = static_cast<uint64_t>(w >> 32);
  if ((static_cast<uint64_t>(w) & 0xffffffffull) != 0 || sticky) top64 |= 1ull;
  return ldexp(__ull2double_rn(top64), 32 * (top - 2) - lz + 32 + ebase);
}

// mag -= d (d >= 0, an integer multiple of 2^ebase); returns true when the
// difference turned negative (mag then holds its magnitude)
template <int K>
__device__ __forceinline__ bool limbs_sub_double(int64_t (&mag)[K], double d, int ebase) {
  if (d != 0.0) {
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
    int be = static_cast<int>((b >> 52) & 0x7ff);
    unsigned long long mm = b & ((1ull << 52) - 1);
    if (be > 0) mm |= (1ull << 52);
    int e = (be > 0 ? be - 1075 : -1074) - ebase;
    int tz = __ffsll(static_cast<long long>(mm)) - 1;
    mm >>= tz;
    e += tz;
    int q0 = e >> 5, r = e & 31;
    unsigned __int128 w = static_cast<unsigned __int128>(mm) << r;
    int64_t p0 = static_cast<int64_t>(static_cast<uint32_t>(w));
    int64_t p1 = static_cast<int64_t>(static_cast<uint32_t>(w >> 32));
    int64_t p2 = static_cast<int64_t>(static_cast<uint32_t>(w >> 64));
#pragma unroll
    for (int q = 0; q < K; ++q)
      mag[q] -= (q == q0 ? p0 : 0) + (q == q0 + 1 ? p1 : 0) + (q == q0 + 2 ? p2 : 0);
  }
  int64_t carry = 0;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    int64_t v = mag[q] + carry;
    carry = v >> 32;
    mag[q] = v - (carry << 32);
  }
  if (carry >= 0) return false;
  int64_t c = 1;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    int64_t v = (0xffffffffll - mag[q]) + c;
    c = v >> 32;
    mag[q] = v & 0xffffffffll;
  }
  return true;
}

// p_t * floor(2^31 / p_t): added to a residue product g (|g| < 2^31 -
// 2^14 for k <= 131071) it makes g nonnegative and below 2^32 without
// changing g mod p_t, so one Barrett step reduces it
__constant__ unsigned kGBias[54] = {
#define MPMM_GB(p) (p) * (2147483648u / (p))
    MPMM_GB(256), MPMM_GB(251), MPMM_GB(243), MPMM_GB(241), MPMM_GB(239), MPMM_GB(233),
    MPMM_GB(229), MPMM_GB(227), MPMM_GB(223), MPMM_GB(211), MPMM_GB(199), MPMM_GB(197),
    MPMM_GB(193), MPMM_GB(191), MPMM_GB(181), MPMM_GB(179), MPMM_GB(173), MPMM_GB(169),
    MPMM_GB(167), MPMM_GB(163), MPMM_GB(157), MPMM_GB(151), MPMM_GB(149), MPMM_GB(139),
    MPMM_GB(137), MPMM_GB(131), MPMM_GB(127), MPMM_GB(125), MPMM_GB(121), MPMM_GB(113),
    MPMM_GB(109), MPMM_GB(107), MPMM_GB(103), MPMM_GB(101), MPMM_GB(97),  MPMM_GB(89),
    MPMM_GB(83),  MPMM_GB(79),  MPMM_GB(73),  MPMM_GB(71),  MPMM_GB(67),  MPMM_GB(61),
    MPMM_GB(59),  MPMM_GB(53),  MPMM_GB(49),  MPMM_GB(47),  MPMM_GB(43),  MPMM_GB(41),
    MPMM_GB(37),  MPMM_GB(31),  MPMM_GB(29),  MPMM_GB(23),  MPMM_GB(19),  MPMM_GB(17)};
#undef MPMM_GB

// CRT table row layout in shared memory (32-bit words): the low KD limbs
// of W_t as doubles (padded to an even count), then the other K - KD limbs
// as uint32 (padded to 4): every row is a whole number of 16-byte vectors.
// All limbs on the FP64 pipe measured best (DD 1024^3 combine: 101 us; 111
// with half the limbs as integer multiply-adds, 114 with all of them).
__host__ __device__ constexpr int kd_limbs(int K) { return K; }
__host__ __device__ constexpr int kd_even(int K) { return (kd_limbs(K) + 1) / 2 * 2; }
__host__ __device__ constexpr int ki_pad(int K) { return (K - kd_limbs(K) + 3) / 4 * 4; }
__host__ __device__ constexpr int row_words(int K) { return 2 * kd_even(K) + ki_pad(K); }
__host__ __device__ constexpr int pwords(int K) { return (K + 3) / 4 * 4; }

// CRT accumulation of one output: acc[q] = sum_t r_t W_t[q] with
// r_t = G_t mod p_t, in K+1 64-bit limb sums.  The low KD limbs run on
// the FP64 pipe -- r_t W_t[q] < 2^40 and sums over <= 54 moduli < 2^46
// are exact in binary64 -- and any others as 32x32->64-bit integer
// multiply-adds.  The G planes are read 8 at
// a time (eight loads in flight).
// address of element e of a residue plane of either representation
template <bool RES8>
__device__ __forceinline__ const void* elem_ptr(const void* base, int64_t e) {
  return RES8 ? static_cast<const void*>(static_cast<const uint8_t*>(base) + e)
              : static_cast<const void*>(static_cast<const int32_t*>(base) + e);
}

// RES8: the planes already hold r_t = G_t mod p_t as bytes (the tcgen05
// residue GEMM reduces in its epilogue); otherwise int32 G_t, reduced here.
// SM: the residue bytes were staged in shared memory (plain loads).
template <int K, bool RES8, int CH, bool SM = false>
__device__ __forceinline__ void crt_accumulate(const void* Gv, int64_t gplane, int N,
                                               const uint32_t* W, uint64_t (&acc)[K + 1]) {
  constexpr int KD = kd_limbs(K), KE = kd_even(K), RW = row_words(K);
  using RT = typename std::conditional<RES8, uint8_t, int32_t>::type;
  const RT* G = static_cast<const RT*>(Gv);
  double a[KD];
#pragma unroll
  for (int q = 0; q < KD; ++q) a[q] = 0.0;
#pragma unroll
  for (int q = 0; q <= K; ++q) acc[q] = 0;
  for (int t0 = 0; t0 < N; t0 += CH) {
    int g[CH];
    const RT* gp = G + t0 * gplane;
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if constexpr (SM)
        g[u] = t0 + u < N ? static_cast<int>(*gp) : 0;
      else
        g[u] = t0 + u < N ? static_cast<int>(__ldcs(gp)) : 0;
      gp += gplane;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int t = t0 + u;
      if (t >= N) break;
      const unsigned p = static_cast<unsigned>(kModsDev[t]);
      const unsigned r = RES8 ? static_cast<unsigned>(g[u])
                              : barrett(static_cast<unsigned>(g[u]) + kGBias[t], kModMu[t], p);
      // r < 2^32 as a double without the XU conversion (I2F.F64 was the
      // kernel's top stall): (2^52 + r) from its bit pattern, minus 2^52,
      // one exact DADD on the FP64 pipe
      const double rd = __hiloint2double(0x43300000, static_cast<int>(r)) - 4503599627370496.0;
      const uint32_t* row = W + t * RW;
      const double2* wd = reinterpret_cast<const double2*>(row);
#pragma unroll
      for (int q2 = 0; q2 < KE / 2; ++q2) {
        const double2 v = wd[q2];
        if (2 * q2 < KD) a[2 * q2] = __fma_rn(rd, v.x, a[2 * q2]);
        if (2 * q2 + 1 < KD) a[2 * q2 + 1] = __fma_rn(rd, v.y, a[2 * q2 + 1]);
      }
      const uint4* wi = reinterpret_cast<const uint4*>(row + 2 * KE);
#pragma unroll
      for (int q4 = 0; q4 < ki_pad(K) / 4; ++q4) {
        const uint4 v = wi[q4];
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (KD + 4 * q4 + e < K) acc[KD + 4 * q4 + e] += static_cast<uint64_t>(r) * w4[e];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < KD; ++q) acc[q] = static_cast<uint64_t>(a[q]);
}

// Multi-limb add/subtract on the carry flag (separate asm volatile
// statements keep their order; nothing between them writes CC).
__device__ __forceinline__ uint32_t add_cc(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t addc_cc(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t sub_cc(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t subc_cc(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t subc(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("subc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// d = a - b over N limbs; returns the borrow out (1 when a < b)
template <int N>
__device__ __forceinline__ uint32_t sub_limbs(uint32_t (&d)[N], const uint32_t (&a)[N],
                                              const uint32_t* b) {
  d[0] = sub_cc(a[0], b[0]);
#pragma unroll
  for (int q = 1; q < N; ++q) d[q] = subc_cc(a[q], b[q]);
  return subc(0u, 0u) & 1u;
}

// Staged CRT table head (32-bit words): P (PW), P/2 (PW), 1/P as a double
// (+2 pad); the weight rows follow.
__host__ __device__ constexpr int table_head(int K) { return 2 * pwords(K) + 4; }

// From the accumulated sums: the centred integer X = (sum mod P) as sign +
// K magnitude limbs.  T: staged table head.  S < N 256 P < 2^14 P, so the
// quotient from the top limbs times 1/P is off by at most one, fixed by
// one conditional add or subtract of P.
template <int K>
__device__ __forceinline__ bool crt_finish(const uint64_t (&acc)[K + 1], const uint32_t* T,
                                           int64_t (&mag)[K]) {
  constexpr int PW = pwords(K);
  const uint32_t* P = T;
  const uint32_t* Ph = T + PW;
  const double invP = *reinterpret_cast<const double*>(T + 2 * PW);
  uint32_t S[K + 1];
  uint64_t carry = 0;
#pragma unroll
  for (int q = 0; q <= K; ++q) {
    const uint64_t v = acc[q] + carry;
    S[q] = static_cast<uint32_t>(v);
    carry = v >> 32;
  }
  double sd = 0.0, sc = 1.0;
#pragma unroll
  for (int q = 0; q <= K; ++q) {
    if (q >= K - 2) sd += static_cast<double>(S[q]) * sc;   // top three limbs
    sc *= 4294967296.0;
  }
  const uint32_t qv = static_cast<uint32_t>(sd * invP);
  uint32_t L[K + 1];                 // qv * P
  uint64_t t = 0;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    t = static_cast<uint64_t>(qv) * P[q] + (t >> 32);
    L[q] = static_cast<uint32_t>(t);
  }
  L[K] = static_cast<uint32_t>(t >> 32);
  uint32_t X[K + 1];
  const uint32_t neg0 = sub_limbs<K + 1>(X, S, L);   // X = S - qv P, maybe negative
  uint32_t Pl[K + 1];
#pragma unroll
  for (int q = 0; q < K; ++q) Pl[q] = P[q];
  Pl[K] = 0;
  if (neg0) {                        // X += P
    X[0] = add_cc(X[0], Pl[0]);
#pragma unroll
    for (int q = 1; q <= K; ++q) X[q] = addc_cc(X[q], Pl[q]);
  } else {                           // X >= P ? X - P : X
    uint32_t Y[K + 1];
    const uint32_t lt = sub_limbs<K + 1>(Y, X, Pl);
#pragma unroll
    for (int q = 0; q <= K; ++q) X[q] = lt ? X[q] : Y[q];
  }
  // centre: X > P/2 -> -(P - X)
  uint32_t Xk[K], D[K];
#pragma unroll
  for (int q = 0; q < K; ++q) Xk[q] = X[q];
  uint32_t Phl[K];
#pragma unroll
  for (int q = 0; q < K; ++q) Phl[q] = Ph[q];
  const bool upper = sub_limbs<K>(D, Phl, Xk) != 0;   // Ph < X
  if (upper) {
    uint32_t Pk[K];
#pragma unroll
    for (int q = 0; q < K; ++q) Pk[q] = P[q];
    sub_limbs<K>(D, Pk, Xk);
#pragma unroll
    for (int q = 0; q < K; ++q) mag[q] = D[q];
  } else {
#pragma unroll
    for (int q = 0; q < K; ++q) mag[q] = Xk[q];
  }
  return upper;
}

// Shared-memory CRT table of one job: the head (P, P/2, 1/P; table_head)
// then the N weight rows (layout above).
template <int K>
struct StagedTable {
  static constexpr int WORDS = table_head(K) + row_words(K) * kNumMods;   // uint32 words
};

template <int K>
__device__ __forceinline__ void stage_table(const uint32_t* __restrict__ table, int N,
                                            uint32_t* sW) {
  constexpr int PW = pwords(K), RW = row_words(K), KD = kd_limbs(K), KE = kd_even(K);
  constexpr int HEAD = table_head(K);
  for (int q = threadIdx.x; q < PW; q += blockDim.x) {
    sW[q] = q < K ? table[q] : 0u;
    // P/2 (P is even: 256 is always the first modulus)
    const uint32_t lo = q < K ? table[q] : 0u, hi = q + 1 < K ? table[q + 1] : 0u;
    sW[PW + q] = (lo >> 1) | (hi << 31);
  }
  if (threadIdx.x == 0) {
    double pd = 0.0, sc = 1.0;
    for (int q = 0; q < K; ++q) {
      pd += static_cast<double>(table[q]) * sc;
      sc *= 4294967296.0;
    }
    *reinterpret_cast<double*>(sW + 2 * PW) = 1.0 / pd;
  }
  for (int q = threadIdx.x; q < N * RW; q += blockDim.x) {
    const int row = q / RW, col = q % RW;
    uint32_t* dst = sW + HEAD + row * RW;
    const uint32_t* src = table + (row + 1) * K;
    if (col < 2 * KE) {            // double limbs, written as their two halves
      const int d = col / 2;
      const double v = d < KD ? static_cast<double>(src[d]) : 0.0;
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
      dst[col] = static_cast<uint32_t>(col % 2 ? bits >> 32 : bits);
    } else {
      const int li = KD + (col - 2 * KE);
      dst[col] = li < K ? src[li] : 0u;
    }
  }
}

// CRT reconstruction of one job's output from a staged table; CH residue
// planes are loaded at a time (measured: 8 best for the register-heavy
// single-job kernel, 16 for the multi-job one, whose occupancy is bounded
// by its shared-memory window).
template <int K, bool RES8, int CH = 8, bool SM = false>
__device__ __forceinline__ bool crt_reconstruct(const void* Gij, int64_t gplane, int N,
                                                const uint32_t* sW, int64_t (&mag)[K]) {
  uint64_t acc[K + 1];
  crt_accumulate<K, RES8, CH, SM>(Gij, gplane, N, sW + table_head(K), acc);
  return crt_finish<K>(acc, sW, mag);
}

template <int COMPS, int K>
__device__ __forceinline__ void round_out(int64_t (&mag)[K], bool neg, int ebase, double* dst,
                                          bool& bad) {
  double out[COMPS];
#pragma unroll
  for (int c = 0; c < COMPS; ++c) {
    double d = limbs_round<K>(mag, ebase);
    out[c] = neg ? -d : d;
    neg = neg ^ limbs_sub_double<K>(mag, d, ebase);
  }
#pragma unroll
  for (int c = 0; c < COMPS; ++c) {
    dst[c] = out[c];
    bad |= !isfinite(out[c]);
  }
}

// Correctly rounded DD (hi, lo) of sign * mag * 2^ebase from the top 128
// bits of the magnitude plus a sticky bit: hi = RN(x) from the window; the
// remainder x - hi = R 2^E + delta (|R| < 2^76, 0 <= delta < 2^E) is
// rounded again when its integer part keeps >= 55 bits, so the sticky bits
// below the window cannot reach the rounding position.  Returns false
// (use the exact limb path) otherwise -- rare: x - hi cancels to within
// 2^54 ulps of the window's last bit.
template <int K>
__device__ __forceinline__ bool round_dd_fast(const int64_t (&mag)[K], bool neg, int ebase,
                                              double& hi, double& lo) {
  int top = -1;
#pragma unroll
  for (int q = 0; q < K; ++q)
    if (mag[q] != 0) top = q;
  if (top < 0) {
    hi = lo = 0.0;
    return true;
  }
  // limbs top-4 .. top; after normalisation the 128-bit window W holds the
  // top 128 bits of the magnitude exactly (the fifth limb fills the bits
  // the shift frees), everything below is the sticky bit
  uint32_t w[5] = {0, 0, 0, 0, 0};
  bool sticky = false;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const uint32_t v = static_cast<uint32_t>(mag[q]);
#pragma unroll
    for (int u = 0; u < 5; ++u)
      if (q == top - 4 + u) w[u] = v;
    if (q < top - 4) sticky |= v != 0;
  }
  using u128 = unsigned __int128;
  const int lz = __clz(w[4]);
  u128 W = (static_cast<u128>(w[4]) << 96) | (static_cast<u128>(w[3]) << 64) |
           (static_cast<u128>(w[2]) << 32) | w[1];
  if (lz) {
    W = (W << lz) | (w[0] >> (32 - lz));
    sticky |= (w[0] << lz) != 0;
  } else {
    sticky |= w[0] != 0;
  }
  const int E = 32 * (top - 3) - lz + ebase;          // weight of W's bit 0
  const uint64_t t = static_cast<uint64_t>(W >> 64), b = static_cast<uint64_t>(W);
  const double h = __ull2double_rn(t | static_cast<uint64_t>((b != 0) | sticky));
  // R = W - H with H = h at the window's scale (h is an integer in [2^63, 2^64])
  bool rneg;
  u128 Rm;
  if (h == 18446744073709551616.0) {                 // rounded up to 2^64
    rneg = true;
    Rm = (~W) + 1;                                    // 2^128 - W
  } else {
    const u128 H = static_cast<u128>(static_cast<uint64_t>(h)) << 64;
    rneg = H > W;
    Rm = rneg ? H - W : W - H;
  }
  bool st2 = sticky;
  if (rneg && sticky) Rm -= 1;                        // -(|R| - delta): integer part |R| - 1
  if (Rm == 0) {
    if (st2) return false;
    hi = ldexp(neg ? -h : h, E + 64);
    lo = 0.0;
    return true;
  }
  const uint64_t rh = static_cast<uint64_t>(Rm >> 64), rl = static_cast<uint64_t>(Rm);
  const int bl = rh ? 128 - __clzll(static_cast<long long>(rh))
                    : 64 - __clzll(static_cast<long long>(rl));
  if (bl < 55) return false;
  const u128 Mn = Rm << (128 - bl);
  const uint64_t mt = static_cast<uint64_t>(Mn >> 64), mb = static_cast<uint64_t>(Mn);
  const double l = __ull2double_rn(mt | static_cast<uint64_t>((mb != 0) | st2));
  const bool lneg = neg ^ rneg;
  hi = ldexp(neg ? -h : h, E + 64);
  lo = ldexp(lneg ? -l : l, E + bl - 64);
  return true;
}

// single job: one output per thread, weights from shared memory
template <int COMPS, int K, bool RES8>
__global__ void __launch_bounds__(128)
combine_single_kernel(CrtJob jb, int m, int n, double* __restrict__ C, int* __restrict__ status) {
  __shared__ __align__(16) uint32_t sW[StagedTable<K>::WORDS];
  // byte residues of this block's 128 outputs, [plane][128] (staged path)
  __shared__ __align__(16) uint8_t sG[RES8 ? kNumMods * 128 : 16];
  // persistent blocks (grid-stride over 128-output tiles): the table is
  // staged once per block
  stage_table<K>(jb.table, jb.N, sW);
  // Staged path (uniform per launch): the tile's outputs are 128
  // consecutive, 16-byte aligned bytes of every plane, fetched by cp.async
  // all at once (N x 8 16-byte chunks in flight per block instead of 8
  // single-byte loads per thread: the per-thread loads left the kernel
  // latency bound).
  const bool staged = RES8 && blockDim.x == 128 && n % 128 == 0 && jb.gpitch % 16 == 0 &&
                      jb.gplane % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(jb.G) & 15) == 0;
  const int64_t total = static_cast<int64_t>(m) * n;
  for (int64_t e0 = static_cast<int64_t>(blockIdx.x) * blockDim.x; e0 < total;
       e0 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (staged) {
      const int i0 = static_cast<int>(e0 / n), j0 = static_cast<int>(e0 % n);
      const uint8_t* g0 =
          static_cast<const uint8_t*>(jb.G) + static_cast<int64_t>(i0) * jb.gpitch + j0;
      for (int c = threadIdx.x; c < jb.N * 8; c += 128)
        cp_async16(sG + c * 16, g0 + (c >> 3) * jb.gplane + (c & 7) * 16, true);
      cp_async_commit();
      cp_async_wait<0>();
    }
    __syncthreads();
    const int64_t e = e0 + threadIdx.x;
    if (e < total) {
      const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
      int64_t mag[K];
      const bool neg =
          staged ? crt_reconstruct<K, RES8, 8, true>(sG + threadIdx.x, 128, jb.N, sW, mag)
                 : crt_reconstruct<K, RES8>(
                       elem_ptr<RES8>(jb.G, static_cast<int64_t>(i) * jb.gpitch + j),
                       jb.gplane, jb.N, sW, mag);
      bool bad = false;
      const int ebase = -(jb.srow[i] + jb.scol[j]);
      if constexpr (COMPS == 2) {
        double hi, lo;
        if (round_dd_fast<K>(mag, neg, ebase, hi, lo)) {
          C[e * 2] = hi;
          C[e * 2 + 1] = lo;
          bad = !isfinite(hi) || !isfinite(lo);
        } else {
          round_out<COMPS, K>(mag, neg, ebase, C + e * COMPS, bad);
        }
      } else {
        round_out<COMPS, K>(mag, neg, ebase, C + e * COMPS, bad);
      }
      if (bad) atomicOr(status, 1);
    }
    __syncthreads();   // sG is refilled for the next tile
  }
}

// ---------------------------------------------------------------------------
// CRT sums on the tensor cores
//
// The bulk of a CUDA-core combine is S_q = sum_t r_t W_t[q]: N x K
// multiply-adds per output (39 x 9 for DD 1024^3).  Splitting each weight
// limb into its four bytes turns that into an integer matrix product --
// residues (outputs x moduli, u8) times weight bytes (moduli x 4K byte
// columns, u8) -- with int32 sums < 54 * 255^2 < 2^22, exact; then
// S_q = sum_b s_{4q+b} 2^(8b) < 2^48 per limb.  One block of 128 threads
// reconstructs 128 outputs: the residues are staged as rows of sA (moduli
// contiguous, zero above N), each warp runs IMMA.16832.U8.U8 (mma.sync
// m16n8k32) over its 32 outputs x 8*NT columns x 64 moduli, the sums go
// through sC to the thread that owns the output, and crt_finish / rounding
// follow as in the CUDA-core kernels (same integer, same bits).
// ---------------------------------------------------------------------------

template <int K>
struct MmaLayout {
  static constexpr int NT = (4 * K + 7) / 8;   // n-tiles of 8 byte columns
  static constexpr int COLS = 8 * NT;
  static constexpr int AST = 20;               // sA / sWB row stride in words (16 used): the
                                               // fragment loads hit 32 distinct banks
  static constexpr int CST = COLS + 4;         // sC row stride: CST/4 odd, LDS.128 conflict-free
  static constexpr int WB_OFF = 0;
  static constexpr int A_OFF = WB_OFF + COLS * AST * 4;
  static constexpr int C_OFF = A_OFF + 128 * AST * 4;
  static constexpr int S_OFF = C_OFF + 128 * CST * 4;          // [kNumMods][128] staged bytes
  static constexpr int H_OFF = S_OFF + kNumMods * 128;         // P, P/2, 1/P
  static constexpr int BYTES = H_OFF + table_head(K) * 4;
};

__device__ __forceinline__ void mma_u8_16832(int (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                             uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Weight bytes sWB[c][t] (c = 4q + b: byte b of W_t[q]; t contiguous,
// zero for t >= N or q >= K) and the head (P, P/2, 1/P) of one job.
template <int K>
__device__ __forceinline__ void stage_mma_tables(const uint32_t* __restrict__ table, int N,
                                                 uint32_t* sWB, uint32_t* sH) {
  using L = MmaLayout<K>;
  for (int idx = threadIdx.x; idx < L::COLS * 16; idx += blockDim.x) {
    const int c = idx >> 4, w = idx & 15;
    const int q = c >> 2, b = c & 3;
    uint32_t v = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = 4 * w + u;
      const uint32_t byte = (q < K && t < N) ? (table[(t + 1) * K + q] >> (8 * b)) & 0xffu : 0u;
      v |= byte << (8 * u);
    }
    sWB[c * L::AST + w] = v;
  }
  constexpr int PW = pwords(K);
  for (int q = threadIdx.x; q < PW; q += blockDim.x) {
    sH[q] = q < K ? table[q] : 0u;
    const uint32_t lo = q < K ? table[q] : 0u, hi = q + 1 < K ? table[q + 1] : 0u;
    sH[PW + q] = (lo >> 1) | (hi << 31);     // P/2 (P is even)
  }
  if (threadIdx.x == 0) {
    double pd = 0.0, sc = 1.0;
    for (int q = 0; q < K; ++q) {
      pd += static_cast<double>(table[q]) * sc;
      sc *= 4294967296.0;
    }
    *reinterpret_cast<double*>(sH + 2 * PW) = 1.0 / pd;
  }
}

// The staged path's condition (uniform per launch): the block's 128 outputs
// are 128 consecutive, 16-byte aligned bytes of every residue plane.
__device__ __forceinline__ bool mma_staged(const CrtJob& jb, int n) {
  return n % 128 == 0 && jb.gpitch % 16 == 0 && jb.gplane % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(jb.G) & 15) == 0;
}

// cp.async the block's residue bytes [t][128] into the staging area (RES8).
__device__ __forceinline__ void mma_prefetch(const CrtJob& jb, int64_t e0, int n,
                                             unsigned char* stage) {
  const int i0 = static_cast<int>(e0 / n), j0 = static_cast<int>(e0 % n);
  const uint8_t* g0 = static_cast<const uint8_t*>(jb.G) + static_cast<int64_t>(i0) * jb.gpitch + j0;
  for (int c = threadIdx.x; c < jb.N * 8; c += blockDim.x)
    cp_async16(stage + c * 16, g0 + (c >> 3) * jb.gplane + (c & 7) * 16, true);
  cp_async_commit();
}

// Reconstruction of the calling thread's output (o = threadIdx.x of 128;
// element (i, j), valid when in range) for one job whose tables are staged
// in `sm`: (neg, mag) exactly as crt_reconstruct returns them.  STAGED:
// the residue bytes are already in the staging area (mma_prefetch, waited).
// Every thread of the block must call it (warp-synchronous MMAs).
struct MmaBufs {
  const uint32_t* wb;      // the job's weight bytes [COLS][AST]
  const uint32_t* head;    // the job's P, P/2, 1/P
  uint32_t* a;             // [128][AST] residue rows
  int* c;                  // [128][CST] sums
  const unsigned char* stage;   // [kNumMods][128] staged residue bytes (staged path)
};

template <int K>
__device__ __forceinline__ MmaBufs mma_bufs(unsigned char* sm) {
  using L = MmaLayout<K>;
  return MmaBufs{reinterpret_cast<const uint32_t*>(sm + L::WB_OFF),
                 reinterpret_cast<const uint32_t*>(sm + L::H_OFF),
                 reinterpret_cast<uint32_t*>(sm + L::A_OFF), reinterpret_cast<int*>(sm + L::C_OFF),
                 sm + L::S_OFF};
}

template <int K, bool RES8>
__device__ __forceinline__ bool crt_reconstruct_mma(const CrtJob& jb, bool staged, bool valid,
                                                    int i, int j, const MmaBufs& bf,
                                                    int64_t (&mag)[K]) {
  using L = MmaLayout<K>;
  const int o = threadIdx.x, lane = o & 31, warp = o >> 5;
  uint32_t* sA = bf.a;
  // 1. this output's residues r_t (t < 64) as 16 words of sA row o
  {
    uint32_t w[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) w[q] = 0u;
    const int N = jb.N;
    if (staged) {
      const unsigned char* stage = bf.stage;
#pragma unroll
      for (int t = 0; t < kNumMods; ++t)
        if (t < N) w[t >> 2] |= static_cast<uint32_t>(stage[t * 128 + o]) << (8 * (t & 3));
    } else if (valid) {
      const int64_t off = static_cast<int64_t>(i) * jb.gpitch + j;
#pragma unroll
      for (int t = 0; t < kNumMods; ++t) {
        if (t < N) {
          uint32_t r;
          if constexpr (RES8) {
            r = __ldcs(static_cast<const uint8_t*>(jb.G) + t * jb.gplane + off);
          } else {
            const int g = __ldcs(static_cast<const int32_t*>(jb.G) + t * jb.gplane + off);
            r = barrett(static_cast<unsigned>(g) + kGBias[t], kModMu[t],
                        static_cast<unsigned>(kModsDev[t]));
          }
          w[t >> 2] |= r << (8 * (t & 3));
        }
      }
    }
    uint4* row = reinterpret_cast<uint4*>(sA + o * L::AST);
#pragma unroll
    for (int q = 0; q < 4; ++q) row[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  }
  __syncwarp();
  // 2. S = R W on the tensor cores, this warp's 32 outputs
  const uint32_t* sWB = bf.wb;
  int acc[2][L::NT][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < L::NT; ++nt)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[mt][nt][v] = 0;
  const int g = lane >> 2, tg = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    uint32_t b[L::NT][2];
#pragma unroll
    for (int nt = 0; nt < L::NT; ++nt) {
      const uint32_t* col = sWB + (nt * 8 + g) * L::AST + ks * 8 + tg;
      b[nt][0] = col[0];
      b[nt][1] = col[4];
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const uint32_t* r0 = sA + (warp * 32 + mt * 16 + g) * L::AST + ks * 8 + tg;
      const uint32_t a[4] = {r0[0], r0[8 * L::AST], r0[4], r0[8 * L::AST + 4]};
#pragma unroll
      for (int nt = 0; nt < L::NT; ++nt) mma_u8_16832(acc[mt][nt], a, b[nt][0], b[nt][1]);
    }
  }
  // 3. the sums to the owning thread
  int* sC = bf.c;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < L::NT; ++nt) {
      int* c0 = sC + (warp * 32 + mt * 16 + g) * L::CST + nt * 8 + 2 * tg;
      *reinterpret_cast<int2*>(c0) = make_int2(acc[mt][nt][0], acc[mt][nt][1]);
      *reinterpret_cast<int2*>(c0 + 8 * L::CST) = make_int2(acc[mt][nt][2], acc[mt][nt][3]);
    }
  __syncwarp();
  uint64_t S[K + 1];
  {
    const int4* my = reinterpret_cast<const int4*>(sC + o * L::CST);
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const int4 v = my[q];
      S[q] = static_cast<uint64_t>(static_cast<uint32_t>(v.x)) +
             (static_cast<uint64_t>(static_cast<uint32_t>(v.y)) << 8) +
             (static_cast<uint64_t>(static_cast<uint32_t>(v.z)) << 16) +
             (static_cast<uint64_t>(static_cast<uint32_t>(v.w)) << 24);
    }
    S[K] = 0;
  }
  __syncwarp();   // sA / sC rows are rewritten by the next job
  return crt_finish<K>(S, bf.head, mag);
}

template <int COMPS, int K, bool RES8>
__global__ void __launch_bounds__(128)
combine_mma_kernel(CrtJob jb, int m, int n, double* __restrict__ C, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smm[];
  using L = MmaLayout<K>;
  // persistent blocks: the tables are staged once per block, not per tile
  stage_mma_tables<K>(jb.table, jb.N, reinterpret_cast<uint32_t*>(smm + L::WB_OFF),
                      reinterpret_cast<uint32_t*>(smm + L::H_OFF));
  const MmaBufs bf = mma_bufs<K>(smm);
  const bool staged = RES8 && mma_staged(jb, n);
  const int64_t total = static_cast<int64_t>(m) * n;
  const int64_t tiles = (total + 127) / 128;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t e0 = tile * 128;
    if (staged) {
      mma_prefetch(jb, e0, n, smm + L::S_OFF);
      cp_async_wait<0>();
    }
    __syncthreads();
    const int64_t e = e0 + threadIdx.x;
    const bool valid = e < total;
    const int i = valid ? static_cast<int>(e / n) : 0, j = valid ? static_cast<int>(e % n) : 0;
    int64_t mag[K];
    const bool neg = crt_reconstruct_mma<K, RES8>(jb, staged, valid, i, j, bf, mag);
    __syncthreads();   // the staging area is refilled for the next tile
    if (!valid) continue;
    bool bad = false;
    const int ebase = -(jb.srow[i] + jb.scol[j]);
    if constexpr (COMPS == 2) {
      double hi, lo;
      if (round_dd_fast<K>(mag, neg, ebase, hi, lo)) {
        C[e * 2] = hi;
        C[e * 2 + 1] = lo;
        bad = !isfinite(hi) || !isfinite(lo);
      } else {
        round_out<COMPS, K>(mag, neg, ebase, C + e * COMPS, bad);
      }
    } else {
      round_out<COMPS, K>(mag, neg, ebase, C + e * COMPS, bad);
    }
    if (bad) atomicOr(status, 1);
  }
}

// ---------------------------------------------------------------------------
// multi-job combine: per-job CRT in registers, the exact sum in a per-thread
// shared-memory window laid out [digit][thread] (conflict-free for any
// per-thread digit index)
// ---------------------------------------------------------------------------

constexpr int kMTB = 128;     // threads per block
constexpr int kMWin = 28;     // largest window (896 bits); the host passes what a plan needs

// One job's reconstructed value (sign + K magnitude limbs, scaled by
// 2^-(s_i + t_j)) added into the thread's exact window, digits of 32 bits
// relative to 2^ebase; *status |= 2 when it does not fit.
template <int K>
__device__ __forceinline__ void window_add(int64_t* wbuf, int tid, int win, const CrtJob& jb,
                                           int i, int j, int ebase, bool neg,
                                           const int64_t (&mag)[K], int* status) {
#define WIN(q) wbuf[(q) * kMTB + tid]
  const int shift = -(jb.srow[i] + jb.scol[j]) - ebase;
  const int q0 = shift >> 5, r = shift & 31;
  if (q0 + K + 1 > win) atomicOr(status, 2);
#pragma unroll
  for (int p = 0; p < K; ++p) {
    uint64_t v = static_cast<uint64_t>(mag[p]) << r;
    int64_t lo = static_cast<int64_t>(v & 0xffffffffull), hi = static_cast<int64_t>(v >> 32);
    if (neg) {
      lo = -lo;
      hi = -hi;
    }
    if (q0 + p < win) WIN(q0 + p) += lo;
    if (q0 + p + 1 < win) WIN(q0 + p + 1) += hi;
  }
#undef WIN
}

// Normalise the window, round it to COMPS non-overlapping doubles (each the
// round-to-nearest of the remaining magnitude), write them to C[e].
template <int COMPS>
__device__ __forceinline__ void window_round(int64_t* wbuf, int tid, int win, int ebase,
                                             double* __restrict__ C, int64_t e, int* status) {
#define WIN(q) wbuf[(q) * kMTB + tid]
  // Full normalisation once (digits to [0, 2^32), sign out), then per
  // component: round the top 96 bits (+ sticky), subtract the double from
  // the digits it covers and propagate the borrow upward only as far as it
  // goes (the digits below are untouched and stay normalised); a negative
  // remainder is negated over its nonzero span [low, top] only (two's
  // complement leaves the zero digits below `low` zero).
  int64_t carry = 0;
  for (int q = 0; q < win; ++q) {
    const int64_t v = WIN(q) + carry;
    carry = v >> 32;
    WIN(q) = v - (carry << 32);
  }
  auto negate = [&](int lo, int hi) {   // two's complement of digits lo..hi
    int64_t c = 1;
    for (int q = lo; q <= hi; ++q) {
      const int64_t v = (0xffffffffll - WIN(q)) + c;
      c = v >> 32;
      WIN(q) = v & 0xffffffffll;
    }
  };
  bool neg = carry < 0;
  int top = win - 1;
  while (top >= 0 && WIN(top) == 0) --top;
  int low = 0;
  while (low <= top && WIN(low) == 0) ++low;
  if (neg) {                       // the whole window was negative
    negate(low, win - 1);
    top = win - 1;
    while (top >= 0 && WIN(top) == 0) --top;
  }
  double out[COMPS];
  for (int c = 0; c < COMPS; ++c) {
    double d = 0.0;
    if (top >= 0) {
      const uint64_t hi = static_cast<uint64_t>(WIN(top));
      const uint64_t mid = top >= 1 ? static_cast<uint64_t>(WIN(top - 1)) : 0;
      const uint64_t lo = top >= 2 ? static_cast<uint64_t>(WIN(top - 2)) : 0;
      const bool sticky = top - 3 >= low;   // digits [low, top-3]: low is nonzero
      const int lz = __clzll(static_cast<long long>(hi)) - 32;
      unsigned __int128 w = (static_cast<unsigned __int128>(hi) << 64) |
                            (static_cast<unsigned __int128>(mid) << 32) | lo;
      w <<= lz;
      uint64_t top64 = static_cast<uint64_t>(w >> 32);
      if ((static_cast<uint64_t>(w) & 0xffffffffull) != 0 || sticky) top64 |= 1ull;
      d = ldexp(__ull2double_rn(top64), 32 * (top - 2) - lz + 32 + ebase);
    }
    out[c] = neg ? -d : d;
    if (d != 0.0) {   // subtract d (a multiple of 2^ebase) from the magnitude
      const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
      const int be = static_cast<int>((b >> 52) & 0x7ff);
      unsigned long long mm = b & ((1ull << 52) - 1);
      if (be > 0) mm |= (1ull << 52);
      int ee = (be > 0 ? be - 1075 : -1074) - ebase;
      const int tz = __ffsll(static_cast<long long>(mm)) - 1;
      mm >>= tz;
      ee += tz;
      const int q0 = ee >> 5, rr = ee & 31;
      const unsigned __int128 ww = static_cast<unsigned __int128>(mm) << rr;
      for (int u = 0; u < 3; ++u)
        if (q0 + u < win)
          WIN(q0 + u) -= static_cast<int64_t>(static_cast<uint32_t>(ww >> (32 * u)));
      // borrow upward from q0 (d's digits span q0 .. q0 + 2 <= top)
      int64_t br = 0;
      int q = q0;
      for (; q < win; ++q) {
        const int64_t v = WIN(q) + br;
        br = v >> 32;
        WIN(q) = v - (br << 32);
        if (q >= q0 + 2 && br == 0) break;
      }
      if (br < 0) {           // d exceeded the remainder: flip the sign
        neg = !neg;
        negate(low, win - 1);
      }
      if (q0 < low) {         // (not expected: d's lowest bit is above `low`)
        low = q0;
      }
      while (low <= top && WIN(low) == 0) ++low;
      if (low > top) {        // remainder exactly zero
        top = -1;
      } else {
        while (top >= 0 && WIN(top) == 0) --top;
      }
    }
  }
#undef WIN
  bool bad = false;
  for (int c = 0; c < COMPS; ++c) {
    C[e * COMPS + c] = out[c];
    bad |= !isfinite(out[c]);
  }
  if (bad) atomicOr(status, 1);
}

template <int COMPS, int K, bool RES8>
__global__ void __launch_bounds__(kMTB)
combine_multi_kernel(const CrtJobs jobs, int njobs, int win, int m, int n,
                     double* __restrict__ C, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smraw[];
  int64_t* wbuf = reinterpret_cast<int64_t*>(smraw);                  // [win][kMTB]
  uint32_t* tabs = reinterpret_cast<uint32_t*>(wbuf + win * kMTB);    // [njobs][WORDS]
  const int tstride = StagedTable<K>::WORDS;
  for (int J = 0; J < njobs; ++J) stage_table<K>(jobs.j[J].table, jobs.j[J].N, tabs + J * tstride);
  // Staged path (uniform per launch, as in combine_single_kernel): each
  // job's residue bytes for the block's 128 outputs arrive by cp.async into
  // one of two buffers while the previous job is reconstructed.
  uint8_t* sG = reinterpret_cast<uint8_t*>(tabs + njobs * tstride);   // [2][kNumMods][kMTB]
  bool staged = RES8 && n % kMTB == 0;
  for (int J = 0; J < njobs; ++J)
    staged = staged && jobs.j[J].gpitch % 16 == 0 && jobs.j[J].gplane % 16 == 0 &&
             (reinterpret_cast<uintptr_t>(jobs.j[J].G) & 15) == 0;
  __syncthreads();   // tables staged
  // persistent blocks (grid-stride over 128-output tiles): the tables above
  // are staged once per block
  const int64_t total = static_cast<int64_t>(m) * n;
  for (int64_t e0 = static_cast<int64_t>(blockIdx.x) * kMTB; e0 < total;
       e0 += static_cast<int64_t>(gridDim.x) * kMTB) {
    auto prefetch = [&](int J) {
      const CrtJob& jb = jobs.j[J];
      const int i0 = static_cast<int>(e0 / n), j0 = static_cast<int>(e0 % n);
      const uint8_t* g0 =
          static_cast<const uint8_t*>(jb.G) + static_cast<int64_t>(i0) * jb.gpitch + j0;
      uint8_t* dst = sG + (J & 1) * kNumMods * kMTB;
      for (int c = threadIdx.x; c < jb.N * (kMTB / 16); c += kMTB)
        cp_async16(dst + c * 16, g0 + (c / (kMTB / 16)) * jb.gplane + (c % (kMTB / 16)) * 16, true);
      cp_async_commit();
    };
    if (staged) prefetch(0);
    [&]() {
      const int tid = threadIdx.x;
      const int64_t e = e0 + tid;
      if (e >= total) return;   // never taken when staged (n % kMTB == 0)
      const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
    #define WIN(q) wbuf[(q) * kMTB + tid]
      for (int q = 0; q < win; ++q) WIN(q) = 0;
      int ebase = 1 << 30;
      for (int J = 0; J < njobs; ++J) ebase = min(ebase, -(jobs.j[J].srow[i] + jobs.j[J].scol[j]));
      for (int J = 0; J < njobs; ++J) {
        const CrtJob& jb = jobs.j[J];
        int64_t mag[K];
        bool neg;
        if (staged) {
          if (J + 1 < njobs) {
            prefetch(J + 1);
            cp_async_wait<1>();
          } else {
            cp_async_wait<0>();
          }
          __syncthreads();
          neg = crt_reconstruct<K, RES8, 16, true>(sG + (J & 1) * kNumMods * kMTB + tid, kMTB,
                                                   jb.N, tabs + J * tstride, mag);
          __syncthreads();   // buffer J & 1 is refilled by the prefetch of job J + 2
        } else {
          neg = crt_reconstruct<K, RES8, 16>(
              elem_ptr<RES8>(jb.G, static_cast<int64_t>(i) * jb.gpitch + j), jb.gplane, jb.N,
              tabs + J * tstride, mag);
        }
        window_add<K>(wbuf, tid, win, jb, i, j, ebase, neg, mag, status);
      }
    #undef WIN
      window_round<COMPS>(wbuf, tid, win, ebase, C, e, status);
    }();
  }
}


// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

cudaError_t oz_scan_launch(int by_cols, const double* X, int64_t ld, int rows, int cols, int comps,
                           int* EL, int* status, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (by_cols) {
    fill_el_kernel<<<(comps * cols + 255) / 256, 256, 0, s>>>(EL, comps, cols);
    dim3 grid((cols + 31) / 32, (rows + 63) / 64);
    if (comps == 2)
      scan_cols_kernel<2><<<grid, 256, 0, s>>>(X, ld, rows, cols, EL, status);
    else
      scan_cols_kernel<4><<<grid, 256, 0, s>>>(X, ld, rows, cols, EL, status);
  } else {
    const unsigned blocks = static_cast<unsigned>(rows);
    if (comps == 2)
      scan_rows_kernel<2><<<blocks, 32 * kScanWarps, 0, s>>>(X, ld, rows, cols, EL, status);
    else
      scan_rows_kernel<4><<<blocks, 32 * kScanWarps, 0, s>>>(X, ld, rows, cols, EL, status);
  }
  return cudaGetLastError();
}

template <int NC, int W>
static cudaError_t residues_go(int by_cols, const double* X, int64_t ld, int rows, int cols,
                               int comps, int c0, const int* shift, int N, int8_t* R,
                               int64_t rpitch, int64_t rplane, cudaStream_t s) {
  if (by_cols) {
    dim3 grid((cols + 31) / 32, (rows + 31) / 32);
    residues_cols_kernel<NC, W><<<grid, 256, 0, s>>>(X, ld, rows, cols, comps, c0, shift, N, R,
                                                      rpitch, rplane);
  } else {
    const int64_t quads = static_cast<int64_t>(rows) * ((cols + 3) / 4);
    residues_rows_kernel<NC, W><<<(unsigned)((quads + 255) / 256), 256, 0, s>>>(
        X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane);
  }
  return cudaGetLastError();
}

template <int NC>
static cudaError_t residues_w(int W, int by_cols, const double* X, int64_t ld, int rows, int cols,
                              int comps, int c0, const int* shift, int N, int8_t* R,
                              int64_t rpitch, int64_t rplane, cudaStream_t s) {
  // word counts are rounded up to an instantiated width (extra words are 0)
  if (W <= 2) return residues_go<NC, 2>(by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
  if (W <= 3) return residues_go<NC, 3>(by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
  if (W <= 4) return residues_go<NC, 4>(by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
  if (W <= 5) return residues_go<NC, 5>(by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
  if (W <= 6) return residues_go<NC, 6>(by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
  if (W <= 8) return residues_go<NC, 8>(by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
  if (W <= kMaxW) return residues_go<NC, kMaxW>(by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
  return cudaErrorInvalidValue;
}

cudaError_t oz_residues_launch(int by_cols, const double* X, int64_t ld, int rows, int cols,
                               int comps, int c0, int c1, const int* shift, int N, int W,
                               int8_t* R, int64_t rpitch, int64_t rplane, cudaStream_t s) {
  if (static_cast<int64_t>(rows) * cols <= 0) return cudaSuccess;
  if (N < 1 || N > kNumMods || W < 1 || W > kMaxW) return cudaErrorInvalidValue;
  switch (c1 - c0) {
    case 1: return residues_w<1>(W, by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
    case 2: return residues_w<2>(W, by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
    case 4: return residues_w<4>(W, by_cols, X, ld, rows, cols, comps, c0, shift, N, R, rpitch, rplane, s);
    default: return cudaErrorInvalidValue;
  }
}

// MPMM_COMBINE=cuda selects the CUDA-core CRT sums (A/B tests); default:
// the tensor-core sums (combine_mma_kernel).
static bool combine_on_cuda_cores() {
  static const bool v = [] {
    const char* e = std::getenv("MPMM_COMBINE");
    return e != nullptr && std::strcmp(e, "cuda") == 0;
  }();
  return v;
}

template <int COMPS, bool RES8>
static cudaError_t combine_mma(const CrtJob& jb, int m, int n, double* C, int* status,
                               unsigned blocks, cudaStream_t s) {
  switch (jb.K) {
#define MPMM_K(KK)                                                                        \
  case KK: {                                                                              \
    auto kern = combine_mma_kernel<COMPS, KK, RES8>;                                      \
    const int smem = MmaLayout<KK>::BYTES;                                                \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);        \
    int dev = 0, sms = 148, occ = 1;                                                      \
    cudaGetDevice(&dev);                                                                  \
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);                    \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem);                 \
    const unsigned grid = std::min<unsigned>(blocks, (unsigned)(sms * (occ > 0 ? occ : 1))); \
    kern<<<grid, 128, smem, s>>>(jb, m, n, C, status);                                    \
    break;                                                                                \
  }
    MPMM_K(1) MPMM_K(2) MPMM_K(3) MPMM_K(4) MPMM_K(5) MPMM_K(6) MPMM_K(7) MPMM_K(8) MPMM_K(9)
    MPMM_K(10) MPMM_K(11) MPMM_K(12)
#undef MPMM_K
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int COMPS, bool RES8>
static cudaError_t combine_single(const CrtJob& jb, int m, int n, double* C, int* status,
                                  unsigned blocks, cudaStream_t s) {
  // the tensor-core sums for byte residues; int32 products (cuBLASLt planes)
  // keep the CUDA-core kernel, which interleaves their Barrett reductions
  // with the sums (measured faster)
  if (RES8 && !combine_on_cuda_cores())
    return combine_mma<COMPS, RES8>(jb, m, n, C, status, blocks, s);
  switch (jb.K) {
#define MPMM_K(KK) \
  case KK:         \
    {                                                                                    \
      auto kern = combine_single_kernel<COMPS, KK, RES8>;                                \
      int dev = 0, sms = 148, occ = 1;                                                   \
      cudaGetDevice(&dev);                                                               \
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);                 \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0);                 \
      kern<<<std::min<unsigned>(blocks, (unsigned)(sms * (occ > 0 ? occ : 1))), 128, 0, s>>>( \
          jb, m, n, C, status);                                                          \
    }                                                                                    \
    break;
    MPMM_K(1) MPMM_K(2) MPMM_K(3) MPMM_K(4) MPMM_K(5) MPMM_K(6) MPMM_K(7) MPMM_K(8) MPMM_K(9)
    MPMM_K(10) MPMM_K(11) MPMM_K(12)
#undef MPMM_K
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int COMPS, bool RES8>
static cudaError_t combine_multi(const CrtJobs& jobs, int njobs, int K, int win, int m, int n,
                                 double* C, int* status, unsigned blocks, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(win) * kMTB * sizeof(int64_t) +
                      static_cast<size_t>(njobs) * (table_head(K) + row_words(K) * kNumMods) *
                          sizeof(uint32_t) +
                      (RES8 ? 2 * kNumMods * kMTB : 0);
  switch (K) {
#define MPMM_K(KK)                                                                            \
  case KK:                                                                                    \
  {                                                                                           \
    auto kern = combine_multi_kernel<COMPS, KK, RES8>;                                        \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
    int dev = 0, sms = 148, occ = 1;                                                          \
    cudaGetDevice(&dev);                                                                      \
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);                        \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kMTB, smem);                    \
    kern<<<std::min<unsigned>(blocks, (unsigned)(sms * (occ > 0 ? occ : 1))), kMTB, smem, s>>>( \
        jobs, njobs, win, m, n, C, status);                                                   \
  }                                                                                           \
    break;
    MPMM_K(1) MPMM_K(2) MPMM_K(3) MPMM_K(4) MPMM_K(5) MPMM_K(6) MPMM_K(7) MPMM_K(8) MPMM_K(9)
    MPMM_K(10) MPMM_K(11) MPMM_K(12)
#undef MPMM_K
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// jobs: HOST array of njobs CrtJob records (device pointers inside); G of
// each job: int32 residue products, or (res8) bytes already reduced mod p_t
cudaError_t oz_combine_launch(int comps, const void* jobs, int njobs, int m, int n, double* C,
                              int* status, cudaStream_t s, bool res8, int win) {
  win = win < 4 ? 4 : (win > kMWin ? kMWin : win);
  int64_t total = static_cast<int64_t>(m) * n;
  if (total <= 0) return cudaSuccess;
  if (jobs == nullptr || njobs < 1 || njobs > kMaxJobs) return cudaErrorInvalidValue;
  const CrtJob* hj = static_cast<const CrtJob*>(jobs);
  int K = 0;
  for (int q = 0; q < njobs; ++q) K = hj[q].K > K ? hj[q].K : K;
  for (int q = 0; q < njobs; ++q)
    if (hj[q].K != K) return cudaErrorInvalidValue;   // host pads every table to one K
  if (njobs == 1) {
    unsigned blocks = static_cast<unsigned>((total + 127) / 128);
    if (res8)
      return comps == 2 ? combine_single<2, true>(*hj, m, n, C, status, blocks, s)
                        : combine_single<4, true>(*hj, m, n, C, status, blocks, s);
    return comps == 2 ? combine_single<2, false>(*hj, m, n, C, status, blocks, s)
                      : combine_single<4, false>(*hj, m, n, C, status, blocks, s);
  }
  CrtJobs all{};
  for (int q = 0; q < njobs; ++q) all.j[q] = hj[q];
  unsigned blocks = static_cast<unsigned>((total + kMTB - 1) / kMTB);
  if (res8)
    return comps == 2 ? combine_multi<2, true>(all, njobs, K, win, m, n, C, status, blocks, s)
                      : combine_multi<4, true>(all, njobs, K, win, m, n, C, status, blocks, s);
  return comps == 2 ? combine_multi<2, false>(all, njobs, K, win, m, n, C, status, blocks, s)
                    : combine_multi<4, false>(all, njobs, K, win, m, n, C, status, blocks, s);
}

// per-row shifts and the bit width of each component range, from the scan
// arrays (device side of the planner): shift[r][o] = -min L (0 when empty),
// beta[r] = max over o of (max E - min L) + 1 (atomic; zeroed by caller)
struct OzRanges {
  int n;
  int c0[4], c1[4];
};

__global__ void oz_shifts_kernel(OzRanges rg, int comps, int odim, const int* __restrict__ EL,
                                 int* __restrict__ shift, int* __restrict__ beta) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  int d = 0;
  if (o < odim) {
    int e = kEmptyE, lo = kEmptyL;
    for (int c = rg.c0[r]; c < rg.c1[r]; ++c) {
      e = max(e, EL[c * odim + o]);
      lo = min(lo, EL[(comps + c) * odim + o]);
    }
    shift[static_cast<int64_t>(r) * odim + o] = lo == kEmptyL ? 0 : -lo;
    d = e == kEmptyE ? 0 : e - lo + 1;
  }
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) d = max(d, __shfl_xor_sync(0xffffffffu, d, k));
  if ((threadIdx.x & 31) == 0 && d > 0) atomicMax(beta + r, d);
}

cudaError_t oz_shifts_launch(int comps, int nranges, const int* ranges, int odim, const int* EL,
                             int* shift, int* beta, cudaStream_t s) {
  if (odim <= 0) return cudaSuccess;
  if (nranges < 1 || nranges > 4) return cudaErrorInvalidValue;
  OzRanges rg{};
  rg.n = nranges;
  for (int r = 0; r < nranges; ++r) {
    rg.c0[r] = ranges[2 * r];
    rg.c1[r] = ranges[2 * r + 1];
  }
  dim3 grid((odim + 255) / 256, nranges);
  oz_shifts_kernel<<<grid, 256, 0, s>>>(rg, comps, odim, EL, shift, beta);
  return cudaGetLastError();
}

}  // namespace mpmm
