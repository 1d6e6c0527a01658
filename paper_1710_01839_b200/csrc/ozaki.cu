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
#include <cstdint>

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
// Lemire fastmod constants ceil(2^64 / p) and 2^32 mod p
__constant__ unsigned long long kModM[54] = {
    0x0100000000000000ull, 0x0105197f7d734042ull, 0x010db20a88f4695aull, 0x010fef010fef0110ull,
    0x0112358e75d30337ull, 0x0119453808ca29c1ull, 0x011e2ef3b3fb8745ull, 0x0120b470c67c0d89ull,
    0x0125e22708092f12ull, 0x013698df3de0747aull, 0x0149539e3b2d066full, 0x014cab88725af6e8ull,
    0x015390948f40feadull, 0x01571ed3c506b39bull, 0x016a13cd15372905ull, 0x016e1f76b4337c6dull,
    0x017ad2208e0ecc36ull, 0x0183c977ab2bedd3ull, 0x01886e5f0abb049aull, 0x01920fb49d0e228eull,
    0x01a16d3f97a4b01bull, 0x01b2036406c80d91ull, 0x01b7d6c3dda338b3ull, 0x01d77b654b82c33aull,
    0x01de5d6e3f8868a5ull, 0x01f44659e4a42716ull, 0x0204081020408103ull, 0x020c49ba5e353f7dull,
    0x021d9ead7cd391fcull, 0x0243f6f0243f6f03ull, 0x02593f69b02593f7ull, 0x02647c69456217edull,
    0x027c45979c952050ull, 0x0288df0cac5b3f5eull, 0x02a3a0fd5c5f02a4ull, 0x02e05c0b81702e06ull,
    0x03159721ed7e7535ull, 0x033d91d2a2067b24ull, 0x0381c0e070381c0full, 0x039b0ad12073615bull,
    0x03d226357e16ece6ull, 0x04325c53ef368eb1ull, 0x0456c797dd49c342ull, 0x04d4873ecade304eull,
    0x05397829cbc14e5full, 0x0572620ae4c415caull, 0x05f417d05f417d06ull, 0x063e7063e7063e71ull,
    0x06eb3e45306eb3e5ull, 0x0842108421084211ull, 0x08d3dcb08d3dcb09ull, 0x0b21642c8590b217ull,
    0x0d79435e50d79436ull, 0x0f0f0f0f0f0f0f10ull};
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

// a mod d for 32-bit a (Lemire, Kaser, Kurz: "Faster remainder by direct
// computation"), M = ceil(2^64 / d)
__device__ __forceinline__ unsigned fastmod(unsigned a, unsigned long long M, unsigned d) {
  unsigned long long low = M * a;
  return static_cast<unsigned>(__umul64hi(low, d));
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

constexpr int kEmptyE = -100000, kEmptyL = 100000;

// one warp per row: E = max top_exp, L = min low_bit over the components
// [c0, c1) of the row's entries
__global__ void scan_rows_kernel(const double* __restrict__ X, int64_t ld, int rows, int cols,
                                 int comps, int c0, int c1, int* __restrict__ E,
                                 int* __restrict__ L) {
  int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (r >= rows) return;
  int e = kEmptyE, lo = kEmptyL;
  for (int k = lane; k < cols; k += 32) {
    const double* p = X + ((int64_t)r * ld + k) * comps;
    for (int c = c0; c < c1; ++c) {
      double v = p[c];
      if (!is_zero(v)) {
        e = max(e, top_exp(v));
        lo = min(lo, low_bit(v));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
  }
  if (lane == 0) {
    E[r] = e;
    L[r] = lo;
  }
}

// columns: a 32-column x 64-row tile per block (coalesced along the row),
// block reduction over the rows, then one atomic per column
__global__ void scan_cols_kernel(const double* __restrict__ X, int64_t ld, int rows, int cols,
                                 int comps, int c0, int c1, int* __restrict__ E,
                                 int* __restrict__ L) {
  __shared__ int se[8][32], sl[8][32];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  int e = kEmptyE, lo = kEmptyL;
  if (j < cols) {
    const int k0 = blockIdx.y * 64;
    for (int k = k0 + ty; k < rows && k < k0 + 64; k += 8) {
      const double* p = X + ((int64_t)k * ld + j) * comps;
      for (int c = c0; c < c1; ++c) {
        double v = p[c];
        if (!is_zero(v)) {
          e = max(e, top_exp(v));
          lo = min(lo, low_bit(v));
        }
      }
    }
  }
  se[ty][tx] = e;
  sl[ty][tx] = lo;
  __syncthreads();
  if (ty == 0 && j < cols) {
    for (int q = 1; q < 8; ++q) {
      e = max(e, se[q][tx]);
      lo = min(lo, sl[q][tx]);
    }
    if (e != kEmptyE) {
      atomicMax(E + j, e);
      atomicMin(L + j, lo);
    }
  }
}

__global__ void fill2_kernel(int* __restrict__ E, int* __restrict__ L, int n) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    E[j] = kEmptyE;
    L[j] = kEmptyL;
  }
}

// Residues of sum_{c < NC} x_{c0+c} 2^shift (an exact integer) modulo the
// first N moduli, centred into int8, for 4 consecutive entries per thread
// (one packed 32-bit store per modulus).  pow2: shared-memory N x xmax
// table of 2^x mod p_t.  All reductions are 32-bit Barrett steps (4
// integer instructions each): a 53-bit mantissa is hi*2^32 + lo, hi < 2^21.
template <int NC>
struct EntryParts {
  unsigned mlo[NC], mhi[NC];
  int ex[NC];
  bool neg[NC], use[NC];

  __device__ __forceinline__ void load(const double* x, int shift, int xmax) {
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double v = x[q];
      use[q] = !is_zero(v);
      unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
      int be = static_cast<int>((b >> 52) & 0x7ff);
      unsigned long long m = b & ((1ull << 52) - 1);
      if (be > 0) m |= (1ull << 52);
      int e = (be > 0 ? be - 1075 : -1074) + shift;
      int tz = use[q] ? __ffsll(static_cast<long long>(m)) - 1 : 0;
      m >>= tz;
      e += tz;                    // >= 0 by the choice of shift (scan_*)
      mlo[q] = static_cast<unsigned>(m);
      mhi[q] = static_cast<unsigned>(m >> 32);
      ex[q] = use[q] ? (e < xmax ? e : xmax - 1) : 0;
      neg[q] = (b >> 63) != 0;
    }
  }

  __device__ __forceinline__ unsigned residue(int t, unsigned p, unsigned mu, unsigned c32,
                                              const uint8_t* pow2, int xmax) const {
    // terms mr * 2^e mod-p factor stay below 2^16; negative terms add
    // p * 2^16 - term, so the sum stays positive and < 2^(17 + log2 NC)
    unsigned acc = 0;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      unsigned mr = barrett(mhi[q] * c32 + barrett(mlo[q], mu, p), mu, p);
      unsigned term = use[q] ? mr * pow2[t * xmax + ex[q]] : 0u;
      acc += neg[q] ? (p << 16) - term : term;
    }
    int r = static_cast<int>(barrett(acc, mu, p));
    if (r >= static_cast<int>((p + 1) / 2)) r -= static_cast<int>(p);   // [-(p-1)/2, p/2)
    return static_cast<unsigned>(r) & 0xffu;
  }
};

__device__ __forceinline__ void load_pow2(const uint8_t* __restrict__ g, uint8_t* s, int n) {
  for (int q = threadIdx.x; q < n; q += blockDim.x) s[q] = g[q];
  __syncthreads();
}

// by_cols 0: A (rows x cols) -> R[t][row][k], k = the column;
// by_cols 1: B (rows=l x cols=n) -> R[t][col][k], k = the row.
// Each thread takes 4 consecutive k of one row/column; the packed int8x4
// stores coalesce along k.  Requires cols (rows) % 4 == 0 (host pads).
template <int NC, int BYCOLS>
__global__ void __launch_bounds__(256)
residues_kernel(const double* __restrict__ X, int64_t ld, int rows, int cols, int comps, int c0,
                const int* __restrict__ shift, int N, const uint8_t* __restrict__ pow2, int xmax,
                int8_t* __restrict__ R, int64_t rpitch, int64_t rplane) {
  extern __shared__ uint8_t spow2[];
  load_pow2(pow2, spow2, N * xmax);
  const int kdim = BYCOLS ? rows : cols;       // the contiguous (k) extent
  const int odim = BYCOLS ? cols : rows;       // rows of R
  const int64_t quads = static_cast<int64_t>(odim) * ((kdim + 3) / 4);
  const int64_t qd = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (qd >= quads) return;
  const int per = (kdim + 3) / 4;
  const int o = static_cast<int>(qd / per), k0 = static_cast<int>(qd % per) * 4;
  const int sh = shift[o];
  EntryParts<NC> ent[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k = k0 + u < kdim ? k0 + u : kdim - 1;
    const double* src = BYCOLS ? X + ((int64_t)k * ld + o) * comps + c0
                               : X + ((int64_t)o * ld + k) * comps + c0;
    ent[u].load(src, sh, xmax);
  }
  const bool full = k0 + 4 <= kdim;
  int8_t* dst = R + static_cast<int64_t>(o) * rpitch + k0;
#pragma unroll 1
  for (int t = 0; t < N; ++t) {
    const unsigned p = static_cast<unsigned>(kModsDev[t]);
    const unsigned mu = kModMu[t];
    const unsigned c32 = kMod2p32[t];
    unsigned word = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) word |= ent[u].residue(t, p, mu, c32, spow2, xmax) << (8 * u);
    if (full) {
      *reinterpret_cast<unsigned*>(dst + t * rplane) = word;
    } else {
      for (int u = 0; k0 + u < kdim; ++u) dst[t * rplane + u] = static_cast<int8_t>(word >> (8 * u));
    }
  }
}

// ---------------------------------------------------------------------------
// CRT reconstruction + exact combination + rounding to DD/QD
// ---------------------------------------------------------------------------

}  // namespace

// Per-job CRT data (device): moduli count, limb count, P limbs, weights.
struct CrtJob {
  const int32_t* G;         // [N][.][gpitch] residue products, plane stride gplane
  const int* srow;          // [m] row shifts
  const int* scol;          // [n] column shifts
  const uint32_t* table;    // [K] P limbs, then [N][K] weight limbs
  int N, K;
  int64_t gpitch, gplane;
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

template <int K>
__device__ __forceinline__ double limbs_double(const uint32_t (&v)[K + 1]) {
  double d = 0.0;
#pragma unroll
  for (int q = 0; q <= K; ++q) d += ldexp(static_cast<double>(v[q]), 32 * q);
  return d;
}

// CRT reconstruction of one job's output (i, j): the centred integer X as
// sign + K magnitude limbs.  sW: P (K limbs) then the N weights (K limbs each).
template <int K>
__device__ __forceinline__ bool crt_reconstruct(const int32_t* __restrict__ Gij, int64_t gplane,
                                                int N, const uint32_t* sW, int64_t (&mag)[K]) {
  const uint32_t* P = sW;
  const uint32_t* W = sW + K;
  uint64_t acc[K + 1];
#pragma unroll
  for (int q = 0; q <= K; ++q) acc[q] = 0;
#pragma unroll 2
  for (int t = 0; t < N; ++t) {
    const unsigned p = static_cast<unsigned>(kModsDev[t]);
    const int g = Gij[t * gplane];
    unsigned r = barrett(static_cast<unsigned>(g), kModMu[t], p);
    if (g < 0) {                 // (g + 2^32) mod p  ->  g mod p
      r = r + p - kMod2p32[t];
      if (r >= p) r -= p;
    }
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] += static_cast<uint64_t>(r) * W[t * K + q];
  }
  uint32_t S[K + 1];
  uint64_t carry = 0;
#pragma unroll
  for (int q = 0; q <= K; ++q) {
    uint64_t v = acc[q] + carry;
    S[q] = static_cast<uint32_t>(v);
    carry = v >> 32;
  }
  uint32_t Pl[K + 1];
#pragma unroll
  for (int q = 0; q < K; ++q) Pl[q] = P[q];
  Pl[K] = 0;
  double qd = floor(limbs_double<K>(S) / limbs_double<K>(Pl));
  const uint64_t qv = qd > 0.0 ? static_cast<uint64_t>(qd) : 0ull;
  int64_t X[K + 1];
  int64_t borrow = 0;
#pragma unroll
  for (int q = 0; q <= K; ++q) {
    uint64_t pq = static_cast<uint64_t>(Pl[q]) * qv;
    int64_t v = static_cast<int64_t>(S[q]) - static_cast<int64_t>(pq & 0xffffffffull) + borrow;
    borrow = (v >> 32) - static_cast<int64_t>(pq >> 32);
    X[q] = v & 0xffffffffll;
  }
  {  // bring X into [0, P): one correction either way
    bool add = borrow < 0;
    bool ge = X[K] != 0;
    if (!add && !ge) {
      bool decided = false;
#pragma unroll
      for (int q = K - 1; q >= 0; --q)
        if (!decided && X[q] != static_cast<int64_t>(Pl[q])) {
          ge = X[q] > static_cast<int64_t>(Pl[q]);
          decided = true;
        }
      if (!decided) ge = true;
    }
    if (add || ge) {
      const int64_t sgn = add ? 1 : -1;
      int64_t c = 0;
#pragma unroll
      for (int q = 0; q <= K; ++q) {
        int64_t v = X[q] + sgn * static_cast<int64_t>(Pl[q]) + c;
        c = v >> 32;
        X[q] = v & 0xffffffffll;
      }
    }
  }
  // centre: X > P/2  ->  -(P - X)
  bool upper = false, decided = false;
#pragma unroll
  for (int q = K - 1; q >= 0; --q) {
    const uint64_t twoq = ((static_cast<uint64_t>(X[q]) << 1) & 0xffffffffull) |
                          (q > 0 ? static_cast<uint64_t>(X[q - 1]) >> 31 : 0ull);
    if (!decided && twoq != Pl[q]) {
      upper = twoq > Pl[q];
      decided = true;
    }
  }
  if ((static_cast<uint64_t>(X[K - 1]) >> 31) != 0 || X[K] != 0) upper = true;
  if (upper) {
    int64_t c = 0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      int64_t v = static_cast<int64_t>(Pl[q]) - X[q] + c;
      c = v >> 32;
      mag[q] = v & 0xffffffffll;
    }
  } else {
#pragma unroll
    for (int q = 0; q < K; ++q) mag[q] = X[q];
  }
  return upper;
}

template <int COMPS, int K>
__global__ void __launch_bounds__(128)
combine_single_kernel(CrtJob jb, int m, int n, double* __restrict__ C, int* __restrict__ status) {
  __shared__ uint32_t sW[(kNumMods + 1) * K];
  for (int q = threadIdx.x; q < (jb.N + 1) * K; q += blockDim.x) sW[q] = jb.table[q];
  __syncthreads();
  int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(m) * n) return;
  const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
  int64_t mag[K];
  bool neg = crt_reconstruct<K>(jb.G + static_cast<int64_t>(i) * jb.gpitch + j, jb.gplane, jb.N,
                                sW, mag);
  const int ebase = -(jb.srow[i] + jb.scol[j]);
  double out[COMPS];
#pragma unroll
  for (int c = 0; c < COMPS; ++c) {
    double d = limbs_round<K>(mag, ebase);
    out[c] = neg ? -d : d;
    neg = neg ^ limbs_sub_double<K>(mag, d, ebase);
  }
  bool bad = false;
#pragma unroll
  for (int c = 0; c < COMPS; ++c) {
    C[e * COMPS + c] = out[c];
    bad |= !isfinite(out[c]);
  }
  if (bad) atomicOr(status, 1);
}

// ---------------------------------------------------------------------------
// multi-job combine: per-job CRT in registers, the exact sum in a per-thread
// shared-memory window laid out [digit][thread] (conflict-free for any
// per-thread digit index)
// ---------------------------------------------------------------------------

constexpr int kMTB = 128;     // threads per block
constexpr int kMWin = 28;     // window digits (896 bits)
constexpr int kMaxJobs = 16;

template <int COMPS, int K>
__global__ void __launch_bounds__(kMTB)
combine_multi_kernel(const CrtJob* __restrict__ jobs, int njobs, int m, int n,
                     double* __restrict__ C, int* __restrict__ status) {
  extern __shared__ unsigned char smraw[];
  int64_t* win = reinterpret_cast<int64_t*>(smraw);                   // [kMWin][kMTB]
  uint32_t* tabs = reinterpret_cast<uint32_t*>(win + kMWin * kMTB);   // [njobs][(55)*K]
  const int tstride = (kNumMods + 1) * K;
  for (int J = 0; J < njobs; ++J)
    for (int q = threadIdx.x; q < (jobs[J].N + 1) * K; q += blockDim.x)
      tabs[J * tstride + q] = jobs[J].table[q];
  __syncthreads();
  const int tid = threadIdx.x;
  int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + tid;
  if (e >= static_cast<int64_t>(m) * n) return;
  const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
#define WIN(q) win[(q) * kMTB + tid]
  for (int q = 0; q < kMWin; ++q) WIN(q) = 0;
  int ebase = 1 << 30;
  for (int J = 0; J < njobs; ++J) ebase = min(ebase, -(jobs[J].srow[i] + jobs[J].scol[j]));
  for (int J = 0; J < njobs; ++J) {
    const CrtJob& jb = jobs[J];
    int64_t mag[K];
    const bool neg = crt_reconstruct<K>(jb.G + static_cast<int64_t>(i) * jb.gpitch + j, jb.gplane,
                                        jb.N, tabs + J * tstride, mag);
    const int shift = -(jb.srow[i] + jb.scol[j]) - ebase;
    const int q0 = shift >> 5, r = shift & 31;
    if (q0 + K + 1 > kMWin) atomicOr(status, 2);
#pragma unroll
    for (int p = 0; p < K; ++p) {
      uint64_t v = static_cast<uint64_t>(mag[p]) << r;
      int64_t lo = static_cast<int64_t>(v & 0xffffffffull), hi = static_cast<int64_t>(v >> 32);
      if (neg) {
        lo = -lo;
        hi = -hi;
      }
      if (q0 + p < kMWin) WIN(q0 + p) += lo;
      if (q0 + p + 1 < kMWin) WIN(q0 + p + 1) += hi;
    }
  }
  auto normalize = [&]() -> bool {
    int64_t carry = 0;
    for (int q = 0; q < kMWin; ++q) {
      int64_t v = WIN(q) + carry;
      carry = v >> 32;
      WIN(q) = v - (carry << 32);
    }
    if (carry >= 0) return false;
    int64_t c = 1;
    for (int q = 0; q < kMWin; ++q) {
      int64_t v = (0xffffffffll - WIN(q)) + c;
      c = v >> 32;
      WIN(q) = v & 0xffffffffll;
    }
    return true;
  };
  bool neg = normalize();
  double out[COMPS];
  for (int c = 0; c < COMPS; ++c) {
    // round-to-nearest of the magnitude
    int top = kMWin - 1;
    while (top >= 0 && WIN(top) == 0) --top;
    double d = 0.0;
    if (top >= 0) {
      uint64_t hi = static_cast<uint64_t>(WIN(top));
      uint64_t mid = top >= 1 ? static_cast<uint64_t>(WIN(top - 1)) : 0;
      uint64_t lo = top >= 2 ? static_cast<uint64_t>(WIN(top - 2)) : 0;
      bool sticky = false;
      for (int q = top - 3; q >= 0; --q) sticky |= (WIN(q) != 0);
      int lz = __clzll(static_cast<long long>(hi)) - 32;
      unsigned __int128 w = (static_cast<unsigned __int128>(hi) << 64) |
                            (static_cast<unsigned __int128>(mid) << 32) | lo;
      w <<= lz;
      uint64_t top64 = static_cast<uint64_t>(w >> 32);
      if ((static_cast<uint64_t>(w) & 0xffffffffull) != 0 || sticky) top64 |= 1ull;
      d = ldexp(__ull2double_rn(top64), 32 * (top - 2) - lz + 32 + ebase);
    }
    out[c] = neg ? -d : d;
    if (d != 0.0) {   // subtract d (a multiple of 2^ebase) from the magnitude
      unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
      int be = static_cast<int>((b >> 52) & 0x7ff);
      unsigned long long mm = b & ((1ull << 52) - 1);
      if (be > 0) mm |= (1ull << 52);
      int ee = (be > 0 ? be - 1075 : -1074) - ebase;
      int tz = __ffsll(static_cast<long long>(mm)) - 1;
      mm >>= tz;
      ee += tz;
      int q0 = ee >> 5, rr = ee & 31;
      unsigned __int128 ww = static_cast<unsigned __int128>(mm) << rr;
      for (int u = 0; u < 3; ++u)
        if (q0 + u < kMWin)
          WIN(q0 + u) -= static_cast<int64_t>(static_cast<uint32_t>(ww >> (32 * u)));
    }
    neg = neg ^ normalize();
  }
#undef WIN
  bool bad = false;
  for (int c = 0; c < COMPS; ++c) {
    C[e * COMPS + c] = out[c];
    bad |= !isfinite(out[c]);
  }
  if (bad) atomicOr(status, 1);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

cudaError_t oz_scan_launch(int by_cols, const double* X, int64_t ld, int rows, int cols, int comps,
                           int c0, int c1, int* E, int* L, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (by_cols) {
    fill2_kernel<<<(cols + 255) / 256, 256, 0, s>>>(E, L, cols);
    dim3 grid((cols + 31) / 32, (rows + 63) / 64);
    scan_cols_kernel<<<grid, 256, 0, s>>>(X, ld, rows, cols, comps, c0, c1, E, L);
  } else {
    int64_t threads = static_cast<int64_t>(rows) * 32;
    scan_rows_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(X, ld, rows, cols, comps,
                                                                       c0, c1, E, L);
  }
  return cudaGetLastError();
}

template <int NC>
static cudaError_t residues_go(int by_cols, const double* X, int64_t ld, int rows, int cols,
                               int comps, int c0, const int* shift, int N, const uint8_t* pow2,
                               int xmax, int8_t* R, int64_t rpitch, int64_t rplane,
                               cudaStream_t s) {
  const int kdim = by_cols ? rows : cols, odim = by_cols ? cols : rows;
  const int64_t quads = static_cast<int64_t>(odim) * ((kdim + 3) / 4);
  const unsigned blocks = static_cast<unsigned>((quads + 255) / 256);
  const size_t smem = static_cast<size_t>(N) * xmax;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (by_cols) {
    cudaFuncSetAttribute(residues_kernel<NC, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    residues_kernel<NC, 1><<<blocks, 256, smem, s>>>(X, ld, rows, cols, comps, c0, shift, N, pow2,
                                                     xmax, R, rpitch, rplane);
  } else {
    cudaFuncSetAttribute(residues_kernel<NC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    residues_kernel<NC, 0><<<blocks, 256, smem, s>>>(X, ld, rows, cols, comps, c0, shift, N, pow2,
                                                     xmax, R, rpitch, rplane);
  }
  return cudaGetLastError();
}

cudaError_t oz_residues_launch(int by_cols, const double* X, int64_t ld, int rows, int cols,
                               int comps, int c0, int c1, const int* shift, int N,
                               const uint8_t* pow2, int xmax, int8_t* R, int64_t rpitch,
                               int64_t rplane, cudaStream_t s) {
  if (static_cast<int64_t>(rows) * cols <= 0) return cudaSuccess;
  if (N < 1 || N > kNumMods) return cudaErrorInvalidValue;
  switch (c1 - c0) {
    case 1: return residues_go<1>(by_cols, X, ld, rows, cols, comps, c0, shift, N, pow2, xmax, R,
                                  rpitch, rplane, s);
    case 2: return residues_go<2>(by_cols, X, ld, rows, cols, comps, c0, shift, N, pow2, xmax, R,
                                  rpitch, rplane, s);
    case 4: return residues_go<4>(by_cols, X, ld, rows, cols, comps, c0, shift, N, pow2, xmax, R,
                                  rpitch, rplane, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int COMPS>
static cudaError_t combine_single(const CrtJob& jb, int m, int n, double* C, int* status,
                                  unsigned blocks, cudaStream_t s) {
  switch (jb.K) {
#define MPMM_K(KK) \
  case KK:         \
    combine_single_kernel<COMPS, KK><<<blocks, 128, 0, s>>>(jb, m, n, C, status); break;
    MPMM_K(1) MPMM_K(2) MPMM_K(3) MPMM_K(4) MPMM_K(5) MPMM_K(6) MPMM_K(7) MPMM_K(8) MPMM_K(9)
    MPMM_K(10) MPMM_K(11) MPMM_K(12)
#undef MPMM_K
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int COMPS>
static cudaError_t combine_multi(const void* jobs, int njobs, int K, int m, int n, double* C,
                                 int* status, unsigned blocks, cudaStream_t s) {
  const CrtJob* J = static_cast<const CrtJob*>(jobs);
  const size_t smem = static_cast<size_t>(kMWin) * kMTB * sizeof(int64_t) +
                      static_cast<size_t>(njobs) * (kNumMods + 1) * K * sizeof(uint32_t);
  switch (K) {
#define MPMM_K(KK)                                                                            \
  case KK:                                                                                    \
    cudaFuncSetAttribute(combine_multi_kernel<COMPS, KK>,                                     \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);             \
    combine_multi_kernel<COMPS, KK><<<blocks, kMTB, smem, s>>>(J, njobs, m, n, C, status);    \
    break;
    MPMM_K(1) MPMM_K(2) MPMM_K(3) MPMM_K(4) MPMM_K(5) MPMM_K(6) MPMM_K(7) MPMM_K(8) MPMM_K(9)
    MPMM_K(10) MPMM_K(11) MPMM_K(12)
#undef MPMM_K
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t oz_combine_launch(int comps, const void* jobs, int njobs, int m, int n, double* C,
                              int* status, cudaStream_t s, const void* host_job) {
  int64_t total = static_cast<int64_t>(m) * n;
  if (total <= 0) return cudaSuccess;
  if (host_job == nullptr || njobs < 1 || njobs > kMaxJobs) return cudaErrorInvalidValue;
  const CrtJob* hj = static_cast<const CrtJob*>(host_job);
  int K = 0;
  for (int q = 0; q < njobs; ++q) K = hj[q].K > K ? hj[q].K : K;
  for (int q = 0; q < njobs; ++q)
    if (hj[q].K != K) return cudaErrorInvalidValue;   // host pads every table to one K
  if (njobs == 1) {
    unsigned blocks = static_cast<unsigned>((total + 127) / 128);
    return comps == 2 ? combine_single<2>(*hj, m, n, C, status, blocks, s)
                      : combine_single<4>(*hj, m, n, C, status, blocks, s);
  }
  unsigned blocks = static_cast<unsigned>((total + kMTB - 1) / kMTB);
  return comps == 2 ? combine_multi<2>(jobs, njobs, K, m, n, C, status, blocks, s)
                    : combine_multi<4>(jobs, njobs, K, m, n, C, status, blocks, s);
}

}  // namespace mpmm
