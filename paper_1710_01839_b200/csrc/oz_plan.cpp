// oz_plan.cpp -- host planner of the exact tensor mode (mpmm_oz_plan).
//
// From the per-component scan arrays of A (rows) and B (columns) it picks
// the cheapest feasible way to cut each operand's components into
// contiguous ranges, and for every range the per-row shift and the bit
// width beta of the scaled integers:
//   job (ra, rb) is feasible when prod(p_1..p_N) > 2 l 2^(beta_a + beta_b)
//   for some N <= 54 and both operands fit the residue kernels' 12 words;
//   cost = sum over jobs of N x (limbs + 4)  (int8 GEMMs and CRT work).
// Every plan covers all component pairs, so the sum of its jobs is the
// exact product (tensor.py documents the scheme).  Pure host code: the
// Python planner it replaces cost ~0.1 ms per product.
#include <cstdint>
#include <vector>

namespace mpmm {

namespace {

constexpr int kMods[54] = {256, 251, 243, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191,
                           181, 179, 173, 169, 167, 163, 157, 151, 149, 139, 137, 131, 127, 125,
                           121, 113, 109, 107, 103, 101, 97,  89,  83,  79,  73,  71,  67,  61,
                           59,  53,  49,  47,  43,  41,  37,  31,  29,  23,  19,  17};
constexpr int kEmptyE = -100000, kEmptyL = 100000;
constexpr int kMaxWords = 12;

struct ProdBits {
  int bitlen[55];    // bit length of prod(p_1..p_n)
  bool pow2[55];     // the product is a power of two
  ProdBits() {
    std::vector<uint32_t> P{1};
    bitlen[0] = 1;
    pow2[0] = true;
    for (int n = 1; n <= 54; ++n) {
      uint64_t carry = 0;
      for (auto& w : P) {
        uint64_t v = static_cast<uint64_t>(w) * kMods[n - 1] + carry;
        w = static_cast<uint32_t>(v);
        carry = v >> 32;
      }
      if (carry) P.push_back(static_cast<uint32_t>(carry));
      int top = 31;
      while (top > 0 && !((P.back() >> top) & 1u)) --top;
      bitlen[n] = 32 * (static_cast<int>(P.size()) - 1) + top + 1;
      int ones = 0;
      for (uint32_t w : P) ones += __builtin_popcount(w);
      pow2[n] = ones == 1;
    }
  }
};

const ProdBits& prod_bits() {
  static const ProdBits pb;
  return pb;
}

// smallest N with prod(p_1..p_N) > 2^bits, or 0
int moduli_count(int bits) {
  const ProdBits& pb = prod_bits();
  for (int n = 1; n <= 54; ++n)
    if (pb.bitlen[n] > bits + 1 || (pb.bitlen[n] == bits + 1 && !pb.pow2[n])) return n;
  return 0;
}

struct Range {
  int c0, c1, beta;
  std::vector<int> shift;
};

// EL: E[comps][od] then L[comps][od]
Range range_stats(const int* EL, int comps, int64_t od, int c0, int c1) {
  Range r{c0, c1, 1, std::vector<int>(od)};
  int d = -1;
  for (int64_t o = 0; o < od; ++o) {
    int e = kEmptyE, lo = kEmptyL;
    for (int c = c0; c < c1; ++c) {
      e = e > EL[c * od + o] ? e : EL[c * od + o];
      lo = lo < EL[(comps + c) * od + o] ? lo : EL[(comps + c) * od + o];
    }
    if (e != kEmptyE && e - lo > d) d = e - lo;
    r.shift[o] = lo == kEmptyL ? 0 : -lo;
  }
  r.beta = (d >= 0 ? d + 1 : 1);
  for (int k = c1 - c0 - 1; k > 0; k >>= 1) ++r.beta;   // + bit_length(c1 - c0 - 1)
  return r;
}

std::vector<std::vector<std::pair<int, int>>> partitions(int comps) {
  if (comps == 2) return {{{0, 2}}, {{0, 1}, {1, 2}}};
  return {{{0, 4}}, {{0, 2}, {2, 4}}, {{0, 1}, {1, 2}, {2, 3}, {3, 4}}};
}

}  // namespace

// returns 0 ok, 4 not representable; jobs: max 16 x 8 ints; shift_a /
// shift_b may be null (the device derives the shifts itself)
int oz_plan(int comps, int64_t m, int64_t n, int64_t l, const int* ela, const int* elb,
            int* njobs, int* jobs, int* na, int* ranges_a, int* shift_a, int* nb, int* ranges_b,
            int* shift_b, int* window_digits) {
  int log_l = 1;
  while ((int64_t{1} << log_l) < l) ++log_l;
  const auto parts = partitions(comps);
  std::vector<Range> ra_cache, rb_cache;
  auto get = [&](std::vector<Range>& cache, const int* EL, int64_t od, int c0, int c1) -> int {
    for (size_t q = 0; q < cache.size(); ++q)
      if (cache[q].c0 == c0 && cache[q].c1 == c1) return static_cast<int>(q);
    cache.push_back(range_stats(EL, comps, od, c0, c1));
    return static_cast<int>(cache.size()) - 1;
  };
  int best_pa = -1, best_pb = -1;
  int64_t best_cost = 0;
  for (size_t pa = 0; pa < parts.size(); ++pa)
    for (size_t pb = 0; pb < parts.size(); ++pb) {
      int64_t sumN = 0;
      int K = 0;
      bool ok = true;
      for (auto a : parts[pa]) {
        for (auto b : parts[pb]) {
          const Range& A = ra_cache[get(ra_cache, ela, m, a.first, a.second)];
          const Range& B = rb_cache[get(rb_cache, elb, n, b.first, b.second)];
          const int N = moduli_count(A.beta + B.beta + log_l + 1);
          if (N == 0 || (A.beta + 33) / 32 > kMaxWords || (B.beta + 33) / 32 > kMaxWords) {
            ok = false;
            break;
          }
          sumN += N;
          const int k = (prod_bits().bitlen[N] + 31) / 32;
          K = k > K ? k : K;
        }
        if (!ok) break;
      }
      if (!ok) continue;
      const int64_t cost = sumN * (K + 4);
      if (best_pa < 0 || cost < best_cost) {
        best_pa = static_cast<int>(pa);
        best_pb = static_cast<int>(pb);
        best_cost = cost;
      }
    }
  if (best_pa < 0) return 4;
  // emit: the chosen partitions' ranges and the jobs
  const auto& PA = parts[best_pa];
  const auto& PB = parts[best_pb];
  *na = static_cast<int>(PA.size());
  *nb = static_cast<int>(PB.size());
  int K = 0;
  for (size_t x = 0; x < PA.size(); ++x) {
    const Range& A = ra_cache[get(ra_cache, ela, m, PA[x].first, PA[x].second)];
    ranges_a[2 * x] = A.c0;
    ranges_a[2 * x + 1] = A.c1;
    if (shift_a)
      for (int64_t o = 0; o < m; ++o) shift_a[x * m + o] = A.shift[o];
  }
  for (size_t y = 0; y < PB.size(); ++y) {
    const Range& B = rb_cache[get(rb_cache, elb, n, PB[y].first, PB[y].second)];
    ranges_b[2 * y] = B.c0;
    ranges_b[2 * y + 1] = B.c1;
    if (shift_b)
      for (int64_t o = 0; o < n; ++o) shift_b[y * n + o] = B.shift[o];
  }
  int q = 0;
  for (size_t x = 0; x < PA.size(); ++x)
    for (size_t y = 0; y < PB.size(); ++y, ++q) {
      const Range& A = ra_cache[get(ra_cache, ela, m, PA[x].first, PA[x].second)];
      const Range& B = rb_cache[get(rb_cache, elb, n, PB[y].first, PB[y].second)];
      const int N = moduli_count(A.beta + B.beta + log_l + 1);
      const int k = (prod_bits().bitlen[N] + 31) / 32;
      K = k > K ? k : K;
      int* J = jobs + 8 * q;
      J[0] = static_cast<int>(x);
      J[1] = static_cast<int>(y);
      J[2] = N;
      J[4] = (A.beta + 33) / 32;
      J[5] = (B.beta + 33) / 32;
      J[6] = A.beta;
      J[7] = B.beta;
    }
  for (int j = 0; j < q; ++j) jobs[8 * j + 3] = K;   // one limb count for the whole combine
  *njobs = q;
  if (window_digits) {
    // multi-job combine window: job scales differ by at most the spread of
    // the row shifts across A's ranges plus that across B's ranges; the
    // largest job then needs K + 1 digits above its offset, +1 for carries
    auto spread = [&](std::vector<Range>& cache, const int* EL, int64_t od,
                      const std::vector<std::pair<int, int>>& parts) {
      int sp = 0;
      for (int64_t o = 0; o < od; ++o) {
        int lo = 1 << 30, hi = -(1 << 30);
        for (auto r : parts) {
          const int sh = cache[get(cache, EL, od, r.first, r.second)].shift[o];
          lo = sh < lo ? sh : lo;
          hi = sh > hi ? sh : hi;
        }
        sp = hi - lo > sp ? hi - lo : sp;
      }
      return sp;
    };
    const int bits = spread(ra_cache, ela, m, PA) + spread(rb_cache, elb, n, PB);
    *window_digits = bits / 32 + K + 2;
  }
  return 0;
}

}  // namespace mpmm
