// strassen.cpp -- native Strassen driver behind mpmm_strassen_dev.
//
// The reference's recursion (pkg/src/mpmm/multiply.py:267-338, eq. (3) of
// the paper) evaluated level by level on one stream: per level one batched
// elementwise launch per operand shape for the 10 operand sums of every
// node (multiply.py:313-321), ONE batched blocked-GEMM launch for all 7^d
// leaves (:294-298, from a zero accumulator), then per level, bottom-up, one
// batched launch for the quadrant combinations (:334-337; the 3-op chains
// of C11/C22 fused) and the crops of padded results (:242-260).  Per
// element the operations and their order are exactly the reference's, so
// the result is bit-identical to it for every level grouping.
//
// Memory: a level-synchronous run keeps every level's operand sums and
// products live until the leaves are done, 4.25 s^2 elements per node of
// size s.  When that exceeds the budget (60 % of free device memory, or
// MPMM_STRASSEN_BUDGET_MB), the top levels run depth first -- the seven
// children one after another, each level-synchronous below -- with
// stream-ordered frees, so siblings reuse the same memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "trace.h"
#include "kernels.h"

namespace mpmm {

namespace {

constexpr int64_t kMaxBatch = 65535;
constexpr size_t kEwiseChunk = 16384;  // elementwise problems per upload + launch (as they are planned)
constexpr size_t kFusedChunk = 1024;   // parents per expand + leaf launch of the fused last level

struct View {
  double* p;
  int64_t ld, rows, cols;
};

struct Node {
  View A, B, C;     // operands and the (possibly padded) product target
  // a leaf whose operand sums are folded into its tile loads:
  // left = A + sa*A2, right = B + sb*B2 (sa, sb in {0, +1, -1})
  View A2{}, B2{};
  int sa = 0, sb = 0;
  View Cout;        // where the product finally goes (== C unless padded)
  bool crop = false;
  View P[7];
};

class Driver {
 public:
  Driver(int comps, int64_t cutoff, int tile, cudaStream_t s, int64_t* stats)
      : comps_(comps), cutoff_(cutoff), tile_(tile), s_(s), stats_(stats) {}

  // The EFT-domain words of the top-level operands and the recursion depth
  // (the leaf launches' gate margins).
  cudaError_t scan_top(const View& A, const View& B, int64_t m, int64_t l, int64_t n) {
    depth_ = 0;
    for (int64_t a = m, b = l, c = n; std::min(a, std::min(b, c)) > cutoff_; ++depth_) {
      a = (a + (a & 1)) / 2;
      b = (b + (b & 1)) / 2;
      c = (c + (c & 1)) / 2;
    }
    if (l == 0) return cudaSuccess;
    return domain_scan(comps_, A.p, A.ld, (int)m, (int)l, B.p, B.ld, (int)n, &words_, s_);
  }

  // scratch allocations of the current scope, freed stream-ordered
  // One stream-ordered allocation for all the scratch matrices a level's
  // nodes are about to ask for (`bytes`, an upper bound; alloc() carves it
  // and falls back to its own allocation when the slab runs out).  A level
  // of 7^5 nodes otherwise makes ~50 000 cudaMallocAsync / cudaFreeAsync
  // calls -- ~0.1 s of host time during which the GPU, already through the
  // few launches of the level above, waits for the leaf launches.
  cudaError_t begin_slab(size_t bytes) {
    slab_ = nullptr;
    slab_left_ = 0;
    if (bytes == 0) return cudaSuccess;
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, s_);
    if (e == cudaErrorMemoryAllocation) {
      // no contiguous block of that size: the nodes allocate one by one
      (void)cudaGetLastError();
      return cudaSuccess;
    }
    if (e != cudaSuccess) return e;
    scope_.push_back(p);
    slab_ = static_cast<char*>(p);
    slab_left_ = bytes;
    return cudaSuccess;
  }
  void end_slab() { slab_ = nullptr, slab_left_ = 0; }
  static size_t slab_round(size_t bytes) { return (bytes + 255) & ~static_cast<size_t>(255); }
  size_t matrix_bytes(int64_t rows, int64_t cols) const {
    return slab_round(static_cast<size_t>(rows * cols * comps_) * sizeof(double));
  }

  cudaError_t alloc(int64_t rows, int64_t cols, bool zero, View* v) {
    size_t bytes = static_cast<size_t>(rows * cols * comps_) * sizeof(double);
    void* p = nullptr;
    cudaError_t e = cudaSuccess;
    if (bytes && slab_round(bytes) <= slab_left_) {
      p = slab_;
      slab_ += slab_round(bytes);
      slab_left_ -= slab_round(bytes);
    } else {
      e = cudaMallocAsync(&p, bytes ? bytes : sizeof(double), s_);
      if (e != cudaSuccess) return e;
      scope_.push_back(p);
    }
    if (zero && bytes) {
      if ((e = cudaMemsetAsync(p, 0, bytes, s_)) != cudaSuccess) return e;
    }
    *v = View{static_cast<double*>(p), cols, rows, cols};
    return cudaSuccess;
  }

  View sub(const View& v, int64_t r0, int64_t c0, int64_t rows, int64_t cols) const {
    return View{v.p + comps_ * (r0 * v.ld + c0), v.ld, rows, cols};
  }

  cudaError_t copy(const View& dst, const View& src, int64_t rows, int64_t cols) {
    const size_t el = comps_ * sizeof(double);
    if (rows == 0 || cols == 0) return cudaSuccess;
    return cudaMemcpy2DAsync(dst.p, dst.ld * el, src.p, src.ld * el, cols * el, rows,
                             cudaMemcpyDeviceToDevice, s_);
  }

  // V itself, or a zero-padded rows x cols copy (multiply.py:206-218)
  cudaError_t padded(const View& v, int64_t rows, int64_t cols, View* out) {
    if (v.rows == rows && v.cols == cols) {
      *out = v;
      return cudaSuccess;
    }
    cudaError_t e = alloc(rows, cols, true, out);
    if (e == cudaSuccess) e = copy(*out, v, v.rows, v.cols);
    return e;
  }

  cudaError_t upload(const void* host, size_t bytes, void** dev) {
    cudaError_t e = cudaMallocAsync(dev, bytes ? bytes : 1, s_);
    if (e != cudaSuccess) return e;
    scope_.push_back(*dev);
    return cudaMemcpyAsync(*dev, host, bytes, cudaMemcpyHostToDevice, s_);
  }

  cudaError_t ewise(const std::vector<EwiseProblem>& items, int64_t rows, int64_t cols) {
    if (items.empty() || rows == 0 || cols == 0) return cudaSuccess;
    void* d = nullptr;
    cudaError_t e = upload(items.data(), items.size() * sizeof(EwiseProblem), &d);
    for (size_t q = 0; e == cudaSuccess && q < items.size(); q += kMaxBatch) {
      const int cnt = static_cast<int>(std::min<size_t>(kMaxBatch, items.size() - q));
      e = ewise_batched_launch(comps_, cnt, (int)rows, (int)cols,
                               static_cast<const EwiseProblem*>(d) + q, s_);
    }
    return e;
  }

  // Leaves with folded operand sums: one launch per <= 65535 problems.
  cudaError_t leaves_fused(const std::vector<Node>& nodes, int64_t m, int64_t l, int64_t n) {
    if (nodes.empty() || m == 0 || n == 0) return cudaSuccess;
    std::vector<SumProblem> probs;
    probs.reserve(nodes.size());
    for (const Node& nd : nodes)
      probs.push_back(SumProblem{nd.A.p, nd.sa ? nd.A2.p : nullptr, nd.B.p,
                                 nd.sb ? nd.B2.p : nullptr, nd.C.p, nd.A.ld, nd.B.ld, nd.C.ld,
                                 nd.sa, nd.sb});
    void* d = nullptr;
    cudaError_t e = upload(probs.data(), probs.size() * sizeof(SumProblem), &d);
    for (size_t q = 0; e == cudaSuccess && q < probs.size(); q += kMaxBatch) {
      GemmArgs g{ALGO_BLOCK, tile_, (int)m, (int)n, (int)l, nullptr, 0, nullptr, 0, nullptr, 0,
                 0, nullptr, s_};
      g.batch = static_cast<int>(std::min<size_t>(kMaxBatch, probs.size() - q));
      g.sprobs = static_cast<const SumProblem*>(d) + q;
      g.gate.words = words_;
      g.gate.margin_lo = depth_ > 0 ? 52 : 0;
      g.gate.margin_hi = depth_ > 0 ? depth_ + 1 : 0;
      e = gemm_checked(comps_, g);
    }
    return e;
  }

  cudaError_t leaves(const std::vector<GemmProblem>& probs, int64_t m, int64_t l, int64_t n) {
    if (probs.empty() || m == 0 || n == 0) return cudaSuccess;
    void* d = nullptr;
    cudaError_t e = upload(probs.data(), probs.size() * sizeof(GemmProblem), &d);
    for (size_t q = 0; e == cudaSuccess && q < probs.size(); q += kMaxBatch) {
      GemmArgs g{ALGO_BLOCK, tile_, (int)m, (int)n, (int)l, nullptr, 0, nullptr, 0, nullptr, 0,
                 0, nullptr, s_};
      g.batch = static_cast<int>(std::min<size_t>(kMaxBatch, probs.size() - q));
      g.probs = static_cast<const GemmProblem*>(d) + q;
      // leaf operands are sums of scanned top-level quadrants: the
      // domain gate with the Strassen margins (domain.cuh)
      g.gate.words = words_;
      g.gate.margin_lo = depth_ > 0 ? 52 : 0;
      g.gate.margin_hi = depth_ > 0 ? depth_ + 1 : 0;
      e = gemm_checked(comps_, g);
    }
    return e;
  }

  static EwiseProblem ew(const View& O, const View& X, const View& Y, int sy) {
    EwiseProblem p{};
    p.X = X.p;
    p.Y = Y.p;
    p.O = O.p;
    p.ldx = X.ld;
    p.ldy = Y.ld;
    p.ldo = O.ld;
    p.nops = 1;
    p.sy = sy;
    p.sz = 1;
    p.sw = 1;
    return p;
  }
  static EwiseProblem ew3(const View& O, const View& X, const View& Y, int sy, const View& Z,
                          int sz, const View& W, int sw) {
    EwiseProblem p = ew(O, X, Y, sy);
    p.Z = Z.p;
    p.W = W.p;
    p.ldz = Z.ld;
    p.ldw = W.ld;
    p.nops = 3;
    p.sz = sz;
    p.sw = sw;
    return p;
  }

  // One level of the recursion for `nodes` (all m x l x n): padding, the
  // operand sums, and the children (returned).  multiply.py:300-332.
  // fuse: the children are leaves whose operand sums the leaf launch folds
  // into its tile loads (no sums materialised at this level).
  cudaError_t expand(std::vector<Node>& nodes, int64_t m, int64_t l, int64_t n,
                     std::vector<Node>* children, bool fuse = false) {
    TraceRange trace_("strassen: operand sums (one level)");
    const int64_t me = m + (m & 1), le = l + (l & 1), ne = n + (n & 1);
    const int64_t hm = me / 2, hl = le / 2, hn = ne / 2;
    std::vector<EwiseProblem> sa, sb;
    // the level's scratch in one allocation: per node the seven products and
    // (unless the sums are folded into the leaves) the ten operand sums,
    // plus the padded copies of odd-sized operands and results
    size_t per = matrix_bytes(7 * hm, hn);
    if (!fuse) per += matrix_bytes(5 * hm, hl) + matrix_bytes(5 * hl, hn);
    if (me != m || le != l) per += matrix_bytes(me, le);
    if (le != l || ne != n) per += matrix_bytes(le, ne);
    if (me != m || ne != n) per += matrix_bytes(me, ne);
    cudaError_t e = begin_slab(per * nodes.size());
    if (e != cudaSuccess) return e;
    for (Node& nd : nodes) {
      View Ap, Bp, ta, tb, pt;
      if ((e = padded(nd.A, me, le, &Ap)) != cudaSuccess) return e;
      if ((e = padded(nd.B, le, ne, &Bp)) != cudaSuccess) return e;
      nd.Cout = nd.C;
      if (me != m || ne != n) {
        if ((e = alloc(me, ne, false, &nd.C)) != cudaSuccess) return e;
        nd.crop = true;
      }
      if ((e = alloc(7 * hm, hn, false, &pt)) != cudaSuccess) return e;
      const View a11 = sub(Ap, 0, 0, hm, hl), a12 = sub(Ap, 0, hl, hm, hl);
      const View a21 = sub(Ap, hm, 0, hm, hl), a22 = sub(Ap, hm, hl, hm, hl);
      const View b11 = sub(Bp, 0, 0, hl, hn), b12 = sub(Bp, 0, hn, hl, hn);
      const View b21 = sub(Bp, hl, 0, hl, hn), b22 = sub(Bp, hl, hn, hl, hn);
      for (int q = 0; q < 7; ++q) nd.P[q] = sub(pt, q * hm, 0, hm, hn);
      if (fuse) {
        // the seven products' operands as (first, second, sign) triples, in
        // the reference's order and signs (multiply.py:313-321)
        const View* xa[7] = {&a11, &a21, &a11, &a22, &a11, &a21, &a12};
        const View* ya[7] = {&a22, &a22, nullptr, nullptr, &a12, &a11, &a22};
        const int sga[7] = {1, 1, 0, 0, 1, -1, -1};
        const View* xb[7] = {&b11, &b11, &b12, &b21, &b22, &b11, &b21};
        const View* yb[7] = {&b22, nullptr, &b22, &b11, nullptr, &b12, &b22};
        const int sgb[7] = {1, 0, -1, -1, 0, 1, 1};
        for (int q = 0; q < 7; ++q) {
          Node c;
          c.A = *xa[q];
          c.B = *xb[q];
          c.sa = sga[q];
          c.sb = sgb[q];
          if (ya[q]) c.A2 = *ya[q];
          if (yb[q]) c.B2 = *yb[q];
          c.C = nd.P[q];
          children->push_back(c);
        }
        if (stats_) {
          stats_[0] += 7;
          stats_[1] += 18;
        }
        continue;
      }
      if ((e = alloc(5 * hm, hl, false, &ta)) != cudaSuccess) return e;
      if ((e = alloc(5 * hl, hn, false, &tb)) != cudaSuccess) return e;
      View SA[5], SB[5];
      for (int q = 0; q < 5; ++q) {
        SA[q] = sub(ta, q * hm, 0, hm, hl);
        SB[q] = sub(tb, q * hl, 0, hl, hn);
      }
      // operand sums of multiply.py:313-321, in the reference's order
      sa.push_back(ew(SA[0], a11, a22, 1));
      sa.push_back(ew(SA[1], a21, a22, 1));
      sa.push_back(ew(SA[2], a11, a12, 1));
      sa.push_back(ew(SA[3], a21, a11, -1));
      sa.push_back(ew(SA[4], a12, a22, -1));
      sb.push_back(ew(SB[0], b11, b22, 1));
      sb.push_back(ew(SB[1], b12, b22, -1));
      sb.push_back(ew(SB[2], b21, b11, -1));
      sb.push_back(ew(SB[3], b11, b12, 1));
      sb.push_back(ew(SB[4], b21, b22, 1));
      // launch the sums planned so far (the GPU works while the host plans on)
      if (sa.size() >= kEwiseChunk) {
        if ((e = ewise(sa, hm, hl)) != cudaSuccess) return e;
        if ((e = ewise(sb, hl, hn)) != cudaSuccess) return e;
        sa.clear();
        sb.clear();
      }
      const View xs[7] = {SA[0], SA[1], a11, a22, SA[2], SA[3], SA[4]};
      const View ys[7] = {SB[0], b11, SB[1], SB[2], b22, SB[3], SB[4]};
      for (int q = 0; q < 7; ++q) {
        Node c;
        c.A = xs[q];
        c.B = ys[q];
        c.C = nd.P[q];
        children->push_back(c);
      }
      if (stats_) {
        stats_[0] += 7;
        stats_[1] += 18;
      }
    }
    end_slab();
    if ((e = ewise(sa, hm, hl)) != cudaSuccess) return e;
    return ewise(sb, hl, hn);
  }

  // C quadrants from the seven products (multiply.py:334-337), then the crop
  cudaError_t combine(const std::vector<Node>& nodes, int64_t m, int64_t n) {
    const int64_t hm = (m + (m & 1)) / 2, hn = (n + (n & 1)) / 2;
    std::vector<EwiseProblem> items;
    for (const Node& nd : nodes) {
      const View* P = nd.P;
      items.push_back(ew3(sub(nd.C, 0, 0, hm, hn), P[0], P[3], 1, P[4], -1, P[6], 1));
      items.push_back(ew(sub(nd.C, 0, hn, hm, hn), P[2], P[4], 1));
      items.push_back(ew(sub(nd.C, hm, 0, hm, hn), P[1], P[3], 1));
      items.push_back(ew3(sub(nd.C, hm, hn, hm, hn), P[0], P[2], 1, P[1], -1, P[5], 1));
      if (items.size() >= kEwiseChunk) {
        if (cudaError_t ce = ewise(items, hm, hn); ce != cudaSuccess) return ce;
        items.clear();
      }
    }
    cudaError_t e = ewise(items, hm, hn);
    for (const Node& nd : nodes)
      if (e == cudaSuccess && nd.crop) e = copy(nd.Cout, nd.C, m, n);
    return e;
  }

  // elements a level-synchronous run of an m x l x n product keeps live
  int64_t footprint(int64_t m, int64_t l, int64_t n) const {
    int64_t nodes = 1, total = 0;
    while (std::min(m, std::min(l, n)) > cutoff_) {
      const int64_t me = m + (m & 1), le = l + (l & 1), ne = n + (n & 1);
      const int64_t hm = me / 2, hl = le / 2, hn = ne / 2;
      int64_t per = 5 * hm * hl + 5 * hl * hn + 7 * hm * hn;
      if (me != m || le != l) per += me * le;
      if (le != l || ne != n) per += le * ne;
      if (me != m || ne != n) per += me * ne;
      total += nodes * per;
      nodes *= 7;
      m = hm;
      l = hl;
      n = hn;
    }
    return total * comps_;
  }

  cudaError_t level_sync(const View& A, const View& B, const View& C, int64_t m, int64_t l,
                         int64_t n) {
    std::vector<std::vector<Node>> levels;
    std::vector<int64_t> lm, ln;
    std::vector<Node> nodes(1);
    nodes[0].A = A;
    nodes[0].B = B;
    nodes[0].C = C;
    cudaError_t e = cudaSuccess;
    bool fused = false;
    while (std::min(m, std::min(l, n)) > cutoff_) {
      std::vector<Node> children;
      const int64_t hm = (m + (m & 1)) / 2, hl = (l + (l & 1)) / 2, hn = (n + (n & 1)) / 2;
      // the last expansion folds its operand sums into the leaf launch
      // when the leaves are small enough for that to pay
      fused = std::min(hm, std::min(hl, hn)) <= cutoff_ &&
              (fuse_ == 1 || (fuse_ < 0 && std::max(hm, std::max(hl, hn)) <= kFuseLeafMax));
      if (fused) {
        // The last expansion launches nothing itself (its sums are folded
        // into the leaves), and planning 7^d leaves takes the host tens of
        // milliseconds: expand and launch the parents in chunks, so the GPU
        // starts on the first leaves while the host plans the rest.
        for (size_t lo = 0; lo < nodes.size(); lo += kFusedChunk) {
          const size_t hi = std::min(nodes.size(), lo + kFusedChunk);
          std::vector<Node> part(nodes.begin() + lo, nodes.begin() + hi), kids;
          kids.reserve(7 * part.size());
          if ((e = expand(part, m, l, n, &kids, true)) != cudaSuccess) return e;
          std::copy(part.begin(), part.end(), nodes.begin() + lo);   // P, C, crop
          if ((e = leaves_fused(kids, hm, hl, hn)) != cudaSuccess) return e;
        }
        levels.push_back(std::move(nodes));
        lm.push_back(m);
        ln.push_back(n);
        nodes.clear();
        break;   // the children were leaves
      }
      if ((e = expand(nodes, m, l, n, &children, false)) != cudaSuccess) return e;
      levels.push_back(std::move(nodes));
      lm.push_back(m);
      ln.push_back(n);
      nodes = std::move(children);
      m = (m + (m & 1)) / 2;
      l = (l + (l & 1)) / 2;
      n = (n + (n & 1)) / 2;
    }
    if (!fused) {
      std::vector<GemmProblem> probs;
      probs.reserve(nodes.size());
      for (const Node& nd : nodes)
        probs.push_back(GemmProblem{nd.A.p, nd.B.p, nd.C.p, nd.A.ld, nd.B.ld, nd.C.ld});
      if ((e = leaves(probs, m, l, n)) != cudaSuccess) return e;
    }
    for (size_t d = levels.size(); d-- > 0;)
      if ((e = combine(levels[d], lm[d], ln[d])) != cudaSuccess) return e;
    return cudaSuccess;
  }

  cudaError_t release() {
    cudaError_t e = cudaSuccess;
    for (void* p : scope_) {
      cudaError_t f = cudaFreeAsync(p, s_);
      if (e == cudaSuccess) e = f;
    }
    scope_.clear();
    return e;
  }

  // Depth first while the level-synchronous footprint is over budget.
  cudaError_t solve(const View& A, const View& B, const View& C, int64_t m, int64_t l,
                    int64_t n, int64_t budget) {
    std::vector<void*> outer;
    outer.swap(scope_);
    cudaError_t e;
    if (std::min(m, std::min(l, n)) <= cutoff_ || footprint(m, l, n) <= budget) {
      e = level_sync(A, B, C, m, l, n);
    } else {
      std::vector<Node> nodes(1), children;
      nodes[0].A = A;
      nodes[0].B = B;
      nodes[0].C = C;
      e = expand(nodes, m, l, n, &children);
      const int64_t hm = (m + (m & 1)) / 2, hl = (l + (l & 1)) / 2, hn = (n + (n & 1)) / 2;
      for (size_t q = 0; e == cudaSuccess && q < children.size(); ++q)
        e = solve(children[q].A, children[q].B, children[q].C, hm, hl, hn, budget);
      if (e == cudaSuccess) e = combine(nodes, m, n);
    }
    cudaError_t f = release();
    scope_.swap(outer);
    return e != cudaSuccess ? e : f;
  }

 private:
  int comps_;
  int64_t cutoff_;
  int tile_;
  cudaStream_t s_;
  int64_t* stats_;
  std::vector<void*> scope_;
  const int* words_ = nullptr;
  int depth_ = 0;
  char* slab_ = nullptr;       // the current level's scratch slab (begin_slab)
  size_t slab_left_ = 0;

 public:
  // fold the last level's operand sums into the leaf launch: 1 always,
  // 0 never, -1 (default) for leaves up to kFuseLeafMax.  Measured on the
  // B200 (tools/exp/strassen_fuse_probe.py): 1.6 % faster with 128^3 leaves,
  // 2-3.5 % slower from 256^3 up (the fold re-sums every operand tile once
  // per CTA column -- +2.5 % FP64 work -- against 48 B per summed element
  // of HBM traffic saved)
  int fuse_ = -1;
  static constexpr int64_t kFuseLeafMax = 128;
};

}  // namespace

cudaError_t strassen_run(int comps, int64_t cutoff, int tile, int64_t m, int64_t l, int64_t n,
                         const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int64_t* stats, cudaStream_t stream) {
  if (m == 0 || n == 0) return cudaSuccess;
  // keep freed scratch in the stream-ordered pool across calls: with the
  // default release threshold (0) every synchronize returns it to the
  // driver and the next call re-maps gigabytes of pages
  cudaError_t pe = retain_default_pool();
  if (pe != cudaSuccess) return pe;
  int64_t budget = 0;
  if (const char* env = std::getenv("MPMM_STRASSEN_BUDGET_MB")) {
    budget = std::atoll(env) * (1 << 20) / 8;
  } else {
    size_t free_b = 0, total_b = 0;
    cudaError_t e = cudaMemGetInfo(&free_b, &total_b);
    if (e != cudaSuccess) return e;
    budget = static_cast<int64_t>(free_b / 8 * 6 / 10);
  }
  Driver d(comps, cutoff, tile, stream, stats);
  if (const char* env = std::getenv("MPMM_STRASSEN_FUSE")) d.fuse_ = env[0] == '0' ? 0 : 1;
  View a{const_cast<double*>(A), lda, m, l}, b{const_cast<double*>(B), ldb, l, n}, c{C, ldc, m, n};
  cudaError_t se = d.scan_top(a, b, m, l, n);
  if (se != cudaSuccess) return se;
  return d.solve(a, b, c, m, l, n, budget);
}

}  // namespace mpmm
