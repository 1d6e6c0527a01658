// gemm.cuh -- generic DD/QD GEMM kernels for sm_100a (bit-exact mirrors).
//
// C (m x n) = A (m x l) * B (l x n), or C += A*B, for a batch of P
// independent problems of one shape (P = 1 for a plain product; the 7^d
// leaves of a Strassen recursion otherwise).  Matrices are row-major views
// of DD (one double2 per element) or QD (two double2) elements with leading
// dimensions in elements: the reference's AoS layout (matrix.py:20,43-48).
//
// Per output element the k loop runs in ascending order from an
// accumulator that starts at zero (overwrite) or at C (accumulate), and
// every step is the reference's multiply-add (Ops::madd, ddqd.cuh), so each
// element is bit-identical to the reference kernels for ANY tiling, tile
// order or batch grouping: tile shapes are performance knobs only.
//
// Kernels are bound by the FP64 pipe (DD: 50 FP64 instructions per
// multiply-add; QD: ~786).  Operand tiles are staged in shared memory with
// cp.async double buffering; each thread owns a TM x TN register tile.
// Two code paths compute a tile, bit for bit the same: gemm_tile (any shape:
// bounds predicates, zero fill) and gemm_tile_interior (the whole tile
// inside C, l a multiple of the k-tile: no predicates, one barrier per
// k-tile, advanced addresses -- every instruction that is not FP64
// arithmetic costs the FP64 pipe an issue cycle).  On interior QD tiles the
// reference's data-dependent zero-term gates are run speculatively
// (QDSpecOps): recorded, voted once per k-tile, the tile recomputed by the
// gated sequence if a vote fails.
//
// Load balance.  At moderate sizes the tile count is a few waves of 148
// SMs, and the last partial wave costs up to half a wave of idle FP64
// pipes.  gemm_lpt is a persistent kernel (one CTA per resident slot) that
// processes whole-wave batches of big tiles first and splits the remaining
// big tiles into four quarter tiles (largest-processing-time-first), so
// every SM ends within about one quarter tile of the others.
#pragma once

#include <mutex>
#include <type_traits>
#include <unordered_map>

#include "common.cuh"
#include "ddqd.cuh"
#include "kernels.h"

namespace mpmm {

struct DDOps {
  static constexpr int V = 1;     // double2 vectors per element
  static constexpr int NACC = 2;  // accumulator doubles
  __device__ __forceinline__ static void madd(double* acc, const double2* a, const double2* b) {
    dd_madd(acc[0], acc[1], a[0].x, a[0].y, b[0].x, b[0].y);
  }
};

// The opt-in faithful DD sequence (dd_madd_fast); same data layout.
struct DDFastOps {
  static constexpr int V = 1;
  static constexpr int NACC = 2;
  __device__ __forceinline__ static void madd(double* acc, const double2* a, const double2* b) {
    dd_madd_fast(acc[0], acc[1], a[0].x, a[0].y, b[0].x, b[0].y);
  }
};

struct QDOps {
  static constexpr int V = 2;
  static constexpr int NACC = 4;
  __device__ __forceinline__ static void madd(double* acc, const double2* a, const double2* b) {
    const double x[4] = {a[0].x, a[0].y, a[1].x, a[1].y};
    const double y[4] = {b[0].x, b[0].y, b[1].x, b[1].y};
    qd_mul_add(acc, x, y);
  }
};

// QD with the speculative dense multiply-add on interior tiles (ddqd.cuh
// qd_mul_add_spec): `madd_spec` records its gates in a per-thread float
// instead of branching on them; gemm_tile_interior checks it once per
// k-tile and, when a gate may have failed, recomputes the tile with `Exact`.
// Everywhere else (edge tiles, the first k-step of a tile, whose
// accumulator is zero) it is QDOps.
struct QDSpecOps : QDOps {
  using Exact = QDOps;
  __device__ __forceinline__ static void madd_spec(double* acc, const double2* a,
                                                   const double2* b, float& m) {
    const double x[4] = {a[0].x, a[0].y, a[1].x, a[1].y};
    const double y[4] = {b[0].x, b[0].y, b[1].x, b[1].y};
    qd_mul_add_spec(acc, x, y, m);
  }
  // after a gated step: the accumulator's own tests, which madd_spec takes
  // as folded from then on
  __device__ __forceinline__ static void spec_seed(const double* acc, float& m) {
    qd_spec_seed(acc, m);
  }
  // a staged operand chunk: the products' share of the 23-term gate
  __device__ __forceinline__ static void spec_stage(double2 v, float& m) { qd_spec_stage(v, m); }
};

// Ops::madd, or Ops::madd_spec recording its gates in m
template <class Ops, bool SPEC>
struct Madd {
  __device__ __forceinline__ static void run(double* acc, const double2* a, const double2* b,
                                             float&) {
    Ops::madd(acc, a, b);
  }
};
template <class Ops>
struct Madd<Ops, true> {
  __device__ __forceinline__ static void run(double* acc, const double2* a, const double2* b,
                                             float& m) {
    Ops::madd_spec(acc, a, b, m);
  }
};

template <class Ops, class = void>
struct IsSpec : std::false_type {};
template <class Ops>
struct IsSpec<Ops, std::void_t<typename Ops::Exact>> : std::true_type {};

// The reference's sequences with its Dekker TwoProd (_kernels.pyx:19-29),
// for operands outside the DFMA-exact domain (domain.cuh).
struct DDDekkerOps {
  static constexpr int V = 1;
  static constexpr int NACC = 2;
  __device__ __forceinline__ static void madd(double* acc, const double2* a, const double2* b) {
    dd_madd<false, true>(acc[0], acc[1], a[0].x, a[0].y, b[0].x, b[0].y);
  }
};

struct QDDekkerOps {
  static constexpr int V = 2;
  static constexpr int NACC = 4;
  __device__ __forceinline__ static void madd(double* acc, const double2* a, const double2* b) {
    const double x[4] = {a[0].x, a[0].y, a[1].x, a[1].y};
    const double y[4] = {b[0].x, b[0].y, b[1].x, b[1].y};
    qd_mul_add<0, 0, true>(acc, x, y);
  }
};

// Tile t of a tiles_m x tiles_n grid in grouped order: kGroupM tile rows
// at a time, column-major inside the group.  The ~296 CTAs resident at once
// then share ~16 A row panels and ~19 B column panels instead of 1-2 A
// panels and every B panel of a row-major sweep, so B is re-read from HBM
// once per 16 tile rows rather than once per tile row (8192^3 DD: 279 GB
// of DRAM reads per launch row-major, profiles/r02f_dd8192_raw.csv).  The
// order never changes a bit: each output tile is computed independently.
constexpr int kGroupM = kTileGroupM;

__device__ __forceinline__ void grouped_tile(int t, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int span = kGroupM * tiles_n;
  const int first = (t / span) * kGroupM;
  const int rows = min(kGroupM, tiles_m - first);
  const int r = t % span;
  tm = first + r % rows;
  tn = r / rows;
}

// Kernels whose tiles need more than the 48 KB default of dynamic shared
// memory opt in once per device (the attribute is per device: the native
// multi-GPU runtime launches the same kernels on several).
inline cudaError_t allow_smem_impl(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, uint64_t> done;   // kernel -> device bit mask
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lock(mu);
  uint64_t& mask = done[kern];
  if (mask & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) mask |= bit;
  return e;
}

template <class Kern>
inline cudaError_t allow_smem(Kern kern, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return allow_smem_impl(reinterpret_cast<const void*>(kern), bytes);
}

// Problem descriptor (pointers as double2 views, leading dims in elements).
struct Prob {
  const double2* A;
  const double2* B;
  double2* C;
  int64_t lda, ldb, ldc;
};

__device__ __forceinline__ Prob get_prob(const GemmProblem* probs, const Prob& single, int p) {
  if (probs == nullptr) return single;
  const GemmProblem& g = probs[p];
  return Prob{reinterpret_cast<const double2*>(g.A), reinterpret_cast<const double2*>(g.B),
              reinterpret_cast<double2*>(g.C), g.lda, g.ldb, g.ldc};
}

// Shared-memory footprint (in double2) of one BM x BN x BK tile pair.
template <class Ops, int BM, int BN, int BK>
struct TileSmem {
  static constexpr int A_STAGE = BM * (BK + 1) * Ops::V;
  static constexpr int B_STAGE = BK * BN * Ops::V;
  static constexpr int TOTAL = 2 * (A_STAGE + B_STAGE);
};

// Streamed operands: k-panel q (kpanel columns of k) is readable once
// flags[q] != 0; flags[-1] is the launch's status word.  The flags are
// written by the copy stream (a 4-byte copy-engine H2D) after the panel's
// H2D, so a CTA spinning here never waits on another kernel; the operand
// tiles are then read through L2 (cp.async.cg), where the DMA writes land.
//
// Tile mode (panel_k == 0, tile_rows > 0): large products stream A by row
// panels and B by column panels in the order the grouped tile raster
// consumes them; flags[q] for A row panel q (tile_rows rows), then
// flags[a_panels + q] for B column panel q (tile_cols columns).  A CTA waits
// once, before its tile, for the panels its rows and columns lie in.
struct KReady {
  const int* flags;
  int panel_k;
  int tile_rows = 0, tile_cols = 0, a_panels = 0;
};

// bounded wait for flags[q] (see wait_k_panel); called by one thread
__device__ __forceinline__ void spin_flag(const KReady& kr, int q) {
  const volatile int* f = kr.flags + q;
  const volatile int* st = kr.flags - 1;
  const long long t0 = clock64();
  while (*f == 0 && (*st & 4) == 0) {
    __nanosleep(200);
    if (clock64() - t0 > (1ll << 32)) {   // ~2.2 s at 1.965 GHz
      atomicOr(const_cast<int*>(kr.flags) - 1, 4);
      break;
    }
  }
}

__device__ __forceinline__ void wait_tile_panels(const KReady& kr, int m0, int n0, int m, int n,
                                                 int bm, int bn) {
  if (kr.flags == nullptr || kr.panel_k != 0) return;
  if (threadIdx.x == 0) {
    spin_flag(kr, (min(m0 + bm, m) - 1) / kr.tile_rows);
    spin_flag(kr, kr.a_panels + (min(n0 + bn, n) - 1) / kr.tile_cols);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void wait_k_panel(const KReady& kr, int k0, int& seen) {
  if (kr.flags == nullptr || kr.panel_k == 0) return;
  const int q = k0 / kr.panel_k;
  if (q <= seen) return;
  if (threadIdx.x == 0) {
    // bounded: a panel that never lands (a broken copy stream) sets bit 2 of
    // the word before the flags and lets the kernel finish instead of
    // hanging the GPU; the host reports it as an error
    const volatile int* f = kr.flags + q;
    const volatile int* st = kr.flags - 1;
    const long long t0 = clock64();
    // once any CTA has timed out, nobody waits again (one bound per launch)
    while (*f == 0 && (*st & 4) == 0) {
      __nanosleep(200);
      if (clock64() - t0 > (1ll << 32)) {   // ~2.2 s at 1.965 GHz
        atomicOr(const_cast<int*>(kr.flags) - 1, 4);
        break;
      }
    }
    __threadfence();
  }
  __syncthreads();
  seen = q;
}

// One CTA computes the BM x BN output tile at (m0, n0) of problem `pr`.
// NT threads: thread (tx, ty) owns rows ty + r*NTY, cols tx + c*NTX.
// accumulate: the accumulator starts at C's value (read through L2).
template <class Ops, int BM, int BN, int BK, int TM, int TN, int NT>
__device__ __forceinline__ void gemm_tile(const Prob& pr, int m, int n, int l, int accumulate,
                                          int m0, int n0, double2* smem, bool& bad,
                                          const KReady kr = KReady{nullptr, 0}) {
  constexpr int V = Ops::V;
  constexpr int NTX = BN / TN, NTY = BM / TM;
  static_assert(NTX * NTY == NT, "thread tile does not cover the CTA tile");
  using S = TileSmem<Ops, BM, BN, BK>;
  // As[stage][row][k][v], Bs[stage][k][col][v]
  auto As = [&](int st, int r, int k, int v) -> double2& {
    return smem[st * S::A_STAGE + (r * (BK + 1) + k) * V + v];
  };
  auto Bs = [&](int st, int k, int c, int v) -> double2& {
    return smem[2 * S::A_STAGE + st * S::B_STAGE + (k * BN + c) * V + v];
  };
  const int tid = threadIdx.x;
  const int tx = tid % NTX, ty = tid / NTX;

  double acc[TM][TN][Ops::NACC];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      int i = m0 + ty + r * NTY, j = n0 + tx + c * NTX;
      bool load = accumulate && i < m && j < n;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        double2 x = load ? __ldcg(pr.C + ((int64_t)i * pr.ldc + j) * V + v)
                         : make_double2(0.0, 0.0);
        acc[r][c][2 * v] = x.x;
        acc[r][c][2 * v + 1] = x.y;
      }
    }

  const int ktiles = (l + BK - 1) / BK;
  auto load = [&](int kt, int st) {
    const int k0 = kt * BK;
#pragma unroll
    for (int e = tid; e < BM * BK * V; e += NT) {
      int v = e % V, el = e / V;
      int row = el / BK, col = el % BK;
      int gi = m0 + row, gk = k0 + col;
      bool ok = gi < m && gk < l;
      const double2* src = ok ? pr.A + ((int64_t)gi * pr.lda + gk) * V + v : pr.A;
      cp_async16(&As(st, row, col, v), src, ok);
    }
#pragma unroll
    for (int e = tid; e < BK * BN * V; e += NT) {
      int v = e % V, el = e / V;
      int row = el / BN, col = el % BN;
      int gk = k0 + row, gj = n0 + col;
      bool ok = gk < l && gj < n;
      const double2* src = ok ? pr.B + ((int64_t)gk * pr.ldb + gj) * V + v : pr.B;
      cp_async16(&Bs(st, row, col, v), src, ok);
    }
  };

  int seen = -1;   // highest k-panel known to have landed (streamed operands)
  wait_tile_panels(kr, m0, n0, m, n, BM, BN);
  if (ktiles > 0) {
    wait_k_panel(kr, 0, seen);
    load(0, 0);
    cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    const int st = kt & 1;
    if (kt + 1 < ktiles) {
      wait_k_panel(kr, (kt + 1) * BK, seen);
      load(kt + 1, st ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int kcount = min(BK, l - kt * BK);
    auto step = [&](int kk) {
      double2 a[TM][V], b[TN][V];
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v) a[r][v] = As(st, ty + r * NTY, kk, v);
#pragma unroll
      for (int c = 0; c < TN; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v) b[c][v] = Bs(st, kk, tx + c * NTX, v);
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) Ops::madd(acc[r][c], a[r], b[c]);
    };
    if (kcount == BK) {
#pragma unroll 2
      for (int kk = 0; kk < BK; ++kk) step(kk);
    } else {
      for (int kk = 0; kk < kcount; ++kk) step(kk);
    }
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      int i = m0 + ty + r * NTY, j = n0 + tx + c * NTX;
      if (i < m && j < n) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          pr.C[((int64_t)i * pr.ldc + j) * V + v] =
              make_double2(acc[r][c][2 * v], acc[r][c][2 * v + 1]);
          bad |= !finite2(acc[r][c][2 * v], acc[r][c][2 * v + 1]);
        }
      }
    }
}

// ---------------------------------------------------------------------------
// Interior tiles (the whole BM x BN tile inside C, l a multiple of BK): the
// same multiply-adds in the same order as gemm_tile, with the instruction
// overhead around them cut down -- the kernel is bound by the FP64 pipe, and
// every LDS / address / loop instruction takes issue and register-file
// cycles from it.  Differences from gemm_tile:
//   * no bounds predicates; the cp.async sources are per-thread pointers
//     advanced once per k-tile, the destinations thread base + immediates;
//   * ONE barrier per k-tile: wait for tile kt (issued a whole k-tile
//     earlier), barrier, issue tile kt+1 into the buffer everybody finished
//     reading before that barrier, compute tile kt;
//   * the k loop steps UNROLL at a time through shared-memory addresses that
//     are advanced, not recomputed; operand fetches are base + immediate.
// ---------------------------------------------------------------------------

#ifndef MPMM_INTERIOR
#define MPMM_INTERIOR 1       // experiments: -DMPMM_INTERIOR=0 (tools/exp/build_variant.py)
#endif
#ifndef MPMM_INTERIOR_UNROLL
#define MPMM_INTERIOR_UNROLL 4
#endif
#ifndef MPMM_INTERIOR_UNROLL_QD
#define MPMM_INTERIOR_UNROLL_QD 1
#endif

// k-steps per trip of the inner loop: the body must stay inside the 32 KB
// instruction cache (a DD multiply-add is ~0.8 KB of code per accumulator,
// a QD one ~20 KB with its exact paths)
template <class Ops>
struct InteriorUnroll {
  static constexpr int value = Ops::V == 1 ? MPMM_INTERIOR_UNROLL : MPMM_INTERIOR_UNROLL_QD;
};

__device__ __forceinline__ void cp_async16_at(uint32_t saddr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
}

__device__ __forceinline__ double2 lds_double2(uint32_t saddr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(saddr));
  return v;
}

// whether gemm_tile_interior's copy mapping covers this configuration
template <class Ops, int BM, int BN, int BK, int NT>
struct InteriorOk {
  static constexpr int V = Ops::V;
  static constexpr bool value = MPMM_INTERIOR != 0 && NT % (BK * V) == 0 && NT % (BN * V) == 0 &&
                                (BM * BK * V) % NT == 0 && (BK * BN * V) % NT == 0 &&
                                BK % InteriorUnroll<Ops>::value == 0;
};

// Returns false when a speculative tile (IsSpec<Ops>) was abandoned: nothing
// was stored, the buffers are free, and the caller recomputes the tile with
// Ops::Exact.  Always true otherwise.
template <class Ops, int BM, int BN, int BK, int TM, int TN, int NT, bool STREAM = false>
__device__ __forceinline__ bool gemm_tile_interior(const Prob& pr, int m, int n, int l,
                                                   int accumulate, int m0, int n0, double2* smem,
                                                   bool& bad, const KReady kr = KReady{nullptr, 0}) {
  constexpr int V = Ops::V;
  constexpr bool SPEC = IsSpec<Ops>::value;
  constexpr int NTX = BN / TN, NTY = BM / TM;
  constexpr int UNROLL = InteriorUnroll<Ops>::value;
  static_assert(NTX * NTY == NT, "thread tile does not cover the CTA tile");
  using S = TileSmem<Ops, BM, BN, BK>;
  constexpr int AROWS = NT / (BK * V);          // A rows covered by one pass of the CTA's copies
  constexpr int BROWS = NT / (BN * V);
  constexpr int ACH = BM / AROWS, BCH = BK / BROWS;   // 16-byte chunks per thread and k-tile
  constexpr uint32_t A_STAGE_B = S::A_STAGE * 16, B_STAGE_B = S::B_STAGE * 16;
  const int tid = threadIdx.x;
  const int tx = tid % NTX, ty = tid / NTX;

  double acc[TM][TN][Ops::NACC];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      const int i = m0 + ty + r * NTY, j = n0 + tx + c * NTX;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        double2 x = accumulate ? __ldcg(pr.C + ((int64_t)i * pr.ldc + j) * V + v)
                               : make_double2(0.0, 0.0);
        acc[r][c][2 * v] = x.x;
        acc[r][c][2 * v + 1] = x.y;
      }
    }

  // copies: thread -> (row, 16-byte column) of the A and B k-tiles
  const int arow = tid / (BK * V), acol = tid % (BK * V);
  const int brow = tid / (BN * V), bcol = tid % (BN * V);
  const double2* asrc = pr.A + (int64_t)(m0 + arow) * pr.lda * V + acol;
  const double2* bsrc = pr.B + ((int64_t)brow * pr.ldb + n0) * V + bcol;
  const int64_t astep = (int64_t)AROWS * pr.lda * V;
  const int64_t bstep = (int64_t)BROWS * pr.ldb * V;
  const int64_t bnext = (int64_t)BK * pr.ldb * V;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const uint32_t adst = sbase + (arow * (BK + 1) * V + acol) * 16;
  const uint32_t bdst = sbase + 2 * A_STAGE_B + (brow * BN * V + bcol) * 16;
  auto load = [&](int st) {
#pragma unroll
    for (int i = 0; i < ACH; ++i)
      cp_async16_at(adst + st * A_STAGE_B + i * (AROWS * (BK + 1) * V * 16), asrc + i * astep);
#pragma unroll
    for (int i = 0; i < BCH; ++i)
      cp_async16_at(bdst + st * B_STAGE_B + i * (BROWS * BN * V * 16), bsrc + i * bstep);
    asrc += BK * V;
    bsrc += bnext;
  };
  // operand fetches: thread base + immediates
  const uint32_t ard = sbase + ty * ((BK + 1) * V * 16);
  const uint32_t brd = sbase + 2 * A_STAGE_B + tx * (V * 16);

  const int ktiles = l / BK;
  int seen = -1;   // highest k-panel known to have landed (streamed operands)
  if constexpr (STREAM) {
    wait_tile_panels(kr, m0, n0, m, n, BM, BN);
    wait_k_panel(kr, 0, seen);
  }
  load(0);
  cp_async_commit();
  float gate_min = 1.0f;   // SPEC: min |high word| over every gate test so far
  for (int kt = 0; kt < ktiles; ++kt) {
    const int st = kt & 1;
    cp_async_wait<0>();
    if constexpr (SPEC) {
      // this thread's own copies of k-tile kt have landed: their limbs'
      // tests, before the vote, so a tile with a zero limb is never started
#pragma unroll
      for (int i = 0; i < ACH; ++i)
        Ops::spec_stage(lds_double2(adst + st * A_STAGE_B + i * (AROWS * (BK + 1) * V * 16)),
                        gate_min);
#pragma unroll
      for (int i = 0; i < BCH; ++i)
        Ops::spec_stage(lds_double2(bdst + st * B_STAGE_B + i * (BROWS * BN * V * 16)),
                        gate_min);
      // the barrier doubles as the vote on the k-tiles computed so far
#ifdef MPMM_SPEC_IGNORE_VOTE   // experiment only: never fall back (wrong on zero terms)
      __syncthreads();
#else
      if (__syncthreads_or(min_hi_is_zero(gate_min))) return false;
#endif
    } else {
      __syncthreads();
    }
    if (kt + 1 < ktiles) {
      if constexpr (STREAM) wait_k_panel(kr, (kt + 1) * BK, seen);
      load(st ^ 1);
      cp_async_commit();
    }
    uint32_t ap = ard + st * A_STAGE_B, bp = brd + st * B_STAGE_B;
    const uint32_t aend = ap + BK * V * 16;
    // one k-step at offset u of the current addresses
    auto step = [&](int u, auto spec) {
      double2 a[TM][V], b[TN][V];
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v)
          a[r][v] = lds_double2(ap + ((r * NTY * (BK + 1) + u) * V + v) * 16);
#pragma unroll
      for (int c = 0; c < TN; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v)
          b[c][v] = lds_double2(bp + ((u * BN + c * NTX) * V + v) * 16);
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c)
          Madd<Ops, decltype(spec)::value>::run(acc[r][c], a[r], b[c], gate_min);
    };
    if constexpr (SPEC) {
      static_assert(BK > UNROLL, "the speculative loop peels its first trip");
      if (kt == 0) {
        // the tile's first k-step meets a zero accumulator (or C's values):
        // that is the gated sequence's business (the whole first trip, so the
        // loop below keeps its trip length)
#pragma unroll 1
        for (int u = 0; u < UNROLL; ++u) {
          step(0, std::false_type{});
          ap += V * 16;
          bp += BN * V * 16;
        }
#pragma unroll
        for (int r = 0; r < TM; ++r)
#pragma unroll
          for (int c = 0; c < TN; ++c) Ops::spec_seed(acc[r][c], gate_min);
      }
    }
#pragma unroll 1
    do {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) step(u, std::integral_constant<bool, SPEC>{});
      ap += UNROLL * V * 16;
      bp += UNROLL * BN * V * 16;
    } while (ap != aend);
  }
  // the buffers are free for the CTA's next tile; SPEC: the last vote
  if constexpr (SPEC) {
    if (__syncthreads_or(min_hi_is_zero(gate_min))) return false;
  } else {
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      const int i = m0 + ty + r * NTY, j = n0 + tx + c * NTX;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        pr.C[((int64_t)i * pr.ldc + j) * V + v] =
            make_double2(acc[r][c][2 * v], acc[r][c][2 * v + 1]);
        bad |= !finite2(acc[r][c][2 * v], acc[r][c][2 * v + 1]);
      }
    }
  return true;
}

// gemm_tile, through the interior path when the tile qualifies (uniform per
// CTA, so the barriers inside never diverge)
template <class Ops, int BM, int BN, int BK, int TM, int TN, int NT, bool STREAM = false>
__device__ __forceinline__ void gemm_tile_any(const Prob& pr, int m, int n, int l, int accumulate,
                                              int m0, int n0, double2* smem, bool& bad,
                                              const KReady kr = KReady{nullptr, 0}) {
  if constexpr (InteriorOk<Ops, BM, BN, BK, NT>::value) {
    if (m0 + BM <= m && n0 + BN <= n && l >= BK && l % BK == 0) {
      if (gemm_tile_interior<Ops, BM, BN, BK, TM, TN, NT, STREAM>(pr, m, n, l, accumulate, m0,
                                                                  n0, smem, bad, kr))
        return;
      if constexpr (IsSpec<Ops>::value) {
        // a gate of the speculative sequence may have failed somewhere in
        // the tile: the exact sequence, from the start (streamed operands:
        // with the same panel waits -- later k-panels may not have landed)
        gemm_tile_interior<typename Ops::Exact, BM, BN, BK, TM, TN, NT, STREAM>(
            pr, m, n, l, accumulate, m0, n0, smem, bad, kr);
      }
      return;
    }
  }
  if constexpr (IsSpec<Ops>::value)
    gemm_tile<typename Ops::Exact, BM, BN, BK, TM, TN, NT>(pr, m, n, l, accumulate, m0, n0, smem,
                                                           bad, kr);
  else
    gemm_tile<Ops, BM, BN, BK, TM, TN, NT>(pr, m, n, l, accumulate, m0, n0, smem, bad, kr);
}

// ---------------------------------------------------------------------------
// Strassen leaves with their operand sums folded into the tile loads
// (multiply.py:313-321): the left operand is X + sa*Y (sa = +-1; 0: X alone)
// and the right one Z + sb*W, each sum the reference's ewise add/sub
// (_kernels.pyx:189-230 DD, :407-452 QD) evaluated per staged element --
// the same bits as the materialised sum, without writing and re-reading it.
// Every thread stages whole elements (all V vectors) of X and Y by
// cp.async, waits for its own copies and forms the sums in place before the
// tile barrier, so the fold adds no barrier.
// ---------------------------------------------------------------------------

struct SumProb {
  const double2* A;
  const double2* A2;
  const double2* B;
  const double2* B2;
  double2* C;
  int64_t lda, ldb, ldc;
  int sa, sb;
};

__device__ __forceinline__ SumProb get_sum_prob(const SumProblem& g) {
  return SumProb{reinterpret_cast<const double2*>(g.A), reinterpret_cast<const double2*>(g.A2),
                 reinterpret_cast<const double2*>(g.B), reinterpret_cast<const double2*>(g.B2),
                 reinterpret_cast<double2*>(g.C), g.lda, g.ldb, g.ldc, g.sa, g.sb};
}

// x <- x + s*y on one staged element (s = +1 / -1): the reference ewise op
template <int V>
__device__ __forceinline__ void fold_sum(double2* x, const double2* y, int s) {
  if constexpr (V == 1) {
    const double yh = s < 0 ? -y[0].x : y[0].x, yl = s < 0 ? -y[0].y : y[0].y;
    double h, lo;
    dd_add(x[0].x, x[0].y, yh, yl, h, lo);
    x[0] = make_double2(h, lo);
  } else {
    const double a[4] = {x[0].x, x[0].y, x[1].x, x[1].y};
    double b[4] = {y[0].x, y[0].y, y[1].x, y[1].y};
    if (s < 0)
      for (int q = 0; q < 4; ++q) b[q] = -b[q];
    double r[4];
    qd_add(a, b, r);
    x[0] = make_double2(r[0], r[1]);
    x[1] = make_double2(r[2], r[3]);
  }
}

template <class Ops, int BM, int BN, int BK>
struct SumSmem {
  using T = TileSmem<Ops, BM, BN, BK>;
  // As, Bs double-buffered, then the Y / W staging of both stages
  static constexpr int TOTAL = 2 * T::TOTAL;
};

template <class Ops, int BM, int BN, int BK, int TM, int TN, int NT>
__device__ __forceinline__ void gemm_tile_sum(const SumProb& pr, int m, int n, int l, int m0,
                                              int n0, double2* smem, bool& bad) {
  constexpr int V = Ops::V;
  constexpr int NTX = BN / TN, NTY = BM / TM;
  static_assert(NTX * NTY == NT, "thread tile does not cover the CTA tile");
  using S = TileSmem<Ops, BM, BN, BK>;
  double2* const Y0 = smem + S::TOTAL;   // staging of the second summands
  auto As = [&](double2* base, int st, int r, int k) -> double2* {
    return base + st * S::A_STAGE + (r * (BK + 1) + k) * V;
  };
  auto Bs = [&](double2* base, int st, int k, int c) -> double2* {
    return base + 2 * S::A_STAGE + st * S::B_STAGE + (k * BN + c) * V;
  };
  const int tid = threadIdx.x;
  const int tx = tid % NTX, ty = tid / NTX;

  double acc[TM][TN][Ops::NACC];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c)
#pragma unroll
      for (int q = 0; q < Ops::NACC; ++q) acc[r][c][q] = 0.0;

  const int ktiles = (l + BK - 1) / BK;
  auto load = [&](int kt, int st) {
    const int k0 = kt * BK;
    for (int el = tid; el < BM * BK; el += NT) {
      const int row = el / BK, col = el % BK;
      const int gi = m0 + row, gk = k0 + col;
      const bool ok = gi < m && gk < l;
      const int64_t off = ((int64_t)gi * pr.lda + gk) * V;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        cp_async16(As(smem, st, row, col) + v, ok ? pr.A + off + v : pr.A, ok);
        if (pr.sa) cp_async16(As(Y0, st, row, col) + v, ok ? pr.A2 + off + v : pr.A2, ok);
      }
    }
    for (int el = tid; el < BK * BN; el += NT) {
      const int row = el / BN, col = el % BN;
      const int gk = k0 + row, gj = n0 + col;
      const bool ok = gk < l && gj < n;
      const int64_t off = ((int64_t)gk * pr.ldb + gj) * V;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        cp_async16(Bs(smem, st, row, col) + v, ok ? pr.B + off + v : pr.B, ok);
        if (pr.sb) cp_async16(Bs(Y0, st, row, col) + v, ok ? pr.B2 + off + v : pr.B2, ok);
      }
    }
  };
  // the sums of this thread's own staged elements (visible to it after
  // its cp.async group completed; the tile barrier publishes them)
  auto fold = [&](int st) {
    if (pr.sa)
      for (int el = tid; el < BM * BK; el += NT) {
        const int row = el / BK, col = el % BK;
        fold_sum<V>(As(smem, st, row, col), As(Y0, st, row, col), pr.sa);
      }
    if (pr.sb)
      for (int el = tid; el < BK * BN; el += NT) {
        const int row = el / BN, col = el % BN;
        fold_sum<V>(Bs(smem, st, row, col), Bs(Y0, st, row, col), pr.sb);
      }
  };

  if (ktiles > 0) {
    load(0, 0);
    cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    const int st = kt & 1;
    if (kt + 1 < ktiles) {
      load(kt + 1, st ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    fold(st);
    __syncthreads();
    const int kcount = min(BK, l - kt * BK);
    auto step = [&](int kk) {
      double2 a[TM][V], b[TN][V];
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int v = 0; v < V; ++v) a[r][v] = As(smem, st, ty + r * NTY, kk)[v];
#pragma unroll
      for (int c = 0; c < TN; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v) b[c][v] = Bs(smem, st, kk, tx + c * NTX)[v];
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) Ops::madd(acc[r][c], a[r], b[c]);
    };
    if (kcount == BK) {
#pragma unroll 2
      for (int kk = 0; kk < BK; ++kk) step(kk);
    } else {
      for (int kk = 0; kk < kcount; ++kk) step(kk);
    }
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      int i = m0 + ty + r * NTY, j = n0 + tx + c * NTX;
      if (i < m && j < n) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          pr.C[((int64_t)i * pr.ldc + j) * V + v] =
              make_double2(acc[r][c][2 * v], acc[r][c][2 * v + 1]);
          bad |= !finite2(acc[r][c][2 * v], acc[r][c][2 * v + 1]);
        }
      }
    }
}

// gemm_tile_sum for interior tiles: the pipeline of gemm_tile_interior (one
// barrier per k-tile, advanced addresses, no predicates) with the operand
// sums formed on each thread's own staged elements before that barrier.
template <class Ops, int BM, int BN, int BK, int NT>
struct SumInteriorOk {
  static constexpr bool value = MPMM_INTERIOR != 0 && NT % BK == 0 && NT % BN == 0 &&
                                (BM * BK) % NT == 0 && (BK * BN) % NT == 0 &&
                                BK % InteriorUnroll<Ops>::value == 0;
};

template <class Ops, int BM, int BN, int BK, int TM, int TN, int NT>
__device__ __forceinline__ void gemm_tile_sum_interior(const SumProb& pr, int l, int m0, int n0,
                                                       double2* smem, bool& bad) {
  constexpr int V = Ops::V;
  constexpr int NTX = BN / TN, NTY = BM / TM;
  constexpr int UNROLL = InteriorUnroll<Ops>::value;
  using S = TileSmem<Ops, BM, BN, BK>;
  constexpr int AROWS = NT / BK, BROWS = NT / BN;       // rows per pass of the CTA's copies
  constexpr int AEL = BM / AROWS, BEL = BK / BROWS;     // elements per thread and k-tile
  constexpr uint32_t A_STAGE_B = S::A_STAGE * 16, B_STAGE_B = S::B_STAGE * 16;
  constexpr uint32_t Y_OFF_B = S::TOTAL * 16;           // staging of the second summands
  const int tid = threadIdx.x;
  const int tx = tid % NTX, ty = tid / NTX;

  double acc[TM][TN][Ops::NACC];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c)
#pragma unroll
      for (int q = 0; q < Ops::NACC; ++q) acc[r][c][q] = 0.0;

  // copies: thread -> (row, element column) of the A and B k-tiles
  const int arow = tid / BK, acol = tid % BK;
  const int brow = tid / BN, bcol = tid % BN;
  const int64_t aoff = ((int64_t)(m0 + arow) * pr.lda + acol) * V;
  const int64_t boff = ((int64_t)brow * pr.ldb + n0 + bcol) * V;
  const double2* asrc = pr.A + aoff;
  const double2* a2src = pr.A2 + aoff;
  const double2* bsrc = pr.B + boff;
  const double2* b2src = pr.B2 + boff;
  const int64_t astep = (int64_t)AROWS * pr.lda * V;
  const int64_t bstep = (int64_t)BROWS * pr.ldb * V;
  const int64_t bnext = (int64_t)BK * pr.ldb * V;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int aidx = (arow * (BK + 1) + acol) * V;                   // in double2
  const int bidx = 2 * S::A_STAGE + (brow * BN + bcol) * V;
  const bool sa = pr.sa != 0, sb = pr.sb != 0;
  auto load = [&](int st) {
#pragma unroll
    for (int i = 0; i < AEL; ++i)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const uint32_t d = sbase + (aidx + st * S::A_STAGE + i * AROWS * (BK + 1) * V + v) * 16;
        cp_async16_at(d, asrc + i * astep + v);
        if (sa) cp_async16_at(d + Y_OFF_B, a2src + i * astep + v);
      }
#pragma unroll
    for (int i = 0; i < BEL; ++i)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const uint32_t d = sbase + (bidx + st * S::B_STAGE + i * BROWS * BN * V + v) * 16;
        cp_async16_at(d, bsrc + i * bstep + v);
        if (sb) cp_async16_at(d + Y_OFF_B, b2src + i * bstep + v);
      }
    asrc += BK * V, a2src += BK * V;
    bsrc += bnext, b2src += bnext;
  };
  // the reference's ewise add/sub on this thread's own staged elements
  auto fold = [&](int st) {
    if (sa) {
#pragma unroll
      for (int i = 0; i < AEL; ++i) {
        double2* x = smem + aidx + st * S::A_STAGE + i * AROWS * (BK + 1) * V;
        fold_sum<V>(x, x + S::TOTAL, pr.sa);
      }
    }
    if (sb) {
#pragma unroll
      for (int i = 0; i < BEL; ++i) {
        double2* x = smem + bidx + st * S::B_STAGE + i * BROWS * BN * V;
        fold_sum<V>(x, x + S::TOTAL, pr.sb);
      }
    }
  };
  const uint32_t ard = sbase + ty * ((BK + 1) * V * 16);
  const uint32_t brd = sbase + 2 * A_STAGE_B + tx * (V * 16);

  const int ktiles = l / BK;
  load(0);
  cp_async_commit();
  for (int kt = 0; kt < ktiles; ++kt) {
    const int st = kt & 1;
    cp_async_wait<0>();
    fold(st);
    __syncthreads();
    if (kt + 1 < ktiles) {
      load(st ^ 1);
      cp_async_commit();
    }
    uint32_t ap = ard + st * A_STAGE_B, bp = brd + st * B_STAGE_B;
    const uint32_t aend = ap + BK * V * 16;
#pragma unroll 1
    do {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        double2 a[TM][V], b[TN][V];
#pragma unroll
        for (int r = 0; r < TM; ++r)
#pragma unroll
          for (int v = 0; v < V; ++v)
            a[r][v] = lds_double2(ap + ((r * NTY * (BK + 1) + u) * V + v) * 16);
#pragma unroll
        for (int c = 0; c < TN; ++c)
#pragma unroll
          for (int v = 0; v < V; ++v)
            b[c][v] = lds_double2(bp + ((u * BN + c * NTX) * V + v) * 16);
#pragma unroll
        for (int r = 0; r < TM; ++r)
#pragma unroll
          for (int c = 0; c < TN; ++c) Ops::madd(acc[r][c], a[r], b[c]);
      }
      ap += UNROLL * V * 16;
      bp += UNROLL * BN * V * 16;
    } while (ap != aend);
  }
  __syncthreads();

#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      const int i = m0 + ty + r * NTY, j = n0 + tx + c * NTX;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        pr.C[((int64_t)i * pr.ldc + j) * V + v] =
            make_double2(acc[r][c][2 * v], acc[r][c][2 * v + 1]);
        bad |= !finite2(acc[r][c][2 * v], acc[r][c][2 * v + 1]);
      }
    }
}

template <class Ops, int BM, int BN, int BK, int TM, int TN, int NT>
__device__ __forceinline__ void gemm_tile_sum_any(const SumProb& pr, int m, int n, int l, int m0,
                                                  int n0, double2* smem, bool& bad) {
  if constexpr (SumInteriorOk<Ops, BM, BN, BK, NT>::value) {
    if (m0 + BM <= m && n0 + BN <= n && l >= BK && l % BK == 0) {
      gemm_tile_sum_interior<Ops, BM, BN, BK, TM, TN, NT>(pr, l, m0, n0, smem, bad);
      return;
    }
  }
  gemm_tile_sum<Ops, BM, BN, BK, TM, TN, NT>(pr, m, n, l, m0, n0, smem, bad);
}

template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
gemm_tiled_sum(const SumProblem* __restrict__ probs, int m, int n, int l,
               int* __restrict__ nonfinite, const DomainGate gate) {
  constexpr int NT = (BM / TM) * (BN / TN);
  extern __shared__ __align__(16) double2 dsmem[];
  if (gate_skip(gate)) return;
  const int tiles_n = (n + BN - 1) / BN, tiles_m = (m + BM - 1) / BM;
  const int per = tiles_m * tiles_n;
  const int p = blockIdx.x / per, t = blockIdx.x % per;
  const SumProb pr = get_sum_prob(probs[p]);
  bool bad = false;
  int tm, tn;
  grouped_tile(t, tiles_m, tiles_n, tm, tn);
  gemm_tile_sum_any<Ops, BM, BN, BK, TM, TN, NT>(pr, m, n, l, tm * BM, tn * BN, dsmem, bad);
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
}

template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB>
cudaError_t launch_tiled_sum(const GemmArgs& g) {
  auto kern = gemm_tiled_sum<Ops, BM, BN, BK, TM, TN, MINB>;
  constexpr size_t bytes = SumSmem<Ops, BM, BN, BK>::TOTAL * sizeof(double2);
  if (cudaError_t attr = allow_smem(kern, bytes); attr != cudaSuccess) return attr;
  int64_t tiles = (int64_t)((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN) * g.batch;
  if (tiles == 0) return cudaSuccess;
  if (tiles > 0x7fffffff) return cudaErrorInvalidValue;
  kern<<<(unsigned)tiles, (BM / TM) * (BN / TN), bytes, g.stream>>>(g.sprobs, g.m, g.n, g.l,
                                                                    g.nonfinite, g.gate);
  return cudaGetLastError();
}

// Plain tiled kernel: one CTA per (problem, tile).  STREAM: the operands
// arrive while it runs (wait_k_panel); a separate instantiation, so the
// resident-operand kernel keeps its code unchanged.
template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB, bool STREAM = false>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
gemm_tiled(const GemmProblem* __restrict__ probs, Prob single, int m, int n, int l,
           int accumulate, int* __restrict__ nonfinite, const KReady kr,
           const DomainGate gate) {
  constexpr int NT = (BM / TM) * (BN / TN);
  extern __shared__ __align__(16) double2 smem[];   // TileSmem<Ops, BM, BN, BK>::TOTAL
  if (gate_skip(gate)) return;
  const int tiles_n = (n + BN - 1) / BN, tiles_m = (m + BM - 1) / BM;
  const int per = tiles_m * tiles_n;
  const int p = blockIdx.x / per, t = blockIdx.x % per;
  const Prob pr = get_prob(probs, single, p);
  bool bad = false;
  int tm, tn;
  grouped_tile(t, tiles_m, tiles_n, tm, tn);
  gemm_tile_any<Ops, BM, BN, BK, TM, TN, NT, STREAM>(pr, m, n, l, accumulate, tm * BM, tn * BN,
                                                     smem, bad, STREAM ? kr : KReady{nullptr, 0});
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
}

// The Dekker (rare-path) launches of the domain gate as persistent CTAs
// striding over the tiles: in the usual in-domain case every CTA exits at
// the gate, so the launch costs one small grid instead of a CTA per tile.
// SUM: Strassen leaves with folded operand sums (SumProblem table).
template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB, bool SUM>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
gemm_persist(const GemmProblem* __restrict__ probs, const SumProblem* __restrict__ sprobs,
             Prob single, int P, int m, int n, int l, int accumulate, int* __restrict__ nonfinite,
             const DomainGate gate) {
  constexpr int NT = (BM / TM) * (BN / TN);
  extern __shared__ __align__(16) double2 dsmem[];
  if (gate_skip(gate)) return;
  const int tiles_n = (n + BN - 1) / BN, tiles_m = (m + BM - 1) / BM;
  const int per = tiles_m * tiles_n;
  const int64_t total = (int64_t)P * per;
  bool bad = false;
  for (int64_t u = blockIdx.x; u < total; u += gridDim.x) {
    const int p = (int)(u / per), t = (int)(u % per);
    const int m0 = (t / tiles_n) * BM, n0 = (t % tiles_n) * BN;
    if constexpr (SUM) {
      gemm_tile_sum_any<Ops, BM, BN, BK, TM, TN, NT>(get_sum_prob(sprobs[p]), m, n, l, m0, n0,
                                                dsmem, bad);
    } else {
      gemm_tile<Ops, BM, BN, BK, TM, TN, NT>(get_prob(probs, single, p), m, n, l, accumulate,
                                             m0, n0, dsmem, bad);
    }
  }
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
}

inline Prob single_prob(const GemmArgs& g);

template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB>
cudaError_t launch_persist(const GemmArgs& g) {
  const bool sum = g.sprobs != nullptr;
  auto kern = sum ? gemm_persist<Ops, BM, BN, BK, TM, TN, MINB, true>
                  : gemm_persist<Ops, BM, BN, BK, TM, TN, MINB, false>;
  const size_t bytes = (sum ? SumSmem<Ops, BM, BN, BK>::TOTAL
                            : TileSmem<Ops, BM, BN, BK>::TOTAL) * sizeof(double2);
  constexpr int NT = (BM / TM) * (BN / TN);
  int dev = 0, sms = 0, occ = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = allow_smem(kern, bytes);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, bytes);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (int64_t)((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN) * g.batch;
  if (tiles == 0) return cudaSuccess;
  const int64_t slots = (int64_t)sms * (occ > 0 ? occ : 1);
  const unsigned grid = (unsigned)(tiles < slots ? tiles : slots);
  kern<<<grid, NT, bytes, g.stream>>>(g.probs, g.sprobs, single_prob(g), g.batch, g.m, g.n, g.l,
                                      g.accumulate, g.nonfinite, g.gate);
  return cudaGetLastError();
}

// Persistent largest-first kernel: big BM x BN tiles in whole waves, then
// the leftover big tiles as quarter tiles (BM/2 x BN/2, TM/2 x TN/2 per
// thread, same thread count).
template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
gemm_lpt(const GemmProblem* __restrict__ probs, Prob single, int P, int m, int n, int l,
         int accumulate, int* __restrict__ nonfinite, const DomainGate gate) {
  constexpr int NT = (BM / TM) * (BN / TN);
  static_assert(TM % 2 == 0 && TN % 2 == 0, "quarter tiles need even thread tiles");
  extern __shared__ __align__(16) double2 smem[];   // TileSmem<Ops, BM, BN, BK>::TOTAL
  if (gate_skip(gate)) return;
  const int tiles_n = (n + BN - 1) / BN, tiles_m = (m + BM - 1) / BM;
  const int per = tiles_m * tiles_n;
  const int T = P * per;
  const int S = gridDim.x;
  const int nbig = (T / S) * S;
  const int units = nbig + 4 * (T - nbig);
  bool bad = false;
  for (int u = blockIdx.x; u < units; u += S) {
    int t, q = -1;
    if (u < nbig) {
      t = u;
    } else {
      t = nbig + (u - nbig) / 4;
      q = (u - nbig) % 4;
    }
    const int p = t / per, tt = t % per;
    const Prob pr = get_prob(probs, single, p);
    int tm, tn;
    grouped_tile(tt, tiles_m, tiles_n, tm, tn);
    int m0 = tm * BM, n0 = tn * BN;
    if (q < 0) {
      gemm_tile_any<Ops, BM, BN, BK, TM, TN, NT>(pr, m, n, l, accumulate, m0, n0, smem, bad);
    } else {
      m0 += (q / 2) * (BM / 2);
      n0 += (q % 2) * (BN / 2);
      if (m0 < m && n0 < n)  // uniform per CTA: no divergent barriers
        gemm_tile_any<Ops, BM / 2, BN / 2, BK, TM / 2, TN / 2, NT>(pr, m, n, l, accumulate, m0,
                                                                  n0, smem, bad);
    }
  }
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
}

// The reference's "simple" algorithm: one thread per output element, the
// operands read straight from global memory (L1/L2), no staging.
template <class Ops>
__global__ void __launch_bounds__(256)
gemm_simple(const GemmProblem* __restrict__ probs, Prob single, int m, int n, int l,
            int accumulate, int* __restrict__ nonfinite, const DomainGate gate) {
  constexpr int V = Ops::V;
  if (gate_skip(gate)) return;
  const int p = blockIdx.z;
  const Prob pr = get_prob(probs, single, p);
  int j = blockIdx.x * 32 + (threadIdx.x & 31);
  int i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= m || j >= n) return;
  double acc[Ops::NACC];
  double2* cp = pr.C + ((int64_t)i * pr.ldc + j) * V;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    double2 x = accumulate ? cp[v] : make_double2(0.0, 0.0);
    acc[2 * v] = x.x;
    acc[2 * v + 1] = x.y;
  }
  const double2* a = pr.A + (int64_t)i * pr.lda * V;
  const double2* b = pr.B + (int64_t)j * V;
  for (int k = 0; k < l; ++k) {
    double2 av[V], bv[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      av[v] = __ldg(a + (int64_t)k * V + v);
      bv[v] = __ldg(b + (int64_t)k * pr.ldb * V + v);
    }
    Ops::madd(acc, av, bv);
  }
  bool bad = false;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    cp[v] = make_double2(acc[2 * v], acc[2 * v + 1]);
    bad |= !finite2(acc[2 * v], acc[2 * v + 1]);
  }
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
}

// ---------------------------------------------------------------------------
// host-side launch helpers
// ---------------------------------------------------------------------------

inline Prob single_prob(const GemmArgs& g) {
  return Prob{reinterpret_cast<const double2*>(g.A), reinterpret_cast<const double2*>(g.B),
              reinterpret_cast<double2*>(g.C), g.lda, g.ldb, g.ldc};
}

template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB>
cudaError_t launch_tiled(const GemmArgs& g) {
  int64_t tiles = (int64_t)((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN) * g.batch;
  if (tiles == 0) return cudaSuccess;
  if (tiles > 0x7fffffff) return cudaErrorInvalidValue;
  const unsigned grid = (unsigned)tiles, nt = (BM / TM) * (BN / TN);
  constexpr size_t bytes = TileSmem<Ops, BM, BN, BK>::TOTAL * sizeof(double2);
  const KReady kr{g.kready, g.kpanel, g.ktile_rows, g.ktile_cols, g.ka_panels};
  if (g.kready != nullptr) {
    auto kern = gemm_tiled<Ops, BM, BN, BK, TM, TN, MINB, true>;
    if (cudaError_t e = allow_smem(kern, bytes); e != cudaSuccess) return e;
    kern<<<grid, nt, bytes, g.stream>>>(g.probs, single_prob(g), g.m, g.n, g.l, g.accumulate,
                                        g.nonfinite, kr, g.gate);
  } else {
    auto kern = gemm_tiled<Ops, BM, BN, BK, TM, TN, MINB, false>;
    if (cudaError_t e = allow_smem(kern, bytes); e != cudaSuccess) return e;
    kern<<<grid, nt, bytes, g.stream>>>(g.probs, single_prob(g), g.m, g.n, g.l, g.accumulate,
                                        g.nonfinite, kr, g.gate);
  }
  return cudaGetLastError();
}

template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB>
cudaError_t launch_lpt(const GemmArgs& g) {
  auto kern = gemm_lpt<Ops, BM, BN, BK, TM, TN, MINB>;
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr size_t bytes = TileSmem<Ops, BM, BN, BK>::TOTAL * sizeof(double2);
  int dev = 0, sms = 0, occ = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = allow_smem(kern, bytes);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, bytes);
  if (e != cudaSuccess) return e;
  int64_t tiles = (int64_t)((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN) * g.batch;
  if (tiles == 0) return cudaSuccess;
  if (tiles * 4 > 0x7fffffff) return cudaErrorInvalidValue;
  int64_t slots = (int64_t)sms * (occ > 0 ? occ : 1);
  // fewer units than slots: launch one CTA per unit (all quarter tiles)
  int64_t units = tiles < slots ? 4 * tiles : slots;
  int grid = (int)(units < slots ? units : slots);
  kern<<<grid, NT, bytes, g.stream>>>(g.probs, single_prob(g), g.batch, g.m, g.n, g.l,
                                      g.accumulate, g.nonfinite, g.gate);
  return cudaGetLastError();
}

template <class Ops>
cudaError_t launch_simple(const GemmArgs& g) {
  if (g.batch > 65535) return cudaErrorInvalidValue;
  dim3 grid((g.n + 31) / 32, (g.m + 7) / 8, g.batch), block(256);
  gemm_simple<Ops><<<grid, block, 0, g.stream>>>(g.probs, single_prob(g), g.m, g.n, g.l,
                                                 g.accumulate, g.nonfinite, g.gate);
  return cudaGetLastError();
}

template <class Kern>
cudaError_t occupancy_of(Kern kern, int threads, Geometry* geo, size_t smem_bytes = 0) {
  geo->threads = threads;
  if (cudaError_t e = allow_smem(kern, smem_bytes); e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&geo->ctas_per_sm, kern, threads,
                                                       smem_bytes);
}

// CTA tile and residency of a gemm_tiled / gemm_lpt configuration
template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB>
cudaError_t tiled_geometry(Geometry* geo) {
  geo->bm = BM, geo->bn = BN;
  return occupancy_of(gemm_tiled<Ops, BM, BN, BK, TM, TN, MINB, false>, (BM / TM) * (BN / TN), geo,
                      TileSmem<Ops, BM, BN, BK>::TOTAL * sizeof(double2));
}

template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB>
cudaError_t lpt_geometry(Geometry* geo) {
  geo->bm = BM, geo->bn = BN;
  return occupancy_of(gemm_lpt<Ops, BM, BN, BK, TM, TN, MINB>, (BM / TM) * (BN / TN), geo,
                      TileSmem<Ops, BM, BN, BK>::TOTAL * sizeof(double2));
}

}  // namespace mpmm
