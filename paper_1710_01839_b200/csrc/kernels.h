// kernels.h -- internal launcher interface shared by the .cu files and the
// C-ABI layer (capi.cu).  Not part of the public ABI (that is
// include/mpmm_cuda.h).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "domain.cuh"

namespace mpmm {

enum Algo { ALGO_SIMPLE = 0, ALGO_BLOCK = 1, ALGO_BLOCK_FAST = 2 };

// CTA tile configurations of the blocked kernels.  The reference's block
// size n_min selects one (tile_for_nmin); results never depend on it.
enum Tile { TILE_16 = 0, TILE_32 = 1, TILE_64 = 2, TILE_32x64 = 3, TILE_LPT = 4, TILE_COUNT = 5 };

// One problem of a batched launch (all problems share m, n, l).  Same
// layout as the 6 x int64 rows the Python side builds for Strassen leaves.
struct GemmProblem {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
};

// One Strassen leaf with its operand sums folded into the tile loads
// (gemm.cuh gemm_tiled_sum): (A + sa*A2) * (B + sb*B2), sa/sb in {0, +1, -1}
// (0: the operand alone); A2 shares A's leading dimension, B2 B's.
struct SumProblem {
  const double* A;
  const double* A2;
  const double* B;
  const double* B2;
  double* C;
  int64_t lda, ldb, ldc;
  int32_t sa, sb;
};

struct GemmArgs {
  int algo;          // ALGO_SIMPLE or ALGO_BLOCK
  int tile;          // Tile (ALGO_BLOCK)
  int m, n, l;
  const double* A;   // element (i,k) at A + comps*(i*lda + k)
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int accumulate;    // 0: acc starts at 0 and C is overwritten; 1: C += A*B
  int* nonfinite;    // device flag, OR-ed with 1 if any output is non-finite (may be null)
  cudaStream_t stream;
  int batch = 1;                         // number of problems
  const GemmProblem* probs = nullptr;    // device array of `batch` problems, or null: A/B/C above
  // Streamed operands (gemm_tiled only): k-panel q of A and B is usable once
  // kready[q] != 0 (set by the copy stream after the panel's H2D); panels
  // are kpanel columns of k.  Null: the operands are already resident.
  const int* kready = nullptr;
  int kpanel = 0;
  // kpanel == 0 with kready set: tile mode -- kready[0 .. ka_panels) flag A
  // row panels of ktile_rows rows, then B column panels of ktile_cols columns
  int ktile_rows = 0, ktile_cols = 0, ka_panels = 0;
  // EFT-domain gate (domain.cuh): with gate.words set, the launch runs only
  // on the side of the domain test gate.want_unsafe selects.
  DomainGate gate{};
  // Strassen leaves with folded operand sums: `batch` SumProblems in device
  // memory (ALGO_BLOCK only; one tile configuration per precision).
  const SumProblem* sprobs = nullptr;
};

// The DFMA mirror kernels (ALGO_SIMPLE / ALGO_BLOCK / ALGO_BLOCK_FAST).
// Tile rows per group of the grouped tile raster (gemm.cuh grouped_tile);
// the streamed host product copies operands in that order.
#ifndef MPMM_GROUP_M
#define MPMM_GROUP_M 16   // experiments: -DMPMM_GROUP_M=n (tools/exp/build_variant.py)
#endif
constexpr int kTileGroupM = MPMM_GROUP_M;

cudaError_t dd_gemm_launch(const GemmArgs& g);
cudaError_t qd_gemm_launch(const GemmArgs& g);
// The same products with the reference's Dekker TwoProd (one tile shape for
// every algorithm: per element the operation sequence is the reference's, so
// the tiling never changes a bit).  No streamed operands.
cudaError_t dd_dekker_launch(const GemmArgs& g);
cudaError_t qd_dekker_launch(const GemmArgs& g);

// Scan the operands of one product (A: m x l, B: l x n views) into the six
// domain words (domain.cuh) of a per-stream buffer; *words receives the
// device pointer, valid in stream order until the next scan on `stream`.
cudaError_t domain_scan(int comps, const double* A, int64_t lda, int m, int l, const double* B,
                        int64_t ldb, int n, const int** words, cudaStream_t stream);
// The same over every problem of a batched launch (one set of words).
cudaError_t domain_scan_batched(int comps, const GemmProblem* probs, int batch, int m, int l,
                                int n, const int** words, cudaStream_t stream);
// A mirror product with the reference's semantics on every input: scan,
// then the DFMA launch gated on the domain and the Dekker launch gated on
// its complement (g.gate's margins are kept; its words are replaced).
// ALGO_BLOCK_FAST (not a mirror) and streamed launches run ungated.
// When `words_out` is non-null the scan's words pointer is stored there.
cudaError_t gemm_checked(int comps, GemmArgs g, const int** words_out = nullptr);
// The two gated launches of gemm_checked for operands already scanned.
cudaError_t gemm_gated(int comps, GemmArgs g, const int* words);

// CTA tile and residency of the kernel a launch would use.
struct Geometry {
  int bm, bn, threads, ctas_per_sm;
};
cudaError_t dd_gemm_geometry(int algo, int tile, Geometry* geo);
cudaError_t qd_gemm_geometry(int algo, int tile, Geometry* geo);

// out = ((x s1 y) s2 z) s3 w for nops = 1, 2, 3 (signs +1/-1), elementwise,
// each step one reference ewise add/sub (_kernels.pyx:207-230, :407-452).
struct EwiseArgs {
  int comps;
  int nops;
  int rows, cols;
  const double* X; int64_t ldx;
  const double* Y; int64_t ldy; int sy;
  const double* Z; int64_t ldz; int sz;
  const double* W; int64_t ldw; int sw;
  double* O; int64_t ldo;
  cudaStream_t stream;
};
cudaError_t ewise_launch(const EwiseArgs& e);

// One problem of a batched elementwise launch (all share rows x cols).
// Layout = 14 int64 words, as built by the Python Strassen planner.
struct EwiseProblem {
  const double* X;
  const double* Y;
  const double* Z;
  const double* W;
  double* O;
  int64_t ldx, ldy, ldz, ldw, ldo;
  int64_t nops, sy, sz, sw;
};
cudaError_t ewise_batched_launch(int comps, int batch, int rows, int cols,
                                 const EwiseProblem* probs, cudaStream_t stream);

cudaError_t nonfinite_launch(int comps, const double* X, int64_t ldx, int rows, int cols,
                             int* flag, cudaStream_t stream);

cudaError_t exact_check_launch(int comps, int l, const double* A, int64_t lda, const double* B,
                               int64_t ldb, const double* C, int64_t ldc, const int64_t* idx_i,
                               const int64_t* idx_j, int64_t count, int u_exp, double* ratio,
                               cudaStream_t stream);

cudaError_t uniform_launch(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                           uint64_t first, int64_t count, double* out, cudaStream_t stream);
cudaError_t assemble_launch(int comps, const double* draws, int64_t count, double* out,
                            cudaStream_t stream);

// exact int8 tensor-core mode (ozaki.cu, int8gemm.cpp)
cudaError_t oz_scan_launch(int by_cols, const double* X, int64_t ld, int rows, int cols, int comps,
                           int* EL, int* status, cudaStream_t s);
cudaError_t oz_residues_launch(int by_cols, const double* X, int64_t ld, int rows, int cols,
                               int comps, int c0, int c1, const int* shift, int N, int W,
                               int8_t* R, int64_t rpitch, int64_t rplane, cudaStream_t s);
// One CRT job of the combine (56 bytes; tensor.py / exact.cpp build them).
struct CrtJob {
  const void* G;            // [N][.][gpitch] residue products (int32) or residues (uint8)
  const int* srow;          // [m] row shifts
  const int* scol;          // [n] column shifts
  const uint32_t* table;    // [K] P limbs, then [N][K] weight limbs
  int N, K;
  int64_t gpitch, gplane;
};
constexpr int kOzMaxJobs = 16;

cudaError_t oz_combine_launch(int comps, const void* jobs, int njobs, int m, int n, double* C,
                              int* status, cudaStream_t s, bool res8 = false, int win = 28);
int oz_plan(int comps, int64_t m, int64_t n, int64_t l, const int* ela, const int* elb,
            int* njobs, int* jobs, int* na, int* ranges_a, int* shift_a, int* nb, int* ranges_b,
            int* shift_b, int* window_digits = nullptr);
cudaError_t oz_shifts_launch(int comps, int nranges, const int* ranges, int odim, const int* EL,
                             int* shift, int* beta, cudaStream_t s);
int int8_gemm_batched(int64_t m, int64_t n, int64_t k, int64_t batch, const int8_t* A,
                      const int8_t* Bt, int32_t* C, void* workspace, size_t ws_size,
                      cudaStream_t stream, std::string* err);

// tcgen05 residue GEMMs (tc_i8.cu): R_t = (A_t * Bt_t^T) mod p_t as uint8
bool tc_residue_gemm_supported(int64_t m, int64_t n, int64_t k);
int tc_residue_gemm_tile_n();
cudaError_t tc_residue_gemm(int64_t m, int64_t n, int64_t k, int batch, const int8_t* A,
                            const int8_t* Bt, uint8_t* R, cudaStream_t s);

// Keep freed stream-ordered allocations of the current device's default
// pool mapped across synchronizations (the default threshold, 0, unmaps
// them at every sync and the next call re-maps gigabytes of pages).
cudaError_t retain_default_pool();

cudaError_t fp64_burn_launch(int op, int blocks, int threads, int64_t iters, double* out,
                             cudaStream_t stream);

}  // namespace mpmm
