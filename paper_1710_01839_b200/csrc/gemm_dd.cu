// gemm_dd.cu -- double-double GEMM kernels for sm_100a (bit-exact mirror).
//
// C (m x n) = A (m x l) * B (l x n), or C += A*B, every matrix a row-major
// view of DD elements (double2 = {hi, lo}) with a leading dimension in
// elements -- the reference's AoS layout (matrix.py:20,43-48), so host
// arrays cross the C-ABI without any re-layout, and Strassen quadrants are
// plain (pointer, ld) views.
//
// Per output element the k loop runs in ascending order from an
// accumulator that starts at (0, 0) (overwrite) or at C (accumulate), and
// every step is the reference's dd_add(c, dd_mul(a, b)) (ddqd.cuh), so each
// element is bit-identical to the reference's dd_simple_rows
// (_kernels.pyx:36-100) / dd_block_cells (:103-186) for ANY tiling: the
// tile shape is a performance knob only (the reference's n_min maps onto
// it, see tile_for_nmin()).
//
// The kernel is bound by the FP64 pipe (50 FP64 instructions per
// multiply-add); shared-memory tiles are staged with
// cp.async double buffering so the loads hide under the arithmetic.
#include "common.cuh"
#include "ddqd.cuh"
#include "kernels.h"

namespace mpmm {

template <int BM, int BN, int BK, int TM, int TN>
struct DDTile {
  static constexpr int NTX = BN / TN;
  static constexpr int NTY = BM / TM;
  static constexpr int NT = NTX * NTY;
  static constexpr int APAD = 1;  // one element of padding per A row
};

template <int BM, int BN, int BK, int TM, int TN, int MINB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
dd_gemm_tiled(const double2* __restrict__ A, int64_t lda, const double2* __restrict__ B,
              int64_t ldb, double2* __restrict__ C, int64_t ldc, int m, int n, int l,
              int accumulate, int tiles_n, int super, int* __restrict__ nonfinite) {
  using T = DDTile<BM, BN, BK, TM, TN>;
  constexpr int NTX = T::NTX, NTY = T::NTY, NT = T::NT;
  __shared__ __align__(16) double2 As[2][BM][BK + T::APAD];
  __shared__ __align__(16) double2 Bs[2][BK][BN];

  // Tile rasterisation: "super" x "super" groups of tiles are walked
  // together (an L2 super-tile; the reference's n_min > 64 maps here).
  int tile = blockIdx.x;
  int tm, tn;
  if (super > 1) {
    int tiles_m = (m + BM - 1) / BM;
    int group = super * tiles_n;               // tiles in one band of super rows
    int band = tile / group;
    int first_m = band * super;
    int rows_in_band = min(super, tiles_m - first_m);
    int in_band = tile - band * group;
    tm = first_m + in_band % rows_in_band;
    tn = in_band / rows_in_band;
  } else {
    tm = tile / tiles_n;
    tn = tile - tm * tiles_n;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int tid = threadIdx.x;
  const int tx = tid % NTX, ty = tid / NTX;

  double ch[TM][TN], cl[TM][TN];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      int i = m0 + ty + r * NTY, j = n0 + tx + c * NTX;
      if (accumulate && i < m && j < n) {
        double2 v = C[(int64_t)i * ldc + j];
        ch[r][c] = v.x;
        cl[r][c] = v.y;
      } else {
        ch[r][c] = 0.0;
        cl[r][c] = 0.0;
      }
    }

  const int ktiles = (l + BK - 1) / BK;
  auto load = [&](int kt, int stage) {
    const int k0 = kt * BK;
#pragma unroll
    for (int e = tid; e < BM * BK; e += NT) {
      int row = e / BK, col = e - (e / BK) * BK;
      int gi = m0 + row, gk = k0 + col;
      bool ok = gi < m && gk < l;
      const double2* src = ok ? A + (int64_t)gi * lda + gk : A;
      cp_async16(&As[stage][row][col], src, ok);
    }
#pragma unroll
    for (int e = tid; e < BK * BN; e += NT) {
      int row = e / BN, col = e - (e / BN) * BN;
      int gk = k0 + row, gj = n0 + col;
      bool ok = gk < l && gj < n;
      const double2* src = ok ? B + (int64_t)gk * ldb + gj : B;
      cp_async16(&Bs[stage][row][col], src, ok);
    }
  };

  if (ktiles > 0) {
    load(0, 0);
    cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    const int stage = kt & 1;
    if (kt + 1 < ktiles) {
      load(kt + 1, stage ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int kcount = min(BK, l - kt * BK);
    if (kcount == BK) {
#pragma unroll 2
      for (int kk = 0; kk < BK; ++kk) {
        double2 a[TM], b[TN];
#pragma unroll
        for (int r = 0; r < TM; ++r) a[r] = As[stage][ty + r * NTY][kk];
#pragma unroll
        for (int c = 0; c < TN; ++c) b[c] = Bs[stage][kk][tx + c * NTX];
#pragma unroll
        for (int r = 0; r < TM; ++r)
#pragma unroll
          for (int c = 0; c < TN; ++c) dd_madd(ch[r][c], cl[r][c], a[r].x, a[r].y, b[c].x, b[c].y);
      }
    } else {
      for (int kk = 0; kk < kcount; ++kk) {
        double2 a[TM], b[TN];
#pragma unroll
        for (int r = 0; r < TM; ++r) a[r] = As[stage][ty + r * NTY][kk];
#pragma unroll
        for (int c = 0; c < TN; ++c) b[c] = Bs[stage][kk][tx + c * NTX];
#pragma unroll
        for (int r = 0; r < TM; ++r)
#pragma unroll
          for (int c = 0; c < TN; ++c) dd_madd(ch[r][c], cl[r][c], a[r].x, a[r].y, b[c].x, b[c].y);
      }
    }
    __syncthreads();
  }

  bool bad = false;
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      int i = m0 + ty + r * NTY, j = n0 + tx + c * NTX;
      if (i < m && j < n) {
        C[(int64_t)i * ldc + j] = make_double2(ch[r][c], cl[r][c]);
        bad |= !finite2(ch[r][c], cl[r][c]);
      }
    }
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
}

// The reference's "simple" algorithm on the GPU: one thread per output
// element, operands read straight from global memory (L1/L2), no shared
// memory staging (_kernels.pyx:36-100 dd_simple_rows).
__global__ void __launch_bounds__(256)
dd_gemm_simple(const double2* __restrict__ A, int64_t lda, const double2* __restrict__ B,
               int64_t ldb, double2* __restrict__ C, int64_t ldc, int m, int n, int l,
               int accumulate, int* __restrict__ nonfinite) {
  int j = blockIdx.x * 32 + (threadIdx.x & 31);
  int i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= m || j >= n) return;
  double ch = 0.0, cl = 0.0;
  if (accumulate) {
    double2 v = C[(int64_t)i * ldc + j];
    ch = v.x;
    cl = v.y;
  }
  const double2* a = A + (int64_t)i * lda;
  const double2* b = B + j;
  for (int k = 0; k < l; ++k) {
    double2 av = __ldg(a + k);
    double2 bv = __ldg(b + (int64_t)k * ldb);
    dd_madd(ch, cl, av.x, av.y, bv.x, bv.y);
  }
  C[(int64_t)i * ldc + j] = make_double2(ch, cl);
  if (nonfinite != nullptr && !finite2(ch, cl)) atomicOr(nonfinite, 1);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

template <int BM, int BN, int BK, int TM, int TN, int MINB>
static cudaError_t launch_tiled(const GemmArgs& g, int super) {
  int tiles_m = (g.m + BM - 1) / BM, tiles_n = (g.n + BN - 1) / BN;
  int64_t tiles = (int64_t)tiles_m * tiles_n;
  if (tiles == 0) return cudaSuccess;
  dim3 grid((unsigned)tiles), block((BM / TM) * (BN / TN));
  dd_gemm_tiled<BM, BN, BK, TM, TN, MINB><<<grid, block, 0, g.stream>>>(
      reinterpret_cast<const double2*>(g.A), g.lda, reinterpret_cast<const double2*>(g.B), g.ldb,
      reinterpret_cast<double2*>(g.C), g.ldc, g.m, g.n, g.l, g.accumulate, tiles_n, super,
      g.nonfinite);
  return cudaGetLastError();
}

template <int BM, int BN, int BK, int TM, int TN, int MINB>
static cudaError_t geometry_tiled(Geometry* geo) {
  geo->bm = BM;
  geo->bn = BN;
  geo->threads = (BM / TM) * (BN / TN);
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &geo->ctas_per_sm, dd_gemm_tiled<BM, BN, BK, TM, TN, MINB>, geo->threads, 0);
}

cudaError_t dd_gemm_geometry(int algo, int tile, Geometry* geo) {
  if (algo == ALGO_SIMPLE) {
    geo->bm = 8;
    geo->bn = 32;
    geo->threads = 256;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&geo->ctas_per_sm, dd_gemm_simple, 256, 0);
  }
  switch (tile) {
    case TILE_16: return geometry_tiled<16, 16, 16, 1, 1, 4>(geo);
    case TILE_32: return geometry_tiled<32, 32, 8, 2, 2, 2>(geo);
    case TILE_64: return geometry_tiled<64, 64, 8, 4, 4, 1>(geo);
    case TILE_32x64: return geometry_tiled<32, 64, 8, 2, 2, 1>(geo);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t dd_gemm_launch(const GemmArgs& g) {
  if (g.m <= 0 || g.n <= 0) return cudaSuccess;
  if (g.algo == ALGO_SIMPLE) {
    dim3 grid((g.n + 31) / 32, (g.m + 7) / 8), block(256);
    dd_gemm_simple<<<grid, block, 0, g.stream>>>(
        reinterpret_cast<const double2*>(g.A), g.lda, reinterpret_cast<const double2*>(g.B),
        g.ldb, reinterpret_cast<double2*>(g.C), g.ldc, g.m, g.n, g.l, g.accumulate, g.nonfinite);
    return cudaGetLastError();
  }
  switch (g.tile) {
    case TILE_16:
      return launch_tiled<16, 16, 16, 1, 1, 4>(g, 1);
    case TILE_32:
      return launch_tiled<32, 32, 8, 2, 2, 2>(g, 1);
    case TILE_64:
      return launch_tiled<64, 64, 8, 4, 4, 1>(g, g.super > 1 ? g.super : 1);
    case TILE_32x64:
      return launch_tiled<32, 64, 8, 2, 2, 1>(g, g.super > 1 ? g.super : 1);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace mpmm
