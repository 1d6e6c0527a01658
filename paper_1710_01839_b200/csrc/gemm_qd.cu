// gemm_qd.cu -- quad-double GEMM kernels for sm_100a (bit-exact mirror).
//
// Same contract as gemm_dd.cu with 4-limb elements (32 bytes, two double2
// per element): each output element runs the reference's
// _qd_mul_add (_kernels.pyx:311-341) for k = 0..l-1 in ascending order, from
// zero (qd_simple_rows, :344-363) or from C (qd_block_cells, :366-404), so
// results are bit-identical to the reference for any tiling.
//
// About 786 FP64 instructions per multiply-add; the two
// _compress4 calls dominate.  The zero-term filter of _compress4 is kept
// exact: a register-only fast path when every term is nonzero (the common
// case) and an out-of-line general path otherwise (qd_mul_add in ddqd.cuh).
#include "common.cuh"
#include "ddqd.cuh"
#include "kernels.h"

namespace mpmm {

template <int BM, int BN, int BK, int TM, int TN, int MINB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
qd_gemm_tiled(const double2* __restrict__ A, int64_t lda, const double2* __restrict__ B,
              int64_t ldb, double2* __restrict__ C, int64_t ldc, int m, int n, int l,
              int accumulate, int tiles_n, int* __restrict__ nonfinite) {
  constexpr int NTX = BN / TN, NTY = BM / TM, NT = NTX * NTY;
  // element (i, k) = two double2: [2*(i*ld + k)] and [2*(i*ld + k) + 1]
  __shared__ __align__(16) double2 As[2][BM][BK + 1][2];
  __shared__ __align__(16) double2 Bs[2][BK][BN][2];

  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x - (blockIdx.x / tiles_n) * tiles_n;
  const int m0 = tm * BM, n0 = tn * BN;
  const int tid = threadIdx.x, tx = tid % NTX, ty = tid / NTX;

  double acc[TM][TN][4];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      int i = m0 + ty + r * NTY, j = n0 + tx + c * NTX;
      if (accumulate && i < m && j < n) {
        const double2* p = C + 2 * ((int64_t)i * ldc + j);
        double2 v0 = p[0], v1 = p[1];
        acc[r][c][0] = v0.x; acc[r][c][1] = v0.y; acc[r][c][2] = v1.x; acc[r][c][3] = v1.y;
      } else {
        acc[r][c][0] = acc[r][c][1] = acc[r][c][2] = acc[r][c][3] = 0.0;
      }
    }

  const int ktiles = (l + BK - 1) / BK;
  auto load = [&](int kt, int stage) {
    const int k0 = kt * BK;
    for (int e = tid; e < BM * BK * 2; e += NT) {
      int half = e & 1, el = e >> 1;
      int row = el / BK, col = el - (el / BK) * BK;
      int gi = m0 + row, gk = k0 + col;
      bool ok = gi < m && gk < l;
      const double2* src = ok ? A + 2 * ((int64_t)gi * lda + gk) + half : A;
      cp_async16(&As[stage][row][col][half], src, ok);
    }
    for (int e = tid; e < BK * BN * 2; e += NT) {
      int half = e & 1, el = e >> 1;
      int row = el / BN, col = el - (el / BN) * BN;
      int gk = k0 + row, gj = n0 + col;
      bool ok = gk < l && gj < n;
      const double2* src = ok ? B + 2 * ((int64_t)gk * ldb + gj) + half : B;
      cp_async16(&Bs[stage][row][col][half], src, ok);
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
    for (int kk = 0; kk < kcount; ++kk) {
      double a[TM][4], b[TN][4];
#pragma unroll
      for (int r = 0; r < TM; ++r) {
        double2 v0 = As[stage][ty + r * NTY][kk][0], v1 = As[stage][ty + r * NTY][kk][1];
        a[r][0] = v0.x; a[r][1] = v0.y; a[r][2] = v1.x; a[r][3] = v1.y;
      }
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        double2 v0 = Bs[stage][kk][tx + c * NTX][0], v1 = Bs[stage][kk][tx + c * NTX][1];
        b[c][0] = v0.x; b[c][1] = v0.y; b[c][2] = v1.x; b[c][3] = v1.y;
      }
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) qd_mul_add(acc[r][c], a[r], b[c]);
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
        double2* p = C + 2 * ((int64_t)i * ldc + j);
        p[0] = make_double2(acc[r][c][0], acc[r][c][1]);
        p[1] = make_double2(acc[r][c][2], acc[r][c][3]);
        bad |= !isfinite(acc[r][c][0]);
        bad |= !finite2(acc[r][c][1], acc[r][c][2]) || !isfinite(acc[r][c][3]);
      }
    }
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
}

// One thread per output element, operands from global memory
// (_kernels.pyx:344-363 qd_simple_rows).
__global__ void __launch_bounds__(256)
qd_gemm_simple(const double2* __restrict__ A, int64_t lda, const double2* __restrict__ B,
               int64_t ldb, double2* __restrict__ C, int64_t ldc, int m, int n, int l,
               int accumulate, int* __restrict__ nonfinite) {
  int j = blockIdx.x * 32 + (threadIdx.x & 31);
  int i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= m || j >= n) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  double2* cp = C + 2 * ((int64_t)i * ldc + j);
  if (accumulate) {
    double2 v0 = cp[0], v1 = cp[1];
    acc[0] = v0.x; acc[1] = v0.y; acc[2] = v1.x; acc[3] = v1.y;
  }
  for (int k = 0; k < l; ++k) {
    const double2* ap = A + 2 * ((int64_t)i * lda + k);
    const double2* bp = B + 2 * ((int64_t)k * ldb + j);
    double2 a0 = __ldg(ap), a1 = __ldg(ap + 1), b0 = __ldg(bp), b1 = __ldg(bp + 1);
    double a[4] = {a0.x, a0.y, a1.x, a1.y}, b[4] = {b0.x, b0.y, b1.x, b1.y};
    qd_mul_add(acc, a, b);
  }
  cp[0] = make_double2(acc[0], acc[1]);
  cp[1] = make_double2(acc[2], acc[3]);
  bool bad = !finite2(acc[0], acc[1]) || !finite2(acc[2], acc[3]);
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
}

template <int BM, int BN, int BK, int TM, int TN, int MINB>
static cudaError_t launch_tiled(const GemmArgs& g) {
  int tiles_m = (g.m + BM - 1) / BM, tiles_n = (g.n + BN - 1) / BN;
  int64_t tiles = (int64_t)tiles_m * tiles_n;
  if (tiles == 0) return cudaSuccess;
  qd_gemm_tiled<BM, BN, BK, TM, TN, MINB><<<(unsigned)tiles, (BM / TM) * (BN / TN), 0, g.stream>>>(
      reinterpret_cast<const double2*>(g.A), g.lda, reinterpret_cast<const double2*>(g.B), g.ldb,
      reinterpret_cast<double2*>(g.C), g.ldc, g.m, g.n, g.l, g.accumulate, tiles_n, g.nonfinite);
  return cudaGetLastError();
}

template <int BM, int BN, int BK, int TM, int TN, int MINB>
static cudaError_t geometry_tiled(Geometry* geo) {
  geo->bm = BM;
  geo->bn = BN;
  geo->threads = (BM / TM) * (BN / TN);
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &geo->ctas_per_sm, qd_gemm_tiled<BM, BN, BK, TM, TN, MINB>, geo->threads, 0);
}

cudaError_t qd_gemm_geometry(int algo, int tile, Geometry* geo) {
  if (algo == ALGO_SIMPLE) {
    geo->bm = 8;
    geo->bn = 32;
    geo->threads = 256;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&geo->ctas_per_sm, qd_gemm_simple, 256, 0);
  }
  switch (tile) {
    case TILE_16: return geometry_tiled<16, 16, 8, 1, 1, 2>(geo);
    case TILE_32: return geometry_tiled<16, 32, 8, 1, 2, 1>(geo);
    case TILE_64: return geometry_tiled<32, 32, 8, 2, 2, 1>(geo);
    case TILE_32x64: return geometry_tiled<8, 32, 8, 1, 1, 4>(geo);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t qd_gemm_launch(const GemmArgs& g) {
  if (g.m <= 0 || g.n <= 0) return cudaSuccess;
  if (g.algo == ALGO_SIMPLE) {
    dim3 grid((g.n + 31) / 32, (g.m + 7) / 8), block(256);
    qd_gemm_simple<<<grid, block, 0, g.stream>>>(
        reinterpret_cast<const double2*>(g.A), g.lda, reinterpret_cast<const double2*>(g.B),
        g.ldb, reinterpret_cast<double2*>(g.C), g.ldc, g.m, g.n, g.l, g.accumulate, g.nonfinite);
    return cudaGetLastError();
  }
  switch (g.tile) {
    case TILE_16:
      return launch_tiled<16, 16, 8, 1, 1, 2>(g);
    case TILE_32:
      return launch_tiled<16, 32, 8, 1, 2, 1>(g);
    case TILE_64:
      return launch_tiled<32, 32, 8, 2, 2, 1>(g);
    case TILE_32x64:
      return launch_tiled<8, 32, 8, 1, 1, 4>(g);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace mpmm
