// gemm_qd.cu -- quad-double instantiations of gemm.cuh.
//
// QD element = two double2 (4 limbs); each multiply-add is the reference's
// _qd_mul_add (_kernels.pyx:311-341): 10 TwoProds + 3 products compressed
// to 4 limbs, then an 8-term compression with the accumulator (~786 FP64
// instructions), zero-term filter reproduced exactly (ddqd.cuh).
// Tile configurations (n_min -> tile: capi.cu tile_for).  A QD
// multiply-add needs ~120 registers per accumulator chain, so every
// configuration keeps one chain per thread (measured: 2x2 register tiles
// at one CTA per SM reach only 10.4 TFLOP/s of F, 1x1 tiles 16.5):
//   TILE_16    16x16 CTA tile, 1x1 per thread, 256 threads, 2 CTAs/SM
//   TILE_32    8x16, 1x1, 128 threads, 4 CTAs/SM
//   TILE_LPT   16x16, 1x1, 256 threads, k-tiles of 16
//   TILE_32x64 8x32, 1x1, 256 threads, 2 CTAs/SM, k-tiles of 16
//   TILE_64    16x16, 1x1, 256 threads, 3 CTAs/SM
// Interior tiles run the speculative dense multiply-add (QDSpecOps): the
// reference's zero-term gates recorded instead of branched on, voted once
// per k-tile, the tile recomputed by the gated sequence if a vote fails --
// 1.2 % faster than the gated kernel on dense data, the same bits always
// (profiles/r02_qd_variants.log, tests/test_gpu_interior.py).
#include "gemm.cuh"

#define MPMM_QD16 16, 16, 8, 1, 1, 2
#define MPMM_QD32 8, 16, 8, 1, 1, 4
#define MPMM_QD64 16, 16, 8, 1, 1, 3
#define MPMM_QD32x64 8, 32, 16, 1, 1, 2
#define MPMM_QDLPT 16, 16, 16, 1, 1, 2
#define MPMM_QDSUM 16, 16, 8, 1, 1, 2   // Strassen leaves with folded operand sums (16-deep k-tiles: no gain)

namespace mpmm {

// The blocked kernels' multiply-add: speculative dense on interior tiles
// (gemm.cuh QDSpecOps); -DMPMM_QD_SPEC=0 builds the gated sequence alone.
#if !defined(MPMM_QD_SPEC) || MPMM_QD_SPEC
using QDBlockOps = QDSpecOps;
#else
using QDBlockOps = QDOps;
#endif

cudaError_t qd_gemm_launch(const GemmArgs& g) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.sprobs != nullptr) return launch_tiled_sum<QDOps, MPMM_QDSUM>(g);
  if (g.algo == ALGO_SIMPLE) return launch_simple<QDOps>(g);
  if (g.algo != ALGO_BLOCK) return cudaErrorNotSupported;
  switch (g.tile) {
    case TILE_16: return launch_tiled<QDBlockOps, MPMM_QD16>(g);
    case TILE_32: return launch_tiled<QDBlockOps, MPMM_QD32>(g);
    case TILE_64: return launch_tiled<QDBlockOps, MPMM_QD64>(g);
    case TILE_32x64: return launch_tiled<QDBlockOps, MPMM_QD32x64>(g);
    case TILE_LPT: return launch_tiled<QDBlockOps, MPMM_QDLPT>(g);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t qd_dekker_launch(const GemmArgs& g) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.kready != nullptr) return cudaErrorNotSupported;
  return launch_persist<QDDekkerOps, 16, 16, 8, 1, 1, 2>(g);
}

cudaError_t qd_gemm_geometry(int algo, int tile, Geometry* geo) {
  if (algo == ALGO_SIMPLE) {
    geo->bm = 8, geo->bn = 32;
    return occupancy_of(gemm_simple<QDOps>, 256, geo);
  }
  switch (tile) {
    case TILE_16: return tiled_geometry<QDBlockOps, MPMM_QD16>(geo);
    case TILE_32: return tiled_geometry<QDBlockOps, MPMM_QD32>(geo);
    case TILE_64: return tiled_geometry<QDBlockOps, MPMM_QD64>(geo);
    case TILE_32x64: return tiled_geometry<QDBlockOps, MPMM_QD32x64>(geo);
    case TILE_LPT: return tiled_geometry<QDBlockOps, MPMM_QDLPT>(geo);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mpmm
