// gemm_qd.cu -- quad-double instantiations of gemm.cuh.
//
// QD element = two double2 (4 limbs); each multiply-add is the reference's
// _qd_mul_add (_kernels.pyx:311-341): 10 TwoProds + 3 products compressed
// to 4 limbs, then an 8-term compression with the accumulator (~786 FP64
// instructions), zero-term filter reproduced exactly (ddqd.cuh).
// Tile configurations (n_min -> tile: capi.cu tile_for):
//   TILE_16    16x16 CTA tile, 1x1 per thread, 256 threads
//   TILE_32    16x32, 1x2, 256 threads
//   TILE_LPT   persistent 32x32 (2x2) tiles in whole waves + 16x16 quarters
//   TILE_32x64 8x32, 1x1, 256 threads
//   TILE_64    32x32, 2x2, 256 threads, plain grid
#include "gemm.cuh"

namespace mpmm {

cudaError_t qd_gemm_launch(const GemmArgs& g) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.algo == ALGO_SIMPLE) return launch_simple<QDOps>(g);
  if (g.algo != ALGO_BLOCK) return cudaErrorNotSupported;
  switch (g.tile) {
    case TILE_16: return launch_tiled<QDOps, 16, 16, 8, 1, 1, 2>(g);
    case TILE_32: return launch_tiled<QDOps, 16, 32, 8, 1, 2, 1>(g);
    case TILE_64: return launch_tiled<QDOps, 32, 32, 8, 2, 2, 1>(g);
    case TILE_32x64: return launch_tiled<QDOps, 8, 32, 8, 1, 1, 2>(g);
    case TILE_LPT: return launch_lpt<QDOps, 32, 32, 8, 2, 2, 1>(g);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t qd_gemm_geometry(int algo, int tile, Geometry* geo) {
  if (algo == ALGO_SIMPLE) {
    geo->bm = 8, geo->bn = 32;
    return occupancy_of(gemm_simple<QDOps>, 256, geo);
  }
  switch (tile) {
    case TILE_16: geo->bm = 16, geo->bn = 16;
      return occupancy_of(gemm_tiled<QDOps, 16, 16, 8, 1, 1, 2>, 256, geo);
    case TILE_32: geo->bm = 16, geo->bn = 32;
      return occupancy_of(gemm_tiled<QDOps, 16, 32, 8, 1, 2, 1>, 256, geo);
    case TILE_64: geo->bm = 32, geo->bn = 32;
      return occupancy_of(gemm_tiled<QDOps, 32, 32, 8, 2, 2, 1>, 256, geo);
    case TILE_32x64: geo->bm = 8, geo->bn = 32;
      return occupancy_of(gemm_tiled<QDOps, 8, 32, 8, 1, 1, 2>, 256, geo);
    case TILE_LPT: geo->bm = 32, geo->bn = 32;
      return occupancy_of(gemm_lpt<QDOps, 32, 32, 8, 2, 2, 1>, 256, geo);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mpmm
