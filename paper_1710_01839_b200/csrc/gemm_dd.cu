// gemm_dd.cu -- double-double instantiations of gemm.cuh.
//
// DD element = one double2 {hi, lo}; each multiply-add is the reference's
// dd_add(c, dd_mul(a, b)) (_kernels.pyx:135-184): 4 DMUL + 3 DFMA + 43 DADD.
// ALGO_BLOCK_FAST runs the same tiles with the opt-in faithful sequence
// dd_madd_fast (15 FP64 instructions, within the north_star bound, NOT
// bit-identical to the reference).
// Tile configurations (n_min -> tile: capi.cu tile_for):
//   TILE_16    16x16 CTA tile, 1x1 per thread, 256 threads, 4 CTAs/SM
//   TILE_32    32x32, 2x2, 256 threads, 2 CTAs/SM, k-tiles of 16
//   TILE_LPT   persistent 64x64 (4x4) tiles in whole waves + 32x32 quarters
//   TILE_32x64 32x64, 2x4, 256 threads, 2 CTAs/SM (0.6-0.8 % faster than
//              TILE_32 in steady state -- fewer LDS per multiply-add --
//              but a coarser wave quantum: profiles/r02_tile_variants2.log)
//   TILE_64    64x64, 4x4, 256 threads, plain grid
#include "gemm.cuh"

// TILE_32's configuration can be overridden at build time (experiments:
// tools/exp/build_variant.py -DMPMM_DD32_CFG=i).
#if !defined(MPMM_DD32_CFG) || MPMM_DD32_CFG == 0
#define MPMM_DD32 32, 32, 16, 2, 2, 2
#elif MPMM_DD32_CFG == 1
#define MPMM_DD32 32, 32, 8, 2, 2, 2
#elif MPMM_DD32_CFG == 2
#define MPMM_DD32 32, 64, 8, 2, 4, 1
#elif MPMM_DD32_CFG == 3
#define MPMM_DD32 64, 32, 8, 4, 2, 1
#elif MPMM_DD32_CFG == 4
#define MPMM_DD32 32, 32, 16, 1, 4, 2
#elif MPMM_DD32_CFG == 5
#define MPMM_DD32 32, 32, 16, 4, 1, 2
#elif MPMM_DD32_CFG == 6
#define MPMM_DD32 32, 64, 8, 2, 4, 2
#endif

// TILE_LPT's configuration (experiments: -DMPMM_LPT_VAR=i)
#if !defined(MPMM_LPT_VAR) || MPMM_LPT_VAR == 0
#define MPMM_LPT_CFG 64, 64, 8, 4, 4, 1
#elif MPMM_LPT_VAR == 1
#define MPMM_LPT_CFG 64, 64, 8, 4, 4, 2
#elif MPMM_LPT_VAR == 2
#define MPMM_LPT_CFG 64, 64, 16, 4, 4, 2
#elif MPMM_LPT_VAR == 3
#define MPMM_LPT_CFG 64, 32, 8, 4, 2, 2
#elif MPMM_LPT_VAR == 4
#define MPMM_LPT_CFG 32, 64, 8, 2, 4, 2
#endif

namespace mpmm {

template <class Ops>
static cudaError_t dd_blocked(const GemmArgs& g) {
  switch (g.tile) {
    case TILE_16: return launch_tiled<Ops, 16, 16, 16, 1, 1, 4>(g);
    case TILE_32: return launch_tiled<Ops, MPMM_DD32>(g);
    case TILE_64: return launch_tiled<Ops, 64, 64, 8, 4, 4, 1>(g);
    case TILE_32x64: return launch_tiled<Ops, 32, 64, 8, 2, 4, 2>(g);
    case TILE_LPT: return launch_lpt<Ops, MPMM_LPT_CFG>(g);
    default: return cudaErrorInvalidValue;
  }
}

template <class Ops, int BM, int BN, int BK, int TM, int TN, int MINB>
static cudaError_t dd_geometry(Geometry* geo) {
  geo->bm = BM, geo->bn = BN;
  return occupancy_of(gemm_tiled<Ops, BM, BN, BK, TM, TN, MINB>, (BM / TM) * (BN / TN), geo);
}

template <class Ops>
static cudaError_t dd32_geometry(Geometry* geo) { return dd_geometry<Ops, MPMM_DD32>(geo); }

cudaError_t dd_gemm_launch(const GemmArgs& g) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.sprobs != nullptr) return launch_tiled_sum<DDOps, 32, 32, 16, 2, 2, 2>(g);
  if (g.algo == ALGO_SIMPLE) return launch_simple<DDOps>(g);
  if (g.algo == ALGO_BLOCK_FAST) return dd_blocked<DDFastOps>(g);
  return dd_blocked<DDOps>(g);
}

cudaError_t dd_dekker_launch(const GemmArgs& g) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.kready != nullptr) return cudaErrorNotSupported;
  return launch_persist<DDDekkerOps, 32, 32, 16, 2, 2, 2>(g);
}

cudaError_t dd_gemm_geometry(int algo, int tile, Geometry* geo) {
  if (algo == ALGO_BLOCK_FAST) {
    switch (tile) {
      case TILE_16: geo->bm = 16, geo->bn = 16;
        return occupancy_of(gemm_tiled<DDFastOps, 16, 16, 16, 1, 1, 4>, 256, geo);
      case TILE_32: return dd32_geometry<DDFastOps>(geo);
      case TILE_64: geo->bm = 64, geo->bn = 64;
        return occupancy_of(gemm_tiled<DDFastOps, 64, 64, 8, 4, 4, 1>, 256, geo);
      case TILE_32x64: geo->bm = 32, geo->bn = 64;
        return occupancy_of(gemm_tiled<DDFastOps, 32, 64, 8, 2, 4, 2>, 256, geo);
      case TILE_LPT: geo->bm = 64, geo->bn = 64;
        return occupancy_of(gemm_lpt<DDFastOps, MPMM_LPT_CFG>, 256, geo);
      default: return cudaErrorInvalidValue;
    }
  }
  if (algo == ALGO_SIMPLE) {
    geo->bm = 8, geo->bn = 32;
    return occupancy_of(gemm_simple<DDOps>, 256, geo);
  }
  switch (tile) {
    case TILE_16: geo->bm = 16, geo->bn = 16;
      return occupancy_of(gemm_tiled<DDOps, 16, 16, 16, 1, 1, 4>, 256, geo);
    case TILE_32: return dd32_geometry<DDOps>(geo);
    case TILE_64: geo->bm = 64, geo->bn = 64;
      return occupancy_of(gemm_tiled<DDOps, 64, 64, 8, 4, 4, 1>, 256, geo);
    case TILE_32x64: geo->bm = 32, geo->bn = 64;
      return occupancy_of(gemm_tiled<DDOps, 32, 64, 8, 2, 4, 2>, 256, geo);
    case TILE_LPT: geo->bm = 64, geo->bn = 64;
      return occupancy_of(gemm_lpt<DDOps, MPMM_LPT_CFG>, 256, geo);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mpmm
