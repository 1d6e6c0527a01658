// gemm_dd.cu -- double-double instantiations of gemm.cuh.
//
// DD element = one double2 {hi, lo}; each multiply-add is the reference's
// dd_add(c, dd_mul(a, b)) (_kernels.pyx:135-184): 4 DMUL + 3 DFMA + 43 DADD.
// ALGO_BLOCK_FAST runs the same tiles with the opt-in faithful sequence
// dd_madd_fast (15 FP64 instructions, within the north_star bound, NOT
// bit-identical to the reference).
// Tile configurations (n_min -> tile: capi.cu tile_for; measured in
// profiles/r02_interior_probe.log, all bitwise equal):
//   TILE_16    16x16 CTA tile, 1x1 per thread, 256 threads, 4 CTAs/SM
//   TILE_32    32x32, 2x4 per thread, 128 threads, 4 CTAs/SM, k-tiles of 16
//              (the finest wave quantum: best at 1024^3; 0.2 % behind
//              TILE_32x64 at 8192^3)
//   TILE_LPT   persistent 64x64 (4x4) tiles in whole waves + 32x32 quarters
//   TILE_32x64 32x64, 2x4, 256 threads, 2 CTAs/SM, k-tiles of 16 (fastest in
//              steady state: 0.512 of the FP64 roofline at 8192^3)
//   TILE_64    64x64, 4x4, 256 threads, 1 CTA/SM, plain grid
// 2x4 register tiles are the sweet spot: 0.75 operand fetches per
// multiply-add at 16 warps per SM; 2x2 needs 1.0, and 4x4 / 2x8 (0.5 /
// 0.625) only fit 8-12 warps per SM and lose more to latency than they save.
#include "gemm.cuh"

// Experiments select another set at build time (tools/exp/build_variant.py
// -DMPMM_DDCFG=i; nvcc splits -D values at commas, hence the index).
#if defined(MPMM_DDCFG) && MPMM_DDCFG == 1
#define MPMM_DD32 32, 32, 32, 2, 2, 2
#define MPMM_DD32x64 32, 64, 8, 2, 4, 2
#define MPMM_DD64 64, 64, 16, 4, 4, 1
#elif defined(MPMM_DDCFG) && MPMM_DDCFG == 3   // 128-thread CTAs, four per SM
#define MPMM_DD32 32, 32, 16, 2, 4, 4
#define MPMM_DD32x64 16, 64, 16, 2, 4, 4
#define MPMM_DD64 32, 32, 32, 2, 4, 4
#elif defined(MPMM_DDCFG) && MPMM_DDCFG == 4   // 2x8 / 4x4 register tiles, 128 threads
#define MPMM_DD32 32, 64, 16, 2, 8, 3
#define MPMM_DD32x64 64, 32, 16, 4, 4, 2
#define MPMM_DD64 64, 32, 16, 4, 4, 3
#elif defined(MPMM_DDCFG) && MPMM_DDCFG == 5   // more warps per SM at fewer registers
#define MPMM_DD32 32, 32, 16, 2, 4, 5
#define MPMM_DD32x64 32, 32, 16, 2, 4, 6
#define MPMM_DD64 32, 32, 16, 2, 2, 6
#elif defined(MPMM_DDCFG) && MPMM_DDCFG == 2
#define MPMM_DD32 64, 32, 16, 4, 2, 2
#define MPMM_DD32x64 32, 64, 32, 2, 4, 2
#define MPMM_DD64 64, 64, 32, 4, 4, 1
#endif
#ifndef MPMM_DD16
#define MPMM_DD16 16, 16, 16, 1, 1, 4
#endif
#ifndef MPMM_DD32
#define MPMM_DD32 32, 32, 16, 2, 4, 4
#endif
#ifndef MPMM_DD64
#define MPMM_DD64 64, 64, 8, 4, 4, 1
#endif
#ifndef MPMM_DD32x64
#define MPMM_DD32x64 32, 64, 16, 2, 4, 2
#endif
#ifndef MPMM_DDLPT
#define MPMM_DDLPT 64, 64, 8, 4, 4, 1
#endif

namespace mpmm {

template <class Ops>
static cudaError_t dd_blocked(const GemmArgs& g) {
  switch (g.tile) {
    case TILE_16: return launch_tiled<Ops, MPMM_DD16>(g);
    case TILE_32: return launch_tiled<Ops, MPMM_DD32>(g);
    case TILE_64: return launch_tiled<Ops, MPMM_DD64>(g);
    case TILE_32x64: return launch_tiled<Ops, MPMM_DD32x64>(g);
    case TILE_LPT: return launch_lpt<Ops, MPMM_DDLPT>(g);
    default: return cudaErrorInvalidValue;
  }
}

template <class Ops>
static cudaError_t dd_blocked_geometry(int tile, Geometry* geo) {
  switch (tile) {
    case TILE_16: return tiled_geometry<Ops, MPMM_DD16>(geo);
    case TILE_32: return tiled_geometry<Ops, MPMM_DD32>(geo);
    case TILE_64: return tiled_geometry<Ops, MPMM_DD64>(geo);
    case TILE_32x64: return tiled_geometry<Ops, MPMM_DD32x64>(geo);
    case TILE_LPT: return lpt_geometry<Ops, MPMM_DDLPT>(geo);
    default: return cudaErrorInvalidValue;
  }
}

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
  if (algo == ALGO_SIMPLE) {
    geo->bm = 8, geo->bn = 32;
    return occupancy_of(gemm_simple<DDOps>, 256, geo);
  }
  if (algo == ALGO_BLOCK_FAST) return dd_blocked_geometry<DDFastOps>(tile, geo);
  return dd_blocked_geometry<DDOps>(tile, geo);
}

}  // namespace mpmm
