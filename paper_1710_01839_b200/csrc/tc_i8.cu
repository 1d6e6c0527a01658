// tc_i8.cu -- residue GEMMs of the exact tensor mode on tcgen05 (sm_100a).
//
// For every modulus t: R_t = (A_t * B_t^T) mod p_t, A_t (m x k) and B_t
// (n x k) int8, K-major (k contiguous, row pitch kp, plane pitch m*kp /
// n*kp), R_t (m x n) uint8 row-major.  The int32 products are exact (k <=
// 131071) and never leave the SM: the accumulator lives in TMEM and the
// epilogue reduces it modulo p_t (one biased Barrett step) before the
// store, so the CRT combine reads one byte per modulus instead of four and
// skips the reduction.
//
// One CTA per 128 x BN output tile of one modulus (grid = n/BN x m/128 x
// N).  Warp 0 issues the TMA loads (128-byte swizzled K-major tiles, a
// 4-stage ring of mbarrier-tracked smem slots); warp 1 allocates TMEM and
// one elected thread issues tcgen05.mma.kind::i8 (M=128, N=BN, K=32, four
// per 128-byte k-block); warps 2-5 wait for the accumulator, tcgen05.ld
// their 32 TMEM lanes (= tile rows) 32 columns at a time, reduce and store.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "kernels.h"

namespace mpmm {

namespace {

__constant__ int kTcMods[54] = {
    256, 251, 243, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191,
    181, 179, 173, 169, 167, 163, 157, 151, 149, 139, 137, 131, 127, 125,
    121, 113, 109, 107, 103, 101, 97,  89,  83,  79,  73,  71,  67,  61,
    59,  53,  49,  47,  43,  41,  37,  31,  29,  23,  19,  17};

constexpr int BM = 128;        // tile rows (TMEM lanes)
constexpr int BK = 128;        // k bytes per stage (one 128-byte swizzle row)
constexpr int UK = 32;         // k per tcgen05.mma.kind::i8
constexpr int STAGES = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// K-major, 128-byte swizzle UMMA smem descriptor: rows of 128 bytes, 8-row
// groups 1024 bytes apart (SBO), LBO unused (1), version 1 (sm100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);          // start address
  d |= static_cast<uint64_t>(1) << 16;                         // LBO (unused)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;                 // SBO
  d |= static_cast<uint64_t>(1) << 46;                         // version
  d |= static_cast<uint64_t>(2) << 61;                         // SWIZZLE_128B
  return d;
}

// instruction descriptor: S32 accumulate, signed int8 A and B, both
// K-major, M = 128, N = BN
template <int BN>
__host__ __device__ constexpr uint32_t i8_idesc() {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(BM >> 4) << 24);
}

template <int BN>
struct TcSmem {
  alignas(1024) int8_t a[STAGES][BM * BK];
  alignas(1024) int8_t b[STAGES][BN * BK];
  uint64_t full[STAGES], empty[STAGES], acc_ready;
  uint32_t tmem_base;
};

template <int BN>
__global__ void __launch_bounds__(192, 1)
residue_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b, int kp, int np,
                    int64_t plane, uint8_t* __restrict__ R) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the swizzled tiles
  TcSmem<BN>& S = *reinterpret_cast<TcSmem<BN>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM, t = blockIdx.z;
  const int kblocks = kp / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);
    }
    mbar_init(&S.acc_ready, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {   // TMEM: BN int32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)),
                 "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    if (lane == 0) {   // TMA producer
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&S.empty[s], ((kb / STAGES) - 1) & 1);
        mbar_expect_tx(&S.full[s], (BM + BN) * BK);
        tma_load_3d(S.a[s], &map_a, &S.full[s], kb * BK, m0, t);
        tma_load_3d(S.b[s], &map_b, &S.full[s], kb * BK, n0, t);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer
      constexpr uint32_t idesc = i8_idesc<BN>();
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&S.full[s], (kb / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(S.a[s]), sb = smem_u32(S.b[s]);
#pragma unroll
        for (int k = 0; k < BK / UK; ++k) {
          const uint64_t da = sw128_desc(sa + k * UK), db = sw128_desc(sb + k * UK);
          const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        // free the slot when these MMAs have read it
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                         "r"(smem_u32(&S.empty[s]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                       "r"(smem_u32(&S.acc_ready))
                   : "memory");
    }
  } else {
    // epilogue: warps 2..5 -> TMEM lane groups (warp % 4) * 32
    const int q = warp & 3;
    mbar_wait(&S.acc_ready, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned p = static_cast<unsigned>(kTcMods[t]);
    const unsigned mu = static_cast<unsigned>((1ull << 32) / p);
    const unsigned bias = p * (2147483648u / p);
    const int row = m0 + q * 32 + lane;
    uint8_t* dst = R + static_cast<int64_t>(t) * plane + static_cast<int64_t>(row) * np + n0;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
          "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
          "[%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      uint32_t w[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        uint32_t packed = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned x = v[4 * e + u] + bias;           // g + p*floor(2^31/p) >= 0
          unsigned r = x - __umulhi(x, mu) * p;
          r = r >= p ? r - p : r;
          packed |= r << (8 * u);
        }
        w[e] = packed;
      }
      uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
      d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
      d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
  }
}

// Persistent variant: one CTA per SM walks the (modulus, row tile, column
// tile) space; two TMEM accumulators (2 x BN columns) let the epilogue of
// one tile overlap the MMAs of the next.  Barriers: full/empty per smem
// stage (TMA <-> MMA), tfull/tempty per accumulator (MMA <-> epilogue).
template <int BN>
struct TcSmemP {
  alignas(1024) int8_t a[STAGES][BM * BK];
  alignas(1024) int8_t b[STAGES][BN * BK];
  uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  uint32_t tmem_base;
};

template <int BN>
__global__ void __launch_bounds__(192, 1)
residue_gemm_persistent(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b, int kp, int mp, int np,
                        int batch, int64_t plane, uint8_t* __restrict__ R) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TcSmemP<BN>& S = *reinterpret_cast<TcSmemP<BN>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = kp / BK;
  const int tn = np / BN, tm = mp / BM;
  const int tiles = tn * tm * batch;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&S.tfull[a], 1);
      mbar_init(&S.tempty[a], 4);          // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)),
                 "n"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    if (lane == 0) {   // TMA producer
      int it = 0;      // global k-block counter (slot / phase)
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int t = tile / (tm * tn), rem = tile % (tm * tn);
        const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&S.empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_expect_tx(&S.full[s], (BM + BN) * BK);
          tma_load_3d(S.a[s], &map_a, &S.full[s], kb * BK, m0, t);
          tma_load_3d(S.b[s], &map_b, &S.full[s], kb * BK, n0, t);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer
      constexpr uint32_t idesc = i8_idesc<BN>();
      int it = 0, local = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
        const int acc_stage = local & 1;
        mbar_wait(&S.tempty[acc_stage], ((local >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc_stage * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&S.full[s], (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(S.a[s]), sb = smem_u32(S.b[s]);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
            const uint64_t da = sw128_desc(sa + k * UK), db = sw128_desc(sb + k * UK);
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  smem_u32(&S.empty[s]))
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&S.tfull[acc_stage]))
            : "memory");
      }
    }
  } else {
    const int q = warp & 3;
    int local = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      const int t = tile / (tm * tn), rem = tile % (tm * tn);
      const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;
      const int acc_stage = local & 1;
      mbar_wait(&S.tfull[acc_stage], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned p = static_cast<unsigned>(kTcMods[t]);
      const unsigned mu = static_cast<unsigned>((1ull << 32) / p);
      const unsigned bias = p * (2147483648u / p);
      const int row = m0 + q * 32 + lane;
      uint8_t* dst = R + static_cast<int64_t>(t) * plane + static_cast<int64_t>(row) * np + n0;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr =
            tmem + acc_stage * BN + (static_cast<uint32_t>(q * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
            "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
            "[%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
              "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
              "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t w[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t packed = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned x = v[4 * e + u] + bias;
            unsigned r = x - __umulhi(x, mu) * p;
            r = r >= p ? r - p : r;
            packed |= r << (8 * u);
          }
          w[e] = packed;
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
        d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
        d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
      // this accumulator may be overwritten by the next-but-one tile
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.tempty[acc_stage]))
                     : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(2 * BN));
  }
}

// Cluster-pair variant for large products: the two CTAs of a cluster work
// on row tiles 2i and 2i+1 of the same column tile, so they share its B
// tile -- each loads one half (128 rows) by TMA multicast into both CTAs'
// smem, halving the B traffic from L2.  A slot is free again only when
// both CTAs' MMAs have read it: every MMA warp commits to the empty
// barrier of BOTH CTAs (arrival count 2).
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c0, int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "h"(mask)
      : "memory");
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
residue_gemm_pair(const __grid_constant__ CUtensorMap map_a,
                  const __grid_constant__ CUtensorMap map_bh, int kp, int mp, int np, int batch,
                  int64_t plane, uint8_t* __restrict__ R) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TcSmemP<BN>& S = *reinterpret_cast<TcSmemP<BN>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = static_cast<int>(cluster_rank());
  const int kblocks = kp / BK;
  const int tn = np / BN, tmp = mp / (2 * BM);          // row-tile pairs
  const int pairs = tn * tmp * batch;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 2);           // both CTAs' MMAs
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&S.tfull[a], 1);
      mbar_init(&S.tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)),
                 "n"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();                       // the peer's barriers exist before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    if (lane == 0) {   // TMA producer: own A tile, one half of the shared B tile
      int it = 0;
      for (int pr = cluster; pr < pairs; pr += nclusters) {
        const int t = pr / (tmp * tn), rem = pr % (tmp * tn);
        const int m0 = ((rem / tn) * 2 + rank) * BM, n0 = (rem % tn) * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&S.empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_expect_tx(&S.full[s], (BM + BN) * BK);
          tma_load_3d(S.a[s], &map_a, &S.full[s], kb * BK, m0, t);
          tma_load_3d_mc(S.b[s] + rank * (BN / 2) * BK, &map_bh, &S.full[s], kb * BK,
                         n0 + rank * (BN / 2), t, 0x3);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer
      constexpr uint32_t idesc = i8_idesc<BN>();
      int it = 0, local = 0;
      for (int pr = cluster; pr < pairs; pr += nclusters, ++local) {
        const int acc_stage = local & 1;
        mbar_wait(&S.tempty[acc_stage], ((local >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc_stage * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&S.full[s], (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(S.a[s]), sb = smem_u32(S.b[s]);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
            const uint64_t da = sw128_desc(sa + k * UK), db = sw128_desc(sb + k * UK);
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          // slot s is free for the producer of either CTA once both have read it
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster"
              ".multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&S.empty[s])),
              "h"(static_cast<uint16_t>(0x3))
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&S.tfull[acc_stage]))
            : "memory");
      }
    }
  } else {
    const int q = warp & 3;
    int local = 0;
    for (int pr = cluster; pr < pairs; pr += nclusters, ++local) {
      const int t = pr / (tmp * tn), rem = pr % (tmp * tn);
      const int m0 = ((rem / tn) * 2 + rank) * BM, n0 = (rem % tn) * BN;
      const int acc_stage = local & 1;
      mbar_wait(&S.tfull[acc_stage], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned p = static_cast<unsigned>(kTcMods[t]);
      const unsigned mu = static_cast<unsigned>((1ull << 32) / p);
      const unsigned bias = p * (2147483648u / p);
      const int row = m0 + q * 32 + lane;
      uint8_t* dst = R + static_cast<int64_t>(t) * plane + static_cast<int64_t>(row) * np + n0;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr =
            tmem + acc_stage * BN + (static_cast<uint32_t>(q * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
            "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
            "[%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
              "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
              "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t w[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t packed = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned x = v[4 * e + u] + bias;
            unsigned r = x - __umulhi(x, mu) * p;
            r = r >= p ? r - p : r;
            packed |= r << (8 * u);
          }
          w[e] = packed;
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
        d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
        d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.tempty[acc_stage]))
                     : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();                       // no CTA leaves while the peer may still signal it
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(2 * BN));
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 3-D int8 map: (k, rows, planes), box (BK, box_rows, 1), 128-byte swizzle
bool make_map(CUtensorMap* map, const int8_t* base, int64_t kp, int64_t rows, int64_t planes,
              int box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kp), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(planes)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(kp),
                                 static_cast<cuuint64_t>(kp * rows)};
  const cuuint32_t box[3] = {BK, static_cast<cuuint32_t>(box_rows), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

}  // namespace

constexpr int kTcBN = 256;

// Shape requirements: m % 128 == 0, n % kTcBN == 0, k % 128 == 0.
bool tc_residue_gemm_supported(int64_t m, int64_t n, int64_t k) {
  return m > 0 && n > 0 && k > 0 && m % BM == 0 && n % kTcBN == 0 && k % BK == 0 &&
         k <= 131071 && encode_fn() != nullptr;
}

int tc_residue_gemm_tile_n() { return kTcBN; }

cudaError_t tc_residue_gemm(int64_t m, int64_t n, int64_t k, int batch, const int8_t* A,
                            const int8_t* Bt, uint8_t* R, cudaStream_t s) {
  if (!tc_residue_gemm_supported(m, n, k) || batch < 1 || batch > 54)
    return cudaErrorInvalidValue;
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, k, m, batch, BM) || !make_map(&mb, Bt, k, n, batch, kTcBN))
    return cudaErrorInvalidValue;
  static const int variant = [] {   // 0 tile, 1 persistent, 2 cluster pair (measurement knob)
    const char* env = std::getenv("MPMM_TC_KERNEL");
    if (env == nullptr) return -1;
    return env[0] == 't' ? 0 : (env[0] == 'p' && env[1] == 'e' ? 1 : 2);
  }();
  // pairs need an even number of 128-row tiles; they pay off on large planes
  const bool pair_ok = (m / BM) % 2 == 0;
  const int use = variant >= 0 ? (variant == 2 && !pair_ok ? 1 : variant)
                               : (pair_ok && m * n * k >= (int64_t{1} << 33) ? 2 : 1);
  if (use == 2) {
    CUtensorMap mbh;
    if (!make_map(&mbh, Bt, k, n, batch, kTcBN / 2)) return cudaErrorInvalidValue;
    const size_t smem = sizeof(TcSmemP<kTcBN>) + 1024;
    auto kern = residue_gemm_pair<kTcBN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
      return e;
    const int64_t pairs = (m / (2 * BM)) * (n / kTcBN) * batch;
    int64_t clusters = sms / 2;
    if (pairs < clusters) clusters = pairs;
    kern<<<static_cast<unsigned>(2 * clusters), 192, smem, s>>>(
        ma, mbh, static_cast<int>(k), static_cast<int>(m), static_cast<int>(n), batch, m * n, R);
    return cudaGetLastError();
  }
  if (use == 0) {
    const size_t smem = sizeof(TcSmem<kTcBN>) + 1024;
    auto kern = residue_gemm_kernel<kTcBN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(static_cast<unsigned>(n / kTcBN), static_cast<unsigned>(m / BM),
              static_cast<unsigned>(batch));
    kern<<<grid, 192, smem, s>>>(ma, mb, static_cast<int>(k), static_cast<int>(n), m * n, R);
    return cudaGetLastError();
  }
  const size_t smem = sizeof(TcSmemP<kTcBN>) + 1024;
  auto kern = residue_gemm_persistent<kTcBN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
    return e;
  const int64_t tiles = (m / BM) * (n / kTcBN) * batch;
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  kern<<<grid, 192, smem, s>>>(ma, mb, static_cast<int>(k), static_cast<int>(m),
                               static_cast<int>(n), batch, m * n, R);
  return cudaGetLastError();
}

}  // namespace mpmm
