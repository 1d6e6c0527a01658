// common.cuh -- shared helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace mpmm {

// 16-byte global->shared async copy (LDGSTS); when !valid the destination is
// zero-filled and the source is not read.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src_bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(src_bytes));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ bool finite2(double a, double b) {
  return isfinite(a) && isfinite(b);
}

}  // namespace mpmm
