// peer.cpp -- B shared over peer memory instead of broadcast (one process
// per GPU): the alternative to the NCCL broadcast for the row-sharded
// product.
//
// The source rank allocates B's device buffer here (cudaMalloc, so the
// buffer is an allocation base and its IPC handle needs no offset) and
// exports a CUDA IPC handle; every other rank maps it (cudaIpcOpenMemHandle,
// peer access enabled lazily) and runs its ordinary GEMM launch with B's
// pointer in the source GPU's memory.  The kernel then pulls B's tiles over
// NVLink/NVSwitch as it consumes them -- the "broadcast" is fused into the
// GEMM's own operand loads, tile by tile, with no collective and no k-panel
// schedule.  Same kernels, same per-element operation order: the results
// are bitwise those of the NCCL path.  (Mapping memory of another process
// on the same device is legal too, which is how the one-GPU tests exercise
// it.)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/mpmm_cuda.h"

namespace mpmm {
int peer_fail(const char* where, cudaError_t e, std::string* err) {
  *err = std::string(where) + ": " + cudaGetErrorString(e);
  return MPMM_ERR_CUDA;
}
}  // namespace mpmm

namespace {
thread_local std::string g_peer_err;
}

extern "C" {

const char* mpmm_peer_last_error(void) { return g_peer_err.c_str(); }

int mpmm_ipc_alloc(int64_t bytes, const void* init, void** ptr, void* handle) {
  if (bytes <= 0 || ptr == nullptr || handle == nullptr) return MPMM_ERR_ARG;
  cudaError_t e = cudaMalloc(ptr, static_cast<size_t>(bytes));
  if (e != cudaSuccess) return mpmm::peer_fail("cudaMalloc", e, &g_peer_err);
  if (init != nullptr &&
      (e = cudaMemcpy(*ptr, init, static_cast<size_t>(bytes), cudaMemcpyDefault)) != cudaSuccess) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return mpmm::peer_fail("cudaMemcpy", e, &g_peer_err);
  }
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *ptr);
  if (e != cudaSuccess) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return mpmm::peer_fail("cudaIpcGetMemHandle", e, &g_peer_err);
  }
  std::memcpy(handle, &h, sizeof h);
  return MPMM_OK;
}

int mpmm_ipc_free(void* ptr) {
  if (ptr == nullptr) return MPMM_OK;
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? MPMM_OK : mpmm::peer_fail("cudaFree", e, &g_peer_err);
}

int mpmm_ipc_open(const void* handle, void** ptr) {
  if (handle == nullptr || ptr == nullptr) return MPMM_ERR_ARG;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? MPMM_OK : mpmm::peer_fail("cudaIpcOpenMemHandle", e, &g_peer_err);
}

int mpmm_ipc_close(void* ptr) {
  if (ptr == nullptr) return MPMM_OK;
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? MPMM_OK : mpmm::peer_fail("cudaIpcCloseMemHandle", e, &g_peer_err);
}

int mpmm_ipc_handle_size(void) { return static_cast<int>(sizeof(cudaIpcMemHandle_t)); }

}  // extern "C"
