// runtime.cpp -- the single-process multi-GPU runtime behind mpmm_init /
// mpmm_gemm_multi / mpmm_finalize.
//
// The reference partitions C's rows over a thread pool
// (pkg/src/mpmm/multiply.py:86-112, :134-160).  Lifted to devices: the
// runtime owns, per GPU, a compute stream, a communication stream and an
// NCCL communicator (ncclCommInitAll over the chosen devices).  For
// C = A*B from host buffers, GPU g owns a contiguous block of C's rows
// (aligned to the 64-row CTA tile); its rows of A go straight from the
// host to it; B goes host -> GPU 0 once and is broadcast by NCCL over
// NVLink in k-panels on the communication streams while the compute
// streams accumulate each landed panel.  There is no reduction: every C
// element has one owner and an ascending k order, so results are bitwise
// identical for any GPU count and any panel split.  Strassen shards run a
// rectangular Strassen on their rows once all of B has landed.
//
// Torch-free: this is what a C/C++ caller of the reference protocol uses.
// The Python package's own multi-GPU path (shard.py) is one process per
// GPU over torch.distributed; both keep the same row/panel geometry.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "trace.h"
#include "kernels.h"

namespace mpmm {

cudaError_t strassen_run(int comps, int64_t cutoff, int tile, int64_t m, int64_t l, int64_t n,
                         const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int64_t* stats, cudaStream_t stream);

namespace {

// NCCL is bound at mpmm_init time, not at link time: a process that also
// hosts PyTorch must use the NCCL build torch loaded (same soname, newer
// symbols), so an already-loaded libnccl.so.2 wins, then MPMM_NCCL_LIB,
// then the default search path.
struct Nccl {
  bool ok = false;
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};
Nccl g_nccl;

bool load_nccl(std::string* err) {
  if (g_nccl.ok) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) {
    if (const char* env = std::getenv("MPMM_NCCL_LIB")) h = dlopen(env, RTLD_NOW);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) {
    *err = std::string("cannot load NCCL (libnccl.so.2): ") + dlerror();
    return false;
  }
  auto sym = [&](const char* name) { return dlsym(h, name); };
  g_nccl.commInitAll = reinterpret_cast<decltype(g_nccl.commInitAll)>(sym("ncclCommInitAll"));
  g_nccl.commDestroy = reinterpret_cast<decltype(g_nccl.commDestroy)>(sym("ncclCommDestroy"));
  g_nccl.broadcast = reinterpret_cast<decltype(g_nccl.broadcast)>(sym("ncclBroadcast"));
  g_nccl.groupStart = reinterpret_cast<decltype(g_nccl.groupStart)>(sym("ncclGroupStart"));
  g_nccl.groupEnd = reinterpret_cast<decltype(g_nccl.groupEnd)>(sym("ncclGroupEnd"));
  g_nccl.errorString = reinterpret_cast<decltype(g_nccl.errorString)>(sym("ncclGetErrorString"));
  if (!g_nccl.commInitAll || !g_nccl.commDestroy || !g_nccl.broadcast || !g_nccl.groupStart ||
      !g_nccl.groupEnd || !g_nccl.errorString) {
    *err = "libnccl.so.2 lacks a required symbol";
    return false;
  }
  g_nccl.ok = true;
  return true;
}

struct Gpu {
  int id = -1;
  cudaStream_t comp = nullptr, comm = nullptr;
  ncclComm_t nccl = nullptr;
};

std::mutex g_mu;
std::vector<Gpu> g_gpus;

struct DeviceGuard {
  int prev = 0;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

int cuda_err(cudaError_t e, const char* where, std::string* err) {
  *err = std::string(where) + ": " + cudaGetErrorString(e);
  return 2;
}

int nccl_err(ncclResult_t r, const char* where, std::string* err) {
  *err = std::string(where) + ": " + g_nccl.errorString(r);
  return 2;
}

#define RT_CU(call)                                    \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return cuda_err(_e, #call, err); \
  } while (0)
#define RT_NC(call)                                    \
  do {                                                 \
    ncclResult_t _r = (call);                          \
    if (_r != ncclSuccess) return nccl_err(_r, #call, err); \
  } while (0)

void destroy_all() {
  for (Gpu& g : g_gpus) {
    cudaSetDevice(g.id);
    if (g.nccl) g_nccl.commDestroy(g.nccl);
    if (g.comp) cudaStreamDestroy(g.comp);
    if (g.comm) cudaStreamDestroy(g.comm);
  }
  g_gpus.clear();
}

}  // namespace

int rt_init(const int* devs, int ndev, std::string* err) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_gpus.empty()) {
    *err = "runtime already initialized (call mpmm_finalize first)";
    return 1;
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    *err = "no CUDA device";
    return 3;
  }
  std::vector<int> ids;
  if (devs == nullptr) {
    for (int g = 0; g < ndev; ++g) ids.push_back(g);
  } else {
    ids.assign(devs, devs + ndev);
  }
  if (ndev < 1 || ndev > count) {
    *err = "ngpus must be in 1.." + std::to_string(count);
    return 1;
  }
  for (size_t q = 0; q < ids.size(); ++q) {
    if (ids[q] < 0 || ids[q] >= count ||
        std::count(ids.begin(), ids.end(), ids[q]) != 1) {
      *err = "device list must name distinct visible devices";
      return 1;
    }
  }
  if (!load_nccl(err)) return 2;
  DeviceGuard guard;
  std::vector<ncclComm_t> comms(ndev);
  RT_NC(g_nccl.commInitAll(comms.data(), ndev, ids.data()));
  g_gpus.resize(ndev);
  for (int g = 0; g < ndev; ++g) {
    g_gpus[g].id = ids[g];
    g_gpus[g].nccl = comms[g];
    cudaError_t e = cudaSetDevice(ids[g]);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g_gpus[g].comp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g_gpus[g].comm, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      destroy_all();
      return cuda_err(e, "runtime stream setup", err);
    }
  }
  return 0;
}

int rt_finalize() {
  std::lock_guard<std::mutex> lock(g_mu);
  DeviceGuard guard;
  destroy_all();
  return 0;
}

int rt_gpus(int* ids, int cap) {
  std::lock_guard<std::mutex> lock(g_mu);
  for (int g = 0; g < static_cast<int>(g_gpus.size()) && g < cap; ++g) ids[g] = g_gpus[g].id;
  return static_cast<int>(g_gpus.size());
}

}  // namespace mpmm

// The schedule of mpmm_gemm_multi, torch-free and GPU-free (so the host
// logic is testable on CPU): GPU g owns C rows [rows[2g], rows[2g+1]) --
// ceil(m / G) rounded up to the 64-row CTA tile, trailing GPUs possibly
// empty --, and B travels in `*npanels` k-panels [kb[p], kb[p+1]).
// panels <= 0: automatic (8 from l >= 1024, l/128 from 256, else 1).
extern "C" int mpmm_multi_plan(int64_t m, int64_t l, int ngpus, int64_t panels, int64_t* rows,
                               int64_t* kb, int* npanels) {
  if (m < 0 || l < 0 || ngpus < 1 || rows == nullptr || kb == nullptr || npanels == nullptr)
    return 1;
  int64_t per = (m + ngpus - 1) / ngpus;
  per = ((per + 63) / 64) * 64;
  for (int g = 0; g < ngpus; ++g) {
    rows[2 * g] = std::min(m, per * g);
    rows[2 * g + 1] = std::min(m, per * (g + 1));
  }
  if (panels < 1) panels = l >= 1024 ? 8 : (l >= 256 ? l / 128 : 1);
  panels = std::max<int64_t>(1, std::min<int64_t>(panels, std::max<int64_t>(l, 1)));
  const int64_t step = l > 0 ? (l + panels - 1) / panels : 1;
  const int P = l > 0 ? static_cast<int>((l + step - 1) / step) : 0;
  for (int p = 0; p <= P; ++p) kb[p] = std::min(l, p * step);
  *npanels = P;
  return 0;
}

namespace mpmm {

int rt_gemm_host(int comps, int algo, int tile, int64_t cutoff, int64_t m, int64_t l, int64_t n,
                 const double* a, const double* b, double* c, int* nonfinite, double* device_ms,
                 int64_t panels, std::string* err) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_gpus.empty()) {
    *err = "runtime not initialized (call mpmm_init)";
    return 1;
  }
  if (nonfinite) *nonfinite = 0;
  if (device_ms) *device_ms = 0.0;
  if (m == 0 || n == 0) return 0;
  DeviceGuard guard;
  const int G = static_cast<int>(g_gpus.size());
  const size_t el = comps * sizeof(double);
  // the schedule (row blocks, k-panels): mpmm_multi_plan
  std::vector<int64_t> plan_rows(2 * G), kb(static_cast<size_t>(std::max<int64_t>(l, 1)) + 2);
  int P = 0;
  if (mpmm_multi_plan(m, l, G, panels, plan_rows.data(), kb.data(), &P) != 0) {
    *err = "bad multi-GPU plan request";
    return 1;
  }
  const bool strassen = algo == 3;

  struct Shard {
    int64_t r0 = 0, r1 = 0;
    double *A = nullptr, *B = nullptr, *C = nullptr;
    int* flag = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr, ready = nullptr;
    std::vector<cudaEvent_t> landed;
  };
  std::vector<Shard> sh(G);
  auto cleanup = [&]() {
    for (int g = 0; g < G; ++g) {
      cudaSetDevice(g_gpus[g].id);
      Shard& s = sh[g];
      for (void* p : {static_cast<void*>(s.A), static_cast<void*>(s.B), static_cast<void*>(s.C),
                      static_cast<void*>(s.flag)})
        if (p) cudaFreeAsync(p, g_gpus[g].comp);
      for (cudaEvent_t e : s.landed) cudaEventDestroy(e);
      if (s.t0) cudaEventDestroy(s.t0);
      if (s.t1) cudaEventDestroy(s.t1);
      if (s.ready) cudaEventDestroy(s.ready);
      cudaStreamSynchronize(g_gpus[g].comp);
    }
  };
  int rc = 0;
  auto body = [&]() -> int {
    // allocation, timing start, A rows
    for (int g = 0; g < G; ++g) {
      Gpu& d = g_gpus[g];
      Shard& s = sh[g];
      RT_CU(cudaSetDevice(d.id));
      s.r0 = plan_rows[2 * g];
      s.r1 = plan_rows[2 * g + 1];
      const int64_t rows = s.r1 - s.r0;
      RT_CU(cudaEventCreate(&s.t0));
      RT_CU(cudaEventCreate(&s.t1));
      RT_CU(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
      RT_CU(cudaEventRecord(s.t0, d.comp));
      RT_CU(cudaMallocAsync(reinterpret_cast<void**>(&s.A), std::max<size_t>(rows * l * el, el),
                            d.comp));
      RT_CU(cudaMallocAsync(reinterpret_cast<void**>(&s.B), std::max<size_t>(l * n * el, el),
                            d.comp));
      RT_CU(cudaMallocAsync(reinterpret_cast<void**>(&s.C), std::max<size_t>(rows * n * el, el),
                            d.comp));
      RT_CU(cudaMallocAsync(reinterpret_cast<void**>(&s.flag), sizeof(int), d.comp));
      RT_CU(cudaMemsetAsync(s.flag, 0, sizeof(int), d.comp));
      RT_CU(cudaEventRecord(s.ready, d.comp));
      RT_CU(cudaStreamWaitEvent(d.comm, s.ready, 0));
      s.landed.resize(P, nullptr);
      for (int p = 0; p < P; ++p)
        RT_CU(cudaEventCreateWithFlags(&s.landed[p], cudaEventDisableTiming));
    }
    // k-panels: A columns and (on GPU 0) B rows from the host, B broadcast
    for (int p = 0; p < P; ++p) {
      const int64_t k0 = kb[p], k1 = kb[p + 1];
      for (int g = 0; g < G; ++g) {
        Gpu& d = g_gpus[g];
        Shard& s = sh[g];
        RT_CU(cudaSetDevice(d.id));
        const int64_t rows = s.r1 - s.r0;
        if (rows > 0)
          RT_CU(cudaMemcpy2DAsync(s.A + k0 * comps, l * el, a + (s.r0 * l + k0) * comps, l * el,
                                  (k1 - k0) * el, rows, cudaMemcpyHostToDevice, d.comm));
        if (g == 0)
          RT_CU(cudaMemcpyAsync(s.B + k0 * n * comps, b + k0 * n * comps, (k1 - k0) * n * el,
                                cudaMemcpyHostToDevice, d.comm));
      }
      if (G > 1) {
        TraceRange trace_("runtime: ncclBroadcast of a B k-panel");
        RT_NC(g_nccl.groupStart());
        for (int g = 0; g < G; ++g) {
          RT_CU(cudaSetDevice(g_gpus[g].id));
          RT_NC(g_nccl.broadcast(sh[0].B + k0 * n * comps, sh[g].B + k0 * n * comps,
                              static_cast<size_t>((k1 - k0) * n * comps), ncclDouble, 0,
                              g_gpus[g].nccl, g_gpus[g].comm));
        }
        RT_NC(g_nccl.groupEnd());
      }
      for (int g = 0; g < G; ++g) {
        Gpu& d = g_gpus[g];
        Shard& s = sh[g];
        RT_CU(cudaSetDevice(d.id));
        RT_CU(cudaEventRecord(s.landed[p], d.comm));
        if (strassen) continue;
        const int64_t rows = s.r1 - s.r0;
        if (rows == 0) continue;
        RT_CU(cudaStreamWaitEvent(d.comp, s.landed[p], 0));
        const bool last = (p == P - 1);
        GemmArgs ga{algo, tile, (int)rows, (int)n, (int)(k1 - k0), s.A + k0 * comps, l,
                    s.B + k0 * n * comps, n, s.C, n, p > 0 ? 1 : 0, last ? s.flag : nullptr,
                    d.comp};
        // per panel: domain scan of its operands, then the gated DFMA /
        // Dekker launches (domain.cuh)
        RT_CU(gemm_checked(comps, ga));
      }
    }
    for (int g = 0; g < G; ++g) {
      Gpu& d = g_gpus[g];
      Shard& s = sh[g];
      RT_CU(cudaSetDevice(d.id));
      const int64_t rows = s.r1 - s.r0;
      // every panel landed (also orders the comm stream's use of the
      // buffers before their stream-ordered free on comp)
      if (P > 0) RT_CU(cudaStreamWaitEvent(d.comp, s.landed[P - 1], 0));
      if (rows == 0) {
        RT_CU(cudaEventRecord(s.t1, d.comp));
        continue;
      }
      if (P == 0 || strassen) {
        if (strassen) {
          RT_CU(strassen_run(comps, cutoff, tile, rows, l, n, s.A, l, s.B, n, s.C, n, nullptr,
                             d.comp));
        } else {   // l == 0: C = 0
          GemmArgs ga{algo, tile, (int)rows, (int)n, 0, s.A, l, s.B, n, s.C, n, 0, nullptr,
                      d.comp};
          RT_CU(comps == 2 ? dd_gemm_launch(ga) : qd_gemm_launch(ga));
        }
        RT_CU(nonfinite_launch(comps, s.C, n, (int)rows, (int)n, s.flag, d.comp));
      }
      RT_CU(cudaMemcpyAsync(c + s.r0 * n * comps, s.C, rows * n * el, cudaMemcpyDeviceToHost,
                            d.comp));
      RT_CU(cudaEventRecord(s.t1, d.comp));
    }
    float worst = 0.f;
    for (int g = 0; g < G; ++g) {
      Gpu& d = g_gpus[g];
      Shard& s = sh[g];
      RT_CU(cudaSetDevice(d.id));
      RT_CU(cudaEventSynchronize(s.t1));
      float ms = 0.f;
      RT_CU(cudaEventElapsedTime(&ms, s.t0, s.t1));
      worst = std::max(worst, ms);
      int f = 0;
      RT_CU(cudaMemcpy(&f, s.flag, sizeof(int), cudaMemcpyDeviceToHost));
      if (nonfinite && f) *nonfinite = 1;
    }
    if (device_ms) *device_ms = worst;
    return 0;
  };
  rc = body();
  cleanup();
  return rc;
}

}  // namespace mpmm
