// domain.cu -- the EFT-domain scan and the gated mirror launches (domain.cuh).
//
// One scan per product reads both operands once (HBM-bound: 16 B per DD
// element, 32 B per QD element, about 0.02 % of a 8192^3 DD product) and
// leaves six words in a per-stream device buffer.  The DFMA launch and the
// Dekker launch that follow both read them; exactly one computes.  The scan
// is self-cleaning (per-block partials, the last block reduces them and
// re-arms the counter), so a product costs no memset and no host sync.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "kernels.h"

namespace mpmm {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanMaxBlocks = 512;   // per operand

struct ScanBuf {
  int words[8];                          // domain words (6 used)
  unsigned counter;                      // blocks finished (re-armed to 0)
  int pad[7];
  int partial[2][kScanMaxBlocks][3];     // per operand, per block: max, 2047-min, nonfinite
};

struct Operand {
  const double* X;
  int64_t ld;      // in elements
  int rows, cols, comps;
};

__device__ __forceinline__ void fold(double x, int& mx, int& mn, int& nf) {
  const unsigned hi = static_cast<unsigned>(__double2hiint(x));
  const unsigned lo = static_cast<unsigned>(__double2loint(x));
  const int e = static_cast<int>((hi >> 20) & 0x7ffu);
  mx = max(mx, e);
  nf |= (e == 0x7ff);
  if (((hi & 0x7fffffffu) | lo) != 0u) mn = max(mn, 2047 - e);
}

__device__ __forceinline__ void scan_operand(const Operand& op, int& mx, int& mn, int& nf) {
  // the row of doubles is cols * comps long; comps is even, so it is a run
  // of double2 vectors
  const int64_t rowvec = (int64_t)op.cols * op.comps / 2;
  const double2* X = reinterpret_cast<const double2*>(op.X);
  const int64_t ldv = op.ld * op.comps / 2;
  if (op.ld == op.cols || op.rows == 1) {
    const int64_t total = (int64_t)op.rows * rowvec;
    const int64_t stride = (int64_t)gridDim.x * kScanThreads;
    int64_t v = (int64_t)blockIdx.x * kScanThreads + threadIdx.x;
    for (; v + 3 * stride < total; v += 4 * stride) {
      double2 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = __ldcs(X + v + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        fold(q[u].x, mx, mn, nf);
        fold(q[u].y, mx, mn, nf);
      }
    }
    for (; v < total; v += stride) {
      const double2 q = __ldcs(X + v);
      fold(q.x, mx, mn, nf);
      fold(q.y, mx, mn, nf);
    }
  } else {
    for (int64_t r = blockIdx.x; r < op.rows; r += gridDim.x)
      for (int64_t c = threadIdx.x; c < rowvec; c += kScanThreads) {
        const double2 q = __ldcs(X + r * ldv + c);
        fold(q.x, mx, mn, nf);
        fold(q.y, mx, mn, nf);
      }
  }
}

// blockIdx.y = 0 scans A, 1 scans B.  With a problem table (batched
// launches) every problem's A (or B) is folded into the same words.
__global__ void __launch_bounds__(kScanThreads)
domain_scan_kernel(Operand a, Operand b, const GemmProblem* probs, int batch, ScanBuf* buf) {
  int mx = 0, mn = 0, nf = 0;
  if (probs == nullptr) {
    scan_operand(blockIdx.y == 0 ? a : b, mx, mn, nf);
  } else {
    for (int p = 0; p < batch; ++p) {
      Operand op = blockIdx.y == 0 ? a : b;
      op.X = blockIdx.y == 0 ? probs[p].A : probs[p].B;
      op.ld = blockIdx.y == 0 ? probs[p].lda : probs[p].ldb;
      scan_operand(op, mx, mn, nf);
    }
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  mn = __reduce_max_sync(0xffffffffu, mn);
  nf = __reduce_or_sync(0xffffffffu, nf);
  __shared__ int red[3][kScanThreads / 32];
  __shared__ bool last;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    red[0][warp] = mx;
    red[1][warp] = mn;
    red[2][warp] = nf;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kScanThreads / 32; ++w) {
      mx = max(mx, red[0][w]);
      mn = max(mn, red[1][w]);
      nf |= red[2][w];
    }
    int* p = buf->partial[blockIdx.y][blockIdx.x];
    p[0] = mx;
    p[1] = mn;
    p[2] = nf;
    __threadfence();
    const unsigned done = atomicAdd(&buf->counter, 1u);
    last = (done == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!last) return;
  // the last block: reduce every block's partial, publish, re-arm
  __threadfence();
  for (int z = 0; z < 2; ++z) {
    int m0 = 0, m1 = 0, m2 = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += kScanThreads) {
      const volatile int* p = buf->partial[z][i];
      m0 = max(m0, p[0]);
      m1 = max(m1, p[1]);
      m2 |= p[2];
    }
    m0 = __reduce_max_sync(0xffffffffu, m0);
    m1 = __reduce_max_sync(0xffffffffu, m1);
    m2 = __reduce_or_sync(0xffffffffu, m2);
    __syncthreads();
    if (lane == 0) {
      red[0][warp] = m0;
      red[1][warp] = m1;
      red[2][warp] = m2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < kScanThreads / 32; ++w) {
        m0 = max(m0, red[0][w]);
        m1 = max(m1, red[1][w]);
        m2 |= red[2][w];
      }
      buf->words[3 * z + 0] = m0;
      buf->words[3 * z + 1] = m1;
      buf->words[3 * z + 2] = m2;
    }
  }
  if (threadIdx.x == 0) {
    buf->counter = 0u;
    __threadfence();
  }
}

// One scan buffer per (device, stream), created on first use and kept.
std::mutex g_mu;
std::map<std::pair<int, cudaStream_t>, ScanBuf*> g_bufs;

cudaError_t scan_buffer(cudaStream_t stream, ScanBuf** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_bufs.find({dev, stream});
  if (it != g_bufs.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  ScanBuf* b = nullptr;
  if ((e = cudaMalloc(reinterpret_cast<void**>(&b), sizeof(ScanBuf))) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b, 0, sizeof(ScanBuf), stream)) != cudaSuccess) {
    cudaFree(b);
    return e;
  }
  g_bufs[{dev, stream}] = b;
  *out = b;
  return cudaSuccess;
}

int scan_blocks(int64_t doubles) {
  int64_t per = (int64_t)kScanThreads * 2 * 8;   // >= 8 double2 per thread
  int64_t b = (doubles + per - 1) / per;
  return static_cast<int>(b < 1 ? 1 : (b > kScanMaxBlocks ? kScanMaxBlocks : b));
}

}  // namespace

cudaError_t domain_scan(int comps, const double* A, int64_t lda, int m, int l, const double* B,
                        int64_t ldb, int n, const int** words, cudaStream_t stream) {
  ScanBuf* buf = nullptr;
  cudaError_t e = scan_buffer(stream, &buf);
  if (e != cudaSuccess) return e;
  const Operand a{A, lda, m, l, comps}, b{B, ldb, l, n, comps};
  const int blocks = std::max(scan_blocks((int64_t)m * l * comps),
                              scan_blocks((int64_t)l * n * comps));
  domain_scan_kernel<<<dim3(blocks, 2), kScanThreads, 0, stream>>>(a, b, nullptr, 0, buf);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  *words = buf->words;
  return cudaSuccess;
}

cudaError_t domain_scan_batched(int comps, const GemmProblem* probs, int batch, int m, int l,
                                int n, const int** words, cudaStream_t stream) {
  ScanBuf* buf = nullptr;
  cudaError_t e = scan_buffer(stream, &buf);
  if (e != cudaSuccess) return e;
  const Operand a{nullptr, 0, m, l, comps}, b{nullptr, 0, l, n, comps};
  const int64_t per = std::max((int64_t)m * l, (int64_t)l * n) * comps * batch;
  domain_scan_kernel<<<dim3(scan_blocks(per), 2), kScanThreads, 0, stream>>>(a, b, probs,
                                                                             batch, buf);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  *words = buf->words;
  return cudaSuccess;
}

cudaError_t gemm_gated(int comps, GemmArgs g, const int* words) {
  g.gate.words = words;
  g.gate.want_unsafe = 0;
  cudaError_t e = comps == 2 ? dd_gemm_launch(g) : qd_gemm_launch(g);
  if (e != cudaSuccess) return e;
  g.gate.want_unsafe = 1;
  return comps == 2 ? dd_dekker_launch(g) : qd_dekker_launch(g);
}

cudaError_t gemm_checked(int comps, GemmArgs g, const int** words_out) {
  if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.algo == ALGO_BLOCK_FAST || g.kready != nullptr || g.l <= 0) {
    g.gate.words = nullptr;
    return comps == 2 ? dd_gemm_launch(g) : qd_gemm_launch(g);
  }
  if ((g.probs != nullptr || g.sprobs != nullptr) && g.gate.words != nullptr) {
    // batched problems the caller has scanned (e.g. Strassen leaves, whose
    // operands derive from one scanned pair; margins set by the caller)
    return gemm_gated(comps, g, g.gate.words);
  }
  if (g.sprobs != nullptr) return cudaErrorInvalidValue;   // the caller scans
  const int* words = nullptr;
  cudaError_t e = g.probs != nullptr
      ? domain_scan_batched(comps, g.probs, g.batch, g.m, g.l, g.n, &words, g.stream)
      : domain_scan(comps, g.A, g.lda, g.m, g.l, g.B, g.ldb, g.n, &words, g.stream);
  if (e != cudaSuccess) return e;
  if (words_out) *words_out = words;
  return gemm_gated(comps, g, words);
}

}  // namespace mpmm
