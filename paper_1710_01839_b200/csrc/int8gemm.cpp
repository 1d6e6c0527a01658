// int8gemm.cpp -- batched exact int8 x int8 -> int32 GEMM through cuBLASLt.
//
// The integer tensor-core products of the exact ("tensor") mode
// (ozaki.cu): one plain library GEMM per CRT modulus, batched.  For batch
// t: C_t (m x n, row-major int32) = A_t (m x k, row-major int8) *
// B_t^T, with B_t stored (n x k, row-major int8) so both operands have k
// contiguous -- cuBLASLt's "TN" integer layout.  int8 products summed in
// int32 are exact while k * 128^2 < 2^31 (k <= 131071; checked).
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <tuple>

namespace mpmm {

namespace {

thread_local cublasLtHandle_t g_lt = nullptr;
thread_local int g_lt_device = -1;
// heuristic picks per (device, m, n, k, batch, workspace): the query costs
// tens of microseconds, the product of a 1024^3 DD call about 45
using AlgoKey = std::tuple<int, int64_t, int64_t, int64_t, int64_t, size_t>;
thread_local std::map<AlgoKey, cublasLtMatmulAlgo_t> g_algos;

}  // namespace

// Returns 0 on success; on failure writes a message into *err.
int int8_gemm_batched(int64_t m, int64_t n, int64_t k, int64_t batch, const int8_t* A,
                      const int8_t* Bt, int32_t* C, void* workspace, size_t ws_size,
                      cudaStream_t stream, std::string* err) {
  if (m <= 0 || n <= 0 || batch <= 0) return 0;
  if (k > 131071) {
    *err = "int8 GEMM inner dimension too large for exact int32 accumulation";
    return 1;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_lt == nullptr || g_lt_device != dev) {
    g_algos.clear();
    if (cublasLtCreate(&g_lt) != CUBLAS_STATUS_SUCCESS) {
      *err = "cublasLtCreate failed";
      return 2;
    }
    g_lt_device = dev;
  }
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  auto cleanup = [&]() {
    if (pref) cublasLtMatmulPreferenceDestroy(pref);
    if (la) cublasLtMatrixLayoutDestroy(la);
    if (lb) cublasLtMatrixLayoutDestroy(lb);
    if (lc) cublasLtMatrixLayoutDestroy(lc);
    if (op) cublasLtMatmulDescDestroy(op);
  };
  auto bad = [&](const char* what) {
    *err = std::string("cuBLASLt: ") + what;
    cleanup();
    return 2;
  };
  if (cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32I, CUDA_R_32I) != CUBLAS_STATUS_SUCCESS)
    return bad("matmul desc");
  cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof ta);
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof tb);
  // column-major views: first operand = Bt as (k x n), second = A as (k x m),
  // D = (n x m) column-major == C (m x n) row-major
  if (cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, k, n, k) != CUBLAS_STATUS_SUCCESS ||
      cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, k, m, k) != CUBLAS_STATUS_SUCCESS ||
      cublasLtMatrixLayoutCreate(&lc, CUDA_R_32I, n, m, n) != CUBLAS_STATUS_SUCCESS)
    return bad("layouts");
  int32_t nb = static_cast<int32_t>(batch);
  int64_t sa = n * k, sb = m * k, sc = m * n;
  cublasLtMatrixLayoutSetAttribute(la, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &nb, sizeof nb);
  cublasLtMatrixLayoutSetAttribute(lb, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &nb, sizeof nb);
  cublasLtMatrixLayoutSetAttribute(lc, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &nb, sizeof nb);
  cublasLtMatrixLayoutSetAttribute(la, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sa, sizeof sa);
  cublasLtMatrixLayoutSetAttribute(lb, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sb, sizeof sb);
  cublasLtMatrixLayoutSetAttribute(lc, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sc, sizeof sc);
  if (cublasLtMatmulPreferenceCreate(&pref) != CUBLAS_STATUS_SUCCESS) return bad("preference");
  uint64_t wss = ws_size;
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wss,
                                       sizeof wss);
  const AlgoKey key{dev, m, n, k, batch, ws_size};
  auto it = g_algos.find(key);
  if (it == g_algos.end()) {
    cublasLtMatmulHeuristicResult_t heur{};
    int found = 0;
    if (cublasLtMatmulAlgoGetHeuristic(g_lt, op, la, lb, lc, lc, pref, 1, &heur, &found) !=
            CUBLAS_STATUS_SUCCESS ||
        found == 0)
      return bad("no int8 algorithm for this shape");
    it = g_algos.emplace(key, heur.algo).first;
  }
  const int32_t alpha = 1, beta = 0;
  cublasStatus_t st = cublasLtMatmul(g_lt, op, &alpha, Bt, la, A, lb, &beta, C, lc, C, lc,
                                     &it->second, workspace, ws_size, stream);
  cleanup();
  if (st != CUBLAS_STATUS_SUCCESS) {
    *err = "cublasLtMatmul failed (status " + std::to_string(static_cast<int>(st)) + ")";
    return 2;
  }
  return 0;
}

}  // namespace mpmm
