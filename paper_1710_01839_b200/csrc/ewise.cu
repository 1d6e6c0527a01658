// ewise.cu -- DD/QD elementwise add/sub (Strassen plumbing), the finite
// check, and the FP64 peak micro-benchmark.
//
// The elementwise kernel evaluates out = ((x s1 y) s2 z) s3 w for one to
// three chained operations; each step is exactly one reference ewise
// add/sub (_kernels.pyx:207-230 DD, :407-452 QD), so a chain is
// bit-identical to the reference's sequence of _ewise calls
// (multiply.py:189-203, :334-337) while reading each operand once and
// writing once (HBM-bound: 16 B per DD operand element).
#include "common.cuh"
#include "ddqd.cuh"
#include "kernels.h"

namespace mpmm {

__device__ __forceinline__ void load_elem(const double* base, int64_t ld, int i, int j, int V,
                                          int sign, double* v) {
  const double2* p = reinterpret_cast<const double2*>(base) + ((int64_t)i * ld + j) * V;
  for (int q = 0; q < V; ++q) {
    double2 x = p[q];
    v[2 * q] = sign < 0 ? -x.x : x.x;
    v[2 * q + 1] = sign < 0 ? -x.y : x.y;
  }
}

// out = ((x sy y) sz z) sw w, one reference ewise op per step.
template <int V>
__device__ __forceinline__ void ewise_elem(const EwiseProblem& e, int i, int j) {
  double x[2 * V], y[2 * V], r[2 * V];
  load_elem(e.X, e.ldx, i, j, V, 1, x);
  load_elem(e.Y, e.ldy, i, j, V, (int)e.sy, y);
  const double* ops[2] = {e.Z, e.W};
  const int64_t lds[2] = {e.ldz, e.ldw};
  const int sg[2] = {(int)e.sz, (int)e.sw};
  if constexpr (V == 1) {
    dd_add(x[0], x[1], y[0], y[1], r[0], r[1]);
    for (int s = 0; s < 2 && s + 2 <= e.nops; ++s) {
      load_elem(ops[s], lds[s], i, j, V, sg[s], y);
      dd_add(r[0], r[1], y[0], y[1], r[0], r[1]);
    }
  } else {
    qd_add(x, y, r);
    for (int s = 0; s < 2 && s + 2 <= e.nops; ++s) {
      load_elem(ops[s], lds[s], i, j, V, sg[s], y);
      double t[4] = {r[0], r[1], r[2], r[3]};
      qd_add(t, y, r);
    }
  }
  double2* o = reinterpret_cast<double2*>(e.O) + ((int64_t)i * e.ldo + j) * V;
  for (int q = 0; q < V; ++q) o[q] = make_double2(r[2 * q], r[2 * q + 1]);
}

template <int V>
__global__ void __launch_bounds__(256)
ewise_kernel(const EwiseProblem* __restrict__ probs, EwiseProblem single, int rows, int cols) {
  const EwiseProblem e = probs ? probs[blockIdx.z] : single;
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  for (int i = blockIdx.y; i < rows; i += gridDim.y) ewise_elem<V>(e, i, j);
}

static cudaError_t ewise_go(int comps, int batch, int rows, int cols, const EwiseProblem* probs,
                            const EwiseProblem& single, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0 || batch <= 0) return cudaSuccess;
  if (batch > 65535) return cudaErrorInvalidValue;
  int threads = cols >= 256 ? 256 : ((cols + 31) / 32) * 32;
  dim3 grid((cols + threads - 1) / threads, rows < 4096 ? rows : 4096, batch);
  if (comps == 2)
    ewise_kernel<1><<<grid, threads, 0, stream>>>(probs, single, rows, cols);
  else
    ewise_kernel<2><<<grid, threads, 0, stream>>>(probs, single, rows, cols);
  return cudaGetLastError();
}

cudaError_t ewise_launch(const EwiseArgs& e) {
  EwiseProblem p{e.X, e.Y, e.Z, e.W, e.O, e.ldx, e.ldy, e.ldz, e.ldw, e.ldo,
                 e.nops, e.sy, e.sz, e.sw};
  return ewise_go(e.comps, 1, e.rows, e.cols, nullptr, p, e.stream);
}

cudaError_t ewise_batched_launch(int comps, int batch, int rows, int cols,
                                 const EwiseProblem* probs, cudaStream_t stream) {
  EwiseProblem none{};
  return ewise_go(comps, batch, rows, cols, probs, none, stream);
}

// multiply.py:124-127 _check_finite: any non-finite component -> flag.
__global__ void nonfinite_kernel(const double* X, int64_t ldx_d, int rows, int row_len,
                                 int* flag) {
  int bad = 0;
  for (int i = blockIdx.y; i < rows; i += gridDim.y)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < row_len; j += gridDim.x * blockDim.x)
      bad |= !isfinite(X[(int64_t)i * ldx_d + j]);
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

cudaError_t nonfinite_launch(int comps, const double* X, int64_t ldx, int rows, int cols,
                             int* flag, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  int row_len = cols * comps;
  dim3 grid((row_len + 255) / 256 < 64 ? (row_len + 255) / 256 : 64, rows < 4096 ? rows : 4096);
  nonfinite_kernel<<<grid, 256, 0, stream>>>(X, ldx * comps, rows, row_len, flag);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// FP64 peak micro-benchmark: 8 independent chains per
// thread of DFMA (op 0, 2 flops each) or DADD (op 1, 1 flop each).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) fp64_burn(int op, int64_t iters, double* out) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  const double a = 0.999999999, b = 1e-9, d = 3.0e-17;
  if (op == 0) {
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = __fma_rn(x[c], a, b);
    }
  } else {
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = x[c] + ((c & 1) ? d : -d);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}

cudaError_t fp64_burn_launch(int op, int blocks, int threads, int64_t iters, double* out,
                             cudaStream_t stream) {
  fp64_burn<<<blocks, threads, 0, stream>>>(op, iters, out);
  return cudaGetLastError();
}

}  // namespace mpmm
