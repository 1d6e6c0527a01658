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

__global__ void __launch_bounds__(256)
dd_ewise_kernel(EwiseArgs e) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int i = blockIdx.y;
  if (j >= e.cols) return;
  const double2* X = reinterpret_cast<const double2*>(e.X);
  const double2* Y = reinterpret_cast<const double2*>(e.Y);
  double2 x = X[(int64_t)i * e.ldx + j];
  double2 y = Y[(int64_t)i * e.ldy + j];
  double h, lo;
  double yh = e.sy < 0 ? -y.x : y.x, yl = e.sy < 0 ? -y.y : y.y;
  dd_add(x.x, x.y, yh, yl, h, lo);
  if (e.nops >= 2) {
    double2 z = reinterpret_cast<const double2*>(e.Z)[(int64_t)i * e.ldz + j];
    double zh = e.sz < 0 ? -z.x : z.x, zl = e.sz < 0 ? -z.y : z.y;
    dd_add(h, lo, zh, zl, h, lo);
  }
  if (e.nops >= 3) {
    double2 w = reinterpret_cast<const double2*>(e.W)[(int64_t)i * e.ldw + j];
    double wh = e.sw < 0 ? -w.x : w.x, wl = e.sw < 0 ? -w.y : w.y;
    dd_add(h, lo, wh, wl, h, lo);
  }
  reinterpret_cast<double2*>(e.O)[(int64_t)i * e.ldo + j] = make_double2(h, lo);
}

__device__ __forceinline__ void qd_load(const double* base, int64_t ld, int i, int j, int sign,
                                        double v[4]) {
  const double2* p = reinterpret_cast<const double2*>(base) + 2 * ((int64_t)i * ld + j);
  double2 a = p[0], b = p[1];
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  if (sign < 0) {
    v[0] = -v[0]; v[1] = -v[1]; v[2] = -v[2]; v[3] = -v[3];
  }
}

__global__ void __launch_bounds__(256)
qd_ewise_kernel(EwiseArgs e) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int i = blockIdx.y;
  if (j >= e.cols) return;
  double x[4], y[4], r[4];
  qd_load(e.X, e.ldx, i, j, 1, x);
  qd_load(e.Y, e.ldy, i, j, e.sy, y);
  qd_add(x, y, r);
  if (e.nops >= 2) {
    qd_load(e.Z, e.ldz, i, j, e.sz, y);
    double t[4] = {r[0], r[1], r[2], r[3]};
    qd_add(t, y, r);
  }
  if (e.nops >= 3) {
    qd_load(e.W, e.ldw, i, j, e.sw, y);
    double t[4] = {r[0], r[1], r[2], r[3]};
    qd_add(t, y, r);
  }
  double2* o = reinterpret_cast<double2*>(e.O) + 2 * ((int64_t)i * e.ldo + j);
  o[0] = make_double2(r[0], r[1]);
  o[1] = make_double2(r[2], r[3]);
}

cudaError_t ewise_launch(const EwiseArgs& e) {
  if (e.rows <= 0 || e.cols <= 0) return cudaSuccess;
  if (e.rows > 65535 * 1024) return cudaErrorInvalidValue;
  int threads = e.cols >= 256 ? 256 : ((e.cols + 31) / 32) * 32;
  dim3 grid((e.cols + threads - 1) / threads, e.rows);
  if (e.rows > 65535) {
    // fall back to row chunks: gridDim.y is limited to 65535
    for (int r0 = 0; r0 < e.rows; r0 += 65535) {
      EwiseArgs c = e;
      int rr = e.rows - r0 < 65535 ? e.rows - r0 : 65535;
      int64_t off = (int64_t)r0 * e.comps;
      c.rows = rr;
      c.X = e.X + off * e.ldx;
      c.Y = e.Y + off * e.ldy;
      if (e.Z) c.Z = e.Z + off * e.ldz;
      if (e.W) c.W = e.W + off * e.ldw;
      c.O = e.O + off * e.ldo;
      cudaError_t err = ewise_launch(c);
      if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
  }
  if (e.comps == 2)
    dd_ewise_kernel<<<grid, threads, 0, e.stream>>>(e);
  else
    qd_ewise_kernel<<<grid, threads, 0, e.stream>>>(e);
  return cudaGetLastError();
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
