// madd_burn.cu -- ceiling of the mirror DD multiply-add sequence on the
// FP64 pipe with no memory traffic: C chains per thread of dd_madd on
// register operands.  nvcc -O3 -fmad=false -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include "../../paper_1710_01839_b200/csrc/ddqd.cuh"
using namespace mpmm;

template <int C>
__global__ void burn(double* out, int iters, double seed) {
  double hi[C], lo[C];
  double ah = seed + threadIdx.x * 1e-9, al = ah * 1e-17;
  double bh = 0.999999, bl = 1e-17;
  for (int c = 0; c < C; ++c) { hi[c] = c * 1e-3; lo[c] = 0; }
  for (int it = 0; it < iters; ++it) {
    ah = ah * 1.0000000001;          // operands change every iteration (no hoisting)
    al = al * 0.9999999999;
#pragma unroll
    for (int c = 0; c < C; ++c) dd_madd(hi[c], lo[c], ah, al, bh + c * 1e-12, bl);
  }
  double s = 0;
  for (int c = 0; c < C; ++c) s += hi[c] + lo[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int C>
void run(int blocks, int threads) {
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  int iters = 2000;
  burn<C><<<blocks, threads>>>(out, 10, 0.5);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  burn<C><<<blocks, threads>>>(out, iters, 0.5);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double madds = (double)blocks * threads * iters * C;
  printf("C=%d blocks=%d threads=%d: %.3f ms, %.2f T FP64 instr/s ((50C+2)/iter)\n", C, blocks,
         threads, ms, madds / C * (50 * C + 2) / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16}) {       // warps per SM
    run<1>(148, 32 * w); run<2>(148, 32 * w); run<4>(148, 32 * w); run<8>(148, 32 * w);
  }
  return 0;
}
