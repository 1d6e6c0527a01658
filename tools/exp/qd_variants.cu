// Experiment: QD "simple" kernel variants (occupancy / outputs per thread).
// nvcc -O3 -std=c++17 -fmad=false -gencode arch=compute_100a,code=sm_100a \
//   -I paper_1710_01839_b200/csrc tools/exp/qd_variants.cu -o /tmp/qdv
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "ddqd.cuh"
using namespace mpmm;

template <int MINB, int TPB>
__global__ void __launch_bounds__(TPB, MINB) qd1(const double2* A, const double2* B, double2* C, int n) {
  int j = blockIdx.x * 32 + (threadIdx.x & 31);
  int i = blockIdx.y * (TPB / 32) + (threadIdx.x >> 5);
  if (i >= n || j >= n) return;
  double acc[4] = {0, 0, 0, 0};
  for (int k = 0; k < n; ++k) {
    const double2* ap = A + 2 * ((long)i * n + k);
    const double2* bp = B + 2 * ((long)k * n + j);
    double2 a0 = __ldg(ap), a1 = __ldg(ap + 1), b0 = __ldg(bp), b1 = __ldg(bp + 1);
    double x[4] = {a0.x, a0.y, a1.x, a1.y}, y[4] = {b0.x, b0.y, b1.x, b1.y};
    qd_mul_add(acc, x, y);
  }
  double2* cp = C + 2 * ((long)i * n + j);
  cp[0] = make_double2(acc[0], acc[1]);
  cp[1] = make_double2(acc[2], acc[3]);
}

// two outputs per thread (columns j and j+32), interleaved
template <int MINB, int TPB>
__global__ void __launch_bounds__(TPB, MINB) qd2(const double2* A, const double2* B, double2* C, int n) {
  int j = blockIdx.x * 64 + (threadIdx.x & 31);
  int i = blockIdx.y * (TPB / 32) + (threadIdx.x >> 5);
  if (i >= n) return;
  double acc0[4] = {0, 0, 0, 0}, acc1[4] = {0, 0, 0, 0};
  for (int k = 0; k < n; ++k) {
    const double2* ap = A + 2 * ((long)i * n + k);
    const double2* bp = B + 2 * ((long)k * n + j);
    double2 a0 = __ldg(ap), a1 = __ldg(ap + 1), b0 = __ldg(bp), b1 = __ldg(bp + 1);
    double2 c0 = __ldg(bp + 64), c1 = __ldg(bp + 65);
    double x[4] = {a0.x, a0.y, a1.x, a1.y}, y[4] = {b0.x, b0.y, b1.x, b1.y};
    double z[4] = {c0.x, c0.y, c1.x, c1.y};
    qd_mul_add(acc0, x, y);
    qd_mul_add(acc1, x, z);
  }
  double2* cp = C + 2 * ((long)i * n + j);
  cp[0] = make_double2(acc0[0], acc0[1]);
  cp[1] = make_double2(acc0[2], acc0[3]);
  cp[64] = make_double2(acc1[0], acc1[1]);
  cp[65] = make_double2(acc1[2], acc1[3]);
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 1024;
  size_t sz = (size_t)n * n * 4;
  std::vector<double> h(sz);
  srand(1);
  for (size_t e = 0; e < (size_t)n * n; ++e) {
    double x0 = 2.0 * rand() / RAND_MAX - 1.0;
    h[4 * e] = x0;
    h[4 * e + 1] = x0 * 0x1p-53 * (2.0 * rand() / RAND_MAX - 1.0);
    h[4 * e + 2] = x0 * 0x1p-106 * (2.0 * rand() / RAND_MAX - 1.0);
    h[4 * e + 3] = x0 * 0x1p-159 * (2.0 * rand() / RAND_MAX - 1.0);
  }
  double *A, *B, *C, *R;
  cudaMalloc(&A, sz * 8); cudaMalloc(&B, sz * 8); cudaMalloc(&C, sz * 8); cudaMalloc(&R, sz * 8);
  cudaMemcpy(A, h.data(), sz * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, h.data(), sz * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<double> ref(sz), got(sz);
  auto run = [&](const char* name, auto launch, bool first) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    cudaMemcpy(first ? ref.data() : got.data(), first ? R : C, sz * 8, cudaMemcpyDeviceToHost);
    bool same = first || memcmp(ref.data(), got.data(), sz * 8) == 0;
    double ideal = (double)n * n * n * 786 / (148.0 * 64 * 1.965e9) * 1e3;
    printf("%-28s %8.3f ms  eff %.3f  %s  err=%s\n", name, best, ideal / best, same ? "same" : "DIFF",
           cudaGetErrorString(cudaGetLastError()));
  };
  const double2* a = (const double2*)A; const double2* b = (const double2*)B;
  run("qd1<3,256> (lib)", [&] { qd1<3, 256><<<dim3(n / 32, n / 8), 256>>>(a, b, (double2*)R, n); }, true);
  run("qd1<4,256>", [&] { qd1<4, 256><<<dim3(n / 32, n / 8), 256>>>(a, b, (double2*)C, n); }, false);
  run("qd1<8,128>", [&] { qd1<8, 128><<<dim3(n / 32, n / 4), 128>>>(a, b, (double2*)C, n); }, false);
  run("qd1<6,128>", [&] { qd1<6, 128><<<dim3(n / 32, n / 4), 128>>>(a, b, (double2*)C, n); }, false);
  run("qd1<2,512>", [&] { qd1<2, 512><<<dim3(n / 32, n / 16), 512>>>(a, b, (double2*)C, n); }, false);
  run("qd2<2,256>", [&] { qd2<2, 256><<<dim3(n / 64, n / 8), 256>>>(a, b, (double2*)C, n); }, false);
  run("qd2<3,128>", [&] { qd2<3, 128><<<dim3(n / 64, n / 4), 128>>>(a, b, (double2*)C, n); }, false);
  run("qd2<4,128>", [&] { qd2<4, 128><<<dim3(n / 64, n / 4), 128>>>(a, b, (double2*)C, n); }, false);
  return 0;
}
