// round_fast_test.cu -- device check of round_dd_fast against limbs read
// from stdin (one case per line: K limbs (hex, low first), neg, ebase);
// prints hi lo as %a.  Compiled with the library's flags.
#include <cstdio>
#include "../../paper_1710_01839_b200/csrc/ozaki.cu"

template <int K>
__global__ void run(const int64_t* mag_in, int neg, int ebase, double* out, int* ok) {
  int64_t mag[K];
  for (int q = 0; q < K; ++q) mag[q] = mag_in[q];
  double hi = 0, lo = 0;
  *ok = mpmm::round_dd_fast<K>(mag, neg != 0, ebase, hi, lo);
  out[0] = hi;
  out[1] = lo;
}

int main() {
  int64_t* dm; double* dout; int* dok;
  cudaMalloc(&dm, 9 * 8); cudaMalloc(&dout, 16); cudaMalloc(&dok, 4);
  unsigned long long v[9];
  int neg, eb;
  while (scanf("%llx %llx %llx %llx %llx %llx %llx %llx %llx %d %d", &v[0], &v[1], &v[2], &v[3],
               &v[4], &v[5], &v[6], &v[7], &v[8], &neg, &eb) == 11) {
    int64_t m[9];
    for (int q = 0; q < 9; ++q) m[q] = (int64_t)v[q];
    cudaMemcpy(dm, m, 72, cudaMemcpyHostToDevice);
    run<9><<<1, 1>>>(dm, neg, eb, dout, dok);
    double o[2]; int ok;
    cudaMemcpy(o, dout, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost);
    printf("%d %a %a\n", ok, o[0], o[1]);
  }
  return 0;
}
