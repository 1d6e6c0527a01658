// ord_burn.cu -- two_sum_ord (magnitude-ordered Fast2Sum) against the
// reference-sequence two_sum: (1) bitwise equality of s and err on random
// and special operand pairs, of DD multiply-add chains and of QD
// multiply-add chains; (2) register-only throughput of the DD and QD
// multiply-add with each variant (FP64 vs ALU pipe balance).
// nvcc -O3 -fmad=false -gencode arch=compute_100a,code=sm_100a ord_burn.cu -o ord_burn
#include <cstdio>
#include <cstdint>
#include <cstring>
#include "../../paper_1710_01839_b200/csrc/ddqd.cuh"
using namespace mpmm;

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ double unif(uint64_t& st) {  // [-1, 1)
  st = mix(st);
  return (double)(int64_t)st * 0x1p-63;
}

// operand with a random class: uniform, wide exponent, tiny/subnormal,
// signed zero, or derived from the other operand (equal, negated, near).
__device__ double pick(uint64_t& st, double other) {
  st = mix(st);
  int cls = st % 10;
  double u = unif(st);
  switch (cls) {
    case 0: return u;
    case 1: return ldexp(u, (int)(mix(st) % 1600) - 1000);
    case 2: return ldexp(u, -1060 + (int)(mix(st) % 40));   // subnormal region
    case 3: return (mix(st) & 1) ? 0.0 : -0.0;
    case 4: return other;
    case 5: return -other;
    case 6: return other * (1.0 + 0x1p-52 * (double)(int)(mix(st) % 5));
    case 7: return ldexp(u, (int)(mix(st) % 120) - 60);
    case 8: return other * 0x1p-53 * u;
    default: return ldexp(u, (int)(mix(st) % 1990) - 1020);
  }
}

__global__ void check_pairs(uint64_t seed, long n, unsigned long long* bad) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t st = seed ^ (uint64_t)i * 0x2545f4914f6cdd1dull;
  double a = pick(st, 0.5);
  double b = pick(st, a);
  if (mix(st) & 1) { double t = a; a = b; b = t; }
  if (!(fabs(a) < 0x1p996) || !(fabs(b) < 0x1p996)) return;
  double e1, e2;
  double s1 = two_sum(a, b, e1);
  double s2 = two_sum_ord(a, b, e2);
  if (__double_as_longlong(s1) != __double_as_longlong(s2) ||
      __double_as_longlong(e1) != __double_as_longlong(e2)) {
    unsigned long long k = atomicAdd(bad, 1ull);
    if (k < 4) printf("pair mismatch a=%a b=%a: s %a/%a e %a/%a\n", a, b, s1, s2, e1, e2);
  }
}

__global__ void check_dd(uint64_t seed, int len, int wide, unsigned long long* bad) {
  uint64_t st = seed ^ (uint64_t)(blockIdx.x * blockDim.x + threadIdx.x) * 0x9e37ull;
  double c1h = 0, c1l = 0, c2h = 0, c2l = 0;
  for (int k = 0; k < len; ++k) {
    double ah = unif(st), bh = unif(st);
    double al = ah * 0x1p-53 * unif(st), bl = bh * 0x1p-53 * unif(st);
    ah = two_sum(ah, al, al);
    bh = two_sum(bh, bl, bl);
    if (wide) {
      int ka = (int)(mix(st) % 61) - 30, kb = (int)(mix(st) % 61) - 30;
      ah = ldexp(ah, ka); al = ldexp(al, ka); bh = ldexp(bh, kb); bl = ldexp(bl, kb);
    }
    if ((mix(st) % 97) == 0) { ah = -c1h / (bh != 0 ? bh : 1.0); al = 0.0; }  // cancellation
    if ((mix(st) % 89) == 0) { al = 0.0; bl = -0.0; }
    dd_madd<false>(c1h, c1l, ah, al, bh, bl);
    dd_madd<true>(c2h, c2l, ah, al, bh, bl);
  }
  if (__double_as_longlong(c1h) != __double_as_longlong(c2h) ||
      __double_as_longlong(c1l) != __double_as_longlong(c2l)) {
    unsigned long long k = atomicAdd(bad, 1ull);
    if (k < 4) printf("dd chain mismatch %a %a vs %a %a\n", c1h, c1l, c2h, c2l);
  }
}

__global__ void check_qd(uint64_t seed, int len, unsigned long long* bad) {
  uint64_t st = seed ^ (uint64_t)(blockIdx.x * blockDim.x + threadIdx.x) * 0x9e37ull;
  double c1[4] = {0, 0, 0, 0}, c2[4] = {0, 0, 0, 0};
  for (int k = 0; k < len; ++k) {
    double x[4], y[4];
    x[0] = unif(st); y[0] = unif(st);
    for (int i = 1; i < 4; ++i) {
      x[i] = ldexp(x[0], -53 * i) * unif(st);
      y[i] = ldexp(y[0], -53 * i) * unif(st);
    }
    if ((mix(st) % 53) == 0) { x[3] = 0.0; }
    if ((mix(st) % 59) == 0) { x[2] = -0.0; y[3] = 0.0; }
    qd_mul_add<0, 0>(c1, x, y);
    qd_mul_add<15, 15>(c2, x, y);
  }
  bool diff = false;
  for (int i = 0; i < 4; ++i) diff |= __double_as_longlong(c1[i]) != __double_as_longlong(c2[i]);
  if (diff) {
    unsigned long long k = atomicAdd(bad, 1ull);
    if (k < 4) printf("qd chain mismatch %a vs %a\n", c1[0], c2[0]);
  }
}

// renorm5 (fast path + fallback) against the general emission loop alone
__global__ void check_renorm(uint64_t seed, long n, unsigned long long* bad) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t st = seed ^ (uint64_t)i * 0x9e3779b97f4a7c15ull;
  double x[5];
  x[0] = unif(st);
  for (int k = 1; k < 5; ++k) {
    st = mix(st);
    int cls = st % 8;
    double u = unif(st);
    x[k] = cls == 0 ? 0.0 : cls == 1 ? -0.0 : cls == 2 ? -x[k - 1] : cls == 3 ? ldexp(u, -1060)
         : ldexp(x[k - 1], -53) * u;
  }
  double a[4], b[4];
  renorm5(x[0], x[1], x[2], x[3], x[4], a);
  double y1 = x[1], y2 = x[2], y3 = x[3], y4 = x[4], s, t;
  s = quick_two_sum(y3, y4, y4);
  t = quick_two_sum(y2, s, y3);
  s = quick_two_sum(y1, t, y2);
  t = quick_two_sum(x[0], s, y1);
  renorm5_emit(t, y1, y2, y3, y4, b);
  for (int k = 0; k < 4; ++k)
    if (__double_as_longlong(a[k]) != __double_as_longlong(b[k])) {
      unsigned long long c = atomicAdd(bad, 1ull);
      if (c < 4) printf("renorm mismatch %a %a %a %a %a\n", x[0], x[1], x[2], x[3], x[4]);
      break;
    }
}

template <int C, bool ORD>
__global__ void burn_dd(double* out, int iters, double seed) {
  double hi[C], lo[C];
  double ah = seed + threadIdx.x * 1e-9, al = ah * 1e-17;
  double bh = 0.999999, bl = 1e-17;
  for (int c = 0; c < C; ++c) { hi[c] = c * 1e-3; lo[c] = 0; }
  for (int it = 0; it < iters; ++it) {
    ah = ah * 1.0000000001;
    al = al * 0.9999999999;
#pragma unroll
    for (int c = 0; c < C; ++c) dd_madd<ORD>(hi[c], lo[c], ah, al, bh + c * 1e-12, bl);
  }
  double s = 0;
  for (int c = 0; c < C; ++c) s += hi[c] + lo[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int M23, int M8>
__global__ void __launch_bounds__(256, 2) burn_qd(double* out, int iters, double seed) {
  double c[4] = {0, 0, 0, 0};
  double x[4] = {seed + threadIdx.x * 1e-9, 1e-17, 1e-34, 1e-51};
  double y[4] = {0.999999, 1.1e-17, 1.2e-34, 1.3e-51};
  for (int it = 0; it < iters; ++it) {
    x[0] = x[0] * 1.0000000001;
    x[1] = x[1] * 0.9999999999;
    qd_mul_add<M23, M8>(c, x, y);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0] + c[1] + c[2] + c[3];
}

template <class K>
float time_kernel(K kern, int blocks, int threads, double* out, int iters) {
  kern<<<blocks, threads>>>(out, 4, 0.5);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<blocks, threads>>>(out, iters, 0.5);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  unsigned long long* bad;
  cudaMallocManaged(&bad, 8);
  *bad = 0;
  long npairs = 1l << 28;
  for (int r = 0; r < 4; ++r) check_pairs<<<(npairs + 255) / 256, 256>>>(1234 + r, npairs, bad);
  cudaDeviceSynchronize();
  printf("pairs: %ld x 4 checked, %llu mismatches\n", npairs, *bad);
  *bad = 0;
  check_dd<<<1184, 128>>>(77, 1024, 0, bad);
  check_dd<<<1184, 128>>>(78, 1024, 1, bad);
  cudaDeviceSynchronize();
  printf("dd chains: 2 x %d of length 1024 (uniform, wide), %llu mismatches\n", 1184 * 128, *bad);
  *bad = 0;
  check_qd<<<592, 128>>>(79, 256, bad);
  cudaDeviceSynchronize();
  printf("qd chains: %d of length 256, %llu mismatches (%s)\n", 592 * 128, *bad,
         cudaGetErrorString(cudaGetLastError()));

  *bad = 0;
  for (int r = 0; r < 4; ++r) check_renorm<<<(npairs + 255) / 256, 256>>>(99 + r, npairs, bad);
  cudaDeviceSynchronize();
  printf("renorm5: %ld x 4 checked, %llu mismatches\n", npairs, *bad);

  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 1024 * 4);
  const double dfma_peak = 148.0 * 64 * 1.965e9;  // FP64 instr/s at boost
  for (int w : {8, 16}) {
    int iters = 2000;
    float m0 = time_kernel(burn_dd<4, false>, 148, 32 * w, out, iters);
    float m1 = time_kernel(burn_dd<4, true>, 148, 32 * w, out, iters);
    double madds = 148.0 * 32 * w * iters * 4;
    printf("DD C=4 warps/SM=%d: mirror %.3f ms (%.1f%% FP64 issue), ord %.3f ms  speed-up %.3f\n", w,
           m0, 100.0 * madds * 50 / (m0 * 1e-3) / dfma_peak, m1, m0 / m1);
  }
  {
    int iters = 200, blocks = 296, threads = 256;
    double madds = (double)blocks * threads * iters;
    float t00 = time_kernel(burn_qd<0, 0>, blocks, threads, out, iters);
    printf("QD mirror: %.3f ms (%.1f%% FP64 issue at 786 instr)\n", t00,
           100.0 * madds * 786 / (t00 * 1e-3) / dfma_peak);
#define QV(a, b) { float t = time_kernel(burn_qd<a, b>, blocks, threads, out, iters); \
      printf("QD M23=%2d M8=%2d: %.3f ms  speed-up %.3f\n", a, b, t, t00 / t); }
    QV(1, 0) QV(3, 0) QV(7, 0) QV(15, 0) QV(5, 0) QV(10, 0) QV(3, 3) QV(7, 7) QV(15, 15) QV(5, 5)
  }
  return 0;
}
