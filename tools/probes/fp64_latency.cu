#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, int n) {
  double acc = a;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < n; ++i) { acc = __dadd_rn(acc, a); acc = __dadd_rn(acc, a); acc = __dadd_rn(acc, a); acc = __dadd_rn(acc, a); }
  long long t1 = clock64();
  double m = a;
  #pragma unroll 1
  for (int i = 0; i < n; ++i) { m = __dmul_rn(m, a); m = __dmul_rn(m, a); m = __dmul_rn(m, a); m = __dmul_rn(m, a); }
  long long t2 = clock64();
  double d = a + 3.0;
  #pragma unroll 1
  for (int i = 0; i < n; ++i) { d = __ddiv_rn(d, a); }
  long long t3 = clock64();
  out[0] = acc + m + d; cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() { double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 24); int n = 4096;
  k<<<1,1>>>(o, c, 1.0000001, n); k<<<1,1>>>(o, c, 1.0000001, n); long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles; DMUL: %.2f; DDIV: %.2f\n", h[0] / (4.0*n), h[1] / (4.0*n), h[2] / (1.0*n)); return 0; }
