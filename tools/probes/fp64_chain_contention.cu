// How many single-lane dependent DADD chains can one SM run before they slow each other down?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, int n, int lanes) {
  double acc = a + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  if ((threadIdx.x & 31) < lanes) {
    #pragma unroll 1
    for (int i = 0; i < n; ++i) { acc = __dadd_rn(acc, a); acc = __dadd_rn(acc, a); acc = __dadd_rn(acc, a); acc = __dadd_rn(acc, a); }
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = acc; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() { double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8); int n = 4096;
  for (int lanes : {1, 32}) for (int warps : {1, 4, 8, 12, 16, 24, 32}) {
    k<<<1, warps * 32>>>(o, c, 1.0000001, n, lanes); k<<<1, warps * 32>>>(o, c, 1.0000001, n, lanes);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("active lanes %2d, warps on the SM %2d: %.2f cycles per dependent DADD\n", lanes, warps, h / (4.0 * n)); }
  return 0; }
