// Dependent-chain latency of DADD / DFMA / LDS.64 on one warp (cycles per op).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, const double* g) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  double s = a;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) s = s + b;
  long long t1 = clock64();
  double f = a;
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) f = fma(f, b, a);
  long long t2 = clock64();
  int idx = threadIdx.x & 7;
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) idx = int(sm[idx]) & 1023;
  long long t3 = clock64();
  out[threadIdx.x] = s + f + idx;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
}
int main() {
  double* out;
  long long* cyc;
  double* g;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 64);
  cudaMalloc(&g, 1024 * 8);
  cudaMemset(g, 0, 1024 * 8);
  for (int w : {32, 128, 512}) {
    k<<<1, w>>>(out, cyc, 1.0, 1e-9, g);
    long long h[3];
    cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
    printf("threads %d: DADD %.2f DFMA %.2f LDS-chain %.2f cycles/op\n", w, h[0] / 4096.0,
           h[1] / 4096.0, h[2] / 4096.0);
  }
  return 0;
}
