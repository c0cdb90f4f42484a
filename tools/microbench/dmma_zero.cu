// Signed-zero padding check: does a DMMA step with a = +0, b = -0 leave c bitwise unchanged (incl. c = -0)?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out) {
  const int lane = threadIdx.x;
  double cs[4] = {-0.0, 0.0, 1.5, -2.25};
  for (int t = 0; t < 4; ++t) {
    double c0 = cs[t], c1 = cs[t];
    double a = 0.0, b = -0.0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    if (lane == 0) { out[2 * t] = c0; out[2 * t + 1] = c1; }
  }
}
int main() {
  double* d; cudaMalloc(&d, 64); k<<<1, 32>>>(d); double h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  for (int t = 0; t < 4; ++t) printf("c=%g -> %g (signbit %d) %g\n", t == 0 ? -0.0 : (t == 1 ? 0.0 : (t == 2 ? 1.5 : -2.25)), h[2*t], __builtin_signbit(h[2*t]) != 0, h[2*t+1]);
  return 0;
}
