// Does mma.sync.m8n8k4.f64 round like four sequential FMAs (k = 0..3)?
#include <cstdio>
#include <cmath>
#include <random>
#include <cuda_runtime.h>

__global__ void k_dmma(const double* A, const double* B, const double* C, double* D) {
  // A 8x4 row-major, B 4x8 col-major, C/D 8x8 row-major; lane layout per PTX:
  // a0 = A[row = lane>>2][col = lane&3]; b0 = B[row = lane&3][col = lane>>2]
  // c0,c1 = C[row = lane>>2][col = 2*(lane&3) + {0,1}]
  const int lane = threadIdx.x;
  double a = A[(lane >> 2) * 4 + (lane & 3)];
  double b = B[(lane >> 2) * 4 + (lane & 3)];  // col-major: col = lane>>2, row = lane&3
  double c0 = C[(lane >> 2) * 8 + 2 * (lane & 3)], c1 = C[(lane >> 2) * 8 + 2 * (lane & 3) + 1];
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  D[(lane >> 2) * 8 + 2 * (lane & 3)] = c0;
  D[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = c1;
}

int main() {
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> u(-1, 1);
  int mism_asc = 0, mism_desc = 0, mism_fused = 0, total = 0;
  double *dA, *dB, *dC, *dD;
  cudaMalloc(&dA, 32 * 8); cudaMalloc(&dB, 32 * 8); cudaMalloc(&dC, 64 * 8); cudaMalloc(&dD, 64 * 8);
  for (int trial = 0; trial < 2000; ++trial) {
    double A[32], B[32], C[64], D[64];
    for (int i = 0; i < 32; ++i) { A[i] = u(g) * pow(2.0, int(u(g) * 20)); B[i] = u(g) * pow(2.0, int(u(g) * 20)); }
    for (int i = 0; i < 64; ++i) C[i] = u(g) * pow(2.0, int(u(g) * 20));
    cudaMemcpy(dA, A, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, B, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C, 512, cudaMemcpyHostToDevice);
    k_dmma<<<1, 32>>>(dA, dB, dC, dD);
    cudaMemcpy(D, dD, 512, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        double s = C[i * 8 + j];
        for (int k = 0; k < 4; ++k) s = fma(A[i * 4 + k], B[j * 4 + k], s);
        double t = C[i * 8 + j];
        for (int k = 3; k >= 0; --k) t = fma(A[i * 4 + k], B[j * 4 + k], t);
        long double f = C[i * 8 + j];
        for (int k = 0; k < 4; ++k) f += (long double)A[i * 4 + k] * (long double)B[j * 4 + k];
        mism_asc += D[i * 8 + j] != s;
        mism_desc += D[i * 8 + j] != t;
        mism_fused += D[i * 8 + j] != (double)f;
        ++total;
      }
  }
  printf("DMMA vs sequential fma k-asc: %d/%d mismatches; k-desc: %d; single-rounding(approx): %d\n",
         mism_asc, total, mism_desc, mism_fused);
  return 0;
}
