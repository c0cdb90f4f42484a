// Does mma.sync.m16n8k{4,8,16}.f64 round like sequential FMAs in ascending k?
// Fragment layouts (PTX ISA, .f64): groupID g = lane>>2, t = lane&3.
//   A (16xK, row): a_i at row g + 8*(i%2), col t + 4*(i/2)
//   B (Kx8, col):  b_i at row t + 4*i, col g
//   C/D (16x8):    c_i at row g + 8*(i/2), col 2*t + (i%2)
// A wrong layout shows up as a large numerical error, not just rounding.
#include <cstdio>
#include <cmath>
#include <random>
#include <cuda_runtime.h>

template <int K>
__global__ void k_mma(const double* A, const double* B, const double* C, double* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[K / 2], b[K / 4], c[4];
  for (int i = 0; i < K / 2; ++i) a[i] = A[(g + 8 * (i % 2)) * K + t + 4 * (i / 2)];
  for (int i = 0; i < K / 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  for (int i = 0; i < 4; ++i) c[i] = C[(g + 8 * (i / 2)) * 8 + 2 * t + (i % 2)];
  if constexpr (K == 4) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  } else if constexpr (K == 8) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  } else {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  for (int i = 0; i < 4; ++i) D[(g + 8 * (i / 2)) * 8 + 2 * t + (i % 2)] = c[i];
}

template <int K>
void run() {
  std::mt19937_64 gen(1);
  std::uniform_real_distribution<double> u(-1, 1);
  int mism = 0, mism_desc = 0, total = 0;
  double maxrel = 0;
  double *dA, *dB, *dC, *dD;
  cudaMalloc(&dA, 16 * K * 8); cudaMalloc(&dB, K * 8 * 8); cudaMalloc(&dC, 128 * 8); cudaMalloc(&dD, 128 * 8);
  for (int trial = 0; trial < 2000; ++trial) {
    double A[16 * K], B[K * 8], C[128], D[128];
    for (int i = 0; i < 16 * K; ++i) A[i] = u(gen) * pow(2.0, int(u(gen) * 20));
    for (int i = 0; i < K * 8; ++i) B[i] = u(gen) * pow(2.0, int(u(gen) * 20));
    for (int i = 0; i < 128; ++i) C[i] = u(gen) * pow(2.0, int(u(gen) * 20));
    cudaMemcpy(dA, A, sizeof(A), cudaMemcpyHostToDevice); cudaMemcpy(dB, B, sizeof(B), cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C, sizeof(C), cudaMemcpyHostToDevice);
    k_mma<K><<<1, 32>>>(dA, dB, dC, dD);
    cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 16; ++i)
      for (int j = 0; j < 8; ++j) {
        double s = C[i * 8 + j], t = C[i * 8 + j], mag = fabs(C[i * 8 + j]);
        for (int k = 0; k < K; ++k) { s = fma(A[i * K + k], B[k * 8 + j], s); mag += fabs(A[i * K + k] * B[k * 8 + j]); }
        for (int k = K - 1; k >= 0; --k) t = fma(A[i * K + k], B[k * 8 + j], t);
        mism += D[i * 8 + j] != s;
        mism_desc += D[i * 8 + j] != t;
        maxrel = fmax(maxrel, fabs(D[i * 8 + j] - s) / mag);
        ++total;
      }
  }
  printf("m16n8k%d: vs sequential fma k-asc %d/%d mismatches, k-desc %d, max rel err %.3g (%s)\n", K, mism,
         total, mism_desc, maxrel, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<4>();
  run<8>();
  run<16>();
  return 0;
}
