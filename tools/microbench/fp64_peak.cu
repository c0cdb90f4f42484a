// FP64 peak micro-benchmark: DFMA (CUDA cores) vs DMMA (mma.sync f64 tensor path) on sm_100a.
// Each thread runs independent FMA chains; throughput = flops / kernel time (CUDA events).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001;
  double d[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-7;
  double d[2][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(d[i][0]), "+d"(d[i][1]), "+d"(d[i][2]), "+d"(d[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int i = 0; i < 2; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb);
      dfma_kernel<<<blocks, tpb>>>(out, 100);
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, tpb>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * (double)blocks * tpb;
      printf("DFMA tpb=%d: %.2f TFLOP/s\n", tpb, fl / ms / 1e9);
    }
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb);
      dmma_m8n8k4<<<blocks, tpb>>>(out, 100);
      cudaEventRecord(e0);
      dmma_m8n8k4<<<blocks, tpb>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * (tpb / 32);
      printf("DMMA m8n8k4 tpb=%d: %.2f TFLOP/s\n", tpb, fl / ms / 1e9);
    }
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb);
      dmma_m16n8k16<<<blocks, tpb>>>(out, 100);
      cudaEventRecord(e0);
      dmma_m16n8k16<<<blocks, tpb>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * 8 * 16 * 2 * (double)iters * blocks * (tpb / 32);
      printf("DMMA m16n8k16 tpb=%d: %.2f TFLOP/s\n", tpb, fl / ms / 1e9);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
