// Do DMMA (tensor path) and DFMA (FP64 pipe) overlap? Half the warps of each
// CTA run m16n8k16 DMMA chains, half DFMA chains; compare the mixed kernel's
// time with each half alone. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ void dfma_loop(double* out, int iters) {
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

__device__ void dmma_loop(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-7;
  double d[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(d[i][0]), "+d"(d[i][1]), "+d"(d[i][2]), "+d"(d[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 12345.678) out[0] = s;
}

// mode 0: all warps DMMA; 1: all DFMA; 2: even warps DMMA, odd DFMA (half each).
__global__ void mix(double* out, int it_mma, int it_fma, int mode) {
  const int w = threadIdx.x >> 5;
  const bool mma = mode == 0 || (mode == 2 && (w & 1) == 0);
  if (mma) dmma_loop(out, it_mma); else dfma_loop(out, it_fma);
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int itm = 4000, itf = 40000, tpb = 512;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      mix<<<sms * 2, tpb>>>(out, itm, itf, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = double(sms) * 2 * tpb / 32;
      const double wm = mode == 0 ? warps : mode == 2 ? warps / 2 : 0;
      const double wf = mode == 1 ? warps : mode == 2 ? warps / 2 : 0;
      const double fl = wm * itm * 4 * 2.0 * 16 * 8 * 16 + wf * 32 * itf * 8 * 2.0;
      if (rep) printf("mode %d (%s): %.3f ms, %.2f TFLOP/s combined\n", mode,
                      mode == 0 ? "DMMA" : mode == 1 ? "DFMA" : "half/half", ms, fl / ms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
