// Latency of a dependent FP64 add chain s = s + a*b (the reference's
// rounded-product reduction) on one warp, with operands from registers and
// from shared memory. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false
#include <cstdio>
__global__ void chain_reg(double* out, long long* cyc, int n, double a) {
  double s = threadIdx.x, b = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { s = s + a * b; b = b * 1.0000001; }
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_add(double* out, long long* cyc, int n, double a) {
  double s = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { s = s + a; }
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_smem(double* out, long long* cyc, int n) {
  __shared__ double col[32 * 130];
  __shared__ double v[256];
  for (int i = threadIdx.x; i < 32 * 130; i += blockDim.x) col[i] = 1.0 + i * 1e-6;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) v[i] = 0.5 + i * 1e-7;
  __syncthreads();
  const double* c = col + (threadIdx.x & 31) * 130;
  double s = 0;
  long long t0 = clock64();
  for (int r = 0; r < n; ++r)
    for (int i = 0; i < 128; ++i) s = s + c[i] * v[i];
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
  const int n = 4096;
  for (int w = 1; w <= 8; w *= 2) {
    chain_add<<<1, 32 * w>>>(o, c, n, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps/CTA=%d  dadd chain: %.2f cycles/elem\n", w, double(h) / n);
    chain_reg<<<1, 32 * w>>>(o, c, n, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps/CTA=%d  dmul+dadd chain (regs): %.2f cycles/elem\n", w, double(h) / n);
    chain_smem<<<1, 32 * w>>>(o, c, 16); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps/CTA=%d  dmul+dadd chain (smem cols): %.2f cycles/elem\n", w, double(h) / (16 * 128));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
