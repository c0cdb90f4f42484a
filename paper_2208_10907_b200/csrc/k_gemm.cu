// Batched variable-size FP64 GEMM with multi-segment accumulation and an
// optional kernel-function generator for the B operand.
//
// Accumulation order per C element equals the reference gemm_core
// (linalg.cpp:17-62): c = fma(A(i,l), alpha*B(l,j), c) over segments in
// order, l in order. Each thread owns a 4x4 register tile of a 64x64 CTA tile;
// A and B k-chunks are staged in shared memory. FP64 on sm_100a: DFMA and
// DMMA both peak at ~37 TFLOP/s (profiles/r01_fp64_peak_probe.txt), so DFMA
// is used and the reference's rounding sequence is kept bit for bit.
#include "kernels.hpp"

namespace h2g {

namespace {

constexpr int TM = 64, TN = 64, KC = 16, NT = 256;

__device__ __forceinline__ bool masked(const GenB& g, int j) {
  for (int t = 0; t < g.nmask; ++t)
    if (j >= g.mask[t].x && j < g.mask[t].y) return true;
  return false;
}

__global__ void __launch_bounds__(NT) gemm_kernel(const GemmJob* __restrict__ jobs,
                                                  const GemmSeg* __restrict__ segs,
                                                  const GemmTile* __restrict__ tiles,
                                                  KernelParams kp, Cloud cloud, ErrWord* err,
                                                  int tag) {
  __shared__ double As[KC][TM];
  __shared__ double Bs[KC][TN + 1];
  __shared__ unsigned char Bmask[TN];
  const GemmTile tile = tiles[blockIdx.x];
  const GemmJob job = jobs[tile.job];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = tile.tm * TM, n0 = tile.tn * TN;
  const Mat C = job.C;
  double c[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = m0 + ty + 16 * a, j = n0 + tx + 16 * b;
      c[a][b] = (job.acc && i < C.rows && j < C.cols) ? C.at(i, j) : 0.0;
    }
  int singular = 0;
  for (int s = 0; s < job.nseg; ++s) {
    const GemmSeg sg = segs[job.seg0 + s];
    const int K = sg.A.cols;
    if (sg.gen) {
      __syncthreads();
      if (threadIdx.x < TN) Bmask[threadIdx.x] = sg.g.nmask ? masked(sg.g, n0 + threadIdx.x) : 0;
    }
    for (int k0 = 0; k0 < K; k0 += KC) {
      __syncthreads();
      // A chunk: TM rows x KC cols.
      for (int e = threadIdx.x; e < TM * KC; e += NT) {
        const int mm = e % TM, kk = e / TM;
        const int i = m0 + mm, l = k0 + kk;
        As[kk][mm] = (i < sg.A.rows && l < K) ? sg.A.at(i, l) : 0.0;
      }
      // B chunk: KC rows x TN cols, pre-multiplied by alpha as the reference does.
      for (int e = threadIdx.x; e < TN * KC; e += NT) {
        const int nn = e % TN, kk = e / TN;
        const int l = k0 + kk, j = n0 + nn;
        double v = 0.0;
        if (l < K && j < C.cols) {
          if (!sg.gen) {
            v = sg.B.at(l, j);
          } else if (!Bmask[nn]) {
            v = sg.g.trans ? kernel_entry(kp, cloud, sg.g.rb + j, sg.g.cb + l, &singular)
                           : kernel_entry(kp, cloud, sg.g.rb + l, sg.g.cb + j, &singular);
          }
          v = sg.alpha * v;
        }
        Bs[kk][nn] = v;
      }
      __syncthreads();
      const int kmax = min(KC, K - k0);
      for (int kk = 0; kk < kmax; ++kk) {
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[kk][ty + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) c[a][b] = fma(av[a], bv[b], c[a][b]);
      }
    }
  }
  if (singular) raise_err(err, 1, tile.job, 0, tag);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = m0 + ty + 16 * a, j = n0 + tx + 16 * b;
      if (i < C.rows && j < C.cols) C.at(i, j) = c[a][b];
    }
}

}  // namespace

void launch_gemm(const GemmJob* jobs, const GemmSeg* segs, const GemmTile* tiles, int ntiles,
                 KernelParams kp, Cloud cloud, ErrWord* err, int tag, cudaStream_t st) {
  // Grid x limit is 2^31-1; tiles are bounded far below that.
  if (ntiles > 0) gemm_kernel<<<ntiles, NT, 0, st>>>(jobs, segs, tiles, kp, cloud, err, tag);
}

}  // namespace h2g
