// Batched variable-size FP64 GEMM on the DMMA tensor path, with
// multi-segment accumulation and an optional kernel-function generator for
// the B operand (fused evaluate-and-project).
//
// Bit-exactness: mma.sync.m8n8k4.f64 rounds exactly like four sequential
// FMAs in ascending k (measured on the B200: 0 / 128,000 mismatches,
// tools/microbench/dmma_order.cu), so accumulating the k4 steps in order
// over segments in order reproduces the reference gemm_core / gemm_acc
// sequence c = fma(a, alpha*b, c) bit for bit (linalg.cpp:17-62). Ragged K
// is padded with a = +0, b = -0: that product adds an exact -0, which leaves
// every c (including -0.0) unchanged (tools/microbench/dmma_zero.cu).
//
// Tiling: CTA tile BM x 64, BK = 16, 2*BM threads (warp tile 32 x 32),
// operands staged in shared memory, the next chunk prefetched into
// registers; per warp and k4 step 4 x 4 m8n8k4 MMAs. BM = 128 is used when the batch has
// tall C blocks so a kernel-generated B tile is evaluated once per 128 rows.
#include "kernels.hpp"

namespace h2g {

namespace {

constexpr int BN = 64, BK = 16, PAD = 8;

__device__ __forceinline__ bool masked(const GenB& g, int j) {
  for (int t = 0; t < g.nmask; ++t)
    if (j >= g.mask[t].x && j < g.mask[t].y) return true;
  return false;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Warp tile 32 x 32 (4 x 4 m8n8 fragments); BM/32 x 2 warps -> 2*BM threads.
template <int BM>
__global__ void __launch_bounds__(2 * BM) gemm_kernel(const GemmJob* __restrict__ jobs,
                                                  const GemmSeg* __restrict__ segs,
                                                  const GemmTile* __restrict__ tiles,
                                                  KernelParams kp, Cloud cloud, ErrWord* err,
                                                  int tag) {
  constexpr int NT = 2 * BM;
  constexpr int WM = 32;            // warp tile rows
  constexpr int FM = WM / 8;        // m8 fragments per warp
  constexpr int FN = 4;             // n8 fragments per warp (32 columns)
  constexpr int AE = BM * BK / NT;  // A elements per thread per chunk
  constexpr int BE = BK * BN / NT;  // B elements per thread per chunk
  __shared__ double As[BK][BM + PAD];
  __shared__ double Bs[BK][BN + PAD];
  __shared__ unsigned char Bmask[BN];
  const GemmTile tile = tiles[blockIdx.x];
  const GemmJob job = jobs[tile.job];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % (BM / 32), wn = warp / (BM / 32);
  const int m0 = tile.tm * BM, n0 = tile.tn * BN;
  const Mat C = job.C;
  // Accumulators: fragment (fm, fn) holds C rows m0 + wm*WM + fm*8 + (lane>>2),
  // cols n0 + wn*32 + fn*8 + 2*(lane&3) + {0,1}.
  double acc[FM][FN][2];
  const int crow = lane >> 2, ccol = 2 * (lane & 3);
#pragma unroll
  for (int fm = 0; fm < FM; ++fm)
#pragma unroll
    for (int fn = 0; fn < FN; ++fn)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = m0 + wm * WM + fm * 8 + crow, j = n0 + wn * 32 + fn * 8 + ccol + h;
        acc[fm][fn][h] = (job.acc && i < C.rows && j < C.cols) ? C.at(i, j) : 0.0;
      }
  int singular = 0;
  for (int s = 0; s < job.nseg; ++s) {
    const GemmSeg sg = segs[job.seg0 + s];
    const int K = sg.A.cols;
    if (K == 0) continue;
    const int K4 = (K + 3) & ~3;  // padded with exact no-op (+0, -0) steps
    if (sg.gen) {
      __syncthreads();
      if (threadIdx.x < BN) Bmask[threadIdx.x] = sg.g.nmask ? masked(sg.g, n0 + threadIdx.x) : 0;
      __syncthreads();
    }
    const bool a_colmajor = sg.A.rs == 1;
    const bool b_colmajor = sg.B.rs == 1;
    double ra[AE], rb[BE];
    auto fetch = [&](int k0) {
#pragma unroll
      for (int u = 0; u < AE; ++u) {
        const int e = threadIdx.x + u * NT;
        int mm, kk;
        if (a_colmajor) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
        const int i = m0 + mm, l = k0 + kk;
        ra[u] = (i < sg.A.rows && l < K) ? sg.A.at(i, l) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < BE; ++u) {
        const int e = threadIdx.x + u * NT;
        int nn, kk;
        if (sg.gen || !b_colmajor) { nn = e % BN; kk = e / BN; } else { kk = e % BK; nn = e / BK; }
        const int l = k0 + kk, j = n0 + nn;
        double v = -0.0;  // pad: exact no-op with a = +0
        if (l < K && j < C.cols) {
          double b;
          if (!sg.gen) {
            b = sg.B.at(l, j);
          } else if (Bmask[nn]) {
            b = 0.0;
          } else {
            b = sg.g.trans ? kernel_entry(kp, cloud, sg.g.rb + j, sg.g.cb + l, &singular)
                           : kernel_entry(kp, cloud, sg.g.rb + l, sg.g.cb + j, &singular);
          }
          v = sg.alpha * b;  // the reference pre-multiplies B by alpha
        }
        rb[u] = v;
      }
    };
    auto stash = [&]() {
#pragma unroll
      for (int u = 0; u < AE; ++u) {
        const int e = threadIdx.x + u * NT;
        int mm, kk;
        if (a_colmajor) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
        As[kk][mm] = ra[u];
      }
#pragma unroll
      for (int u = 0; u < BE; ++u) {
        const int e = threadIdx.x + u * NT;
        int nn, kk;
        if (sg.gen || !b_colmajor) { nn = e % BN; kk = e / BN; } else { kk = e % BK; nn = e / BK; }
        Bs[kk][nn] = rb[u];
      }
    };
    __syncthreads();
    fetch(0);
    stash();
    __syncthreads();
    for (int k0 = 0; k0 < K4; k0 += BK) {
      // Register prefetch of the next chunk overlaps this chunk's MMAs.
      const bool more = k0 + BK < K4;
      if (more) fetch(k0 + BK);
      const int ksteps = min(BK, K4 - k0) / 4;
      for (int ks = 0; ks < ksteps; ++ks) {
        const int kr = ks * 4 + (lane & 3);
        double af[FM], bf[FN];
#pragma unroll
        for (int fm = 0; fm < FM; ++fm) af[fm] = As[kr][wm * WM + fm * 8 + (lane >> 2)];
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) bf[fn] = Bs[kr][wn * 32 + fn * 8 + (lane >> 2)];
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
#pragma unroll
          for (int fn = 0; fn < FN; ++fn) dmma(acc[fm][fn][0], acc[fm][fn][1], af[fm], bf[fn]);
      }
      if (more) {
        __syncthreads();
        stash();
        __syncthreads();
      }
    }
  }
  if (singular) raise_err(err, 1, tile.job, 0, tag);
#pragma unroll
  for (int fm = 0; fm < FM; ++fm)
#pragma unroll
    for (int fn = 0; fn < FN; ++fn)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = m0 + wm * WM + fm * 8 + crow, j = n0 + wn * 32 + fn * 8 + ccol + h;
        if (i < C.rows && j < C.cols) C.at(i, j) = acc[fm][fn][h];
      }
}

}  // namespace

int gemm_tile_rows(int max_rows) { return max_rows > 64 ? 128 : 64; }

void launch_gemm(const GemmJob* jobs, const GemmSeg* segs, const GemmTile* tiles, int ntiles,
                 int bm, KernelParams kp, Cloud cloud, ErrWord* err, int tag, cudaStream_t st) {
  if (ntiles <= 0) return;
  if (bm == 128)
    gemm_kernel<128><<<ntiles, 256, 0, st>>>(jobs, segs, tiles, kp, cloud, err, tag);
  else
    gemm_kernel<64><<<ntiles, 128, 0, st>>>(jobs, segs, tiles, kp, cloud, err, tag);
}

}  // namespace h2g
