// Batched kernel-block evaluation (near-field arena, solve inputs, basis
// members), batched strided copies/adds, and sequential Frobenius norms.
#include "kernels.hpp"

namespace h2g {

namespace {

constexpr int T = 64, NT = 256;

// Tile -> (job, tile index within the job) from the per-job prefix sums of tile
// counts (the host uploads njobs + 1 integers instead of two per tile).
__device__ __forceinline__ int find_job(const int* __restrict__ ptr, int njobs, int tile, int& idx) {
  int lo = 0, hi = njobs;  // ptr[lo] <= tile < ptr[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (ptr[mid] <= tile) lo = mid; else hi = mid;
  }
  idx = tile - ptr[lo];
  return lo;
}

// assemble_block (kernels.cpp:242-268) over 64x64 tiles; rows fastest so a
// column-major destination is written coalesced. The near-field arena write
// is the HBM-bound phase (8 B per entry).
__global__ void __launch_bounds__(NT) eval_kernel(const EvalJob* __restrict__ jobs,
                                                  const int* __restrict__ tile_ptr, int njobs,
                                                  KernelParams kp, Cloud cloud, ErrWord* err,
                                                  int tag) {
  // A thread's row is fixed (NT is a multiple of T): its point stays in
  // registers; the tile's 64 column points are staged in shared memory and
  // read as warp-wide broadcasts (a warp's 32 entries share one column).
  __shared__ double cpt[T][4];
  int ti;
  const int jb = find_job(tile_ptr, njobs, blockIdx.x, ti);
  const EvalJob job = jobs[jb];
  const int tpr = (job.out.rows + T - 1) / T;
  const int r0 = (ti % tpr) * T, c0 = (ti / tpr) * T;
  {
    const int jj = threadIdx.x >> 2, comp = threadIdx.x & 3;  // NT = 4 T
    double v = 0.0;
    if (c0 + jj < job.out.cols) {
      const int64_t pj = job.cb + int64_t(c0 + jj) * job.cstep;
      const double* src = comp == 0 ? cloud.x : comp == 1 ? cloud.y : comp == 2 ? cloud.z : cloud.q;
      v = src[pj];
    }
    cpt[jj][comp] = v;
  }
  const int i = r0 + (threadIdx.x % T);
  double xi = 0.0, yi = 0.0, zi = 0.0;
  if (i < job.out.rows) {
    const int64_t pi = job.rb + int64_t(i) * job.rstep;
    xi = cloud.x[pi];
    yi = cloud.y[pi];
    zi = cloud.z[pi];
  }
  __syncthreads();
  int singular = 0;
  if (i < job.out.rows) {
    double* dst = &job.out.at(i, c0);
    const int jn = min(T, job.out.cols - c0);
#pragma unroll 4
    for (int jj = threadIdx.x / T; jj < jn; jj += NT / T)
      dst[int64_t(jj) * job.out.cs] =
          kernel_pair(kp, xi, yi, zi, cpt[jj][0], cpt[jj][1], cpt[jj][2], cpt[jj][3], &singular);
  }
  if (singular) raise_err(err, 1, jb, 0, tag);
}

// dst = (add ? dst : 0) + alpha * src  — the reference's add_block computes
// dst[i] += alpha * src[i], contracted to fma(alpha, src, dst).
__global__ void __launch_bounds__(NT) copy_kernel(const CopyJob* __restrict__ jobs,
                                                  const int* __restrict__ tile_ptr, int njobs) {
  int ti;
  const CopyJob job = jobs[find_job(tile_ptr, njobs, blockIdx.x, ti)];
  const int tpr = (job.dst.rows + T - 1) / T;
  const int r0 = (ti % tpr) * T, c0 = (ti / tpr) * T;
  for (int e = threadIdx.x; e < T * T; e += NT) {
    const int i = r0 + (e % T), j = c0 + (e / T);
    if (i >= job.dst.rows || j >= job.dst.cols) continue;
    double v;
    if (job.src.p == nullptr) {
      v = job.ident ? (i == j ? 1.0 : 0.0) : 0.0;
      if (job.add) v = job.dst.at(i, j);
    } else if (job.add) {
      v = fma(job.alpha, job.src.at(i, j), job.dst.at(i, j));
    } else {
      v = job.alpha == 1.0 ? job.src.at(i, j) : job.alpha * job.src.at(i, j);
    }
    job.dst.at(i, j) = v;
  }
}

__global__ void __launch_bounds__(NT) accum_kernel(const AccJob* __restrict__ jobs,
                                                   const AccSrc* __restrict__ srcs,
                                                   const int* __restrict__ tile_ptr, int njobs) {
  int ti;
  const AccJob job = jobs[find_job(tile_ptr, njobs, blockIdx.x, ti)];
  const int tpr = (job.dst.rows + T - 1) / T;
  const int r0 = (ti % tpr) * T, c0 = (ti / tpr) * T;
  for (int e = threadIdx.x; e < T * T; e += NT) {
    const int i = r0 + (e % T), j = c0 + (e / T);
    if (i >= job.dst.rows || j >= job.dst.cols) continue;
    double v = job.zero_init ? 0.0 : job.dst.at(i, j);
    for (int s = 0; s < job.nsrc; ++s) {
      const AccSrc sr = srcs[job.src0 + s];
      v = fma(sr.alpha, sr.src.at(i, j), v);
    }
    job.dst.at(i, j) = v;
  }
}

__global__ void permute_rows_kernel(Mat dst, Mat src, const int64_t* idx, int scatter) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t rows = scatter ? src.rows : dst.rows;
  if (e >= rows * dst.cols) return;
  const int64_t i = e % rows, j = e / rows;
  if (scatter) dst.at(idx[i], j) = src.at(i, j);
  else dst.at(i, j) = src.at(idx[i], j);
}

// norm_frobenius (linalg.cpp:604-609): s += d*d over storage order. GCC's
// vectorised reduction (see k_qr.cu, pattern P2): 4-wide groups of rounded
// squares added in order; tails (and sizes <= 3) fused. One warp per matrix:
// the lanes load 32 consecutive elements (coalesced, one chunk ahead) and
// square them; the in-order sum runs on every lane from shuffled squares, so
// the dependent chain is one DADD per element.
__global__ void norms_kernel(const NormJob* __restrict__ jobs, int njobs) {
  const int w = int((blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (w >= njobs) return;
  const NormJob job = jobs[w];
  const int rows = job.a.rows;
  const int64_t tc = int64_t(rows) * job.a.cols;
  // Element e = (e % rows, e / rows) of the column-major walk; (i0, j0) is the
  // walk position of the current chunk's lane 0.
  int i0 = 0;
  int64_t j0 = 0;
  auto elem = [&](int64_t base_i, int64_t base_j, int off, int64_t e, int64_t lim) {
    if (e >= lim) return 0.0;
    int64_t i = base_i + off, j = base_j;
    while (i >= rows) {
      i -= rows;
      ++j;
    }
    return job.a.at(i, j);
  };
  auto advance = [&](int by) {
    i0 += by;
    while (i0 >= rows) {
      i0 -= rows;
      ++j0;
    }
  };
  double s = 0.0;
  if (tc <= 3) {
    for (int64_t e = 0; e < tc; ++e) {
      const double d = elem(0, 0, int(e), e, tc);
      s = fma(d, d, s);
    }
  } else {
    const int64_t v4 = tc & ~int64_t(3);
    double cur = elem(i0, j0, lane, lane, v4);
    for (int64_t e0 = 0; e0 < v4; e0 += 32) {
      advance(32);
      const double nxt = elem(i0, j0, lane, e0 + 32 + lane, v4);  // next chunk in flight
      const double sq = cur * cur;
      const int cnt = v4 - e0 < 32 ? int(v4 - e0) : 32;
      for (int l = 0; l < cnt; ++l) s = s + __shfl_sync(0xffffffffu, sq, l);
      cur = nxt;
    }
    for (int64_t e = v4; e < tc; ++e) {  // fused tail (<= 3 elements)
      const double d = job.a.at(e % rows, e / rows);
      s = fma(d, d, s);
    }
  }
  if (lane == 0) *job.out = sqrt(s);
}

// y = A x by direct summation in the ORIGINAL point order, each y_i
// accumulated over j in order like matmul(A, x) (solve.cpp:234-239).
__global__ void __launch_bounds__(256) matvec_kernel(KernelParams kp, Cloud c, const double* x,
                                                     double* y, int nrhs, int* singular) {
  __shared__ double sx[256], sy[256], sz[256], sq[256];
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const bool live = i < c.n;
  double acc[4] = {0, 0, 0, 0};
  const double xi = live ? c.x[i] : 0.0, yi = live ? c.y[i] : 0.0, zi = live ? c.z[i] : 0.0;
  int sing = 0;
  for (int r0 = 0; r0 < nrhs; r0 += 4) {
    const int nr = min(4, nrhs - r0);
    for (int a = 0; a < 4; ++a) acc[a] = 0.0;
    for (int64_t j0 = 0; j0 < c.n; j0 += 256) {
      __syncthreads();
      const int64_t jj = j0 + threadIdx.x;
      if (jj < c.n) {
        sx[threadIdx.x] = c.x[jj];
        sy[threadIdx.x] = c.y[jj];
        sz[threadIdx.x] = c.z[jj];
        sq[threadIdx.x] = c.q[jj];
      }
      __syncthreads();
      const int cnt = int(c.n - j0 < 256 ? c.n - j0 : 256);
      if (!live) continue;
      for (int t = 0; t < cnt; ++t) {
        const double a = kernel_pair(kp, xi, yi, zi, sx[t], sy[t], sz[t], sq[t], &sing);
        for (int q = 0; q < nr; ++q) acc[q] = fma(a, x[(r0 + q) * c.n + j0 + t], acc[q]);
      }
    }
    if (live)
      for (int q = 0; q < nr; ++q) y[(r0 + q) * c.n + i] = acc[q];
  }
  if (sing) *singular = 1;
}

}  // namespace

void launch_matvec(KernelParams kp, Cloud c, const double* x, double* y, int nrhs, int* singular,
                   cudaStream_t st) {
  if (c.n > 0) matvec_kernel<<<unsigned((c.n + 255) / 256), 256, 0, st>>>(kp, c, x, y, nrhs, singular);
}

void launch_eval(const EvalJob* jobs, const int* tile_ptr, int njobs, int ntiles, KernelParams kp, Cloud cloud,
                 ErrWord* err, int tag, cudaStream_t st) {
  if (ntiles > 0) eval_kernel<<<ntiles, NT, 0, st>>>(jobs, tile_ptr, njobs, kp, cloud, err, tag);
}

void launch_copy(const CopyJob* jobs, const int* tile_ptr, int njobs, int ntiles, cudaStream_t st) {
  if (ntiles > 0) copy_kernel<<<ntiles, NT, 0, st>>>(jobs, tile_ptr, njobs);
}

void launch_accum(const AccJob* jobs, const AccSrc* srcs, const int* tile_ptr, int njobs, int ntiles,
                  cudaStream_t st) {
  if (ntiles > 0) accum_kernel<<<ntiles, NT, 0, st>>>(jobs, srcs, tile_ptr, njobs);
}

void launch_permute_rows(Mat dst, Mat src, const int64_t* idx, int scatter, cudaStream_t st) {
  const int64_t rows = scatter ? src.rows : dst.rows;
  const int64_t tot = rows * dst.cols;
  if (tot > 0) permute_rows_kernel<<<unsigned((tot + 255) / 256), 256, 0, st>>>(dst, src, idx, scatter);
}

void launch_norms(const NormJob* jobs, int njobs, cudaStream_t st) {
  if (njobs > 0) norms_kernel<<<(njobs + 3) / 4, 128, 0, st>>>(jobs, njobs);  // a warp per matrix
}

}  // namespace h2g
