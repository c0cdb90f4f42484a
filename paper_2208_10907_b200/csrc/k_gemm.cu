// Batched variable-size FP64 GEMM on the DMMA tensor path, with
// multi-segment accumulation and an optional kernel-function generator for
// the B operand (fused evaluate-and-project).
//
// Bit-exactness: mma.sync.m16n8k16.f64 rounds exactly like sixteen
// sequential FMAs in ascending k (measured on the B200: 0 / 256,000
// mismatches, tools/microbench/dmma16_order.cu), so accumulating the k16
// steps in order over segments in order reproduces the reference gemm_core /
// gemm_acc sequence c = fma(a, alpha*b, c) bit for bit (linalg.cpp:17-62).
// Ragged K is padded with a = +0, b = -0: that product adds an exact -0,
// which leaves every c (including -0.0) unchanged
// (tools/microbench/dmma_zero.cu).
//
// Tiling: CTA tile BM x 64, BK = 16 (one MMA k-step), 2*BM threads, warp
// tile 32 x 32 (2 m16 x 4 n8 fragments). Operands go through two shared-
// memory stages (one barrier per k-step); the next chunk is prefetched into
// registers while the current one feeds the MMAs. Row strides of 132 / 68
// doubles (= 4 mod 16) make every fragment load conflict-free. BM = 128 is
// used when the batch has tall C blocks so a kernel-generated B tile is
// evaluated once per 128 rows.
#include <cstdlib>
#include <type_traits>

#include "kernels.hpp"

namespace h2g {

namespace {

constexpr int BN = 64, BK = 16;

__device__ __forceinline__ bool masked(const GenB& g, int j) {
  for (int t = 0; t < g.nmask; ++t)
    if (j >= g.mask[t].x && j < g.mask[t].y) return true;
  return false;
}

// D = A(16x16) B(16x8) + D. Fragments (PTX ISA, .f64; g = lane>>2, t = lane&3):
// a_i = A[g + 8(i%2)][t + 4(i/2)], b_i = B[t + 4i][g], c_i = C[g + 8(i/2)][2t + i%2].
__device__ __forceinline__ void dmma16(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int BM>
struct Smem {
  static constexpr int SA = BM + 4, SB = BN + 4;  // = 4 (mod 16): conflict-free fragments
  double A[2][BK][SA];
  double B[2][BK][SB];
  unsigned char Bmask[BN];
};

template <int BM>
__global__ void __launch_bounds__(2 * BM) gemm_kernel(const GemmJob* __restrict__ jobs,
                                                  const GemmSeg* __restrict__ segs,
                                                  const GemmTile* __restrict__ tiles,
                                                  KernelParams kp, Cloud cloud, ErrWord* err,
                                                  int tag) {
  constexpr int NT = 2 * BM;
  constexpr int AE = BM * BK / NT;  // A elements per thread per chunk (8)
  constexpr int BE = BK * BN / NT;  // B elements per thread per chunk
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem<BM>& sm = *reinterpret_cast<Smem<BM>*>(smraw);
  const GemmTile tile = tiles[blockIdx.x];
  const GemmJob job = jobs[tile.job];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % (BM / 32), wn = warp / (BM / 32);
  const int g = lane >> 2, t = lane & 3;
  const int m0 = tile.tm * BM, n0 = tile.tn * BN;
  const Mat C = job.C;
  // acc[fm][fn][i]: C row m0 + wm*32 + fm*16 + g + 8(i/2), col n0 + wn*32 + fn*8 + 2t + i%2.
  double acc[2][4][4];
#pragma unroll
  for (int fm = 0; fm < 2; ++fm)
#pragma unroll
    for (int fn = 0; fn < 4; ++fn)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm * 32 + fm * 16 + g + 8 * (i / 2), c = n0 + wn * 32 + fn * 8 + 2 * t + (i % 2);
        acc[fm][fn][i] = (job.acc && r < C.rows && c < C.cols) ? (job.Cin.p ? job.Cin.at(r, c) : C.at(r, c)) : 0.0;
      }
  int singular = 0;
  int buf = 0;
  for (int s = 0; s < job.nseg; ++s) {
    const GemmSeg sg = segs[job.seg0 + s];
    const int K = sg.A.cols;
    if (K == 0) continue;
    const int K16 = (K + 15) & ~15;  // padded with exact no-op (+0, -0) steps
    if (sg.gen) {
      __syncthreads();
      if (threadIdx.x < BN) sm.Bmask[threadIdx.x] = sg.g.nmask ? masked(sg.g, n0 + threadIdx.x) : 0;
      __syncthreads();
    }
    const bool a_colmajor = sg.A.rs == 1;
    const bool b_colmajor = sg.B.rs == 1;
    // Generated B: every thread owns one C column of the tile (nn = tid % BN,
    // NT is a multiple of BN) and BE k-rows per chunk. The column's point is
    // loaded once per segment; a chunk row's point is warp-uniform.
    const int nnT = threadIdx.x % BN;
    const int jT = n0 + nnT;
    bool liveT = false;
    double xT = 0.0, yT = 0.0, zT = 0.0, qT = 0.0;
    if (sg.gen) {
      liveT = jT < C.cols && !sm.Bmask[nnT];
      if (liveT) {
        const int64_t tp = (sg.g.trans ? sg.g.rb : sg.g.cb) + int64_t(jT) * sg.g.jstep;
        xT = cloud.x[tp];
        yT = cloud.y[tp];
        zT = cloud.z[tp];
        qT = cloud.q[tp];
      }
    }
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
      if (sg.gen) {
#pragma unroll
        for (int u = 0; u < BE; ++u) {
          const int l = k0 + threadIdx.x / BN + u * (NT / BN);
          double v = -0.0;  // pad: exact no-op with a = +0
          if (l < K && jT < C.cols) {
            double b = 0.0;
            if (liveT) {
              const int64_t cp = sg.g.trans ? sg.g.cb + l : sg.g.rb + l;
              const double xc = cloud.x[cp], yc = cloud.y[cp], zc = cloud.z[cp];
              // K(i, j): i = rb + row, j = cb + col of the generated block.
              b = sg.g.trans ? kernel_pair(kp, xT, yT, zT, xc, yc, zc, cloud.q[cp], &singular)
                             : kernel_pair(kp, xc, yc, zc, xT, yT, zT, qT, &singular);
            }
            v = sg.alpha * b;  // the reference pre-multiplies B by alpha
          }
          rb[u] = v;
        }
      } else {
#pragma unroll
        for (int u = 0; u < BE; ++u) {
          const int e = threadIdx.x + u * NT;
          int nn, kk;
          if (!b_colmajor) { nn = e % BN; kk = e / BN; } else { kk = e % BK; nn = e / BK; }
          const int l = k0 + kk, j = n0 + nn;
          rb[u] = (l < K && j < C.cols) ? sg.alpha * sg.B.at(l, j) : -0.0;
        }
      }
    };
    auto stash = [&](int bb) {
#pragma unroll
      for (int u = 0; u < AE; ++u) {
        const int e = threadIdx.x + u * NT;
        int mm, kk;
        if (a_colmajor) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
        sm.A[bb][kk][mm] = ra[u];
      }
#pragma unroll
      for (int u = 0; u < BE; ++u) {
        const int e = threadIdx.x + u * NT;
        int nn, kk;
        if (sg.gen || !b_colmajor) { nn = e % BN; kk = e / BN; } else { kk = e % BK; nn = e / BK; }
        sm.B[bb][kk][nn] = rb[u];
      }
    };
    fetch(0);
    __syncthreads();  // previous segment's last reads of this buffer are done
    stash(buf);
    __syncthreads();
    for (int k0 = 0; k0 < K16; k0 += BK) {
      // Register prefetch of the next chunk overlaps this chunk's MMAs. A
      // plain chunk's loads are issued first (their latency hides behind
      // the MMAs); a generated chunk is evaluated after the MMAs are issued,
      // so the evaluation's dependent FP64 chains overlap the tensor work.
      const bool more = k0 + BK < K16;
      if (more && !sg.gen) fetch(k0 + BK);
      double af[2][8];
#pragma unroll
      for (int fm = 0; fm < 2; ++fm)
#pragma unroll
        for (int i = 0; i < 8; ++i)
          af[fm][i] = sm.A[buf][t + 4 * (i / 2)][wm * 32 + fm * 16 + g + 8 * (i % 2)];
#pragma unroll
      for (int fn = 0; fn < 4; ++fn) {
        double bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) bf[i] = sm.B[buf][t + 4 * i][wn * 32 + fn * 8 + g];
#pragma unroll
        for (int fm = 0; fm < 2; ++fm) dmma16(acc[fm][fn], af[fm], bf);
      }
      if (more && sg.gen) fetch(k0 + BK);
      if (more) {
        stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
  if (singular) raise_err(err, 1, tile.job, 0, tag);
#pragma unroll
  for (int fm = 0; fm < 2; ++fm)
#pragma unroll
    for (int fn = 0; fn < 4; ++fn)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm * 32 + fm * 16 + g + 8 * (i / 2), c = n0 + wn * 32 + fn * 8 + 2 * t + (i % 2);
        if (r < C.rows && c < C.cols) C.at(r, c) = acc[fm][fn][i];
      }
}

// ---- warp-specialised BM = 128 path ----------------------------------------
// 8 consumer warps only issue DMMAs (warp tile 32 x 32 as above); 4 producer
// warps fill an NS-stage shared-memory ring of BK = 32 chunks: plain operands
// by cp.async, generated B by evaluating the kernel function (row points of
// the chunk staged in shared memory first). Full/empty mbarriers per stage;
// the producers run up to NS chunks ahead, so the tensor work of one chunk
// overlaps the loads and evaluations of the next ones.
namespace ws {
constexpr int BM = 128, BKW = 32, NSW = 4, NC = 256, NP = 256, NTW = NC + NP;
struct Smem {
  static constexpr int SA = BM + 4, SB = BN + 4;
  double A[NSW][BKW][SA];
  double B[NSW][BKW][SB];
  double P[NSW][BKW][4];  // generated chunk: row points (x, y, z, q)
  double alpha[NSW];
  unsigned long long full[NSW], empty[NSW];
};

__device__ __forceinline__ unsigned su32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
// Arrives when all of this thread's earlier cp.async copies have completed.
__device__ __forceinline__ void mb_arrive_cp_async(unsigned long long* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp8(double* smem, const double* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(su32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp16(double* smem, const double* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(smem)), "l"(gmem) : "memory");
}

// KIND only names the instantiation (0 = general, 1 = member Gram matrices)
// so profiles can tell the launches apart.
template <int KIND>
__global__ void __launch_bounds__(NTW, 1) gemm_ws_kernel(const GemmJob* __restrict__ jobs,
                                                        const GemmSeg* __restrict__ segs,
                                                        const GemmTile* __restrict__ tiles,
                                                        KernelParams kp, Cloud cloud, ErrWord* err, int tag) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& sm = *reinterpret_cast<Smem*>(smraw);
  const GemmTile tile = tiles[blockIdx.x];
  const GemmJob job = jobs[tile.job];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = tile.tm * BM, n0 = tile.tn * BN;
  const Mat C = job.C;
  if (threadIdx.x < NSW) {
    mb_init(&sm.full[threadIdx.x], 2 * NP);  // per producer thread: release arrive + cp.async arrive
    mb_init(&sm.empty[threadIdx.x], NC / 32);  // one per consumer warp
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  int nchunks = 0;
  for (int s = 0; s < job.nseg; ++s) nchunks += (segs[job.seg0 + s].A.cols + BKW - 1) / BKW;

  if (warp >= NC / 32) {
    // ---------------- producers ----------------
    // Register split of the 512-thread CTA (64K registers): producers give
    // theirs to the consumers' accumulators (warpgroup-aligned setmaxnreg).
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
    const int pt = threadIdx.x - NC;  // 0 .. NP-1
    int singular = 0;
    int ps = 0, pk = 0, loaded = -1;
    const int nnT = pt % BN, jT = n0 + nnT;
    bool liveT = false;
    double xT = 0.0, yT = 0.0, zT = 0.0, qT = 0.0;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int st = ch % NSW;
      if (ch >= NSW) mb_wait(&sm.empty[st], ((ch / NSW) - 1) & 1);
      while (pk >= segs[job.seg0 + ps].A.cols) {
        ++ps;
        pk = 0;
      }
      const GemmSeg& sg = segs[job.seg0 + ps];
      const Mat A = sg.A;
      const int K = A.cols;
      const double alpha = sg.alpha;
      const bool gen = sg.gen;
      if (pt == 0) sm.alpha[st] = gen ? 1.0 : alpha;
      const bool a_colmajor = A.rs == 1;
      // Column-major A with 16-byte aligned columns: row pairs by 16-byte
      // cp.async (half the copy instructions).
      const bool a_pairs = a_colmajor && (A.cs % 2 == 0) && ((reinterpret_cast<uintptr_t>(A.p) & 15) == 0);
      if (a_pairs) {
#pragma unroll 2
        for (int u = 0; u < BM * BKW / (2 * NP); ++u) {
          const int e = pt + u * NP;
          const int mm = 2 * (e % (BM / 2)), kk = e / (BM / 2);
          const int i = m0 + mm, l = pk + kk;
          double* dst = &sm.A[st][kk][mm];
          if (l < K && i + 1 < A.rows) {
            cp16(dst, &A.at(i, l));
          } else {
            if (i < A.rows && l < K) cp8(dst, &A.at(i, l)); else dst[0] = 0.0;
            dst[1] = 0.0;
          }
        }
      } else
#pragma unroll 2
      for (int u = 0; u < BM * BKW / NP; ++u) {
        const int e = pt + u * NP;
        int mm, kk;
        if (a_colmajor) { mm = e % BM; kk = e / BM; } else { kk = e % BKW; mm = e / BKW; }
        const int i = m0 + mm, l = pk + kk;
        double* dst = &sm.A[st][kk][mm];
        if (i < A.rows && l < K)
          cp8(dst, &A.at(i, l));
        else
          *dst = 0.0;  // +0: with b = -0 an exact no-op
      }
      if (gen) {
        if (loaded != ps) {
          loaded = ps;
          bool masked_col = false;
          for (int q = 0; q < sg.g.nmask; ++q)
            if (jT >= sg.g.mask[q].x && jT < sg.g.mask[q].y) masked_col = true;
          liveT = jT < C.cols && !masked_col;
          if (liveT) {
            const int64_t tp = (sg.g.trans ? sg.g.rb : sg.g.cb) + int64_t(jT) * sg.g.jstep;
            xT = cloud.x[tp];
            yT = cloud.y[tp];
            zT = cloud.z[tp];
            qT = cloud.q[tp];
          }
        }
        if (pt < 4 * BKW) {  // stage the chunk's row points: thread pt loads component pt % 4 of row pt / 4
          const int l = pk + pt / 4, comp = pt % 4;
          double v = 0.0;
          if (l < K) {
            const int64_t cp = sg.g.trans ? sg.g.cb + l : sg.g.rb + l;
            const double* src = comp == 0 ? cloud.x : comp == 1 ? cloud.y : comp == 2 ? cloud.z : cloud.q;
            v = src[cp];
          }
          sm.P[st][pt / 4][comp] = v;
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(NP) : "memory");
        if (pk + BKW <= K && jT < C.cols) {
          // Full chunk: the BKW * BN / NP entries of this thread are
          // independent chains (sqrt / div / exp); evaluated branch-free per
          // kernel kind so they interleave.
          constexpr int NE = BKW * BN / NP;
          double vals[NE];
          auto gen = [&](auto kind_tag) {
            constexpr int KD = decltype(kind_tag)::value;
            if (sg.g.trans) {
#pragma unroll
              for (int u = 0; u < NE; ++u) {
                const double* q = sm.P[st][pt / BN + u * (NP / BN)];
                vals[u] = kernel_pair_k<KD>(kp, xT, yT, zT, q[0], q[1], q[2], q[3], &singular);
              }
            } else {
#pragma unroll
              for (int u = 0; u < NE; ++u) {
                const double* q = sm.P[st][pt / BN + u * (NP / BN)];
                vals[u] = kernel_pair_k<KD>(kp, q[0], q[1], q[2], xT, yT, zT, qT, &singular);
              }
            }
          };
          if (!liveT) {
#pragma unroll
            for (int u = 0; u < NE; ++u) vals[u] = 0.0;
          } else if (kp.kind == 0) {
            gen(std::integral_constant<int, 0>{});
          } else if (kp.kind == 1) {
            gen(std::integral_constant<int, 1>{});
          } else {
            gen(std::integral_constant<int, 2>{});
          }
#pragma unroll
          for (int u = 0; u < NE; ++u) sm.B[st][pt / BN + u * (NP / BN)][nnT] = alpha * vals[u];
        } else
#pragma unroll 2
        for (int u = 0; u < BKW * BN / NP; ++u) {
          const int kk = pt / BN + u * (NP / BN);
          const int l = pk + kk;
          double v = -0.0;  // pad: exact no-op with a = +0
          if (l < K && jT < C.cols) {
            double b = 0.0;
            if (liveT) {
              const double* q = sm.P[st][kk];
              // K(i, j): i = rb + row, j = cb + col of the generated block.
              b = sg.g.trans ? kernel_pair(kp, xT, yT, zT, q[0], q[1], q[2], q[3], &singular)
                             : kernel_pair(kp, q[0], q[1], q[2], xT, yT, zT, qT, &singular);
            }
            v = alpha * b;  // the reference pre-multiplies B by alpha
          }
          sm.B[st][kk][nnT] = v;
        }
      } else {
        const Mat B = sg.B;
        const bool b_colmajor = B.rs == 1;
        const double pad = alpha < 0.0 ? 0.0 : -0.0;  // -0 after the consumer's alpha scaling
        // Row-major B (columns contiguous, e.g. the Gram's A^T) with 16-byte
        // aligned rows: column pairs by 16-byte cp.async.
        const bool b_pairs = !b_colmajor && B.cs == 1 && (B.rs % 2 == 0) &&
                             ((reinterpret_cast<uintptr_t>(B.p) & 15) == 0);
        if (b_pairs) {
#pragma unroll 4
          for (int u = 0; u < BKW * BN / (2 * NP); ++u) {
            const int e = pt + u * NP;
            const int nn = 2 * (e % (BN / 2)), kk = e / (BN / 2);
            const int l = pk + kk, j = n0 + nn;
            double* dst = &sm.B[st][kk][nn];
            if (l < K && j + 1 < C.cols) {
              cp16(dst, &B.at(l, j));
            } else {
              if (l < K && j < C.cols) cp8(dst, &B.at(l, j)); else dst[0] = pad;
              dst[1] = pad;
            }
          }
        } else
#pragma unroll 4
        for (int u = 0; u < BKW * BN / NP; ++u) {
          const int e = pt + u * NP;
          int nn, kk;
          if (b_colmajor) { kk = e % BKW; nn = e / BKW; } else { nn = e % BN; kk = e / BN; }
          const int l = pk + kk, j = n0 + nn;
          double* dst = &sm.B[st][kk][nn];
          if (l < K && j < C.cols)
            cp8(dst, &B.at(l, j));
          else
            *dst = pad;
        }
      }
      pk += BKW;
      mb_arrive_cp_async(&sm.full[st]);
      mb_arrive(&sm.full[st]);
    }
    if (singular) raise_err(err, 1, tile.job, 0, tag);
    return;
  }

  // ---------------- consumers ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 160;\n" ::: "memory");
  const int wm = warp % (BM / 32), wn = warp / (BM / 32);
  const int g = lane >> 2, t = lane & 3;
  double acc[2][4][4];
#pragma unroll
  for (int fm = 0; fm < 2; ++fm)
#pragma unroll
    for (int fn = 0; fn < 4; ++fn)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm * 32 + fm * 16 + g + 8 * (i / 2), c = n0 + wn * 32 + fn * 8 + 2 * t + (i % 2);
        acc[fm][fn][i] = (job.acc && r < C.rows && c < C.cols) ? (job.Cin.p ? job.Cin.at(r, c) : C.at(r, c)) : 0.0;
      }
  for (int ch = 0; ch < nchunks; ++ch) {
    const int st = ch % NSW;
    mb_wait(&sm.full[st], (ch / NSW) & 1);
    const double al = sm.alpha[st];
    // One A fragment live at a time (the B fragments are re-read per fm):
    // keeps the consumers within the 128 registers of a 512-thread CTA.
#pragma unroll
    for (int ks = 0; ks < BKW; ks += 16) {
#pragma unroll
      for (int fm = 0; fm < 2; ++fm) {
        double af[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = sm.A[st][ks + t + 4 * (i / 2)][wm * 32 + fm * 16 + g + 8 * (i % 2)];
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
          double bf[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) bf[i] = sm.B[st][ks + t + 4 * i][wn * 32 + fn * 8 + g];
          if (al != 1.0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) bf[i] = al * bf[i];
          }
          dmma16(acc[fm][fn], af, bf);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mb_arrive(&sm.empty[st]);
  }
#pragma unroll
  for (int fm = 0; fm < 2; ++fm)
#pragma unroll
    for (int fn = 0; fn < 4; ++fn)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm * 32 + fm * 16 + g + 8 * (i / 2), c = n0 + wn * 32 + fn * 8 + 2 * t + (i % 2);
        if (r < C.rows && c < C.cols) C.at(r, c) = acc[fm][fn][i];
      }
}
}  // namespace ws

template <int BM>
void launch_bm(const GemmJob* jobs, const GemmSeg* segs, const GemmTile* tiles, int ntiles,
               KernelParams kp, Cloud cloud, ErrWord* err, int tag, cudaStream_t st) {
  const int smem = int(sizeof(Smem<BM>));
  smem_attr((const void*)gemm_kernel<BM>, smem, "gemm smem attribute");
  gemm_kernel<BM><<<ntiles, 2 * BM, smem, st>>>(jobs, segs, tiles, kp, cloud, err, tag);
}

}  // namespace

int gemm_tile_rows(int max_rows) { return max_rows > 64 ? 128 : 64; }

void launch_gemm(const GemmJob* jobs, const GemmSeg* segs, const GemmTile* tiles, int ntiles,
                 int bm, KernelParams kp, Cloud cloud, ErrWord* err, int tag, cudaStream_t st, int kind) {
  if (ntiles <= 0) return;
  static const bool use_ws = getenv("H2G_GEMM_CLASSIC") == nullptr;
  if (bm == 128 && use_ws) {
    const int smem = int(sizeof(ws::Smem));
    smem_attr((const void*)ws::gemm_ws_kernel<0>, smem, "gemm_ws smem attribute");
    smem_attr((const void*)ws::gemm_ws_kernel<1>, smem, "gemm_ws smem attribute");
    if (kind == 1)
      ws::gemm_ws_kernel<1><<<ntiles, ws::NTW, smem, st>>>(jobs, segs, tiles, kp, cloud, err, tag);
    else
      ws::gemm_ws_kernel<0><<<ntiles, ws::NTW, smem, st>>>(jobs, segs, tiles, kp, cloud, err, tag);
  } else if (bm == 128)
    launch_bm<128>(jobs, segs, tiles, ntiles, kp, cloud, err, tag, st);
  else
    launch_bm<64>(jobs, segs, tiles, ntiles, kp, cloud, err, tag, st);
}

}  // namespace h2g
