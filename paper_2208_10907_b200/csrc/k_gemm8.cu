// Persistent warp-specialised FP64 GEMM for plain (materialised) operands, on
// mma.sync.m8n8k4.f64 fragments.
//
// Why a second GEMM kernel: the wide skeleton products of the factorization
// have C blocks of rank x |J| with rank = cap (100) or two merged ranks (200).
// With the 128-row tiles of k_gemm.cu, 22 % of every issued DMMA is padding.
// The FP64 tensor instruction the hardware executes is DMMA.8x8x4 either way
// (an m16n8k16 is eight of them in SASS), so issuing m8n8k4 directly gives an
// 8-row granularity for free: a CTA tile is up to 13 row fragments (104 rows)
// x 128 columns, and a job's rows are split evenly over its row tiles
// (100 -> 13 fragments, 200 -> 13 + 12).
//
// Bit-exactness is unchanged: m8n8k4 rounds like four sequential FMAs in
// ascending k (tools/microbench/dmma_order.cu), chunks and segments are
// consumed in order, and the K/row/column pads are the same exact no-ops
// (a = +0, b = -0) as in k_gemm.cu, so every C element sees the reference's
// c = fma(a, alpha*b, c) sequence (linalg.cpp:17-62).
//
// Structure: one CTA per SM, taking tiles from a per-launch ticket. 4
// producer warps copy operand chunks of BK = 32 with 16-byte cp.async along
// whichever direction is contiguous in HBM, into a 3-stage ring whose layout
// (k-major or m/n-major, both conflict-free for the fragment loads) is
// recorded per stage; they run ahead across tile boundaries, so a tile's first
// chunks are in flight while the consumers still store the previous tile. 8
// consumer warps each own 16 columns x all row fragments of the tile.
#include <cstdlib>

#include "kernels.hpp"

namespace h2g {

namespace p8 {

constexpr int TM = 104, TN = 128, BK = 32, NS = 3, NC = 256, NP = 128, NT = NC + NP;
constexpr int MF = TM / 8;
constexpr int SK = BK + 4;     // k-major row stride (= 4 mod 16): fragment loads conflict-free
constexpr int SAM = TM + 4;    // A m-major stride (108 = 12 mod 16)
constexpr int SBN = TN + 4;    // B n-major stride (132 = 4 mod 16)
constexpr int A_ST = TM * SK > BK * SAM ? TM * SK : BK * SAM;
constexpr int B_ST = TN * SK > BK * SBN ? TN * SK : BK * SBN;

struct Meta {
  double alpha;
  int a_kmajor, b_kmajor;
  int tile;  // tile this stage belongs to; -1: no more tiles (the consumers leave)
  int nch;   // chunks of that tile; 0: a data-less stage announcing a tile without chunks
};
struct Smem {
  double A[NS][A_ST];
  double B[NS][B_ST];
  Meta meta[NS];
  unsigned long long full[NS], empty[NS];
  int next_tile;
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
// D(8x8) += A(8x4) B(4x8). Fragments (g = lane>>2, t = lane&3):
// a = A[g][t], b = B[t][g], c_i = C[g][2t + i].
__device__ __forceinline__ void dmma8(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Two consecutive elements along the contiguous direction: one 16-byte copy
// when both exist and the source is aligned, else element copies / pads.
__device__ __forceinline__ void copy_pair(double* dst, const double* src, bool ok0, bool ok1, double pad) {
  if (ok1 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    cp16(dst, src);
  } else {
    if (ok0) cp8(dst, src); else dst[0] = pad;
    if (ok1) cp8(dst + 1, src + 1); else dst[1] = pad;
  }
}

// One BK chunk of a warp's 16 columns x MFT row fragments, straight-line (no
// per-fragment branches, so the fragment loads of a k-step are issued ahead of
// its DMMAs). Strides are in bytes; operand layouts vary per ring stage.
// Fragments beyond the tile's own row count read unwritten shared memory:
// row r of A only ever reaches row r of C, and those rows are never stored.
__device__ __forceinline__ double lds64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
template <int MFT>
__device__ __forceinline__ void consume(double (&acc)[MF][2][2], unsigned ap, unsigned sAm8, unsigned sAk4,
                                        unsigned bp, unsigned sBn8, unsigned sBk4, double al) {
  // Rolling prefetch: fragment fm of the next k-step is loaded right after
  // this step's DMMAs on it are issued, so a load has a whole k-step to land.
  double a[MFT];
#pragma unroll
  for (int fm = 0; fm < MFT; ++fm) a[fm] = lds64(ap + fm * sAm8);
  double b0 = lds64(bp), b1 = lds64(bp + sBn8);
#pragma unroll
  for (int k4 = 0; k4 < BK / 4; ++k4) {
    double nb0 = 0.0, nb1 = 0.0;
    if (k4 + 1 < BK / 4) {
      nb0 = lds64(bp + (k4 + 1) * sBk4);
      nb1 = lds64(bp + sBn8 + (k4 + 1) * sBk4);
    }
    b0 = al * b0;  // the reference pre-multiplies B by alpha (1.0 * b is exact)
    b1 = al * b1;
#pragma unroll
    for (int fm = 0; fm < MFT; ++fm) {
      dmma8(acc[fm][0], a[fm], b0);
      dmma8(acc[fm][1], a[fm], b1);
      if (k4 + 1 < BK / 4) a[fm] = lds64(ap + fm * sAm8 + (k4 + 1) * sAk4);
    }
    b0 = nb0;
    b1 = nb1;
  }
}

struct TileGeom {
  int m0, mf, n0;
};
__device__ __forceinline__ TileGeom geom(const GemmTile& t, int rows) {
  const int nt = (rows + TM - 1) / TM, F = (rows + 7) >> 3;
  const int f0 = t.tm * F / nt, f1 = (t.tm + 1) * F / nt;
  return TileGeom{8 * f0, f1 - f0, t.tn * TN};
}

// What a consumer needs of its tile, read through volatile pointers so that a
// second call re-loads instead of keeping the first one's registers alive.
struct CInfo {
  int lower;
  double* p;
  int64_t rs, cs;
  const double* ip;  // initial accumulator source (C itself, or the job's Cin)
  int64_t irs, ics;
  int rows, cols, m0, mf, n0, acc, seg0, nseg;
};
__device__ __forceinline__ CInfo load_info(const GemmJob* jobs, const GemmTile* tiles, int ti) {
  const volatile GemmTile* vt = tiles + ti;
  GemmTile tile;
  tile.job = vt->job;
  tile.tm = vt->tm;
  tile.tn = vt->tn;
  const volatile GemmJob* vj = jobs + tile.job;
  CInfo ci;
  ci.p = vj->C.p;
  ci.rs = vj->C.rs;
  ci.cs = vj->C.cs;
  ci.rows = vj->C.rows;
  ci.cols = vj->C.cols;
  ci.acc = vj->acc;
  ci.lower = vj->lower;
  ci.ip = vj->Cin.p ? vj->Cin.p : ci.p;
  ci.irs = vj->Cin.p ? vj->Cin.rs : ci.rs;
  ci.ics = vj->Cin.p ? vj->Cin.cs : ci.cs;
  ci.seg0 = vj->seg0;
  ci.nseg = vj->nseg;
  const TileGeom tg = geom(tile, ci.rows);
  ci.m0 = tg.m0;
  ci.mf = tg.mf;
  ci.n0 = tg.n0;
  return ci;
}

// A consumer warp's share of its tile: columns [n0 + nb, + 16) and the row
// fragments it needs. For a symmetric job the fragments entirely above the
// warp's first column are skipped (returns the number skipped).
__device__ __forceinline__ int warp_window(CInfo& ci, int nb) {
  int fs = 0;
  if (ci.lower) {
    fs = (ci.n0 + nb - ci.m0) >> 3;
    fs = fs < 0 ? 0 : (fs > ci.mf ? ci.mf : fs);
    ci.m0 += 8 * fs;
    ci.mf -= fs;
  }
  return fs;
}

__global__ void __launch_bounds__(NT, 1) gemm_p8_kernel(const GemmJob* __restrict__ jobs,
                                                       const GemmSeg* __restrict__ segs,
                                                       const GemmTile* __restrict__ tiles, int ntiles,
                                                       int* __restrict__ counter) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& sm = *reinterpret_cast<Smem*>(smraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < NS) {
    mb_init(&sm.full[threadIdx.x], 2 * NP);   // per producer thread: release arrive + cp.async arrive
    mb_init(&sm.empty[threadIdx.x], NC / 32);  // one per consumer warp
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  unsigned gc = 0;  // chunk counter over all of this CTA's tiles (ring position)

  if (warp >= NC / 32) {
    // ---------------- producers ----------------
    const int pt = threadIdx.x - NC;
    // Tiles are handed out dynamically (one atomic per tile): their K extents
    // differ by up to 4x inside a launch, and a static round-robin left 5 % of
    // the SM-cycles idle at the end of the largest launch.
    auto announce = [&](int tile_id, int nch) {  // a data-less stage
      const int st = gc % NS;
      if (gc >= NS) mb_wait(&sm.empty[st], ((gc / NS) - 1) & 1);
      if (pt == 0) sm.meta[st] = Meta{1.0, 1, 1, tile_id, nch};
      mb_arrive_cp_async(&sm.full[st]);
      mb_arrive(&sm.full[st]);
      ++gc;
    };
    while (true) {
      if (pt == 0) sm.next_tile = atomicAdd(counter, 1);
      asm volatile("bar.sync 1, %0;\n" ::"n"(NP) : "memory");
      const int ti = sm.next_tile;
      asm volatile("bar.sync 1, %0;\n" ::"n"(NP) : "memory");  // everyone has read it before the next overwrite
      if (ti >= ntiles) {
        announce(-1, 0);
        break;
      }
      const GemmTile tile = tiles[ti];
      const GemmJob job = jobs[tile.job];
      const TileGeom tg = geom(tile, job.C.rows);
      const int mrows = tg.mf * 8, ccols = job.C.cols;
      int nch = 0;
      for (int s = 0; s < job.nseg; ++s) nch += (segs[job.seg0 + s].A.cols + BK - 1) / BK;
      if (nch == 0) {
        announce(ti, 0);
        continue;
      }
      for (int s = 0; s < job.nseg; ++s) {
        const GemmSeg& sg = segs[job.seg0 + s];
        const Mat A = sg.A, B = sg.B;
        const int K = A.cols;
        const double alpha = sg.alpha;
        const double bpad = alpha < 0.0 ? 0.0 : -0.0;  // -0 after the consumer's alpha scaling
        const bool a_km = A.rs != 1, b_km = B.rs == 1 || B.cs != 1;
        for (int pk = 0; pk < K; pk += BK, ++gc) {
          const int st = gc % NS;
          if (gc >= NS) mb_wait(&sm.empty[st], ((gc / NS) - 1) & 1);
          if (pt == 0) sm.meta[st] = Meta{alpha, a_km ? 1 : 0, b_km ? 1 : 0, ti, nch};
          double* As = sm.A[st];
          double* Bs = sm.B[st];
          if (a_km) {
            // k contiguous (row-major A) or general strides: As[row][k].
            const int kk = (pt & 15) * 2, l = pk + kk;
            const bool pairs = A.cs == 1;
            for (int row = pt >> 4; row < mrows; row += NP / 16) {
              const int i = tg.m0 + row;
              double* dst = &As[row * SK + kk];
              const bool in = i < A.rows;
              if (pairs) {
                copy_pair(dst, A.p + int64_t(i) * A.rs + l, in && l < K, in && l + 1 < K, 0.0);
              } else {
                if (in && l < K) cp8(dst, &A.at(i, l)); else dst[0] = 0.0;
                if (in && l + 1 < K) cp8(dst + 1, &A.at(i, l + 1)); else dst[1] = 0.0;
              }
            }
          } else {
            // m contiguous (column-major A): As[k][m].
            for (int kk = pt >> 3; kk < BK; kk += NP / 8) {
              const int l = pk + kk;
              const double* col = A.p + int64_t(l) * A.cs;
              for (int mm = (pt & 7) * 2; mm < mrows; mm += 16) {
                const int i = tg.m0 + mm;
                copy_pair(&As[kk * SAM + mm], col + i, l < K && i < A.rows, l < K && i + 1 < A.rows, 0.0);
              }
            }
          }
          if (b_km) {
            // k contiguous (column-major B) or general strides: Bs[n][k].
            const int kk = (pt & 15) * 2, l = pk + kk;
            const bool pairs = B.rs == 1;
#pragma unroll 2
            for (int nn = pt >> 4; nn < TN; nn += NP / 16) {
              const int j = tg.n0 + nn;
              double* dst = &Bs[nn * SK + kk];
              const bool in = j < ccols;
              if (pairs) {
                copy_pair(dst, B.p + int64_t(j) * B.cs + l, in && l < K, in && l + 1 < K, bpad);
              } else {
                if (in && l < K) cp8(dst, &B.at(l, j)); else dst[0] = bpad;
                if (in && l + 1 < K) cp8(dst + 1, &B.at(l + 1, j)); else dst[1] = bpad;
              }
            }
          } else {
            // n contiguous (row-major B): Bs[k][n].
            for (int kk = pt >> 3; kk < BK; kk += NP / 8) {
              const int l = pk + kk;
              const double* rowp = B.p + int64_t(l) * B.rs;
#pragma unroll 2
              for (int nn = (pt & 7) * 2; nn < TN; nn += 16) {
                const int j = tg.n0 + nn;
                copy_pair(&Bs[kk * SBN + nn], rowp + j, l < K && j < ccols, l < K && j + 1 < ccols, bpad);
              }
            }
          }
          mb_arrive_cp_async(&sm.full[st]);
          mb_arrive(&sm.full[st]);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  // Register budget: 104 accumulator + 26 fragment registers leave little
  // else, so nothing about the tile stays live across the chunk loop: the
  // epilogue re-reads the descriptors (volatile loads, a few L2 hits per tile).
  const int g = lane >> 2, t = lane & 3;
  // Column group of the warp: warps w and w + 4 share a scheduler, and in a
  // symmetric tile the work falls with the column index, so the second four
  // take the groups in reverse (group s and 7 - s per scheduler).
  const int nb = 16 * (warp < 4 ? warp : 11 - warp);
  while (true) {
    // The first stage of a tile names it (and says how many chunks follow).
    int st = gc % NS;
    mb_wait(&sm.full[st], (gc / NS) & 1);
    const int ti = sm.meta[st].tile;
    const int nch = sm.meta[st].nch;
    if (ti < 0) break;  // no more tiles
    double acc[MF][2][2];
    int mfc = 0, fskip = 0;
    {
      CInfo ci = load_info(jobs, tiles, ti);
      fskip = warp_window(ci, nb);
      const int c0 = ci.n0 + nb;
      mfc = (c0 < ci.cols && ci.mf > 0) ? (ci.mf >= 10 ? ci.mf : ((ci.mf + 1) & ~1)) : 0;  // 0: idle warp
      const int64_t rstep = 8 * ci.irs;
#pragma unroll
      for (int fn = 0; fn < 2; ++fn)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int c = c0 + fn * 8 + 2 * t + i;
          const double* cp = ci.ip + int64_t(ci.m0 + g) * ci.irs + int64_t(c) * ci.ics;
#pragma unroll
          for (int fm = 0; fm < MF; ++fm) {
            const int r = ci.m0 + fm * 8 + g;
            acc[fm][fn][i] = (ci.acc && fm < ci.mf && r < ci.rows && c < ci.cols) ? cp[fm * rstep] : 0.0;
          }
        }
    }
    if (nch == 0) {  // the announcing stage carried no data
      __syncwarp();
      if (lane == 0) mb_arrive(&sm.empty[st]);
      ++gc;
    }
    for (int ch = 0; ch < nch; ++ch, ++gc) {
      st = gc % NS;
      if (ch > 0) mb_wait(&sm.full[st], (gc / NS) & 1);
      if (mfc > 0) {
        const Meta me = sm.meta[st];
        const unsigned sAm = me.a_kmajor ? SK : 1, sAk = me.a_kmajor ? 1 : SAM;
        const unsigned sBn = me.b_kmajor ? SK : 1, sBk = me.b_kmajor ? 1 : SBN;
        const unsigned ap = su32(sm.A[st]) + 8 * ((g + 8 * fskip) * sAm + t * sAk);
        const unsigned bp = su32(sm.B[st]) + 8 * ((nb + g) * sBn + t * sBk);
        const unsigned sAm8 = 64 * sAm, sAk4 = 32 * sAk, sBn8 = 64 * sBn, sBk4 = 32 * sBk;
        switch (mfc) {
          case 2: consume<2>(acc, ap, sAm8, sAk4, bp, sBn8, sBk4, me.alpha); break;
          case 4: consume<4>(acc, ap, sAm8, sAk4, bp, sBn8, sBk4, me.alpha); break;
          case 6: consume<6>(acc, ap, sAm8, sAk4, bp, sBn8, sBk4, me.alpha); break;
          case 8: consume<8>(acc, ap, sAm8, sAk4, bp, sBn8, sBk4, me.alpha); break;
          case 10: consume<10>(acc, ap, sAm8, sAk4, bp, sBn8, sBk4, me.alpha); break;
          case 11: consume<11>(acc, ap, sAm8, sAk4, bp, sBn8, sBk4, me.alpha); break;
          case 12: consume<12>(acc, ap, sAm8, sAk4, bp, sBn8, sBk4, me.alpha); break;
          default: consume<13>(acc, ap, sAm8, sAk4, bp, sBn8, sBk4, me.alpha); break;
        }
      }
      __syncwarp();
      if (lane == 0) mb_arrive(&sm.empty[st]);
    }
    if (mfc > 0) {
      CInfo ci = load_info(jobs, tiles, ti);
      warp_window(ci, nb);
      const int c0 = ci.n0 + nb;
      const int64_t rstep = 8 * ci.rs;
#pragma unroll
      for (int fn = 0; fn < 2; ++fn)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int c = c0 + fn * 8 + 2 * t + i;
          double* cp = ci.p + int64_t(ci.m0 + g) * ci.rs + int64_t(c) * ci.cs;
#pragma unroll
          for (int fm = 0; fm < MF; ++fm) {
            const int r = ci.m0 + fm * 8 + g;
            if (fm < ci.mf && r < ci.rows && c < ci.cols) cp[fm * rstep] = acc[fm][fn][i];
          }
        }
    }
  }
}

}  // namespace p8

int gemm_p8_row_tiles(int rows) { return (rows + p8::TM - 1) / p8::TM; }
int gemm_p8_col_tiles(int cols) { return (cols + p8::TN - 1) / p8::TN; }
int gemm_p8_tile_cols() { return p8::TN; }
int gemm_p8_row_end(int rows, int tm) {
  const int nt = (rows + p8::TM - 1) / p8::TM, F = (rows + 7) >> 3;
  const int end = 8 * ((tm + 1) * F / nt);
  return end < rows ? end : rows;
}

void launch_gemm_p8(const GemmJob* jobs, const GemmSeg* segs, const GemmTile* tiles, int ntiles,
                    int* counter, cudaStream_t st) {
  if (ntiles <= 0) return;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int smem = int(sizeof(p8::Smem));
  smem_attr((const void*)p8::gemm_p8_kernel, smem, "gemm_p8 smem attribute");
  p8::gemm_p8_kernel<<<ntiles < sms ? ntiles : sms, p8::NT, smem, st>>>(jobs, segs, tiles, ntiles, counter);
}

}  // namespace h2g
