// Host-visible descriptors and launchers of the batched sm_100a kernels.
#pragma once
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace h2g {

void cuda_check(cudaError_t e, const char* what);                   // batch.cu
void smem_attr(const void* kernel, size_t bytes, const char* what);  // batch.cu

// ---- batched GEMM (k_gemm.cu) ---------------------------------------------
// C = [acc ? C : 0] + sum_s A_s * (alpha_s * B_s), each C element accumulated
// with fma over the segments in order and over k in order: the reference's
// gemm_core / gemm_acc order (linalg.cpp:17-62, :86-126).
// B may be generated on the fly from the kernel function (fused
// evaluate-and-project; never materialises far-field blocks):
//   trans = 0: B(l, j) = K(x[rb + l], x[cb + j]) (q of cb + j)
//   trans = 1: B(l, j) = K(x[rb + j], x[cb + l]) (q of cb + l)
// with columns inside mask ranges [a, b) forced to zero (the column zeroing
// of ulv.cpp:365-371 / :433-440).
struct GenB {
  int64_t rb = 0, cb = 0;
  int trans = 0;
  int jstep = 1;  // column j addresses point base + j * jstep (sampled far-field columns)
  int nmask = 0;
  const int2* mask = nullptr;  // device pointer
};
struct GemmSeg {
  Mat A, B;
  double alpha = 1.0;
  int gen = 0;
  GenB g;
};
struct GemmJob {
  Mat C;
  int seg0 = 0, nseg = 0;
  int acc = 0;   // 1: C starts from its own contents
  Mat Cin;       // Cin.p != nullptr (with acc = 1): C starts from Cin instead (same shape)
  int lower = 0; // symmetric C: only entries on or below the diagonal are needed
};
struct GemmTile {
  int job, tm, tn;
};
// tm indexes BM-row tiles; BM = gemm_tile_rows(max C rows in the batch).
int gemm_tile_rows(int max_rows);
void launch_gemm(const GemmJob* jobs, const GemmSeg* segs, const GemmTile* tiles, int ntiles,
                 int bm, KernelParams kp, Cloud cloud, ErrWord* err, int tag, cudaStream_t st,
                 int kind = 0);

// Persistent m8n8k4 kernel for plain operands (k_gemm8.cu): tiles are up to
// 104 rows (a job's 8-row fragments split evenly over gemm_p8_row_tiles) x 128
// columns; GemmTile {job, row tile, column tile}.
int gemm_p8_row_tiles(int rows);
int gemm_p8_col_tiles(int cols);
int gemm_p8_tile_cols();
int gemm_p8_row_end(int rows, int tm);  // one past the last row of row tile tm
// counter: a zeroed device integer of this launch's own (dynamic tile hand-out).
void launch_gemm_p8(const GemmJob* jobs, const GemmSeg* segs, const GemmTile* tiles, int ntiles,
                    int* counter, cudaStream_t st);

// ---- batched kernel-block evaluation (k_eval.cu) ---------------------------
// out(i, j) = K(x[rb + i], x[cb + j]) (assemble_block, kernels.cpp:242-268).
// rstep / cstep > 1 evaluate a strided sample of the row / column points
// (sampled far-field members, Options::sample_cols; not in the reference).
struct EvalJob {
  Mat out;
  int64_t rb, cb;
  int rstep = 1, cstep = 1;
};
// tile_ptr: njobs + 1 prefix sums of the jobs' 64 x 64 tile counts (the kernels find their job by bisection).
void launch_eval(const EvalJob* jobs, const int* tile_ptr, int njobs, int ntiles, KernelParams kp, Cloud cloud,
                 ErrWord* err, int tag, cudaStream_t st);

// ---- batched copies / adds / zero-fills (k_eval.cu) -----------------------
// dst = (add ? dst : 0) + alpha * src (add_block alpha form, matrix.cpp:55-64);
// src.p == nullptr means zero-fill (or identity when ident = 1).
struct CopyJob {
  Mat dst, src;
  double alpha = 1.0;
  int add = 0;
  int ident = 0;
};
void launch_copy(const CopyJob* jobs, const int* tile_ptr, int njobs, int ntiles, cudaStream_t st);

// ---- ordered accumulation: dst = (zero ? 0 : dst) then, for s in order,
// dst = fma(alpha_s, src_s, dst) — a chain of the reference's add_block calls.
struct AccJob {
  Mat dst;
  int src0, nsrc;
  int zero_init;
};
struct AccSrc {
  Mat src;
  double alpha;
};
void launch_accum(const AccJob* jobs, const AccSrc* srcs, const int* tile_ptr, int njobs, int ntiles,
                  cudaStream_t st);

// Row gather/scatter of a multi-column vector block: dst(i, :) = src(idx[i], :)
// (scatter = 0) or dst(idx[i], :) = src(i, :) (scatter = 1).
void launch_permute_rows(Mat dst, Mat src, const int64_t* idx, int scatter, cudaStream_t st);

// Direct-summation y = A x over a cloud (original order), x/y n x nrhs col-major.
void launch_matvec(KernelParams kp, Cloud c, const double* x, double* y, int nrhs, int* singular,
                   cudaStream_t st);

// ---- Frobenius norms, sequential order (norm_frobenius, linalg.cpp:604-609)
struct NormJob {
  Mat a;
  double* out;
};
void launch_norms(const NormJob* jobs, int njobs, cudaStream_t st);

// ---- batched LU with block-local partial pivoting (k_lu.cu) ----------------
// lu_factor (linalg.cpp:352-388) in place on A (n x n); perm[i] = forward map.
struct LuJob {
  Mat A;
  int64_t* perm;
  double tol;
};
void launch_lu(const LuJob* jobs, int njobs, int max_n, ErrWord* err, int tag, cudaStream_t st);
// Blocked LU of a batch of blocks (panels of 32 columns; bitwise equal to
// lu_kernel): amax + identity perm, per panel step: panel factorization (one
// CTA per block), panel-row updates, then a DMMA GEMM trailing update by the
// caller. Blocks smaller than the current panel offset sit the step out.
void launch_lu_amax(const LuJob* jobs, int njobs, double* out, cudaStream_t st);  // out[job]; identity perms
void launch_lu_panel(const LuJob* jobs, int njobs, int max_n, int kb, int nb, const double* amax, ErrWord* err,
                     int tag, cudaStream_t st);
void launch_lu_rows(const LuJob* jobs, int njobs, int max_n, int kb, int nb, cudaStream_t st);

// LuFactors solve family (linalg.cpp:404-559), in place on X.
enum SolveKind : int {
  SOLVE_FULL = 0,         // X <- A^-1 X        (solve_in_place)
  SOLVE_LOWER = 1,        // X <- L^-1 P X      (solve_lower_in_place)
  SOLVE_UPPER = 2,        // X <- U^-1 X        (solve_upper_in_place)
  SOLVE_TRANSPOSE = 3,    // X <- A^-T X        (solve_transpose_in_place)
  SOLVE_RIGHT = 4,        // X <- X A^-1        (solve_right_in_place)
  SOLVE_UPPER_RIGHT = 5,  // X <- X U^-1        (solve_upper_right_in_place)
};
struct SolveJob {
  Mat lu;
  const int64_t* perm;
  Mat X;
  int kind;
};
// Chunks: each CTA handles one (job, chunk) of RHS columns (left solves) or
// rows (right solves); chunk width chosen on the host.
struct SolveChunk {
  int job, c0, nc;
};
void launch_solve(const SolveJob* jobs, const SolveChunk* chunks, int nchunks,
                  size_t smem_doubles, cudaStream_t st);
int solve_chunk_width(int m);

// Blocked left solves: one diagonal block [kb, kb + nb) (nb <= 32) for all
// RHS columns; tiles = (job, 128-column group).
struct TrsmBlockJob {
  Mat lu, X;
  int kb, nb;
  int lower;
};
void launch_trsm_block(const TrsmBlockJob* jobs, const int2* tiles, int ntiles, cudaStream_t st);
// Fused blocked left solve (FULL / LOWER / UPPER): tiles = (job, chunk of
// trsm_chunk_cols() RHS columns); the chunk stays in shared memory.
void launch_trsm_chunk(const SolveJob* jobs, const int2* tiles, int ntiles, int max_m, cudaStream_t st);
int trsm_chunk_cols();
// dst(i, :) = src(perm[i], :); tiles = (job, 4096-element chunk).
struct GatherJob {
  Mat dst, src;
  const int64_t* perm;
};
void launch_gather_rows(const GatherJob* jobs, const int2* tiles, int ntiles, cudaStream_t st);

// ---- batched column-pivoted Householder QR with member stopping (k_qr.cu)
// run_pivoted_qr + form_q (linalg.cpp:137-185, :216-332) as used by
// basis_from_members (compression.cpp:111-146).
struct QrJob {
  Mat A;               // input members concatenation, m x n (any strides)
  int m, n;            // work: column-major m x n, element (i, j) at work[j * ldw + i]
  const int64_t* member_off;  // nmem + 1 offsets (device)
  int nmem;
  double tol, member_tol;
  int cap;             // <= 0: none
  double* work;        // m x n column-major working copy (R), may alias A
  int64_t ldw;
  double* scratch;     // >= 3 n + nmem*2 doubles + m*kmax reflectors
  double* Q;           // output m x m row-major (Q[i*m + j])
  int* rank_out;
  double* dbg = nullptr;  // optional per-job phase cycle counters (profiling)
};
void launch_qr(const QrJob* jobs, int njobs, int max_m, int max_nmem, int cluster,
               cudaStream_t st);
// CTAs per basis (thread-block cluster size) for a batch of njobs bases.
int qr_cluster_size(int njobs, int min_n, int max_m, int max_nmem);
// Co-resident clusters of g CTAs; largest cluster a basis of n columns uses.
int qr_fit(int g, int max_m, int max_nmem);
int qr_max_cluster(int n);
size_t qr_scratch_doubles(int m, int n, int nmem);
// Blocked QR mode (k_qrb.cu): same job interface, reflectors accumulated NB at
// a time; rounding differs from the reference (tolerance parity).
size_t qrb_scratch_doubles(int m, int n, int nmem);
int qrb_max_rows();
void launch_qrb(const QrJob* jobs, int njobs, int max_m, int max_nmem, int cluster, cudaStream_t st);
int qrb_cluster_size(int njobs, int min_n, int max_m, int max_nmem);

// ---- member compression (k_pchol.cu, qr_mode = 2) ------------------------------
// Diagonally pivoted Cholesky of a member's Gram matrix G = M M^T: writes
// count[0] <= kmax columns R with R R^T = G up to a dropped trace <= eta tr(G).
struct PcholJob {
  const double* G;  // m x m column-major
  int64_t ldg;
  double* R;        // m x kmax column-major
  int64_t ldr;
  int m, kmax;
  double eta;
  int* count;
};
void launch_pchol(const PcholJob* jobs, int njobs, int max_m, int max_k, cudaStream_t st);

}  // namespace h2g
