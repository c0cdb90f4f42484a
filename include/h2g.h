/* h2g — C-ABI of the B200-native dependency-free H2-ULV hot path.
 *
 * Plain pointers and sizes only; an opaque handle owns all device memory.
 * Each entry point replaces one piece of the reference's C++ API
 * (/root/reference/proj/include/h2ulv), cited per function. Every function
 * returns 0 on success or nonzero with h2g_last_error() set to the
 * reference's error message (e.g. "singular block in LU of S^RR at step 3",
 * "basis does not absorb fill-in at level 5 block (2,7)").
 * Host/device: pointers are host memory unless the *_dev variant is used.
 * There is no CPU fallback: every call runs sm_100a kernels and fails when no
 * CUDA device is present.
 */
#ifndef H2G_H
#define H2G_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct h2g_problem h2g_problem;

/* KernelSpec (kernels.hpp:15-23): kind 0 = Laplace, 1 = Yukawa,
 * 2 = Gaussian q_j (exp(-alpha_m r^2) + [r == 0] eta_reg) / permittivity_scale
 * (BASELINE configs[2]: alpha_m = 1/0.1, eta_reg = 1e-2, scale 1; not in the
 * reference, so its parity is by residual only). */
typedef struct {
  int32_t kind;
  double alpha_m;
  double permittivity_scale;
  double eta_reg;
} h2g_kernel;

/* FactorOptions (ulv.hpp:29-45) + AdmissibilityRule (geometry.hpp:60-67). */
typedef struct {
  double tol;                   /* RankDecision tol (default 1e-8) */
  int64_t cap;                  /* <= 0: no cap */
  double rr_pivot_tol;          /* 1e-13 */
  int32_t absorb_coupling;      /* 1 */
  double abort_residual_factor; /* 100 */
  int32_t structure;            /* 0 = h2 (strong, nodep), 1 = hss (weak), 2 = blr2 (flat, weak) */
  double eta;                   /* strong admissibility eta (1.0) */
  int64_t qr_mem_budget;        /* bytes of QR working memory per chunk, <= 0: default */
  int32_t qr_mode;              /* 0 = exact (the reference's rounding, bit-exact),
                                   1 = blocked (NB = 32 reflectors per panel update;
                                   same decisions, parity within tolerance),
                                   2 = compressed (each member of width >= 48 replaced by
                                   a pivoted-Cholesky factor of its Gram matrix, then the
                                   blocked QR; same stopping rule, tolerance parity,
                                   meant for tol >= 2.5e-7; below it the blocked
                                   mode runs) */
  int32_t reference_compat;     /* 1 = the reference's h2/nodep assembly, bit for bit,
                                   including its covered-coupling defect (ulv.cpp:424-463,
                                   :583-603); 0 = corrected assembly (covered T terms, far
                                   fills at upper levels, neighbour content from every
                                   overlapping target; oracle/fix_reference.py), accurate
                                   to the tolerance */
} h2g_options;

const char* h2g_last_error(void);
int h2g_version(void);

/* Handle lifetime: replaces constructing Pipeline (report.hpp:73-99). */
int h2g_create(h2g_problem** out);
void h2g_destroy(h2g_problem* p);
int h2g_set_kernel(h2g_problem* p, const h2g_kernel* k);
int h2g_set_options(h2g_problem* p, const h2g_options* o);
/* B200 extension (no reference counterpart): far-field basis members wider than
 * sample_cols columns are replaced by a strided sample of about sample_cols of
 * their columns - the reference concatenates every far-field column
 * (compression.cpp:153-177, ulv.cpp:476-521), O(N) per box. 0 = off (the
 * reference's members, the default); otherwise >= 64. Parity by tolerance. */
int h2g_set_sampling(h2g_problem* p, int64_t sample_cols);

/* Device memory (no reference counterpart): blocks come from a process-wide arena
 * carved out of a few large cudaMalloc'd segments (the first one
 * H2G_ARENA_FRACTION, default 0.7, of the free memory at first use), so a
 * repeated factorization makes no allocator call in its steady state.
 * h2g_trim_memory returns every segment that is entirely free to the driver. */
void h2g_trim_memory(void);

/* build_cluster_tree (geometry.hpp:58) + classify_blocks (hstructure.hpp:55)
 * + materialize_dense (hstructure.hpp:101-103) = Pipeline::build
 * (report.cpp:79-91). xyz is AoS n x 3, q has n charges. */
int h2g_build(h2g_problem* p, int64_t n, const double* xyz, const double* q, int64_t leaf);
int h2g_build_dev(h2g_problem* p, int64_t n, const double* d_xyz, const double* d_q, int64_t leaf);

/* prepare_factor_inputs + factorize = build_and_factorize (ulv.hpp:121-123),
 * Pipeline::factor (report.cpp:93-106). */
int h2g_factor(h2g_problem* p);

/* solve (solve.hpp:10): b, x are n x nrhs column-major in the ORIGINAL order. */
int h2g_solve(h2g_problem* p, int64_t nrhs, const double* b, double* x);
int h2g_solve_dev(h2g_problem* p, int64_t nrhs, const double* d_b, double* d_x);

/* ---- inspection (ClusterTree / BlockStructure / HMatrix / ULVFactors) ---- */
int h2g_levels(h2g_problem* p);
int h2g_tree_perm(h2g_problem* p, int64_t* original_index);          /* geometry.hpp:40 */
int h2g_nodes(h2g_problem* p, int64_t* begin_end, double* center_radius); /* heap order */
int h2g_reordered_points(h2g_problem* p, double* xyz, double* q);
int64_t h2g_list_count(h2g_problem* p, int level, int far); /* -1: bad level */
int h2g_list(h2g_problem* p, int level, int far, int64_t* ptr, int64_t* idx); /* hstructure.hpp:41-42 */
int64_t h2g_near_entries(h2g_problem* p);
int h2g_near_dense(h2g_problem* p, double* out); /* HMatrix::leaf_dense, row-major over blocks */
int h2g_num_factor_levels(h2g_problem* p);
int h2g_factor_level(h2g_problem* p, int li, int64_t* ranks); /* returns tree level, -1: bad li */
int64_t h2g_cutoff(h2g_problem* p, int64_t* dims);           /* count | level << 32 */
int64_t h2g_top_n(h2g_problem* p);
int h2g_top(h2g_problem* p, double* lu, int64_t* perm);      /* ULVFactors::top */
int64_t h2g_basis(h2g_problem* p, int level, int64_t k, int side, double* sq); /* dim | rank<<32, -1: bad index */
double h2g_max_fill_residual(h2g_problem* p);
/* LevelFactors of factorized level li (ulv.hpp:60-68): returns the box count m
 * (-1 on error) and fills dims/ranks (m each, may be NULL) and use_z. */
int h2g_level_dims(h2g_problem* p, int li, int64_t* dims, int64_t* ranks, int32_t* use_z);
/* DenseSystem::block(i, j) of level li (compression.hpp:33): rows/cols out;
 * out (column-major rows x cols) may be NULL to query the shape. */
int h2g_level_block(h2g_problem* p, int li, int64_t i, int64_t j, int64_t* rows, int64_t* cols,
                    double* out);
/* Packed LU factors of level li, box k (linalg.hpp:73-92): which = 0 the
 * cached diagonal LU of the DenseSystem (DenseSystem::diag_lu), 1 the pivot
 * LU of S^RR (ClusterFactors::pivot). n out; lu (n x n) / perm (n) may be NULL. */
int h2g_level_lu(h2g_problem* p, int li, int which, int64_t k, int64_t* n, double* lu, int64_t* perm);
/* ClusterFactors::urs (which 0, rdim x sdim) / lsr (which 1, sdim x rdim). */
int h2g_level_elim(h2g_problem* p, int li, int64_t k, int which, int64_t* rows, int64_t* cols, double* out);
/* assemble_block (kernels.hpp:38-39) of a host cloud (AoS xyz, charges q),
 * evaluated on the device: out = K(rows [r0, r1), cols [c0, c1)), column-major. */
int h2g_assemble_block(const h2g_kernel* k, int64_t n, const double* xyz, const double* q, int64_t r0,
                       int64_t r1, int64_t c0, int64_t c1, double* out);

/* Timings [tree, classify, near, factor, solve] (s); counted flops
 * [fill_precompute, basis, skeleton, factorize, assemble, solve] following the
 * reference ledger rules (flops.hpp); launches = kernels launched so far. */
int h2g_stats(h2g_problem* p, double* t5, double* f6, int64_t* launches);
/* Kernel-function entries evaluated so far (FlopCounter::kernel_evals, flops.hpp). */
int64_t h2g_kernel_evals(h2g_problem* p);

/* Launch everything on a caller-owned cudaStream_t (before h2g_build). */
int h2g_set_stream(h2g_problem* p, void* stream);
/* Device (CUDA-event) seconds of the last [build, factor, solve]. */
int h2g_stats_dev(h2g_problem* p, double* t3);
/* Per-kernel-family CUDA-event timing: enable, reset, and read family idx
 * (returns 0 past the end): total ms, launches, algorithmic flops and bytes. */
int h2g_set_profile(h2g_problem* p, int on);
/* Host wall seconds per reference phase (fill_precompute, basis, skeleton,
 * factorize, assemble); returns 0 past the end. */
int h2g_phase_seconds(h2g_problem* p, int idx, char* name, int name_len, double* sec);
int h2g_reset_profile(h2g_problem* p);
int h2g_kernel_stats(h2g_problem* p, int idx, char* name, int name_len, double* ms,
                     int64_t* launches, double* flops, double* bytes);

/* Matrix-free direct-summation product y = A x on the ORIGINAL ordering
 * (replaces matvec_dense_oracle, solve.cpp:234-239, without its N guard). */
int h2g_matvec(h2g_problem* p, int64_t nrhs, const double* x, double* y);

/* ---- multi-GPU level partition (one process per GPU) ----
 * The reference has no multi-process path (its MPI plan is offline only,
 * partition_plan_json, report.cpp:245-296); these follow that plan: rank r of
 * P owns the contiguous box range [m r / P, m (r+1) / P) of every level with
 * m >= P boxes, coarser levels are replicated. The partitioned stages (basis
 * construction: member concats + pivoted QR) run only on owned boxes and
 * all-gather their outputs, so every rank ends with the single-GPU factors,
 * bit for bit. Set the communicator before h2g_factor. */
typedef struct h2g_comm h2g_comm;
int h2g_nccl_unique_id(void* id128); /* ncclGetUniqueId, 128 bytes (rank 0; broadcast it) */
/* NCCL communicator over the node's GPUs (ncclCommInitRank; collective). */
int h2g_comm_nccl(int nranks, int rank, const void* id128, h2g_comm** out);
/* Host-mediated exchange (tests, or a host transport): fn is called with a
 * host buffer holding this rank's bytes [offs[rank], offs[rank+1]) and must
 * fill in the other ranks' segments (an all-gather-v); returns 0 on success. */
typedef int (*h2g_host_allgather_fn)(void* user, void* host_buf, const int64_t* byte_offs, int nranks);
int h2g_comm_host(int nranks, int rank, h2g_host_allgather_fn fn, void* user, h2g_comm** out);
void h2g_comm_destroy(h2g_comm* c); /* problems using it keep it alive */
/* Partition this problem's factorization over the communicator's ranks
 * (NULL: single GPU). Call before h2g_factor. */
int h2g_set_comm(h2g_problem* p, h2g_comm* c);
/* Box range [lo, hi) of an m-box level owned by rank (host logic, no GPU). */
int h2g_partition_range(int64_t m, int nranks, int rank, int64_t* lo, int64_t* hi);

/* ---- seeded point clouds (host code, no device needed) ----
 * generate_uniform_cube / generate_line / generate_sphere_surface
 * (geometry.cpp:42-95, SplitMix64 prng.hpp:10-29) bit for bit, plus the two
 * BASELINE.json geometries the reference lacks. xyz is AoS n x 3, q = 1.
 * `spheres` is the sphere count (perfect cube) for H2G_GEOM_SPHERE and the
 * ellipsoid count for H2G_GEOM_ELLIPSOIDS; `spacing` is the sphere lattice
 * spacing (RunConfig default 3.0). Errors: h2g_points_last_error(). */
enum {
  H2G_GEOM_CUBE = 0,
  H2G_GEOM_LINE = 1,
  H2G_GEOM_SPHERE = 2,          /* Fibonacci lattice per sphere (the reference's "sphere") */
  H2G_GEOM_UNIFORM_SPHERE = 3,  /* i.i.d. uniform on the unit sphere */
  H2G_GEOM_ELLIPSOIDS = 4       /* union of seeded random ellipsoids */
};
int h2g_generate_points(int32_t geometry, int64_t n, uint64_t seed, int64_t spheres, double spacing,
                        double* xyz, double* q);
const char* h2g_points_last_error(void);

/* ---- single-primitive entry points (kernel parity tests) ---- */
/* lu_factor (linalg.cpp:352-388) on one n x n column-major block. */
int h2g_lu_factor(int64_t n, const double* a, double tol, double* lu, int64_t* perm);
/* basis_from_members (compression.cpp:111-146): concat dim x width column-major,
 * nmem members with offsets; writes square [Qr | Qs] (dim x dim) and rank. */
int h2g_basis_from_members(int64_t dim, int64_t width, const double* concat, int64_t nmem,
                           const int64_t* offsets, double tol, int64_t cap, int64_t min_rank,
                           double* sq, int64_t* rank);
/* The same through a chosen QR mode (h2g_options.qr_mode: 0 exact, 1 blocked,
 * 2 compressed); h2g_basis_from_members is qr_mode 0. */
int h2g_basis_from_members_mode(int64_t dim, int64_t width, const double* concat, int64_t nmem,
                                const int64_t* offsets, double tol, int64_t cap, int64_t min_rank,
                                int32_t qr_mode, double* sq, int64_t* rank);
/* LuFactors solve family (linalg.cpp:404-559) with the given packed factors:
 * kind 0 solve, 1 lower, 2 upper, 3 transpose, 4 right, 5 upper_right. */
int h2g_lu_solve(int64_t n, const double* lu, const int64_t* perm, int kind, int64_t rows,
                 int64_t cols, double* x);
/* gemm (linalg.cpp:86-116): C = alpha op(A) op(B) (+ C when acc). */
int h2g_gemm(int64_t m, int64_t n, int64_t k, double alpha, const double* a, int transa,
             const double* b, int transb, int acc, double* c);
/* The device's restatement of glibc's exp (the Yukawa kernel's std::exp,
 * kernels.cpp:36,58) evaluated on the host: y[i] = exp(x[i]), bitwise equal
 * to glibc >= 2.28 on x86-64 with FMA for |x| < 512 (host code, no device). */
int h2g_exp_glibc_host(int64_t n, const double* x, double* y);

#ifdef __cplusplus
}
#endif
#endif
