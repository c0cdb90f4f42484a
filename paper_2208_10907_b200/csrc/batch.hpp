// Host-side batching layer: stream-ordered device slabs, matrix handles and
// job builders. A factorization stage (one parallel_for of the reference)
// becomes a handful of batched launches: the host collects every task's
// jobs, uploads the descriptors once and launches one kernel per job type.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "kernels.hpp"

namespace h2g {

void cuda_check(cudaError_t e, const char* what);
// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the
// current device (kept per device and kernel; thread-safe; checked).
void smem_attr(const void* kernel, size_t bytes, const char* what);

using Slab = std::shared_ptr<void>;

// Device memory arena (arena.cu): best-fit blocks carved from a few large
// cudaMalloc'd segments; stream-ordered reuse on the releasing stream.
void* arena_alloc(size_t bytes, cudaStream_t st);  // nullptr when the device is exhausted
void arena_free(void* p, cudaStream_t st);
void arena_stream_gone(cudaStream_t st);  // the stream was synchronised and is being retired
size_t arena_free_bytes();
void trim_device_memory();  // give entirely free segments back to the driver

struct Ctx {
  cudaStream_t stream = nullptr;
  ErrWord* err = nullptr;  // device
  KernelParams kp;
  Cloud cloud;
  // statistics
  int64_t launches = 0;
  double flops = 0;  // algorithmic (reference counting rules)
  double kernel_evals = 0;  // kernel-function entries evaluated (FlopCounter::kernel_evals)
  std::map<std::string, double> phase_flops;
  std::string phase = "other";
  void add_flops(double f) {
    flops += f;
    phase_flops[phase] += f;
  }
  Slab alloc(size_t bytes);
  // Free device memory as the chunking budgets should see it: the driver's, plus the arena's free blocks.
  size_t free_bytes() const;
  // Blocks from the arena (default) or from cudaMallocAsync (H2G_NO_ARENA=1, and
  // factorizations that need most of the device: Problem::factor decides).
  bool use_arena = getenv("H2G_NO_ARENA") == nullptr;
  // Pinned staging arena for descriptor uploads: a copy from pageable memory
  // larger than a few KB makes cudaMemcpyAsync wait for the stream, which
  // serialises host preparation with the GPU. Regions are handed out
  // linearly and recycled at every sync (all staged copies have run).
  char* pin = nullptr;
  size_t pin_cap = 0, pin_head = 0;
  const void* stage(const void* src, size_t bytes);
  char* stage_reserve(size_t bytes);  // a region of the staging arena to fill (nullptr: does not fit)
  // Zeroed device integers, one per launch that hands work out dynamically
  // (k_gemm8.cu): a slab of them, re-zeroed (stream-ordered) when used up.
  Slab tickets;
  int tickets_used = 0;
  int* ticket();
  Ctx() = default;
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
  ~Ctx();
  // QR mode: exact (the reference's rounding, k_qr.cu) or blocked (k_qrb.cu);
  // set per factorization from Options::qr_mode (H2G_QR_MODE overrides).
  bool qr_blocked = false;
  // Compressed QR mode (qr_mode = 2): members replaced by pivoted-Cholesky
  // factors of their Gram matrices before the (blocked) QR (k_pchol.cu).
  bool qr_compress = false;
  // Same mode: wide A^-1 / A^-T applications as GEMMs with explicit inverses
  // (tolerance parity; SolveBatch::run).
  bool fast_solve = false;
  void sync();            // stream sync + error word check
  void check_err();       // throws the reference's message for device errors
  // Names of the LU batches launched since the last sync, by tag: a singular
  // pivot is reported (with the reference's message) at the next sync
  // without making every LU batch a synchronisation point.
  std::map<int, std::vector<std::string>> lu_names;
  int lu_tag = 0;
  // Per-kernel CUDA-event timing on the launching stream (bench roofline).
  struct ProfAgg {
    double ms = 0, flops = 0, bytes = 0;
    int64_t launches = 0;
  };
  struct ProfRec {
    std::string name;
    cudaEvent_t a, b;
    double flops, bytes;
    std::string phase;
  };
  bool prof = false;
  bool prof_detail = getenv("H2G_PROF_DETAIL") != nullptr;  // per-phase kernel names
  std::vector<ProfRec> prec;
  // H2G_TIMELINE: also account the idle time between consecutive profiled
  // kernels as "gap@<phase>" (host-side launch preparation, syncs).
  bool prof_gaps = getenv("H2G_TIMELINE") != nullptr;
  cudaEvent_t last_end = nullptr;
  std::string last_name;
  std::map<std::string, ProfAgg> pagg;
  cudaEvent_t prof_begin();
  void prof_end(const char* name, cudaEvent_t a, double flops, double bytes);
  void prof_resolve();  // after a sync: fold finished records into pagg
};

void host_prof_report();  // H2G_HOST_PROF: host time inside the batch launchers

struct DMat {
  Mat m;
  Slab owner;
  int rows() const { return m.rows; }
  int cols() const { return m.cols; }
};

// Allocate several compact column-major matrices in one slab.
std::vector<DMat> alloc_mats(Ctx& c, const std::vector<std::pair<int, int>>& shapes);
DMat alloc_mat(Ctx& c, int rows, int cols);

struct LuF {
  DMat lu;
  Slab pslab;
  int64_t* perm = nullptr;
  int n() const { return lu.rows(); }
};

template <class T>
T* upload(Ctx& c, const std::vector<T>& v, Slab& keep) {
  if (v.empty()) return nullptr;
  keep = c.alloc(sizeof(T) * v.size());
  cuda_check(cudaMemcpyAsync(keep.get(), c.stage(v.data(), sizeof(T) * v.size()),
                             sizeof(T) * v.size(), cudaMemcpyHostToDevice, c.stream),
             "upload");
  return static_cast<T*>(keep.get());
}

// Several descriptor arrays of one launch in ONE device block and ONE copy
// (an allocation and a cudaMemcpyAsync per array cost ~7 us of host time each,
// four arrays per GEMM launch, ~1,100 launches per factorization).
struct UploadPart {
  const void* src;
  size_t bytes;
  void** dst;  // receives the device address (nullptr when bytes == 0)
};
inline void upload_parts(Ctx& c, Slab& keep, std::initializer_list<UploadPart> parts) {
  size_t total = 0;
  for (auto& p : parts) total += (p.bytes + 255) & ~size_t(255);
  for (auto& p : parts) *p.dst = nullptr;
  if (total == 0) return;
  keep = c.alloc(total);
  char* dev = static_cast<char*>(keep.get());
  char* pin = c.stage_reserve(total);
  size_t off = 0;
  for (auto& p : parts) {
    if (p.bytes == 0) continue;
    *p.dst = dev + off;
    if (pin)
      memcpy(pin + off, p.src, p.bytes);
    else  // larger than the staging arena: one (pageable) copy per array
      cuda_check(cudaMemcpyAsync(dev + off, p.src, p.bytes, cudaMemcpyHostToDevice, c.stream), "upload");
    off += (p.bytes + 255) & ~size_t(255);
  }
  if (pin) cuda_check(cudaMemcpyAsync(dev, pin, total, cudaMemcpyHostToDevice, c.stream), "upload");
}

// ---- GEMM -----------------------------------------------------------------
struct GemmBatch {
  std::vector<GemmJob> jobs;
  std::vector<GemmSeg> segs;
  std::vector<int2> masks;
  std::vector<int> seg_mask_off;  // per seg: offset into masks or -1
  const char* name = nullptr;     // profiling name (default "gemm")
  std::vector<char> lower;        // per job: only tiles touching the lower triangle (symmetric C)
  // Begin a job; add segments with seg()/seg_gen() afterwards.
  void job(Mat C, bool acc) {
    GemmJob j;
    j.C = C;
    j.seg0 = int(segs.size());
    j.nseg = 0;
    j.acc = acc ? 1 : 0;
    jobs.push_back(j);
    lower.push_back(0);
  }
  // C = Cin + sum of segments (the accumulator starts from another matrix).
  void job_from(Mat C, Mat Cin) {
    job(C, true);
    jobs.back().Cin = Cin;
  }
  void seg(Mat A, Mat B, double alpha = 1.0) {
    GemmSeg s;
    s.A = A;
    s.B = B;
    s.alpha = alpha;
    s.gen = 0;
    segs.push_back(s);
    seg_mask_off.push_back(-1);
    jobs.back().nseg++;
  }
  // B generated from the kernel function: trans = 0 -> B(l,j) = K(rb+l, cb+j).
  void seg_gen(Mat A, int64_t rb, int64_t cb, int Bcols, bool trans, double alpha,
               const std::vector<int2>& mask = {}, int jstep = 1) {
    GemmSeg s;
    s.A = A;
    s.B = Mat{nullptr, A.cols, Bcols, 0, 0};
    s.alpha = alpha;
    s.gen = 1;
    s.g.rb = rb;
    s.g.cb = cb;
    s.g.trans = trans ? 1 : 0;
    s.g.jstep = jstep;
    s.g.nmask = int(mask.size());
    seg_mask_off.push_back(mask.empty() ? -1 : int(masks.size()));
    masks.insert(masks.end(), mask.begin(), mask.end());
    segs.push_back(s);
    jobs.back().nseg++;
  }
  void run(Ctx& c, int tag = 0);
  bool empty() const { return jobs.empty(); }
};

// C = op products convenience: C = A * B (fresh) as one job.
inline void gemm1(GemmBatch& b, Mat C, Mat A, Mat B, double alpha = 1.0, bool acc = false) {
  b.job(C, acc);
  b.seg(A, B, alpha);
}

// ---- kernel-block evaluation ------------------------------------------------
struct EvalBatch {
  std::vector<EvalJob> jobs;
  void add(Mat out, int64_t rb, int64_t cb, int rstep = 1, int cstep = 1) {
    jobs.push_back({out, rb, cb, rstep, cstep});
  }
  void run(Ctx& c, int tag = 0);
};

// ---- copies / adds ----------------------------------------------------------
struct CopyBatch {
  std::vector<CopyJob> jobs;
  void copy(Mat dst, Mat src) { jobs.push_back({dst, src, 1.0, 0, 0}); }
  void add(Mat dst, Mat src, double alpha) { jobs.push_back({dst, src, alpha, 1, 0}); }
  void zero(Mat dst) { jobs.push_back({dst, Mat{}, 1.0, 0, 0}); }
  void ident(Mat dst) { jobs.push_back({dst, Mat{}, 1.0, 0, 1}); }
  void run(Ctx& c);
};

// ---- ordered accumulation ---------------------------------------------------------
struct AccBatch {
  std::vector<AccJob> jobs;
  std::vector<AccSrc> srcs;
  void job(Mat dst, bool zero_init) { jobs.push_back({dst, int(srcs.size()), 0, zero_init ? 1 : 0}); }
  void src(Mat s, double alpha) {
    srcs.push_back({s, alpha});
    jobs.back().nsrc++;
  }
  void run(Ctx& c);
};

// ---- norms --------------------------------------------------------------------
struct NormBatch {
  std::vector<Mat> mats;
  int add(Mat a) {
    mats.push_back(a);
    return int(mats.size()) - 1;
  }
  std::vector<double> run(Ctx& c);  // synchronous
};

// ---- LU -------------------------------------------------------------------------
struct LuBatch {
  std::vector<LuJob> jobs;
  std::vector<std::string> names;
  void add(const LuF& f, double tol, std::string name) {
    jobs.push_back({f.lu.m, f.perm, tol});
    names.push_back(std::move(name));
  }
  void run(Ctx& c);
};
LuF alloc_lu(Ctx& c, int n);
std::vector<LuF> alloc_lus(Ctx& c, const std::vector<int>& ns);

// ---- LU solves --------------------------------------------------------------------
struct SolveBatch {
  std::vector<SolveJob> jobs;
  void add(const LuF& f, Mat X, int kind) {
    if (X.rows == 0 || X.cols == 0 || f.n() == 0) return;
    jobs.push_back({f.lu.m, f.perm, X, kind});
  }
  void run(Ctx& c);
};

// ---- pivoted QR bases ----------------------------------------------------------------
// One basis_from_members call: a row-major dim x width concatenation.
struct QrBatch {
  struct Item {
    DMat concat;           // m x n view (row-major)
    int m, n;
    std::vector<int64_t> offs;
    double tol;
    int cap;
    bool inplace;  // factor the concat itself (it is consumed)
    int fixed = 0;  // compressed mode: members [0, fixed) are already compressed
    // Compressed mode: views[s].p != nullptr -> member s is that m x w_s matrix (not
    // stored in the concat): its Gram GEMM reads it in place, only its compressed
    // columns enter the panel.
    std::vector<Mat> views;
  };
  std::vector<Item> items;
  int add(DMat concat, int m, int n, std::vector<int64_t> offs, double tol, int cap,
          bool inplace = false) {
    items.push_back({std::move(concat), m, n, std::move(offs), tol, cap, inplace});
    return int(items.size()) - 1;
  }
  // Runs all QRs (in memory-bounded chunks); returns Q (row-major m x m in a
  // DMat whose view is Q as an m x m matrix) and ranks.
  void run(Ctx& c, std::vector<DMat>& Q, std::vector<int>& rank, size_t mem_budget);
  // Compressed mode only: replace the wide members of every item now (the
  // items then own narrow panels; run() does not compress them again).
  void compress(Ctx& c, size_t mem_budget);
  bool compressed = false;
};

}  // namespace h2g
