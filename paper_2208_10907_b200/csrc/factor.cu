// Level-parallel (dependency-free) H2-ULV factorization and solve on the GPU.
//
// Host C++ walks the reference's NodepDriver schedule (ulv.cpp:293-760) and
// turns every parallel_for stage into batched sm_100a launches (batch.hpp).
// All numerics run on the device; the host only enumerates jobs from the
// integer block structure and reads back the discrete ranks once per basis
// stage. Within a stage every element sees the reference's rounding sequence,
// so factors and solutions are bitwise equal to the reference (Laplace).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <future>
#include <set>
#include <stdexcept>

#include "h2.hpp"

namespace h2g {

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct PhaseTimer {
  Ctx& c;
  Stats& st;
  std::string prev;
  double t0;
  PhaseTimer(Ctx& c_, Stats& s, const char* name) : c(c_), st(s), prev(c_.phase), t0(now_s()) {
    c.phase = name;
  }
  ~PhaseTimer() {
    st.phase_seconds[c.phase] += now_s() - t0;
    c.phase = prev;
  }
};

// CUDA-event interval on the problem stream (device time of a phase).
struct DevTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit DevTimer(cudaStream_t st) : s(st) {
    cuda_check(cudaEventCreate(&a), "event");
    cuda_check(cudaEventCreate(&b), "event");
    cuda_check(cudaEventRecord(a, s), "event");
  }
  double stop() {
    float ms = 0;
    cuda_check(cudaEventRecord(b, s), "event");
    cuda_check(cudaEventSynchronize(b), "event");
    cuda_check(cudaEventElapsedTime(&ms, a, b), "event");
    return ms * 1e-3;
  }
  ~DevTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

}  // namespace

bool Structure::is_near(int l, int64_t i, int64_t j) const {
  const int64_t* b = near(l, i);
  return std::binary_search(b, b + nnear(l, i), j);
}
bool Structure::is_far(int l, int64_t i, int64_t j) const {
  const int64_t* b = far(l, i);
  return std::binary_search(b, b + nfar(l, i), j);
}

Problem::Problem() {
  cuda_check(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking), "stream");
  // Keep freed stream-ordered memory in the pool: the factorization reuses
  // tens of GB of panel memory level after level, and re-mapping it from
  // the driver at every synchronisation costs seconds.
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "device");
  cudaMemPool_t pool;
  cuda_check(cudaDeviceGetDefaultMemPool(&pool, dev), "mempool");
  uint64_t keep = ~uint64_t(0);
  cuda_check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "mempool attr");
  cuda_check(cudaMalloc(&c.err, sizeof(ErrWord)), "err");
  cuda_check(cudaMemset(c.err, 0, sizeof(ErrWord)), "err");
}

void Problem::use_stream(cudaStream_t s) {
  c.tickets.reset();  // (re-created, and zeroed, on the new stream)
  cuda_check(cudaStreamSynchronize(c.stream), "stream");
  arena_stream_gone(c.stream);
  if (own_stream_) cudaStreamDestroy(c.stream);
  c.stream = s;
  own_stream_ = false;
}

Problem::~Problem() {
  // Release device objects before the stream they free on.
  U.clear();
  V.clear();
  levels.clear();
  top = LuF{};
  near.clear();
  near_slab.reset();
  orig_slab.reset();
  c.tickets.reset();
  if (c.stream) cudaStreamSynchronize(c.stream);
  arena_stream_gone(c.stream);  // its released blocks are now usable from any stream
  cudaFree(c.err);
  if (c.stream && own_stream_) cudaStreamDestroy(c.stream);
}

// Memory regime, decided before a build allocates anything. The arena cannot
// re-map: a factorization whose piece sets (rank x N per box, three alive at
// the upper levels) take most of the device needs the driver
// pool's ability to serve a 50 GB request from scattered free memory. Such
// problems go back to the stream-ordered allocator (after handing the arena's
// free segments back to the driver).
void Problem::choose_allocator(int64_t n, int64_t leaf) {
  size_t fr = 0, tot = 0;
  cuda_check(cudaMemGetInfo(&fr, &tot), "meminfo");
  const double boxes = double(int64_t(1) << tree_levels(n, leaf));
  const double rank = opt.cap > 0 ? double(opt.cap) : double(leaf);
  const double piece_set = 8.0 * rank * double(n) * boxes;
  const bool roomy = 3.5 * piece_set < 0.5 * double(tot);
  if (c.use_arena && !roomy) {
    c.use_arena = false;
    c.sync();
    trim_device_memory();
  } else if (!c.use_arena && roomy && getenv("H2G_NO_ARENA") == nullptr) {
    c.use_arena = true;
  }
}

// Pipeline::build (report.cpp:79-91): tree, classification, near field.
void Problem::build(const double* d_xyz, const double* d_q, int64_t n, int64_t leaf) {
  // A rebuild invalidates any previous factorization.
  factored = false;
  built = false;
  U.clear();
  V.clear();
  levels.clear();
  top = LuF{};
  near.clear();
  near_slab.reset();
  orig_slab.reset();
  if (leaf >= 2 && n >= 2 * leaf) choose_allocator(n, leaf);
  double t0 = now_s();
  DevTimer dt(c.stream);
  build_tree_device(T, d_xyz, d_q, n, leaf, c.stream);
  const int L = T.levels;
  const int64_t nn = (int64_t(1) << (L + 1)) - 1;
  be.resize(2 * nn);
  cuda_check(cudaMemcpyAsync(be.data(), T.be, sizeof(int64_t) * 2 * nn, cudaMemcpyDeviceToHost,
                             c.stream),
             "be d2h");
  std::vector<double> hq(size_t(std::max<int64_t>(n, 1)));
  if (n > 0)
    cuda_check(cudaMemcpyAsync(hq.data(), d_q, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, c.stream),
               "q d2h");
  c.sync();
  uniform_q = n > 0 && std::all_of(hq.begin(), hq.begin() + n, [&](double v) { return v == hq[0]; });
  double t1 = now_s();
  classify_device(T, opt.eta, opt.structure != 0 ? 1 : 0, S, c.stream);
  if (opt.structure == 2) {
    // BLR^2 (classify_blocks, hstructure.cpp:75-87): flat, every leaf pair
    // classified at the leaf level with the weak rule -- the diagonal block is
    // dense, every other leaf pair is far -- and no coarser levels.
    const int L = T.levels;
    for (int l = 1; l < L; ++l) {
      const int64_t m = int64_t(1) << l;
      S.level[l].near_ptr.assign(m + 1, 0);
      S.level[l].far_ptr.assign(m + 1, 0);
      S.level[l].near_idx.clear();
      S.level[l].far_idx.clear();
    }
    const int64_t m = int64_t(1) << L;
    auto& lv = S.level[L];
    lv.near_ptr.resize(m + 1);
    lv.far_ptr.resize(m + 1);
    lv.near_idx.resize(m);
    lv.far_idx.resize(m * (m - 1));
    for (int64_t i = 0; i <= m; ++i) {
      lv.near_ptr[i] = i;
      lv.far_ptr[i] = i * (m - 1);
    }
    for (int64_t i = 0; i < m; ++i) {
      lv.near_idx[i] = i;
      int64_t t = i * (m - 1);
      for (int64_t j = 0; j < m; ++j)
        if (j != i) lv.far_idx[t++] = j;
    }
  }
  double t2 = now_s();
  c.cloud = Cloud{T.x, T.y, T.z, T.q, n};
  {
    orig_slab = c.alloc(sizeof(double) * 4 * n);
    double* o = static_cast<double*>(orig_slab.get());
    DMat src{Mat{const_cast<double*>(d_xyz), int(n), 3, 3, 1}, Slab()};
    CopyBatch cb;
    cb.copy(Mat{o, int(n), 3, 1, n}, src.m);
    cb.run(c);
    cuda_check(cudaMemcpyAsync(o + 3 * n, d_q, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream), "q");
    orig = Cloud{o, o + n, o + 2 * n, o + 3 * n, n};
  }
  // materialize_dense (hstructure.cpp:142-164): one arena, blocks aligned with near CSR.
  const auto& LP = S.level[L];
  std::vector<std::pair<int, int>> shapes;
  for (int64_t i = 0; i < (int64_t(1) << L); ++i)
    for (int64_t t = LP.near_ptr[i]; t < LP.near_ptr[i + 1]; ++t)
      shapes.push_back({int(range_size(L, i)), int(range_size(L, LP.near_idx[t]))});
  near = alloc_mats(c, shapes);
  near_slab = near.empty() ? Slab() : near[0].owner;
  EvalBatch eb;
  size_t at = 0;
  for (int64_t i = 0; i < (int64_t(1) << L); ++i)
    for (int64_t t = LP.near_ptr[i]; t < LP.near_ptr[i + 1]; ++t, ++at)
      eb.add(near[at].m, range_begin(L, i), range_begin(L, LP.near_idx[t]));
  {
    PhaseTimer pt(c, stats, "assemble");
    eb.run(c);
    c.sync();
  }
  stats.t_tree = t1 - t0;
  stats.t_classify = t2 - t1;
  stats.t_near = now_s() - t2;
  stats.t_build_dev = dt.stop();
  c.prof_resolve();
  built = true;
}

// ---------------------------------------------------------------------------
namespace {

struct Driver {
  Problem& P;
  Ctx& c;
  const Structure& S;
  const Options& opt;
  int L;
  // child big layer (points x rank), per cluster of the previously processed level
  std::vector<Mat> Ubig, Vbig;
  std::vector<DMat> big_owner;
  std::vector<PieceMap> carried;
  // Single-GPU: the two children's carried pieces toward a target are
  // allocated as the row blocks of one parent-stacked matrix (stacked_[parent]),
  // so build_upper_pieces takes the stack as it is instead of copying it.
  std::vector<PieceMap> stacked_;
  // Allocate carried pieces for boxes [0, m) of a level: keys[t] = (box, target),
  // rows[t] = the piece's row count; out[t] is a view into its parent's stack.
  std::vector<DMat> alloc_stacked(int64_t m, const std::vector<std::pair<int64_t, TargetKey>>& keys,
                                  const std::vector<int>& rows) {
    std::map<std::pair<int64_t, TargetKey>, std::array<int, 2>> h;  // (parent, tk) -> child row counts
    for (size_t t = 0; t < keys.size(); ++t) {
      auto& e = h.try_emplace({keys[t].first >> 1, keys[t].second}, std::array<int, 2>{-1, -1}).first->second;
      e[keys[t].first & 1] = rows[t];
    }
    std::vector<std::pair<int, int>> shapes;
    for (auto& [key, e] : h) {
      if (e[0] < 0 || e[1] < 0) throw std::logic_error("alloc_stacked: a child piece is missing");
      shapes.push_back({e[0] + e[1], int(rs(key.second.first, key.second.second))});
    }
    auto mats = alloc_mats(c, shapes);
    stacked_.assign(size_t(m / 2), {});
    std::map<std::pair<int64_t, TargetKey>, size_t> at;
    size_t q = 0;
    for (auto& [key, e] : h) {
      stacked_[size_t(key.first)][key.second] = mats[q];
      at[key] = q++;
    }
    std::vector<DMat> out(keys.size());
    for (size_t t = 0; t < keys.size(); ++t) {
      const std::pair<int64_t, TargetKey> key{keys[t].first >> 1, keys[t].second};
      const DMat& S2 = mats[at.at(key)];
      const int r0 = (keys[t].first & 1) ? h.at(key)[0] : 0;
      out[t].m = Mat{S2.m.p + r0, rows[t], S2.m.cols, 1, S2.m.cs};
      out[t].owner = S2.owner;
    }
    return out;
  }

  Driver(Problem& p) : P(p), c(p.c), S(p.S), opt(p.opt), L(p.T.levels) {}

  int64_t rb(int l, int64_t i) const { return P.range_begin(l, i); }
  int64_t rs(int l, int64_t i) const { return P.range_size(l, i); }

  static int find_near(const Structure& S, int l, int64_t i, int64_t j) {
    const int64_t* b = S.near(l, i);
    const int64_t n = S.nnear(l, i);
    const int64_t* it = std::lower_bound(b, b + n, j);
    if (it == b + n || *it != j) return -1;
    return int(S.level[l].near_ptr[i] + (it - b));
  }
  Mat block(const SysL& sys, int64_t i, int64_t j) const {
    const int t = find_near(S, sys.lvl, i, j);
    if (t < 0) throw std::out_of_range("DenseSystem::block: no dense block");
    return sys.blocks[t].m;
  }

  std::vector<TargetKey> ancestor_far_partners(int lvl, int64_t K) const {
    std::vector<TargetKey> out;
    int64_t a = K;
    for (int l2 = lvl - 1; l2 >= 1; --l2) {
      a >>= 1;
      for (int64_t t = 0; t < S.nfar(l2, a); ++t) out.push_back({l2, S.far(l2, a)[t]});
    }
    return out;
  }
  std::vector<TargetKey> targets_of(int lvl, int64_t k) const {
    std::vector<TargetKey> t;
    for (int64_t x = 0; x < S.nfar(lvl, k); ++x) t.push_back({lvl, S.far(lvl, k)[x]});
    for (auto& p : ancestor_far_partners(lvl, k)) t.push_back(p);
    return t;
  }
  TargetKey covering_target(int lvl, int64_t i, int64_t j) const {
    int64_t a = i, b = j;
    int tl = lvl;
    while (tl > 1) {
      a >>= 1;
      b >>= 1;
      --tl;
      if (S.is_far(tl, a, b)) return {tl, b};
      if (S.is_near(tl, a, b)) throw std::logic_error("covering_target: covering pair is dense");
    }
    throw std::logic_error("covering_target: no covering far block");
  }
  // Columns of target range jr covered by level-lvl near partners of p
  // (ulv.cpp:365-371 / :433-440); all_zero when one equals jr.
  std::vector<int2> mask_for(int lvl, int64_t p, int64_t jb, int64_t je, bool& all_zero) const {
    std::vector<int2> m;
    all_zero = false;
    for (int64_t t = 0; t < S.nnear(lvl, p); ++t) {
      const int64_t jn = S.near(lvl, p)[t];
      const int64_t a = rb(lvl, jn), b = a + rs(lvl, jn);
      if (a >= jb && b <= je) {
        m.push_back(make_int2(int(a - jb), int(b - jb)));
        if (a == jb && b == je) all_zero = true;
      }
    }
    return m;
  }

  // Targets of a piece map whose column ranges overlap target tk's range
  // (tree ranges nest, so each is inside tk's range or contains it): the
  // column slice [src, src + len) of that piece lands at [dst, dst + len).
  struct Overlap {
    TargetKey tk;
    int src, dst, len;
  };
  std::vector<Overlap> overlapping(const PieceMap& pm, const TargetKey& tk) const {
    std::vector<Overlap> out;
    const int64_t jb = rb(tk.first, tk.second), je = jb + rs(tk.first, tk.second);
    for (auto& [tk2, pc] : pm) {
      const int64_t b2 = rb(tk2.first, tk2.second), e2 = b2 + rs(tk2.first, tk2.second);
      const int64_t lo = std::max(jb, b2), hi = std::min(je, e2);
      if (lo < hi) out.push_back({tk2, int(lo - b2), int(lo - jb), int(hi - lo)});
    }
    return out;
  }

  // ---- precompute_fillins (compression.cpp:55-109) -------------------------
  FillSet precompute_fillins(SysL& sys) {
    PhaseTimer pt(c, P.stats, "fill_precompute");
    FillSet out;
    const int l = sys.lvl;
    const int64_t m = sys.m;
    if (!sys.offdiag) return out;
    sys.diag_lu = alloc_lus(c, sys.dims);
    {
      CopyBatch cb;
      LuBatch lb;
      for (int64_t p = 0; p < m; ++p) {
        cb.copy(sys.diag_lu[p].lu.m, block(sys, p, p));
        lb.add(sys.diag_lu[p], opt.rr_pivot_tol, "diagonal block " + std::to_string(p));
      }
      cb.run(c);
      lb.run(c);
    }
    // W_pj = A_pp^-1 A_pj for every off-diagonal near block.
    std::map<std::pair<int64_t, int64_t>, DMat> W;
    {
      std::vector<std::pair<int64_t, int64_t>> keys;
      std::vector<std::pair<int, int>> shapes;
      for (int64_t p = 0; p < m; ++p)
        for (int64_t t = 0; t < S.nnear(l, p); ++t) {
          const int64_t j = S.near(l, p)[t];
          if (j == p) continue;
          keys.push_back({p, j});
          shapes.push_back({sys.dims[p], sys.dims[j]});
        }
      auto mats = alloc_mats(c, shapes);
      CopyBatch cb;
      SolveBatch sb;
      for (size_t t = 0; t < keys.size(); ++t) {
        cb.copy(mats[t].m, block(sys, keys[t].first, keys[t].second));
        sb.add(sys.diag_lu[keys[t].first], mats[t].m, SOLVE_FULL);
        W[keys[t]] = mats[t];
      }
      cb.run(c);
      sb.run(c);
    }
    // Targets: (c, j) sharing a common near p (both != p).
    std::set<std::pair<int64_t, int64_t>> targets;
    for (int64_t p = 0; p < m; ++p)
      for (int64_t a = 0; a < S.nnear(l, p); ++a) {
        const int64_t cc = S.near(l, p)[a];
        if (cc == p) continue;
        for (int64_t b = 0; b < S.nnear(l, p); ++b) {
          const int64_t j = S.near(l, p)[b];
          if (j == p) continue;
          targets.insert({cc, j});
        }
      }
    std::vector<std::pair<int, int>> shapes;
    for (auto& t : targets) shapes.push_back({sys.dims[t.first], sys.dims[t.second]});
    auto mats = alloc_mats(c, shapes);
    GemmBatch gb;
    size_t at = 0;
    for (auto& t : targets) {
      const auto [cc, j] = t;
      gb.job(mats[at].m, false);
      for (int64_t a = 0; a < S.nnear(l, cc); ++a) {
        const int64_t p = S.near(l, cc)[a];
        if (p == cc || p == j) continue;
        auto it = W.find({p, j});
        if (it == W.end()) continue;
        gb.seg(block(sys, cc, p), it->second.m, -1.0);
      }
      out[t] = mats[at++];
    }
    gb.run(c);
    return out;
  }

  // ---- basis_from_members (compression.cpp:111-146) batched -----------------
  // A member list is realised straight into a column-major dim x width
  // concat that the QR then factors in place. Boxes are processed in chunks so the
  // concatenations (O(N) wide in the reference's exact-member scheme) never
  // exceed the memory budget.
  struct Members {
    int dim = 0;
    int width = 0;
    std::vector<int64_t> offs{0};
    DMat concat;
    int fixed = 0;  // compressed mode: members [0, fixed) are already compressed
    Mat slice(int off, int w) const {
      const int ld = std::max(2, (dim + 1) & ~1);
      return Mat{concat.m.p + int64_t(off) * ld, dim, w, 1, ld};
    }
    // Compressed mode: member s read in place from views[s] (see QrBatch::Item).
    std::vector<Mat> views;
    void set_view(size_t s, const Mat& v) {
      if (views.size() < offs.size() - 1) views.resize(offs.size() - 1);
      views[s] = v;
    }
    int add(int w) {
      const int off = width;
      width += w;
      offs.push_back(width);
      return off;
    }
    // Column-major (ld = dim): each member column is contiguous, so the QR's
    // column tiles are contiguous HBM ranges.
    size_t bytes() const {
      return sizeof(double) * size_t(std::max(2, (dim + 1) & ~1)) * size_t(std::max(width, 1));
    }
  };
  // Column stride = dim rounded up to even: 16-byte aligned column segments
  // for the QR's TMA bulk copies.
  static int ldc(int dim) { return std::max(2, (dim + 1) & ~1); }
  void alloc_concat(Members& M) {
    M.concat = alloc_mat(c, ldc(M.dim), std::max(M.width, 1));
    M.concat.m = Mat{M.concat.m.p, M.dim, M.width, 1, ldc(M.dim)};
  }

  // Sampled far-field members (Options::sample_cols > 0): a member of w
  // columns wider than sample_cols keeps every step-th column.
  struct Samp {
    int step, count;
  };
  Samp samp(int64_t w) const {
    if (opt.sample_cols <= 0 || w <= opt.sample_cols) return {1, int(w)};
    const int step = int((w + opt.sample_cols - 1) / opt.sample_cols);
    return {step, int((w + step - 1) / step)};
  }
  static Mat sample_cols_view(const Mat& a, const Samp& sp) {
    return Mat{a.p, a.rows, sp.count, a.rs, a.cs * sp.step};
  }

  using FillFn = std::function<void(int64_t, int64_t)>;
  using SinkFn = std::function<void(int64_t, const Mat&, int, const Mat&, int)>;

  // For boxes [0, m): allocate concats chunk by chunk, fill(k0, k1), QR all
  // of the chunk's row (and col) concats in place, then sink(k, Qrow, rrow,
  // Qcol, rcol) per box while the Q's are alive.
  void run_bases(std::vector<Members>& rows, std::vector<Members>* cols, const FillFn& fill,
                 const SinkFn& sink, const std::function<void()>& flush = {}) {
    const int64_t m = int64_t(rows.size());
    if (P.comm && P.comm->partitioned(m))
      run_bases_partitioned(rows, cols, fill, sink, flush);
    else
      run_bases_range(rows, cols, fill, sink, flush, 0, m);
  }

  // Multi-GPU: this rank builds and factors the concats of its own box range
  // only; the Q's (and ranks) land in one box-ordered slab, so each owner's
  // boxes are one contiguous segment, all-gathered in place; then every rank
  // runs the sink for every box exactly as the single-GPU path does.
  void run_bases_partitioned(std::vector<Members>& rows, std::vector<Members>* cols,
                             const FillFn& fill, const SinkFn& sink,
                             const std::function<void()>& flush) {
    Comm& cm = *P.comm;
    const int64_t m = int64_t(rows.size());
    const int nq = cols ? 2 : 1;
    std::vector<int64_t> qoff(m + 1, 0);
    for (int64_t k = 0; k < m; ++k) qoff[k + 1] = qoff[k] + int64_t(nq) * rows[k].dim * rows[k].dim;
    Slab qslab = c.alloc(sizeof(double) * size_t(std::max<int64_t>(qoff[m], 1)));
    Slab rslab = c.alloc(sizeof(int) * size_t(nq * m));
    double* qa = static_cast<double*>(qslab.get());
    int* ra = static_cast<int*>(rslab.get());
    auto qview = [&](int64_t k, int side) {
      const int d = rows[k].dim;
      return Mat{qa + qoff[k] + int64_t(side) * d * d, d, d, std::max(d, 1), 1};  // row-major like QrBatch
    };
    std::vector<int> rk(size_t(nq * m), 0);
    CopyBatch qcopies;
    run_bases_range(rows, cols, fill,
                    [&](int64_t k, const Mat& qu, int ru, const Mat& qv, int rv) {
                      if (rows[k].dim > 0) qcopies.copy(qview(k, 0), qu);
                      rk[size_t(nq * k)] = ru;
                      if (cols) {
                        if (rows[k].dim > 0) qcopies.copy(qview(k, 1), qv);
                        rk[size_t(nq * k + 1)] = rv;
                      }
                    },
                    [&]() {
                      qcopies.run(c);
                      qcopies.jobs.clear();
                    },
                    cm.lo(m), cm.hi(m));
    cuda_check(cudaMemcpyAsync(ra, c.stage(rk.data(), sizeof(int) * rk.size()), sizeof(int) * rk.size(),
                               cudaMemcpyHostToDevice, c.stream),
               "ranks h2d");
    std::vector<int64_t> qb(cm.size + 1), rb(cm.size + 1);
    for (int r = 0; r <= cm.size; ++r) {
      const int64_t k = r == cm.size ? m : cm.lo(m, r);
      qb[r] = int64_t(sizeof(double)) * qoff[k];
      rb[r] = int64_t(sizeof(int)) * nq * k;
    }
    {
      PhaseTimer pt(c, P.stats, "exchange");
      cm.allgatherv(qa, qb, c.stream);
      cm.allgatherv(ra, rb, c.stream);
    }
    cuda_check(cudaMemcpyAsync(rk.data(), ra, sizeof(int) * rk.size(), cudaMemcpyDeviceToHost, c.stream),
               "ranks d2h");
    c.sync();
    for (int64_t k = 0; k < m; ++k)
      sink(k, qview(k, 0), rk[size_t(nq * k)], cols ? qview(k, 1) : Mat{}, cols ? rk[size_t(nq * k + 1)] : 0);
    if (flush) flush();
  }

  // Multi-GPU: the box range this rank computes in a partitioned stage of an
  // m-box level ([0, m) when single-GPU or the level is replicated).
  std::pair<int64_t, int64_t> own_range(int64_t m) const {
    if (P.comm && P.comm->partitioned(m)) return {P.comm->lo(m), P.comm->hi(m)};
    return {0, m};
  }

  // All-gather matrices allocated by one alloc_mats call in non-decreasing
  // box order (box[t] = box of mats[t]): every owner's matrices are one
  // contiguous byte range of the slab.
  void exchange_mats(const std::vector<DMat>& mats, const std::vector<int64_t>& box, int64_t m) {
    if (!(P.comm && P.comm->partitioned(m)) || mats.empty()) return;
    Comm& cm = *P.comm;
    PhaseTimer pt(c, P.stats, "exchange");
    char* base = reinterpret_cast<char*>(mats[0].m.p);
    const DMat& last = mats.back();
    const int64_t end = reinterpret_cast<char*>(last.m.p) - base +
                        int64_t(sizeof(double)) * int64_t((size_t(last.m.rows) * last.m.cols + 3) & ~size_t(3));
    std::vector<int64_t> offs(cm.size + 1, end);
    size_t t = 0;
    for (int r = 0; r < cm.size; ++r) {
      const int64_t lo = cm.lo(m, r);
      while (t < mats.size() && box[t] < lo) ++t;
      if (t < mats.size()) offs[r] = reinterpret_cast<char*>(mats[t].m.p) - base;
    }
    cm.allgatherv(base, offs, c.stream);
  }

  // Boxes [kb, ke): chunked concat fill -> in-place QR -> sink.
  void run_bases_range(std::vector<Members>& rows, std::vector<Members>* cols, const FillFn& fill,
                       const SinkFn& sink, const std::function<void()>& flush, int64_t kb, int64_t ke) {
    if (c.qr_compress) {
      run_bases_range_compressed(rows, cols, fill, sink, flush, kb, ke);
      return;
    }
    const int64_t m = ke;
    int64_t k0 = kb;
    while (k0 < m) {
      size_t bytes = 0;
      int64_t k1 = k0;
      while (k1 < m) {
        size_t need = rows[k1].bytes() + (cols ? (*cols)[k1].bytes() : 0);
        need += need / 16 + 65536;
        if (k1 > k0 && bytes + need > opt.qr_mem_budget) break;
        bytes += need;
        ++k1;
      }
      const bool hp = getenv("H2G_HOST_PROF") != nullptr;
      double ht0 = now_s();
      for (int64_t k = k0; k < k1; ++k) {
        alloc_concat(rows[k]);
        if (cols) alloc_concat((*cols)[k]);
      }
      double ht1 = now_s();
      fill(k0, k1);
      if (hp) c.sync();
      double ht2 = now_s();
      QrBatch qb;
      for (int64_t k = k0; k < k1; ++k)
        qb.add(rows[k].concat, rows[k].dim, rows[k].width, rows[k].offs, opt.tol, opt.cap, true);
      if (cols)
        for (int64_t k = k0; k < k1; ++k)
          qb.add((*cols)[k].concat, (*cols)[k].dim, (*cols)[k].width, (*cols)[k].offs, opt.tol,
                 opt.cap, true);
      std::vector<DMat> Q;
      std::vector<int> rank;
      qb.run(c, Q, rank, opt.qr_mem_budget);
      double ht3 = now_s();
      const int64_t nk = k1 - k0;
      for (int64_t k = k0; k < k1; ++k) {
        const Mat qc = cols ? Q[nk + (k - k0)].m : Mat{};
        const int rc = cols ? rank[nk + (k - k0)] : 0;
        sink(k, Q[k - k0].m, rank[k - k0], qc, rc);
      }
      // One launch for the whole chunk's sink copies; the Q's and concats
      // are released stream-ordered behind them (cudaFreeAsync).
      if (flush) flush();
      if (hp) c.sync();
      double ht4 = now_s();
      for (int64_t k = k0; k < k1; ++k) {
        rows[k].concat = DMat{};
        if (cols) (*cols)[k].concat = DMat{};
      }
      if (hp) {
        c.sync();
        fprintf(stderr, "HOSTPROF run_bases boxes=%ld alloc %.3f fill %.3f qr %.3f sink %.3f free %.3f\n",
                long(k1 - k0), ht1 - ht0, ht2 - ht1, ht3 - ht2, ht4 - ht3, now_s() - ht4);
      }
      k0 = k1;
    }
  }

  // Compressed mode: the member panels are filled and compressed chunk by
  // chunk (the wide panels never coexist beyond the memory budget), then one
  // QR launch factors every compressed panel of the range and the sinks run.
  void run_bases_range_compressed(std::vector<Members>& rows, std::vector<Members>* cols,
                                  const FillFn& fill, const SinkFn& sink,
                                  const std::function<void()>& flush, int64_t kb, int64_t ke) {
    QrBatch all;
    all.compressed = true;
    int64_t k0 = kb;
    while (k0 < ke) {
      size_t bytes = 0;
      int64_t k1 = k0;
      while (k1 < ke) {
        size_t need = rows[k1].bytes() + (cols ? (*cols)[k1].bytes() : 0);
        need += need / 16 + 65536;
        if (k1 > k0 && bytes + need > opt.qr_mem_budget) break;
        bytes += need;
        ++k1;
      }
      for (int64_t k = k0; k < k1; ++k) {
        alloc_concat(rows[k]);
        if (cols) alloc_concat((*cols)[k]);
      }
      fill(k0, k1);
      QrBatch qb;
      for (int64_t k = k0; k < k1; ++k) {
        qb.add(rows[k].concat, rows[k].dim, rows[k].width, rows[k].offs, opt.tol, opt.cap, true);
        qb.items.back().fixed = rows[k].fixed;
        qb.items.back().views = rows[k].views;
        rows[k].concat = DMat{};
      }
      if (cols)
        for (int64_t k = k0; k < k1; ++k) {
          qb.add((*cols)[k].concat, (*cols)[k].dim, (*cols)[k].width, (*cols)[k].offs, opt.tol, opt.cap, true);
          (*cols)[k].concat = DMat{};
        }
      qb.compress(c, opt.qr_mem_budget);
      if (save_rows_) {  // keep a copy of each compressed row panel (the QR consumes it)
        CopyBatch cb;
        for (int64_t k = k0; k < k1; ++k) {
          const auto& it = qb.items[size_t(k - k0)];
          saved_rows_[size_t(k)].offs = it.offs;
          saved_rows_[size_t(k)].dim = it.m;
          saved_rows_[size_t(k)].width = it.n;
          saved_rows_[size_t(k)].concat = alloc_mat(c, ldc(it.m), std::max(it.n, 1));
          saved_rows_[size_t(k)].concat.m = Mat{saved_rows_[size_t(k)].concat.m.p, it.m, it.n, 1, ldc(it.m)};
          if (it.n > 0 && it.m > 0) cb.copy(saved_rows_[size_t(k)].concat.m, it.concat.m);
        }
        cb.run(c);
      }
      for (auto& it : qb.items) all.items.push_back(std::move(it));
      k0 = k1;
    }
    // all.items: per chunk, the chunk's rows then its cols; map back per box.
    std::vector<size_t> at_row(size_t(ke - kb)), at_col(size_t(ke - kb));
    {
      size_t t = 0;
      int64_t a = kb;
      while (a < ke) {
        // recover the chunk boundaries in the same way as above
        size_t bytes = 0;
        int64_t b = a;
        while (b < ke) {
          size_t need = rows[b].bytes() + (cols ? (*cols)[b].bytes() : 0);
          need += need / 16 + 65536;
          if (b > a && bytes + need > opt.qr_mem_budget) break;
          bytes += need;
          ++b;
        }
        for (int64_t k = a; k < b; ++k) at_row[size_t(k - kb)] = t++;
        if (cols)
          for (int64_t k = a; k < b; ++k) at_col[size_t(k - kb)] = t++;
        a = b;
      }
    }
    std::vector<DMat> Q;
    std::vector<int> rank;
    all.run(c, Q, rank, opt.qr_mem_budget);
    for (int64_t k = kb; k < ke; ++k) {
      const size_t r = at_row[size_t(k - kb)];
      const Mat qc = cols ? Q[at_col[size_t(k - kb)]].m : Mat{};
      const int rc = cols ? rank[at_col[size_t(k - kb)]] : 0;
      sink(k, Q[r].m, rank[r], qc, rc);
    }
    if (flush) flush();
  }

  // Compressed mode, leaf coupling: the provisional pass's compressed row
  // panels, reused as the first members of the final row panels.
  bool save_rows_ = false;
  std::vector<Members> saved_rows_;

  // Off-diagonal fills of a level indexed by row and by column, each list in
  // the FillSet's (map) order, so that "for every fill with key.first == i"
  // walks the same entries in the same order without scanning the map.
  struct FillIndex {
    std::vector<std::vector<const DMat*>> by_row, by_col;
  };
  static FillIndex index_fills(const FillSet& fills, int64_t m) {
    FillIndex x;
    x.by_row.resize(m);
    x.by_col.resize(m);
    for (auto& [key, F] : fills) {
      if (key.first == key.second) continue;
      x.by_row[key.first].push_back(&F);
      x.by_col[key.second].push_back(&F);
    }
    return x;
  }

  // Rank-equalised square bases (compression.cpp:224-229 / ulv.cpp:507-511):
  // the min_rank extension of basis_from_members re-splits the same Q.
  SinkFn square_sink(std::vector<Basis>& Ub, std::vector<Basis>& Vb, CopyBatch& cb) {
    return [this, &Ub, &Vb, &cb](int64_t k, const Mat& qu, int ru, const Mat& qv, int rv) {
      const int dim = qu.rows;
      const int r = std::min(dim, std::max(ru, rv));
      auto sq = alloc_mats(c, {{dim, dim}, {dim, dim}});
      for (int side = 0; side < 2; ++side) {
        Basis& B = side == 0 ? Ub[k] : Vb[k];
        B.SQ = sq[side];
        B.dim = dim;
        B.rank = r;
        const Mat q = side == 0 ? qu : qv;
        if (dim == 0) continue;
        if (dim - r > 0) cb.copy(B.SQ.m.sub(0, 0, dim, dim - r), q.sub(0, r, dim, dim - r));
        if (r > 0) cb.copy(B.SQ.m.sub(0, dim - r, dim, r), q.sub(0, 0, dim, r));
      }
    };
  }

  // ---- build_leaf_bases (compression.cpp:193-234) ---------------------------
  void build_leaf_bases(SysL& sys, const FillSet& fills) {
    PhaseTimer pt(c, P.stats, "basis");
    const int64_t m = sys.m;
    const bool coupling = opt.absorb_coupling && opt.structure == 0 && sys.offdiag;
    // Row members: fills (i, j != i) | A(i, far j) | A(i, ancestor far J) [+ coupling].
    std::vector<Members> rows(m), cols(m);
    const FillIndex FI = index_fills(fills, m);
    for (int64_t i = 0; i < m; ++i) {
      Members& R = rows[i];
      R.dim = sys.dims[i];
      for (const DMat* F : FI.by_row[i]) R.add(F->cols());
      for (int64_t t = 0; t < S.nfar(L, i); ++t) R.add(samp(rs(L, S.far(L, i)[t])).count);
      for (auto [l2, J] : ancestor_far_partners(L, i)) R.add(samp(rs(l2, J)).count);
      Members& C = cols[i];
      C.dim = sys.dims[i];
      for (const DMat* F : FI.by_col[i]) C.add(F->rows());
      for (int64_t t = 0; t < S.nfar(L, i); ++t) C.add(samp(rs(L, S.far(L, i)[t])).count);
      for (auto [l2, I] : ancestor_far_partners(L, i)) C.add(samp(rs(l2, I)).count);
    }
    auto fill_base_rows = [&](std::vector<Members>& R, int64_t k0, int64_t k1, CopyBatch& cb,
                              EvalBatch& eb) {
      for (int64_t i = k0; i < k1; ++i) {
        int off = 0;
        for (const DMat* F : FI.by_row[i]) {
          cb.copy(R[i].slice(off, F->cols()), F->m);
          off += F->cols();
        }
        for (int64_t t = 0; t < S.nfar(L, i); ++t) {
          const int64_t j = S.far(L, i)[t];
          const Samp sp = samp(rs(L, j));
          eb.add(R[i].slice(off, sp.count), rb(L, i), rb(L, j), 1, sp.step);
          off += sp.count;
        }
        for (auto [l2, J] : ancestor_far_partners(L, i)) {
          const Samp sp = samp(rs(l2, J));
          eb.add(R[i].slice(off, sp.count), rb(L, i), rb(l2, J), 1, sp.step);
          off += sp.count;
        }
      }
    };
    std::vector<DMat> X(m);
    std::vector<int> provR(m, 0);
    std::vector<std::vector<std::pair<int64_t, int>>> couple_at(m);
    bool reuse = false;
    bool col_reuse = false;
    std::vector<int> col_reuse_off;
    if (coupling) {
      // Provisional row bases (compression.cpp:203-211), kept as Qs_p.
      std::vector<Members> prow = rows;
      std::vector<DMat> provQs(m);
      CopyBatch provcopies;
      // Compressed mode: the provisional members' compressed panels are kept
      // and become the first members of the final row panels (the final
      // row members are the provisional ones plus the coupling products).
      reuse = c.qr_compress;
      save_rows_ = reuse;
      if (reuse) saved_rows_.assign(size_t(m), Members{});
      run_bases(prow, nullptr,
                [&](int64_t k0, int64_t k1) {
                  CopyBatch cb;
                  EvalBatch eb;
                  fill_base_rows(prow, k0, k1, cb, eb);
                  cb.run(c);
                  eb.run(c);
                },
                [&](int64_t p, const Mat& q, int r, const Mat&, int) {
                  provR[p] = r;
                  provQs[p] = alloc_mat(c, sys.dims[p], r);
                  if (r > 0) provcopies.copy(provQs[p].m, q.sub(0, 0, sys.dims[p], r));
                },
                [&]() {
                  provcopies.run(c);
                  provcopies.jobs.clear();
                });
      save_rows_ = false;
      if (reuse && P.uniform_q && getenv("H2G_NO_COL_REUSE") == nullptr) {
        // Equal charges: the column members A(j, i)^T (j far) and A(I, i)^T (I
        // an ancestor's far partner) equal the row members A(i, j), A(i, I)
        // bit for bit and come in the same order, so the final column panels
        // take the provisional pass's compressed far/ancestor members first
        // (already compressed) and their own fill members after them.
        const auto [lo, hi] = own_range(m);
        col_reuse_off.assign(size_t(m), 0);
        for (int64_t i = lo; i < hi; ++i) {
          const Members& sv = saved_rows_[size_t(i)];
          const size_t nf = FI.by_row[i].size();
          const size_t nmem = sv.offs.size() - 1;
          Members C;
          C.dim = sys.dims[i];
          for (size_t s = nf; s < nmem; ++s) C.add(int(sv.offs[s + 1] - sv.offs[s]));
          C.fixed = int(nmem - nf);
          for (const DMat* F : FI.by_col[i]) C.add(F->rows());
          col_reuse_off[size_t(i)] = int(sv.offs[nf]);
          cols[i] = std::move(C);
        }
        col_reuse = true;
      }
      if (reuse) {
        const auto [lo, hi] = own_range(m);
        for (int64_t i = 0; i < m; ++i) {
          Members R;
          R.dim = sys.dims[i];
          if (i >= lo && i < hi) {
            R.offs = saved_rows_[size_t(i)].offs;
            R.width = saved_rows_[size_t(i)].width;
          }
          R.fixed = int(R.offs.size()) - 1;
          rows[i] = std::move(R);
        }
      }
      // X_p = A_pp^-1 Qs_p; coupling member A_ip X_p for p in near(i).
      SolveBatch sb;
      for (int64_t p = 0; p < m; ++p) {
        X[p] = provQs[p];
        if (provR[p] > 0) sb.add(sys.diag_lu[p], X[p].m, SOLVE_FULL);
      }
      sb.run(c);
      for (int64_t i = 0; i < m; ++i)
        for (int64_t t = 0; t < S.nnear(L, i); ++t) {
          const int64_t p = S.near(L, i)[t];
          if (p == i || provR[p] == 0) continue;
          couple_at[i].push_back({p, rows[i].add(provR[p])});
        }
    }
    CopyBatch sqcopies;
    run_bases(rows, &cols,
              [&](int64_t k0, int64_t k1) {
                CopyBatch cb;
                EvalBatch eb;
                GemmBatch gb;
                if (reuse) {
                  for (int64_t i = k0; i < k1; ++i) {
                    const Members& sv = saved_rows_[size_t(i)];
                    if (sv.width > 0 && sv.dim > 0) cb.copy(rows[i].slice(0, sv.width), sv.concat.m);
                  }
                } else {
                  fill_base_rows(rows, k0, k1, cb, eb);
                }
                for (int64_t i = k0; i < k1; ++i)
                  for (auto [p, off] : couple_at[i])
                    gemm1(gb, rows[i].slice(off, provR[p]), block(sys, i, p), X[p].m);
                // Column members: F(c, j)^T | A(i, j)^T | A(I, j)^T.
                for (int64_t j = k0; j < k1 && col_reuse; ++j) {
                  // reused far/ancestor members first, then the fill members
                  Members& C = cols[j];
                  const Members& sv = saved_rows_[size_t(j)];
                  const int w0 = sv.width - col_reuse_off[size_t(j)];
                  if (w0 > 0 && C.dim > 0)
                    cb.copy(C.slice(0, w0), sv.concat.m.sub(0, col_reuse_off[size_t(j)], C.dim, w0));
                  int off = w0;
                  for (const DMat* F : FI.by_col[j]) {
                    cb.copy(C.slice(off, F->rows()).t(), F->m);
                    off += F->rows();
                  }
                }
                for (int64_t j = k0; j < k1 && !col_reuse; ++j) {
                  Members& C = cols[j];
                  int off = 0;
                  for (const DMat* F : FI.by_col[j]) {
                    cb.copy(C.slice(off, F->rows()).t(), F->m);
                    off += F->rows();
                  }
                  for (int64_t t = 0; t < S.nfar(L, j); ++t) {
                    const int64_t i = S.far(L, j)[t];
                    const Samp sp = samp(rs(L, i));
                    eb.add(C.slice(off, sp.count).t(), rb(L, i), rb(L, j), sp.step, 1);
                    off += sp.count;
                  }
                  for (auto [l2, I] : ancestor_far_partners(L, j)) {
                    const Samp sp = samp(rs(l2, I));
                    eb.add(C.slice(off, sp.count).t(), rb(l2, I), rb(L, j), sp.step, 1);
                    off += sp.count;
                  }
                }
                cb.run(c);
                eb.run(c);
                gb.run(c);
              },
              [&](int64_t k, const Mat& qu, int ru, const Mat& qv, int rv) {
                square_sink(P.U[L], P.V[L], sqcopies)(k, qu, ru, qv, rv);
              },
              [&]() {
                sqcopies.run(c);
                sqcopies.jobs.clear();
              });
    saved_rows_.clear();
  }

  // A column-major copy (even leading dimension) of a strided view, queued on
  // cb: generated-B GEMM producers move such A operands by 16-byte pairs.
  DMat colmajor_copy(CopyBatch& cb, const Mat& src) {
    const int ld = (src.rows + 1) & ~1;
    DMat d = alloc_mat(c, std::max(ld, 2), std::max(src.cols, 1));
    d.m = Mat{d.m.p, src.rows, src.cols, 1, std::max(ld, 2)};
    if (src.rows > 0 && src.cols > 0) cb.copy(d.m, src);
    return d;
  }

  // Leaf pieces with the kernel block generated inside the GEMM (every
  // A(p, J) is re-evaluated for each box c having p as a near neighbour and
  // J as a target; H2G_LEAF_GEN=1).
  void leaf_pieces_generated(SysL& sys, const std::vector<std::pair<int64_t, TargetKey>>& pkeys,
                             const std::vector<DMat>& mats, const std::map<int64_t, DMat>& usT,
                             const std::map<std::pair<int64_t, int64_t>, DMat>& qcm, int64_t lo, int64_t hi) {
    const auto& Ub = P.U[L];
    GemmBatch gb;
    for (size_t t = 0; t < pkeys.size(); ++t) {
      const auto [cc, tk] = pkeys[t];
      if (cc < lo || cc >= hi) continue;
      const int64_t jb = rb(tk.first, tk.second), je = jb + rs(tk.first, tk.second);
      const int w = int(je - jb);
      gb.job(mats[t].m, false);
      gb.seg_gen(Ub[cc].rank > 0 ? usT.at(cc).m : Ub[cc].Qs().t(), rb(L, cc), jb, w, false, 1.0);
      if (Ub[cc].rank > 0 && sys.offdiag)
        for (int64_t x = 0; x < S.nnear(L, cc); ++x) {
          const int64_t p = S.near(L, cc)[x];
          if (p == cc) continue;
          bool all_zero;
          auto mask = mask_for(L, p, jb, je, all_zero);
          if (all_zero) continue;
          gb.seg_gen(qcm.at({cc, p}).m, rb(L, p), jb, w, false, -1.0, mask);
        }
    }
    gb.run(c);
  }

  // Leaf pieces from materialized kernel blocks (the default): per target J
  // the rows every piece toward J needs -- A(c, J) of each box c with target
  // J, and A(p, J) with p's near columns zeroed for each of their near
  // neighbours p -- are evaluated ONCE into one column-major block and shared
  // by all the pieces' GEMM segments (the generated path evaluates A(p, J)
  // once per (c, p, J), ~26 times at the bench size). Targets are processed
  // in chunks under a memory budget. Same values (one kernel_pair per entry,
  // masked entries +0), same segments in the same order: bit-identical pieces.
  struct Plan {
    TargetKey tk;
    int64_t jb = 0;
    int w = 0, rows = 0;
    std::map<std::pair<int64_t, int>, int> off;  // (box, masked) -> row offset
    std::vector<std::pair<int64_t, int>> order;  // row blocks in layout order
    std::vector<size_t> jobs;                     // indices into pkeys
    // neighbour p -> which block its term reads: 1 = the masked copy, 0 = the
    // unmasked block (p has no near column inside the target, so the two are
    // the same values and one evaluation serves both), -1 = all zero (skipped)
    std::map<int64_t, int> nb;
  };
  // pkeys of build_leaf_pieces: (box, target) in box order, targets_of order.
  std::vector<std::pair<int64_t, TargetKey>> leaf_piece_keys() const {
    std::vector<std::pair<int64_t, TargetKey>> pkeys;
    for (int64_t cc = 0; cc < (int64_t(1) << L); ++cc)
      for (auto& tk : targets_of(L, cc)) pkeys.push_back({cc, tk});
    return pkeys;
  }
  // positive: per box, rank > 0 (nullptr: assume so). Reads the integer structure only.
  std::vector<Plan> make_leaf_plans(const std::vector<std::pair<int64_t, TargetKey>>& pkeys, bool offdiag,
                                    int64_t lo, int64_t hi, const std::vector<char>* positive) const {
    std::map<TargetKey, size_t> at;
    std::vector<Plan> plans;
    auto add_rows = [&](Plan& pl, int64_t box, int masked) {
      if (pl.off.count({box, masked})) return;
      pl.off[{box, masked}] = pl.rows;
      pl.order.push_back({box, masked});
      pl.rows += int(rs(L, box));
    };
    for (size_t t = 0; t < pkeys.size(); ++t) {
      const auto [cc, tk] = pkeys[t];
      if (cc < lo || cc >= hi) continue;
      auto it = at.find(tk);
      if (it == at.end()) {
        it = at.emplace(tk, plans.size()).first;
        plans.emplace_back();
        plans.back().tk = tk;
        plans.back().jb = rb(tk.first, tk.second);
        plans.back().w = int(rs(tk.first, tk.second));
      }
      Plan& pl = plans[it->second];
      pl.jobs.push_back(t);
      add_rows(pl, cc, 0);
      if ((!positive || (*positive)[size_t(cc)]) && offdiag)
        for (int64_t x = 0; x < S.nnear(L, cc); ++x) {
          const int64_t p = S.near(L, cc)[x];
          if (p == cc) continue;
          auto known = pl.nb.find(p);
          if (known == pl.nb.end()) {
            bool all_zero;
            const auto mk = mask_for(L, p, pl.jb, pl.jb + pl.w, all_zero);
            known = pl.nb.emplace(p, all_zero ? -1 : (mk.empty() ? 0 : 1)).first;
          }
          if (known->second >= 0) add_rows(pl, p, known->second);
        }
    }
    return plans;
  }
  std::future<std::vector<Plan>> leaf_plan_future_;

  void leaf_pieces_materialized(SysL& sys, const std::vector<std::pair<int64_t, TargetKey>>& pkeys,
                                const std::vector<DMat>& mats, const std::map<int64_t, DMat>& usT,
                                const std::map<std::pair<int64_t, int64_t>, DMat>& qcm, int64_t lo,
                                int64_t hi) {
    const auto& Ub = P.U[L];
    // The plans depend on the integer structure only (given that every own box
    // has a nonzero rank): Driver::run starts computing them on a host thread
    // while the fills and the bases keep the device busy.
    bool ranks_ok = true;
    for (int64_t cc = lo; cc < hi; ++cc) ranks_ok = ranks_ok && Ub[cc].rank > 0;
    std::vector<Plan> plans;
    if (leaf_plan_future_.valid()) {
      plans = leaf_plan_future_.get();
      if (!ranks_ok) plans.clear();
    }
    if (plans.empty()) {
      std::vector<char> pos(size_t(sys.m));
      for (int64_t cc = 0; cc < sys.m; ++cc) pos[size_t(cc)] = Ub[cc].rank > 0;
      plans = make_leaf_plans(pkeys, sys.offdiag, lo, hi, &pos);
    }
    const size_t fr = c.free_bytes();
    const size_t budget = std::max<size_t>(size_t(1) << 28, fr / 3);
    // Equal charges: A(I, c)^T == A(c, I) bit for bit, so the first transfer
    // level's ancestor-partner column members (A(I, c) Vs_c)^T = Vs_c^T A(c, I)
    // are plain GEMMs on the kernel blocks materialised here for the pieces
    // (same operands, same k order as the kernel-generated GEMM of
    // build_transfers, which they replace: 71 ms at 11 TF/s at the bench size).
    // leaf_cols_[c]: r_c x (widths of ancestor_far_partners(L - 1, c >> 1)).
    leaf_cols_.clear();
    std::map<std::pair<int64_t, TargetKey>, Mat> leaf_col_dst;
    if (P.uniform_q && L >= 3 && getenv("H2G_NO_LEAF_COLS") == nullptr) {
      const auto& Vb = P.V[L];
      std::vector<std::pair<int, int>> shp;
      size_t need = 0;
      const int64_t mleaf = int64_t(1) << L;
      for (int64_t cc = 0; cc < mleaf; ++cc) {
        int w = 0;
        for (auto [l2, I] : ancestor_far_partners(L - 1, cc >> 1)) w += samp(rs(l2, I)).count;
        shp.push_back({Vb[cc].rank, w});
        need += sizeof(double) * size_t(Vb[cc].rank) * size_t(w);
      }
      if (need < fr / 4) {
        leaf_cols_ = alloc_mats(c, shp);
        for (int64_t cc = lo; cc < hi; ++cc) {
          int off = 0;
          for (auto [l2, I] : ancestor_far_partners(L - 1, cc >> 1)) {
            const int w = samp(rs(l2, I)).count;  // (sampled members: the same strided columns)
            leaf_col_dst[{cc, TargetKey{l2, I}}] = leaf_cols_[size_t(cc)].m.sub(0, off, Vb[cc].rank, w);
            off += w;
          }
        }
      }
    }
    size_t p0 = 0;
    while (p0 < plans.size()) {
      size_t p1 = p0, bytes = 0;
      while (p1 < plans.size()) {
        const size_t need = sizeof(double) * size_t(plans[p1].rows) * size_t(plans[p1].w);
        if (p1 > p0 && bytes + need > budget) break;
        bytes += need;
        ++p1;
      }
      std::vector<std::pair<int, int>> bshapes;
      for (size_t q = p0; q < p1; ++q) bshapes.push_back({plans[q].rows, plans[q].w});
      auto B = alloc_mats(c, bshapes);
      EvalBatch eb;
      CopyBatch zb;
      for (size_t q = p0; q < p1; ++q) {
        const Plan& pl = plans[q];
        const Mat Bm = B[q - p0].m;
        for (auto [box, masked] : pl.order) {
          const int r0 = pl.off.at({box, masked}), nr = int(rs(L, box));
          eb.add(Bm.sub(r0, 0, nr, pl.w), rb(L, box), pl.jb);
          if (masked) {
            bool all_zero;
            for (auto& r : mask_for(L, box, pl.jb, pl.jb + pl.w, all_zero))
              zb.zero(Bm.sub(r0, r.x, nr, r.y - r.x));
          }
        }
      }
      eb.run(c);
      zb.run(c);
      GemmBatch gb;
      for (size_t q = p0; q < p1; ++q) {
        const Plan& pl = plans[q];
        const Mat Bm = B[q - p0].m;
        auto rows_of = [&](int64_t box, int masked) {
          return Bm.sub(pl.off.at({box, masked}), 0, int(rs(L, box)), pl.w);
        };
        for (size_t t : pl.jobs) {
          const int64_t cc = pkeys[t].first;
          gb.job(mats[t].m, false);
          gb.seg(Ub[cc].rank > 0 ? usT.at(cc).m : Ub[cc].Qs().t(), rows_of(cc, 0), 1.0);
          if (Ub[cc].rank > 0 && sys.offdiag)
            for (int64_t x = 0; x < S.nnear(L, cc); ++x) {
              const int64_t p = S.near(L, cc)[x];
              if (p == cc) continue;
              const auto nbp = pl.nb.find(p);
              if (nbp == pl.nb.end() || nbp->second < 0) continue;
              gb.seg(qcm.at({cc, p}).m, rows_of(p, nbp->second), -1.0);
            }
          const auto lc = leaf_col_dst.find({cc, pl.tk});
          if (lc != leaf_col_dst.end() && lc->second.rows > 0)
            gemm1(gb, lc->second, P.V[L][cc].Qs().t(), sample_cols_view(rows_of(cc, 0), samp(pl.w)));
        }
      }
      gb.run(c);
      p0 = p1;  // B is freed (stream-ordered) when it goes out of scope
    }
    if (!leaf_cols_.empty()) {  // multi-GPU: every rank needs every leaf's members
      std::vector<int64_t> box;
      for (int64_t cc = 0; cc < (int64_t(1) << L); ++cc) box.push_back(cc);
      exchange_mats(leaf_cols_, box, int64_t(1) << L);
    }
  }
  // First transfer level's ancestor-partner column members per leaf (see above).
  std::vector<DMat> leaf_cols_;

  // ---- build_leaf_pieces (ulv.cpp:336-401) -----------------------------------
  void build_leaf_pieces(SysL& sys, const FillSet& fills, std::vector<PieceMap>& pieces,
                         double* level_max) {
    PhaseTimer pt(c, P.stats, "skeleton");
    const int64_t m = sys.m;
    const auto& Ub = P.U[L];
    const auto& Vb = P.V[L];
    pieces.assign(m, {});
    // q_cp = (A_pp^-T A_cp^T Us_c)^T for near p != c.
    std::map<std::pair<int64_t, int64_t>, DMat> qT;  // stored as B = dims_p x r_c (q = B^T)
    // Multi-GPU: the pieces of this rank's boxes only, then all-gathered.
    const auto [lo, hi] = own_range(m);
    if (sys.offdiag) {
      std::vector<std::pair<int64_t, int64_t>> keys;
      std::vector<std::pair<int, int>> shapes;
      for (int64_t cc = lo; cc < hi; ++cc) {
        if (Ub[cc].rank == 0) continue;
        for (int64_t t = 0; t < S.nnear(L, cc); ++t) {
          const int64_t p = S.near(L, cc)[t];
          if (p == cc) continue;
          keys.push_back({cc, p});
          shapes.push_back({sys.dims[p], Ub[cc].rank});
        }
      }
      auto mats = alloc_mats(c, shapes);
      GemmBatch gb;
      SolveBatch sb;
      for (size_t t = 0; t < keys.size(); ++t) {
        const auto [cc, p] = keys[t];
        gemm1(gb, mats[t].m, block(sys, cc, p).t(), Ub[cc].Qs());
        sb.add(sys.diag_lu[p], mats[t].m, SOLVE_TRANSPOSE);
        qT[keys[t]] = mats[t];
      }
      gb.run(c);
      sb.run(c);
    }
    // The generated-B GEMM's A operands, stored column-major with an even
    // leading dimension (Us_c^T and q_cp; the views above are transposes):
    // the producers then move A by 16-byte row pairs. Same values, same order.
    std::map<int64_t, DMat> usT;
    std::map<std::pair<int64_t, int64_t>, DMat> qcm;
    {
      CopyBatch cb;
      for (int64_t cc = lo; cc < hi; ++cc)
        if (Ub[cc].rank > 0) usT[cc] = colmajor_copy(cb, Ub[cc].Qs().t());
      for (auto& [key, m] : qT) qcm[key] = colmajor_copy(cb, m.m.t());
      cb.run(c);
    }
    // Pieces: Us_c^T A(c, J) - sum_p q_cp A(p, J)[masked].
    std::vector<std::pair<int64_t, TargetKey>> pkeys;
    std::vector<std::pair<int, int>> shapes;
    for (int64_t cc = 0; cc < m; ++cc)
      for (auto& tk : targets_of(L, cc)) {
        pkeys.push_back({cc, tk});
        shapes.push_back({Ub[cc].rank, int(rs(tk.first, tk.second))});
      }
    std::vector<DMat> mats;
    stacked_.clear();
    if (!(P.comm && P.comm->partitioned(m)) && m >= 2) {
      // carried pieces (coarser targets) in their parents' stacks, own-level ones apart
      std::vector<std::pair<int64_t, TargetKey>> ck;
      std::vector<int> cr;
      std::vector<std::pair<int, int>> own;
      for (size_t t = 0; t < pkeys.size(); ++t)
        if (pkeys[t].second.first < L) {
          ck.push_back(pkeys[t]);
          cr.push_back(shapes[t].first);
        } else {
          own.push_back(shapes[t]);
        }
      auto cm = alloc_stacked(m, ck, cr);
      auto om = alloc_mats(c, own);
      size_t a = 0, b = 0;
      for (size_t t = 0; t < pkeys.size(); ++t) mats.push_back(pkeys[t].second.first < L ? cm[a++] : om[b++]);
    } else {
      mats = alloc_mats(c, shapes);
    }
    for (size_t t = 0; t < pkeys.size(); ++t) pieces[pkeys[t].first][pkeys[t].second] = mats[t];
    {
      PhaseTimer pt2(c, P.stats, "skeleton_leaf_pieces");
      static const bool generated = getenv("H2G_LEAF_GEN") != nullptr;
      if (generated)
        leaf_pieces_generated(sys, pkeys, mats, usT, qcm, lo, hi);
      else
        leaf_pieces_materialized(sys, pkeys, mats, usT, qcm, lo, hi);
    }
    {
      std::vector<int64_t> box(pkeys.size());
      for (size_t t = 0; t < pkeys.size(); ++t) box[t] = pkeys[t].first;
      exchange_mats(mats, box, m);
    }
    // Fill content: project, measure absorption, add into the target piece.
    observe_and_add_fills(L, fills, pieces, level_max, true);
  }

  // uf = Us_c^T F, proj = uf Vs_j; observe_fill (ulv.cpp:140-147); for leaf,
  // add uf into far / covering pieces (ulv.cpp:380-400).
  void observe_and_add_fills(int lvl, const FillSet& fills, std::vector<PieceMap>& pieces,
                             double* level_max, bool add_to_pieces) {
    const auto& Ub = P.U[lvl];
    const auto& Vb = P.V[lvl];
    std::vector<std::pair<int64_t, int64_t>> keys;
    std::vector<std::pair<int, int>> shapes;
    for (auto& [key, F] : fills) {
      if (key.first == key.second) continue;
      keys.push_back(key);
      shapes.push_back({Ub[key.first].rank, F.cols()});
      shapes.push_back({Ub[key.first].rank, Vb[key.second].rank});
    }
    auto mats = alloc_mats(c, shapes);
    GemmBatch g1, g2;
    NormBatch nb;
    for (size_t t = 0; t < keys.size(); ++t) {
      const auto [cc, j] = keys[t];
      const DMat& F = fills.at(keys[t]);
      gemm1(g1, mats[2 * t].m, Ub[cc].Qs().t(), F.m);
      gemm1(g2, mats[2 * t + 1].m, mats[2 * t].m, Vb[j].Qs());
      nb.add(F.m);
      nb.add(mats[2 * t + 1].m);
    }
    g1.run(c);
    g2.run(c);
    auto norms = nb.run(c);
    for (size_t t = 0; t < keys.size(); ++t)
      observe_fill(lvl, keys[t].first, keys[t].second, norms[2 * t], norms[2 * t + 1], level_max);
    if (!add_to_pieces) return;
    CopyBatch cb;
    for (size_t t = 0; t < keys.size(); ++t) {
      const auto [cc, j] = keys[t];
      const Mat uf = mats[2 * t].m;
      if (S.is_far(lvl, cc, j)) {
        cb.add(pieces[cc].at({lvl, j}).m, uf, 1.0);
      } else if (!S.is_near(lvl, cc, j)) {
        TargetKey tk = covering_target(lvl, cc, j);
        const int off = int(rb(lvl, j) - rb(tk.first, tk.second));
        const Mat& pc = pieces[cc].at(tk).m;
        cb.add(pc.sub(0, off, pc.rows, uf.cols), uf, 1.0);
      }
    }
    cb.run(c);
  }

  void observe_fill(int lvl, int64_t cc, int64_t j, double nf, double kept, double* level_max) {
    const double resid = std::sqrt(std::max(0.0, nf * nf - kept * kept));
    if (nf > 0.0 && level_max) *level_max = std::max(*level_max, resid / nf);
    if (resid > opt.abort_residual_factor * opt.tol * nf && nf > 1e-300)
      throw std::runtime_error("basis does not absorb fill-in at level " + std::to_string(lvl) +
                               " block (" + std::to_string(cc) + "," + std::to_string(j) + ")");
  }

  // cols_to_merged (ulv.cpp:468-474) of a piece whose rows come in up to two
  // row blocks (vconcat of carried children), written into out (rows x dims_J).
  void cols_to_merged(GemmBatch& gb, Mat out, const std::vector<Mat>& row_blocks, int64_t J) {
    const Mat v0 = Vbig[2 * J], v1 = Vbig[2 * J + 1];
    int r = 0;
    for (const Mat& pb : row_blocks) {
      if (pb.rows > 0) {
        gemm1(gb, out.sub(r, 0, pb.rows, v0.cols), pb.sub(0, 0, pb.rows, v0.rows), v0);
        gemm1(gb, out.sub(r, v0.cols, pb.rows, v1.cols), pb.sub(0, v0.rows, pb.rows, v1.rows), v1);
      }
      r += pb.rows;
    }
  }

  // ---- build_upper_pieces (ulv.cpp:405-464) ----------------------------------
  void build_upper_pieces(SysL& sys, const FillSet& fills, std::vector<PieceMap>& stack,
                          std::vector<PieceMap>& merged) {
    PhaseTimer pt(c, P.stats, "skeleton");
    const int lvl = sys.lvl;
    const int64_t m = sys.m;
    stack.assign(m, {});
    {
      std::vector<std::pair<int64_t, TargetKey>> keys;
      std::vector<std::pair<int, int>> shapes;
      for (int64_t K = 0; K < m; ++K)
        for (auto& tk : targets_of(lvl, K)) {
          if (!carried[2 * K].count(tk) || !carried[2 * K + 1].count(tk))
            throw std::logic_error("build_upper_pieces: missing child piece");
          keys.push_back({K, tk});
          shapes.push_back({sys.dims[K], int(rs(tk.first, tk.second))});
        }
      if (int64_t(stacked_.size()) == m) {
        for (auto& [K, tk] : keys) stack[K][tk] = stacked_[size_t(K)].at(tk);  // already stacked: no copy
        stacked_.clear();
      } else {
        auto mats = alloc_mats(c, shapes);
        CopyBatch cb;
        for (size_t t = 0; t < keys.size(); ++t) {
          const auto [K, tk] = keys[t];
          const Mat a = carried[2 * K].at(tk).m, b = carried[2 * K + 1].at(tk).m;
          if (a.rows) cb.copy(mats[t].m.sub(0, 0, a.rows, a.cols), a);
          if (b.rows) cb.copy(mats[t].m.sub(a.rows, 0, b.rows, b.cols), b);
          stack[K][tk] = mats[t];
        }
        cb.run(c);
      }
    }
    merged.assign(m, {});
    if (sys.offdiag) {
      // g(P, tk) = A_PP^-1 (stack[P][tk] with P's near columns zeroed), shared across K.
      // Multi-GPU: corrected pieces of this rank's boxes only (all-gathered
      // below); the g's they need may belong to neighbours (recomputed).
      const auto [lo, hi] = own_range(m);
      // Tolerance-parity mode: reassociate A_KP (A_PP^-1 S_P) as (A_KP A_PP^-1) S_P,
      // with W_KP = A_KP A_PP^-1 formed once per near pair, so the wide
      // A_PP^-1 S_P products are never formed (g then holds the masked S_P).
      const bool reassoc = c.fast_solve;
      std::map<std::pair<int64_t, int64_t>, DMat> Wkp;
      if (reassoc) {
        // W_KP^T = A_PP^-T A_KP^T: one transpose solve per (K, P) near pair.
        std::vector<std::pair<int64_t, int64_t>> pk;
        std::vector<std::pair<int, int>> ws;
        for (int64_t K = lo; K < hi; ++K)
          for (int64_t x = 0; x < S.nnear(lvl, K); ++x) {
            const int64_t Pp = S.near(lvl, K)[x];
            if (Pp == K || sys.dims[K] == 0 || sys.dims[Pp] == 0) continue;
            pk.push_back({K, Pp});
            ws.push_back({sys.dims[Pp], sys.dims[K]});
          }
        auto wm = alloc_mats(c, ws);
        CopyBatch wc;
        SolveBatch wsb;
        for (size_t t = 0; t < pk.size(); ++t) {
          const auto [K, Pp] = pk[t];
          wc.copy(wm[t].m, block(sys, K, Pp).t());
          wsb.add(sys.diag_lu[Pp], wm[t].m, SOLVE_TRANSPOSE);
          Wkp[pk[t]] = wm[t];
        }
        wc.run(c);
        wsb.run(c);
      }
      // corrected = stack - sum_P A_KP g(P, tk), accumulated over P in order.
      std::vector<std::pair<int64_t, TargetKey>> keys;
      std::vector<std::pair<int, int>> cshapes;
      std::vector<size_t> first_of(size_t(m) + 1, 0);  // keys of box K: [first_of[K], first_of[K + 1])
      for (int64_t K = 0; K < m; ++K) {
        first_of[size_t(K)] = keys.size();
        for (auto& [tk, piece] : stack[K]) {
          keys.push_back({K, tk});
          cshapes.push_back({piece.rows(), piece.cols()});
        }
      }
      first_of[size_t(m)] = keys.size();
      auto cm = alloc_mats(c, cshapes);
      for (size_t t = 0; t < keys.size(); ++t) merged[keys[t].first][keys[t].second] = cm[t];
      // Boxes are processed in chunks so that the g's alive at once stay within
      // a third of the free memory (they are as large as a whole piece set).
      const size_t fr = c.free_bytes();
      const size_t budget = std::max<size_t>(size_t(1) << 28, fr / 3);
      auto needed_by = [&](int64_t K, std::vector<std::pair<int64_t, TargetKey>>& out) {
        for (int64_t x = 0; x < S.nnear(lvl, K); ++x) {
          const int64_t Pp = S.near(lvl, K)[x];
          if (Pp == K) continue;
          for (auto& [tk, piece] : stack[K]) {
            if (opt.reference_compat ? !stack[Pp].count(tk) : overlapping(stack[Pp], tk).empty())
              continue;
            out.push_back({Pp, tk});
          }
        }
      };
      int64_t K0 = lo;
      while (K0 < hi) {
        std::set<std::pair<int64_t, TargetKey>> needset;
        size_t bytes = 0;
        int64_t K1 = K0;
        while (K1 < hi) {
          std::vector<std::pair<int64_t, TargetKey>> nk;
          needed_by(K1, nk);
          size_t add = 0;
          for (auto& key : nk)
            if (!needset.count(key))
              add += sizeof(double) * size_t(sys.dims[key.first]) * size_t(rs(key.second.first, key.second.second));
          if (K1 > K0 && bytes + add > budget) break;
          for (auto& key : nk) needset.insert(key);
          bytes += add;
          ++K1;
        }
        std::map<std::pair<int64_t, TargetKey>, DMat> g;
        std::vector<std::pair<int, int>> shapes;
        std::vector<std::pair<int64_t, TargetKey>> gkeys;
        std::vector<std::vector<int2>> gmasks;
        for (auto& [Pp, tk] : needset) {
          const int64_t jb = rb(tk.first, tk.second), je = jb + rs(tk.first, tk.second);
          bool all_zero;
          auto mask = mask_for(lvl, Pp, jb, je, all_zero);
          if (all_zero) continue;
          gkeys.push_back({Pp, tk});
          gmasks.push_back(mask);
          shapes.push_back({sys.dims[Pp], int(je - jb)});
        }
        auto mats = alloc_mats(c, shapes);
        CopyBatch cb, zb;
        SolveBatch sb;
        for (size_t t = 0; t < gkeys.size(); ++t) {
          const auto [Pp, tk] = gkeys[t];
          if (opt.reference_compat) {
            cb.copy(mats[t].m, stack[Pp].at(tk).m);
          } else {
            // P's content over J's columns from every target of P overlapping J
            // (oracle/fix_reference.py fix 3); the rest are P's near columns.
            // (only the columns no target covers are zero-filled, not the whole block)
            auto ov = overlapping(stack[Pp], tk);
            std::sort(ov.begin(), ov.end(), [](const Overlap& a, const Overlap& b) { return a.dst < b.dst; });
            int at = 0;
            for (auto& o : ov) {
              if (o.dst > at) zb.zero(mats[t].m.sub(0, at, mats[t].rows(), o.dst - at));
              cb.copy(mats[t].m.sub(0, o.dst, mats[t].rows(), o.len),
                      stack[Pp].at(o.tk).m.sub(0, o.src, mats[t].rows(), o.len));
              at = std::max(at, o.dst + o.len);
            }
            if (at < mats[t].cols()) zb.zero(mats[t].m.sub(0, at, mats[t].rows(), mats[t].cols() - at));
          }
          if (opt.reference_compat)
            for (auto& r : gmasks[t]) zb.zero(mats[t].m.sub(0, r.x, mats[t].rows(), r.y - r.x));
          if (!reassoc) sb.add(sys.diag_lu[Pp], mats[t].m, SOLVE_FULL);
          g[gkeys[t]] = mats[t];
        }
        if (opt.reference_compat) {
          cb.run(c);
          zb.run(c);
        } else {
          zb.run(c);  // zero-fill first, then the overlapping slices, then the masks
          cb.run(c);
          CopyBatch mz;
          for (size_t t = 0; t < gkeys.size(); ++t)
            for (auto& r : gmasks[t]) mz.zero(mats[t].m.sub(0, r.x, mats[t].rows(), r.y - r.x));
          mz.run(c);
        }
        sb.run(c);
        CopyBatch cc;
        GemmBatch gb;
        for (size_t t = first_of[size_t(K0)]; t < first_of[size_t(K1)]; ++t) {
          const auto [K, tk] = keys[t];
          bool any = false;
          for (int64_t x = 0; x < S.nnear(lvl, K); ++x) {
            const int64_t Pp = S.near(lvl, K)[x];
            if (Pp == K) continue;
            auto it = g.find({Pp, tk});
            if (it == g.end()) continue;
            // the accumulator starts from the stacked piece (no copy into cm first)
            if (!any) gb.job_from(cm[t].m, stack[K].at(tk).m);
            any = true;
            gb.seg(reassoc ? Wkp.at({K, Pp}).m.t() : block(sys, K, Pp), it->second.m, -1.0);
          }
          if (!any) cc.copy(cm[t].m, stack[K].at(tk).m);
        }
        cc.run(c);
        gb.run(c);
        K0 = K1;  // this chunk's g's are released stream-ordered behind its GEMMs
      }
      std::vector<int64_t> box(keys.size());
      for (size_t t = 0; t < keys.size(); ++t) box[t] = keys[t].first;
      exchange_mats(cm, box, m);
    } else {
      merged = stack;
    }
    // Covered fills: expand merged columns to raw columns, add into the covering slice.
    std::vector<std::pair<int64_t, int64_t>> fk;
    std::vector<std::pair<int, int>> shapes;
    for (auto& [key, F] : fills) {
      const auto [cc, j] = key;
      if (cc == j || S.is_near(lvl, cc, j)) continue;
      // The reference adds only covered fills here; far ones are lost
      // (oracle/fix_reference.py fix 2).
      if (opt.reference_compat && S.is_far(lvl, cc, j)) continue;
      fk.push_back(key);
      shapes.push_back({F.rows(), int(rs(lvl, j))});
    }
    if (fk.empty()) return;
    auto raws = alloc_mats(c, shapes);
    GemmBatch gb;
    CopyBatch cb;
    for (size_t t = 0; t < fk.size(); ++t) {
      const auto [cc, j] = fk[t];
      const Mat F = fills.at(fk[t]).m;
      const Mat v0 = Vbig[2 * j], v1 = Vbig[2 * j + 1];
      gemm1(gb, raws[t].m.sub(0, 0, F.rows, v0.rows), F.sub(0, 0, F.rows, v0.cols), v0.t());
      gemm1(gb, raws[t].m.sub(0, v0.rows, F.rows, v1.rows), F.sub(0, v0.cols, F.rows, v1.cols), v1.t());
      TargetKey tk = S.is_far(lvl, cc, j) ? TargetKey{lvl, j} : covering_target(lvl, cc, j);
      const int off = int(rb(lvl, j) - rb(tk.first, tk.second));
      const Mat pc = merged[cc].at(tk).m;
      cb.add(pc.sub(0, off, pc.rows, raws[t].cols()), raws[t].m, 1.0);
    }
    gb.run(c);
    cb.run(c);
  }

  // ---- build_transfers_nodep (ulv.cpp:476-521) --------------------------------
  void build_transfers(SysL& sys, const FillSet& fills, const std::vector<PieceMap>& merged) {
    PhaseTimer pt(c, P.stats, "basis");
    const int lvl = sys.lvl;
    const int64_t m = sys.m;
    std::vector<Members> rows(m), cols(m);
    const FillIndex FI = index_fills(fills, m);
    for (int64_t k = 0; k < m; ++k) {
      rows[k].dim = cols[k].dim = sys.dims[k];
      for (const DMat* F : FI.by_row[k]) rows[k].add(F->cols());
      for (auto& [tk, piece] : merged[k]) rows[k].add(samp(piece.cols()).count);
      for (const DMat* F : FI.by_col[k]) cols[k].add(F->rows());
      for (int64_t t = 0; t < S.nfar(lvl, k); ++t) cols[k].add(sys.dims[S.far(lvl, k)[t]]);
      for (auto [l2, I] : ancestor_far_partners(lvl, k)) cols[k].add(samp(rs(l2, I)).count);
    }
    for (int64_t k = 0; k < m; ++k)
      if (sys.dims[k] == 0 && rows[k].width > 0)
        throw std::runtime_error("compute_transfer: rank-0 children with nonzero parent blocks");
    // Tolerance modes: the ancestor-partner column members are nested. With
    // Vbig_c = blockdiag(Vbig of c's children) Vs_c, the member of child c
    // toward I is Vs_c^T times c's own member toward I of the previous (finer)
    // level, so from the second transfer level on no kernel entry is evaluated
    // again (the reference evaluates A(I, c) Vbig_c from scratch at every
    // level, ulv.cpp:495-501). The members of this level are kept for the next.
    const bool nest = c.fast_solve && lvl + 1 < L && int64_t(prev_cols_.size()) == 2 * m;
    std::vector<DMat> keepm;
    std::vector<int> anc_off(m, 0), anc_w(m, 0);
    for (int64_t k = 0; k < m; ++k) {
      anc_off[k] = cols[k].width;
      for (auto [l2, I] : ancestor_far_partners(lvl, k)) {
        const int w = samp(rs(l2, I)).count;
        anc_off[k] -= w;
        anc_w[k] += w;
      }
    }
    if (c.fast_solve && lvl >= 3) {
      size_t need = 0;
      for (int64_t k = 0; k < m; ++k) need += sizeof(double) * size_t(sys.dims[k]) * size_t(anc_w[k]);
      const size_t fr = c.free_bytes();
      if (need < fr / 4) {
        std::vector<std::pair<int, int>> ks;
        for (int64_t k = 0; k < m; ++k) ks.push_back({sys.dims[k], anc_w[k]});
        keepm = alloc_mats(c, ks);
      }
    }
    CopyBatch sqcopies;
    run_bases(rows, &cols,
              [&](int64_t k0, int64_t k1) {
                CopyBatch cb;
                GemmBatch gb;
                CopyBatch kb;            // this level's ancestor members -> keepm
                std::vector<DMat> keep;  // A operands alive until the GEMMs are queued
                for (int64_t k = k0; k < k1; ++k) {
                  int off = 0;
                  for (const DMat* F : FI.by_row[k]) {
                    cb.copy(rows[k].slice(off, F->cols()), F->m);
                    off += F->cols();
                  }
                  size_t mem = FI.by_row[k].size();
                  for (auto& [tk, piece] : merged[k]) {
                    const Samp sp = samp(piece.cols());
                    // compressed mode: the Gram GEMM reads the piece in place (no copy into the panel)
                    if (c.qr_compress)
                      rows[k].set_view(mem, sample_cols_view(piece.m, sp));
                    else
                      cb.copy(rows[k].slice(off, sp.count), sample_cols_view(piece.m, sp));
                    off += sp.count;
                    ++mem;
                  }
                  off = 0;
                  for (const DMat* F : FI.by_col[k]) {
                    cb.copy(cols[k].slice(off, F->rows()).t(), F->m);
                    off += F->rows();
                  }
                  for (int64_t t = 0; t < S.nfar(lvl, k); ++t) {
                    const int64_t i = S.far(lvl, k)[t];
                    const Mat piece = merged[i].at({lvl, k}).m;
                    cols_to_merged(gb, cols[k].slice(off, piece.rows).t(), {piece}, k);
                    off += piece.rows;
                  }
                  const auto anc = ancestor_far_partners(lvl, k);
                  if (anc.empty()) continue;
                  const Mat v0 = Vbig[2 * k], v1 = Vbig[2 * k + 1];
                  if (!keepm.empty() && anc_w[k] > 0 && sys.dims[k] > 0)
                    kb.copy(keepm[k].m, cols[k].slice(anc_off[k], anc_w[k]));
                  if (lvl + 1 == L && int64_t(leaf_cols_.size()) == 2 * m) {
                    // children are leaves: their members were formed beside the leaf pieces
                    const Mat dst = cols[k].slice(off, anc_w[k]);
                    if (v0.cols > 0 && anc_w[k] > 0) cb.copy(dst.sub(0, 0, v0.cols, anc_w[k]), leaf_cols_[2 * k].m);
                    if (v1.cols > 0 && anc_w[k] > 0)
                      cb.copy(dst.sub(v0.cols, 0, v1.cols, anc_w[k]), leaf_cols_[2 * k + 1].m);
                    continue;
                  }
                  if (nest && prev_cols_[2 * k].m.p && prev_cols_[2 * k + 1].m.p) {
                    // prev_cols_[c]: c's ancestor members of the finer level, in
                    // ancestor_far_partners(lvl + 1, c) order = far(lvl, k), then anc.
                    int skip = 0;
                    for (int64_t t = 0; t < S.nfar(lvl, k); ++t) skip += samp(rs(lvl, S.far(lvl, k)[t])).count;
                    const Mat q0 = P.V[lvl + 1][2 * k].Qs().t(), q1 = P.V[lvl + 1][2 * k + 1].Qs().t();
                    const Mat p0 = prev_cols_[2 * k].m, p1 = prev_cols_[2 * k + 1].m;
                    const Mat dst = cols[k].slice(off, anc_w[k]);
                    if (v0.cols > 0) gemm1(gb, dst.sub(0, 0, v0.cols, anc_w[k]), q0, p0.sub(0, skip, p0.rows, anc_w[k]));
                    if (v1.cols > 0)
                      gemm1(gb, dst.sub(v0.cols, 0, v1.cols, anc_w[k]), q1, p1.sub(0, skip, p1.rows, anc_w[k]));
                    continue;
                  }
                  // Vbig_c^T column-major (even ld) for the generated GEMMs' A.
                  keep.push_back(colmajor_copy(cb, v0.t()));
                  const Mat v0T = keep.back().m;
                  keep.push_back(colmajor_copy(cb, v1.t()));
                  const Mat v1T = keep.back().m;
                  for (auto [l2, I] : anc) {
                    // (A(I, c0) Vbig_c0 | A(I, c1) Vbig_c1)^T, B generated in-kernel.
                    const Samp sp = samp(rs(l2, I));
                    const int w = sp.count;
                    const Mat dst = cols[k].slice(off, w);
                    gb.job(dst.sub(0, 0, v0.cols, w), false);
                    gb.seg_gen(v0T, rb(l2, I), rb(lvl + 1, 2 * k), w, true, 1.0, {}, sp.step);
                    gb.job(dst.sub(v0.cols, 0, v1.cols, w), false);
                    gb.seg_gen(v1T, rb(l2, I), rb(lvl + 1, 2 * k + 1), w, true, 1.0, {}, sp.step);
                    off += w;
                  }
                }
                cb.run(c);
                gb.run(c);
                kb.run(c);
              },
              [&](int64_t k, const Mat& qu, int ru, const Mat& qv, int rv) {
                square_sink(P.U[lvl], P.V[lvl], sqcopies)(k, qu, ru, qv, rv);
              },
              [&]() {
                sqcopies.run(c);
                sqcopies.jobs.clear();
              });
    if (!keepm.empty()) {  // multi-GPU: every rank needs every box's members at replicated levels
      std::vector<int64_t> box;
      for (int64_t k = 0; k < m; ++k) box.push_back(k);
      exchange_mats(keepm, box, m);
    }
    prev_cols_ = std::move(keepm);
    if (lvl + 1 == L) leaf_cols_.clear();
  }
  // Transfer stage, tolerance modes: per box of the previous (finer) transfer
  // level, its ancestor-partner column members (dims x sum of sampled widths).
  std::vector<DMat> prev_cols_;

  // ---- assemble_level (ulv.cpp:526-607) ----------------------------------------
  void assemble_level(SysL& sys, const FillSet& fills, const std::vector<PieceMap>& pieces,
                      const std::vector<PieceMap>& merged, std::vector<DMat>& diag_S,
                      std::map<std::pair<int64_t, int64_t>, DMat>& far_ss,
                      std::map<std::pair<int64_t, int64_t>, DMat>& dense_ss, double* level_max) {
    PhaseTimer pt(c, P.stats, "factorize");
    const int lvl = sys.lvl;
    const bool is_leaf = lvl == L;
    const int64_t m = sys.m;
    const auto& Ub = P.U[lvl];
    const auto& Vb = P.V[lvl];
    // Diagonal skeletons: [Ur Us]^T (A_kk + F_kk) [Vr Vs].
    {
      std::vector<std::pair<int, int>> shapes;
      for (int64_t k = 0; k < m; ++k) {
        shapes.push_back({sys.dims[k], sys.dims[k]});
        shapes.push_back({sys.dims[k], sys.dims[k]});
        shapes.push_back({sys.dims[k], sys.dims[k]});
      }
      auto mats = alloc_mats(c, shapes);
      CopyBatch cb, ab;
      GemmBatch g1, g2;
      diag_S.assign(m, {});
      for (int64_t k = 0; k < m; ++k) {
        const Mat D = mats[3 * k].m, T1 = mats[3 * k + 1].m;
        cb.copy(D, block(sys, k, k));
        auto it = fills.find({k, k});
        if (it != fills.end()) ab.add(D, it->second.m, 1.0);
        gemm1(g1, T1, Ub[k].SQ.m.t(), D);
        gemm1(g2, mats[3 * k + 2].m, T1, Vb[k].SQ.m);
        diag_S[k] = mats[3 * k + 2];
      }
      cb.run(c);
      ab.run(c);
      g1.run(c);
      g2.run(c);
    }
    // Far skeletons from the pieces.
    {
      std::vector<std::pair<int64_t, int64_t>> keys;
      std::vector<std::pair<int, int>> shapes;
      for (int64_t k = 0; k < m; ++k)
        for (int64_t t = 0; t < S.nfar(lvl, k); ++t) {
          const int64_t j = S.far(lvl, k)[t];
          keys.push_back({k, j});
          shapes.push_back({Ub[k].rank, Vb[j].rank});
          if (!is_leaf) {
            shapes.push_back({sys.dims[k], sys.dims[j]});
            shapes.push_back({Ub[k].rank, sys.dims[j]});
          }
        }
      auto mats = alloc_mats(c, shapes);
      GemmBatch g1, g2, g3;
      const int per = is_leaf ? 1 : 3;
      for (size_t t = 0; t < keys.size(); ++t) {
        const auto [k, j] = keys[t];
        const Mat Sm = mats[per * t].m;
        if (is_leaf) {
          gemm1(g1, Sm, pieces[k].at({lvl, j}).m, Vb[j].Qs());
        } else {
          const Mat y = mats[per * t + 1].m, ty = mats[per * t + 2].m;
          cols_to_merged(g1, y, {merged[k].at({lvl, j}).m}, j);
          gemm1(g2, ty, Ub[k].Qs().t(), y);
          gemm1(g3, Sm, ty, Vb[j].Qs());
        }
        far_ss[keys[t]] = mats[per * t];
      }
      g1.run(c);
      g2.run(c);
      g3.run(c);
    }
    if (!sys.offdiag) return;
    // Off-diagonal near content: projected fills + T terms over far (p, j).
    std::vector<std::pair<int64_t, int64_t>> pairs;
    for (int64_t k = 0; k < m; ++k)
      for (int64_t t = 0; t < S.nnear(lvl, k); ++t) {
        const int64_t j = S.near(lvl, k)[t];
        if (j != k) pairs.push_back({k, j});
      }
    // Fill projections (uf, proj) and their observation.
    std::map<std::pair<int64_t, int64_t>, DMat> proj;
    {
      std::vector<std::pair<int64_t, int64_t>> keys;
      std::vector<std::pair<int, int>> shapes;
      for (auto& kj : pairs) {
        auto it = fills.find(kj);
        if (it == fills.end()) continue;
        keys.push_back(kj);
        shapes.push_back({Ub[kj.first].rank, it->second.cols()});
        shapes.push_back({Ub[kj.first].rank, Vb[kj.second].rank});
      }
      auto mats = alloc_mats(c, shapes);
      GemmBatch g1, g2;
      NormBatch nb;
      for (size_t t = 0; t < keys.size(); ++t) {
        const auto [k, j] = keys[t];
        const Mat F = fills.at(keys[t]).m;
        gemm1(g1, mats[2 * t].m, Ub[k].Qs().t(), F);
        gemm1(g2, mats[2 * t + 1].m, mats[2 * t].m, Vb[j].Qs());
        nb.add(F);
        nb.add(mats[2 * t + 1].m);
        proj[keys[t]] = mats[2 * t + 1];
      }
      g1.run(c);
      g2.run(c);
      auto norms = nb.run(c);
      for (size_t t = 0; t < keys.size(); ++t)
        observe_fill(lvl, keys[t].first, keys[t].second, norms[2 * t], norms[2 * t + 1], level_max);
    }
    // g(p, j) = A_pp^-1 content(p, j), shared across k.
    std::vector<std::tuple<int64_t, int64_t, int64_t>> triples;  // (k, j, p)
    std::set<std::pair<int64_t, int64_t>> gneed;
    for (auto [k, j] : pairs)
      for (int64_t x = 0; x < S.nnear(lvl, k); ++x) {
        const int64_t p = S.near(lvl, k)[x];
        if (p == k || p == j) continue;
        // The reference takes only far (p, j); corrected mode every p not
        // near j (oracle/fix_reference.py fix 1).
        if (opt.reference_compat ? !S.is_far(lvl, p, j) : S.is_near(lvl, p, j)) continue;
        triples.push_back({k, j, p});
        gneed.insert({p, j});
      }
    std::map<std::pair<int64_t, int64_t>, DMat> g;
    {
      std::vector<std::pair<int64_t, int64_t>> keys(gneed.begin(), gneed.end());
      std::vector<std::pair<int, int>> shapes;
      for (auto [p, j] : keys) shapes.push_back({sys.dims[p], sys.dims[j]});
      auto mats = alloc_mats(c, shapes);
      EvalBatch eb;
      GemmBatch gb;
      SolveBatch sb;
      for (size_t t = 0; t < keys.size(); ++t) {
        const auto [p, j] = keys[t];
        if (is_leaf) {
          eb.add(mats[t].m, rb(lvl, p), rb(lvl, j));
        } else {
          // far: the (lvl, j) pieces; covered: j's slice of the covering target's
          const TargetKey tk = S.is_far(lvl, p, j) ? TargetKey{lvl, j} : covering_target(lvl, p, j);
          const int off = int(rb(lvl, j) - rb(tk.first, tk.second)), w = int(rs(lvl, j));
          const Mat a0 = carried[2 * p].at(tk).m, a1 = carried[2 * p + 1].at(tk).m;
          cols_to_merged(gb, mats[t].m, {a0.sub(0, off, a0.rows, w), a1.sub(0, off, a1.rows, w)}, j);
        }
        sb.add(sys.diag_lu[p], mats[t].m, SOLVE_FULL);
        g[keys[t]] = mats[t];
      }
      eb.run(c);
      gb.run(c);
      sb.run(c);
    }
    // T terms: t = Us_k^T (A_kp g), term = t Vs_j, D -= term (in p order).
    std::vector<std::pair<int, int>> shapes;
    for (auto [k, j, p] : triples) {
      shapes.push_back({sys.dims[k], sys.dims[j]});
      shapes.push_back({Ub[k].rank, sys.dims[j]});
      shapes.push_back({Ub[k].rank, Vb[j].rank});
    }
    auto tm = alloc_mats(c, shapes);
    GemmBatch g1, g2, g3;
    for (size_t t = 0; t < triples.size(); ++t) {
      const auto [k, j, p] = triples[t];
      gemm1(g1, tm[3 * t].m, block(sys, k, p), g.at({p, j}).m);
      gemm1(g2, tm[3 * t + 1].m, Ub[k].Qs().t(), tm[3 * t].m);
      gemm1(g3, tm[3 * t + 2].m, tm[3 * t + 1].m, Vb[j].Qs());
    }
    g1.run(c);
    g2.run(c);
    g3.run(c);
    std::vector<std::pair<int, int>> dshapes;
    std::vector<std::pair<int64_t, int64_t>> dkeys;
    std::map<std::pair<int64_t, int64_t>, std::vector<size_t>> terms_of;
    for (size_t t = 0; t < triples.size(); ++t)
      terms_of[{std::get<0>(triples[t]), std::get<1>(triples[t])}].push_back(t);
    for (auto kj : pairs) {
      if (!proj.count(kj) && !terms_of.count(kj)) continue;
      dkeys.push_back(kj);
      dshapes.push_back({Ub[kj.first].rank, Vb[kj.second].rank});
    }
    auto dm = alloc_mats(c, dshapes);
    AccBatch acc;
    for (size_t t = 0; t < dkeys.size(); ++t) {
      acc.job(dm[t].m, true);
      auto pi = proj.find(dkeys[t]);
      if (pi != proj.end()) acc.src(pi->second.m, 1.0);
      auto ti = terms_of.find(dkeys[t]);
      if (ti != terms_of.end())
        for (size_t x : ti->second) acc.src(tm[3 * x + 2].m, -1.0);
      dense_ss[dkeys[t]] = dm[t];
    }
    acc.run(c);
  }

  // ---- eliminate_level (ulv.cpp:25-48, :609-630) --------------------------------
  void eliminate_level(SysL& sys, std::vector<DMat>& diag_S, LevelF& lf) {
    PhaseTimer pt(c, P.stats, "factorize");
    const int64_t m = sys.m;
    lf.elim.assign(m, {});
    std::vector<int> rr;
    std::vector<std::pair<int, int>> shapes;
    for (int64_t k = 0; k < m; ++k) {
      const int rank = P.U[sys.lvl][k].rank;
      const int rdim = sys.dims[k] - rank, sdim = rank;
      lf.elim[k].rdim = rdim;
      lf.elim[k].sdim = sdim;
      rr.push_back(rdim);
      shapes.push_back({rdim, sdim});
      shapes.push_back({sdim, rdim});
    }
    auto lus = alloc_lus(c, rr);
    auto mats = alloc_mats(c, shapes);
    CopyBatch cb;
    LuBatch lb;
    for (int64_t k = 0; k < m; ++k) {
      ElimF& e = lf.elim[k];
      e.piv = lus[k];
      e.urs = mats[2 * k];
      e.lsr = mats[2 * k + 1];
      if (e.rdim == 0) continue;
      const Mat Sk = diag_S[k].m;
      cb.copy(e.piv.lu.m, Sk.sub(0, 0, e.rdim, e.rdim));
      if (e.sdim) {
        cb.copy(e.urs.m, Sk.sub(0, e.rdim, e.rdim, e.sdim));
        cb.copy(e.lsr.m, Sk.sub(e.rdim, 0, e.sdim, e.rdim));
      }
      lb.add(e.piv, opt.rr_pivot_tol, "S^RR");
    }
    cb.run(c);
    lb.run(c);
    SolveBatch s1;
    GemmBatch gb;
    for (int64_t k = 0; k < m; ++k) {
      ElimF& e = lf.elim[k];
      if (e.rdim == 0 || e.sdim == 0) continue;
      s1.add(e.piv, e.urs.m, SOLVE_LOWER);
      s1.add(e.piv, e.lsr.m, SOLVE_UPPER_RIGHT);
      gb.job(diag_S[k].m.sub(e.rdim, e.rdim, e.sdim, e.sdim), true);
      gb.seg(e.lsr.m, e.urs.m, -1.0);
    }
    s1.run(c);
    gb.run(c);
  }

  // ---- merge (ulv.cpp:632-671) ---------------------------------------------------
  SysL merge(const SysL& sys, const std::vector<DMat>& diag_S,
             const std::map<std::pair<int64_t, int64_t>, DMat>& far_ss,
             const std::map<std::pair<int64_t, int64_t>, DMat>& dense_ss) {
    PhaseTimer pt(c, P.stats, "factorize");
    const int lvl = sys.lvl;
    const int64_t mp = int64_t(1) << (lvl - 1);
    SysL next;
    next.lvl = lvl - 1;
    next.m = int(mp);
    next.dims.resize(mp);
    const auto& Ub = P.U[lvl];
    for (int64_t I = 0; I < mp; ++I) next.dims[I] = Ub[2 * I].rank + Ub[2 * I + 1].rank;
    std::vector<std::pair<int, int>> shapes;
    const auto& LP = S.level[lvl - 1];
    for (int64_t I = 0; I < mp; ++I)
      for (int64_t t = LP.near_ptr[I]; t < LP.near_ptr[I + 1]; ++t)
        shapes.push_back({next.dims[I], next.dims[LP.near_idx[t]]});
    next.blocks = alloc_mats(c, shapes);
    CopyBatch cb;
    for (int64_t I = 0; I < mp; ++I)
      for (int64_t t = LP.near_ptr[I]; t < LP.near_ptr[I + 1]; ++t) {
        const int64_t J = LP.near_idx[t];
        const Mat B = next.blocks[t].m;
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b) {
            const int64_t ci = 2 * I + a, cj = 2 * J + b;
            const int r0 = a == 0 ? 0 : Ub[2 * I].rank;
            const int c0 = b == 0 ? 0 : Ub[2 * J].rank;
            const int nr = Ub[ci].rank, nc = Ub[cj].rank;
            if (nr == 0 || nc == 0) continue;
            const Mat dst = B.sub(r0, c0, nr, nc);
            if (ci == cj) {
              const int rd = diag_S[ci].rows() - nr;
              cb.copy(dst, diag_S[ci].m.sub(rd, rd, nr, nr));
            } else if (far_ss.count({ci, cj})) {
              cb.copy(dst, far_ss.at({ci, cj}).m);
            } else if (dense_ss.count({ci, cj})) {
              cb.copy(dst, dense_ss.at({ci, cj}).m);
            } else {
              cb.zero(dst);
            }
          }
      }
    cb.run(c);
    next.offdiag = false;
    for (int64_t I = 0; I < mp && !next.offdiag; ++I)
      for (int64_t t = LP.near_ptr[I]; t < LP.near_ptr[I + 1]; ++t)
        if (LP.near_idx[t] != I) next.offdiag = true;
    return next;
  }

  // ---- assemble_top_nodep (ulv.cpp:691-708) --------------------------------------
  void assemble_top(SysL& sys) {
    PhaseTimer pt(c, P.stats, "factorize");
    const int lvl = sys.lvl;
    const int64_t m = sys.m;
    P.cutoff_level = lvl;
    P.cutoff_dims = sys.dims;
    std::vector<int64_t> off(m + 1, 0);
    for (int64_t k = 0; k < m; ++k) off[k + 1] = off[k] + sys.dims[k];
    P.top = alloc_lu(c, int(off[m]));
    const Mat A = P.top.lu.m;
    CopyBatch zb, cb;
    GemmBatch gb;
    zb.zero(A);
    for (int64_t i = 0; i < m; ++i) {
      for (int64_t t = 0; t < S.nnear(lvl, i); ++t) {
        const int64_t j = S.near(lvl, i)[t];
        if (sys.dims[i] && sys.dims[j])
          cb.copy(A.sub(int(off[i]), int(off[j]), sys.dims[i], sys.dims[j]), block(sys, i, j));
      }
      for (int64_t t = 0; t < S.nfar(lvl, i); ++t) {
        const int64_t j = S.far(lvl, i)[t];
        cols_to_merged(gb, A.sub(int(off[i]), int(off[j]), sys.dims[i], sys.dims[j]),
                       {carried[2 * i].at({lvl, j}).m, carried[2 * i + 1].at({lvl, j}).m}, j);
      }
    }
    zb.run(c);
    cb.run(c);
    gb.run(c);
    LuBatch lb;
    lb.add(P.top, 1e-15, "top system");
    lb.run(c);
  }

  // ---- finish_blr2 (ulv.cpp:762-781) ---------------------------------------------
  // The flat variant's remaining skeleton grid is the top system itself:
  // diagonal SS corners, far and dense skeleton couplings, one LU.
  void finish_blr2(const SysL& sys, const std::vector<DMat>& diag_S,
                   const std::map<std::pair<int64_t, int64_t>, DMat>& far_ss,
                   const std::map<std::pair<int64_t, int64_t>, DMat>& dense_ss) {
    PhaseTimer pt(c, P.stats, "factorize");
    const int64_t m = sys.m;
    const auto& Ub = P.U[sys.lvl];
    P.cutoff_level = sys.lvl;
    P.cutoff_dims.assign(m, 0);
    std::vector<int64_t> off(m + 1, 0);
    for (int64_t k = 0; k < m; ++k) {
      P.cutoff_dims[k] = Ub[k].rank;
      off[k + 1] = off[k] + Ub[k].rank;
    }
    P.top = alloc_lu(c, int(off[m]));
    const Mat A = P.top.lu.m;
    CopyBatch zb, cb;
    zb.zero(A);
    for (int64_t k = 0; k < m; ++k) {
      const int r = Ub[k].rank;
      if (r == 0) continue;
      const int rd = diag_S[k].rows() - r;
      cb.copy(A.sub(int(off[k]), int(off[k]), r, r), diag_S[k].m.sub(rd, rd, r, r));
    }
    for (const auto* ss : {&far_ss, &dense_ss})
      for (auto& [key, SS] : *ss)
        if (SS.rows() && SS.cols())
          cb.copy(A.sub(int(off[key.first]), int(off[key.second]), SS.rows(), SS.cols()), SS.m);
    zb.run(c);
    cb.run(c);
    LuBatch lb;
    lb.add(P.top, 1e-15, "top system");
    lb.run(c);
  }

  // ---- lift_layer (compression.cpp:302-322) --------------------------------------
  void make_layer(int lvl) {
    const int64_t m = int64_t(1) << lvl;
    std::vector<Mat> nu(m), nv(m);
    if (lvl == L) {
      for (int64_t i = 0; i < m; ++i) {
        nu[i] = P.U[L][i].Qs();
        nv[i] = P.V[L][i].Qs();
      }
      big_owner.clear();
    } else {
      std::vector<std::pair<int, int>> shapes;
      for (int64_t k = 0; k < m; ++k) {
        shapes.push_back({int(rs(lvl, k)), P.U[lvl][k].rank});
        shapes.push_back({int(rs(lvl, k)), P.V[lvl][k].rank});
      }
      auto mats = alloc_mats(c, shapes);
      GemmBatch gb;
      for (int64_t k = 0; k < m; ++k) {
        for (int side = 0; side < 2; ++side) {
          const Mat Tq = side == 0 ? P.U[lvl][k].Qs() : P.V[lvl][k].Qs();
          const auto& child = side == 0 ? Ubig : Vbig;
          const Mat u0 = child[2 * k], u1 = child[2 * k + 1];
          const Mat out = mats[2 * k + side].m;
          if (Tq.cols == 0) continue;
          gemm1(gb, out.sub(0, 0, u0.rows, Tq.cols), u0, Tq.sub(0, 0, u0.cols, Tq.cols));
          gemm1(gb, out.sub(u0.rows, 0, u1.rows, Tq.cols), u1, Tq.sub(u0.cols, 0, u1.cols, Tq.cols));
        }
        nu[k] = mats[2 * k].m;
        nv[k] = mats[2 * k + 1].m;
      }
      gb.run(c);
      std::vector<DMat> keep = std::move(mats);
      big_owner_next_ = std::move(keep);
    }
    Ubig = std::move(nu);
    Vbig = std::move(nv);
  }
  std::vector<DMat> big_owner_next_;

  // ---- NodepDriver::run (ulv.cpp:710-760) -----------------------------------------
  void run() {
    SysL sys;
    sys.lvl = L;
    sys.m = 1 << L;
    sys.dims.resize(sys.m);
    for (int64_t i = 0; i < sys.m; ++i) sys.dims[i] = int(rs(L, i));
    sys.blocks = P.near;
    sys.offdiag = false;
    for (int64_t i = 0; i < sys.m && !sys.offdiag; ++i)
      for (int64_t t = 0; t < S.nnear(L, i); ++t)
        if (S.near(L, i)[t] != i) sys.offdiag = true;
    P.U.assign(L + 1, {});
    P.V.assign(L + 1, {});
    for (int l = 0; l <= L; ++l) {
      P.U[l].resize(size_t(1) << l);
      P.V[l].resize(size_t(1) << l);
    }
    if (getenv("H2G_LEAF_GEN") == nullptr) {
      const auto [plo, phi] = own_range(sys.m);
      const bool offdiag = sys.offdiag;
      leaf_plan_future_ = std::async(std::launch::async, [this, plo = plo, phi = phi, offdiag] {
        return make_leaf_plans(leaf_piece_keys(), offdiag, plo, phi, nullptr);
      });
    }
    // prepare_factor_inputs (ulv.cpp:1108-1126)
    FillSet fills;
    if (opt.structure == 0 && sys.offdiag) fills = precompute_fillins(sys);
    FillSet basis_fills;
    for (auto& [k, F] : fills)
      if (k.first != k.second) basis_fills[k] = F;
    build_leaf_bases(sys, basis_fills);

    // H2G_HOST_PROF: host seconds per driver stage (enqueue + any syncs).
    const bool hp = getenv("H2G_HOST_PROF") != nullptr;
    double hpt = now_s();
    auto mark = [&](const char* what) {
      if (!hp) return;
      const double t = now_s();
      fprintf(stderr, "HOSTSTAGE level %d %-18s %.4f s\n", sys.lvl, what, t - hpt);
      hpt = t;
    };
    mark("leaf_bases");
    while (true) {
      const bool is_leaf = sys.lvl == L;
      std::vector<PieceMap> pieces, stack, merged;
      P.max_fill_resid.push_back(0.0);
      double* lm = &P.max_fill_resid.back();
      if (is_leaf) {
        build_leaf_pieces(sys, fills, pieces, lm);
        mark("leaf_pieces");
      } else {
        fills = precompute_fillins(sys);
        mark("fills");
        build_upper_pieces(sys, fills, stack, merged);
        mark("upper_pieces");
        build_transfers(sys, fills, merged);
        mark("transfers");
      }
      std::vector<DMat> diag_S;
      std::map<std::pair<int64_t, int64_t>, DMat> far_ss, dense_ss;
      assemble_level(sys, fills, pieces, merged, diag_S, far_ss, dense_ss, lm);
      mark("assemble");
      LevelF lf;
      lf.level = sys.lvl;
      lf.dims = sys.dims;
      lf.ranks.resize(sys.m);
      for (int64_t k = 0; k < sys.m; ++k) lf.ranks[k] = P.U[sys.lvl][k].rank;
      eliminate_level(sys, diag_S, lf);
      mark("eliminate");
      lf.use_z = sys.offdiag;
      // project_pieces (ulv.cpp:675-689)
      {
        PhaseTimer pt(c, P.stats, "skeleton");
        std::vector<PieceMap> next(sys.m);
        GemmBatch gb;
        std::vector<std::pair<int64_t, TargetKey>> keys;
        std::vector<std::pair<int, int>> shapes;
        const auto& src = is_leaf ? pieces : merged;
        for (int64_t k = 0; k < sys.m; ++k)
          for (auto& [tk, piece] : src[k]) {
            if (tk.first == sys.lvl) continue;
            if (is_leaf) {
              next[k][tk] = piece;
            } else {
              keys.push_back({k, tk});
              shapes.push_back({P.U[sys.lvl][k].rank, piece.cols()});
            }
          }
        const bool part = P.comm && P.comm->partitioned(sys.m);
        if (is_leaf) {
          if (part) stacked_.clear();  // (single-GPU: build_leaf_pieces stacked them)
        } else {
          stacked_.clear();
        }
        std::vector<DMat> mats;
        if (!is_leaf && !part && sys.m >= 2) {
          std::vector<int> pr;
          for (auto& sh : shapes) pr.push_back(sh.first);
          mats = alloc_stacked(sys.m, keys, pr);
        } else {
          mats = alloc_mats(c, shapes);
        }
        const auto [lo, hi] = own_range(sys.m);  // multi-GPU: own boxes, then all-gathered
        std::vector<int64_t> box(keys.size());
        for (size_t t = 0; t < keys.size(); ++t) {
          const auto [k, tk] = keys[t];
          next[k][tk] = mats[t];
          box[t] = k;
          if (k >= lo && k < hi) gemm1(gb, mats[t].m, P.U[sys.lvl][k].Qs().t(), src[k].at(tk).m);
        }
        gb.run(c);
        exchange_mats(mats, box, sys.m);
        carried = std::move(next);
      }
      mark("project_pieces");
      make_layer(sys.lvl);
      big_owner = std::move(big_owner_next_);
      if (opt.structure == 2) {  // BLR^2: one level, then the flat top system
        finish_blr2(sys, diag_S, far_ss, dense_ss);
        lf.sys = std::move(sys);
        P.levels.push_back(std::move(lf));
        break;
      }
      SysL next = merge(sys, diag_S, far_ss, dense_ss);
      mark("layer+merge");
      lf.sys = std::move(sys);
      P.levels.push_back(std::move(lf));
      const int next_lvl = next.lvl;
      int64_t total = 0;
      for (int d : next.dims) total += d;
      if (next_lvl <= 1 || total <= 4 * P.T.leaf) {
        assemble_top(next);
        break;
      }
      sys = std::move(next);
    }
  }
};

}  // namespace

void Problem::factor() {
  if (!built) throw std::logic_error("Pipeline::factor: build() first");
  if (factored) return;
  const double t0 = now_s();
  DevTimer dt(c.stream);
  if (auto_budget_) {
    const size_t fr = c.free_bytes();
    opt.qr_mem_budget = std::max<size_t>(size_t(1) << 28, fr / 3);
  }
  c.phase_flops.clear();
  const char* qm = getenv("H2G_QR_MODE");  // experiment override
  const int qmode = qm ? (std::string(qm) == "compressed" ? 2 : std::string(qm) == "blocked" ? 1 : 0) : opt.qr_mode;
  c.qr_blocked = qmode >= 1;
  c.qr_compress = qmode == 2;
  c.fast_solve = qmode == 2 && getenv("H2G_EXACT_SOLVES") == nullptr;
  levels.clear();
  max_fill_resid.clear();
  Driver d(*this);
  d.run();
  c.sync();
  stats.t_factor_dev = dt.stop();
  stats.t_factor = now_s() - t0;
  c.prof_resolve();
  host_prof_report();
  for (auto& [k, v] : c.phase_flops) stats.phase_flops[k] += v;
  stats.launches = c.launches;
  stats.max_fill_residual = 0;
  for (double r : max_fill_resid) stats.max_fill_residual = std::max(stats.max_fill_residual, r);
  factored = true;
}

void Problem::matvec(const double* d_x, double* d_y, int nrhs) {
  if (!built) throw std::logic_error("matvec: build() first");
  Slab flag = c.alloc(sizeof(int));
  cuda_check(cudaMemsetAsync(flag.get(), 0, sizeof(int), c.stream), "memset");
  launch_matvec(c.kp, orig, d_x, d_y, nrhs, static_cast<int*>(flag.get()), c.stream);
  int h = 0;
  cuda_check(cudaMemcpyAsync(&h, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream), "flag");
  c.sync();
  if (h) throw std::runtime_error("assemble_block: singular evaluation (r + eta_reg == 0)");
}

// ---- solve (solve.cpp:17-224), all right-hand sides at once -------------------
void Problem::solve(const double* d_b, double* d_x, int nrhs) {
  if (!factored) throw std::logic_error("Pipeline::solve_rhs: factor() first");
  const double t0 = now_s();
  DevTimer dt(c.stream);
  const int64_t n = T.n;
  const int L = T.levels;
  const std::string saved_phase = c.phase;
  c.phase = "solve";
  DMat bp = alloc_mat(c, int(n), nrhs);
  launch_permute_rows(bp.m, Mat{const_cast<double*>(d_b), int(n), nrhs, 1, n}, T.order, 0, c.stream);
  // r[k]: leaf segments (views).
  std::vector<Mat> r(size_t(1) << L);
  for (int64_t k = 0; k < (int64_t(1) << L); ++k)
    r[k] = bp.m.sub(int(range_begin(L, k)), 0, int(range_size(L, k)), nrhs);
  std::vector<std::vector<DMat>> z_all(levels.size());
  std::vector<DMat> keep;
  for (size_t li = 0; li < levels.size(); ++li) {
    const LevelF& lf = levels[li];
    const int lvl = lf.level;
    const int64_t m = int64_t(lf.dims.size());
    std::vector<Mat> rt = r;
    if (lf.use_z) {
      std::vector<std::pair<int, int>> shapes;
      for (int64_t p = 0; p < m; ++p) shapes.push_back({lf.dims[p], nrhs});
      for (int64_t k = 0; k < m; ++k) shapes.push_back({lf.dims[k], nrhs});
      std::vector<std::pair<int64_t, int64_t>> prods;
      for (int64_t k = 0; k < m; ++k)
        for (int64_t t = 0; t < S.nnear(lvl, k); ++t)
          if (S.near(lvl, k)[t] != k) {
            prods.push_back({k, S.near(lvl, k)[t]});
            shapes.push_back({lf.dims[k], nrhs});
          }
      auto mats = alloc_mats(c, shapes);
      CopyBatch cb;
      SolveBatch sb;
      for (int64_t p = 0; p < m; ++p) {
        cb.copy(mats[p].m, r[p]);
        sb.add(lf.sys.diag_lu[p], mats[p].m, SOLVE_FULL);
      }
      cb.run(c);
      sb.run(c);
      GemmBatch gb;
      for (size_t t = 0; t < prods.size(); ++t) {
        const auto [k, p] = prods[t];
        const int tt = Driver::find_near(S, lvl, k, p);
        gemm1(gb, mats[2 * m + t].m, lf.sys.blocks[tt].m, mats[p].m);
      }
      gb.run(c);
      AccBatch acc;
      size_t t = 0;
      for (int64_t k = 0; k < m; ++k) {
        acc.job(mats[m + k].m, true);
        acc.src(r[k], 1.0);
        for (; t < prods.size() && prods[t].first == k; ++t) acc.src(mats[2 * m + t].m, -1.0);
        rt[k] = mats[m + k].m;
      }
      acc.run(c);
      keep.insert(keep.end(), mats.begin(), mats.end());
    }
    // c = [Ur Us]^T rt; z = L^-1 P c_R; s = c_S - L^SR z.
    std::vector<std::pair<int, int>> shapes;
    for (int64_t k = 0; k < m; ++k) {
      shapes.push_back({lf.dims[k], nrhs});
      shapes.push_back({lf.elim[k].sdim, nrhs});
    }
    auto mats = alloc_mats(c, shapes);
    GemmBatch g1, g2;
    SolveBatch sb;
    AccBatch acc;
    z_all[li].resize(m);
    std::vector<Mat> s(m);
    for (int64_t k = 0; k < m; ++k) {
      const ElimF& el = lf.elim[k];
      const Mat cvec = mats[2 * k].m;
      gemm1(g1, cvec, U[lvl][k].SQ.m.t(), rt[k]);
      const Mat z = cvec.sub(0, 0, el.rdim, nrhs);
      if (el.rdim > 0) sb.add(el.piv, z, SOLVE_LOWER);
      s[k] = cvec.sub(el.rdim, 0, el.sdim, nrhs);
      if (el.rdim > 0 && el.sdim > 0) {
        gemm1(g2, mats[2 * k + 1].m, el.lsr.m, z);
        acc.job(s[k], false);
        acc.src(mats[2 * k + 1].m, -1.0);
      }
      z_all[li][k] = DMat{z, mats[2 * k].owner};
    }
    g1.run(c);
    sb.run(c);
    g2.run(c);
    acc.run(c);
    keep.insert(keep.end(), mats.begin(), mats.end());
    // Stack skeleton parts for the next system.
    const int64_t mp = m / 2;
    std::vector<std::pair<int, int>> pshapes;
    for (int64_t I = 0; I < mp; ++I) pshapes.push_back({s[2 * I].rows + s[2 * I + 1].rows, nrhs});
    auto nr = alloc_mats(c, pshapes);
    CopyBatch cb;
    std::vector<Mat> rn(mp);
    for (int64_t I = 0; I < mp; ++I) {
      if (s[2 * I].rows) cb.copy(nr[I].m.sub(0, 0, s[2 * I].rows, nrhs), s[2 * I]);
      if (s[2 * I + 1].rows) cb.copy(nr[I].m.sub(s[2 * I].rows, 0, s[2 * I + 1].rows, nrhs), s[2 * I + 1]);
      rn[I] = nr[I].m;
    }
    cb.run(c);
    keep.insert(keep.end(), nr.begin(), nr.end());
    r = std::move(rn);
  }
  // Top dense solve.
  const int tn = top.n();
  DMat y = alloc_mat(c, tn, nrhs);
  {
    CopyBatch cb;
    int at = 0;
    for (auto& piece : r) {
      if (piece.rows) cb.copy(y.m.sub(at, 0, piece.rows, nrhs), piece);
      at += piece.rows;
    }
    cb.run(c);
    SolveBatch sb;
    sb.add(top, y.m, SOLVE_FULL);
    sb.run(c);
  }
  std::vector<Mat> ys;
  {
    // The downward pass splits parent segments into their children; a top
    // system at the last factorized level itself (BLR^2) is regrouped by pairs.
    std::vector<int> seg(cutoff_dims.begin(), cutoff_dims.end());
    if (!levels.empty() && cutoff_level == levels.back().level) {
      std::vector<int> pairs;
      for (size_t k = 0; k + 1 < seg.size(); k += 2) pairs.push_back(seg[k] + seg[k + 1]);
      seg = pairs;
    }
    int at = 0;
    for (int d : seg) {
      ys.push_back(y.m.sub(at, 0, d, nrhs));
      at += d;
    }
  }
  // Downward pass.
  for (int64_t li = int64_t(levels.size()) - 1; li >= 0; --li) {
    const LevelF& lf = levels[li];
    const int lvl = lf.level;
    const int64_t m = int64_t(lf.dims.size());
    std::vector<std::pair<int, int>> shapes;
    for (int64_t k = 0; k < m; ++k) {
      shapes.push_back({lf.elim[k].rdim, nrhs});
      shapes.push_back({lf.dims[k], nrhs});
    }
    auto mats = alloc_mats(c, shapes);
    GemmBatch g1, g2;
    AccBatch acc;
    SolveBatch sb;
    std::vector<Mat> yfull(m);
    for (int64_t k = 0; k < m; ++k) {
      const ElimF& el = lf.elim[k];
      const int64_t parent = k >> 1;
      const int off = (k & 1) ? lf.ranks[k - 1] : 0;
      const Mat yskel = ys[parent].sub(off, 0, lf.ranks[k], nrhs);
      const Mat yr = z_all[li][k].m;
      if (el.rdim > 0) {
        if (el.sdim > 0) {
          gemm1(g1, mats[2 * k].m, el.urs.m, yskel);
          acc.job(yr, false);
          acc.src(mats[2 * k].m, -1.0);
        }
        sb.add(el.piv, yr, SOLVE_UPPER);
      }
      // x_k = [V_r V_s] [y_R; y_S] as one product over the stacked vector.
      const Basis& Vk = V[lvl][k];
      g2.job(mats[2 * k + 1].m, false);
      if (el.rdim > 0) g2.seg(Vk.SQ.m.sub(0, 0, Vk.dim, el.rdim), yr);
      if (el.sdim > 0) g2.seg(Vk.SQ.m.sub(0, el.rdim, Vk.dim, el.sdim), yskel);
      yfull[k] = mats[2 * k + 1].m;
    }
    g1.run(c);
    acc.run(c);
    sb.run(c);
    g2.run(c);
    keep.insert(keep.end(), mats.begin(), mats.end());
    ys = std::move(yfull);
  }
  // Leaf segments back to the original ordering.
  DMat xp = alloc_mat(c, int(n), nrhs);
  {
    CopyBatch cb;
    for (int64_t k = 0; k < (int64_t(1) << L); ++k)
      if (ys[k].rows) cb.copy(xp.m.sub(int(range_begin(L, k)), 0, ys[k].rows, nrhs), ys[k]);
    cb.run(c);
  }
  launch_permute_rows(Mat{d_x, int(n), nrhs, 1, n}, xp.m, T.order, 1, c.stream);
  c.sync();
  c.phase = saved_phase;
  stats.t_solve_dev = dt.stop();
  stats.t_solve = now_s() - t0;
  c.prof_resolve();
}

}  // namespace h2g
