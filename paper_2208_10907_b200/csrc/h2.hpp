// The B200 H2-ULV problem: device-resident tree, structure, near-field arena,
// factors, and the solve. Mirrors the reference's proj/include API objects
// (ClusterTree, BlockStructure, HMatrix, SharedBasisSet, ULVFactors).
#pragma once
#include <array>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "batch.hpp"
#include "comm.hpp"
#include "tree.hpp"

namespace h2g {

struct Options {  // FactorOptions (ulv.hpp:29-45) + RunConfig bits
  double tol = 1e-8;
  int cap = 0;  // <= 0: none
  double rr_pivot_tol = 1e-13;
  bool absorb_coupling = true;
  double abort_residual_factor = 100.0;
  int structure = 0;  // 0 h2 (strong, nodep), 1 hss (weak), 2 blr2 (flat, weak)
  double eta = 1.0;
  size_t qr_mem_budget = size_t(8) << 30;  // auto (free/3) unless set
  int qr_mode = 0;  // 0 exact (k_qr.cu, bit-exact), 1 blocked (k_qrb.cu, tolerance parity)
  // true: the reference's assembly bit for bit (covered couplings skipped,
  // ulv.cpp:424-463, :583-603); false: corrected (oracle/fix_reference.py).
  bool reference_compat = true;
  // > 0: far-field basis members wider than this many columns are replaced by
  // a strided sample of about this many of their columns (the north star's
  // "far-field samples"; the reference concatenates every column,
  // compression.cpp:153-177, ulv.cpp:476-521). 0 = the reference's members.
  int sample_cols = 0;
};

struct Basis {  // SharedBasis (hstructure.hpp:61-69): square [Qr | Qs]
  DMat SQ;
  int dim = 0, rank = 0;
  Mat Qs() const { return SQ.m.sub(0, dim - rank, dim, rank); }
  Mat Qr() const { return SQ.m.sub(0, 0, dim, dim - rank); }
};

struct SysL {  // DenseSystem (compression.hpp:21-38) aligned with the level's near CSR
  int lvl = 0;
  int m = 0;
  std::vector<int> dims;
  std::vector<DMat> blocks;  // blocks[near_ptr[i] + c]
  std::vector<LuF> diag_lu;
  bool offdiag = false;
};

struct ElimF {  // ClusterFactors (ulv.hpp:48-54)
  LuF piv;
  DMat urs, lsr;
  int rdim = 0, sdim = 0;
};

struct LevelF {  // LevelFactors (ulv.hpp:60-68)
  int level = 0;
  std::vector<int> dims, ranks;
  std::vector<ElimF> elim;
  SysL sys;
  bool use_z = false;
};

using TargetKey = std::pair<int, int64_t>;
using PieceMap = std::map<TargetKey, DMat>;
using FillSet = std::map<std::pair<int64_t, int64_t>, DMat>;

struct Stats {
  double t_tree = 0, t_classify = 0, t_near = 0, t_factor = 0, t_solve = 0;
  double t_build_dev = 0, t_factor_dev = 0, t_solve_dev = 0;  // CUDA events
  std::map<std::string, double> phase_flops, phase_seconds;
  int64_t launches = 0;
  double kernel_evals = 0;
  double max_fill_residual = 0;
};

class Problem {
 public:
  Ctx c;
  DeviceTree T;
  Structure S;
  std::vector<int64_t> be;  // host copy of node ranges
  Slab near_slab;
  std::vector<DMat> near;  // leaf near blocks aligned with S.level[L] near CSR
  Options opt;
  Stats stats;
  Slab orig_slab;  // original-order SoA cloud (matrix-free matvec)
  Cloud orig;
  // factors
  std::vector<std::vector<Basis>> U, V;
  std::vector<LevelF> levels;
  int cutoff_level = 0;
  std::vector<int> cutoff_dims;
  LuF top;
  std::vector<double> max_fill_resid;
  bool built = false, factored = false;
  // All charges equal: A(I, i)^T == A(i, I) bit for bit (kernel_pair is
  // symmetric in the two points), so column members can reuse row members.
  bool uniform_q = false;
  bool auto_budget_ = true;
  // Multi-GPU level partition (null: single GPU). The partitioned stages
  // compute only this rank's box range and all-gather their outputs, so
  // every rank ends with the single-GPU factors bit for bit.
  std::shared_ptr<Comm> comm;

  Problem();
  ~Problem();
  void set_kernel(const KernelParams& kp) { c.kp = kp; }
  // Run on a caller-owned stream (e.g. torch's) instead of the private one.
  void use_stream(cudaStream_t s);
  bool own_stream_ = true;
  void build(const double* d_xyz, const double* d_q, int64_t n, int64_t leaf);  // device inputs
  void choose_allocator(int64_t n, int64_t leaf);  // arena or stream-ordered pool, by predicted footprint
  void factor();
  // b and x: device, n x nrhs column-major, ORIGINAL point order.
  void solve(const double* d_b, double* d_x, int nrhs);
  void matvec(const double* d_x, double* d_y, int nrhs);
  int64_t range_begin(int l, int64_t i) const { return be[2 * ((int64_t(1) << l) - 1 + i)]; }
  int64_t range_end(int l, int64_t i) const { return be[2 * ((int64_t(1) << l) - 1 + i) + 1]; }
  int64_t range_size(int l, int64_t i) const { return range_end(l, i) - range_begin(l, i); }
  int leaf_level() const { return T.levels; }
};

}  // namespace h2g
