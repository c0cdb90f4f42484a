// Drives the B200 path through the drop-in header tree (include/h2ulv/) the
// way a caller of the reference's Pipeline would (report.hpp:73-99), and
// prints what tests/test_facade.py checks against the reference's golden
// fixtures: tree permutation and solution bit hashes, the ranks, the
// residual, and the reference's exception types/messages.
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "h2ulv/prng.hpp"
#include "h2ulv/report.hpp"

using namespace h2ulv;

static uint64_t fnv(const void* p, size_t n64) {
  uint64_t h = 0xcbf29ce484222325ULL;
  const auto* v = static_cast<const uint64_t*>(p);
  for (size_t i = 0; i < n64; ++i) {
    h ^= v[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 4096;
  const int64_t leaf = argc > 2 ? atoll(argv[2]) : 128;
  if (argc > 3 && std::strcmp(argv[3], "report") == 0) {  // RunReport::to_json of run_pipeline
    RunConfig cfg;
    cfg.n = n;
    cfg.leaf_size = leaf;
    cfg.scale = 1.0;
    cfg.reg = 1e-3;
    cfg.tol = 1e-8;
    printf("%s\n", run_pipeline(cfg).to_json().c_str());
    return 0;
  }
  // Configuration errors are the reference's invalid_argument (report.cpp:43-58).
  try {
    RunConfig bad;
    bad.n = 100;
    bad.leaf_size = 256;
    Pipeline p(bad);
    printf("{\"error\": \"validate did not throw\"}\n");
    return 1;
  } catch (const std::invalid_argument& e) {
    printf("{\"invalid_argument\": \"%s\"}\n", e.what());
  }
  try {
    RunConfig cfg;
    cfg.n = n;
    cfg.leaf_size = leaf;
    cfg.scale = 1.0;
    cfg.reg = 1e-3;
    cfg.tol = 1e-8;
    Pipeline pipe(cfg);
    pipe.factor();
    Matrix b(n, 1);
    SplitMix64 rng(7);
    for (int64_t i = 0; i < n; ++i) b(i, 0) = rng.next_signed();
    Matrix x = solve(pipe.factors(), b);  // solve(const ULVFactors&, const Matrix&)
    Matrix y = pipe.matvec(x);
    double rn = 0, bn = 0;
    for (int64_t i = 0; i < n; ++i) {
      rn += (y(i, 0) - b(i, 0)) * (y(i, 0) - b(i, 0));
      bn += b(i, 0) * b(i, 0);
    }
    // The free-function path: build_cluster_tree -> classify_blocks ->
    // materialize_dense -> build_and_factorize -> solve (hstructure.hpp,
    // ulv.hpp, solve.hpp), against the Pipeline's tree, lists and x.
    const HMatrix& H = pipe.hmatrix();
    ClusterTreeResult t2 = build_cluster_tree(pipe.original_cloud(), leaf);
    BlockStructure s2 = classify_blocks(t2.tree, AdmissibilityRule{}, StructureVariant::h2);
    bool same_lists = H.structure.levels == s2.levels;
    for (int l = 1; l <= s2.levels && same_lists; ++l)
      same_lists = H.structure.level[size_t(l)].near_cols == s2.level[size_t(l)].near_cols &&
                   H.structure.level[size_t(l)].far_cols == s2.level[size_t(l)].far_cols;
    HMatrix H2 = materialize_dense(s2, t2.tree, t2.cloud, pipe.kernel(), StructureVariant::h2);
    FactorOptions fo;
    fo.tol = cfg.tol;
    ULVFactors f2 = build_and_factorize(H2, fo);
    Matrix x2 = solve(f2, b);
    bool same_near = H2.leaf_dense.size() == H.leaf_dense.size();
    for (size_t i = 0; i < H.leaf_dense.size() && same_near; ++i)
      for (size_t c = 0; c < H.leaf_dense[i].size() && same_near; ++c)
        same_near = fnv(H.leaf_dense[i][c].data(), size_t(H.leaf_dense[i][c].size())) ==
                    fnv(H2.leaf_dense[i][c].data(), size_t(H2.leaf_dense[i][c].size()));
    int64_t rank_sum = 0;
    for (const auto& lf : pipe.factors().levels)
      for (int64_t v : lf.ranks) rank_sum += v;
    const ClusterTree& t = H.tree;
    printf("{\"n\": %lld, \"levels\": %d, \"perm_fnv\": %llu, \"x_fnv\": %llu, \"residual\": %.17g, "
           "\"same_tree\": %s, \"same_lists\": %s, \"same_near\": %s, \"same_x_free_api\": %s, "
           "\"rank_sum\": %lld}\n",
           (long long)n, t.levels, (unsigned long long)fnv(t.original_index.data(), size_t(n)),
           (unsigned long long)fnv(x.data(), size_t(n)), std::sqrt(rn / bn),
           t.original_index == t2.tree.original_index ? "true" : "false", same_lists ? "true" : "false",
           same_near ? "true" : "false",
           fnv(x.data(), size_t(n)) == fnv(x2.data(), size_t(n)) ? "true" : "false", (long long)rank_sum);
  } catch (const std::runtime_error& e) {
    printf("{\"runtime_error\": \"%s\"}\n", e.what());
    return 2;
  }
  return 0;
}
