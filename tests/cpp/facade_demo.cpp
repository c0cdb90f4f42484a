// Drives the B200 path through the C++ façade (include/h2ulv_b200.hpp) the
// way a caller of the reference's Pipeline would (report.hpp:73-99), and
// prints what tests/test_facade.py checks against the reference's golden
// fixtures: tree permutation and solution bit hashes, the ranks, the
// residual, and the reference's exception types/messages.
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "h2ulv_b200.hpp"

using namespace h2ulv_b200;

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
    Matrix x = solve(pipe, b);
    Matrix y = pipe.matvec(x);
    double rn = 0, bn = 0;
    for (int64_t i = 0; i < n; ++i) {
      rn += (y(i, 0) - b(i, 0)) * (y(i, 0) - b(i, 0));
      bn += b(i, 0) * b(i, 0);
    }
    ClusterTreeResult t = pipe.tree();
    ClusterTreeResult t2 = build_cluster_tree(pipe.original_cloud(), leaf);
    BlockStructure s = pipe.structure();
    BlockStructure s2 = classify_blocks(pipe.original_cloud(), leaf, AdmissibilityRule{});
    bool same_lists = s.levels == s2.levels;
    for (int l = 1; l <= s.levels && same_lists; ++l)
      same_lists = s.level[size_t(l)].near_cols == s2.level[size_t(l)].near_cols &&
                   s.level[size_t(l)].far_cols == s2.level[size_t(l)].far_cols;
    int64_t rank_sum = 0;
    for (auto& [lvl, r] : pipe.ranks())
      for (int64_t v : r) rank_sum += v;
    printf("{\"n\": %lld, \"levels\": %d, \"perm_fnv\": %llu, \"x_fnv\": %llu, \"residual\": %.17g, "
           "\"same_tree\": %s, \"same_lists\": %s, \"rank_sum\": %lld}\n",
           (long long)n, t.tree.levels, (unsigned long long)fnv(t.tree.original_index.data(), size_t(n)),
           (unsigned long long)fnv(x.data(), size_t(n)), std::sqrt(rn / bn),
           t.tree.original_index == t2.tree.original_index ? "true" : "false", same_lists ? "true" : "false",
           (long long)rank_sum);
  } catch (const std::runtime_error& e) {
    printf("{\"runtime_error\": \"%s\"}\n", e.what());
    return 2;
  }
  return 0;
}
