/* TEST INFRASTRUCTURE ONLY — CPU restatement of the bit-exact front half of
 * the reference H2-ULV path. Never linked into the product; loaded by tests/
 * and smoke() through ctypes as the checker. Pinned against the compiled
 * reference (oracle/_ref/libh2ref.so) in tests/test_oracle.py. */
#ifndef H2ORACLE_H
#define H2ORACLE_H
#include <stdint.h>

/* geometry.cpp:42-52 / :54-62 / :64-95 */
int  or_generate(int geometry, int64_t n, uint64_t seed, int64_t spheres, double spacing,
                 double* xyz, double* q);
double or_domain_diameter(int64_t n, const double* xyz);          /* geometry.cpp:28-40 */
double or_default_eta_reg(double diam, int64_t n);                 /* kernels.cpp:228-230 */
int  or_tree_levels(int64_t n, int64_t leaf);                       /* geometry.cpp:234-235 */
/* build_cluster_tree (geometry.cpp:222-261): xyz/q permuted in place,
 * order[i] = original index, nodes_be 2*(2^(L+1)-1), nodes_geo 4*(...). */
int  or_build_tree(int64_t n, int64_t leaf, double* xyz, double* q, int64_t* order,
                   int64_t* nodes_be, double* nodes_geo);
/* classify_blocks (hstructure.cpp:64-114) for one level given the parent
 * near CSR; returns counts through *nnear/*nfar when outputs are NULL. */
int  or_classify(int levels, const double* nodes_geo, double eta, int weak,
                 int64_t* near_ptr_all, int64_t* near_idx_all, int64_t* far_ptr_all,
                 int64_t* far_idx_all, int64_t* near_total, int64_t* far_total);
/* assemble_block (kernels.cpp:242-268), column-major rows x cols. */
int  or_assemble_block(int kind, double alpha_m, double scale, double reg, const double* xyz,
                       const double* q, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                       double* out);
uint64_t or_fnv64(const int64_t* v, int64_t n);
#endif
