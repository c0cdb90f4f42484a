/* TEST INFRASTRUCTURE ONLY — CPU restatement of the bit-exact front half of
 * the reference (/root/reference/proj). It is the checker for the GPU tree,
 * classification and near-field kernels, never the product. Compiled with
 * -ffp-contract=off; the FMAs GCC -O3 -mfma contracts in the reference are
 * written out explicitly with fma() so results are bitwise identical
 * (pinned in tests/test_oracle.py against oracle/_ref/libh2ref.so). */
#include "h2oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- SplitMix64 (prng.hpp:14-25) ---- */
typedef struct { uint64_t s; } smx;
static uint64_t smx_u64(smx* r) {
  uint64_t z = (r->s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double smx_double(smx* r) { return (double)(smx_u64(r) >> 11) * 0x1.0p-53; }

/* dist2 (geometry.cpp:17-20) as contracted by GCC: fma(dz,dz,fma(dx,dx,dy*dy)). */
static double dist2(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return fma(dz, dz, fma(dx, dx, dy * dy));
}

int or_generate(int geometry, int64_t n, uint64_t seed, int64_t spheres, double spacing,
                double* xyz, double* q) {
  if (n < 2) return 1;
  smx rng = {seed};
  for (int64_t i = 0; i < n; ++i) q[i] = 1.0;
  if (geometry == 0) { /* geometry.cpp:42-52 */
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) xyz[3 * i + d] = smx_double(&rng);
    return 0;
  }
  if (geometry == 1) { /* geometry.cpp:54-62 */
    for (int64_t i = 0; i < n; ++i) {
      xyz[3 * i] = smx_double(&rng);
      xyz[3 * i + 1] = 0.0;
      xyz[3 * i + 2] = 0.0;
    }
    return 0;
  }
  /* Fibonacci-lattice spheres on a cubic lattice (geometry.cpp:64-95). */
  int64_t side = (int64_t)llround(cbrt((double)spheres));
  if (side < 1 || side * side * side != spheres) return 2;
  const double origin = -0.5 * spacing * (double)(side - 1);
  const double golden = (1.0 + sqrt(5.0)) / 2.0;
  int64_t remaining = n, sphere_idx = 0, at = 0;
  for (int64_t ix = 0; ix < side; ++ix)
    for (int64_t iy = 0; iy < side; ++iy)
      for (int64_t iz = 0; iz < side; ++iz, ++sphere_idx) {
        const int64_t left = spheres - sphere_idx;
        const int64_t m = (remaining + left - 1) / left;
        remaining -= m;
        const double c0 = origin + spacing * ix, c1 = origin + spacing * iy,
                     c2 = origin + spacing * iz;
        const double phase = smx_double(&rng) * 2.0 * M_PI;
        for (int64_t t = 0; t < m; ++t) {
          const double z = 1.0 - 2.0 * (t + 0.5) / (double)m;
          const double zz = fma(-z, z, 1.0); /* 1 - z*z contracted */
          const double r = sqrt(zz > 0.0 ? zz : 0.0);
          const double phi = fma(2.0 * M_PI, t / golden, phase);
          xyz[3 * at] = fma(r, cos(phi), c0);
          xyz[3 * at + 1] = fma(r, sin(phi), c1);
          xyz[3 * at + 2] = c2 + z;
          ++at;
        }
      }
  return 0;
}

/* PointCloud::domain_diameter (geometry.cpp:28-40). */
double or_domain_diameter(int64_t n, const double* xyz) {
  double lo[3] = {1.7976931348623157e308, 1.7976931348623157e308, 1.7976931348623157e308};
  double hi[3] = {-1.7976931348623157e308, -1.7976931348623157e308, -1.7976931348623157e308};
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      const double v = xyz[3 * i + d];
      if (v < lo[d]) lo[d] = v;
      if (v > hi[d]) hi[d] = v;
    }
  /* GCC's contraction of the unrolled loop: fma(d2,d2, d0*d0 + d1*d1). */
  const double d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
  return sqrt(fma(d2, d2, d0 * d0 + d1 * d1));
}

double or_default_eta_reg(double diam, int64_t n) { return 1e-3 * diam / cbrt((double)n); }

int or_tree_levels(int64_t n, int64_t leaf) {
  int levels = 0;
  while (((int64_t)1 << levels) * leaf < n) ++levels;
  return levels;
}

/* ---- 2-means split (geometry.cpp:130-204) ---- */
typedef struct {
  double* xyz;
  double* q;
  int64_t* order;
  /* scratch */
  char* assign;
  int64_t* idx;
  int64_t* tmp_idx;
  double* margin;
  double* tp;
  double* tq;
  int64_t* to;
} splitter;

/* Stable merge sort of idx by margin (std::stable_sort with a < b). */
static void stable_sort_idx(int64_t* idx, int64_t* tmp, const double* key, int64_t n) {
  for (int64_t w = 1; w < n; w *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
      int64_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) tmp[o++] = (key[idx[b]] < key[idx[a]]) ? idx[b++] : idx[a++];
      while (a < mid) tmp[o++] = idx[a++];
      while (b < hi) tmp[o++] = idx[b++];
    }
    memcpy(idx, tmp, sizeof(int64_t) * n);
  }
}

static int64_t split(splitter* sp, int64_t begin, int64_t end, int64_t min_side) {
  const int64_t len = end - begin;
  const int64_t ncand = len < 32 ? len : 32;
  int64_t cand[32];
  for (int64_t i = 0; i < ncand; ++i) cand[i] = begin + (ncand == 1 ? 0 : i * (len - 1) / (ncand - 1));
  double best = -1.0;
  double c1[3], c2[3];
  memcpy(c1, sp->xyz + 3 * begin, sizeof c1);
  memcpy(c2, sp->xyz + 3 * (end - 1), sizeof c2);
  for (int64_t a = 0; a < ncand; ++a)
    for (int64_t b = a + 1; b < ncand; ++b) {
      const double d = dist2(sp->xyz + 3 * cand[a], sp->xyz + 3 * cand[b]);
      if (d > best) {
        best = d;
        memcpy(c1, sp->xyz + 3 * cand[a], sizeof c1);
        memcpy(c2, sp->xyz + 3 * cand[b], sizeof c2);
      }
    }
  char* assign = sp->assign;
  memset(assign, 0, (size_t)len);
  for (int iter = 0; iter < 100; ++iter) {
    int changed = 0;
    double s1[3] = {0, 0, 0}, s2[3] = {0, 0, 0};
    int64_t n1 = 0;
    for (int64_t i = 0; i < len; ++i) {
      const double* p = sp->xyz + 3 * (begin + i);
      const char a = dist2(p, c2) < dist2(p, c1) ? 1 : 0;
      if (a != assign[i]) {
        assign[i] = a;
        changed = 1;
      }
      if (a == 0) {
        ++n1;
        for (int d = 0; d < 3; ++d) s1[d] += p[d];
      } else {
        for (int d = 0; d < 3; ++d) s2[d] += p[d];
      }
    }
    if (n1 > 0)
      for (int d = 0; d < 3; ++d) c1[d] = s1[d] / n1;
    if (len - n1 > 0)
      for (int d = 0; d < 3; ++d) c2[d] = s2[d] / (len - n1);
    if (!changed && iter > 0) break;
  }
  for (int64_t i = 0; i < len; ++i) {
    const double* p = sp->xyz + 3 * (begin + i);
    sp->idx[i] = i;
    sp->margin[i] = dist2(p, c1) - dist2(p, c2);
  }
  stable_sort_idx(sp->idx, sp->tmp_idx, sp->margin, len);
  int64_t n1 = 0;
  for (int64_t i = 0; i < len; ++i)
    if (sp->margin[sp->idx[i]] < 0.0) ++n1;
  if (n1 < min_side) n1 = min_side;
  if (n1 > len - min_side) n1 = len - min_side;
  for (int64_t i = 0; i < len; ++i) {
    memcpy(sp->tp + 3 * i, sp->xyz + 3 * (begin + sp->idx[i]), 3 * sizeof(double));
    sp->tq[i] = sp->q[begin + sp->idx[i]];
    sp->to[i] = sp->order[begin + sp->idx[i]];
  }
  memcpy(sp->xyz + 3 * begin, sp->tp, 3 * sizeof(double) * len);
  memcpy(sp->q + begin, sp->tq, sizeof(double) * len);
  memcpy(sp->order + begin, sp->to, sizeof(int64_t) * len);
  return begin + n1;
}

int or_build_tree(int64_t n, int64_t leaf, double* xyz, double* q, int64_t* order,
                  int64_t* be, double* geo) {
  if (leaf < 2) return 1;
  if (n < 2 * leaf) return 2;
  int distinct = 0;
  for (int64_t i = 1; i < n && !distinct; ++i)
    if (dist2(xyz + 3 * i, xyz) > 0.0) distinct = 1;
  if (!distinct) return 3;
  const int levels = or_tree_levels(n, leaf);
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  splitter sp = {xyz, q, order, malloc((size_t)n), malloc(8 * (size_t)n), malloc(8 * (size_t)n),
                 malloc(8 * (size_t)n), malloc(24 * (size_t)n), malloc(8 * (size_t)n),
                 malloc(8 * (size_t)n)};
  be[0] = 0;
  be[1] = n;
  for (int level = 0; level < levels; ++level) {
    const int64_t base = ((int64_t)1 << level) - 1, cbase = ((int64_t)1 << (level + 1)) - 1;
    const int64_t min_side = (int64_t)1 << (levels - level - 1);
    for (int64_t i = 0; i < ((int64_t)1 << level); ++i) {
      const int64_t b = be[2 * (base + i)], e = be[2 * (base + i) + 1];
      const int64_t mid = split(&sp, b, e, min_side);
      be[2 * (cbase + 2 * i)] = b;
      be[2 * (cbase + 2 * i) + 1] = mid;
      be[2 * (cbase + 2 * i + 1)] = mid;
      be[2 * (cbase + 2 * i + 1) + 1] = e;
    }
  }
  /* compute_geometry (geometry.cpp:207-218) */
  const int64_t nn = ((int64_t)1 << (levels + 1)) - 1;
  for (int64_t k = 0; k < nn; ++k) {
    const int64_t b = be[2 * k], e = be[2 * k + 1];
    double c[3] = {0, 0, 0};
    for (int64_t i = b; i < e; ++i)
      for (int d = 0; d < 3; ++d) c[d] += xyz[3 * i + d];
    for (int d = 0; d < 3; ++d) c[d] /= (double)(e - b);
    double r2 = 0.0;
    for (int64_t i = b; i < e; ++i) {
      const double d2 = dist2(xyz + 3 * i, c);
      if (d2 > r2) r2 = d2;
    }
    for (int d = 0; d < 3; ++d) geo[4 * k + d] = c[d];
    geo[4 * k + 3] = sqrt(r2);
  }
  free(sp.assign); free(sp.idx); free(sp.tmp_idx); free(sp.margin);
  free(sp.tp); free(sp.tq); free(sp.to);
  return 0;
}

/* admissible (geometry.cpp:263-277): 1 = admissible (far), 0 = near. */
static int is_admissible(const double* geo, int level, int64_t a, int64_t b, double eta, int weak) {
  if (weak) return a != b;
  const double* na = geo + 4 * (((int64_t)1 << level) - 1 + a);
  const double* nb = geo + 4 * (((int64_t)1 << level) - 1 + b);
  const double d = sqrt(dist2(na, nb));
  return d > eta * (na[3] + nb[3]);
}

/* classify_blocks (hstructure.cpp:64-114), h2/hss variants. Global row g of
 * level l, cluster i is g = 2^l - 2 + i. Per-row lists come out sorted
 * because each row's candidates are the children of its parent's (sorted)
 * near list, generated in ascending order. */
int or_classify(int levels, const double* geo, double eta, int weak, int64_t* near_ptr,
                int64_t* near_idx, int64_t* far_ptr, int64_t* far_idx, int64_t* near_total,
                int64_t* far_total) {
  const int64_t rows_total = ((int64_t)1 << (levels + 1)) - 2;
  int64_t* nptr = calloc((size_t)rows_total + 1, 8);
  int64_t* fptr = calloc((size_t)rows_total + 1, 8);
  int64_t cap = 1024, ncount = 0, fcount = 0;
  int64_t* nidx = malloc(8 * (size_t)cap);
  int64_t fcap = 1024;
  int64_t* fidx = malloc(8 * (size_t)fcap);
  for (int l = 1; l <= levels; ++l) {
    const int64_t m = (int64_t)1 << l, g0 = m - 2, pg0 = (m >> 1) - 2;
    for (int64_t i = 0; i < m; ++i) {
      const int64_t g = g0 + i;
      nptr[g] = ncount;
      fptr[g] = fcount;
      /* candidates: level 1 -> {0,1}; else children of parent's near list */
      int64_t pcount = (l == 1) ? 1 : (nptr[pg0 + (i >> 1) + 1] - nptr[pg0 + (i >> 1)]);
      for (int64_t t = 0; t < pcount; ++t) {
        const int64_t J = (l == 1) ? 0 : nidx[nptr[pg0 + (i >> 1)] + t];
        for (int64_t cj = 0; cj < 2; ++cj) {
          const int64_t j = 2 * J + cj;
          if (is_admissible(geo, l, i, j, eta, weak)) {
            if (fcount == fcap) fidx = realloc(fidx, 8 * (size_t)(fcap *= 2));
            fidx[fcount++] = j;
          } else {
            if (ncount == cap) nidx = realloc(nidx, 8 * (size_t)(cap *= 2));
            nidx[ncount++] = j;
          }
        }
      }
      nptr[g + 1] = ncount;
      fptr[g + 1] = fcount;
    }
  }
  *near_total = ncount;
  *far_total = fcount;
  if (near_ptr) {
    memcpy(near_ptr, nptr, 8 * ((size_t)rows_total + 1));
    memcpy(far_ptr, fptr, 8 * ((size_t)rows_total + 1));
    memcpy(near_idx, nidx, 8 * (size_t)ncount);
    memcpy(far_idx, fidx, 8 * (size_t)fcount);
  }
  free(nptr); free(fptr); free(nidx); free(fidx);
  return 0;
}

/* assemble_block (kernels.cpp:242-268): r = sqrt(fma(dz,dz,fma(dx,dx,dy*dy))).
 * kind 2 (Gaussian, BASELINE configs[2]) is NOT in the reference: q_j (exp(-alpha_m r^2)
 * + [r^2 == 0] reg) / scale; parity unpinned (our definition, checked by residual). */
int or_assemble_block(int kind, double alpha_m, double scale, double reg, const double* xyz,
                      const double* q, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                      double* out) {
  const int64_t nr = r1 - r0;
  for (int64_t j = c0; j < c1; ++j)
    for (int64_t i = r0; i < r1; ++i) {
      if (kind == 2) {
        const double r2 = dist2(xyz + 3 * i, xyz + 3 * j);
        out[(j - c0) * nr + (i - r0)] = q[j] * (exp(-alpha_m * r2) + (r2 == 0.0 ? reg : 0.0)) / scale;
        continue;
      }
      const double r = sqrt(dist2(xyz + 3 * i, xyz + 3 * j));
      const double denom = scale * (r + reg);
      if (denom == 0.0) return 1;
      out[(j - c0) * nr + (i - r0)] = kind == 0 ? q[j] / denom : q[j] * exp(-alpha_m * r) / denom;
    }
  return 0;
}

uint64_t or_fnv64(const int64_t* v, int64_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < n; ++i) {
    h ^= (uint64_t)v[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}
