// Seeded point clouds (host code): the reference's generators bit for bit
// (SplitMix64, prng.hpp:10-29; generate_uniform_cube / generate_line /
// generate_sphere_surface, geometry.cpp:42-95) plus the two BASELINE.json
// geometries the reference lacks (i.i.d. uniform sphere, union of random
// ellipsoids). Points are an input of the hot path, so this is host C++; it
// calls libm (glibc) cos/sin/sqrt/cbrt like the reference does, and spells
// out with std::fma every contraction GCC makes in the reference's
// -march=native build (checked bit for bit against oracle/_ref).
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/h2g.h"

namespace {

thread_local std::string g_points_err;

struct SplitMix64 {  // prng.hpp:10-29
  uint64_t s;
  uint64_t next_u64() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double next_double() { return double(next_u64() >> 11) * 0x1.0p-53; }
};

// geometry.cpp:64-95: Fibonacci lattices on a cubic lattice of unit spheres.
void fib_spheres(int64_t n, int64_t spheres, double spacing, uint64_t seed, double* xyz) {
  const int64_t side = int64_t(std::llround(std::cbrt(double(spheres))));
  if (side < 1 || side * side * side != spheres)
    throw std::invalid_argument("generate_sphere_surface: spheres must be a perfect cube count");
  SplitMix64 rng{seed};
  const double origin = -0.5 * spacing * double(side - 1);
  const double golden = (1.0 + std::sqrt(5.0)) / 2.0;
  const double two_pi = 2.0 * M_PI;
  int64_t remaining = n, sphere_idx = 0, at = 0;
  for (int64_t ix = 0; ix < side; ++ix)
    for (int64_t iy = 0; iy < side; ++iy)
      for (int64_t iz = 0; iz < side; ++iz, ++sphere_idx) {
        const int64_t left = spheres - sphere_idx;
        const int64_t m = (remaining + left - 1) / left;
        remaining -= m;
        const double c0 = origin + spacing * double(ix), c1 = origin + spacing * double(iy),
                     c2 = origin + spacing * double(iz);
        const double phase = rng.next_double() * 2.0 * M_PI;
        for (int64_t t = 0; t < m; ++t) {
          const double z = 1.0 - 2.0 * (double(t) + 0.5) / double(m);
          const double zz = std::fma(-z, z, 1.0);  // 1 - z*z, contracted
          const double r = std::sqrt(zz > 0.0 ? zz : 0.0);
          const double phi = std::fma(two_pi, double(t) / golden, phase);
          xyz[3 * at] = std::fma(r, std::cos(phi), c0);
          xyz[3 * at + 1] = std::fma(r, std::sin(phi), c1);
          xyz[3 * at + 2] = c2 + z;
          ++at;
        }
      }
}

// Unit vector from two uniform draws: z = 2u - 1, phi = 2 pi u'.
inline void unit_from(double u, double v, double* out) {
  const double z = 2.0 * u - 1.0;
  const double phi = 2.0 * M_PI * v;
  const double zz = 1.0 - z * z;
  const double r = std::sqrt(zz > 0.0 ? zz : 0.0);
  out[0] = r * std::cos(phi);
  out[1] = r * std::sin(phi);
  out[2] = z;
}

}  // namespace

extern "C" {

const char* h2g_points_last_error(void) { return g_points_err.c_str(); }

int h2g_generate_points(int32_t geometry, int64_t n, uint64_t seed, int64_t spheres, double spacing,
                        double* xyz, double* q) {
  try {
    if (n < 2) throw std::invalid_argument("generate: n must be >= 2");
    for (int64_t i = 0; i < n; ++i) q[i] = 1.0;
    SplitMix64 rng{seed};
    switch (geometry) {
      case H2G_GEOM_CUBE:  // geometry.cpp:42-52: point i = draws 3i..3i+2
        for (int64_t i = 0; i < 3 * n; ++i) xyz[i] = rng.next_double();
        break;
      case H2G_GEOM_LINE:  // geometry.cpp:54-62
        for (int64_t i = 0; i < n; ++i) {
          xyz[3 * i] = rng.next_double();
          xyz[3 * i + 1] = 0.0;
          xyz[3 * i + 2] = 0.0;
        }
        break;
      case H2G_GEOM_SPHERE:
        fib_spheres(n, spheres, spacing, seed, xyz);
        break;
      case H2G_GEOM_UNIFORM_SPHERE:  // BASELINE configs[1] as worded: i.i.d. on the unit sphere
        for (int64_t i = 0; i < n; ++i) {
          const double u = rng.next_double(), v = rng.next_double();
          unit_from(u, v, xyz + 3 * i);
        }
        break;
      case H2G_GEOM_ELLIPSOIDS: {  // BASELINE configs[4]: `spheres` ellipsoids,
        // semi-axes U(0.05, 0.2), centres U[0,1]^3, point i on ellipsoid i % count
        const int64_t count = spheres;
        if (count < 1) throw std::invalid_argument("generate: ellipsoid count must be >= 1");
        double* geo = new double[size_t(6 * count)];
        for (int64_t e = 0; e < 3 * count; ++e) geo[e] = rng.next_double();
        for (int64_t e = 0; e < 3 * count; ++e) geo[3 * count + e] = 0.05 + 0.15 * rng.next_double();
        for (int64_t i = 0; i < n; ++i) {
          const int64_t e = i % count;
          const double u = rng.next_double(), v = rng.next_double();
          double d[3];
          unit_from(u, v, d);
          for (int k = 0; k < 3; ++k) xyz[3 * i + k] = geo[3 * e + k] + geo[3 * count + 3 * e + k] * d[k];
        }
        delete[] geo;
        break;
      }
      default:
        throw std::invalid_argument("generate: unknown geometry " + std::to_string(geometry));
    }
    return 0;
  } catch (const std::exception& e) {
    g_points_err = e.what();
    return 1;
  }
}

}  // extern "C"
