// host_rng.hpp — host-side randomness of the hot path.
//
// Probe vectors, the pathwise RFF base draws and the SGD minibatch index
// stream stay on the host so their values are bitwise those of the
// reference's mt19937_64 streams (SURVEY K8 / §7 "SGD RNG parity").
#pragma once

#include <stdint.h>

#include <cmath>
#include <limits>
#include <random>
#include <stdexcept>
#include <vector>

namespace wgp {

// proj/include/warmgp/common.hpp:25-30
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// common.hpp:34-36
inline uint64_t derive_seed(uint64_t base, uint64_t stream) {
  return splitmix64(splitmix64(base) ^ splitmix64(stream + 0x51ed2701ab0a3c11ULL));
}
// common.hpp:40-47
inline uint64_t uniform_below(std::mt19937_64& rng, uint64_t bound) {
  const uint64_t limit =
      std::numeric_limits<uint64_t>::max() - std::numeric_limits<uint64_t>::max() % bound;
  uint64_t v;
  do {
    v = rng();
  } while (v >= limit);
  return v % bound;
}
// common.hpp:50-52
inline double uniform_unit(std::mt19937_64& rng) {
  return static_cast<double>(rng() >> 11) * 0x1.0p-53;
}

// proj/src/estimator.cpp:21-37 (column-major fill), written to `out` with
// leading dimension ld.
template <class T>
void sample_probes_host(int64_t n, int s, int dist, uint64_t seed, T* out, int64_t ld) {
  if (n < 1 || s < 1) throw std::invalid_argument("sample_probes: n and s must be >= 1");
  std::mt19937_64 rng(seed);
  if (dist == 0) {
    std::normal_distribution<double> normal(0.0, 1.0);
    for (int j = 0; j < s; ++j)
      for (int64_t i = 0; i < n; ++i) out[i + j * ld] = static_cast<T>(normal(rng));
  } else {
    for (int j = 0; j < s; ++j)
      for (int64_t i = 0; i < n; ++i) out[i + j * ld] = static_cast<T>((rng() & 1u) ? 1.0 : -1.0);
  }
}

// Pathwise-probe base randomness (BASELINE a12), draw order: omega_z (F x d,
// f-major), chi2_3 (F, three squared normals each), phase b = 2 pi U[0,1) (F),
// w (F x s column-major), eps (n x s column-major, leading dim ld).
struct RffBase {
  int F = 0, d = 0, s = 0;
  std::vector<double> omega_z, chi2, b, w;
  std::vector<float> eps;  // ld x s
};

inline RffBase rff_base_host(int64_t n, int d, int F, int s, uint64_t seed, int64_t ld) {
  if (n < 1 || d < 1 || F < 1 || s < 1) throw std::invalid_argument("rff_base: bad sizes");
  RffBase r;
  r.F = F;
  r.d = d;
  r.s = s;
  r.omega_z.resize(static_cast<size_t>(F) * d);
  r.chi2.resize(F);
  r.b.resize(F);
  r.w.resize(static_cast<size_t>(F) * s);
  r.eps.assign(static_cast<size_t>(ld) * s, 0.f);
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> normal(0.0, 1.0);
  for (int f = 0; f < F; ++f)
    for (int k = 0; k < d; ++k) r.omega_z[static_cast<size_t>(f) * d + k] = normal(rng);
  for (int f = 0; f < F; ++f) {
    double acc = 0.0;
    for (int q = 0; q < 3; ++q) {
      const double z = normal(rng);
      acc += z * z;
    }
    r.chi2[f] = acc;
  }
  for (int f = 0; f < F; ++f) r.b[f] = 2.0 * M_PI * uniform_unit(rng);
  for (int j = 0; j < s; ++j)
    for (int f = 0; f < F; ++f) r.w[static_cast<size_t>(j) * F + f] = normal(rng);
  for (int j = 0; j < s; ++j)
    for (int64_t i = 0; i < n; ++i) r.eps[i + j * ld] = static_cast<float>(normal(rng));
  return r;
}

}  // namespace wgp
