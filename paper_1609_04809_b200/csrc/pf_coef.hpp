// pf_coef.hpp — the counter-based lognormal(0, 1) cell coefficient:
// kappa = exp(z), z by Box-Muller on two 53-bit uniforms in (0, 1] drawn from splitmix64
// keyed by (seed, cell number), so every rank and the device agree without communication.
// Restated in oracle/coef.py.
#pragma once

#include <cmath>
#include <cstdint>

namespace pf {

inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

inline double lognormal_kappa(uint64_t seed, int64_t cell) {
  const uint64_t a = splitmix64(seed ^ splitmix64(static_cast<uint64_t>(cell) * 2 + 1));
  const uint64_t b = splitmix64(a);
  const double u1 = (static_cast<double>(a >> 11) + 1.0) / 9007199254740992.0;
  const double u2 = (static_cast<double>(b >> 11) + 1.0) / 9007199254740992.0;
  const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::acos(-1.0) * u2);
  return std::exp(z);
}

}  // namespace pf
