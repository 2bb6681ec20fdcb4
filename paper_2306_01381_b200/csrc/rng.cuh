// rng.cuh — the reference's counter-based generator (quantcodec/rng.hpp:13-61)
// as host/device functions.  A draw is a pure function of (key, counter), so
// every element of every message is an independent lane of work on the GPU.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define QGNN_HD __host__ __device__ __forceinline__
#else
#define QGNN_HD inline
#endif

namespace qgnn_b200 {

constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ull;

// rng.hpp:52-57
QGNN_HD uint64_t rng_mix(uint64_t z) {
  z += kPhi;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// rng.hpp:15
QGNN_HD uint64_t rng_seed_key(uint64_t seed) { return rng_mix(seed ^ 0x6a09e667f3bcc909ull); }
// rng.hpp:17-22
QGNN_HD uint64_t rng_fork(uint64_t key, uint64_t coord) { return rng_mix(key ^ rng_mix(coord + kPhi)); }
// rng.hpp:30 (counter already incremented)
QGNN_HD uint64_t rng_u64(uint64_t key, uint64_t ctr) { return rng_mix(key + ctr * kPhi); }
// rng.hpp:33 — the 53-bit integer behind next_double(): u = (r >> 11) * 2^-53
QGNN_HD uint64_t rng_u53(uint64_t key, uint64_t ctr) { return rng_u64(key, ctr) >> 11; }

// rng.hpp:36-41 (host side; counter advanced in place)
inline uint64_t rng_next_below(uint64_t key, uint64_t& ctr, uint64_t n) {
  const uint64_t limit = ~uint64_t{0} - ~uint64_t{0} % n;
  uint64_t x = rng_u64(key, ++ctr);
  while (x >= limit) x = rng_u64(key, ++ctr);
  return x % n;
}

}  // namespace qgnn_b200
