// Random streams for the two transport modes.
//
// Exact mode replays the reference's streams bit-for-bit: xoshiro256** whose
// 4x64-bit state is seeded by four splitmix64 draws from
// seed + 0x9E3779B97F4A7C15 * stream_id, with stream_id = (purpose << 56) ^
// (step << 40) ^ history and uniform() = ((u >> 11) + 0.5) * 2^-53
// (proj/include/hww/rng.hpp:10-80).
//
// Fast mode uses counter-based Philox4x32-10: every particle owns the stream
// (key = seed ^ step, counter = {lineage lo, lineage hi, draw index, purpose})
// so draws need no state in HBM beyond a 32-bit counter per particle.
#pragma once

#include <stdint.h>

#include "libm_log.h"

namespace hwwg {

enum StreamPurpose : uint64_t { kSource = 0, kFlight = 1, kWindow = 2, kComb = 3 };

HWWG_HD uint64_t stream_id(uint64_t step, uint64_t history, uint64_t purpose) {
  return (purpose << 56) ^ (step << 40) ^ history;
}

HWWG_HD uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

struct Xoshiro {
  uint64_t s0, s1, s2, s3;

  HWWG_HD static uint64_t splitmix(uint64_t& x) {
    x += 0x9E3779B97F4A7C15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }

  HWWG_HD void seed(uint64_t seed_value, uint64_t id) {
    uint64_t x = seed_value + 0x9E3779B97F4A7C15ULL * id;
    s0 = splitmix(x);
    s1 = splitmix(x);
    s2 = splitmix(x);
    s3 = splitmix(x);
    if ((s0 | s1 | s2 | s3) == 0) s0 = 1;
  }

  HWWG_HD uint64_t next() {
    const uint64_t out = rotl64(s1 * 5, 7) * 9;
    const uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = rotl64(s3, 45);
    return out;
  }

  // Uniform deviate strictly inside (0,1); the integer->double conversion and
  // the scaling are exact, so no rounding mode question arises.
  HWWG_HD double uniform() { return ((double)(next() >> 11) + 0.5) * 0x1.0p-53; }
  HWWG_HD double uniform_pm1() { return HWWG_SUB(HWWG_MUL(2.0, uniform()), 1.0); }
};

// ------------------------------------------------------------ Philox4x32-10
struct U4 {
  uint32_t x, y, z, w;
};

HWWG_HD void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#if defined(__CUDA_ARCH__)
  lo = a * b;
  hi = __umulhi(a, b);
#else
  const uint64_t p = (uint64_t)a * (uint64_t)b;
  lo = (uint32_t)p;
  hi = (uint32_t)(p >> 32);
#endif
}

HWWG_HD U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c.x, hi0, lo0);
    mulhilo32(0xCD9E8D57u, c.z, hi1, lo1);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Philox4x32-10 with the round keys precomputed (rk[2r] = k0 + r * 0x9E3779B9,
// rk[2r+1] = k1 + r * 0xBB67AE85: philox_round_keys): the same function as
// philox4x32_10, without the key schedule's adds — with rk in kernel
// parameters every key is a constant-bank operand of its XOR.
HWWG_HD void philox_round_keys(uint32_t k0, uint32_t k1, uint32_t rk[20]) {
  for (int r = 0; r < 10; ++r) {
    rk[2 * r] = k0 + (uint32_t)r * 0x9E3779B9u;
    rk[2 * r + 1] = k1 + (uint32_t)r * 0xBB67AE85u;
  }
}
HWWG_HD U4 philox4x32_10_rk(U4 c, const uint32_t (&rk)[20]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c.x, hi0, lo0);
    mulhilo32(0xCD9E8D57u, c.z, hi1, lo1);
    c = U4{hi1 ^ c.y ^ rk[2 * r], lo1, hi0 ^ c.w ^ rk[2 * r + 1], lo0};
  }
  return c;
}

// Two uniforms in (0,1) from one Philox block (53 bits each).
// One event's deviates from one Philox block: a 53-bit uniform (flight
// distance) and two 32-bit uniforms (collision type / roulette, scattering).
HWWG_HD void philox_uniform3(U4 r, double& a, double& b, double& c) {
  const uint64_t ua = ((uint64_t)r.x << 32 | r.y) >> 11;
  a = ((double)ua + 0.5) * 0x1.0p-53;
  b = ((double)r.z + 0.5) * 0x1.0p-32;
  c = ((double)r.w + 0.5) * 0x1.0p-32;
}

HWWG_HD void philox_uniform2(U4 r, double& a, double& b) {
  const uint64_t ua = ((uint64_t)r.x << 32 | r.y) >> 11;
  const uint64_t ub = ((uint64_t)r.z << 32 | r.w) >> 11;
  a = ((double)ua + 0.5) * 0x1.0p-53;
  b = ((double)ub + 0.5) * 0x1.0p-53;
}

}  // namespace hwwg
