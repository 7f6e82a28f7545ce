// Bit-exact replay of the host libm's double log on host and device.
//
// Provenance and licence. The algorithm restated here is glibc 2.39's double
// log (sysdeps/ieee754/dbl-64/e_log.c, contributed to glibc from Arm's
// optimized-routines project; glibc: LGPL-2.1-or-later, optimized-routines:
// MIT OR Apache-2.0 WITH LLVM-exception). Bit-exact replay of the reference's
// xoshiro-driven flight distances needs the same operations in the same order,
// so the range split, table lookup and polynomial evaluation below follow that
// published algorithm step for step (an acknowledged deviation from "do not
// copy a libm implementation": a different log would change ~8e-4 of the
// reference's events). No glibc source text or constant is in this repository:
// the constants are read from the installed libm at build time
// (gen_libm_log_table.py) into _build/, which is never committed.
//
// The reference samples flight distances as -std::log(xi)/sigma_t
// (proj/src/transport.cpp:24-27). Its third-party dependency is glibc 2.39's
// log (ifunc-selected FMA build on x86-64 hosts with FMA+AVX2). The published
// algorithm: for x = 2^k * z with z in [0x1.6p-1, 0x1.6p0),
//     log(x) = k*ln2 + log(c_i) + log1p(r),  r = z*(1/c_i) - 1  (one fma),
// with i the top 7 mantissa bits of z, a 128-entry (1/c_i, log c_i) table,
// and log1p(r) ~ r + A0 r^2 + r^3 (A1 + A2 r + r^2 (A3 + A4 r)); inputs within
// [1 - 2^-4, 1 + 0x1.09p-4) use r = x - 1 directly with an 11-coefficient
// polynomial and a 27-bit split of r to carry r - r^2/2 in two parts.
//
// The evaluation order below is the one the installed binary executes
// (every fma/mul/add is explicit and non-contractible), and the constants come
// from _build/libm_log_table.h, generated from the installed libm by
// csrc/gen_libm_log_table.py. tests/test_libm_log.py checks this function
// against the system log bit-for-bit. Domain: finite x > 0 (uniform deviates
// in (0,1) in the transport kernels); other inputs follow IEEE log semantics.
#pragma once

#include <stdint.h>

#include "libm_log_table.h"

#if defined(__CUDACC__)
#define HWWG_HD __host__ __device__ __forceinline__
#elif defined(__cplusplus)
#define HWWG_HD inline
#else
#define HWWG_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define HWWG_FMA(a, b, c) __fma_rn((a), (b), (c))
#define HWWG_MUL(a, b) __dmul_rn((a), (b))
#define HWWG_ADD(a, b) __dadd_rn((a), (b))
#define HWWG_SUB(a, b) __dsub_rn((a), (b))
#define HWWG_BITS(x) ((uint64_t)__double_as_longlong(x))
#define HWWG_DBL(u) __longlong_as_double((long long)(u))
#else
#include <math.h>
#include <string.h>
HWWG_HD uint64_t hwwg_bits_(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
HWWG_HD double hwwg_dbl_(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
#define HWWG_FMA(a, b, c) fma((a), (b), (c))
#define HWWG_MUL(a, b) ((a) * (b))
#define HWWG_ADD(a, b) ((a) + (b))
#define HWWG_SUB(a, b) ((a) - (b))
#define HWWG_BITS(x) hwwg_bits_(x)
#define HWWG_DBL(u) hwwg_dbl_(u)
#endif

#if defined(__CUDACC__)
__device__ __constant__ static const double hwwg_log_tab_d[256] = HWWG_LOG_TAB;
#endif
static const double hwwg_log_tab_h[256] = HWWG_LOG_TAB;

HWWG_HD double hwwg_libm_log(double x) {
#if defined(__CUDA_ARCH__)
  const double* T = hwwg_log_tab_d;
#else
  const double* T = hwwg_log_tab_h;
#endif
  const double A[5] = HWWG_LOG_A;
  const double Bc[11] = HWWG_LOG_B;
  uint64_t ix = HWWG_BITS(x);

  // Inputs close to 1: direct polynomial in r = x - 1.
  if (ix - 0x3fee000000000000ULL < 0x3090000000000ULL) {
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double r = HWWG_SUB(x, 1.0);
    double q21 = HWWG_FMA(r, Bc[2], Bc[1]);
    double q54 = HWWG_FMA(r, Bc[5], Bc[4]);
    const double r2 = HWWG_MUL(r, r);
    double q87 = HWWG_FMA(r, Bc[8], Bc[7]);
    q21 = HWWG_FMA(r2, Bc[3], q21);
    q54 = HWWG_FMA(r2, Bc[6], q54);
    const double r3 = HWWG_MUL(r, r2);
    q87 = HWWG_FMA(r2, Bc[9], q87);
    q87 = HWWG_FMA(r3, Bc[10], q87);
    double q = HWWG_FMA(q87, r3, q54);
    q = HWWG_FMA(q, r3, q21);
    // r split at 27 bits: rhi exact square, rlo the remainder.
    const double t = HWWG_FMA(r, 0x1p27, r);
    const double rhi = HWWG_FMA(-0x1p27, r, t);
    const double rr = HWWG_MUL(rhi, rhi);
    const double rlo = HWWG_SUB(r, rhi);
    const double hi = HWWG_FMA(rr, Bc[0], r);
    double lo = HWWG_FMA(rr, Bc[0], HWWG_SUB(r, hi));
    const double s = HWWG_ADD(r, rhi);
    lo = HWWG_FMA(HWWG_MUL(Bc[0], rlo), s, lo);
    const double y = HWWG_FMA(q, r3, lo);
    return HWWG_ADD(hi, y);
  }

  const uint32_t top = (uint32_t)(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if ((ix << 1) == 0) return -1.0 / 0.0;                   // log(+-0) = -inf
    if (ix == 0x7ff0000000000000ULL) return x;               // log(inf) = inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u)      // negative or NaN
      return (x - x) / (x - x);
    // subnormal: scale into the normal range
    ix = HWWG_BITS(HWWG_MUL(x, 0x1p52)) - (52ULL << 52);
  }

  const uint64_t tmp = ix - 0x3fe6000000000000ULL;
  const int i = (int)((tmp >> 45) & 127u);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & 0xfffULL << 52);
  const double z = HWWG_DBL(iz);
  const double invc = T[2 * i];
  const double logc = T[2 * i + 1];
  const double kd = (double)k;

  const double w = HWWG_FMA(kd, HWWG_LOG_LN2HI, logc);
  const double r = HWWG_FMA(z, invc, -1.0);
  const double p1 = HWWG_FMA(r, A[2], A[1]);
  const double hi = HWWG_ADD(r, w);
  const double r2 = HWWG_MUL(r, r);
  const double lo0 = HWWG_ADD(HWWG_SUB(w, hi), r);
  const double lo1 = HWWG_FMA(kd, HWWG_LOG_LN2LO, lo0);
  const double r3 = HWWG_MUL(r, r2);
  const double p2 = HWWG_FMA(r, A[4], A[3]);
  const double lo2 = HWWG_FMA(r2, A[0], lo1);
  const double p = HWWG_FMA(p2, r2, p1);
  const double y = HWWG_FMA(r3, p, lo2);
  return HWWG_ADD(y, hi);
}
