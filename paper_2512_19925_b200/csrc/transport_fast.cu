// Throughput (Philox) mode: event-driven particle transport on sm_100a.
//
// The reference's per-history xoshiro streams force history-serial order; this
// mode instead gives every particle its own counter-based Philox4x32-10
// stream (counter = {history, lineage key lo, lineage key hi, step<<16 | draw},
// key = seed), so any particle can advance independently and the result is a
// statistically equivalent estimator of the same physics (SURVEY.md §7 hard
// part 1; parity = combined standard errors, tests/test_gpu_statistical.py).
// One Philox block per event: flight, collision channel and scattering
// deviates (the roulette deviate after a scatter is the channel one recycled).
//
// Work model — a persistent grid (2 CTAs of 14 warps per SM, or one 24-warp
// CTA for large tally copies), one particle per
// lane, one EVENT per loop trip (free flight -> census | cell crossing |
// collision), with refill: a lane whose particle terminated takes the next
// unit of work from
//   1. its warp's run-length-encoded split stack (LIFO, like the reference;
//      the bottom kSmemStack records in shared memory),
//   2. the source bank, through a per-warp reservation of kClaim particles
//      claimed one trip ahead (first one static) and prefetched into L1; comb
//      teeth are (x, mu) only (FastArgs::n_packed) and get their weight, time,
//      cell and identity here,
//   3. the global pool of split records other warps donated (ticket queue).
// A split never materialises its daughters: it pushes ONE record (state, n-1
// copies) and lanes pop daughters from it — the bank-expansion step done by
// ballot + prefix-popcount inside the warp. Backlogs are shared with idle
// warps (halves of a long run or whole records, up to one per idle warp per
// trip), so the heavy cold-start split trees (config 2 step 1: p99 1108
// segments per history) spread over the whole GPU instead of pinning one warp.
// Roulette and unchanged windows cost no memory traffic.
//
// Tallies: block-private shared-memory histograms over the segment's batch
// range (track-length by batch and cell, census phi/J/F, census weight by
// batch, edge currents, per-cell track counts), flushed once per block with
// fp64 REDs. Where the wider slots fit, these scores are fixed-point integers
// added as 16-bit limbs with native 32-bit shared atomics, kept from wrapping
// by a rolling carry sweep (see fix_add / fix_sweep); in the cold start the
// census scores of identical split copies are grouped by an exact MATCH on
// (cell, w, mu) first (census_groups). Otherwise fp64 slots (CAS loops) with
// census scores run-aggregated across the warp, and global REDs
// warp-aggregated (MATCH.ANY groups, REDUX fixed-point sums) when the
// histograms do not fit in shared memory (I = 4000).
//
// Census thinning (FastArgs::precomb, the cold start): every lane combs the
// census particles it banks at the spacing s0 and banks each once with its
// teeth' weight n s0 (or not at all), so the x60 raw census never
// materialises; the comb at the next step start combs the ~8 x target records.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "fast.cuh"
#include "libm_log_table.h"
#include "rng.cuh"

namespace hwwg {

namespace {

// Block shapes (warps per SM at <= 72 registers): 2 blocks of 14 warps (28),
// 2 of 12 (24), or 1 block of 24 warps when the block's shared-memory tallies
// fit only once per SM or reach 96 KB (config 3's 1000 cells). One
// shared-memory tally set per block; the driver picks the shape per launch
// (C5: 2 x 14 2.54e10 seg/s against 2 x 12 2.43e10; C3: 1 x 24 2.0e10
// against 2 x 14 1.5e10).
constexpr int kMaxWarpsPerSm = 28;

// -DHWWG_FAST_PROF: per-phase clock64 accounting of the loop (lane 0 of every
// warp), summed over the grid into g_fprof: [0] refill [1] event [2] census
// [3] tally [4] split [5] trips [6] idle cycles (waiting on the pool)
// [7] warp lifetime cycles
#ifdef HWWG_FAST_PROF
__device__ unsigned long long g_fprof[12];
// trips and live lanes per 5 us bin since the segment's reset, per segment (<= 8)
constexpr int kHistBins = 120;
__device__ unsigned int g_fhist[8][kHistBins][2];
#define FPROF_DECL                                                                   \
  unsigned long long fp_t = clock64(), fp_c[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, fp_trip = 0, \
                     fp_k0 = fp_t;
#define FPROF(k)                          \
  do {                                    \
    const unsigned long long t_ = clock64(); \
    fp_c[k] += t_ - fp_t;                 \
    fp_t = t_;                            \
  } while (0)
#else
#define FPROF_DECL
#define FPROF(k) \
  do {           \
  } while (0)
#endif
#ifndef HWWG_KDONATE
#define HWWG_KDONATE 256
#endif
#ifndef HWWG_KSHARE
#define HWWG_KSHARE 64
#endif
#ifndef HWWG_BACKOFF
#define HWWG_BACKOFF 2048
#endif
constexpr unsigned kDonate = HWWG_KDONATE;  // pending local daughters above which splits go global
constexpr unsigned kCensusChunk = 64;  // census slots a warp reserves at a time
#ifndef HWWG_KCLAIM
#define HWWG_KCLAIM 32
#endif
constexpr unsigned kClaim = HWWG_KCLAIM;  // source particles a warp reserves per claim
#ifndef HWWG_KCLAIM_TAIL
#define HWWG_KCLAIM_TAIL 4
#endif
constexpr unsigned kClaimTail = HWWG_KCLAIM_TAIL;  // claim size near the end of the source
// (measured on config 2: 32 static + 4 in the last 2 claims per warp, 8.0e9 ->
// 8.3e9 seg/s against uniform 16-particle claims)
#ifndef HWWG_CLAIM_ZONE
#define HWWG_CLAIM_ZONE 2  // the tail zone, in kClaim-particle claims per warp
#endif
constexpr unsigned kShare = HWWG_KSHARE;
#ifndef HWWG_POLL_EVERY
#define HWWG_POLL_EVERY 4
#endif
constexpr unsigned kPollEvery = HWWG_POLL_EVERY;  // trips between looks at the pool counters
#ifndef HWWG_SMEM_STACK
#define HWWG_SMEM_STACK 24  // measured: 8 -> 16 is +2% on config 2, 16 -> 24 +0.7% on config 5 (split stacks stay on chip)
#endif
// split-stack records per warp kept in shared memory: HWWG_SMEM_STACK for the
// 12/14-warp blocks, 16 for the 24-warp block, whose shared memory goes to a
// large tally copy (config 3: 16 is 1.3% faster than 24; config 5 at 2 x 14
// warps: 24 is 0.7% faster than 16)
template <int kW>
__host__ __device__ constexpr int smem_stack() { return kW >= 24 ? 16 : HWWG_SMEM_STACK; }
#ifndef HWWG_KPIECE
#define HWWG_KPIECE 32
#endif
constexpr unsigned kPiece = HWWG_KPIECE;  // smallest run piece handed to an idle warp

// A daughter's lineage key (the Philox counter's middle words): a bijective
// one-multiply mix of (parent key, parent draw counter, daughter index) — the
// keys only need to stay distinct within a history (Philox does the mixing),
// and the cold start draws ~6e8 of them.
__device__ __forceinline__ unsigned long long mix_lineage(unsigned long long z) {
  z *= 0x9E3779B97F4A7C15ULL;
  return z ^ (z >> 32);
}

struct Lane {
  double x, mu, w, t, inv_mu;
  int cell;
  int bslot;  // tally batch slot (batch, or batch - b_lo for shared-memory tallies)
  unsigned hist, ctr;
  unsigned long long key;
  bool alive;
  bool fis;  // a fission secondary whose direction and window game are pending
};

// split records with this bit in `ctr` hold fission secondaries (each draws its
// own direction and plays the window game when popped), not identical copies
constexpr unsigned kFissionRec = 0x80000000u;

// One Philox4x32-10 block per event: flight, collision type and scattering
// deviates (the roulette deviate after a scatter is the collision-type one
// recycled: given u1 < sigma_s/sigma_t, u1 * sigma_t / sigma_s is uniform and
// independent of that decision).
__device__ __forceinline__ void draw3(const FastArgs& a, Lane& p, double& u0, double& u1,
                                      double& u2) {
  const U4 c{p.hist, (unsigned)p.key, (unsigned)(p.key >> 32), (a.step << 16) | (p.ctr & 0xffffu)};
  ++p.ctr;
  philox_uniform3(philox4x32_10_rk(c, a.rk), u0, u1, u2);
}

// tally.hpp:130-134 batch_of = floor(h B / H): an fp64 estimate from the
// precomputed B / H, corrected by one integer comparison (the estimate is off
// by at most one; no division)
__device__ __forceinline__ int batch_fast(unsigned h, unsigned long long H, int B, double bmul) {
  int b = (int)((double)h * bmul);
  if (H * (unsigned)B < (1ULL << 32)) {  // every product below fits 32 bits (h < H, b < B)
    const unsigned hb = h * (unsigned)B, H32 = (unsigned)H;
    if ((unsigned)(b + 1) * H32 <= hb) ++b;
    else if (b > 0 && (unsigned)b * H32 > hb) --b;
    return b < B ? b : B - 1;
  }
  const unsigned long long hb = (unsigned long long)h * (unsigned)B;
  if ((unsigned long long)(b + 1) * H <= hb) ++b;
  else if (b > 0 && (unsigned long long)b * H > hb) --b;
  return b < B ? b : B - 1;
}

__constant__ double c_logtab[256] = HWWG_LOG_TAB;

// mesh.cpp:26-40 for a comb tooth's x: the uniform estimate by a multiplication
// (any estimate within one cell becomes the unique c with edges[c] <= x <
// edges[c+1] under the +-1 guards), else a binary search over the edges in
// shared memory; -1 outside the mesh
__device__ __forceinline__ int locate_cell_mul(const MeshView& m, double x, double inv_w0,
                                               const double* e) {
  if (x < m.x_min || x > m.x_max) return -1;
  if (x == m.x_max) return m.I - 1;
  if (m.uniform) {
    int c = (int)((x - m.x_min) * inv_w0);
    c = c < 0 ? 0 : (c >= m.I ? m.I - 1 : c);
    if (x < e[c]) --c;
    else if (x >= e[c + 1]) ++c;
    return c;
  }
  int lo = 0, hi = m.I + 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (e[mid] > x) hi = mid;
    else lo = mid + 1;
  }
  return lo - 1;
}

// 1 / x to within an ulp: the MUFU reciprocal estimate and two Newton steps
// (the IEEE division's 1 / mu cost a slow-path check per direction change);
// x = 0 keeps the IEEE answer (+-inf)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  // (no division in the select: it would be computed on every call)
  const long long inf = 0x7ff0000000000000LL | (__double_as_longlong(x) & (long long)0x8000000000000000ULL);
  return x == 0.0 ? __longlong_as_double(inf) : r;
}

// -ln(u) for a deviate u in (0, 1) (the flight distance in mean free paths):
// the table-driven algorithm of libm_log.h (k ln2 + log c + log1p(r), 128-entry
// (1/c, log c) table from the installed libm, degree-6 polynomial) with the
// table in shared memory and no special-case paths (u is normal and below 1).
// Near u = 1 the near-1 branch the exact replay keeps is dropped: the absolute
// error stays ~1e-17 (a distance of 1e-17 mean free paths), which no estimator
// can see; the exact mode keeps the bit-exact replay.
__device__ __forceinline__ double neg_log_unit(double u, const double* __restrict__ T) {
  const double A[5] = HWWG_LOG_A;
  const unsigned long long ix = (unsigned long long)__double_as_longlong(u);
  const unsigned long long tmp = ix - 0x3fe6000000000000ULL;
  const int i = (int)((tmp >> 45) & 127u);
  const int k = (int)((long long)tmp >> 52);
  const double z = __longlong_as_double((long long)(ix - (tmp & (0xfffULL << 52))));
  const double invc = T[2 * i], logc = T[2 * i + 1];
  const double kd = (double)k;
  const double w = fma(kd, HWWG_LOG_LN2HI, logc);
  const double r = fma(z, invc, -1.0);
  const double r2 = r * r;
  const double p = fma(fma(r, A[4], A[3]), r2, fma(r, A[2], A[1]));
  const double lo = fma(r2, A[0], fma(kd, HWWG_LOG_LN2LO, (w - (r + w)) + r));
  return -((r + w) + fma(r2 * r, p, lo));
}

// split records carry the parent's cell | batch slot << 16 (daughters keep the
// history's batch: no per-daughter batch division)
__device__ __forceinline__ void load_rec(Lane& p, const FastStackRec& r, unsigned j) {
  p.x = r.x;
  p.mu = r.mu;
  p.w = r.w;
  p.t = r.t;
  p.cell = (int)(r.cell & 0xffffu);
  p.bslot = (int)(r.cell >> 16);
  p.hist = r.hist;
  p.key = mix_lineage(r.key ^ ((unsigned long long)r.ctr << 40) ^ ((unsigned long long)j << 8) ^
                0x5bd1e995ULL);
  p.ctr = 0;
  p.inv_mu = r.inv_mu;
  p.alive = true;
  p.fis = (r.ctr & kFissionRec) != 0;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Warp-aggregated atomic add: lanes with the same key (MATCH.ANY) are summed,
// then the group's lowest lane issues ONE atomic. key < 0: no contribution.
// Must be called by all 32 lanes. In the cold-start steps most of a warp sits
// in a few cells around the pulse, where per-lane fp64 CAS loops on shared
// memory serialise.
__device__ __forceinline__ unsigned agg_group(int key) {
  const int lane = threadIdx.x & 31;
  return __match_any_sync(0xffffffffu, key >= 0 ? key : -1 - lane);
}

// Sum of v over the lanes of `grp` (a MATCH.ANY group holding this lane) with
// three integer REDUX ops, whatever the group size: every value is put on the
// fixed-point grid 2^-56 below the group's largest magnitude (finer than the
// fp64 rounding of any sum that includes that value) and the 64-bit integer
// sum is exact; one rounding back to fp64. Non-finite groups take shuffles.
__device__ __forceinline__ double group_sum(unsigned grp, double v) {
  const unsigned e = ((unsigned)__double2hiint(v) >> 20) & 0x7ffu;
  const unsigned emax = __reduce_max_sync(grp, e);
  if (emax == 0x7ffu) {  // inf/nan somewhere in the group
    double t = 0.0;
    for (unsigned m = grp; m; m &= m - 1) t += __shfl_sync(grp, v, __ffs(m) - 1);
    return t;
  }
  if (emax < 64u) return 0.0;  // every |v| < 2^-959
  const int sh = 56 - ((int)emax - 1023);  // |v * 2^sh| < 2^57: 32 lanes sum below 2^62
  const long long q = __double2ll_rn(v * __hiloint2double((sh + 1023) << 20, 0));
  const unsigned lo = (unsigned)q & 0x1fffffu;
  const unsigned mid = (unsigned)(q >> 21) & 0x1fffffu;
  const int hi = (int)(q >> 42);
  const unsigned slo = __reduce_add_sync(grp, lo);
  const unsigned smid = __reduce_add_sync(grp, mid);
  const int shi = __reduce_add_sync(grp, hi);
  const long long tot = ((long long)shi << 42) + ((long long)smid << 21) + (long long)slo;
  return (double)tot * __hiloint2double((1023 - sh) << 20, 0);
}

__device__ __forceinline__ bool group_leader(unsigned grp) {
  return (int)(threadIdx.x & 31) == __ffs(grp) - 1;
}

// (lanes without a contribution are singleton groups and must stay out of the
// REDUX ops: sync reductions run once per distinct member mask)
__device__ __forceinline__ void agg_add(double* base, int key, double v) {
  if (!__any_sync(0xffffffffu, key >= 0)) return;
  const unsigned grp = agg_group(key);
  if (key >= 0) {
    const double s = group_sum(grp, v);
    if (group_leader(grp)) atomicAdd(base + key, s);
  }
}

__device__ __forceinline__ void agg_add3(double* b0, double* b1, double* b2, int key, double v0,
                                         double v1, double v2) {
  if (!__any_sync(0xffffffffu, key >= 0)) return;
  const unsigned grp = agg_group(key);
  if (key >= 0) {
    const double s0 = group_sum(grp, v0);
    const double s1 = group_sum(grp, v1);
    const double s2 = group_sum(grp, v2);
    if (group_leader(grp)) {
      atomicAdd(b0 + key, s0);
      atomicAdd(b1 + key, s1);
      atomicAdd(b2 + key, s2);
    }
  }
}

// The census weight by batch (tally.hpp:65-72 census_weight_batch) of one
// trip: runs of census lanes keyed by the batch slot alone — usually one run
// per warp (all its census lanes hold histories of one batch), which takes a
// plain butterfly sum and one add.
template <class AddW>
__device__ __forceinline__ void census_weight_runs_t(AddW add_w, bool c, int b, double v) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned cm = __ballot_sync(full, c);
  if (!cm) return;
  const int b0 = __shfl_sync(full, b, __ffs(cm) - 1);
  if (!__any_sync(full, c && b != b0)) {
    double w = c ? v : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(full, w, o);
    if (lane == __ffs(cm) - 1) add_w(b0, w);
    return;
  }
  const unsigned below = cm & ((1u << lane) - 1u);
  const int prev = below ? 31 - __clz(below) : lane;
  const unsigned upto = (2u << lane) - 1u;
  const int pb = __shfl_sync(full, b, prev);
  const bool hb_head = c && (prev == lane || pb != b);
  const unsigned bheads = __ballot_sync(full, hb_head);
  const unsigned bhb = bheads & upto;
  const int bstart = bhb ? 31 - __clz(bhb) : 0;
  double w = c ? v : 0.0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(full, w, o);
    if (lane - o >= bstart) w += t;
  }
  const unsigned above = cm & ~upto;
  const int next = above ? __ffs(above) - 1 : -1;
  if (c && (next < 0 || ((bheads >> next) & 1u))) add_w(b, w);
}
__device__ __forceinline__ void census_weight_runs(double* cwb, bool c, int b, double v) {
  census_weight_runs_t([&](int bb, double w) { atomicAdd(cwb + bb, w); }, c, b, v);
}

// Census scores of one trip, summed over runs of census lanes with equal
// (batch slot, cell) in lane order, then one set of adds per run. Split copies
// that reach census without colliding are identical and were handed to
// adjacent lanes, and every census lane of a warp usually shares the batch
// slot, so per-lane CAS loops on these addresses serialise (measured: about
// half of the steady-state transport time). A segmented Hillis-Steele scan
// over the warp (non-census lanes carry zeros) costs a fixed 5 steps.
// AddCell(cell, s0, s1, s2): the run's phi/J/F adds (fp64 or fixed-point slots)
template <class AddCell>
__device__ __forceinline__ void census_runs(AddCell add_cell, double* cwb, int cell, int b,
                                            double v0, double v1, double v2, double v3) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const bool c = cell >= 0;
  const unsigned cm = __ballot_sync(full, c);
  if (!cm) return;
  const int key = c ? (b << 16) | cell : -1;  // cell < 2^16 in this mode
  const unsigned below = cm & ((1u << lane) - 1u);
  const int prev = below ? 31 - __clz(below) : lane;
  const int pkey = __shfl_sync(full, key, prev);
  const bool head = c && (prev == lane || pkey != key);
  const unsigned heads = __ballot_sync(full, head);
  const unsigned upto = (2u << lane) - 1u;  // lanes 0..lane (all 32 for lane 31)
  const unsigned hb = heads & upto;
  const int start = hb ? 31 - __clz(hb) : 0;
  double s0 = c ? v0 : 0.0, s1 = c ? v1 : 0.0, s2 = c ? v2 : 0.0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t0 = __shfl_up_sync(full, s0, o);
    const double t1 = __shfl_up_sync(full, s1, o);
    const double t2 = __shfl_up_sync(full, s2, o);
    if (lane - o >= start) {
      s0 += t0;
      s1 += t1;
      s2 += t2;
    }
  }
  const unsigned above = cm & ~upto;  // census lanes after this one
  const int next = above ? __ffs(above) - 1 : -1;
  if (c && (next < 0 || ((heads >> next) & 1u))) add_cell(cell, s0, s1, s2);  // last lane of its run
  census_weight_runs(cwb, c, b, v3);
}

// Census scores of one trip on fixed-point slots, grouped by exact equality:
// split copies popped from one record carry the same (w, mu), and those that
// reach census in one cell (and batch slot) score identical phi/J/F. Three
// MATCH.ANY ops (cell|batch, then w and mu bit patterns) give each lane the
// lanes whose scores equal its own; the group's lowest lane adds n times the
// score (one rounding onto the fixed-point grid, as a single add), so identical
// copies cost one set of slot adds and no scan. Lanes with equal cells but
// other (w, mu) form their own groups (their per-lane adds conflict rarely).
template <class AddCell, class AddW>
__device__ __forceinline__ void census_groups(AddCell add_cell, AddW add_w, int cell, int b,
                                              double w, double mu, double v0, double v1,
                                              double v2) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const bool c = cell >= 0;
  if (!__any_sync(full, c)) return;
  unsigned g = __match_any_sync(full, c ? (b << 16) | cell : -1 - lane);
  g &= __match_any_sync(full, (unsigned long long)__double_as_longlong(w));
  g &= __match_any_sync(full, (unsigned long long)__double_as_longlong(mu));
  if (c && lane == __ffs(g) - 1) {
    const double n = (double)__popc(g);
    add_cell(cell, n * v0, n * v1, n * v2);
  }
  // (run-aggregated: in the cold start every census lane of a warp adds to one
  // batch slot — per-lane limb adds cost C5's step 1 27 -> 31 ms)
  census_weight_runs_t(add_w, c, b, w);
}

// track-length score (keyed by batch slot and cell) plus the per-cell count
template <class Count>
__device__ __forceinline__ void agg_add_count_t(double* base, Count* cnt, int key, double v,
                                                int cell) {
  if (!__any_sync(0xffffffffu, key >= 0)) return;
  const unsigned grp = agg_group(key);
  if (key >= 0) {
    const double s = group_sum(grp, v);
    if (group_leader(grp)) {
      atomicAdd(base + key, s);
      atomicAdd(cnt + cell, (Count)__popc(grp));
    }
  }
}
__device__ __forceinline__ void agg_add_count(double* base, unsigned* cnt, int key, double v,
                                              int cell) {
  agg_add_count_t<unsigned>(base, cnt, key, v, cell);
}
__device__ __forceinline__ void agg_add_count_global(double* base, unsigned long long* cnt,
                                                     int key, double v, int cell) {
  agg_add_count_t<unsigned long long>(base, cnt, key, v, cell);
}

// Fixed-point track, edge and census phi/J/F tallies (kFix). Shared-memory fp64
// adds are CAS loops on sm_100 (ATOMS.CAST.SPIN.64: load, add, compare-and-swap,
// retry) and sat on every event's dependency chain; 32-bit integer ATOMS.ADD is
// native and needs no reply. A score v is put on the launch's grid 2^-k (k
// chosen on the host so the largest expected score is ~2^40 grid units: see
// fast_fix_exponent) as a 64-bit integer q and added as four 16-bit limbs into
// the four 32-bit words of its slot: independent, fire-and-forget adds. A limb
// word would wrap after 2^16 adds; instead of capping the adds, every warp
// sweeps the next 32 slots of a block-shared cursor every 8 loop trips and
// moves each low word's carry (its high half) into the next word with two
// atomics (fix_sweep: the slot's value is unchanged, concurrent adds are not
// lost). Each sweep takes ceil(slots / 4096) slots per lane, so a slot is
// swept at least once per 8 x 4096 / 32 = 1024 warp trips of the block, i.e.
// before 2^15 lane adds: a word stays below 2^16 + 2^15 x 2^16 < 2^32. A score beyond 2^62 grid units (and NaN)
// goes to the global tally with a native fp64 RED. The flush recombines the
// limbs exactly into one fp64 value per slot (three roundings), so a tally
// carries the fp64 sum of the quantised scores: 2^-40 of the expected largest
// score, ~1e-12 relative.
constexpr unsigned kSweepEvery = 8;  // warp loop trips between carry sweeps

__device__ __forceinline__ double pow2(int k) {  // 2^k, |k| <= 1022
  return __hiloint2double((k + 1023) << 20, 0);
}

__device__ __forceinline__ bool fix_add(double* slot, double v, double scale) {
  const double sv = v * scale;
  if (!(fabs(sv) < 0x1p62)) return false;  // also NaN
  const long long q = __double2ll_rn(sv);
  unsigned* w = reinterpret_cast<unsigned*>(slot);
  atomicAdd(w + 0, (unsigned)q & 0xffffu);
  atomicAdd(w + 1, (unsigned)(q >> 16) & 0xffffu);
  atomicAdd(w + 2, (unsigned)(q >> 32) & 0xffffu);
  // the signed top limb (two's complement) only where it is not zero: scores
  // are sized to ~2^40 grid units, so for the non-negative ones (track lengths,
  // census phi and weights) the whole warp skips this add. One shared atomic
  // and its conflict passes less per score: C5 +3.2% (cold start 26.9 ->
  // 25.2 ms), C4 +4%. Skipping zero middle limbs as well did not pay: ptxas
  // turns each test into a divergent BSSY/BRA/BSYNC region (predicated
  // red.shared too), which costs C3 2-3% and the steady steps gain nothing.
  const unsigned top = (unsigned)(q >> 48);
  if (top) atomicAdd(w + 3, top);
  return true;
}

// Carry of one slot's low words into the next word (slot: 4 limb words). The
// carry is taken with one atomic AND that clears the word's high half and
// returns what it held, so two warps sweeping the same slot at once (a narrow
// tally window cycles its cursor through few slots) move each carry exactly
// once: a read-then-subtract let both subtract the same carry and wrap the low
// word below zero. Adds racing with the sweep are not lost either way.
__device__ __forceinline__ void fix_sweep_slot(unsigned* w) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (*(volatile unsigned*)(w + i) >> 16) {  // (cheap look first: carries are rare)
      const unsigned c = atomicAnd(w + i, 0xffffu) >> 16;
      if (c) atomicAdd(w + i + 1, c);
    }
  }
}

__device__ __forceinline__ double fix_value(const double* slot, double inv_scale) {
  const unsigned* w = reinterpret_cast<const unsigned*>(slot);
  const double v = (double)(int)w[3] * 0x1p48 + (double)w[2] * 0x1p32 +
                   (double)w[1] * 0x1p16 + (double)w[0];  // each term exact
  return v * inv_scale;
}

// Shared-memory tally views (block-private).
struct SmemTally {
  double* trk;    // nb * I, batch b at (b - b_lo); kFix: 16-B limb slots
  double* cphi;   // I
  double* cJ;     // I
  double* cF;     // I
  double* edge;   // I + 1; kFix: 16-B limb slots
  double* cwb;    // nb
  double* bclo;   // 2
  unsigned* trc;  // I
};


// kShf: the fp64 tallies live in block-private shared memory (smem_tallies ==
// 1), statically, so the atomics compile to shared-memory CAS loops with no
// generic-address dispatch.
// kWin: the fixed-point histograms cover a window of cells [t_lo, t_lo + t_n)
// (FastArgs), where a mesh's full histograms do not fit shared memory (config
// 4's 4000 cells) but the step's particles stay in a narrow region around the
// pulse; scores outside the window go to the global tallies with fp64 REDs.
template <bool kUniform, bool kShf, bool kFix, int kW, bool kWin = false>
__global__ void __launch_bounds__(32 * kW, kMaxWarpsPerSm / kW) k_fast_segment(FastArgs a) {
  static_assert(kShf || !kFix, "fixed-point tallies live in shared memory");
  static_assert(!kWin || kFix, "windowed tallies are fixed-point");
  // (programmatic dependent launch: the block-private setup below — zeroed
  // histograms, mesh edges, log table — overlaps the window-update kernel this
  // launch follows; griddepcontrol.wait comes before the first read of anything
  // that kernel writes: the centres, the window flags, the pool counters)
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  // per-warp RLE split stack: the bottom kSmemStack records on chip (steady
  // state rarely goes deeper), the rest in global memory
  FastStackRec* stk = a.stacks + (size_t)gwarp * a.stack_cap;
  constexpr int kSmemStack = smem_stack<kW>();
  __shared__ FastStackRec s_stk[kW][kSmemStack];
  FastStackRec* s_my = s_stk[threadIdx.x >> 5];
#define STK(i) (*((i) < kSmemStack ? &s_my[(i)] : &stk[(i)]))
  int sp = 0;
  unsigned pend = 0;  // daughters pending in the local stack (warp-uniform)
  bool src_done = false;
  const int I = a.mesh.I;
  const double* __restrict__ edges = a.mesh.edges;
  const CellInfo* __restrict__ cells = a.mesh.cells;
  bool windows = false;  // (read after griddepcontrol.wait below)
  // smem_tallies: 0 all global REDs; 1 all block-private shared memory; 2 fp64
  // tallies as global REDs (native, fire-and-forget) and the integer track
  // counts in shared memory (shared fp64 adds are CAS loops on sm_100)
  const bool sh = a.smem_tallies != 0;       // shared memory in use (zero + flush)
  constexpr bool shf = kShf;                 // fp64 tallies in shared memory
  constexpr int slotw = kFix ? 2 : 1;
  // dynamic shared memory: [tallies (mode-dependent words) | window centres I |
  // edges I + 1], offsets precomputed on the host (FastArgs::so)
  SmemTally S;
  S.trc = reinterpret_cast<unsigned*>(smem);
  S.trk = smem + a.so.trk;
  S.cphi = smem + a.so.cphi;
  S.cJ = smem + a.so.cJ;
  S.cF = smem + a.so.cF;
  S.edge = smem + a.so.edge;
  S.cwb = smem + a.so.cwb;
  S.bclo = smem + a.so.bclo;
  const size_t tally_words = a.so.cent;
  // (grid scales 2^k from the launch arguments: constant-bank operands, no registers)
  const double fix_trk = a.fix_s_trk, fix_edge = a.fix_s_edge, fix_cw = a.fix_s_cw;
  __shared__ unsigned s_sweep;  // kFix: the carry sweep's slot cursor
  // kFix: the fixed-point slots, contiguous from S.trk (track nb*I, census
  // phi/J/F 3*I, edges I+1, census weight by batch nb)
  // tally window: cells [tlo, tlo + tn) (the whole mesh unless kWin)
  const int tlo = kWin ? a.t_lo : 0;
  const int tn = kWin ? a.t_n : I;
  // window cell of a global cell (-1 outside; edges: [0, tn])
  auto wcell = [&](int c) -> int {
    if constexpr (kWin) {
      const unsigned u = (unsigned)(c - tlo);
      return u < (unsigned)tn ? (int)u : -1;
    } else {
      return c;
    }
  };
  auto wedge = [&](int e) -> int {
    if constexpr (kWin) {
      const unsigned u = (unsigned)(e - tlo);
      return u <= (unsigned)tn ? (int)u : -1;
    } else {
      return e;
    }
  };
  const unsigned fix_slots = a.fix_slots;  // nb*tn + 4*tn + 1 + nb (launch_fast_segment)
  // slots per lane per sweep: every slot is swept within 4096 / 32 sweeps
  const unsigned fix_spl = a.fix_spl;
  if (kFix && threadIdx.x == 0) s_sweep = 0u;
  for (size_t i = threadIdx.x; i < tally_words; i += blockDim.x) smem[i] = 0.0;
  double* s_cent = smem + a.so.cent;  // read at every window site: keep it on chip
  // mesh edges (read at every event) and the log table, on chip
  double* s_edge = smem + a.so.edgex;
  for (int e = threadIdx.x; e <= I; e += blockDim.x) s_edge[e] = edges[e];
  __shared__ double s_logtab[256];
  for (int j = threadIdx.x; j < 256; j += blockDim.x) s_logtab[j] = c_logtab[j];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the window update has completed
  windows = a.centers != nullptr && (a.active == nullptr || *a.active != 0);
  if (windows)
    for (int i = threadIdx.x; i < I; i += blockDim.x) s_cent[i] = a.centers[i];
  __shared__ double s_w0;  // the weight of every comb tooth (the comb spacing, on the device)
  if (threadIdx.x == 0) s_w0 = a.n_packed ? *a.src_w0 : 0.0;
  // census thinning (FastArgs::precomb): each lane's distance to its next tooth,
  // in (0, s0], starting at a uniform offset; kept in global memory (L1-resident,
  // touched only at census events) off the event loop's registers and shared memory
  double* pc_need = a.pc_need + (size_t)gwarp * 32 + lane;
  if (a.precomb) {
    const U4 r = philox4x32_10(U4{(unsigned)gwarp, (unsigned)lane, a.pc_key, a.step}, a.k0 ^ 0x85ebca6bu,
                               a.k1 ^ 0xc2b2ae35u);
    double u, v;
    philox_uniform2(r, u, v);
    *pc_need = u * a.pc_s0;
  }
  __syncthreads();
  if (a.span && threadIdx.x == 0) atomicMin(&a.span[0], globaltimer());
  // per-lane event counters: 32 bits is plenty within one launch (registers
  // are what bounds occupancy here)
  unsigned n_coll = 0, n_cen = 0;
  // window-game, grazing and leakage events are rare: block counters in shared
  // memory (native 32-bit ATOMS.ADD) and a global RED for the leaked weight
  __shared__ unsigned s_rare[6];  // splits, daughters, capped, r.kills, r.survivals, grazing
  if (threadIdx.x < 6) s_rare[threadIdx.x] = 0u;
  __syncthreads();
  volatile unsigned long long* ctl = a.pool.ctl;

  unsigned n_iter = 0;
#ifdef HWWG_FAST_PROF
  unsigned n_ev = 0;  // events (timeline word 3): -DHWWG_FAST_PROF builds only (a register)
#endif
  // this warp's census chunk [wcur, wend), carried across the step's segments
  unsigned long long wcur = a.warp_cursor[2 * gwarp];
  unsigned wleft = (unsigned)(a.warp_cursor[2 * gwarp + 1] - wcur);  // <= kCensusChunk
  // (the timeline's start stamp goes out now: no register held through the loop)
  if (a.timeline && lane == 0) a.timeline[kTimelineWords * gwarp + 0] = globaltimer();
  Lane p;
  p.alive = false;
  p.fis = false;
  bool holding = true;  // this warp counts in pool.ctl[2] (active warps)
  bool declared = false;  // this warp has set pool.ctl[3] (backlog declared)
  // source reservation (warp-uniform) and the claim in flight (lane 0)
  // (32-bit: the driver keeps a segment's source below 2^32 - 2^26 particles)
  const unsigned n_src = (unsigned)a.n_src;
  const unsigned n_packed = (unsigned)a.n_packed;
  unsigned r_lo = (unsigned)gwarp * kClaim, r_hi = r_lo + kClaim;
  if (r_lo >= n_src) r_lo = r_hi = 0, src_done = true;
  else if (r_hi > n_src) r_hi = n_src;
  unsigned r_next = 0;
  bool r_pend = false;
  // claim size: kClaim, then kClaimTail once a claim lands in the last
  // HWWG_CLAIM_ZONE * kClaim particles per warp of the source, so the final reservations do
  // not pin a warp's worth of unstarted histories while other warps idle
  unsigned csz = kClaim;
  const unsigned tail_zone = gridDim.x * kW * kClaim * (unsigned)HWWG_CLAIM_ZONE;
  unsigned long long ticket = ~0ULL;  // lane 0: pool slot this warp waits on
  // The pool counters are reset without knowing this grid (fast_pool_reset:
  // active = kPoolSentinel, source head = 0), so the reset can ride on the
  // kernel before this one; the first thread turns the sentinel into the warp
  // count (until it lands, `active` cannot read zero) and claims start after
  // the static first reservations.
  if (blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(const_cast<unsigned long long*>(&ctl[2]),
              (unsigned long long)gridDim.x * kW - kPoolSentinel);
  const unsigned claim0 = gridDim.x * kW * kClaim;

  FPROF_DECL
#ifdef HWWG_FAST_PROF
  unsigned dg_maxpend = 0, dg_given = 0, dg_donated = 0, dg_taken = 0;  // timeline words 4..7
#endif
  while (true) {
#ifdef HWWG_FAST_PROF
    dg_maxpend = max(dg_maxpend, pend);
#endif
#ifdef HWWG_FAST_PROF
    fp_trip = clock64();
    fp_t = fp_trip;
#endif
    // ---- refill idle lanes: local split stack, then source bank, then pool
    // Work sharing. A backlog on this warp's stack while other warps sit idle
    // is the tail of a heavy split tree: one split of thousands of daughters,
    // or a deep tree of small ones, would otherwise drain 32 lanes at a time on
    // one warp while the grid waits. Hand the idle warps up to one piece each
    // in a single trip: split the top run into pieces (daughter index ranges
    // stay disjoint through the base offset) or give away whole records from
    // the top of the stack, keeping at least one trip of work here.
    // (the pool counters are one hot L2 line: a warp with a backlog looks at
    // them every kPollEvery-th trip, and declares the backlog once)
    if (pend > kShare && sp > 0 && (n_iter % kPollEvery) == 0) {
      unsigned open = 0;
      if (lane == 0) {
        if (!declared) ctl[3] = 1;  // declare a backlog: idle warps wait for work
        const unsigned long long t1 = ctl[1], t0 = ctl[0];
        open = t1 > t0 ? (unsigned)min(t1 - t0, 32ULL) : 0u;
      }
      declared = true;
      open = __shfl_sync(0xffffffffu, open, 0);
      if (open) {
        HWWG_CHECK(sp >= 1 && sp <= a.stack_cap);
        FastStackRec& top = STK(sp - 1);
        const unsigned cnt = top.count;
        const bool split_top = cnt >= 2 * kPiece;
        unsigned m = split_top ? min(open, cnt / kPiece - 1) : min(open, (unsigned)(sp - 1));
        const unsigned piece = split_top ? cnt / (m + 1) : 0u;
        unsigned long long s0 = 0;
        if (m && lane == 0) {
          atomicAdd(const_cast<unsigned long long*>(&ctl[2]), (unsigned long long)m);
          s0 = atomicAdd(const_cast<unsigned long long*>(&ctl[0]), (unsigned long long)m);
          if (s0 + m > a.pool.cap) {  // pool full: donate what fits, return the rest
            const unsigned fit = s0 < a.pool.cap ? (unsigned)(a.pool.cap - s0) : 0u;
            atomicAdd(const_cast<unsigned long long*>(&ctl[2]), (unsigned long long)(fit - m));
          }
        }
        s0 = __shfl_sync(0xffffffffu, s0, 0);
        if (m) {
          if (s0 + m > a.pool.cap) m = s0 < a.pool.cap ? (unsigned)(a.pool.cap - s0) : 0u;
          unsigned given = 0;
          if (lane < (int)m) {
            FastStackRec g = split_top ? top : STK(sp - 1 - lane);
            if (split_top) {
              g.base = top.base + lane * piece;
              g.count = piece;
            }
            given = g.count;
            g.ready = 0u;
            FastStackRec* pr = a.pool.recs + s0 + lane;
            *pr = g;
            __threadfence();
            *(volatile unsigned*)&pr->ready = 1u;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) given += __shfl_xor_sync(0xffffffffu, given, o);
          __syncwarp();
          if (split_top) {
            if (lane == 0) {
              top.count = cnt - m * piece;
              top.base += m * piece;
            }
          } else {
            sp -= (int)m;
          }
          pend -= given;
#ifdef HWWG_FAST_PROF
          dg_given += m;
#endif
          __syncwarp();
        }
      }
    }
    FPROF(8);
    unsigned need = __ballot_sync(0xffffffffu, !p.alive);
    // Pops from the top record: the bottom kSmemStack records are on chip, and
    // the two address spaces take separate paths so the on-chip one compiles
    // to shared-memory loads (a generic pointer to either cost address
    // resolution on every field of the record)
    auto pop = [&](FastStackRec& r) {
      const unsigned k = __popc(need);
      const unsigned cnt = r.count;
      const unsigned take = k < cnt ? k : cnt;
      const unsigned rank = __popc(need & lt);
      if (!p.alive && rank < take) load_rec(p, r, r.base + cnt - rank);
      __syncwarp();
      if (lane == 0) r.count = cnt - take;
      __syncwarp();
      pend -= take;
      if (cnt == take) --sp;
    };
    while (need && sp > 0) {
      HWWG_CHECK(sp >= 1 && sp <= a.stack_cap);
      if (sp <= kSmemStack) pop(s_my[sp - 1]);
      else pop(stk[sp - 1]);
      need = __ballot_sync(0xffffffffu, !p.alive);
    }
    FPROF(9);
    // Source claims: a warp holds a reservation [r_lo, r_hi) of up to kClaim
    // particles. Its first reservation is static (no atomic: every warp would
    // otherwise hit the one counter at launch); later ones are claimed one
    // trip AHEAD (after the event, see below), so the round trip of the
    // global atomic overlaps a whole event instead of stalling the refill.
    for (int pass = 0; pass < 2 && need && !src_done; ++pass) {
      if (r_lo == r_hi) {
        unsigned nb = 0;
        if (lane == 0)
          nb = r_pend ? r_next : claim0 + (unsigned)atomicAdd(a.src_head, (unsigned long long)csz);
        nb = __shfl_sync(0xffffffffu, nb, 0);
        r_pend = false;
        if (nb >= n_src) {
          src_done = true;
          break;
        }
        r_lo = nb;
        r_hi = nb + csz < n_src ? nb + csz : n_src;
        if (n_src - nb < tail_zone) csz = kClaimTail;
        // warm L1 with the new reservation once: its later refills hit on chip
        if ((unsigned)lane < r_hi - r_lo) {
          const unsigned kk = r_lo + lane;
          const unsigned pi =
              a.scramble && (kk | 1023u) < n_src ? (kk & ~1023u) | (__brev(kk) >> 22) : kk;
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a.src.xm + pi));
          if (pi >= n_packed) {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.src.wt + pi));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.src.meta + pi));
          }
        }
      }
      const unsigned k = __popc(need);
      const unsigned avail = r_hi - r_lo;
      const unsigned take = k < avail ? k : avail;
      const unsigned base = r_lo;
      r_lo += take;
      const unsigned rank = __popc(need & lt);
      if (!p.alive && rank < take) {
        // Claims walk the source in bit-reversed order inside 1024-particle
        // blocks: the bank is in census order, i.e. runs of daughters of one
        // split, and consecutive particles in one warp would collide on the
        // same tally cells (shared-memory CAS retries).
        const unsigned k = base + rank;
        const unsigned idx = a.scramble && (k | 1023u) < n_src ? (k & ~1023u) | (__brev(k) >> 22) : k;
        {
          HWWG_CHECK(idx < n_src);
          const double2 xm = a.src.xm[idx];
          p.x = xm.x;
          p.mu = xm.y;
          if (idx < n_packed) {  // a comb tooth: (x, mu) only (FastArgs::n_packed)
            p.w = s_w0;
            p.t = a.src_t0;
            p.cell = locate_cell_mul(a.mesh, p.x, a.inv_w0, s_edge);
            p.ctr = 0;
            p.hist = a.src_hist0 + idx;
            p.key = 0;
          } else {
            const double2 wt = a.src.wt[idx];
            const uint4 m = a.src.meta[idx];
            p.w = wt.x;
            p.t = wt.y;
            p.cell = (int)(m.x & 0xffffu);
            p.ctr = m.x >> 16;
            p.hist = m.y;
            p.key = ((unsigned long long)m.w << 32) | m.z;
          }
          p.inv_mu = rcp_nr(p.mu);
          p.bslot = batch_fast(p.hist, a.H, a.B, a.bmul) - (shf ? a.b_lo : 0);
          p.alive = p.w > 0.0;
          p.fis = false;
        }
      }
      need = __ballot_sync(0xffffffffu, !p.alive);
    }
    FPROF(10);
    const bool any_alive = need != 0xffffffffu;
    if (!any_alive && sp == 0 && src_done) {
      // Out of local work: claim a donated record, or leave when no warp can
      // donate any more (pool drained and no active warp).
      if (holding) {
        if (lane == 0) {
          __threadfence();
          atomicAdd(const_cast<unsigned long long*>(&ctl[2]), ~0ULL);  // active--
        }
        holding = false;
      }
      // Ticket queue: an idle warp takes the next pool slot (one atomicAdd, no
      // CAS storms) and waits for a donor to fill it. `active` counts busy
      // warps PLUS donated records not yet picked up (a donor adds one per
      // record before publishing it; the consumer inherits that unit), so
      // active == 0 means nothing can ever fill an outstanding ticket.
      int got = 0;  // 1: record ready in our slot, -1: finished
      // With no backlog declared anywhere (ctl[3]) there is nothing to wait
      // for: leave now rather than poll (the spread-out steady-state steps).
      if (lane == 0 && ticket == ~0ULL && ctl[3] == 0) got = -1;
      if (lane == 0 && got == 0) {
        if (ticket == ~0ULL) ticket = atomicAdd(const_cast<unsigned long long*>(&ctl[1]), 1ULL);
        if (ticket >= a.pool.cap) {
          got = -1;
        } else {
          HWWG_CHECK(ticket < a.pool.cap);
          const FastStackRec* pr = a.pool.recs + ticket;
          unsigned backoff = 32;
          while (true) {
            if (*(volatile const unsigned*)&pr->ready) {
              got = 1;
              break;
            }
            if (ctl[2] == 0) {
              __threadfence();
              if (*(volatile const unsigned*)&pr->ready) {
                got = 1;
                break;
              }
              got = -1;
              break;
            }
            __nanosleep(backoff);
            backoff = backoff < HWWG_BACKOFF ? backoff * 2 : HWWG_BACKOFF;  // idle polling costs issue slots
          }
        }
      }
      got = __shfl_sync(0xffffffffu, got, 0);
#ifdef HWWG_FAST_PROF
      fp_c[6] += clock64() - fp_trip;
#endif
      if (got < 0) break;
      const unsigned long long slot = __shfl_sync(0xffffffffu, ticket, 0);
      ticket = ~0ULL;
      holding = true;  // the record's active unit is ours now
      FastStackRec* pr = a.pool.recs + slot;
      __syncwarp();
      __threadfence();
      if (lane == 0) {
        STK(0) = *pr;
        STK(0).ready = 0;
        pr->ready = 0;  // slots are reused by the next segment
      }
      __syncwarp();
      sp = 1;
      pend = STK(0).count;
#ifdef HWWG_FAST_PROF
      ++dg_taken;
#endif
      continue;
    }
    if (!any_alive) continue;
    if (kFix && (n_iter % kSweepEvery) == 0) {  // carry sweep of the next 32 * spl slots
      unsigned c0 = 0;
      if (lane == 0) c0 = atomicAdd(&s_sweep, 32u * fix_spl);
      c0 = __shfl_sync(0xffffffffu, c0, 0);
      for (unsigned k = 0; k < fix_spl; ++k)
        fix_sweep_slot(reinterpret_cast<unsigned*>(S.trk) + 4 * ((c0 + 32u * k + lane) % fix_slots));
    }
#ifdef HWWG_FAST_PROF
    if (p.alive) ++n_ev;
#endif
    ++n_iter;
#ifdef HWWG_FAST_PROF
    if (lane == 0) {
      const unsigned long long dt_ns = globaltimer() - ctl[4];
      const int bin = (int)min(dt_ns / 5000ULL, (unsigned long long)(kHistBins - 1));
      const int sg = a.seg < 8 ? a.seg : 7;
      atomicAdd(&g_fhist[sg][bin][0], 1u);
      atomicAdd(&g_fhist[sg][bin][1], (unsigned)__popc(~need));
    }
#endif
    FPROF(0);

    // ---- one event per live lane; tally contributions are collected per lane
    // and committed warp-aggregated after the event (see agg_add)
    unsigned split_n = 0;
    bool fis_rec = false;  // the record pushed this trip holds fission secondaries
    int trk_key = -1, cen_cell = -1, cen_b = -1, edge_key = -1, trk_cell = 0;
    double trk_v = 0.0, cen_phi = 0.0, cen_J = 0.0, cen_F = 0.0, cen_w = 0.0, edge_v = 0.0;
    if (p.alive) {
      const CellInfo ci = kUniform ? a.cell0 : cells[p.cell];
      // edge position: the host table, or the same x_min + e*w (unfused) in registers
      auto edge_x = [&](int e) { return s_edge[e]; };
      double u0, u1, u2;
      draw3(a, p, u0, u1, u2);
      bool window_site = false;
      if (p.fis) {  // a fission secondary: its direction, then the window game (transport.cpp:181-185)
        p.fis = false;
        p.mu = 2.0 * u2 - 1.0;
        p.inv_mu = rcp_nr(p.mu);
        window_site = true;
      } else {
        const double d_census = ci.speed * (a.t_end - p.t);
        const double d_coll = neg_log_unit(u0, s_logtab) * ci.inv_sigma_t;
        double d_b = __longlong_as_double(0x7ff0000000000000LL);
        int edge = -1;
        if (p.mu > 0.0) {
          edge = p.cell + 1;
          d_b = (edge_x(edge) - p.x) * p.inv_mu;
        } else if (p.mu < 0.0) {
          edge = p.cell;
          d_b = (edge_x(edge) - p.x) * p.inv_mu;
        }
        double d = d_census;
        if (d_coll < d) d = d_coll;
        if (d_b < d) d = d_b;
        // (a d_b < 0 from rounding at an edge is a crossing, as in the reference:
        // transport.cpp:135-164 takes min{} as is and tests d == d_boundary)
        if (d > 0.0) {
          trk_v = p.w * d * ci.inv_dx * a.inv_dt;
          trk_key = p.bslot * I + p.cell;
          HWWG_CHECK(p.cell >= 0 && p.cell < I && p.bslot >= 0 && (!shf || p.bslot < a.nb) &&
                     p.bslot < a.B);
          trk_cell = p.cell;
        }
        if (d == d_census) {
          p.x += d * p.mu;
          p.t = a.t_end;
          cen_phi = ci.speed * p.w * ci.inv_dx;
          cen_J = cen_phi * p.mu;
          cen_F = cen_phi * (1.0 / 3.0 - p.mu * p.mu);
          cen_cell = p.cell;
          cen_w = p.w;
          cen_b = p.bslot;
          ++n_cen;
          p.alive = false;  // banked below, after the warp reconverges
        } else if (d == d_b) {
          p.x = edge_x(edge);
          p.t += d * ci.inv_speed;
          const bool domain = edge == 0 || edge == I;
          edge_v = (p.mu > 0 ? p.w : -p.w) * a.inv_dt;
          edge_key = edge;
          HWWG_CHECK(edge >= 0 && edge <= I);
          if (domain) {
            const double amu = fabs(p.mu);
            if (amu < 1e-10) {
              atomicAdd(&s_rare[5], 1u);
            } else {
              const double bc = p.w * (0.5 - amu) * rcp_nr(amu) * a.inv_dt;
              if (shf) atomicAdd(&S.bclo[edge == 0 ? 0 : 1], bc);
              else atomicAdd(&a.t.boundary_closure[edge == 0 ? 0 : 1], bc);
            }
            atomicAdd(&a.t.dcount[0], p.w);
            p.alive = false;
          } else {
            p.cell += p.mu > 0.0 ? 1 : -1;
            window_site = true;
          }
        } else {  // collision
          p.x += d * p.mu;
          p.t += d * ci.inv_speed;
          ++n_coll;
          const double xi = u1 * ci.sigma_t;
          if (xi < ci.sigma_s) {
            p.mu = 2.0 * u2 - 1.0;
            p.inv_mu = rcp_nr(p.mu);
            u1 = xi * ci.inv_sigma_s;  // recycled roulette deviate for the window game below
            window_site = true;
          } else if (xi < ci.sigma_s + ci.sigma_f) {
            // fission (transport.cpp:29-40, 179-188): floor(nu) + Bernoulli(frac)
            // secondaries, the Bernoulli deviate the unused scattering one; this
            // lane becomes the first secondary, the rest go on the stack as one
            // fission record; each secondary's direction and window game follow
            // on its own next trip (the parent itself is not windowed)
            const double fl = floor(ci.nu_f);
            const double frac = ci.nu_f - fl;
            const unsigned n = (unsigned)fl + (frac > 0.0 && u2 < frac ? 1u : 0u);
            if (n == 0) {
              p.alive = false;
            } else {
              p.fis = true;
              split_n = n;
              fis_rec = true;
            }
          } else {  // capture
            p.alive = false;
          }
        }
      }
      if (window_site && windows) {  // ww.cpp:46-72 (split conserves, roulette unbiased)
        HWWG_CHECK(p.cell >= 0 && p.cell < I);
        const double c = s_cent[p.cell];
        if (p.w > c * a.rho) {
          double n = ceil(p.w * rcp_nr(c));  // (no IEEE division: its slow-path call)
          if (n > 1e6) {
            n = 1e6;
            atomicAdd(&s_rare[2], 1u);
          }
          split_n = (unsigned)n;
          p.w = p.w * rcp_nr(n);
          atomicAdd(&s_rare[0], 1u);
          atomicAdd(&s_rare[1], split_n - 1);
        } else if (p.w < c * a.inv_rho) {
          if (u1 * c < p.w) {
            p.w = c;
            atomicAdd(&s_rare[4], 1u);
          } else {
            p.alive = false;
            atomicAdd(&s_rare[3], 1u);
          }
        }
      }
    }
    FPROF(1);
    // ---- look-ahead source claim: the reservation is spent and lanes will need
    // particles; the atomic's latency hides behind the census and tally work
    if (r_lo == r_hi && !r_pend && !src_done) {
      if (lane == 0) r_next = claim0 + (unsigned)atomicAdd(a.src_head, (unsigned long long)csz);
      r_pend = true;
    }
    // ---- bank census particles. Slots come from a per-warp chunk of the census
    // bank (one global atomic per kCensusChunk particles, not one per warp per
    // iteration: a single shared counter hit by every warp serialised whole
    // segments). Chunk tails left at the end of a step become zero-weight
    // records (fill_census_holes), which the comb never selects.
    {
      bool bank = cen_cell >= 0;
      double w_bank = p.w;
      if (a.precomb && bank) {  // census thinning: this particle's teeth on the lane's comb
        double need = *pc_need;
        if (p.w < need) {
          need -= p.w;
          bank = false;
        } else {
          const double r = p.w - need;  // past the first tooth
          const double k = floor(r * a.pc_inv_s0);
          double rem = r - k * a.pc_s0;  // in [0, s0) up to rounding
          rem = rem < 0.0 ? 0.0 : (rem >= a.pc_s0 ? 0.0 : rem);
          need = a.pc_s0 - rem;
          w_bank = (k + 1.0) * a.pc_s0;
        }
        *pc_need = need;
      }
      const unsigned cmask = __ballot_sync(0xffffffffu, bank);
      if (cmask) {
        const unsigned k = __popc(cmask);
        const unsigned avail = wleft;
        unsigned long long nb = 0;
        if (k > avail) {
          if (lane == 0) nb = atomicAdd(a.census_count, (unsigned long long)kCensusChunk);
          nb = __shfl_sync(0xffffffffu, nb, 0);
        }
        if (bank) {
          const unsigned rank = __popc(cmask & lt);
          const unsigned long long slot = rank < avail ? wcur + rank : nb + (rank - avail);
          if (slot < a.census_cap) {  // t = t_end, the cell follows from x
            a.census.xm[slot] = make_double2(p.x, p.mu);
            a.census.w[slot] = w_bank;
          }
        }
        if (k > avail) {
          wcur = nb + (k - avail);
          wleft = kCensusChunk - (k - avail);
        } else {
          wcur += k;
          wleft -= k;
        }
      }
    }

    FPROF(2);
    // ---- commit the event's tallies, warp-aggregated (lanes sharing a cell
    // are summed with shuffles first: one CAS per distinct address, not per lane)
    if (!kFix && a.aggregate) {  // cold-start segments (never with fixed-point slots): most lanes share a few cells
      if (shf) {
        agg_add_count(S.trk, S.trc, trk_key, trk_v, trk_cell);
        agg_add3(S.cphi, S.cJ, S.cF, cen_cell, cen_phi, cen_J, cen_F);
        agg_add(S.cwb, cen_b, cen_w);
        agg_add(S.edge, edge_key, edge_v);
      } else {
        agg_add_count_global(a.t.track_flux_batch, a.t.tracks, trk_key, trk_v, trk_cell);
        agg_add3(a.t.census_phi, a.t.census_current, a.t.census_closure, cen_cell, cen_phi,
                 cen_J, cen_F);
        agg_add(a.t.census_weight_batch, cen_b, cen_w);
        agg_add(a.t.edge_current, edge_key, edge_v);
      }
    } else {  // spread population: per-lane atomics, no warp synchronisation
      double* trk = kShf ? S.trk : a.t.track_flux_batch;
      double* cphi = kShf ? S.cphi : a.t.census_phi;
      double* cJ = kShf ? S.cJ : a.t.census_current;
      double* cF = kShf ? S.cF : a.t.census_closure;
      double* cwb = kShf ? S.cwb : a.t.census_weight_batch;
      // kFix: the census weight by batch on limb slots too (no shared fp64 CAS loop)
      auto fix_cwb = [&](int bb, double w) {
        if (!fix_add(S.cwb + 2 * bb, w, fix_cw)) atomicAdd(a.t.census_weight_batch + a.b_lo + bb, w);
      };
      double* edg = kShf ? S.edge : a.t.edge_current;
      if (trk_key >= 0) {
        const int wc = wcell(trk_cell);
        if (!kFix) atomicAdd(trk + trk_key, trk_v);
        else if (wc < 0 || !fix_add(S.trk + 2 * (kWin ? p.bslot * tn + wc : trk_key), trk_v, fix_trk))
          atomicAdd(a.t.track_flux_batch + (size_t)a.b_lo * I + trk_key, trk_v);
        if (sh && wc >= 0) atomicAdd(S.trc + wc, 1u);
        else atomicAdd(a.t.tracks + trk_cell, 1ULL);
      }
#if !defined(HWWG_CENSUS_PER_LANE)
      // census scores: fixed-point slots take per-lane native adds in a spread
      // population (no conflict cost worth a warp scan); in the cold start and
      // with fp64 slots they are run-aggregated (census_runs)
      if (kFix && !a.census_runs) {
        if (cen_cell >= 0) {
          const int wc = wcell(cen_cell);
          if (wc < 0 || !fix_add(S.cphi + 2 * wc, cen_phi, fix_trk)) atomicAdd(a.t.census_phi + cen_cell, cen_phi);
          if (wc < 0 || !fix_add(S.cJ + 2 * wc, cen_J, fix_trk)) atomicAdd(a.t.census_current + cen_cell, cen_J);
          if (wc < 0 || !fix_add(S.cF + 2 * wc, cen_F, fix_trk)) atomicAdd(a.t.census_closure + cen_cell, cen_F);
        }
        // per lane, not run-aggregated: a spread population's census lanes rarely
        // share a slot, and a run scan costs issue slots (C5 +2%, C2 +2.3%)
        if (cen_cell >= 0) fix_cwb(cen_b, cen_w);
      } else if (kFix) {  // cold start: identical split copies reach census together
        census_groups(
            [&](int cell, double s0, double s1, double s2) {
              const int wc = wcell(cell);
              if (wc < 0 || !fix_add(S.cphi + 2 * wc, s0, fix_trk)) atomicAdd(a.t.census_phi + cell, s0);
              if (wc < 0 || !fix_add(S.cJ + 2 * wc, s1, fix_trk)) atomicAdd(a.t.census_current + cell, s1);
              if (wc < 0 || !fix_add(S.cF + 2 * wc, s2, fix_trk)) atomicAdd(a.t.census_closure + cell, s2);
            },
            fix_cwb, cen_cell, cen_b, cen_w, p.mu, cen_phi, cen_J, cen_F);
      } else {
        census_runs(
            [&](int cell, double s0, double s1, double s2) {
              atomicAdd(cphi + cell, s0);
              atomicAdd(cJ + cell, s1);
              atomicAdd(cF + cell, s2);
            },
            cwb, cen_cell, cen_b, cen_phi, cen_J, cen_F, cen_w);
      }
#else
      if (cen_cell >= 0) {
        atomicAdd(cphi + cen_cell, cen_phi);
        atomicAdd(cJ + cen_cell, cen_J);
        atomicAdd(cF + cen_cell, cen_F);
        atomicAdd(cwb + cen_b, cen_w);
      }
#endif
      if (edge_key >= 0) {
        const int we = wedge(edge_key);
        if (!kFix) atomicAdd(edg + edge_key, edge_v);
        else if (we < 0 || !fix_add(S.edge + 2 * we, edge_v, fix_edge))
          atomicAdd(a.t.edge_current + edge_key, edge_v);
      }
    }

    FPROF(3);
    // ---- push split records: local stack while shallow, else donate to the pool
    const unsigned smask = __ballot_sync(0xffffffffu, split_n > 1);
    if (smask) {
      const unsigned dau = split_n > 1 ? split_n - 1 : 0;
      unsigned tot = dau;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      // donate only a real backlog, and only while idle warps hold open tickets
      bool donate = pend + tot > kDonate;  // warp-uniform
      if (donate) {
        int open = 0;
        if (lane == 0) {
          if (!declared) ctl[3] = 1;  // declare a backlog: idle warps wait for donations
          open = ctl[1] > ctl[0] ? 1 : 0;
        }
        declared = true;
        donate = __shfl_sync(0xffffffffu, open, 0) != 0;
      }
      const FastStackRec rec{p.x, p.mu, p.w, p.t, (unsigned)p.cell | ((unsigned)p.bslot << 16),
                             p.hist, p.key, p.ctr | (fis_rec ? kFissionRec : 0u), dau, 0u,
                             0u, p.inv_mu};  // base 0: daughters 1..dau
      bool push_local = dau > 0 && !donate;
      // one pair of atomics per warp: the donated records' active units, then
      // their slots (ordered before this warp's own decrement by the fence on
      // the idle path; the donor counts as active meanwhile)
      const unsigned dmask = __ballot_sync(0xffffffffu, dau > 0 && donate);
      unsigned long long dbase = 0;
      if (dmask && lane == 0) {
        atomicAdd(const_cast<unsigned long long*>(&ctl[2]), (unsigned long long)__popc(dmask));
        dbase = atomicAdd(const_cast<unsigned long long*>(&ctl[0]), (unsigned long long)__popc(dmask));
      }
      dbase = __shfl_sync(0xffffffffu, dbase, 0);
#ifdef HWWG_FAST_PROF
      dg_donated += __popc(dmask);
#endif
      if (dau > 0 && donate) {
        const unsigned long long slot = dbase + __popc(dmask & lt);
        if (slot < a.pool.cap) {
          FastStackRec* pr = a.pool.recs + slot;
          *pr = rec;
          __threadfence();
          *(volatile unsigned*)&pr->ready = 1u;
        } else {
          atomicAdd(const_cast<unsigned long long*>(&ctl[2]), ~0ULL);
          push_local = true;  // pool full: keep it
        }
      }
      const unsigned lmask = __ballot_sync(0xffffffffu, push_local);
      if (push_local) {
        const int slot = sp + (int)__popc(lmask & lt);
        if (slot < kSmemStack) s_my[slot] = rec;
        else if (slot < a.stack_cap) stk[slot] = rec;
        else atomicCAS(&a.err->code, 0, HWWG_ESTACK);
      }
      unsigned ld = push_local ? dau : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ld += __shfl_xor_sync(0xffffffffu, ld, o);
      pend += ld;
      sp += __popc(lmask);
      if (sp > a.stack_cap) sp = a.stack_cap;
      __syncwarp();
    }
    FPROF(4);
#ifdef HWWG_FAST_PROF
    fp_c[5] += 1;
#endif
  }
#ifdef HWWG_FAST_PROF
  fp_c[7] = clock64() - fp_k0;
  if (lane == 0)
    for (int k = 0; k < 12; ++k) atomicAdd(&g_fprof[k], fp_c[k]);
#endif

  if (a.fill_tail) {  // k_fill_holes for this warp's chunk tail
    for (unsigned k = lane; k < wleft; k += 32) {
      const unsigned long long slot = wcur + k;
      if (slot < a.census_cap) {
        a.census.xm[slot] = make_double2(a.x_fill, 0.5);
        a.census.w[slot] = 0.0;
      }
    }
  }
  if (lane == 0) {
    a.warp_cursor[2 * gwarp] = wcur;
    a.warp_cursor[2 * gwarp + 1] = wcur + wleft;
  }
  if (a.timeline) {
#ifdef HWWG_FAST_PROF
    unsigned long long ev = n_ev;
#else
    unsigned long long ev = 0;  // (events are counted in -DHWWG_FAST_PROF builds)
#endif
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ev += __shfl_down_sync(0xffffffffu, ev, o);
    if (lane == 0) {
      a.timeline[kTimelineWords * gwarp + 1] = n_iter;
      a.timeline[kTimelineWords * gwarp + 2] = globaltimer();
      a.timeline[kTimelineWords * gwarp + 3] = ev;
#ifdef HWWG_FAST_PROF
      a.timeline[kTimelineWords * gwarp + 4] = dg_maxpend;
      a.timeline[kTimelineWords * gwarp + 5] = dg_given;
      a.timeline[kTimelineWords * gwarp + 6] = dg_donated;
      a.timeline[kTimelineWords * gwarp + 7] = dg_taken;
#endif
    }
  }

  // ---- flush block-private tallies
  if (shf && !kFix && a.flush_replicas) {
    // into one of R global replicas of the smem layout (R-fold less same-address
    // contention than every block adding into the one tally set at segment end);
    // k_flush_reduce folds the replicas into the tallies
    __syncthreads();
    double* rep = a.flush_scratch + (size_t)(blockIdx.x % a.flush_replicas) * a.flush_stride;
    const int nd = (a.nb + 4) * I + 1 + a.nb + 2;
    for (int i = threadIdx.x; i < nd; i += blockDim.x) {
      const double v = S.trk[i];
      if (v != 0.0) atomicAdd(rep + i, v);
    }
    unsigned long long* rc = reinterpret_cast<unsigned long long*>(rep + nd);
    for (int i = threadIdx.x; i < I; i += blockDim.x)
      if (S.trc[i]) atomicAdd(rc + i, (unsigned long long)S.trc[i]);
  } else if (shf) {
    __syncthreads();
    const int nb = a.nb;
    const double inv_trk = kFix ? pow2(-a.fix_k_trk) : 0.0;
    const double inv_edge = kFix ? pow2(-a.fix_k_edge) : 0.0;
    for (int i = threadIdx.x; i < nb * tn; i += blockDim.x) {
      const double v = kFix ? fix_value(S.trk + 2 * i, inv_trk) : S.trk[i];
      // (window slot i = batch i / tn, cell tlo + i % tn)
      const size_t g = kWin ? (size_t)(i / tn) * I + tlo + i % tn : (size_t)i;
      if (v != 0.0) atomicAdd(&a.t.track_flux_batch[(size_t)a.b_lo * I + g], v);
    }
    for (int i = threadIdx.x; i < tn; i += blockDim.x) {
      const double vp = kFix ? fix_value(S.cphi + 2 * i, inv_trk) : S.cphi[i];
      const double vj = kFix ? fix_value(S.cJ + 2 * i, inv_trk) : S.cJ[i];
      const double vf = kFix ? fix_value(S.cF + 2 * i, inv_trk) : S.cF[i];
      if (vp != 0.0) atomicAdd(&a.t.census_phi[tlo + i], vp);
      if (vj != 0.0) atomicAdd(&a.t.census_current[tlo + i], vj);
      if (vf != 0.0) atomicAdd(&a.t.census_closure[tlo + i], vf);
      if (S.trc[i]) atomicAdd(&a.t.tracks[tlo + i], (unsigned long long)S.trc[i]);
    }
    for (int i = threadIdx.x; i <= tn; i += blockDim.x) {
      const double v = kFix ? fix_value(S.edge + 2 * i, inv_edge) : S.edge[i];
      if (v != 0.0) atomicAdd(&a.t.edge_current[tlo + i], v);
    }
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
      const double v = kFix ? fix_value(S.cwb + 2 * i, pow2(-a.fix_k_cw)) : S.cwb[i];
      if (v != 0.0) atomicAdd(&a.t.census_weight_batch[a.b_lo + i], v);
    }
    if (threadIdx.x < 2 && S.bclo[threadIdx.x] != 0.0)
      atomicAdd(&a.t.boundary_closure[threadIdx.x], S.bclo[threadIdx.x]);
  } else if (sh) {
    __syncthreads();
    for (int i = threadIdx.x; i < I; i += blockDim.x)
      if (S.trc[i]) atomicAdd(&a.t.tracks[i], (unsigned long long)S.trc[i]);
  } else {
    __syncthreads();
  }
  if (threadIdx.x < 6 && s_rare[threadIdx.x]) {
    // s_rare[0..4] follow UCounter kSplits..kRouletteSurvivals; [5] is grazing
    const int slot = threadIdx.x < 5 ? kSplits + (int)threadIdx.x : kGrazingDiscarded;
    atomicAdd(&a.t.ucount[slot], (unsigned long long)s_rare[threadIdx.x]);
  }

  // ---- counters (warp-aggregated)
  auto wsum = [](unsigned v32) {
    unsigned long long v = v32;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
  };
  const unsigned long long coll = wsum(n_coll), cen = wsum(n_cen);
  if (lane == 0) {
    unsigned long long* u = a.t.ucount;
    if (coll) atomicAdd(&u[kCollisions], coll);
    if (cen) atomicAdd(&u[kCensusCount], cen);
  }
  if (a.span) {  // the block's end, after all its warps
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&a.span[1], globaltimer());
  }
}

#undef STK

// Folds the flush replicas into the tallies and re-zeroes them: one owner per
// word, so plain adds (the layout is k_fast_segment's shared-memory layout from
// the track-batch block on: trk[nb*I], cphi, cJ, cF [I], edge[I+1], cwb[nb],
// bclosure[2], then the track counts as u64[I]).
__global__ void k_flush_reduce(double* scratch, int R, size_t stride, int I, int nb, int b_lo,
                               TallyPtrs t) {
  const int nd = (nb + 4) * I + 1 + nb + 2;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nd + I; w += gridDim.x * blockDim.x) {
    if (w < nd) {
      double v = 0.0;
      for (int r = 0; r < R; ++r) {
        double* q = scratch + (size_t)r * stride + w;
        v += *q;
        *q = 0.0;
      }
      if (v == 0.0) continue;
      double* dst;
      if (w < nb * I) dst = t.track_flux_batch + (size_t)b_lo * I + w;
      else if (w < (nb + 1) * I) dst = t.census_phi + (w - nb * I);
      else if (w < (nb + 2) * I) dst = t.census_current + (w - (nb + 1) * I);
      else if (w < (nb + 3) * I) dst = t.census_closure + (w - (nb + 2) * I);
      else if (w < (nb + 4) * I + 1) dst = t.edge_current + (w - (nb + 3) * I);
      else if (w < (nb + 4) * I + 1 + nb) dst = t.census_weight_batch + b_lo + (w - ((nb + 4) * I + 1));
      else dst = t.boundary_closure + (w - ((nb + 4) * I + 1 + nb));
      *dst += v;
    } else {
      unsigned long long c = 0;
      for (int r = 0; r < R; ++r) {
        unsigned long long* q = reinterpret_cast<unsigned long long*>(scratch + (size_t)r * stride + nd) + (w - nd);
        c += *q;
        *q = 0ULL;
      }
      if (c) t.tracks[w - nd] += c;
    }
  }
}

// Source bank from AoS particles (the pulse source, host-bank round trips).
__global__ void k_aos_to_fast(const hwwg_particle* __restrict__ in, uint64_t n, const MeshView m,
                              FastBank out, uint64_t hist0) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 a = reinterpret_cast<const double2*>(in)[2 * i];
  const double2 b = reinterpret_cast<const double2*>(in)[2 * i + 1];
  out.xm[i] = a;
  out.wt[i] = b;
  const int c = locate_cell(m, a.x);
  out.meta[i] = make_uint4((unsigned)(c < 0 ? 0 : c), (unsigned)(hist0 + i), 0u, 0u);
}

}  // namespace

size_t fast_smem_bytes(int I, int nb) {
  return ((size_t)(nb + 4) * I + 1 + nb + 2) * sizeof(double) + (size_t)(I + 1) / 2 * 8 + 16;
}
size_t fast_smem_count_bytes(int I) { return (size_t)(I + 1) / 2 * 8 + 16; }
size_t fast_smem_fix_bytes(int I, int nb) {
  return ((size_t)2 * ((size_t)nb * I + 4 * (size_t)I + 1 + nb) + 2) * sizeof(double) +
         (size_t)(I + 1) / 2 * 8 + 16;
}
// Grid exponent k for the fixed-point tallies: the largest expected score
// (vmax) lands near 2^40 grid units, leaving 2^22 of headroom below the 2^62
// guard and 2^-40 of vmax as resolution. False when vmax is unusable (the
// driver then keeps the fp64 layout).
bool fast_fix_exponent(double vmax, int* k) {
  if (!(vmax > 0.0) || !std::isfinite(vmax)) return false;
  const int e = 40 - std::ilogb(vmax);
  *k = e < -1000 ? -1000 : (e > 1000 ? 1000 : e);
  return true;
}
size_t fast_smem_centers_bytes(int I) { return (size_t)(2 * I + 1) * 8; }  // centres + edges
size_t fast_flush_stride(int I, int B) { return (size_t)(B + 4) * I + 1 + B + 2 + I; }

int fast_max_warps_per_sm() { return kMaxWarpsPerSm; }

// -DHWWG_FAST_PROF builds: read and clear the loop phase accounting (0 otherwise)
int fast_prof_read(unsigned long long out[12], unsigned* hist) {
#ifdef HWWG_FAST_PROF
  if (hist) {
    HWWG_CUDA(cudaMemcpyFromSymbol(hist, g_fhist, sizeof(g_fhist)));
    std::vector<unsigned> zh(sizeof(g_fhist) / sizeof(unsigned), 0u);
    HWWG_CUDA(cudaMemcpyToSymbol(g_fhist, zh.data(), sizeof(g_fhist)));
  }
  HWWG_CUDA(cudaMemcpyFromSymbol(out, g_fprof, 12 * sizeof(unsigned long long)));
  const unsigned long long z[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  HWWG_CUDA(cudaMemcpyToSymbol(g_fprof, z, sizeof z));
  return 1;
#else
  (void)out;
  (void)hist;
  return 0;
#endif
}

void configure_fast_kernel();

using FastKernel = void (*)(FastArgs);
// fix: 0 fp64 tallies, 1 fixed-point, 2 fixed-point over a cell window (kWin)
template <int kW>
FastKernel fast_kernel_w(int uniform, int shf, int fix) {
  return uniform && fix == 2 ? k_fast_segment<true, true, true, kW, true>
         : fix == 2          ? k_fast_segment<false, true, true, kW, true>
         : uniform && fix   ? k_fast_segment<true, true, true, kW>
         : uniform && shf ? k_fast_segment<true, true, false, kW>
         : uniform        ? k_fast_segment<true, false, false, kW>
         : fix            ? k_fast_segment<false, true, true, kW>
         : shf            ? k_fast_segment<false, true, false, kW>
                          : k_fast_segment<false, false, false, kW>;
}
FastKernel fast_kernel(int uniform, int shf, int fix, int warps) {
  return warps == 24   ? fast_kernel_w<24>(uniform, shf, fix)
         : warps == 14 ? fast_kernel_w<14>(uniform, shf, fix)
                       : fast_kernel_w<12>(uniform, shf, fix);
}

// resident blocks per SM of the instantiation a launch will use (the
// persistent grid must be fully resident: idle warps wait on busy ones)
int fast_blocks_per_sm(size_t smem, int uniform, int shf, int fix, int warps) {
  // memoised per device: the driver asks several times per segment, and the
  // host must stay ahead of ~20 us segments (config 1)
  static std::mutex m;
  static std::map<std::tuple<int, size_t, int, int, int, int>, int> memo;
  int dev = 0;
  HWWG_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_tuple(dev, smem, uniform, shf, fix, warps);
  {
    std::lock_guard<std::mutex> lk(m);
    const auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  configure_fast_kernel();
  int n = 0;
  HWWG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &n, fast_kernel(uniform, shf, fix, warps), 32 * warps, smem));
  std::lock_guard<std::mutex> lk(m);
  memo[key] = n;
  return n;
}

namespace {
__global__ void k_segment_reset(unsigned long long* ctl, unsigned long long* src_head,
                                unsigned long long* span) {
  fast_pool_reset(ctl, src_head, span);
}
}  // namespace

void configure_fast_kernel() {
  static thread_local int done_dev = -1;  // this thread configured this device already
  int dev = 0;
  HWWG_CUDA(cudaGetDevice(&dev));
  if (dev == done_dev) return;
  static DynSmemCache configured[24];
  int i = 0;
  for (int w : kFastBlockWarps)
    for (int u = 0; u < 2; ++u)
      for (int sh = 0; sh < 2; ++sh)
        for (int f = 0; f <= 2 * sh; ++f) {
          // the block's static shared memory (its split-stack bottoms) comes first
          const FastKernel k = fast_kernel(u, sh, f, w);
          cudaFuncAttributes fa{};
          HWWG_CUDA(cudaFuncGetAttributes(&fa, k));
          ensure_dyn_smem(k, std::min<size_t>(200 * 1024, 227 * 1024 - fa.sharedSizeBytes),
                          configured[i++]);
        }
  done_dev = dev;
}

void launch_fast_segment(const FastArgs& a0, int blocks, size_t smem, cudaStream_t s) {
  configure_fast_kernel();
  FastArgs a = a0;
  // fixed-point grid scales and sweep parameters, once per launch (kernel
  // parameters: constant-bank operands in the event loop)
  a.fix_s_trk = std::ldexp(1.0, a.fix_k_trk);
  a.fix_s_edge = std::ldexp(1.0, a.fix_k_edge);
  a.fix_s_cw = std::ldexp(1.0, a.fix_k_cw);
  {
    const unsigned tn = (a.smem_tallies == 1 && a.fix && a.t_win) ? (unsigned)a.t_n : (unsigned)a.mesh.I;
    a.fix_slots = (unsigned)a.nb * tn + 4 * tn + 1 + (unsigned)a.nb;
    a.fix_spl = (a.fix_slots + 4095u) / 4096u;
  }
  {  // the dynamic shared-memory layout (SmemOffsets; smem_view's order)
    // (the histograms span the tally window's cells, the centres and edges the mesh)
    const unsigned I = (unsigned)a.mesh.I, nb = (unsigned)a.nb;
    const unsigned T = (a.smem_tallies == 1 && a.fix && a.t_win) ? (unsigned)a.t_n : I;
    const unsigned slotw = (a.smem_tallies == 1 && a.fix) ? 2u : 1u;
    SmemOffsets& o = a.so;
    o.trk = (T + 1) / 2;
    o.cphi = o.trk + slotw * nb * T;
    o.cJ = o.cphi + slotw * T;
    o.cF = o.cJ + slotw * T;
    o.edge = o.cF + slotw * T;
    o.cwb = o.edge + slotw * (T + 1);
    o.bclo = o.cwb + slotw * nb;
    o.cent = a.smem_tallies == 1 ? o.bclo + 2 : (a.smem_tallies ? (I + 1) / 2 : 0);
    o.edgex = o.cent + I;
  }
  if (!a.pool_reset_done) k_segment_reset<<<1, 1, 0, s>>>(a.pool.ctl, a.src_head, a.span);
  const bool shf = a.smem_tallies == 1;
  const int fix = shf && a.fix ? (a.t_win ? 2 : 1) : 0;
  const FastKernel k = fast_kernel(a.uniform, shf, fix, a.warps);
  // programmatic dependent launch: the grid may be scheduled while the kernel
  // before it (the window update) drains; every block waits for it
  // (griddepcontrol.wait) before touching memory
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(32 * a.warps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  HWWG_CUDA(cudaLaunchKernelEx(&cfg, k, a));
  if (shf && !fix && a.flush_replicas) {
    k_flush_reduce<<<32, 256, 0, s>>>(a.flush_scratch, a.flush_replicas, a.flush_stride, a.mesh.I,
                                      a.nb, a.b_lo, a.t);
    HWWG_CUDA(cudaGetLastError());
  }
}

void launch_aos_to_fast(const hwwg_particle* in, uint64_t n, const MeshView& m, FastBank out,
                        uint64_t hist0, cudaStream_t s) {
  if (!n) return;
  k_aos_to_fast<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, n, m, out, hist0);
  HWWG_CUDA(cudaGetLastError());
}

}  // namespace hwwg
