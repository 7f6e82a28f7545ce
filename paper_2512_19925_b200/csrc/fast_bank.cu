// Throughput-mode bank kernels: the parallel comb (population control at step
// start, proj/src/popctrl.cpp:7-42) and bank format conversions.
//
// The comb keeps the reference's estimator — teeth spaced W/target apart with
// one random offset walk the cumulative-weight axis of the bank — but the
// cumulative weights are exact fixed-point integers summed in tiles (two
// passes, O(n/4096) scratch) instead of a serial fp64 walk, and each particle
// writes the teeth that fall in its cumulative-weight interval. Tooth k lands
// at perm(k) (fast.cuh Perm). The multi-GPU pieces (a local CUB scan, teeth
// placed by binary search against a global origin) are at the end.
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "common.cuh"
#include "fast.cuh"
#include "rng.cuh"

namespace hwwg {

namespace {

__global__ void k_extract_w(CensusBank b, uint64_t n, double* w) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = b.w[i];
}

// mesh.cpp:26-40 with the uniform estimate by a multiplication with 1 / w0:
// the +-1 guards turn any estimate within one cell of the truth into the
// unique c with edges[c] <= x < edges[c+1], so the result equals locate_cell's
// (throughput mode only; the exact mode keeps the reference's division)
__device__ __forceinline__ int locate_cell_mul(const MeshView& m, double x, double inv_w0) {
  if (!m.uniform) return locate_cell(m, x);
  if (x < m.x_min || x > m.x_max) return -1;
  if (x == m.x_max) return m.I - 1;
  int c = (int)((x - m.x_min) * inv_w0);
  if (c >= m.I) c = m.I - 1;
  if (c < 0) c = 0;
  if (x < m.edges[c]) --c;
  else if (x >= m.edges[c + 1]) ++c;
  return c;
}

__device__ __forceinline__ void write_tooth(const FastCombArgs& a, double2 xm, uint64_t k,
                                            double spacing, double inv_w0) {
  HWWG_CHECK(k < a.target);
  const uint64_t p = a.perm(k);
  HWWG_CHECK(p < a.target);
  a.out.xm[p] = xm;
  if (a.packed_out) return;  // the transport derives (w, t), cell and identity
  const int c = locate_cell_mul(a.mesh, xm.x, inv_w0);  // as advance_history locates a start (transport.cpp:95)
  a.out.wt[p] = make_double2(spacing, a.t_bank);
  a.out.meta[p] = make_uint4((unsigned)(c < 0 ? 0 : c), (unsigned)p, 0u, 0u);
}

__device__ __forceinline__ void write_teeth(const FastCombArgs& a, uint64_t src, uint64_t k0,
                                            uint64_t k1, double spacing) {
  HWWG_CHECK(src < a.n && k1 <= a.target);
  const double2 xm = a.bank.xm[src];
  const int c = locate_cell(a.mesh, xm.x);  // as advance_history locates a start (transport.cpp:95)
  for (uint64_t k = k0; k < k1; ++k) {
    const uint64_t p = a.perm(k);
    HWWG_CHECK(p < a.target);
    a.out.xm[p] = xm;
    if (a.packed_out) continue;
    a.out.wt[p] = make_double2(spacing, a.t_bank);
    // fresh identity for the new step: history = its slot, key 0, draw 0
    a.out.meta[p] = make_uint4((unsigned)(c < 0 ? 0 : c), (unsigned)p, 0u, 0u);
  }
}

// ---- single-GPU comb: two passes over the bank in 4096-particle tiles ------
// The cumulative weights are exact integers: every weight becomes
// floor(w * 2^s), with 2^s chosen from a bound on the bank total known before
// the comb (the step's census-weight tallies, or the pulse strength) so the
// total stays below 2^61. Integer tile sums are associative, so tile starts are
// exact and both sides of every tile boundary see the same prefix; each tile
// then recomputes its particles' prefixes in a block scan and every particle
// writes the teeth in its cumulative-weight interval (particle j owns teeth
// [cnt(P_{j-1}), cnt(P_j)), cnt(v) = #{k : T_k < v}, T_k = offset + k *
// spacing: monotone in v and evaluated identically on both sides of every
// boundary, so the teeth partition [0, target)). Two reads of the weights,
// O(n / 4096) scratch, no n-sized prefix. Quantisation moves a tooth
// boundary by < n * 2^-60 of the total.
#ifndef HWWG_CB_ITEMS
#define HWWG_CB_ITEMS 16
#endif
constexpr int kCbThreads = 256, kCbItems = HWWG_CB_ITEMS, kCbTile = kCbThreads * kCbItems;

// scratch (8-byte words of FastCombArgs::prefix): [0] scale, [1] integer
// total, [2] spacing and [3] offset in integer units, [4] done-block counter,
// then tile sums [nt] and tile starts [nt] (uint64)
struct CbScratch {
  double* base;
  uint64_t nt;
  __device__ double& scale() const { return base[0]; }
  __device__ unsigned long long& total() const { return reinterpret_cast<unsigned long long*>(base)[1]; }
  __device__ double& spacing_i() const { return base[2]; }
  __device__ double& offset_i() const { return base[3]; }
  __device__ unsigned* done() const { return reinterpret_cast<unsigned*>(base + 4); }
  __device__ unsigned long long* tsum() const { return reinterpret_cast<unsigned long long*>(base + 8); }
  __device__ unsigned long long* tstart() const {
    return reinterpret_cast<unsigned long long*>(base + 8 + nt);
  }
};

__device__ __forceinline__ unsigned long long fixed_w(double w, double scale) {
  return w > 0.0 ? (unsigned long long)(w * scale) : 0ULL;  // truncation: monotone
}

// Block (kCbThreads) exclusive scan of one value per thread; `total` = block sum.
template <class T>
__device__ __forceinline__ T block_exclusive_256(T v, T* red, T& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T p = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += p;
  }
  __syncthreads();  // red reuse
  if (lane == 31) red[wid] = inc;
  __syncthreads();
  T before = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kCbThreads / 32; ++w) {
    if (w < wid) before += red[w];
    all += red[w];
  }
  total = all;
  return before + inc - v;
}

// Block (kCbThreads) exclusive max-scan of one value per thread (0 for thread 0).
__device__ __forceinline__ unsigned block_exclusive_max_256(unsigned v, unsigned* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned p = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = max(inc, p);
  }
  __syncthreads();  // red reuse
  if (lane == 31) red[wid] = inc;
  __syncthreads();
  unsigned before = 0;
#pragma unroll
  for (int w = 0; w < kCbThreads / 32; ++w)
    if (w < wid) before = max(before, red[w]);
  const unsigned prev = __shfl_up_sync(0xffffffffu, inc, 1);
  return max(before, lane ? prev : 0u);
}

// Is this the last block of the grid to finish? (the counter resets itself)
__device__ __forceinline__ bool last_block(unsigned* done) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(done, 1u);
    last = prev == gridDim.x - 1;
    if (last) *done = 0;
  }
  __syncthreads();
  return last;
}

// 2^s with W * (1 + 2^-10) < 2^(61 - s): the integer total stays below 2^61
__device__ __forceinline__ double comb_scale(const FastCombArgs& a) {
  double W = a.hint_host;
  for (int b = 0; b < a.hint_n; ++b) W += a.hint_batches[b];
  int e = 0;
  frexp(W > 0.0 ? W * (1.0 + 0x1p-10) : 1.0, &e);
  return ldexp(1.0, 61 - e);
}

// pass 1: integer tile sums; the last block scans them into tile starts and
// forms the comb scalars (popctrl.cpp:15-20: spacing W/target, one offset
// from the step's comb stream)
__global__ void __launch_bounds__(kCbThreads) k_cb_sums(FastCombArgs a) {
  __shared__ unsigned long long red[kCbThreads / 32];
  const CbScratch S{a.prefix, (a.n + kCbTile - 1) / kCbTile};
  const double scale = comb_scale(a);
  const uint64_t t0 = (uint64_t)blockIdx.x * kCbTile;
  unsigned long long q = 0;
  double ld[kCbItems];  // all loads in flight first
#pragma unroll
  for (int i = 0; i < kCbItems; ++i) {
    const uint64_t j = t0 + threadIdx.x + i * kCbThreads;
    ld[i] = j < a.n ? a.bank.w[j] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < kCbItems; ++i) q += fixed_w(ld[i], scale);
  unsigned long long t;
  block_exclusive_256(q, red, t);
  if (threadIdx.x == 0) S.tsum()[blockIdx.x] = t;
  if (!last_block(S.done())) return;
  const uint64_t per = (S.nt + kCbThreads - 1) / kCbThreads;
  const uint64_t lo = threadIdx.x * per < S.nt ? threadIdx.x * per : S.nt;
  const uint64_t hi = lo + per < S.nt ? lo + per : S.nt;
  unsigned long long v = 0;
  for (uint64_t i = lo; i < hi; ++i) v += S.tsum()[i];
  unsigned long long total;
  unsigned long long r = block_exclusive_256(v, red, total);
  for (uint64_t i = lo; i < hi; ++i) {
    S.tstart()[i] = r;
    r += S.tsum()[i];
  }
  if (threadIdx.x == 0) {
    S.scale() = scale;
    S.total() = total;
    const double W = (double)total / scale;
    const double spacing = W / (double)a.target;
    Xoshiro rng;
    rng.seed(a.seed, a.stream);
    const double u = rng.uniform();
    a.scalars[0] = W;
    a.scalars[1] = spacing;
    a.scalars[2] = u * spacing;
    a.scalars[3] = spacing * (double)a.target;
    const double sp_i = (double)total / (double)a.target;
    S.spacing_i() = sp_i;
    S.offset_i() = u * sp_i;
  }
}

// #{k : offset + k * spacing < v} (as ceil((v - offset) / spacing), the
// division by a multiplication with the reciprocal: a monotone function of v,
// evaluated identically on both sides of every particle boundary), clamped to
// [0, target]. (A division per boundary ran fp64 division's slow path.)
__device__ __forceinline__ uint64_t teeth_below_i(double v, double off, double inv_sp,
                                                  uint64_t target) {
  if (!(v > off)) return 0;
  const double e = ceil((v - off) * inv_sp);
  return e >= (double)target ? target : (uint64_t)e;
}

// pass 2: per tile, weights staged through shared memory, integer prefixes by
// a block scan (blocked order: thread i owns particles 16i .. 16i+15), every
// particle's tooth bound cnt(P_j) into shared memory; the tile's teeth are the
// contiguous range [cnt(tile start), cnt(tile end)), written by consecutive
// threads, each finding its source particle by binary search over the bounds
// (writing per particle diverged: with ~1 tooth per 60 particles after the
// cold start, most warps ran the write path for one lane)
// padded shared-memory indices: blocked reads (thread t, item i at 16t + i)
// and striped writes both stay free of bank conflicts
__device__ __forceinline__ int pad_d(int j) { return j + (j >> 4); }  // doubles
__device__ __forceinline__ int pad_u(int j) { return j + (j >> 5); }  // 32-bit words

__global__ void __launch_bounds__(kCbThreads) k_cb_scatter(FastCombArgs a) {
  __shared__ double wv[kCbTile + kCbTile / 16];  // weights, then the tooth bounds
  __shared__ unsigned long long red[kCbThreads / 32];
  __shared__ unsigned long long s_k0;
  const CbScratch S{a.prefix, (a.n + kCbTile - 1) / kCbTile};
  const double scale = S.scale(), inv_sp = 1.0 / S.spacing_i(), off_i = S.offset_i();
  const double spacing = a.scalars[1];
  const uint64_t t0 = (uint64_t)blockIdx.x * kCbTile;
  const int m = a.n - t0 < (uint64_t)kCbTile ? (int)(a.n - t0) : kCbTile;
  {  // all 16 loads in flight before the first use (one round trip per tile)
    double ld[kCbItems];
#pragma unroll
    for (int i = 0; i < kCbItems; ++i) {
      const int j = threadIdx.x + i * kCbThreads;
      ld[i] = j < m ? a.bank.w[t0 + j] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kCbItems; ++i) wv[pad_d(threadIdx.x + i * kCbThreads)] = ld[i];
  }
  __syncthreads();
  unsigned long long q[kCbItems];
  unsigned long long mine = 0;
#pragma unroll
  for (int i = 0; i < kCbItems; ++i) {
    q[i] = fixed_w(wv[pad_d(threadIdx.x * kCbItems + i)], scale);
    mine += q[i];
  }
  unsigned long long tot;
  const unsigned long long start = S.tstart()[blockIdx.x];
  unsigned long long run = start + block_exclusive_256(mine, red, tot);
  if (threadIdx.x == 0) s_k0 = teeth_below_i((double)start, off_i, inv_sp, a.target);
  __syncthreads();  // every weight is read: wv becomes the bound table
  const uint64_t k0 = s_k0;
  unsigned* khi = reinterpret_cast<unsigned*>(wv);  // cnt(P_j) - k0 per particle
#pragma unroll
  for (int i = 0; i < kCbItems; ++i) {
    run += q[i];
    khi[pad_u(threadIdx.x * kCbItems + i)] =
        (unsigned)(teeth_below_i((double)run, off_i, inv_sp, a.target) - k0);
  }
  __syncthreads();
  const unsigned nT = khi[pad_u(kCbTile - 1)];  // the tile's teeth (padding holds the last bound)
  // Tooth -> particle table, kCbTile teeth per round: every particle marks its
  // first tooth of the round with its index, and a block max-scan carries each
  // mark over the particle's remaining teeth (particles own consecutive,
  // ordered tooth ranges), so the writes below need no per-tooth search.
  unsigned* own = khi + pad_u(kCbTile);  // the upper half of wv, free once the bounds exist
  const double inv_w0 = a.mesh.uniform ? 1.0 / a.mesh.w0 : 0.0;
  for (unsigned R0 = 0; R0 < nT; R0 += kCbTile) {
    const unsigned R1 = nT - R0 < (unsigned)kCbTile ? nT : R0 + kCbTile;
#pragma unroll
    for (int i = 0; i < kCbItems; ++i) own[pad_u(threadIdx.x * kCbItems + i)] = 0u;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kCbItems; ++i) {
      const int j = threadIdx.x * kCbItems + i;
      if (j < m) {
        const unsigned lo = j ? khi[pad_u(j - 1)] : 0u, hi = khi[pad_u(j)];
        const unsigned first = lo > R0 ? lo : R0;
        if (first < hi && first < R1) own[pad_u(first - R0)] = (unsigned)j;
      }
    }
    __syncthreads();
    unsigned run = 0;  // blocked inclusive max-scan of the marks
    unsigned v[kCbItems];
#pragma unroll
    for (int i = 0; i < kCbItems; ++i) {
      run = max(run, own[pad_u(threadIdx.x * kCbItems + i)]);
      v[i] = run;
    }
    const unsigned before = block_exclusive_max_256(run, reinterpret_cast<unsigned*>(red));
#pragma unroll
    for (int i = 0; i < kCbItems; ++i) own[pad_u(threadIdx.x * kCbItems + i)] = max(v[i], before);
    __syncthreads();
    // teeth of the round, 4 per thread in flight (their particles' loads first)
    for (unsigned r0 = R0 + threadIdx.x; r0 < R1; r0 += 4 * kCbThreads) {
      double2 xm[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned r = r0 + q * kCbThreads;
        if (r < R1) {
          const unsigned j = own[pad_u(r - R0)];
          HWWG_CHECK((int)j < m && khi[pad_u(j)] > r && (j == 0 || khi[pad_u(j - 1)] <= r));
          xm[q] = a.bank.xm[t0 + j];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned r = r0 + q * kCbThreads;
        if (r < R1) write_tooth(a, xm[q], k0 + r, spacing, inv_w0);
      }
    }
    __syncthreads();  // the table is rebuilt for the next round
  }
  // teeth stranded past the integer total by round-off go to the last particle
  // with weight (popctrl.cpp:31-37)
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kCbThreads - 1) {
    const uint64_t k_end = teeth_below_i((double)S.total(), off_i, inv_sp, a.target);
    if (k_end < a.target) {
      uint64_t src = a.n - 1;
      while (src > 0 && !(fixed_w(a.bank.w[src], scale) > 0)) --src;
      write_teeth(a, src, k_end, a.target, spacing);
    }
  }
}

struct WeightOf {
  __host__ __device__ double operator()(const double2& v) const { return v.x; }
};

__global__ void k_local_total(const double* prefix, uint64_t n, double* sc) {
  sc[0] = n ? prefix[n - 1] : 0.0;
}

__global__ void k_comb_teeth_range(FastCombArgs a, double spacing, double offset, double origin,
                                   uint64_t k_lo, uint64_t k_hi, FastBank out) {
  const uint64_t k = k_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k_hi) return;
  const double T = offset + (double)k * spacing;
  uint64_t lo = 0, hi = a.n;  // first local particle with T < origin + prefix
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (T < origin + a.prefix[mid]) hi = mid;
    else lo = mid + 1;
  }
  uint64_t s = lo < a.n ? lo : a.n - 1;
  if (lo >= a.n)
    while (s > 0 && a.bank.w[s] <= 0.0) --s;
  const uint64_t o = k - k_lo;
  const double2 xm = a.bank.xm[s];
  const int c = locate_cell(a.mesh, xm.x);
  out.xm[o] = xm;
  out.wt[o] = make_double2(spacing, a.t_bank);
  out.meta[o] = make_uint4((unsigned)(c < 0 ? 0 : c), (unsigned)k, 0u, 0u);
}

__global__ void k_fast_permute(FastBank in, FastBank out, uint64_t n, Perm perm, PieceTable t) {
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const uint64_t s = perm(c);
  HWWG_CHECK(s < n);
  uint64_t g = c, rem = c;  // global id of local slot c
  for (int i = 0; i < t.n; ++i) {
    if (rem < t.cnt[i]) {
      g = t.lo[i] + rem;
      break;
    }
    rem -= t.cnt[i];
  }
  out.xm[c] = in.xm[s];
  out.wt[c] = in.wt[s];
  out.meta[c] = make_uint4(in.meta[s].x & 0xffffu, (unsigned)g, 0u, 0u);
}

// one warp per transport warp's chunk tail (<= kCensusChunk slots), lanes in parallel
__global__ void k_fill_holes(CensusBank c, uint64_t cap, const unsigned long long* cur, int warps,
                             double x_fill) {
  const int w = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= warps) return;
  const unsigned long long end = cur[2 * w + 1] < cap ? cur[2 * w + 1] : cap;
  for (unsigned long long s = cur[2 * w] + lane; s < end; s += 32) {
    c.xm[s] = make_double2(x_fill, 0.5);
    c.w[s] = 0.0;
  }
}

// Drop zero-weight holes while converting to AoS (order is free in this mode).
__global__ void k_compact_aos(CensusBank in, uint64_t n, double t, hwwg_particle* out,
                              unsigned long long* count) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool keep = i < n && in.w[i] > 0.0;
  const unsigned mask = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0 && mask) base = atomicAdd(count, (unsigned long long)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) {
    const unsigned long long j = base + __popc(mask & ((1u << lane) - 1u));
    double2* o = reinterpret_cast<double2*>(out) + 2 * j;
    o[0] = in.xm[i];
    o[1] = make_double2(in.w[i], t);
  }
}

__global__ void k_aos_to_census(const hwwg_particle* __restrict__ in, uint64_t n, CensusBank out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 a = reinterpret_cast<const double2*>(in)[2 * i];
  const double2 b = reinterpret_cast<const double2*>(in)[2 * i + 1];
  out.xm[i] = a;
  out.w[i] = b.x;
}

// The pulse as a census bank from its directions alone (e2e host round trip:
// every pulse particle shares x0, w0 and t = 0, so only mu crosses PCIe).
__global__ void k_mu_to_census(const double* __restrict__ mu, uint64_t n, double x0, double w0,
                               CensusBank out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out.xm[i] = make_double2(x0, mu[i]);
  out.w[i] = w0;
}

// The throughput step's start in one launch (instead of four memsets and a
// reset kernel, each of which serialised the launch pipeline): zero the tally
// slab and the warps' census cursors, the census counter and the error word,
// and reset the first segment's pool counters.
__global__ void k_step_start(double* slab, size_t slab_words, unsigned long long* cursor,
                             size_t cursor_words, unsigned long long* counter, DevError* err,
                             unsigned long long* ctl, unsigned long long* src_head,
                             unsigned long long* span) {
  const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = i0; i < slab_words; i += stride) slab[i] = 0.0;
  for (size_t i = i0; i < cursor_words; i += stride) cursor[i] = 0ULL;
  if (i0 == 0) {
    *counter = 0ULL;
    err->code = 0;
    err->pad = 0;
    err->history = 0ULL;
    fast_pool_reset(ctl, src_head, span);
  }
}

__global__ void k_track_from_batches(TallyPtrs t, int I, int B) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I) return;
  double s = 0.0;
  for (int b = 0; b < B; ++b) s += t.track_flux_batch[(size_t)b * I + i];
  t.track_flux[i] = s;
}

__global__ void k_fast_to_aos_packed(FastBank in, uint64_t n, uint64_t n_packed, const double* w0,
                                     double t0, hwwg_particle* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2* o = reinterpret_cast<double2*>(out) + 2 * i;
  o[0] = in.xm[i];
  o[1] = i < n_packed ? make_double2(*w0, t0) : in.wt[i];
}

__global__ void k_fill_wt(double2* wt, uint64_t n, const double* w0, double t0) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) wt[i] = make_double2(*w0, t0);
}

__global__ void k_fast_to_aos(FastBank in, uint64_t n, hwwg_particle* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2* o = reinterpret_cast<double2*>(out) + 2 * i;
  o[0] = in.xm[i];
  o[1] = in.wt[i];
}

// e2e host round trip, packed wire format: a combed bank carries one (w, t)
// pair for every particle (w = the comb spacing, t = the census time), so only
// (x, mu) crosses PCIe. The check flags a bank where that does not hold.
__global__ void k_check_uniform(const double2* __restrict__ wt, uint64_t n, unsigned* flag,
                                double2* first) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 v = wt[i], f = wt[0];
  if (i == 0) *first = f;
  if (v.x != f.x || v.y != f.y) *flag = 1u;
}

// (x, mu) from the host into the SoA bank: cell, identity, and (w, t) when the
// host bank was packed uniform.
__global__ void k_xm_to_fast(FastBank out, uint64_t n, const MeshView m, uint64_t hist0,
                             int uniform, double w0, double t0, PieceTable pieces) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = out.xm[i].x;
  if (uniform) out.wt[i] = make_double2(w0, t0);
  const int c = locate_cell(m, x);
  uint64_t g = hist0 + i;  // history: hist0 + i, or the rank's i-th owned id (pieces)
  if (pieces.n) {
    uint64_t rem = i;
    for (int k = 0; k < pieces.n; ++k) {
      if (rem < pieces.cnt[k]) {
        g = pieces.lo[k] + rem;
        break;
      }
      rem -= pieces.cnt[k];
    }
  }
  out.meta[i] = make_uint4((unsigned)(c < 0 ? 0 : c), (unsigned)g, 0u, 0u);
}

// Config-3 volumetric source on the device (Philox mode; DESIGN.md "Config-3
// features"): particle j of the step's box emission gets x ~ U[x_lo, x_hi],
// t ~ U[ta, tb], mu ~ U(-1, 1) from two Philox blocks keyed by (seed ^ a source
// constant; j, step) — a stream no transport event uses — weight w, history
// hist0 + i.  j = j0 + i: any rank samples any slice of the same emission.
__global__ void k_volume_source(FastBank out, uint64_t n, uint64_t j0, uint64_t hist0,
                                const MeshView m, unsigned k0, unsigned k1, unsigned step,
                                double x_lo, double x_hi, double ta, double tb, double w) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t j = j0 + i;
  const unsigned sk0 = k0 ^ 0x3c6ef372u, sk1 = k1 ^ 0xa54ff53au;
  double ux, ut, umu, unused;
  philox_uniform2(philox4x32_10(U4{(unsigned)j, (unsigned)(j >> 32), step, 0u}, sk0, sk1), ux, ut);
  philox_uniform2(philox4x32_10(U4{(unsigned)j, (unsigned)(j >> 32), step, 1u}, sk0, sk1), umu,
                  unused);
  const double x = x_lo + (x_hi - x_lo) * ux;
  const double t = ta + (tb - ta) * ut;
  const double mu = 2.0 * umu - 1.0;
  const int c = locate_cell(m, x);
  out.xm[i] = make_double2(x, mu);
  out.wt[i] = make_double2(w, t);
  out.meta[i] = make_uint4((unsigned)(c < 0 ? 0 : c), (unsigned)(hist0 + i), 0u, 0u);
}

}  // namespace

void launch_volume_source(FastBank out, uint64_t n, uint64_t j0, uint64_t hist0, const MeshView& m,
                          unsigned k0, unsigned k1, unsigned step, double x_lo, double x_hi,
                          double ta, double tb, double w, cudaStream_t s) {
  if (!n) return;
  k_volume_source<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, n, j0, hist0, m, k0, k1, step,
                                                              x_lo, x_hi, ta, tb, w);
  HWWG_CUDA(cudaGetLastError());
}

void launch_check_uniform(const double2* wt, uint64_t n, unsigned* flag, double2* first,
                          cudaStream_t s) {
  HWWG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), s));
  if (!n) return;
  k_check_uniform<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(wt, n, flag, first);
  HWWG_CUDA(cudaGetLastError());
}

void launch_xm_to_fast(FastBank out, uint64_t n, const MeshView& m, uint64_t hist0, int uniform,
                       double w0, double t0, cudaStream_t s, const PieceTable* pieces) {
  if (!n) return;
  PieceTable t{};
  if (pieces) t = *pieces;
  k_xm_to_fast<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, n, m, hist0, uniform, w0, t0, t);
  HWWG_CUDA(cudaGetLastError());
}

using WeightIt = cub::TransformInputIterator<double, WeightOf, const double2*>;

size_t fast_comb_temp_bytes(uint64_t n) {
  size_t bytes = 0, b2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, (const double*)nullptr, (double*)nullptr, (int)n);
  cub::DeviceScan::InclusiveSum(nullptr, b2, WeightIt(nullptr, WeightOf()), (double*)nullptr, (int)n);
  return bytes > b2 ? bytes : b2;
}

size_t fast_comb_scratch_words(uint64_t n) { return 8 + 2 * ((n + kCbTile - 1) / kCbTile) + 8; }

void launch_fast_comb(const FastCombArgs& a, cudaStream_t s) {
  const unsigned nt = (unsigned)((a.n + kCbTile - 1) / kCbTile);
  HWWG_CUDA(cudaMemsetAsync(a.prefix + 4, 0, sizeof(double), s));  // done-block counter
  k_cb_sums<<<nt, kCbThreads, 0, s>>>(a);  // + tile starts, scalars (last block)
  k_cb_scatter<<<nt, kCbThreads, 0, s>>>(a);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_comb_local_scan(const FastCombArgs& a, cudaStream_t s) {
  if (a.n) {
    k_extract_w<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a.bank, a.n, a.prefix);
    size_t bytes = a.temp_bytes;
    HWWG_CUDA(cub::DeviceScan::InclusiveSum(a.temp, bytes, a.prefix, a.prefix, (int)a.n, s));
  }
  k_local_total<<<1, 1, 0, s>>>(a.prefix, a.n, a.scalars);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_comb_teeth_range(const FastCombArgs& a, double spacing, double offset,
                                  double origin, uint64_t k_lo, uint64_t k_hi, FastBank out,
                                  cudaStream_t s) {
  const uint64_t n = k_hi - k_lo;
  if (!n || !a.n) return;
  k_comb_teeth_range<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, spacing, offset, origin,
                                                                 k_lo, k_hi, out);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_permute(FastBank in, FastBank out, uint64_t n, Perm perm, const PieceTable& t,
                         cudaStream_t s) {
  if (!n) return;
  k_fast_permute<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, out, n, perm, t);
  HWWG_CUDA(cudaGetLastError());
}

static uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    const uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

Perm make_perm(uint64_t n, uint64_t seed, uint64_t step) {
  const uint64_t nt = n >> 5;  // whole 32-element tiles
  if (nt < 3) return Perm{0, 0, 0, 0};
  uint64_t a = (uint64_t)((double)nt * 0.6180339887498949);
  if (a < 1) a = 1;
  while (gcd_u64(a, nt) != 1) ++a;  // a few steps at most (coprimes are dense)
  uint64_t z = seed ^ (step * 0x9E3779B97F4A7C15ULL);  // splitmix64 of (seed, step): the offset
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  const unsigned long long m = (unsigned long long)(((unsigned __int128)1 << 64) / nt);
  return Perm{nt, a % nt, z % nt, m};
}

void launch_fill_census_holes(CensusBank census, uint64_t cap,
                              const unsigned long long* warp_cursor, int warps, double x_fill,
                              cudaStream_t s) {
  k_fill_holes<<<(warps + 7) / 8, 256, 0, s>>>(census, cap, warp_cursor, warps, x_fill);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_compact_aos(CensusBank in, uint64_t n, double t, hwwg_particle* out,
                             unsigned long long* count, cudaStream_t s) {
  HWWG_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned long long), s));
  if (!n) return;
  k_compact_aos<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, n, t, out, count);
  HWWG_CUDA(cudaGetLastError());
}

void launch_mu_to_census(const double* mu, uint64_t n, double x0, double w0, CensusBank out,
                         cudaStream_t s) {
  if (!n) return;
  k_mu_to_census<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(mu, n, x0, w0, out);
  HWWG_CUDA(cudaGetLastError());
}

void launch_aos_to_census(const hwwg_particle* in, uint64_t n, CensusBank out, cudaStream_t s) {
  if (!n) return;
  k_aos_to_census<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, n, out);
  HWWG_CUDA(cudaGetLastError());
}

void launch_step_start(double* slab, size_t slab_words, unsigned long long* cursor,
                       size_t cursor_words, unsigned long long* counter, DevError* err,
                       unsigned long long* ctl, unsigned long long* src_head,
                       unsigned long long* span, int sms, cudaStream_t s) {
  k_step_start<<<2 * sms, 256, 0, s>>>(slab, slab_words, cursor, cursor_words, counter, err, ctl,
                                       src_head, span);
  HWWG_CUDA(cudaGetLastError());
}

void launch_track_from_batches(TallyPtrs t, int I, int B, cudaStream_t s) {
  k_track_from_batches<<<(I + 255) / 256, 256, 0, s>>>(t, I, B);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_to_aos_packed(FastBank in, uint64_t n, uint64_t n_packed, const double* w0,
                               double t0, hwwg_particle* out, cudaStream_t s) {
  if (!n) return;
  k_fast_to_aos_packed<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, n, n_packed, w0, t0, out);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fill_wt(double2* wt, uint64_t n, const double* w0, double t0, cudaStream_t s) {
  if (!n) return;
  k_fill_wt<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(wt, n, w0, t0);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_to_aos(FastBank in, uint64_t n, hwwg_particle* out, cudaStream_t s) {
  if (!n) return;
  k_fast_to_aos<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, n, out);
  HWWG_CUDA(cudaGetLastError());
}

}  // namespace hwwg
