// Throughput-mode bank kernels: the parallel comb (population control at step
// start, proj/src/popctrl.cpp:7-42) and bank format conversions.
//
// The comb keeps the reference's estimator — teeth spaced W/target apart with
// one random offset walk the cumulative-weight axis of the bank — but the
// cumulative weights come from a parallel scan (CUB fp64 scan into an n-sized
// prefix; exact fixed-point integers in tiles, with O(n/2048) scratch, for
// banks beyond the preallocated prefix) instead of a serial walk, and each
// particle writes the teeth that fall in its cumulative-weight interval.
// Teeth land in bank order.
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "common.cuh"
#include "fast.cuh"
#include "rng.cuh"

namespace hwwg {

namespace {

__global__ void k_extract_w(FastBank b, uint64_t n, double* w) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = b.wt[i].x;
}

// Particle-parallel teeth: particle i owns the teeth k with
// prefix[i-1] <= T_k < prefix[i], T_k = offset + k * spacing — exactly the
// teeth whose first index with T_k < prefix[idx] is i (the search definition),
// since cnt(v) = #{k : T_k < v} is evaluated with the same fp64 T_k on both
// sides of every boundary. Reads and writes are coalesced and there is no
// search; teeth stranded past the total by round-off go to the last particle
// with weight (popctrl.cpp:31-37).
__device__ __forceinline__ uint64_t teeth_below(double v, double offset, double spacing,
                                                uint64_t target) {
  double e = ceil((v - offset) / spacing);
  uint64_t k = e <= 0.0 ? 0 : (e >= (double)target ? target : (uint64_t)e);
  while (k > 0 && !(offset + (double)(k - 1) * spacing < v)) --k;
  while (k < target && offset + (double)k * spacing < v) ++k;
  return k;
}

__device__ __forceinline__ void write_teeth(const FastCombArgs& a, uint64_t src, uint64_t k0,
                                            uint64_t k1, double spacing) {
  const double2 xm = a.bank.xm[src];
  const double2 wt = a.bank.wt[src];
  const uint4 m = a.bank.meta[src];
  for (uint64_t k = k0; k < k1; ++k) {
    const uint64_t p = a.perm(k);
    a.out.xm[p] = xm;
    a.out.wt[p] = make_double2(spacing, wt.y);
    // fresh identity for the new step: history = its slot, key 0, draw 0
    a.out.meta[p] = make_uint4(m.x & 0xffffu, (unsigned)p, 0u, 0u);
  }
}

// popctrl.cpp:15-20 comb scalars (W, spacing, the offset drawn from the
// step's comb stream, the output weight), formed by every block from the
// scan's last prefix (the same values everywhere); block 0 records them.
__device__ __forceinline__ void comb_scalars(const FastCombArgs& a, double& spacing,
                                             double& offset) {
  __shared__ double sc[2];
  if (threadIdx.x == 0) {
    const double W = a.prefix[a.n - 1];
    const double sp = W / (double)a.target;
    Xoshiro r;
    r.seed(a.seed, a.stream);
    const double off = r.uniform() * sp;
    sc[0] = sp;
    sc[1] = off;
    if (blockIdx.x == 0) {
      a.scalars[0] = W;
      a.scalars[1] = sp;
      a.scalars[2] = off;
      a.scalars[3] = sp * (double)a.target;
    }
  }
  __syncthreads();
  spacing = sc[0];
  offset = sc[1];
}

__global__ void k_comb_scatter(FastCombArgs a) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double spacing, offset;
  comb_scalars(a, spacing, offset);
  if (i >= a.n) return;
  const uint64_t k0 = i ? teeth_below(a.prefix[i - 1], offset, spacing, a.target) : 0;
  const uint64_t k1 = teeth_below(a.prefix[i], offset, spacing, a.target);
  if (k0 < k1) write_teeth(a, i, k0, k1, spacing);
  if (i == a.n - 1 && k1 < a.target) {  // stranded teeth
    uint64_t s = i;
    while (s > 0 && a.bank.wt[s].x <= 0.0) --s;
    write_teeth(a, s, k1, a.target, spacing);
  }
}

// ---- single-GPU comb without an n-sized prefix (memory-wall banks) ---------
// The cumulative weights are exact integers: every weight becomes
// floor(w * 2^k) (k chosen so the bank total stays below 2^62), tiles of 2048
// sum and scan in uint64, so prefixes are associative, monotone and identical
// on both sides of every tile boundary — each particle recomputes its own
// prefix in its tile's block scan and writes its teeth. Scratch is O(n/2048)
// words instead of 8 B per census slot (the step-1 census of config 4 is 1.9e9
// particles). Quantisation moves a tooth boundary by < n * 2^-62 of the total.
constexpr int kFcThreads = 256, kFcItems = 8, kFcTile = kFcThreads * kFcItems;

// scratch layout (8-byte words): [0] scale, [1] integer total, [2] spacing in
// integer units, [3] offset in integer units, [4] done-block counter, then tile
// sums (fp64) [nt], tile integer sums [nt], tile integer starts [nt]
struct FcScratch {
  double* base;
  uint64_t nt;
  __device__ double& scale() const { return base[0]; }
  __device__ unsigned long long& total() const { return reinterpret_cast<unsigned long long*>(base)[1]; }
  __device__ double& spacing_i() const { return base[2]; }
  __device__ double& offset_i() const { return base[3]; }
  __device__ unsigned* done() const { return reinterpret_cast<unsigned*>(base + 4); }
  __device__ double* fsum() const { return base + 5; }
  __device__ unsigned long long* isum() const { return reinterpret_cast<unsigned long long*>(base + 5 + nt); }
  __device__ unsigned long long* istart() const {
    return reinterpret_cast<unsigned long long*>(base + 5 + 2 * nt);
  }
};

__device__ __forceinline__ unsigned long long fixed_w(double w, double scale) {
  return w > 0.0 ? (unsigned long long)(w * scale) : 0ULL;  // truncation: monotone
}

// Block (kFcThreads) exclusive scan of one value per thread; returns the
// thread's exclusive prefix, `total` the block sum (all threads).
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
  for (int w = 0; w < kFcThreads / 32; ++w) {
    if (w < wid) before += red[w];
    all += red[w];
  }
  total = all;
  return before + inc - v;
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

// pass 1 (kInteger = false): fp64 tile sums, then the last block derives the
// fixed-point scale from their total; pass 2: integer tile sums, then the last
// block scans them into tile starts and writes the comb scalars.
template <bool kInteger>
__global__ void __launch_bounds__(kFcThreads) k_fc_tile_sums(FastCombArgs a) {
  __shared__ double fred[kFcThreads / 32];
  __shared__ unsigned long long ired[kFcThreads / 32];
  const FcScratch S{a.prefix, (a.n + kFcTile - 1) / kFcTile};
  const uint64_t k0 = (uint64_t)blockIdx.x * kFcTile;
  const double scale = kInteger ? S.scale() : 0.0;
  double f = 0.0;
  unsigned long long q = 0;
  for (int j = threadIdx.x; j < kFcTile; j += kFcThreads) {
    const uint64_t k = k0 + j;
    if (k < a.n) {
      const double w = a.bank.wt[k].x;
      if (kInteger) q += fixed_w(w, scale);
      else f += w > 0.0 ? w : 0.0;
    }
  }
  if (kInteger) {
    unsigned long long t;
    block_exclusive_256(q, ired, t);
    if (threadIdx.x == 0) S.isum()[blockIdx.x] = t;
  } else {
    double t;
    block_exclusive_256(f, fred, t);
    if (threadIdx.x == 0) S.fsum()[blockIdx.x] = t;
  }
  if (!last_block(S.done())) return;
  // the last block: every tile sum is visible (fence + counter)
  const uint64_t per = (S.nt + kFcThreads - 1) / kFcThreads;
  const uint64_t lo = threadIdx.x * per < S.nt ? threadIdx.x * per : S.nt;
  const uint64_t hi = lo + per < S.nt ? lo + per : S.nt;
  if (!kInteger) {
    double v = 0.0;
    for (uint64_t t = lo; t < hi; ++t) v += S.fsum()[t];
    double W;
    block_exclusive_256(v, fred, W);
    if (threadIdx.x == 0) {
      // total * scale < 2^62 with room for the fp64 sum's own rounding
      int e = 0;
      frexp(W > 0.0 ? W * (1.0 + 0x1p-20) : 1.0, &e);
      S.scale() = ldexp(1.0, 62 - e);
      a.scalars[0] = W;
    }
    return;
  }
  unsigned long long v = 0;
  for (uint64_t t = lo; t < hi; ++t) v += S.isum()[t];
  unsigned long long r_total;
  unsigned long long r = block_exclusive_256(v, ired, r_total);
  for (uint64_t t = lo; t < hi; ++t) {
    S.istart()[t] = r;
    r += S.isum()[t];
  }
  if (threadIdx.x == 0) {
    S.total() = r_total;
    const double W = a.scalars[0];
    const double spacing = W / (double)a.target;
    Xoshiro rng;
    rng.seed(a.seed, a.stream);
    const double u = rng.uniform();
    a.scalars[1] = spacing;
    a.scalars[2] = u * spacing;
    a.scalars[3] = spacing * (double)a.target;
    const double sp_i = (double)r_total / (double)a.target;
    S.spacing_i() = sp_i;
    S.offset_i() = u * sp_i;
  }
}

// Per tile: weights staged through shared memory, exact integer prefixes by a
// block scan (blocked order), then the teeth written particle-parallel in
// striped order so consecutive lanes write consecutive teeth.
__global__ void __launch_bounds__(kFcThreads) k_fc_scatter(FastCombArgs a) {
  __shared__ double wv[kFcTile];
  __shared__ unsigned long long P[kFcTile];
  __shared__ unsigned long long red[kFcThreads / 32];
  const FcScratch S{a.prefix, (a.n + kFcTile - 1) / kFcTile};
  const double scale = S.scale(), sp_i = S.spacing_i(), off_i = S.offset_i();
  const double spacing = a.scalars[1];
  const uint64_t t0 = (uint64_t)blockIdx.x * kFcTile;
  const int m = a.n - t0 < (uint64_t)kFcTile ? (int)(a.n - t0) : kFcTile;
  for (int j = threadIdx.x; j < kFcTile; j += kFcThreads) wv[j] = j < m ? a.bank.wt[t0 + j].x : 0.0;
  __syncthreads();
  unsigned long long q[kFcItems];
  unsigned long long mine = 0;
#pragma unroll
  for (int i = 0; i < kFcItems; ++i) {
    q[i] = fixed_w(wv[threadIdx.x * kFcItems + i], scale);
    mine += q[i];
  }
  unsigned long long tot;
  unsigned long long run = S.istart()[blockIdx.x] + block_exclusive_256(mine, red, tot);
#pragma unroll
  for (int i = 0; i < kFcItems; ++i) {
    run += q[i];
    P[threadIdx.x * kFcItems + i] = run;  // inclusive
  }
  __syncthreads();
  const unsigned long long start = S.istart()[blockIdx.x];
  for (int j = threadIdx.x; j < m; j += kFcThreads) {
    const uint64_t k = t0 + j;
    const uint64_t lo = teeth_below((double)(j ? P[j - 1] : start), off_i, sp_i, a.target);
    const uint64_t hi = teeth_below((double)P[j], off_i, sp_i, a.target);
    if (lo < hi) write_teeth(a, k, lo, hi, spacing);
    if (k == a.n - 1 && hi < a.target) {  // stranded teeth (popctrl.cpp:31-37)
      uint64_t src = k;
      while (src > 0 && !(fixed_w(a.bank.wt[src].x, scale) > 0)) --src;
      write_teeth(a, src, hi, a.target, spacing);
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
    while (s > 0 && a.bank.wt[s].x <= 0.0) --s;
  const uint64_t o = k - k_lo;
  out.xm[o] = a.bank.xm[s];
  out.wt[o] = make_double2(spacing, a.bank.wt[s].y);
  out.meta[o] = make_uint4(a.bank.meta[s].x & 0xffffu, (unsigned)k, 0u, 0u);
}

__global__ void k_fast_permute(FastBank in, FastBank out, uint64_t n, Perm perm, PieceTable t) {
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const uint64_t s = perm(c);
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
__global__ void k_fill_holes(FastBank c, uint64_t cap, const unsigned long long* cur, int warps,
                             double x_fill, double t_fill) {
  const int w = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= warps) return;
  const unsigned long long end = cur[2 * w + 1] < cap ? cur[2 * w + 1] : cap;
  for (unsigned long long s = cur[2 * w] + lane; s < end; s += 32) {
    c.xm[s] = make_double2(x_fill, 0.5);
    c.wt[s] = make_double2(0.0, t_fill);
    c.meta[s] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// Drop zero-weight holes while converting to AoS (order is free in this mode).
__global__ void k_compact_aos(FastBank in, uint64_t n, hwwg_particle* out,
                              unsigned long long* count) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool keep = i < n && in.wt[i].x > 0.0;
  const unsigned mask = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0 && mask) base = atomicAdd(count, (unsigned long long)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) {
    const unsigned long long j = base + __popc(mask & ((1u << lane) - 1u));
    double2* o = reinterpret_cast<double2*>(out) + 2 * j;
    o[0] = in.xm[i];
    o[1] = in.wt[i];
  }
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
                             int uniform, double w0, double t0) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = out.xm[i].x;
  if (uniform) out.wt[i] = make_double2(w0, t0);
  const int c = locate_cell(m, x);
  out.meta[i] = make_uint4((unsigned)(c < 0 ? 0 : c), (unsigned)(hist0 + i), 0u, 0u);
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
                       double w0, double t0, cudaStream_t s) {
  if (!n) return;
  k_xm_to_fast<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, n, m, hist0, uniform, w0, t0);
  HWWG_CUDA(cudaGetLastError());
}

using WeightIt = cub::TransformInputIterator<double, WeightOf, const double2*>;

size_t fast_comb_temp_bytes(uint64_t n) {
  size_t bytes = 0, b2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, (const double*)nullptr, (double*)nullptr, (int)n);
  cub::DeviceScan::InclusiveSum(nullptr, b2, WeightIt(nullptr, WeightOf()), (double*)nullptr, (int)n);
  return bytes > b2 ? bytes : b2;
}

size_t fast_comb_scratch_words(uint64_t n) { return 5 + 3 * ((n + kFcTile - 1) / kFcTile) + 4; }

void launch_fast_comb(const FastCombArgs& a, cudaStream_t s) {
  // inclusive fp64 scan of the weights straight from the SoA bank (n-sized prefix)
  size_t bytes = a.temp_bytes;
  HWWG_CUDA(cub::DeviceScan::InclusiveSum(a.temp, bytes, WeightIt(a.bank.wt, WeightOf()), a.prefix,
                                          (int)a.n, s));
  k_comb_scatter<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_comb_tiled(const FastCombArgs& a, cudaStream_t s) {
  const unsigned nt = (unsigned)((a.n + kFcTile - 1) / kFcTile);
  HWWG_CUDA(cudaMemsetAsync(a.prefix + 4, 0, sizeof(double), s));  // done-block counter
  k_fc_tile_sums<false><<<nt, kFcThreads, 0, s>>>(a);  // + the scale (last block)
  k_fc_tile_sums<true><<<nt, kFcThreads, 0, s>>>(a);   // + tile starts, scalars
  k_fc_scatter<<<nt, kFcThreads, 0, s>>>(a);
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
  if (nt < 3) return Perm{0, 0, 0};
  uint64_t a = (uint64_t)((double)nt * 0.6180339887498949);
  if (a < 1) a = 1;
  while (gcd_u64(a, nt) != 1) ++a;  // a few steps at most (coprimes are dense)
  uint64_t z = seed ^ (step * 0x9E3779B97F4A7C15ULL);  // splitmix64 of (seed, step): the offset
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return Perm{nt, a % nt, z % nt};
}

void launch_fill_census_holes(FastBank census, uint64_t cap, const unsigned long long* warp_cursor,
                              int warps, double x_fill, double t_fill, cudaStream_t s) {
  k_fill_holes<<<(warps + 7) / 8, 256, 0, s>>>(census, cap, warp_cursor, warps, x_fill, t_fill);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_compact_aos(FastBank in, uint64_t n, hwwg_particle* out,
                             unsigned long long* count, cudaStream_t s) {
  HWWG_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned long long), s));
  if (!n) return;
  k_compact_aos<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, n, out, count);
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

void launch_fast_to_aos(FastBank in, uint64_t n, hwwg_particle* out, cudaStream_t s) {
  if (!n) return;
  k_fast_to_aos<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, n, out);
  HWWG_CUDA(cudaGetLastError());
}

}  // namespace hwwg
