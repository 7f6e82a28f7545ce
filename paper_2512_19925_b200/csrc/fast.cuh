// Throughput (Philox) mode: SoA particle bank, transport and comb interfaces.
#pragma once

#include "common.cuh"

namespace hwwg {

// 48 B per particle, three 128-bit words.
struct FastBank {
  double2* xm;  // {x, mu}
  double2* wt;  // {w, t}
  uint4* meta;  // {cell | draw << 16, history, lineage key lo, lineage key hi}
};

// Census bank (the transport's output, the next comb's input): 24 B per
// particle. Every census particle sits at t = t_end of its step and is located
// again from x when it next moves (mesh.cpp:26-40, as advance_history does at
// a history's start), so only (x, mu) and w are kept — half the 48 B source
// record, in the largest buffers of a run (the x63 cold-start census).
struct CensusBank {
  double2* xm;  // {x, mu}
  double* w;
};

// One run-length-encoded split record (72 B): `count` identical daughters.
struct FastStackRec {
  double x, mu, w, t;
  unsigned cell, hist;
  unsigned long long key;
  unsigned ctr, count;  // daughters base+1 .. base+count remain
  unsigned ready, base;  // ready: set last when the record sits in the global pool
  double inv_mu;  // 1 / mu, carried so a popped daughter needs no division
};

// Global pool of split records shared by all warps of a segment kernel (load
// balance for heavy split trees) plus the termination counter.
struct FastPool {
  FastStackRec* recs;
  unsigned long long* ctl;  // [0] tail (reserved), [1] head (claimed), [2] active warps
  unsigned cap;
  unsigned warps;  // warps in the grid
};

// Pool counter reset before a transport launch, independent of its grid:
// active warps = kPoolSentinel (the kernel's first thread swaps in its warp
// count), source claims counted from the end of the static reservations.
constexpr unsigned long long kPoolSentinel = 1ULL << 40;
// span (nullable): the launch's [first block start, last block end] in
// globaltimer ns, reset to [~0, 0] here and stamped by the transport blocks
__device__ __forceinline__ void fast_pool_reset(unsigned long long* ctl,
                                                unsigned long long* src_head,
                                                unsigned long long* span) {
  if (span) {
    span[0] = ~0ULL;
    span[1] = 0ULL;
  }
  ctl[0] = 0;
  ctl[1] = 0;
  ctl[2] = kPoolSentinel;  // every warp starts active (holding source work)
  ctl[3] = 0;              // no backlog declared yet
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  ctl[4] = t;  // segment start (diagnostics)
  *src_head = 0;
}

// Dynamic shared-memory layout of the transport kernel, in doubles from its
// base (filled by launch_fast_segment): the track counts at 0, the tally
// histograms, then the window centres and the mesh edges. Passed precomputed so
// the event loop's address arithmetic takes constant-bank operands instead of
// re-deriving the layout from I and nb (the compiler rematerialises it under
// register pressure).
struct SmemOffsets {
  unsigned trk, cphi, cJ, cF, edge, cwb, bclo, cent, edgex;
};

struct FastArgs {
  FastBank src;  // this segment's source particles
  unsigned long long n_src;
  // Source slots [0, n_packed) are comb teeth stored as (x, mu) alone (the
  // comb's packed output): weight *src_w0 (the comb spacing, in device
  // memory), time src_t0, cell located from x, history src_hist0 + slot,
  // lineage key 0, draw 0. Slots from n_packed on are full records.
  unsigned long long n_packed;
  const double* src_w0;
  double src_t0, inv_w0;
  unsigned src_hist0;
  unsigned long long* src_head;  // refill cursor (zeroed per segment)
  CensusBank census;
  unsigned long long* census_count;
  uint64_t census_cap;
  MeshView mesh;
  double t_end, inv_dt;
  unsigned k0, k1, step;  // Philox key (seed) and step
  unsigned rk[20];        // the key's round keys (philox_round_keys)
  uint64_t H;
  int B;
  double bmul;  // B / H (batch_of without a division)
  int b_lo, nb;  // batches touched by this segment: [b_lo, b_lo + nb)
  int smem_tallies;  // 0 global REDs, 1 shared-memory tallies, 2 fp64 global + counts shared
  int aggregate;     // 1: warp-aggregate tally atomics (cold start: lanes share cells)
  int census_runs;   // fixed-point slots: 1 run-aggregates census scores (cold start)
  int scramble;      // 1: claim source particles in bit-reversed order within 1024-blocks
  // 1: fixed-point track/edge tallies in shared memory (smem_tallies == 1, no
  // aggregation): scores on the grid 2^-fix_k_* (fast_fix_exponent)
  int fix, fix_k_trk, fix_k_edge, fix_k_cw;  // ... census weight by batch on 2^-fix_k_cw
  // t_win = 1 (with fix): the fixed-point histograms cover cells [t_lo, t_lo +
  // t_n) only (the step's particles' reach, config 4); other scores go to the
  // global tallies with fp64 REDs
  int t_win, t_lo, t_n;
  // set by launch_fast_segment: the grid scales 2^fix_k_* and the carry sweep's
  // slot count and slots per lane
  double fix_s_trk, fix_s_edge, fix_s_cw;
  unsigned fix_slots, fix_spl;
  int warps;            // warps per block: 12 (2 blocks per SM) or 24 (1 block per SM)
  int pool_reset_done;  // 1: the kernel before this launch reset the pool counters
  int pdl;              // 1: programmatic dependent launch after the previous kernel
  // [first block start, last block end] (globaltimer ns) of this launch, reset
  // with the pool counters: the transport time without per-launch CUDA events
  // (events between the segment kernels serialised the launch pipeline: -4%)
  unsigned long long* span;
  // 1 (the step's last segment, whose grid holds every warp with a census
  // chunk): each warp writes zero-weight records (x_fill, t_fill) into the
  // unused tail of its chunk on exit, instead of a separate fill launch
  int fill_tail;
  double x_fill;
  // Uniform generated mesh (edges[e] == x_min + e*w bit-for-bit, edges[I] ==
  // x_max) with one material: geometry and cross sections come from registers,
  // no per-event table loads.
  int uniform;
  double x_min, x_max, w_gen;
  CellInfo cell0;
  const double* centers;
  const int* active;
  double rho, inv_rho;
  TallyPtrs t;
  FastStackRec* stacks;  // per-warp local stacks
  int stack_cap;
  FastPool pool;
  DevError* err;
  int seg;  // segment index within the step (diagnostics)
  unsigned long long* timeline;  // optional per-warp words (kTimelineWords)
  unsigned long long* warp_cursor;  // per warp {next, end} of its census chunk (zeroed per step)
  // shared-memory tallies flush into flush_replicas zeroed global replicas
  // (fast_flush_stride words each), folded in by a reduce kernel; 0: direct
  double* flush_scratch;
  size_t flush_stride;
  int flush_replicas;
  // Census thinning (precomb = 1; the cold start, where the census is x60-x150
  // the next step's histories). Every lane carries its own systematic comb of
  // spacing pc_s0 over the census particles it banks: a particle of weight w
  // starting at lane position P (the lane's census weight so far plus a uniform
  // offset in [0, s0) drawn per launch from pc_key) holds n = #{k : k s0 in
  // [P, P + w)} teeth and is banked once, with weight n s0, or not at all
  // (n = 0). E[n s0] = w for every particle, so the banked census is an
  // unbiased, equal-quantum restatement of the census; the comb at the next
  // step start (popctrl.cpp:7-42) then combs this ~(W / s0)-record bank to the
  // target instead of the raw census. Census tallies and counters score the
  // unthinned particles.
  int precomb;
  double pc_s0, pc_inv_s0;
  unsigned pc_key;
  double* pc_need;  // 32 per warp of the grid
  SmemOffsets so;   // set by launch_fast_segment
};
size_t fast_flush_stride(int I, int B);  // words per flush replica (nb <= B)

// Zero-weight records in the unused tails of the warps' census chunks, and the
// count of slots the census bank spans.
void launch_fill_census_holes(CensusBank census, uint64_t cap,
                              const unsigned long long* warp_cursor, int warps, double x_fill,
                              cudaStream_t s);
// Step start of the throughput mode in one launch: zero the tally slab, the
// warp census cursors, the census counter and the error word; reset the first
// segment's pool counters (fast_pool_reset).
void launch_step_start(double* slab, size_t slab_words, unsigned long long* cursor,
                       size_t cursor_words, unsigned long long* counter, DevError* err,
                       unsigned long long* ctl, unsigned long long* src_head,
                       unsigned long long* span, int sms, cudaStream_t s);
// Compact the census bank (drop zero-weight holes) into AoS particles at time t.
void launch_fast_compact_aos(CensusBank in, uint64_t n, double t, hwwg_particle* out,
                             unsigned long long* count, cudaStream_t s);
// The pulse (x0, mu[i], w0, t = 0) into a census bank from its directions alone.
void launch_mu_to_census(const double* mu, uint64_t n, double x0, double w0, CensusBank out,
                         cudaStream_t s);
// AoS particles (all at one time: the pulse source, a host-held census) into a census bank.
void launch_aos_to_census(const hwwg_particle* in, uint64_t n, CensusBank out, cudaStream_t s);

// resident blocks per SM of the transport instantiation (uniform mesh, shared
// tallies, fixed-point slots, warps per block: 12 or 24) with `smem` dynamic
// shared memory, and the most warps per SM any instantiation holds
// (fix: 0 fp64, 1 fixed-point, 2 fixed-point over a cell window)
int fast_blocks_per_sm(size_t smem, int uniform, int shf, int fix, int warps);
// transport block shapes (warps per block): 2 x 12, 2 x 14 (where the
// registers and the tallies' shared memory allow 28 warps) or 1 x 24 per SM
constexpr int kFastBlockWarps[3] = {12, 14, 24};
int fast_max_warps_per_sm();
// per-warp census cursor words (FastArgs::warp_cursor: next, end)
constexpr int kWarpCursorWords = 2;
// timeline words per warp: {t0, loop trips, t_exit, events} and, in
// -DHWWG_FAST_PROF builds, {max pending daughters, pieces shared, split
// records donated, pool records taken}
constexpr int kTimelineWords = 8;
// -DHWWG_FAST_PROF builds: loop phase sums; hist (optional, 8 x 120 x 2
// unsigned): trips and live lanes per 5 us bin of each segment
int fast_prof_read(unsigned long long out[12], unsigned* hist);
constexpr int kFastHistWords = 8 * 120 * 2;
size_t fast_smem_bytes(int I, int nb);
size_t fast_smem_count_bytes(int I);  // smem_tallies == 2: the track counts only
size_t fast_smem_fix_bytes(int I, int nb);  // smem_tallies == 1 with fixed-point track/edge slots
bool fast_fix_exponent(double vmax, int* k);  // grid exponent for the largest expected score
size_t fast_smem_centers_bytes(int I);  // window centres and mesh edges (after the tallies)
void launch_fast_segment(const FastArgs& a, int blocks, size_t smem, cudaStream_t s);
void launch_aos_to_fast(const hwwg_particle* in, uint64_t n, const MeshView& m, FastBank out,
                        uint64_t hist0, cudaStream_t s);

// Bijection on [0, n) that spreads runs of consecutive k evenly over [0, n):
// 32-element tiles t = k / 32 move to tile (a t + b) mod nt with a ~ 0.618 nt
// coprime to nt (a Weyl sequence), in-tile order and the last n % 32 elements
// stay. The comb writes tooth k at perm(k) — whole 512-byte tiles per array, so
// the writes stay coalesced — and the next step's contiguous history ranges
// (its window-update segments) become even samples of the census bank.
// The census of the throughput engine is stored in completion order: early
// slots hold the particles that reached census in few events, i.e. the
// ballistic ones near the wave front, and taken in bank order the first 25% of
// the next step's histories over-represented the front in the mid-step
// partial snapshot (driver.cpp:204-218) whose closure steers the windows
// (measured: phi_hybrid at the front cell 15 standard errors above the exact
// engine, tests/test_gpu_stat_pin.py). The reference's bank is in history
// order, exchangeable across histories; the permutation restores that.
// nt == 0: identity.
struct Perm {
  unsigned long long nt, a, b;
  unsigned long long m;  // floor(2^64 / nt): Barrett reduction (no 64-bit division call)
  __host__ __device__ unsigned long long operator()(unsigned long long k) const {
    const unsigned long long t = k >> 5;
    if (t >= nt) return k;
    const unsigned long long x = a * t + b;  // < 2^64 (a, b < nt < 2^27, t < nt)
#if defined(__CUDA_ARCH__)
    unsigned long long r = x - __umul64hi(x, m) * nt;
    if (r >= nt) r -= nt;
#else
    const unsigned long long r = x % nt;
#endif
    return (r << 5) | (k & 31ULL);
  }
};
Perm make_perm(uint64_t n, uint64_t seed, uint64_t step);

// Parallel comb (popctrl.cpp:7-42 semantics with a parallel fp64 scan).
struct FastCombArgs {
  CensusBank bank;
  double t_bank;  // the time of every particle of the bank (the census time)
  MeshView mesh;  // teeth locate their cell from x
  uint64_t n, target;
  uint64_t seed, stream;
  double* prefix;   // n
  double* scalars;  // [0] W, [1] spacing, [2] offset, [3] output weight
  FastBank out;
  void* temp;
  size_t temp_bytes;
  Perm perm;  // tooth k is written at perm(k), as history perm(k) (n == 0: identity)
  // 1: write (x, mu) only (FastArgs::n_packed: the transport derives the
  // rest of a tooth); 0: full 48 B records
  int packed_out;
  // a bound-grade estimate of the bank's total weight (hint_host plus the
  // hint_n device doubles at hint_batches: the step's census weight per
  // batch), which fixes the comb's integer scale before it reads the bank
  const double* hint_batches;
  int hint_n;
  double hint_host;
};
size_t fast_comb_temp_bytes(uint64_t n);
// Single-GPU comb of a bank of any size: `prefix` is fast_comb_scratch_words(n)
// words of scratch, `temp` unused.
void launch_fast_comb(const FastCombArgs& a, cudaStream_t s);
size_t fast_comb_scratch_words(uint64_t n);
// Multi-GPU comb pieces: local inclusive scan (scalars[0] = local total, 0 for
// an empty bank), and teeth [k_lo, k_hi) placed against origin + local prefix.
void launch_fast_comb_local_scan(const FastCombArgs& a, cudaStream_t s);
void launch_fast_comb_teeth_range(const FastCombArgs& a, double spacing, double offset,
                                  double origin, uint64_t k_lo, uint64_t k_hi, FastBank out,
                                  cudaStream_t s);
// Multi-rank local permutation of a rank's combed source (the multi-GPU comb
// places teeth by contiguous ranges, so the permutation follows the
// rebalance): out[c] = in[perm(c)] for c < n, with history id hist[c] (the
// rank's owned global ids: `pieces` ranges of (first id, count), in order).
struct PieceTable {
  int n;
  unsigned long long lo[9], cnt[9];
};
void launch_fast_permute(FastBank in, FastBank out, uint64_t n, Perm perm, const PieceTable& t,
                         cudaStream_t s);
// track_flux[i] = sum_b track_flux_batch[b][i] (fast mode scores batches only)
void launch_track_from_batches(TallyPtrs t, int I, int B, cudaStream_t s);
void launch_fast_to_aos(FastBank in, uint64_t n, hwwg_particle* out, cudaStream_t s);
// the same for a source whose first n_packed slots are comb teeth (x, mu only):
// w = *w0 (device), t = t0
void launch_fast_to_aos_packed(FastBank in, uint64_t n, uint64_t n_packed, const double* w0,
                               double t0, hwwg_particle* out, cudaStream_t s);
// (w, t) of the first n slots (comb teeth) written out: w = *w0 (device), t = t0
void launch_fill_wt(double2* wt, uint64_t n, const double* w0, double t0, cudaStream_t s);
// e2e packed host round trip: flag (zeroed here) = 1 unless every (w, t) equals
// wt[0] (copied to *first); and (x, mu) already in out.xm -> cell, identity
// hist0 + i, and (w0, t0) when uniform.
void launch_check_uniform(const double2* wt, uint64_t n, unsigned* flag, double2* first,
                          cudaStream_t s);
// Config-3 volumetric source particles j0 .. j0+n-1 of a step (Philox mode),
// written to out[0..n) as histories hist0 .. hist0+n-1.
void launch_volume_source(FastBank out, uint64_t n, uint64_t j0, uint64_t hist0, const MeshView& m,
                          unsigned k0, unsigned k1, unsigned step, double x_lo, double x_hi,
                          double ta, double tb, double w, cudaStream_t s);
// (pieces: multi-rank, history of slot i = the rank's i-th owned id; null: hist0 + i)
void launch_xm_to_fast(FastBank out, uint64_t n, const MeshView& m, uint64_t hist0, int uniform,
                       double w0, double t0, cudaStream_t s, const PieceTable* pieces = nullptr);

}  // namespace hwwg
