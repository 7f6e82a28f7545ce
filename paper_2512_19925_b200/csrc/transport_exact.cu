// Exact-mode history kernel: bit-exact replay of hww::run_segment_parallel
// (proj/src/transport.cpp:81-237) on sm_100a — events, census AND tallies.
//
// Why it is built this way: the reference's daughters share their parent
// history's flight/window streams and run depth-first on a LIFO stack
// (transport.cpp:100-107, 199-202), so a history's event sequence is
// inherently serial; and its fp64 tallies are sums in one specific order —
// sequential over the events of each 256-history chunk into a fresh TallySet,
// then chunk sums merged in chunk order (transport.cpp:219-236). One GPU
// thread per 256-history chunk runs that chunk's histories in order into
// chunk-private accumulators (plain adds, no atomics), and k_merge_chunks adds
// the chunk sums into the running tallies in chunk order, so every tally —
// and hence every LOSM solve and window centre downstream — is bit-identical
// to the reference, not merely within rounding. Integer tallies (tracks per
// cell, counters) are order-free and use atomics.
//
// The daughter stack is run-length encoded: a split pushes its n-1 identical
// copies as ONE run (entry, n-1) (transport.cpp:65-66), so the pop order is
// the reference's while storage is O(split events) — measured depth <= 9 runs
// on BASELINE configs 1/2/4/5 (oracle diagnostics); capacity 64 here.
//
// Arithmetic parity: compiled with -fmad=false (no FMA contraction, like the
// reference's x86-64 baseline build), IEEE div.rn, and log is the bit-exact
// libm replay in libm_log.h. Census records are appended with a
// (history << 24 | emission index) key and radix-sorted afterwards, restoring
// the reference's history-major, depth-first order (transport.cpp:146, 233-236).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "rng.cuh"
#include "transport.cuh"

namespace hwwg {

namespace {

constexpr int kMaxRuns = 64;
constexpr uint64_t kMaxEventsPerHistory = 1000000ULL;  // transport.hpp:97
constexpr double kMaxSplitDaughters = 1000000.0;        // ww.hpp:53
constexpr double kGrazingMu = 1e-10;                    // tally.hpp:48

struct Run {
  double x, mu, w, t;
  int cell;
  unsigned count;
};

struct Local {
  unsigned long long u[kNumUCounters];
  double leak, aborted;  // chunk-sequential, like StepCounters of a chunk
};

// Chunk-private fp64 accumulators (one hww::TallySet per chunk), added to in
// place by the chunk-serial kernel.
struct Sink {
  double* track;  // I
  double* cphi;   // I
  double* cJ;     // I
  double* cF;     // I
  double* edge;   // I+1
  double* bclo;   // 2
  double* cwb;    // B
  double* trackb; // span*I, batch b stored at (b - b0)
  int b0;
  int I;
  Local* c;       // leak / aborted: chunk-sequential registers
  __device__ __forceinline__ void track_add(int cell, int batch, double v) const {
    track[cell] += v;
    trackb[(size_t)(batch - b0) * I + cell] += v;
  }
  __device__ __forceinline__ void census_add(int cell, int batch, double phi, double J, double F,
                                             double w) const {
    cphi[cell] += phi;
    cJ[cell] += J;
    cF[cell] += F;
    cwb[batch] += w;
  }
  __device__ __forceinline__ void edge_add(int e, double v) const { edge[e] += v; }
  __device__ __forceinline__ void bclo_add(int side, double v) const { bclo[side] += v; }
  __device__ __forceinline__ void leak_add(double w) const { c->leak += w; }
  __device__ __forceinline__ void aborted_add(double w) const { c->aborted += w; }
};

__device__ __forceinline__ void set_error(DevError* e, int code, unsigned long long h) {
  if (atomicCAS(&e->code, 0, code) == 0) e->history = h;
}

struct History {
  const ExactArgs& a;
  Local& c;
  Run* stk;
  int sp;
  Xoshiro flight, win;
  unsigned long long h;

  __device__ __forceinline__ bool push(double x, double mu, double w, double t, int cell,
                                       unsigned count) {
    if (sp == kMaxRuns) {
      set_error(a.err, HWWG_ESTACK, h);
      return false;
    }
    stk[sp] = Run{x, mu, w, t, cell, count};
    ++sp;
    return true;
  }

  // ww.cpp:46-72 + transport.cpp:54-77 applied in place; false = particle dies.
  __device__ __forceinline__ bool window_game(double x, double mu, double& w, double t,
                                              int cell) {
    const double center = a.centers[cell];
    const double floor_ = center / a.rho;
    const double ceil_ = center * a.rho;
    if (w > ceil_) {
      double n = ceil(w / center);
      if (n > kMaxSplitDaughters) {
        n = kMaxSplitDaughters;
        ++c.u[kCappedSplits];
      }
      const int daughters = (int)n;
      ++c.u[kSplits];
      c.u[kSplitDaughters] += (unsigned long long)(daughters - 1);
      w = w / n;
      if (daughters > 1 && !push(x, mu, w, t, cell, (unsigned)(daughters - 1))) {
        sp = 0;
        return false;
      }
      return true;
    }
    if (w < floor_) {
      const double survival = w / center;
      if (win.uniform() < survival) {
        ++c.u[kRouletteSurvivals];
        w = center;
        return true;
      }
      ++c.u[kRouletteKills];
      return false;
    }
    return true;
  }
};

// advance_history (transport.cpp:81-192) for source index i into sink S
// (chunk accumulators, or the tally log of the history-parallel path).
template <class SinkT>
__device__ void run_history(const ExactArgs& a, uint64_t i, Local& c, Run* stk, SinkT& S) {
  const unsigned long long h = a.h_begin + i;
  const double2 s0 = reinterpret_cast<const double2*>(a.src)[2 * i];
  const double2 s1 = reinterpret_cast<const double2*>(a.src)[2 * i + 1];
  // transport.cpp:91-98
  if (!isfinite(s0.x) || !isfinite(s1.x) || s1.x <= 0.0) {
    ++c.u[kNanAborts];
    return;
  }
  const int start_cell = locate_cell(a.mesh, s0.x);
  if (start_cell < 0 || !(s1.y >= a.t_begin && s1.y < a.t_end)) {
    set_error(a.err, HWWG_EINVAL, h);
    return;
  }

  History hs{a, c, stk, 0, {}, {}, h};
  hs.flight.seed(a.seed, stream_id(a.step, h, kFlight));  // transport.cpp:199-202
  hs.win.seed(a.seed, stream_id(a.step, h, kWindow));
  const int batch = batch_of(h, a.H, a.B);
  const bool windows = a.centers != nullptr && (a.active == nullptr || *a.active != 0);
  const int I = a.mesh.I;
  const double* edges = a.mesh.edges;

  hs.push(s0.x, s0.y, s1.x, s1.y, start_cell, 1u);
  unsigned long long events = 0;
  unsigned seq = 0;
  // A census record is written one census later (or at the history's end):
  // the slot atomic's round trip then overlaps the events in between.
  unsigned long long pend_slot = ~0ULL, pend_key = 0;
  double2 pend_a = make_double2(0.0, 0.0), pend_b = make_double2(0.0, 0.0);
  auto flush_census = [&]() {
    if (pend_slot < a.census_cap) {
      double2* dst = reinterpret_cast<double2*>(a.census) + 2 * pend_slot;
      dst[0] = pend_a;
      dst[1] = pend_b;
      a.census_keys[pend_slot] = pend_key;
    }
    pend_slot = ~0ULL;
  };

  while (hs.sp > 0) {
    Run& top = stk[hs.sp - 1];
    double x = top.x, mu = top.mu, w = top.w, t = top.t;
    int cell = top.cell;
    if (--top.count == 0) --hs.sp;

    bool alive = true;
    while (alive) {
      if (++events > kMaxEventsPerHistory) {  // transport.cpp:111-118
        ++c.u[kEventCapAborts];
        S.aborted_add(w);
        for (int r = 0; r < hs.sp; ++r)
          for (unsigned j = 0; j < stk[r].count; ++j) S.aborted_add(stk[r].w);
        hs.sp = 0;
        break;
      }
      const CellInfo ci = a.mesh.cells[cell];
      const double d_census = ci.speed * (a.t_end - t);
      const double d_collision = -hwwg_libm_log(hs.flight.uniform()) / ci.sigma_t;
      double d_boundary = __longlong_as_double(0x7ff0000000000000LL);
      int edge = -1;
      if (mu > 0.0) {
        edge = cell + 1;
        d_boundary = (edges[edge] - x) / mu;
      } else if (mu < 0.0) {
        edge = cell;
        d_boundary = (edges[edge] - x) / mu;
      }
      double d = d_census;  // std::min({...}) keeps the first smallest
      if (d_collision < d) d = d_collision;
      if (d_boundary < d) d = d_boundary;

      if (d > 0.0) {  // score_track, tally.hpp:51-56
        const double sc = w * d * (ci.inv_dx * a.inv_dt);
        S.track_add(cell, batch, sc);
        atomicAdd(&a.t.tracks[cell], 1ULL);
      }

      if (d == d_census) {  // transport.cpp:141-149
        x += d * mu;
        t = a.t_end;
        const double base = ci.speed * w * ci.inv_dx;  // score_census, tally.hpp:65-72
        S.census_add(cell, batch, base, base * mu, base * (1.0 / 3.0 - mu * mu), w);
        ++c.u[kCensusCount];
        flush_census();
        pend_slot = atomicAdd(a.census_count, 1ULL);
        pend_a = make_double2(x, mu);
        pend_b = make_double2(w, t);
        pend_key = (h << 24) | seq;
        ++seq;
        alive = false;
        continue;
      }

      if (d == d_boundary) {  // transport.cpp:151-164
        x = edges[edge];
        t += d / ci.speed;
        const bool domain = edge == 0 || edge == I;
        S.edge_add(edge, (mu > 0 ? w : -w) * a.inv_dt);  // tally.hpp:77-92
        if (domain) {
          const double amu = mu > 0 ? mu : -mu;
          if (amu < kGrazingMu) {
            ++c.u[kGrazingDiscarded];
          } else {
            S.bclo_add(edge == 0 ? 0 : 1, w * (0.5 - amu) / amu * a.inv_dt);
          }
          S.leak_add(w);
          alive = false;
          continue;
        }
        cell += mu > 0.0 ? 1 : -1;
        if (windows) alive = hs.window_game(x, mu, w, t, cell);
        continue;
      }

      // collision, transport.cpp:166-190; sample_collision :29-40
      x += d * mu;
      t += d / ci.speed;
      ++c.u[kCollisions];
      const double xi = hs.flight.uniform() * ci.sigma_t;
      if (xi < ci.sigma_s) {
        mu = hs.flight.uniform_pm1();
        if (windows) alive = hs.window_game(x, mu, w, t, cell);
      } else if (xi < ci.sigma_s + ci.sigma_f) {
        const double fl = floor(ci.nu_f);
        const double frac = ci.nu_f - fl;
        int ns = (int)fl;
        if (frac > 0.0 && hs.flight.uniform() < frac) ++ns;
        for (int s = 0; s < ns; ++s) {
          double ws = w;
          const double mus = hs.flight.uniform_pm1();
          if (!windows || hs.window_game(x, mus, ws, t, cell)) {
            if (!hs.push(x, mus, ws, t, cell, 1u)) {
              hs.sp = 0;
              break;
            }
          }
        }
        alive = false;
      } else {
        alive = false;
      }
    }
  }
  flush_census();
}

__device__ __forceinline__ Sink chunk_sink(const ExactArgs& a, int c) {
  const ChunkLayout& L = a.chunks;
  double* b = L.base + (size_t)c * L.stride;
  const int I = a.mesh.I;
  Sink s;
  s.track = b;
  s.cphi = b + I;
  s.cJ = b + 2 * I;
  s.cF = b + 3 * I;
  s.edge = b + 4 * I;
  s.bclo = b + 5 * I + 1;
  s.cwb = b + 5 * I + 5;
  s.trackb = b + 5 * I + 5 + a.B;
  s.b0 = batch_of(a.h_begin + (uint64_t)c * kChunk, a.H, a.B);
  s.I = I;
  s.c = nullptr;
  return s;
}

// One thread per 256-history chunk (run_segment_serial on the chunk,
// transport.cpp:194-207), histories in order.
__global__ void __launch_bounds__(64) k_exact_chunks(ExactArgs a) {
  Run stk[kMaxRuns];
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.chunks.count) return;
  Sink S = chunk_sink(a, c);
  double* dcnt = a.chunks.base + (size_t)c * a.chunks.stride + 5 * a.mesh.I + 3;
  Local l;
  S.c = &l;
#pragma unroll
  for (int k = 0; k < kNumUCounters; ++k) l.u[k] = 0;
  l.leak = dcnt[0];
  l.aborted = dcnt[1];
  const uint64_t lo = (uint64_t)c * kChunk;
  const uint64_t hi = lo + kChunk < a.n ? lo + kChunk : a.n;
  for (uint64_t i = lo; i < hi; ++i) run_history(a, i, l, stk, S);
  dcnt[0] = l.leak;
  dcnt[1] = l.aborted;
  l.u[kHistoriesScored] = hi - lo;
#pragma unroll
  for (int k = 0; k < kNumUCounters; ++k)
    if (l.u[k]) atomicAdd(&a.t.ucount[k], l.u[k]);
}

constexpr size_t kReplaySmemMax = 96 * 1024;

// ---- history-parallel path ------------------------------------------------
// The tally contributions of one history, in event order, appended to its own
// block chain in the log (slots of the chunk layout: track 0, census phi I,
// J 2I, F 3I, edge 4I, bclosure 5I+1, leak 5I+3, aborted 5I+4, census weight
// by batch 5I+5, track by batch 5I+5+B).
struct LogSink {
  ExactLog L;
  DevError* err;
  unsigned I, B;
  int b0;
  unsigned cur = ~0u, pos = kLogBlock, first = ~0u, total = 0;
  unsigned long long own = 0;      // the history's first block: its own index, no atomic
  unsigned long long dyn_base = 0;  // later blocks: dyn_base + a shared counter
  bool full = false;
  __device__ __forceinline__ void put(unsigned slot, double v) {
    if (pos == kLogBlock) {
      const unsigned long long nb = cur == ~0u ? own : dyn_base + atomicAdd(L.blocks, 1ULL);
      if (nb >= L.cap_blocks) {  // the step replays with a larger arena; a full
        if (!full) atomicCAS(&err->code, 0, kLogOverflow);  // history keeps
        full = true;                                         // counting its demand
        atomicMax(L.blocks + 1, nb + 1);
      } else if (!full) {
        if (cur == ~0u) first = (unsigned)nb;
        else L.next[cur] = (unsigned)nb;
        cur = (unsigned)nb;
      }
      pos = 0;
    }
    if (!full) {
      const size_t e = (size_t)cur * kLogBlock + pos;
      L.slot[e] = slot;
      L.val[e] = v;
    }
    ++pos;
    ++total;
  }
  __device__ __forceinline__ void track_add(int cell, int batch, double v) {
    put((unsigned)cell, v);
    put(5 * I + 5 + B + (unsigned)(batch - b0) * I + (unsigned)cell, v);
  }
  __device__ __forceinline__ void census_add(int cell, int batch, double phi, double J, double F,
                                             double w) {
    put(I + (unsigned)cell, phi);
    put(2 * I + (unsigned)cell, J);
    put(3 * I + (unsigned)cell, F);
    put(5 * I + 5 + (unsigned)batch, w);
  }
  __device__ __forceinline__ void edge_add(int e, double v) { put(4 * I + (unsigned)e, v); }
  __device__ __forceinline__ void bclo_add(int side, double v) { put(5 * I + 1 + side, v); }
  __device__ __forceinline__ void leak_add(double w) { put(5 * I + 3, w); }
  __device__ __forceinline__ void aborted_add(double w) { put(5 * I + 4, w); }
};

// One thread per history: the physics of every history runs concurrently; the
// fp64 tallies go to the log, integer tallies and counters straight to their
// (order-free) atomics, census records as in the chunk path.
__global__ void __launch_bounds__(128) k_exact_histories(ExactArgs a) {
  Run stk[kMaxRuns];
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool on = i < a.n;
  Local l;
#pragma unroll
  for (int k = 0; k < kNumUCounters; ++k) l.u[k] = 0;
  if (on) {
    LogSink S;
    S.L = a.log;
    S.err = a.err;
    S.I = (unsigned)a.mesh.I;
    S.B = (unsigned)a.B;
    S.b0 = batch_of(a.h_begin + (i / kChunk) * kChunk, a.H, a.B);
    S.own = i;
    S.dyn_base = a.n;
    run_history(a, i, l, stk, S);
    a.log.first[i] = S.first;
    a.log.count[i] = S.total;
    l.u[kHistoriesScored] = 1;
  }
#pragma unroll
  for (int k = 0; k < kNumUCounters; ++k) {
    unsigned long long v = l.u[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&a.t.ucount[k], v);
  }
}

// One warp per chunk: the chunk's accumulators in shared memory, the log of
// its histories added in history and event order. 32 consecutive entries are
// loaded at once; entries with distinct slots commute, entries with the same
// slot (MATCH.ANY group) are added by the group's first lane in lane order —
// exactly the chunk-serial sequence of adds per slot.
template <bool kSmem>
__global__ void __launch_bounds__(32) k_exact_replay(ExactArgs a) {
  extern __shared__ double smem_acc[];
  if (a.err->code == kLogOverflow) return;  // the step replays
  const ChunkLayout& L = a.chunks;
  const int c = blockIdx.x;
  const int lane = threadIdx.x;
  double* base = L.base + (size_t)c * L.stride;
  double* acc = kSmem ? smem_acc : base;
  if (kSmem) {
    for (size_t k = lane; k < L.stride; k += 32) acc[k] = base[k];
    __syncwarp();
  }
  __shared__ unsigned s_blk[32], s_ord[32], s_last[32];
  const uint64_t lo = (uint64_t)c * kChunk;
  const uint64_t hi = lo + kChunk < a.n ? lo + kChunk : a.n;
  // 32 histories at a time: their logs concatenated in history order, taken
  // 32 entries per window (lane = entry), so short logs share a window. Two-
  // stage pipeline: window w+1's entries are located and loaded before window
  // w is summed; a history's first block is its own index, later blocks come
  // from the chain, whose next link is fetched one window ahead.
  for (uint64_t g = lo; g < hi; g += 32) {
    const uint64_t h = g + lane;
    const unsigned cnt = h < hi ? a.log.count[h] : 0u;
    unsigned cur_blk = (unsigned)h;  // lane j: history g + j's current block ...
    unsigned cur_ord = 0;            // ... its ordinal in the chain ...
    unsigned nreg = ~0u;             // a next link this lane fetched for some history
    unsigned inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned p = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += p;
    }
    const unsigned off = inc - cnt;  // exclusive: the history's first entry
    const unsigned total = __shfl_sync(0xffffffffu, inc, 31);
    if (lane < 32) s_last[lane] = 32u;  // no prefetched link yet
    __syncwarp();
    // locate window p's entries and issue their loads (advances the chain state)
    auto locate = [&](unsigned p, unsigned& slot, double& v, bool& valid) {
      // the link prefetched for this lane's history (by the lane in s_last)
      const unsigned src = s_last[lane];
      const unsigned got = __shfl_sync(0xffffffffu, nreg, src & 31);
      const unsigned my_nxt = src < 32 ? got : ~0u;
      const unsigned q = p + lane;
      valid = q < total;
      int j = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const unsigned oc = __shfl_sync(0xffffffffu, off, (j + st) & 31);
        if (j + st < 32 && oc <= q) j += st;
      }
      const unsigned e = q - __shfl_sync(0xffffffffu, off, j);
      const unsigned ord = e / kLogBlock;
      const unsigned bj = __shfl_sync(0xffffffffu, cur_blk, j);
      const unsigned oj = __shfl_sync(0xffffffffu, cur_ord, j);
      const unsigned nj = __shfl_sync(0xffffffffu, my_nxt, j);
      const unsigned cj = __shfl_sync(0xffffffffu, cnt, j);
      unsigned blk = bj;
      slot = 0;
      v = 0.0;
      if (valid) {
        if (ord != oj) blk = nj != ~0u ? nj : a.log.next[bj];  // one block on at most
        const size_t ent = (size_t)blk * kLogBlock + (e % kLogBlock);
        slot = a.log.slot[ent];
        v = a.log.val[ent];
      }
      __syncwarp();
      // the history's last entry in this window carries its chain position on
      // and fetches the following link when the log continues past this block
      const int jn = __shfl_down_sync(0xffffffffu, j, 1);
      const bool last = valid && (lane == 31 || jn != j || q + 1 >= total);
      nreg = ~0u;
      if (last) {
        s_blk[j] = blk;
        s_ord[j] = ord;
        if ((ord + 1) * kLogBlock < cj) {
          nreg = a.log.next[blk];
          s_last[j] = (unsigned)lane;
        } else {
          s_last[j] = 32u;
        }
      }
      __syncwarp();
      const bool seen = cnt > 0 && off < p + 32 && off + cnt > p;
      if (seen) {
        cur_blk = s_blk[lane];
        cur_ord = s_ord[lane];
      }
      __syncwarp();
    };
    auto add = [&](unsigned slot, double v, bool valid) {
      const unsigned grp = __match_any_sync(0xffffffffu, valid ? slot : 0xffffffffu - lane);
      const bool leader = valid && lane == __ffs(grp) - 1;
      double sum = 0.0;
      unsigned rest = 0;
      if (leader) {
        sum = acc[slot] + v;
        rest = grp & (grp - 1);  // the group's other lanes, ascending
      }
      while (__any_sync(0xffffffffu, rest != 0)) {
        const int src = rest ? __ffs(rest) - 1 : lane;
        const double o = __shfl_sync(0xffffffffu, v, src);
        if (rest) {
          sum += o;
          rest &= rest - 1;
        }
      }
      if (leader) acc[slot] = sum;
      __syncwarp();
    };
    if (total == 0) continue;
    unsigned slot_a, slot_b = 0;
    double v_a, v_b = 0.0;
    bool ok_a, ok_b = false;
    locate(0, slot_a, v_a, ok_a);
    for (unsigned p = 0; p < total; p += 32) {
      const bool more = p + 32 < total;
      if (more) locate(p + 32, slot_b, v_b, ok_b);  // in flight while window p is added
      add(slot_a, v_a, ok_a);
      slot_a = slot_b;
      v_a = v_b;
      ok_a = ok_b;
    }
  }
  if (kSmem)
    for (size_t k = lane; k < L.stride; k += 32) base[k] = acc[k];
}

// Chunk accumulators start at zero (a fresh TallySet per chunk,
// transport.cpp:220-227) — or, when the segment is a single chunk, at the
// running tallies (run_segment_serial straight into them, transport.cpp:216-217).
__global__ void k_chunk_init(ExactArgs a) {
  const ChunkLayout& L = a.chunks;
  const int I = a.mesh.I, B = a.B;
  const size_t total = (size_t)L.count * L.stride;
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= total) return;
  double v = 0.0;
  if (L.count == 1) {
    const TallyPtrs& T = a.t;
    const int b0 = batch_of(a.h_begin, a.H, B);
    if (k < (size_t)I) v = T.track_flux[k];
    else if (k < 2 * (size_t)I) v = T.census_phi[k - I];
    else if (k < 3 * (size_t)I) v = T.census_current[k - 2 * I];
    else if (k < 4 * (size_t)I) v = T.census_closure[k - 3 * I];
    else if (k < 5 * (size_t)I + 1) v = T.edge_current[k - 4 * I];
    else if (k < 5 * (size_t)I + 3) v = T.boundary_closure[k - (5 * I + 1)];
    else if (k < 5 * (size_t)I + 5) v = T.dcount[k - (5 * I + 3)];
    else if (k < 5 * (size_t)I + 5 + B) v = T.census_weight_batch[k - (5 * I + 5)];
    else {
      const size_t j = k - (5 * (size_t)I + 5 + B);
      const int b = b0 + (int)(j / I);
      if (b < B) v = T.track_flux_batch[(size_t)b * I + j % I];
    }
  }
  L.base[k] = v;
}

// merge_from in chunk order (tally.cpp:8-26; transport.cpp:233-236): one
// thread per tally slot walks the chunks sequentially.
__global__ void k_merge_chunks(ExactArgs a) {
  const ChunkLayout& L = a.chunks;
  const int I = a.mesh.I, B = a.B;
  const int slots = 5 * I + 5 + B + B * I;  // chunk-layout slots + the global batch table
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= slots) return;
  const TallyPtrs& T = a.t;
  double* dst;
  int local;  // slot inside a chunk, or -1 for the batch table
  int b = 0, cell = 0;
  if (s < 5 * I + 5 + B) {
    local = s;
    if (s < I) dst = &T.track_flux[s];
    else if (s < 2 * I) dst = &T.census_phi[s - I];
    else if (s < 3 * I) dst = &T.census_current[s - 2 * I];
    else if (s < 4 * I) dst = &T.census_closure[s - 3 * I];
    else if (s < 5 * I + 1) dst = &T.edge_current[s - 4 * I];
    else if (s < 5 * I + 3) dst = &T.boundary_closure[s - (5 * I + 1)];
    else if (s < 5 * I + 5) dst = &T.dcount[s - (5 * I + 3)];
    else dst = &T.census_weight_batch[s - (5 * I + 5)];
  } else {
    local = -1;
    const int j = s - (5 * I + 5 + B);
    b = j / I;
    cell = j % I;
    dst = &T.track_flux_batch[(size_t)b * I + cell];
  }
  if (L.count == 1) {  // accumulated in place from the running values
    if (local >= 0) {
      *dst = L.base[local];
    } else {
      const int b0 = batch_of(a.h_begin, a.H, B);
      if (b >= b0 && b < b0 + L.span) *dst = L.base[5 * I + 5 + B + (size_t)(b - b0) * I + cell];
    }
    return;
  }
  // chunks in order; loads run kAhead chunks ahead of the (sequential) adds
  constexpr int kAhead = 8;
  double acc = *dst;
  if (local >= 0) {
    const double* p = L.base + local;
    int c = 0;
    for (; c + kAhead <= L.count; c += kAhead) {
      double v[kAhead];
#pragma unroll
      for (int k = 0; k < kAhead; ++k) v[k] = p[(size_t)(c + k) * L.stride];
#pragma unroll
      for (int k = 0; k < kAhead; ++k) acc += v[k];
    }
    for (; c < L.count; ++c) acc += p[(size_t)c * L.stride];
  } else {
    // the chunks whose batch window [b0, b0 + span) holds b form one run
    // (b0 is non-decreasing in c): find it, then add in chunk order
    auto b0_of = [&](int c) { return batch_of(a.h_begin + (uint64_t)c * kChunk, a.H, B); };
    int lo = 0, hi = L.count;  // first c with b0 + span > b
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (b0_of(m) + L.span > b) hi = m;
      else lo = m + 1;
    }
    const int c_lo = lo;
    hi = L.count;  // first c with b0 > b
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (b0_of(m) > b) hi = m;
      else lo = m + 1;
    }
    const int c_hi = lo;
    const size_t row = 5 * I + 5 + B + (size_t)cell;
    int c = c_lo;
    for (; c + kAhead <= c_hi; c += kAhead) {
      double v[kAhead];
#pragma unroll
      for (int k = 0; k < kAhead; ++k)
        v[k] = L.base[(size_t)(c + k) * L.stride + row + (size_t)(b - b0_of(c + k)) * I];
#pragma unroll
      for (int k = 0; k < kAhead; ++k) acc += v[k];
    }
    for (; c < c_hi; ++c) acc += L.base[(size_t)c * L.stride + row + (size_t)(b - b0_of(c)) * I];
  }
  *dst = acc;
}

__global__ void k_iota(unsigned* v, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (unsigned)i;
}

__global__ void k_gather(const hwwg_particle* __restrict__ src, const unsigned* __restrict__ idx,
                         hwwg_particle* __restrict__ dst, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double2* s = reinterpret_cast<const double2*>(src) + 2 * (uint64_t)idx[i];
    double2* d = reinterpret_cast<double2*>(dst) + 2 * i;
    d[0] = s[0];
    d[1] = s[1];
  }
}

int host_batch_of(uint64_t h, uint64_t H, int B) {
  if (H == 0) return 0;
  const int b = (int)(h * (uint64_t)B / H);
  return b < B ? b : B - 1;
}

}  // namespace

ChunkLayout chunk_layout(uint64_t n, uint64_t h_begin, uint64_t H, int I, int B) {
  ChunkLayout L{};
  L.count = (int)((n + kChunk - 1) / kChunk);
  int span = 1;  // batches touched by one chunk (contiguous slices of H/B histories)
  for (int c = 0; c < L.count; ++c) {
    const uint64_t lo = h_begin + (uint64_t)c * kChunk;
    const uint64_t len = n - (uint64_t)c * kChunk < (uint64_t)kChunk ? n - (uint64_t)c * kChunk
                                                                     : (uint64_t)kChunk;
    const int sp = host_batch_of(lo + len - 1, H, B) - host_batch_of(lo, H, B) + 1;
    if (sp > span) span = sp;
  }
  L.span = span;
  L.stride = (size_t)5 * I + 5 + B + (size_t)span * I;
  return L;
}


void launch_exact_segment(const ExactArgs& a, cudaStream_t s) {
  if (a.n == 0) return;
  const size_t total = (size_t)a.chunks.count * a.chunks.stride;
  k_chunk_init<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(a);
  if (a.log.slot) {
    HWWG_CUDA(cudaMemsetAsync(a.log.blocks, 0, sizeof(unsigned long long), s));
    k_exact_histories<<<(unsigned)((a.n + 127) / 128), 128, 0, s>>>(a);
    const size_t smem = a.chunks.stride * sizeof(double);
    if (smem <= kReplaySmemMax) {  // chunk accumulators in shared memory
      static DynSmemCache configured;
      ensure_dyn_smem(k_exact_replay<true>, smem, configured);
      k_exact_replay<true><<<(unsigned)a.chunks.count, 32, smem, s>>>(a);
    } else {
      k_exact_replay<false><<<(unsigned)a.chunks.count, 32, 0, s>>>(a);
    }
  } else {
    k_exact_chunks<<<(unsigned)((a.chunks.count + 63) / 64), 64, 0, s>>>(a);
  }
  const int slots = 5 * a.mesh.I + 5 + a.B + a.B * a.mesh.I;
  k_merge_chunks<<<(slots + 255) / 256, 256, 0, s>>>(a);
  HWWG_CUDA(cudaGetLastError());
}

size_t census_sort_temp_bytes(uint64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const unsigned*)nullptr,
                                  (unsigned*)nullptr, (int)n, 0, 64);
  return bytes;
}

void sort_census(const CensusSortArgs& a, cudaStream_t s) {
  if (a.n == 0) return;
  const unsigned threads = 256;
  const unsigned blocks = (unsigned)((a.n + threads - 1) / threads);
  k_iota<<<blocks, threads, 0, s>>>(a.idx_in, a.n);
  size_t bytes = a.temp_bytes;
  HWWG_CUDA(cub::DeviceRadixSort::SortPairs(a.temp, bytes, a.keys_in, a.keys_out, a.idx_in,
                                            a.idx_out, (int)a.n, a.begin_bit, a.end_bit, s));
  k_gather<<<blocks, threads, 0, s>>>(a.records, a.idx_out, a.out, a.n);
  HWWG_CUDA(cudaGetLastError());
}

}  // namespace hwwg
