/*
 * TEST INFRASTRUCTURE — CPU oracle (checker only; see hww_oracle.h).
 *
 * Plain-C restatement of the reference's hot path and its callers, function
 * by function, with the reference file:line each one follows. Arithmetic is
 * written in the reference's evaluation order and the file is compiled with
 * -ffp-contract=off and no -march (the reference's own flags,
 * proj/CMakeLists.txt:1-19), so results are bit-identical to
 * oracle/_ref/libhww_ref.so. log() is the system libm's, exactly as the
 * reference calls std::log (proj/src/transport.cpp:26).
 *
 * The daughter stack is run-length encoded: split copies are identical at
 * push time (proj/src/transport.cpp:65-66), so a run (entry, count) pops in
 * exactly the reference's LIFO order.
 */
#include "hww_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[512];
const char* orc_last_error(void) { return g_err; }
static void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

/* ---------------------------------------------------------------- RNG --- */
/* proj/include/hww/rng.hpp:10-59: splitmix64 seeding of xoshiro256**. */
typedef struct { uint64_t s[4]; } orc_rng;

static uint64_t sm64_next(uint64_t* x) {
  uint64_t z;
  *x += 0x9E3779B97F4A7C15ULL;
  z = *x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint64_t rot64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

static void rng_init(orc_rng* r, uint64_t seed, uint64_t id) {
  uint64_t x = seed + 0x9E3779B97F4A7C15ULL * id;
  for (int i = 0; i < 4; ++i) r->s[i] = sm64_next(&x);
  if ((r->s[0] | r->s[1] | r->s[2] | r->s[3]) == 0) r->s[0] = 1;
}
static uint64_t rng_u64(orc_rng* r) {
  const uint64_t out = rot64(r->s[1] * 5, 7) * 9;
  const uint64_t t = r->s[1] << 17;
  r->s[2] ^= r->s[0];
  r->s[3] ^= r->s[1];
  r->s[1] ^= r->s[2];
  r->s[0] ^= r->s[3];
  r->s[2] ^= t;
  r->s[3] = rot64(r->s[3], 45);
  return out;
}
/* rng.hpp:51-56 */
static double rng_uniform(orc_rng* r) {
  return ((double)(rng_u64(r) >> 11) + 0.5) * 0x1.0p-53;
}
static double rng_pm1(orc_rng* r) { return 2.0 * rng_uniform(r) - 1.0; }

/* rng.hpp:73-76 */
uint64_t orc_stream_id(uint64_t step, uint64_t history, uint64_t purpose) {
  return (purpose << 56) ^ (step << 40) ^ history;
}
enum { P_SOURCE = 0, P_FLIGHT = 1, P_WINDOW = 2, P_COMB = 3 };

void orc_stream_uniforms(uint64_t seed, uint64_t id, uint64_t n, double* out) {
  orc_rng r;
  rng_init(&r, seed, id);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_uniform(&r);
}
void orc_stream_u64(uint64_t seed, uint64_t id, uint64_t n, uint64_t* out) {
  orc_rng r;
  rng_init(&r, seed, id);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_u64(&r);
}

/* The reference's log, element-wise (std::log, transport.cpp:26). */
void orc_log_array(const double* x, uint64_t n, double* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = log(x[i]);
}

/* --------------------------------------------------------------- mesh --- */
typedef struct {
  const double* edges;
  double* widths;
  int cells;
  int uniform;
} orc_mesh;

/* proj/src/mesh.cpp:9-24 (widths and the 1e-12 uniformity test). */
static int mesh_init(orc_mesh* m, const double* edges, int cells) {
  m->edges = edges;
  m->cells = cells;
  m->widths = (double*)malloc(sizeof(double) * (size_t)(cells > 0 ? cells : 1));
  if (cells < 1) {
    set_err("mesh needs at least one cell");
    return -1;
  }
  for (int i = 1; i <= cells; ++i)
    if (!(edges[i] > edges[i - 1])) {
      set_err("mesh edges must be strictly increasing");
      return -1;
    }
  for (int c = 0; c < cells; ++c) m->widths[c] = edges[c + 1] - edges[c];
  m->uniform = 1;
  for (int c = 0; c < cells; ++c)
    if (!(fabs(m->widths[c] - m->widths[0]) <= 1e-12 * m->widths[0])) m->uniform = 0;
  return 0;
}
static void mesh_free(orc_mesh* m) { free(m->widths); }

/* proj/src/mesh.cpp:26-40; returns -1 outside [x_min, x_max]. */
static int mesh_locate(const orc_mesh* m, double x) {
  const double lo = m->edges[0], hi = m->edges[m->cells];
  if (x < lo || x > hi) return -1;
  if (x == hi) return m->cells - 1;
  if (m->uniform) {
    int c = (int)((x - lo) / m->widths[0]);
    if (c >= m->cells) c = m->cells - 1;
    if (x < m->edges[c]) --c;
    else if (x >= m->edges[c + 1]) ++c;
    return c;
  }
  /* upper_bound: first edge strictly greater than x */
  int a = 0, b = m->cells + 1;
  while (a < b) {
    const int mid = (a + b) / 2;
    if (m->edges[mid] > x) b = mid;
    else a = mid + 1;
  }
  return a - 1;
}

int32_t orc_locate(const double* edges, int32_t cells, double x) {
  orc_mesh m;
  if (mesh_init(&m, edges, cells)) {
    mesh_free(&m);
    return -2;
  }
  const int c = mesh_locate(&m, x);
  mesh_free(&m);
  return c;
}

/* proj/src/mesh.cpp:42-50 */
void orc_uniform_edges(double x_min, double x_max, int32_t cells, double* out) {
  const double w = (x_max - x_min) / cells;
  for (int e = 0; e <= cells; ++e) out[e] = x_min + e * w;
  out[cells] = x_max;
}

/* proj/src/transport.cpp:13-22 + proj/src/driver.cpp:309-316 */
void orc_pulse_source(uint64_t seed, uint64_t histories, double x0, double strength,
                      orc_particle* out) {
  orc_rng r;
  rng_init(&r, seed, orc_stream_id(0, 0, P_SOURCE));
  const double total = strength * (double)histories;
  const double w = total / (double)histories;
  for (uint64_t h = 0; h < histories; ++h) {
    out[h].x = x0;
    out[h].mu = rng_pm1(&r);
    out[h].w = w;
    out[h].t = 0.0;
  }
}

/* Config-3 extension (the reference driver has
 * no volumetric source): n particles of the isotropic source box [x_lo, x_hi] x
 * [ta, tb], one sequential source stream per step (stream (step, 0, source));
 * per particle x, then t, then mu; weight rate * (tb - ta) * H_cfg / n. */
void orc_volume_source(uint64_t seed, int step, uint64_t n, double x_lo, double x_hi, double ta,
                       double tb, double rate, uint64_t h_cfg, orc_particle* out) {
  orc_rng r;
  rng_init(&r, seed, orc_stream_id((uint64_t)step, 0, P_SOURCE));
  const double w = rate * (tb - ta) * (double)h_cfg / (double)n;
  for (uint64_t h = 0; h < n; ++h) {
    out[h].x = x_lo + (x_hi - x_lo) * rng_uniform(&r);
    out[h].t = ta + (tb - ta) * rng_uniform(&r);
    out[h].mu = rng_pm1(&r);
    out[h].w = w;
  }
}

/* The LOSM source q_i of a step (losm.cpp:101-103 pass-through): the box's
 * emission integrated over cell i, averaged over the step:
 * rate * ((tb - ta) / dt) * |cell_i n [x_lo, x_hi]| / (x_hi - x_lo). */
void orc_volume_q(const double* edges, int I, double x_lo, double x_hi, double ta, double tb,
                  double dt, double rate, double* q) {
  const double tfrac = (tb - ta) / dt;
  const double bw = x_hi - x_lo;
  for (int i = 0; i < I; ++i) {
    const double lo = edges[i] > x_lo ? edges[i] : x_lo;
    const double hi = edges[i + 1] < x_hi ? edges[i + 1] : x_hi;
    const double len = hi > lo ? hi - lo : 0.0;
    q[i] = rate * tfrac * len / bw;
  }
}

/* --------------------------------------------------------------- bank --- */
static int bank_push(orc_bank* b, const orc_particle* p) {
  if (b->n == b->cap) {
    uint64_t nc = b->cap ? b->cap * 2 : 1024;
    orc_particle* d = (orc_particle*)realloc(b->data, nc * sizeof(orc_particle));
    if (!d) {
      set_err("out of memory growing census bank");
      return -1;
    }
    b->data = d;
    b->cap = nc;
  }
  b->data[b->n++] = *p;
  return 0;
}
void orc_bank_free(orc_bank* b) {
  free(b->data);
  b->data = NULL;
  b->n = b->cap = 0;
}

/* ---------------------------------------------------------- transport --- */
typedef struct {
  orc_mesh mesh;
  const orc_material* mats;
  double t_begin, t_end;
  uint64_t seed;
  int step;
  uint64_t histories_total;
  int batches;
  const double* centers; /* NULL: analog */
  double rho;
} seg_ctx;

typedef struct {
  orc_particle p;
  int cell;
  uint32_t count; /* identical copies in this run */
} stack_run;

typedef struct {
  stack_run* r;
  uint32_t n, cap, max_n;
} run_stack;

static void stack_push(run_stack* s, const orc_particle* p, int cell, uint32_t count) {
  if (s->n == s->cap) {
    s->cap = s->cap ? s->cap * 2 : 64;
    s->r = (stack_run*)realloc(s->r, s->cap * sizeof(stack_run));
  }
  s->r[s->n].p = *p;
  s->r[s->n].cell = cell;
  s->r[s->n].count = count;
  ++s->n;
  if (s->n > s->max_n) s->max_n = s->n;
}

/* tally.hpp:130-134 */
static int batch_of(uint64_t h, uint64_t H, int B) {
  if (H == 0) return 0;
  const int b = (int)(h * (uint64_t)B / H);
  return b < B ? b : B - 1;
}

/* ww.cpp:46-72 + transport.cpp:54-77: returns 0 when the particle dies. */
static int window_game(orc_particle* p, int cell, const seg_ctx* c, run_stack* st,
                       orc_rng* wrng, orc_counters* k) {
  const double center = c->centers[cell];
  const double floor_ = center / c->rho;
  const double ceil_ = center * c->rho;
  if (p->w > ceil_) {
    double n = ceil(p->w / center);
    int capped = 0;
    if (n > 1000000.0) {
      n = 1000000.0;
      capped = 1;
    }
    const int daughters = (int)n;
    ++k->splits;
    k->split_daughters += (uint64_t)daughters - 1;
    if (capped) ++k->capped_splits;
    p->w = p->w / n;
    if (daughters > 1) stack_push(st, p, cell, (uint32_t)(daughters - 1));
    return 1;
  }
  if (p->w < floor_) {
    const double survival = p->w / center;
    if (rng_uniform(wrng) < survival) {
      ++k->roulette_survivals;
      p->w = center;
      return 1;
    }
    ++k->roulette_kills;
    return 0;
  }
  return 1;
}

/* proj/src/transport.cpp:81-192 */
static int advance_history(const orc_particle* start, const seg_ctx* c, orc_tallies* ts,
                           orc_counters* k, uint64_t* tracks, orc_bank* census,
                           orc_rng* flight, orc_rng* wrng, int batch, run_stack* st) {
  const orc_mesh* mesh = &c->mesh;
  const int last_cell = mesh->cells - 1;
  const double inv_dt = 1.0 / (c->t_end - c->t_begin);
  const int I = mesh->cells;

  if (!isfinite(start->x) || !isfinite(start->w) || start->w <= 0.0) {
    ++k->nan_aborts;
    return 0;
  }
  const int start_cell = mesh_locate(mesh, start->x);
  if (start_cell < 0) {
    set_err("history starts outside the mesh");
    return -1;
  }
  if (!(start->t >= c->t_begin && start->t < c->t_end)) {
    set_err("history starts outside the time step");
    return -1;
  }

  st->n = 0;
  stack_push(st, start, start_cell, 1);
  uint64_t events = 0;

  while (st->n > 0) {
    stack_run* top = &st->r[st->n - 1];
    orc_particle p = top->p;
    int cell = top->cell;
    if (--top->count == 0) --st->n;

    int alive = 1;
    while (alive) {
      if (++events > 1000000ULL) { /* kMaxEventsPerHistory, transport.hpp:97 */
        ++k->event_cap_aborts;
        k->aborted_weight += p.w;
        for (uint32_t r = 0; r < st->n; ++r)
          for (uint32_t j = 0; j < st->r[r].count; ++j) k->aborted_weight += st->r[r].p.w;
        st->n = 0;
        break;
      }
      const orc_material* mat = &c->mats[cell];
      const double inv_dx = 1.0 / mesh->widths[cell];

      const double d_census = mat->speed * (c->t_end - p.t);
      if (!(mat->sigma_t > 0)) {
        set_err("sigma_t must be > 0");
        return -1;
      }
      const double d_collision = -log(rng_uniform(flight)) / mat->sigma_t;
      double d_boundary = INFINITY;
      int edge = -1;
      if (p.mu > 0.0) {
        edge = cell + 1;
        d_boundary = (mesh->edges[edge] - p.x) / p.mu;
      } else if (p.mu < 0.0) {
        edge = cell;
        d_boundary = (mesh->edges[edge] - p.x) / p.mu;
      }
      /* std::min({...}) keeps the first smallest (transport.cpp:135) */
      double d = d_census;
      if (d_collision < d) d = d_collision;
      if (d_boundary < d) d = d_boundary;

      if (d > 0.0) { /* score_track, tally.hpp:51-56 */
        const double sc = p.w * d * (inv_dx * inv_dt);
        ts->track_flux[cell] += sc;
        ts->track_flux_batch[(size_t)batch * I + cell] += sc;
        ++tracks[cell];
      }

      if (d == d_census) { /* transport.cpp:141-149; score_census tally.hpp:65-72 */
        p.x += d * p.mu;
        p.t = c->t_end;
        const double base = mat->speed * p.w * inv_dx;
        ts->census_phi[cell] += base;
        ts->census_current[cell] += base * p.mu;
        ts->census_closure[cell] += base * (1.0 / 3.0 - p.mu * p.mu);
        ts->census_weight_batch[batch] += p.w;
        ++k->census_count;
        if (census && bank_push(census, &p)) return -1;
        alive = 0;
        continue;
      }

      if (d == d_boundary) { /* transport.cpp:151-164; tally.hpp:77-92 */
        p.x = mesh->edges[edge];
        p.t += d / mat->speed;
        const int domain = edge == 0 || edge == last_cell + 1;
        ts->edge_current[edge] += (p.mu > 0 ? p.w : -p.w) * inv_dt;
        if (domain) {
          const double amu = p.mu > 0 ? p.mu : -p.mu;
          if (amu < 1e-10) {
            ++ts->grazing_discarded;
          } else {
            const double sc = p.w * (0.5 - amu) / amu * inv_dt;
            if (edge == 0) ts->boundary_closure_left += sc;
            else ts->boundary_closure_right += sc;
          }
          k->leakage_weight += p.w;
          alive = 0;
          continue;
        }
        cell += p.mu > 0.0 ? 1 : -1;
        if (c->centers) alive = window_game(&p, cell, c, st, wrng, k);
        continue;
      }

      /* collision, transport.cpp:166-190; sample_collision :29-40 */
      p.x += d * p.mu;
      p.t += d / mat->speed;
      ++k->collisions;
      const double xi = rng_uniform(flight) * mat->sigma_t;
      if (xi < mat->sigma_s) {
        p.mu = rng_pm1(flight);
        if (c->centers) alive = window_game(&p, cell, c, st, wrng, k);
      } else if (xi < mat->sigma_s + mat->sigma_f) {
        const double fl = floor(mat->nu_f);
        const double frac = mat->nu_f - fl;
        int ns = (int)fl;
        if (frac > 0.0 && rng_uniform(flight) < frac) ++ns;
        for (int s = 0; s < ns; ++s) {
          orc_particle sec = p;
          sec.mu = rng_pm1(flight);
          if (!c->centers || window_game(&sec, cell, c, st, wrng, k))
            stack_push(st, &sec, cell, 1);
        }
        alive = 0;
      } else {
        alive = 0;
      }
    }
  }
  return 0;
}

static int seg_serial(const seg_ctx* c, const orc_particle* src, uint64_t n,
                      uint64_t h_begin, orc_tallies* t, orc_counters* k, uint64_t* tracks,
                      orc_bank* census, run_stack* st) {
  for (uint64_t i = 0; i < n; ++i) { /* transport.cpp:194-207 */
    const uint64_t h = h_begin + i;
    orc_rng flight, wrng;
    rng_init(&flight, c->seed, orc_stream_id((uint64_t)c->step, h, P_FLIGHT));
    rng_init(&wrng, c->seed, orc_stream_id((uint64_t)c->step, h, P_WINDOW));
    const int batch = batch_of(h, c->histories_total, c->batches);
    if (advance_history(&src[i], c, t, k, tracks, census, &flight, &wrng, batch, st))
      return -1;
    ++t->histories_scored;
  }
  return 0;
}

static void counters_merge(orc_counters* a, const orc_counters* b) {
  a->collisions += b->collisions;
  a->splits += b->splits;
  a->split_daughters += b->split_daughters;
  a->capped_splits += b->capped_splits;
  a->roulette_kills += b->roulette_kills;
  a->roulette_survivals += b->roulette_survivals;
  a->census_count += b->census_count;
  a->event_cap_aborts += b->event_cap_aborts;
  a->nan_aborts += b->nan_aborts;
  a->leakage_weight += b->leakage_weight;
  a->aborted_weight += b->aborted_weight;
}

/* tally.cpp:8-26 */
static void tallies_merge(orc_tallies* a, const orc_tallies* b, int I, int B) {
  for (int i = 0; i < I; ++i) {
    a->track_flux[i] += b->track_flux[i];
    a->census_phi[i] += b->census_phi[i];
    a->census_current[i] += b->census_current[i];
    a->census_closure[i] += b->census_closure[i];
  }
  for (size_t i = 0; i < (size_t)B * I; ++i) a->track_flux_batch[i] += b->track_flux_batch[i];
  for (int j = 0; j < B; ++j) a->census_weight_batch[j] += b->census_weight_batch[j];
  for (int e = 0; e <= I; ++e) a->edge_current[e] += b->edge_current[e];
  a->boundary_closure_left += b->boundary_closure_left;
  a->boundary_closure_right += b->boundary_closure_right;
  a->histories_scored += b->histories_scored;
  a->grazing_discarded += b->grazing_discarded;
}

typedef struct {
  double* block;
  orc_tallies t;
} owned_tallies;

static void tallies_alloc(owned_tallies* o, int I, int B) {
  const size_t n = (size_t)I * 4 + (size_t)B * I + B + I + 1;
  o->block = (double*)calloc(n, sizeof(double));
  double* p = o->block;
  o->t.track_flux = p; p += I;
  o->t.track_flux_batch = p; p += (size_t)B * I;
  o->t.census_phi = p; p += I;
  o->t.census_current = p; p += I;
  o->t.census_closure = p; p += I;
  o->t.census_weight_batch = p; p += B;
  o->t.edge_current = p;
  o->t.boundary_closure_left = o->t.boundary_closure_right = 0.0;
  o->t.histories_scored = o->t.grazing_discarded = 0;
}
static void tallies_zero(owned_tallies* o, int I, int B) {
  const size_t n = (size_t)I * 4 + (size_t)B * I + B + I + 1;
  memset(o->block, 0, n * sizeof(double));
  o->t.boundary_closure_left = o->t.boundary_closure_right = 0.0;
  o->t.histories_scored = o->t.grazing_discarded = 0;
}

uint32_t orc_max_stack_runs_seen = 0; /* diagnostics: deepest RLE stack so far */

/* transport.cpp:209-237 (chunk > 0) or :194-207 (chunk <= 0). */
static int run_segment_ctx(const seg_ctx* c, const orc_particle* src, uint64_t n,
                           uint64_t h_begin, int chunk, orc_tallies* t, orc_counters* k,
                           uint64_t* tracks, orc_bank* census, uint32_t* max_runs) {
  run_stack st = {0};
  int rc = 0;
  const int I = c->mesh.cells, B = c->batches;
  const uint64_t chunks = chunk > 0 ? (n + (uint64_t)chunk - 1) / (uint64_t)chunk : 1;
  if (chunk <= 0 || chunks <= 1) {
    rc = seg_serial(c, src, n, h_begin, t, k, tracks, census, &st);
  } else {
    owned_tallies ct;
    tallies_alloc(&ct, I, B);
    uint64_t* ctracks = (uint64_t*)calloc((size_t)I, sizeof(uint64_t));
    orc_bank cb = {0};
    for (uint64_t ch = 0; ch < chunks && rc == 0; ++ch) {
      const uint64_t lo = ch * (uint64_t)chunk;
      const uint64_t hi = lo + (uint64_t)chunk < n ? lo + (uint64_t)chunk : n;
      orc_counters ck;
      memset(&ck, 0, sizeof ck);
      tallies_zero(&ct, I, B);
      memset(ctracks, 0, sizeof(uint64_t) * (size_t)I);
      cb.n = 0;
      rc = seg_serial(c, src + lo, hi - lo, h_begin + lo, &ct.t, &ck, ctracks,
                      census ? &cb : NULL, &st);
      if (rc) break;
      tallies_merge(t, &ct.t, I, B);
      if (census)
        for (uint64_t j = 0; j < cb.n; ++j)
          if (bank_push(census, &cb.data[j])) { rc = -1; break; }
      counters_merge(k, &ck);
      for (int i = 0; i < I; ++i) tracks[i] += ctracks[i];
    }
    orc_bank_free(&cb);
    free(ctracks);
    free(ct.block);
  }
  if (max_runs) *max_runs = st.max_n > *max_runs ? st.max_n : *max_runs;
  if (st.max_n > orc_max_stack_runs_seen) orc_max_stack_runs_seen = st.max_n;
  free(st.r);
  return rc;
}

int orc_run_segment(const double* edges, int32_t cells, const orc_material* mats,
                    double t_begin, double t_end, uint64_t seed, int32_t step,
                    uint64_t histories_total, int32_t batches, const orc_particle* source,
                    uint64_t n, uint64_t h_begin, const double* centers, double rho,
                    int32_t chunk, orc_tallies* t, orc_counters* counters,
                    uint64_t* tracks_per_cell, orc_bank* census, uint32_t* max_stack_runs) {
  seg_ctx c;
  memset(&c, 0, sizeof c);
  if (mesh_init(&c.mesh, edges, cells)) {
    mesh_free(&c.mesh);
    return -1;
  }
  c.mats = mats;
  c.t_begin = t_begin;
  c.t_end = t_end;
  c.seed = seed;
  c.step = step;
  c.histories_total = histories_total;
  c.batches = batches;
  c.centers = centers;
  c.rho = rho;
  const int rc = run_segment_ctx(&c, source, n, h_begin, chunk, t, counters,
                                 tracks_per_cell, census, max_stack_runs);
  mesh_free(&c.mesh);
  return rc;
}

/* ------------------------------------------------------------- tallies --- */
/* tally.cpp:43-48: histories in batch b under the contiguous-slice rule. */
static uint64_t batch_size(uint64_t H, int B, int b) {
  const uint64_t lo = ((uint64_t)b * H + (uint64_t)B - 1) / (uint64_t)B;
  const uint64_t hi = ((uint64_t)(b + 1) * H + (uint64_t)B - 1) / (uint64_t)B;
  return hi - lo;
}

/* tally.cpp:68-128 */
int orc_report(int32_t I, int32_t B, const orc_tallies* t, uint64_t histories,
               uint64_t histories_total, double normalization, int32_t snapshot,
               double* phi_track, double* sigma, double* phi_census, double* current,
               double* closure, double* edge, double* scalars) {
  double norm;
  if (snapshot) {
    if (histories == 0) {
      set_err("partial snapshot needs histories >= 1");
      return -1;
    }
    if (histories_total == 0) histories_total = histories;
    if (normalization <= 0.0) normalization = (double)histories_total;
    norm = normalization * (double)histories / (double)histories_total;
  } else {
    if (histories == 0) {
      set_err("finalize needs histories >= 1");
      return -1;
    }
    if (t->histories_scored != histories) {
      set_err("finalize: histories_scored does not match");
      return -1;
    }
    if (normalization <= 0.0) normalization = (double)histories;
    norm = normalization;
  }
  /* means_only, tally.cpp:51-66 */
  const double inv_h = 1.0 / norm;
  for (int i = 0; i < I; ++i) {
    phi_track[i] = t->track_flux[i] * inv_h;
    phi_census[i] = t->census_phi[i] * inv_h;
    current[i] = t->census_current[i] * inv_h;
    closure[i] = t->census_closure[i] * inv_h;
  }
  for (int e = 0; e <= I; ++e) edge[e] = t->edge_current[e] * inv_h;
  scalars[0] = t->boundary_closure_left * inv_h;
  scalars[1] = t->boundary_closure_right * inv_h;
  double cw = 0.0;
  for (int b = 0; b < B; ++b) cw += t->census_weight_batch[b];
  scalars[2] = cw * inv_h;
  scalars[3] = 0.0;
  scalars[4] = 0.0;
  if (sigma)
    for (int i = 0; i < I; ++i) sigma[i] = 0.0;
  if (!snapshot && B >= 2 && histories >= (uint64_t)B) {
    const double scale = (double)histories / normalization;
    double* inv_nb = (double*)malloc(sizeof(double) * (size_t)B);
    for (int b = 0; b < B; ++b) {
      const uint64_t nb = batch_size(histories, B, b);
      inv_nb[b] = nb ? 1.0 / (double)nb : 0.0;
    }
    const double ih = 1.0 / (double)histories;
    scalars[4] = 1.0;
    if (sigma)
      for (int i = 0; i < I; ++i) {
        const double mean = t->track_flux[i] * ih;
        double ss = 0.0;
        for (int b = 0; b < B; ++b) {
          const double bm = t->track_flux_batch[(size_t)b * I + i] * inv_nb[b];
          const double d = bm - mean;
          ss += d * d;
        }
        sigma[i] = scale * sqrt(ss / ((double)B * (B - 1)));
      }
    double wsum = 0.0;
    for (int b = 0; b < B; ++b) wsum += t->census_weight_batch[b];
    const double wmean = wsum * ih;
    double ss = 0.0;
    for (int b = 0; b < B; ++b) {
      const double bm = t->census_weight_batch[b] * inv_nb[b];
      const double d = bm - wmean;
      ss += d * d;
    }
    scalars[3] = scale * sqrt(ss / ((double)B * (B - 1)));
    free(inv_nb);
  }
  return 0;
}

/* ---------------------------------------------------------------- LOSM --- */
/* banded.cpp:8-38 (in place on copies). */
int orc_solve_tridiagonal(int32_t n, const double* lower, const double* diag,
                          const double* upper, const double* rhs, double* x) {
  double* a = (double*)malloc(sizeof(double) * (size_t)n * 5);
  double* b = a + n;
  double* c = b + n;
  double* r = c + n;
  double* fill = r + n;
  memcpy(a, lower, sizeof(double) * (size_t)n);
  memcpy(b, diag, sizeof(double) * (size_t)n);
  memcpy(c, upper, sizeof(double) * (size_t)n);
  memcpy(r, rhs, sizeof(double) * (size_t)n);
  memset(fill, 0, sizeof(double) * (size_t)n);
  int rc = 0;
  for (int k = 0; k + 1 < n; ++k) {
    if (fabs(a[k + 1]) > fabs(b[k])) {
      double tmp;
      tmp = b[k]; b[k] = a[k + 1]; a[k + 1] = tmp;
      tmp = c[k]; c[k] = b[k + 1]; b[k + 1] = tmp;
      if (k + 2 < n) { tmp = fill[k]; fill[k] = c[k + 1]; c[k + 1] = tmp; }
      tmp = r[k]; r[k] = r[k + 1]; r[k + 1] = tmp;
    }
    if (b[k] == 0.0) { rc = -1 - k; goto done; }
    const double m = a[k + 1] / b[k];
    a[k + 1] = 0.0;
    b[k + 1] -= m * c[k];
    if (k + 2 < n) c[k + 1] -= m * fill[k];
    r[k + 1] -= m * r[k];
  }
  if (b[n - 1] == 0.0) { rc = -n; goto done; }
  x[n - 1] = r[n - 1] / b[n - 1];
  if (n >= 2) x[n - 2] = (r[n - 2] - c[n - 2] * x[n - 1]) / b[n - 2];
  for (int k = n - 3; k >= 0; --k) x[k] = (r[k] - c[k] * x[k + 1] - fill[k] * x[k + 2]) / b[k];
done:
  if (rc) set_err("singular low-order system at pivot row %d", -1 - rc);
  free(a);
  return rc;
}

static double removal(const orc_material* m) {
  return m->sigma_t - m->sigma_s - m->nu_f * m->sigma_f; /* material.hpp:15 */
}

/* losm.cpp:43-165: check_inputs + assemble + solve + unpack. */
int orc_assemble_solve(int32_t I, const double* edges, const orc_material* mats,
                       const double* phi_prev, const double* J_prev, double J_L, double J_R,
                       int32_t implicit, const double* F_now, double PL_now, double PR_now,
                       const double* F_prev, double PL_prev, double PR_prev, double theta,
                       double dt, const double* q, double* phi_out, double* J_out) {
  if (!(theta >= 0.5 && theta <= 1.0)) { set_err("theta must lie in [1/2, 1]"); return -1; }
  if (!(dt > 0.0)) { set_err("dt must be > 0"); return -1; }
  for (int i = 0; i < I + 2; ++i)
    if (!isfinite(phi_prev[i])) { set_err("NaN in previous flux"); return -1; }
  for (int i = 0; i < I + 1; ++i)
    if (!isfinite(J_prev[i])) { set_err("NaN in previous current"); return -1; }
  for (int i = 0; i < I + 2; ++i)
    if (!isfinite(F_prev[i])) { set_err("NaN in closures"); return -1; }

  const int n = 2 * I + 3;
  double* lo = (double*)calloc((size_t)n * 5, sizeof(double));
  double* di = lo + n;
  double* up = di + n;
  double* rh = up + n;
  double* u = rh + n;
  const double* Fs = implicit ? F_now : F_prev;
  const double PLs = implicit ? PL_now : PL_prev;
  const double PRs = implicit ? PR_now : PR_prev;
  /* ghost widths, mesh.hpp:30-33 */
#define GW(i) (((i) <= 0 || (i) >= I + 1) ? 0.0 : (edges[(i)] - edges[(i)-1]))
#define QQ(i) (q ? q[(i)] : 0.0)

  di[0] = 0.5; /* left boundary row, losm.cpp:88-91 */
  up[0] = 1.0;
  rh[0] = 2.0 * J_L + PLs;
  for (int i = 1; i <= I; ++i) { /* balance rows, losm.cpp:94-104 */
    const int m = 2 * i;
    const double dx = GW(i);
    const orc_material* mt = &mats[i - 1];
    const double tau = dx / (mt->speed * dt);
    lo[m] = -theta;
    di[m] = tau + theta * removal(mt) * dx;
    up[m] = theta;
    rh[m] = tau * phi_prev[i] + theta * QQ(i - 1) +
            (theta - 1.0) * (J_prev[i] - J_prev[i - 1] + removal(mt) * dx * phi_prev[i] -
                             QQ(i - 1));
  }
  for (int i = 0; i <= I; ++i) { /* first-moment rows, losm.cpp:107-130 */
    const int m = 2 * i + 1;
    const double dx_l = GW(i);
    const double dx_r = GW(i + 1);
    const double dx_hat = 0.5 * (dx_r + dx_l);
    double num_sig = 0.0, num_vel = 0.0;
    if (dx_l > 0.0) {
      num_sig += mats[i - 1].sigma_t * dx_l;
      num_vel += dx_l / mats[i - 1].speed;
    }
    if (dx_r > 0.0) {
      num_sig += mats[i].sigma_t * dx_r;
      num_vel += dx_r / mats[i].speed;
    }
    const double sig_hat = num_sig / (dx_l + dx_r);
    const double inv_speed_hat = num_vel / (dx_l + dx_r);
    const double tau = dx_hat * inv_speed_hat / dt;
    lo[m] = -theta / 3.0;
    di[m] = tau + theta * sig_hat * dx_hat;
    up[m] = theta / 3.0;
    rh[m] = tau * J_prev[i] + theta * (Fs[i + 1] - Fs[i]) +
            (theta - 1.0) * ((phi_prev[i + 1] - phi_prev[i]) / 3.0 +
                             sig_hat * dx_hat * J_prev[i] - (F_prev[i + 1] - F_prev[i]));
  }
  {
    const int m = 2 * I + 2; /* right boundary row, losm.cpp:133-136 */
    lo[m] = 1.0;
    di[m] = -0.5;
    rh[m] = 2.0 * J_R - PRs;
  }
#undef GW
#undef QQ
  const int rc = orc_solve_tridiagonal(n, lo, di, up, rh, u);
  if (rc == 0) {
    for (int i = 0; i <= I + 1; ++i) phi_out[i] = u[2 * i];
    for (int i = 0; i <= I; ++i) J_out[i] = u[2 * i + 1];
  }
  free(lo);
  return rc ? -1 : 0;
}

/* losm.cpp:12-32 */
int orc_edge_currents(const double* cc, int32_t I, const double* edges, double* out) {
  if (I < 2) {
    set_err("edge interpolation needs at least two cells");
    return -1;
  }
  out[0] = cc[0];
  out[I] = cc[I - 1];
  for (int e = 1; e < I; ++e) {
    const double xl = 0.5 * (edges[e - 1] + edges[e]);
    const double xr = 0.5 * (edges[e] + edges[e + 1]);
    const double t = (edges[e] - xl) / (xr - xl);
    out[e] = (1.0 - t) * cc[e - 1] + t * cc[e];
  }
  return 0;
}

/* filters.cpp:11-24 */
int orc_moving_average(const double* g, int32_t M, int32_t k, double* out) {
  if (k < 0) {
    set_err("moving average half-width must be >= 0");
    return -1;
  }
  if (k == 0 || M == 0) {
    memmove(out, g, sizeof(double) * (size_t)M);
    return 0;
  }
  for (int m = 0; m < M; ++m) {
    int km = k;
    if (m < km) km = m;
    if (M - 1 - m < km) km = M - 1 - m;
    double sum = 0.0;
    for (int l = -km; l <= km; ++l) sum += g[m + l];
    out[m] = sum / (2 * km + 1);
  }
  return 0;
}

/* filters.cpp:26-52: direct O(M^2) transform. std::polar(1, a) is (cos a, sin
 * a); real * complex scales both parts; the synthesis multiplies complex
 * numbers as (ac - bd) + (ad + bc)i; modes with min(j, M-j) > cutoff are
 * zeroed and skipped (spectrum == 0+0i). Only the real part is kept. */
int orc_fourier_lowpass(const double* g, int32_t M, int32_t cutoff, double* out) {
  if (cutoff < 0) {
    set_err("fourier cutoff must be >= 0");
    return -1;
  }
  if (M <= 1) {
    memmove(out, g, sizeof(double) * (size_t)(M > 0 ? M : 0));
    return 0;
  }
  const double w0 = 2.0 * 3.141592653589793 / M; /* std::numbers::pi */
  double* sre = (double*)calloc((size_t)M, sizeof(double));
  double* sim = (double*)calloc((size_t)M, sizeof(double));
  for (int j = 0; j < M; ++j) {
    const int mj = j < M - j ? j : M - j;
    if (mj > cutoff) continue;
    double re = 0.0, im = 0.0;
    for (int m = 0; m < M; ++m) {
      const double a = -w0 * j * m;
      re += g[m] * cos(a);
      im += g[m] * sin(a);
    }
    sre[j] = re;
    sim[j] = im;
  }
  for (int m = 0; m < M; ++m) {
    double re = 0.0;
    for (int j = 0; j < M; ++j) {
      if (sre[j] == 0.0 && sim[j] == 0.0) continue;
      const double a = w0 * j * m;
      const double c = cos(a), d = sin(a);
      re += sre[j] * c - sim[j] * d;
    }
    out[m] = re / M;
  }
  free(sre);
  free(sim);
  return 0;
}

/* ww.cpp:8-32 */
int orc_build_centers(const double* phi, int32_t n, double eps_min, double rho,
                      double* centers) {
  if (!(eps_min > 0.0 && eps_min < 1.0)) { set_err("eps_min must lie in (0,1)"); return -1; }
  if (!(rho >= 1.0)) { set_err("rho must be >= 1"); return -1; }
  double mx = 0.0;
  for (int i = 0; i < n; ++i)
    if (phi[i] > mx) mx = phi[i];
  for (int i = 0; i < n; ++i) centers[i] = 1.0;
  if (!(mx > 0.0) || !isfinite(mx)) return 1;
  for (int i = 0; i < n; ++i) {
    const double cl = phi[i] > 0.0 ? phi[i] : 0.0;
    centers[i] = (cl / mx) * (1.0 - eps_min) + eps_min;
  }
  return 0;
}

/* ww.cpp:74-87 */
int orc_update_thresholds(uint64_t H, const double* f, int32_t n, uint64_t* out) {
  double prev = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!(f[i] > prev && f[i] < 1.0)) {
      set_err("update fractions must increase within (0,1)");
      return -1;
    }
    prev = f[i];
    out[i] = (uint64_t)ceil(f[i] * (double)H);
  }
  return 0;
}

/* popctrl.cpp:7-42 */
int orc_uniform_comb(const orc_particle* bank, uint64_t n, uint64_t target, uint64_t seed,
                     uint64_t stream_id, orc_particle* out, double* in_w, double* out_w) {
  if (n == 0) { set_err("cannot comb an empty bank"); return -1; }
  if (target < 1) { set_err("comb target must be positive"); return -1; }
  orc_rng r;
  rng_init(&r, seed, stream_id);
  double W = 0.0;
  for (uint64_t i = 0; i < n; ++i) W += bank[i].w;
  const double spacing = W / (double)target;
  const double offset = rng_uniform(&r) * spacing;
  double cum = 0.0;
  uint64_t tooth = 0;
  for (uint64_t i = 0; i < n; ++i) {
    cum += bank[i].w;
    while (tooth < target && offset + (double)tooth * spacing < cum) {
      out[tooth] = bank[i];
      out[tooth].w = spacing;
      ++tooth;
    }
  }
  while (tooth < target) {
    out[tooth] = bank[n - 1];
    out[tooth].w = spacing;
    ++tooth;
  }
  double ow = 0.0;
  for (uint64_t i = 0; i < target; ++i) ow += out[i].w;
  *in_w = W;
  *out_w = ow;
  return 0;
}

/* -------------------------------------------------------------- driver --- */
typedef struct {
  orc_config cfg;
  double* edges;
  double* layers;
  orc_material* mats;
  orc_mesh mesh;
  int I, B;
  orc_bank bank;
  int next_step;
  /* RunState, driver.hpp:80-86 */
  int has_prev_report;
  double *prev_phi_census, *prev_current, *prev_closure, *prev_phi_track;
  double prev_PL, prev_PR;
  int has_prev_grid;
  double* prev_grid;
  /* last StepRecord arrays */
  double *r_phi_track, *r_sigma, *r_phi_census, *r_current, *r_closure, *r_edge;
  double *r_centers, *r_hybrid;
  uint64_t* r_tracks;
  int r_has_centers, r_has_hybrid;
  double* q_step; /* volumetric-source LOSM q of the current step, or NULL */
} orc_driver;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* filters.cpp:54-87: apply_filter (config.hpp filter(): moving average for
 * hww_ma, Fourier low-pass for hww_fourier, none otherwise). */
static int apply_filter(const double* g, int len, const orc_config* c, double* out) {
  if (c->mode == 3) return orc_moving_average(g, len, c->ma_base_k, out);
  return orc_fourier_lowpass(g, len, c->fourier_cutoff, out);
}
static int filter_interior(double* g, int len, const orc_config* c) {
  if ((c->mode != 3 && c->mode != 4) || len <= 2) return 0; /* FilterSpec::none */
  double* tmp = (double*)malloc(sizeof(double) * (size_t)len);
  const int rc = apply_filter(g + 1, len - 2, c, tmp);
  memcpy(g + 1, tmp, sizeof(double) * (size_t)(len - 2));
  free(tmp);
  return rc;
}
static int filter_all(double* g, int len, const orc_config* c) {
  if (c->mode != 3 && c->mode != 4) return 0;
  double* tmp = (double*)malloc(sizeof(double) * (size_t)len);
  const int rc = apply_filter(g, len, c, tmp);
  memcpy(g, tmp, sizeof(double) * (size_t)len);
  free(tmp);
  return rc;
}

/* driver.cpp:29-37 */
static void extrap(const double* cells, int I, double* out) {
  out[0] = cells[0];
  memcpy(out + 1, cells, sizeof(double) * (size_t)I);
  out[I + 1] = cells[I - 1];
}

/* config.cpp:27-69 (the subset the drivers need to agree on). */
static int validate(const orc_config* c) {
  const int hybrid = c->mode >= 2;
  if (!(c->sigma_t > 0) || c->sigma_s < 0 || c->sigma_s > c->sigma_t || c->sigma_f < 0 ||
      c->sigma_f > c->sigma_t || c->sigma_s + c->sigma_f > c->sigma_t || c->nu_f < 0 ||
      !(c->speed > 0)) { set_err("invalid material"); return -1; }
  if (c->histories_per_step < 1) { set_err("histories_per_step must be >= 1"); return -1; }
  if (!(c->theta >= 0.5 && c->theta <= 1.0)) { set_err("theta must lie in [1/2, 1]"); return -1; }
  if (!(c->rho >= 1.0)) { set_err("rho must be >= 1"); return -1; }
  if (!(c->eps_min > 0.0 && c->eps_min < 1.0)) { set_err("eps_min must lie in (0,1)"); return -1; }
  if (c->u_ww < 0) { set_err("u_ww must be >= 0"); return -1; }
  if (hybrid) {
    if (c->n_fractions != c->u_ww) { set_err("update_fractions count must equal u_ww"); return -1; }
    double prev = 0.0;
    for (int i = 0; i < c->n_fractions; ++i) {
      if (!(c->fractions[i] > 0.0 && c->fractions[i] < 1.0) || !(c->fractions[i] > prev)) {
        set_err("bad update fractions");
        return -1;
      }
      prev = c->fractions[i];
    }
  }
  if (c->mode == 3 && c->ma_base_k < 0) { set_err("ma_base_k must be >= 0"); return -1; }
  if (c->mode == 4 && c->fourier_cutoff < 0) { set_err("fourier_cutoff must be >= 0"); return -1; }
  if (c->batches < 2) { set_err("batches must be >= 2"); return -1; }
  if (!(c->x_min < c->x_max) || c->cells < 1 || !(c->t_end > 0.0) || c->time_steps < 1 ||
      (!c->no_pulse && (!(c->strength > 0.0) || c->x0 < c->x_min || c->x0 > c->x_max))) {
    set_err("invalid geometry/time/source");
    return -1;
  }
  if (c->n_regions < 0 || c->n_regions > 8) { set_err("n_regions must lie in [0, 8]"); return -1; }
  for (int r = 0; r < c->n_regions; ++r) {
    const double* m = c->region_mat[r];
    if (!(m[0] > 0) || m[1] < 0 || m[1] + m[2] > m[0] || m[2] < 0 || m[3] < 0 || !(m[4] > 0) ||
        (r > 0 && !(c->region_x_hi[r] > c->region_x_hi[r - 1]))) {
      set_err("invalid material region");
      return -1;
    }
  }
  if (c->vol_rate > 0.0 && (!(c->vol_x_lo < c->vol_x_hi) || c->vol_x_lo < c->x_min ||
                            c->vol_x_hi > c->x_max || !(c->vol_t_lo < c->vol_t_hi) ||
                            c->vol_histories < 1)) {
    set_err("invalid volumetric source");
    return -1;
  }
  if (c->no_pulse && !(c->vol_rate > 0.0)) { set_err("no source at all"); return -1; }
  return 0;
}

void* orc_driver_create(const orc_config* c) {
  if (validate(c)) return NULL;
  orc_driver* d = (orc_driver*)calloc(1, sizeof(orc_driver));
  d->cfg = *c;
  d->I = c->cells;
  d->B = c->batches;
  const int I = d->I;
  d->edges = (double*)malloc(sizeof(double) * (size_t)(I + 1));
  orc_uniform_edges(c->x_min, c->x_max, I, d->edges);
  mesh_init(&d->mesh, d->edges, I);
  d->layers = (double*)malloc(sizeof(double) * (size_t)(c->time_steps + 1));
  { /* time_grid.hpp:22-29 */
    const double dt = (c->t_end - 0.0) / c->time_steps;
    for (int n = 0; n <= c->time_steps; ++n) d->layers[n] = 0.0 + n * dt;
    d->layers[c->time_steps] = c->t_end;
  }
  d->mats = (orc_material*)malloc(sizeof(orc_material) * (size_t)I);
  for (int i = 0; i < I; ++i) {
    d->mats[i].sigma_t = c->sigma_t;
    d->mats[i].sigma_s = c->sigma_s;
    d->mats[i].sigma_f = c->sigma_f;
    d->mats[i].nu_f = c->nu_f;
    d->mats[i].speed = c->speed;
    if (c->n_regions > 0) { /* first region whose upper bound exceeds the cell centre */
      const double xc = 0.5 * (d->edges[i] + d->edges[i + 1]);
      int r = 0;
      while (r < c->n_regions - 1 && !(xc < c->region_x_hi[r])) ++r;
      d->mats[i].sigma_t = c->region_mat[r][0];
      d->mats[i].sigma_s = c->region_mat[r][1];
      d->mats[i].sigma_f = c->region_mat[r][2];
      d->mats[i].nu_f = c->region_mat[r][3];
      d->mats[i].speed = c->region_mat[r][4];
    }
  }
  if (!c->no_pulse) {
    d->bank.cap = d->bank.n = c->histories_per_step;
    d->bank.data = (orc_particle*)malloc(sizeof(orc_particle) * d->bank.n);
    orc_pulse_source(c->seed, c->histories_per_step, c->x0, c->strength, d->bank.data);
  }
  d->next_step = 1;
  double** arrs[] = {&d->prev_phi_census, &d->prev_current, &d->prev_closure,
                     &d->prev_phi_track, &d->prev_grid, &d->r_phi_track, &d->r_sigma,
                     &d->r_phi_census, &d->r_current, &d->r_closure, &d->r_centers,
                     &d->r_hybrid};
  for (size_t i = 0; i < sizeof arrs / sizeof arrs[0]; ++i)
    *arrs[i] = (double*)calloc((size_t)I + 2, sizeof(double));
  d->r_edge = (double*)calloc((size_t)I + 1, sizeof(double));
  d->r_tracks = (uint64_t*)calloc((size_t)I, sizeof(uint64_t));
  return d;
}

void orc_driver_destroy(void* h) {
  orc_driver* d = (orc_driver*)h;
  if (!d) return;
  free(d->edges); free(d->layers); free(d->mats); mesh_free(&d->mesh);
  orc_bank_free(&d->bank);
  free(d->prev_phi_census); free(d->prev_current); free(d->prev_closure);
  free(d->prev_phi_track); free(d->prev_grid);
  free(d->r_phi_track); free(d->r_sigma); free(d->r_phi_census); free(d->r_current);
  free(d->r_closure); free(d->r_edge); free(d->r_centers); free(d->r_hybrid);
  free(d->r_tracks);
  free(d);
}

typedef struct {
  double *phi, *J, *F, PL, PR; /* filtered HybridInputs (driver.hpp:15-21) */
} hyb_inputs;

/* driver.cpp:72-95 */
static int hybrid_windows(orc_driver* d, const hyb_inputs* prev, int implicit,
                          const double* F_now, double PL_now, double PR_now, double theta,
                          double dt, int* active, double* centers, double* phi_hybrid,
                          int* has_hybrid) {
  const int I = d->I;
  double* phi_out = (double*)malloc(sizeof(double) * (size_t)(I + 2));
  double* J_out = (double*)malloc(sizeof(double) * (size_t)(I + 1));
  const int rc = orc_assemble_solve(I, d->edges, d->mats, prev->phi, prev->J, 0.0, 0.0,
                                    implicit, F_now, PL_now, PR_now, prev->F, prev->PL,
                                    prev->PR, theta, dt, d->q_step, phi_out, J_out);
  int ok = 1;
  if (rc == 0) {
    memcpy(phi_hybrid, phi_out + 1, sizeof(double) * (size_t)I);
    *has_hybrid = 1;
    orc_build_centers(phi_hybrid, I, d->cfg.eps_min, d->cfg.rho, centers);
    *active = 1;
  } else {
    if (!*active) {
      for (int i = 0; i < I; ++i) centers[i] = 1.0;
      *active = 1;
    }
    fprintf(stderr, "warning: low-order solve failed (%s); keeping previous windows\n",
            g_err);
    ok = 0;
  }
  free(phi_out);
  free(J_out);
  return ok;
}

/* driver.cpp:99-284 */
int orc_driver_step(void* h, orc_step_out* out) {
  orc_driver* d = (orc_driver*)h;
  const orc_config* c = &d->cfg;
  const int I = d->I, B = d->B;
  if (d->next_step > c->time_steps) {
    set_err("run already complete");
    return -1;
  }
  const int step = d->next_step;
  memset(out, 0, sizeof *out);
  out->step = step;
  out->t_begin = d->layers[step - 1];
  out->t_end = d->layers[step];
  const double dt = d->layers[step] - d->layers[step - 1];
  const double t0 = now_s();
  const uint64_t target = c->target_population ? c->target_population : c->histories_per_step;

  /* population control, driver.cpp:111-129 */
  orc_bank source = {0};
  const double bank_cap = c->comb_overflow_factor * (double)target;
  if (d->bank.n == 0 && (c->no_pulse || c->vol_rate > 0.0)) {
    /* volumetric-source runs before any census exists: nothing to comb */
    out->comb_in = out->comb_out = 0;
  } else if (c->comb_overflow_factor <= 1.0 || (double)d->bank.n > bank_cap) {
    if (d->bank.n == 0) {
      set_err("cannot comb an empty bank");
      return -1;
    }
    source.n = source.cap = target;
    source.data = (orc_particle*)malloc(sizeof(orc_particle) * target);
    orc_uniform_comb(d->bank.data, d->bank.n, target, c->seed,
                     orc_stream_id((uint64_t)step, 0, P_COMB), source.data,
                     &out->comb_in_weight, &out->comb_out_weight);
    out->comb_in = d->bank.n;
    out->comb_out = target;
    orc_bank_free(&d->bank);
  } else {
    double w = 0.0;
    for (uint64_t i = 0; i < d->bank.n; ++i) w += d->bank.data[i].w;
    out->comb_in = out->comb_out = d->bank.n;
    out->comb_in_weight = out->comb_out_weight = w;
    source = d->bank;
    memset(&d->bank, 0, sizeof d->bank);
  }
  /* volumetric source particles born in this step follow the combed census */
  double* qv = NULL;
  if (c->vol_rate > 0.0) {
    const double ta = out->t_begin > c->vol_t_lo ? out->t_begin : c->vol_t_lo;
    const double tb = out->t_end < c->vol_t_hi ? out->t_end : c->vol_t_hi;
    if (tb > ta) {
      const uint64_t n0 = source.n, nv = c->vol_histories;
      source.data = (orc_particle*)realloc(source.data, sizeof(orc_particle) * (n0 + nv));
      source.n = source.cap = n0 + nv;
      orc_volume_source(c->seed, step, nv, c->vol_x_lo, c->vol_x_hi, ta, tb, c->vol_rate,
                        c->histories_per_step, source.data + n0);
      qv = (double*)malloc(sizeof(double) * (size_t)I);
      orc_volume_q(d->edges, I, c->vol_x_lo, c->vol_x_hi, ta, tb, dt, c->vol_rate, qv);
    }
  }
  d->q_step = qv;
  const uint64_t H = source.n;

  /* windows, driver.cpp:136-167 */
  int active = 0;
  double* centers = (double*)calloc((size_t)I, sizeof(double));
  hyb_inputs fin = {0};
  fin.phi = (double*)calloc((size_t)I + 2, sizeof(double));
  fin.J = (double*)calloc((size_t)I + 1, sizeof(double));
  fin.F = (double*)calloc((size_t)I + 2, sizeof(double));
  const double theta_eff = step == 1 ? 1.0 : c->theta;
  const int hybrid = c->mode >= 2;
  int failed = 0;
  d->r_has_hybrid = 0;
  if (c->mode == 1) { /* lww */
    if (d->has_prev_report) {
      if (orc_build_centers(d->prev_phi_track, I, c->eps_min, c->rho, centers) == 0)
        active = 1;
    }
  } else if (hybrid) {
    if (step == 1) { /* analytic_pulse_inputs, driver.cpp:51-61 */
      if (!c->no_pulse) {
        const int cell = mesh_locate(&d->mesh, c->x0);
        fin.phi[cell + 1] = c->speed * c->strength / d->mesh.widths[cell];
      }
    } else { /* hybrid_inputs_from_report, driver.cpp:41-49 */
      extrap(d->prev_phi_census, I, fin.phi);
      extrap(d->prev_closure, I, fin.F);
      if (orc_edge_currents(d->prev_current, I, d->edges, fin.J)) return -1;
      fin.PL = d->prev_PL;
      fin.PR = d->prev_PR;
    }
    /* apply_filter_pipeline(nullptr, F, phi, J), filters.cpp:76-84 */
    filter_interior(fin.F, I + 2, c);
    filter_interior(fin.phi, I + 2, c);
    filter_all(fin.J, I + 1, c);
    if (d->has_prev_grid) {
      memcpy(centers, d->prev_grid, sizeof(double) * (size_t)I);
      active = 1;
    }
    failed = !hybrid_windows(d, &fin, 0, NULL, 0.0, 0.0, theta_eff, dt, &active, centers,
                             d->r_hybrid, &d->r_has_hybrid) ||
             failed;
  }

  /* thresholds, driver.cpp:170-177 */
  uint64_t thr[8];
  int nthr = 0;
  if (hybrid && c->u_ww > 0) {
    uint64_t raw[8];
    orc_update_thresholds(H, c->fractions, c->n_fractions, raw);
    for (int i = 0; i < c->n_fractions; ++i) {
      if (raw[i] >= H) continue;
      if (nthr > 0 && raw[i] <= thr[nthr - 1]) continue;
      thr[nthr++] = raw[i];
    }
  }
  out->n_thresholds = nthr;
  for (int i = 0; i < nthr; ++i) out->thresholds[i] = thr[i];

  /* segments, driver.cpp:181-219 */
  seg_ctx sc;
  memset(&sc, 0, sizeof sc);
  sc.mesh = d->mesh;
  sc.mats = d->mats;
  sc.t_begin = out->t_begin;
  sc.t_end = out->t_end;
  sc.seed = c->seed;
  sc.step = step;
  sc.histories_total = H;
  sc.batches = B;
  sc.rho = c->rho;
  owned_tallies tl;
  tallies_alloc(&tl, I, B);
  orc_counters k;
  memset(&k, 0, sizeof k);
  memset(d->r_tracks, 0, sizeof(uint64_t) * (size_t)I);
  orc_bank census = {0};
  uint64_t h_done = 0;
  int rc = 0;
  double* snap = (double*)malloc(sizeof(double) * (size_t)(5 * I + 8));
  double* F_now = (double*)malloc(sizeof(double) * (size_t)(I + 2));
  for (int u = 0; u <= nthr && rc == 0; ++u) {
    const uint64_t h_stop = u < nthr ? thr[u] : H;
    sc.centers = active ? centers : NULL;
    rc = run_segment_ctx(&sc, source.data + h_done, h_stop - h_done, h_done, 256, &tl.t, &k,
                         d->r_tracks, &census, NULL);
    h_done = h_stop;
    if (rc || u == nthr) break;
    /* partial_snapshot + implicit closure, driver.cpp:206-217 */
    double* s_phi = snap;
    double* s_cphi = s_phi + I;
    double* s_cur = s_cphi + I;
    double* s_clo = s_cur + I;
    double* s_edge = s_clo + I;
    double* s_sc = s_edge + I + 1;
    orc_report(I, B, &tl.t, h_done, H, (double)c->histories_per_step, 1, s_phi, NULL, s_cphi,
               s_cur, s_clo, s_edge, s_sc);
    extrap(s_clo, I, F_now);
    filter_interior(F_now, I + 2, c);
    const int ok = hybrid_windows(d, &fin, 1, F_now, s_sc[0], s_sc[1], theta_eff, dt, &active,
                                  centers, d->r_hybrid, &d->r_has_hybrid);
    failed = failed || !ok;
    if (ok) ++out->updates_applied;
  }
  free(snap);
  free(F_now);
  if (rc) {
    free(tl.block);
    orc_bank_free(&census);
    orc_bank_free(&source);
    free(d->q_step);
    d->q_step = NULL;
    free(centers);
    free(fin.phi); free(fin.J); free(fin.F);
    return -1;
  }

  /* finalize, driver.cpp:221-229 */
  double sc5[5];
  if (orc_report(I, B, &tl.t, H, H, (double)c->histories_per_step, 0, d->r_phi_track,
                 d->r_sigma, d->r_phi_census, d->r_current, d->r_closure, d->r_edge, sc5))
    return -1;
  out->tau = now_s() - t0;
  out->histories = H;
  out->hybrid_solve_failed = failed;
  out->counters = k;
  uint64_t seg = 0;
  for (int i = 0; i < I; ++i) seg += d->r_tracks[i];
  out->segments = seg;
  out->census_weight = sc5[2];
  out->census_weight_sigma = sc5[3];
  out->boundary_closure_left = sc5[0];
  out->boundary_closure_right = sc5[1];
  out->sigma_valid = (int)sc5[4];
  /* fom without a reference, driver.cpp:272-275; metrics.cpp:34-55 */
  out->fom_sigma_l2 = NAN;
  if (out->sigma_valid) {
    const double tau = out->tau > 1e-9 ? out->tau : 1e-9;
    double sum = 0.0;
    for (int i = 0; i < I; ++i) {
      if (d->r_sigma[i] == 0.0) continue;
      const double f = 1.0 / (tau * d->r_sigma[i] * d->r_sigma[i]);
      sum += f * f * d->mesh.widths[i];
    }
    out->fom_sigma_l2 = sqrt(sum);
  }
  d->r_has_centers = active;
  if (active) memcpy(d->r_centers, centers, sizeof(double) * (size_t)I);
  out->has_windows = active;
  out->has_hybrid = d->r_has_hybrid;

  /* state hand-off, driver.cpp:278-281 */
  orc_bank_free(&d->bank);
  d->bank = census;
  out->census_size = census.n;
  d->has_prev_report = 1;
  memcpy(d->prev_phi_census, d->r_phi_census, sizeof(double) * (size_t)I);
  memcpy(d->prev_current, d->r_current, sizeof(double) * (size_t)I);
  memcpy(d->prev_closure, d->r_closure, sizeof(double) * (size_t)I);
  memcpy(d->prev_phi_track, d->r_phi_track, sizeof(double) * (size_t)I);
  d->prev_PL = sc5[0];
  d->prev_PR = sc5[1];
  if (active) {
    memcpy(d->prev_grid, centers, sizeof(double) * (size_t)I);
    d->has_prev_grid = 1;
  }
  free(tl.block);
  orc_bank_free(&source);
  free(d->q_step);
  d->q_step = NULL;
  free(centers);
  free(fin.phi); free(fin.J); free(fin.F);
  ++d->next_step;
  return 0;
}

void orc_driver_arrays(void* h, double* phi_track, double* phi_sigma, double* phi_census,
                       double* current_census, double* closure_census, double* edge_current,
                       double* ww_centers, double* phi_hybrid, uint64_t* tracks_per_cell) {
  orc_driver* d = (orc_driver*)h;
  const size_t I = (size_t)d->I;
  if (phi_track) memcpy(phi_track, d->r_phi_track, I * sizeof(double));
  if (phi_sigma) memcpy(phi_sigma, d->r_sigma, I * sizeof(double));
  if (phi_census) memcpy(phi_census, d->r_phi_census, I * sizeof(double));
  if (current_census) memcpy(current_census, d->r_current, I * sizeof(double));
  if (closure_census) memcpy(closure_census, d->r_closure, I * sizeof(double));
  if (edge_current) memcpy(edge_current, d->r_edge, (I + 1) * sizeof(double));
  if (ww_centers && d->r_has_centers) memcpy(ww_centers, d->r_centers, I * sizeof(double));
  if (phi_hybrid && d->r_has_hybrid) memcpy(phi_hybrid, d->r_hybrid, I * sizeof(double));
  if (tracks_per_cell) memcpy(tracks_per_cell, d->r_tracks, I * sizeof(uint64_t));
}

uint64_t orc_driver_bank(void* h, orc_particle* out, uint64_t cap) {
  orc_driver* d = (orc_driver*)h;
  if (out) memcpy(out, d->bank.data, (d->bank.n < cap ? d->bank.n : cap) * sizeof(orc_particle));
  return d->bank.n;
}
