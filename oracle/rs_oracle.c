/* oracle/rs_oracle.c — TEST INFRASTRUCTURE ONLY (see rs_oracle.h).
 *
 * A deliberately plain, single-threaded C restatement of the reference
 * routesim hot path.  It recomputes every router snapshot from scratch each
 * tick exactly as the reference does (no incremental aggregates), so it is
 * an independent check on the engine's incremental bookkeeping.  Compile
 * with -ffp-contract=off (oracle/Makefile): fp64 clocks must see separate
 * multiply/add roundings to match the reference.
 *
 * File:line citations are relative to /root/reference/proj/include/routesim.
 */
#include "rs_oracle.h"

#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

int ora_cmp_double(const void* a, const void* b);

/* ------------------------------------------------------------------ rng */

uint64_t ora_mix_seed(uint64_t seed, uint64_t stream) { /* rng.hpp:11-16 */
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* std::mt19937_64 (the engine of Rng, rng.hpp:21-27). */
typedef struct {
  uint64_t s[312];
  int idx;
} mt64;

static void mt64_seed(mt64* m, uint64_t seed) {
  m->s[0] = seed;
  for (int i = 1; i < 312; ++i) {
    m->s[i] = 6364136223846793005ULL * (m->s[i - 1] ^ (m->s[i - 1] >> 62)) + (uint64_t)i;
  }
  m->idx = 312;
}

static uint64_t mt64_next(mt64* m) {
  if (m->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (m->s[i] & 0xFFFFFFFF80000000ULL) | (m->s[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      m->s[i] = m->s[(i + 156) % 312] ^ xa;
    }
    m->idx = 0;
  }
  uint64_t y = m->s[m->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void ora_mt19937_64(uint64_t seed, int64_t count, uint64_t* out) {
  mt64 m;
  mt64_seed(&m, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = mt64_next(&m);
}

static double rng_uniform(mt64* m) { /* rng.hpp:29 */
  return (double)(mt64_next(m) >> 11) * 0x1.0p-53;
}

static uint64_t rng_uniform_below(mt64* m, uint64_t n) { /* rng.hpp:32-35 */
  uint64_t k = (uint64_t)(rng_uniform(m) * (double)n);
  return k < n ? k : n - 1;
}

/* ----------------------------------------------------- buckets, predictor */

static int bucket_of(const int64_t* edges, int n, int64_t tokens) { /* predictor.hpp:34-40 */
  int b = 0;
  for (int i = 1; i < n; ++i)
    if (tokens >= edges[i]) b = i;
  return b;
}

static int64_t upper_bound_tokens(const rs_batch_cfg* c, int bucket) { /* predictor.hpp:44-51 */
  if (bucket + 1 < c->n_predictor_edges) return c->predictor_edges[bucket + 1];
  return c->predictor_top_cap;
}

static int predict_one(const rs_batch_cfg* c, mt64* rng, int32_t prompt,
                       int32_t decode, uint8_t task, const uint8_t* given, int64_t i) {
  if (c->predictor_mode == RS_PREDICTOR_GIVEN) return given[i];
  if (c->predictor_mode == RS_PREDICTOR_EMPIRICAL) { /* predictor.hpp:146-158 */
    int band = bucket_of(c->band_edges, c->n_band_edges, prompt);
    return c->empirical_table[task][band];
  }
  /* predict_simulated, predictor.hpp:98-110 */
  int n = c->n_predictor_edges;
  int tb = bucket_of(c->predictor_edges, n, decode);
  if (n == 1) return 0;
  if (rng_uniform(rng) < c->accuracy[task]) return tb;
  if (tb == 0) return 1;
  if (tb == n - 1) return n - 2;
  return rng_uniform(rng) < 0.5 ? tb - 1 : tb + 1;
}

int ora_predict_buckets(const rs_batch_cfg* c, int64_t n, const int32_t* prompt,
                        const int32_t* decode, const uint8_t* task,
                        const uint8_t* given, uint64_t seed, uint8_t* out) {
  mt64* rng = (mt64*)malloc(sizeof(mt64));
  if (!rng) return -1;
  mt64_seed(rng, seed);
  for (int64_t i = 0; i < n; ++i)
    out[i] = (uint8_t)predict_one(c, rng, prompt[i], decode[i], task[i], given, i);
  free(rng);
  return 0;
}

/* ------------------------------------------------------------------ mlp */

/* Mlp::forward (mlp.hpp:54-68) with affine (mlp.hpp:139-152): acc = b[o];
 * acc += w[o][i] * x[i] in index order; ReLU on all but the last layer. */
static void mlp_forward(const rs_batch_cfg* c, const double* x, double* q) {
  double bufa[RS_MAX_WIDTH], bufb[RS_MAX_WIDTH];
  const double* p = c->rl_params;
  const double* cur = x;
  double* nxt = bufa;
  for (int l = 0; l < c->rl_num_layers; ++l) {
    int ni = c->rl_dims[l], no = c->rl_dims[l + 1];
    const double* w = p;
    const double* b = p + (size_t)ni * no;
    double* dst = (l + 1 == c->rl_num_layers) ? q : nxt;
    for (int o = 0; o < no; ++o) {
      double acc = b[o];
      for (int i = 0; i < ni; ++i) acc += w[(size_t)o * ni + i] * cur[i];
      dst[o] = acc;
    }
    if (l + 1 < c->rl_num_layers)
      for (int o = 0; o < no; ++o) dst[o] = dst[o] > 0.0 ? dst[o] : 0.0;
    p += (size_t)ni * no + no;
    cur = dst;
    nxt = (nxt == bufa) ? bufb : bufa;
  }
}

static int argmax_action(const double* q, int n) { /* dqn.hpp:82-90 */
  int best = 0;
  for (int a = 1; a < n; ++a)
    if (q[a] > q[best]) best = a;
  return best;
}

int ora_mlp_forward(const rs_batch_cfg* c, const double* states, int32_t batch,
                    double* q_out, int32_t* greedy_out) {
  if (c->rl_num_layers < 1 || c->rl_num_layers > RS_MAX_LAYERS) return -1;
  for (int l = 0; l <= c->rl_num_layers; ++l)
    if (c->rl_dims[l] < 1 || c->rl_dims[l] > RS_MAX_WIDTH) return -1;
  int din = c->rl_dims[0], dout = c->rl_dims[c->rl_num_layers];
  for (int b = 0; b < batch; ++b) {
    double* q = q_out + (size_t)b * dout;
    mlp_forward(c, states + (size_t)b * din, q);
    if (greedy_out) greedy_out[b] = argmax_action(q, dout);
  }
  return 0;
}

/* ------------------------------------------------------------ simulator */

typedef struct { /* Instance::RunningEntry, instance.hpp:91-95 */
  uint32_t req;
  int32_t prompt_remaining;
  uint64_t admit_seq;
} run_entry;

typedef struct { /* std::deque<uint32_t> as a ring */
  uint32_t* buf;
  int64_t cap, head, size;
} deque32;

static uint32_t dq_at(const deque32* d, int64_t i) { return d->buf[(d->head + i) % d->cap]; }
static void dq_push_back(deque32* d, uint32_t v) {
  d->buf[(d->head + d->size) % d->cap] = v;
  d->size++;
}
static void dq_push_front(deque32* d, uint32_t v) {
  d->head = (d->head + d->cap - 1) % d->cap;
  d->buf[d->head] = v;
  d->size++;
}
static void dq_erase(deque32* d, int64_t i) { /* erase(begin()+i), order kept */
  for (int64_t k = i; k + 1 < d->size; ++k)
    d->buf[(d->head + k) % d->cap] = d->buf[(d->head + k + 1) % d->cap];
  d->size--;
}

typedef struct {
  double clock;
  uint64_t admit_seq;
  run_entry* run;
  int32_t n_run;
  deque32 wait;
} inst_t;

typedef struct { /* InstanceFeatures (instance.hpp:69-83) + token mass */
  int32_t dbc[RS_MAX_BUCKETS];
  double capacity, t_hat_c;
  int64_t pending_prompt, out_dec_est, out_true, kv_in_use, free_kv;
  int64_t reserved, free_reserved, token_sum;
  int32_t running, waiting;
} feat_t;

typedef struct {
  const rs_batch_cfg* c;
  int64_t n;
  const double* arrival;
  const int32_t* prompt;
  const int32_t* decode;
  /* Request mutable fields (request.hpp:51-62) */
  int32_t* pred;
  int32_t* dest; /* decode_estimate_tokens */
  double *routed, *first, *completion;
  int32_t *emitted, *preempt, *assigned;
  inst_t* inst;
  deque32 rq; /* router_queue_ */
  int64_t cursor, completed, tick, infeasible;
  double clock;
  int32_t* scratch; /* per-iteration emission list */
  int error, error_instance;
} sim_t;

static int64_t dec_est(const sim_t* s, uint32_t r) { /* request.hpp:63-66 */
  return s->dest[r] > 0 ? s->dest[r] : s->decode[r];
}
static int64_t reserved_tokens(const sim_t* s, uint32_t r) { /* instance.hpp:365-368 */
  int64_t d = dec_est(s, r), e = s->emitted[r];
  return (int64_t)s->prompt[r] + (d > e ? d : e);
}
static int64_t decode_left(const sim_t* s, uint32_t r) { /* instance.hpp:370-372 */
  int64_t v = dec_est(s, r) - s->emitted[r];
  return v > 0 ? v : 0;
}
static int64_t footprint(const sim_t* s, const run_entry* e) { /* instance.hpp:375-378 */
  return (int64_t)(s->prompt[e->req] - e->prompt_remaining) + s->emitted[e->req];
}
static int64_t kv_in_use(const sim_t* s, const inst_t* I) {
  int64_t t = 0;
  for (int i = 0; i < I->n_run; ++i) t += footprint(s, &I->run[i]);
  return t;
}

static void admit_waiting(sim_t* s, inst_t* I) { /* instance.hpp:149-195 */
  const rs_batch_cfg* c = s->c;
  int64_t reserved = 0;
  for (int i = 0; i < I->n_run; ++i) reserved += reserved_tokens(s, I->run[i].req);
  while (I->wait.size > 0 && I->n_run < c->max_batch_size) {
    int64_t pick = I->wait.size;
    if (c->batching == RS_BATCHING_FCFS) {
      uint32_t h = dq_at(&I->wait, 0);
      if (reserved + reserved_tokens(s, h) <= c->kv_capacity_tokens) pick = 0;
    } else if (c->batching == RS_BATCHING_BIN_PACKING) {
      int64_t best = -1;
      for (int64_t i = 0; i < I->wait.size; ++i) {
        uint32_t r = dq_at(&I->wait, i);
        int64_t size = reserved_tokens(s, r);
        if (reserved + size <= c->kv_capacity_tokens && size > best) {
          best = size;
          pick = i;
        }
      }
    } else {
      int64_t best = INT64_MAX;
      for (int64_t i = 0; i < I->wait.size; ++i) {
        uint32_t r = dq_at(&I->wait, i);
        int64_t left = decode_left(s, r);
        if (reserved + reserved_tokens(s, r) <= c->kv_capacity_tokens && left < best) {
          best = left;
          pick = i;
        }
      }
    }
    if (pick >= I->wait.size) break;
    uint32_t r = dq_at(&I->wait, pick);
    dq_erase(&I->wait, pick);
    I->run[I->n_run].req = r;
    I->run[I->n_run].prompt_remaining = s->prompt[r];
    I->run[I->n_run].admit_seq = I->admit_seq++;
    I->n_run++;
    reserved += reserved_tokens(s, r);
  }
}

/* Instance::step (instance.hpp:203-277); returns completions or -1 and adds
 * IterationOutcome::tokens_emitted to *tokens. */
static int inst_step(sim_t* s, inst_t* I, int* tokens) {
  const rs_batch_cfg* c = s->c;
  const rs_profile* p = &c->profile;
  admit_waiting(s, I);
  if (I->n_run == 0) return -1; /* logic_error: none admissible */
  int any_prefill = 0;
  for (int i = 0; i < I->n_run; ++i)
    if (I->run[i].prompt_remaining > 0) { any_prefill = 1; break; }
  /* indices of running entries that emit this iteration */
  int32_t* emit = s->scratch;
  int n_emit = 0;
  double elapsed;
  if (any_prefill) {
    int64_t kv_before = kv_in_use(s, I);
    int64_t budget = c->chunk_size > 0 ? (int64_t)c->chunk_size : INT64_MAX;
    int64_t processed = 0;
    for (int i = 0; i < I->n_run; ++i) {
      run_entry* e = &I->run[i];
      if (e->prompt_remaining == 0) {
        if (c->chunk_size > 0) emit[n_emit++] = i; /* co-decoding */
        continue;
      }
      if (budget <= 0) continue;
      int64_t take = e->prompt_remaining < budget ? e->prompt_remaining : budget;
      e->prompt_remaining -= (int32_t)take;
      budget -= take;
      processed += take;
    }
    /* prompt_batch_time, latency.hpp:68-74 */
    elapsed = p->prompt_time_intercept + p->prompt_time_per_token * (double)processed +
              p->decode_time_per_token * (double)kv_before;
  } else {
    /* decode_batch_time with the running COUNT, instance.hpp:244-245 */
    elapsed = p->decode_time_base + p->decode_time_per_token * (double)I->n_run;
    for (int i = 0; i < I->n_run; ++i) emit[n_emit++] = i;
  }
  I->clock += elapsed;
  *tokens += n_emit;
  for (int k = 0; k < n_emit; ++k) {
    uint32_t r = I->run[emit[k]].req;
    s->emitted[r] += 1;
    if (!(s->first[r] >= 0.0)) s->first[r] = I->clock;
  }
  /* completions, back to front, order of survivors kept (instance.hpp:265-273) */
  int done = 0;
  for (int i = I->n_run; i-- > 0;) {
    uint32_t r = I->run[i].req;
    if (s->emitted[r] >= s->decode[r]) {
      s->completion[r] = I->clock;
      for (int k = i; k + 1 < I->n_run; ++k) I->run[k] = I->run[k + 1];
      I->n_run--;
      done++;
    }
  }
  /* preempt_if_needed, instance.hpp:282-299 */
  while (kv_in_use(s, I) > c->kv_capacity_tokens && I->n_run > 1) {
    int victim = 0;
    for (int i = 1; i < I->n_run; ++i)
      if (I->run[i].admit_seq > I->run[victim].admit_seq) victim = i;
    uint32_t r = I->run[victim].req;
    for (int k = victim; k + 1 < I->n_run; ++k) I->run[k] = I->run[k + 1];
    I->n_run--;
    s->preempt[r] += 1;
    dq_push_front(&I->wait, r);
  }
  return done;
}

static void snapshot(const sim_t* s, const inst_t* I, feat_t* f) { /* instance.hpp:317-360 */
  const rs_batch_cfg* c = s->c;
  memset(f, 0, sizeof(*f));
  int64_t min_left = INT64_MAX;
  for (int i = 0; i < I->n_run; ++i) {
    uint32_t r = I->run[i].req;
    f->reserved += reserved_tokens(s, r);
    int64_t left = decode_left(s, r);
    if (left < min_left) min_left = left;
    if (I->run[i].prompt_remaining <= 0) f->dbc[bucket_of(c->state_edges, c->n_state_edges, left)]++;
    f->pending_prompt += I->run[i].prompt_remaining;
    f->out_dec_est += left;
    int64_t tl = (int64_t)s->decode[r] - s->emitted[r];
    f->out_true += tl > 0 ? tl : 0;
    f->token_sum += (int64_t)s->prompt[r] + s->emitted[r]; /* instance_loads, env.hpp:341-354 */
  }
  for (int64_t k = 0; k < I->wait.size; ++k) {
    uint32_t r = dq_at(&I->wait, k);
    f->reserved += reserved_tokens(s, r);
    f->pending_prompt += s->prompt[r];
    f->out_dec_est += decode_left(s, r);
    int64_t tl = (int64_t)s->decode[r] - s->emitted[r];
    f->out_true += tl > 0 ? tl : 0;
    f->token_sum += (int64_t)s->prompt[r] + s->emitted[r];
  }
  f->kv_in_use = kv_in_use(s, I);
  f->free_kv = c->kv_capacity_tokens - f->kv_in_use;
  f->free_reserved = c->kv_capacity_tokens - f->reserved;
  double frac = 1.0 - (double)f->kv_in_use / (double)c->kv_capacity_tokens;
  f->capacity = frac < 0.0 ? 0.0 : (frac > 1.0 ? 1.0 : frac);
  f->t_hat_c = I->n_run == 0 ? 0.0 : c->profile.decode_time_base * (double)min_left;
  f->running = I->n_run;
  f->waiting = (int32_t)I->wait.size;
}

static void inject_arrivals(sim_t* s) { /* env.hpp:357-375 */
  const rs_batch_cfg* c = s->c;
  while (s->cursor < s->n && s->arrival[s->cursor] <= s->clock) {
    int64_t i = s->cursor;
    (void)c;
    s->dest[i] = (int32_t)upper_bound_tokens(c, s->pred[i]);
    dq_push_back(&s->rq, (uint32_t)i);
    s->cursor++;
  }
}

/* ------------------------------------------------------------- policies */

typedef struct {
  uint64_t rr_next, dsl_next;
  double mc_next_allowed;
  int64_t dsl_cutoff;
  mt64 rng; /* epsilon-greedy stream */
} pol_t;

static int can_accept(const feat_t* f, const sim_t* s, uint32_t head) { /* policies.hpp:44-48 */
  return f->free_reserved >= reserved_tokens(s, head) &&
         f->running + f->waiting < s->c->max_batch_size;
}

static double round2(double x) { return round(x * 100.0) / 100.0; } /* env.hpp:82 */

static int decide(sim_t* s, pol_t* P, const feat_t* F) {
  const rs_batch_cfg* c = s->c;
  const rs_profile* pr = &c->profile;
  int m = c->num_instances;
  int has_head = s->rq.size > 0;
  uint32_t head = has_head ? dq_at(&s->rq, 0) : 0;
  switch (c->policy) {
    case RS_POLICY_ROUND_ROBIN: { /* policies.hpp:50-69 */
      if (!has_head) return m;
      int t = (int)(P->rr_next % (uint64_t)m);
      if (!can_accept(&F[t], s, head)) return m;
      P->rr_next++;
      return t;
    }
    case RS_POLICY_DEDICATED_SMALL_LARGE: { /* policies.hpp:73-104 */
      if (!has_head) return m;
      int t;
      if (m < 2) t = 0;
      else if (dec_est(s, head) >= P->dsl_cutoff) t = 0;
      else t = 1 + (int)(P->dsl_next % (uint64_t)(m - 1));
      if (!can_accept(&F[t], s, head)) return m;
      if (m >= 2 && t >= 1) P->dsl_next++;
      return t;
    }
    case RS_POLICY_DECODE_BALANCER: { /* policies.hpp:108-127 */
      if (!has_head) return m;
      int best = -1;
      for (int i = 0; i < m; ++i) {
        if (!can_accept(&F[i], s, head)) continue;
        if (best < 0 || F[i].out_true < F[best].out_true) best = i;
      }
      return best < 0 ? m : best;
    }
    case RS_POLICY_JSQ: { /* policies.hpp:131-146 */
      if (!has_head) return m;
      int best = 0;
      for (int i = 1; i < m; ++i)
        if (F[i].pending_prompt + F[i].out_dec_est < F[best].pending_prompt + F[best].out_dec_est)
          best = i;
      return best;
    }
    case RS_POLICY_MAX_CAPACITY: { /* policies.hpp:150-170 */
      if (!has_head || s->clock < P->mc_next_allowed) return m;
      int best = 0;
      for (int i = 1; i < m; ++i)
        if (F[i].capacity > F[best].capacity) best = i;
      if (F[best].free_reserved < reserved_tokens(s, head)) return m;
      P->mc_next_allowed = s->clock + 1.0;
      return best;
    }
    case RS_POLICY_MIN_MIN: { /* policies.hpp:193-206 */
      if (!has_head) return m;
      int best = 0;
      double rb = (double)F[0].pending_prompt * pr->prompt_time_per_token +
                  (double)F[0].out_dec_est * pr->decode_time_base;
      for (int i = 1; i < m; ++i) {
        double ri = (double)F[i].pending_prompt * pr->prompt_time_per_token +
                    (double)F[i].out_dec_est * pr->decode_time_base;
        if (ri < rb) { best = i; rb = ri; }
      }
      return best;
    }
    case RS_POLICY_EARLIEST_AVAILABLE: { /* policies.hpp:214-228 */
      if (!has_head) return m;
      for (int i = 0; i < m; ++i)
        if (F[i].free_reserved >= reserved_tokens(s, head)) return i;
      return m;
    }
    case RS_POLICY_WORKLOAD_AWARE: {
      if (!has_head) return m;
      const rs_impact* im = &c->impact;
      int64_t p = s->prompt[head], d = dec_est(s, head);
      int best = -1;
      double best_score = 0.0;
      for (int l = 0; l < m; ++l) {
        if (!can_accept(&F[l], s, head)) continue;
        double avail = pr->decode_time_base * (double)F[l].out_dec_est; /* latency.hpp:96-99 */
        double pcost = pr->prompt_time_per_token * (double)(F[l].pending_prompt + p);
        /* mixing_for, impact.hpp:51-77 */
        double pi = (double)p;
        double lead = (im->prompt_exponent == 2) ? pi * pi : pi;
        double t_p = im->grad1 * (lead + (double)F[l].token_sum);
        double r_p = (t_p <= im->epsilon_s) ? 1.0 : 1.0 - t_p / im->epsilon_s;
        double r_d = -im->grad2 * (double)(F[l].token_sum + p + d);
        double mix = im->alpha * r_p + (1.0 - im->alpha) * r_d;
        double score = (avail + pcost) - im->epsilon_s * mix;
        if (best < 0 || score < best_score) { best = l; best_score = score; }
      }
      return best < 0 ? m : best;
    }
    case RS_POLICY_RL: { /* RlPolicy (dqn.hpp:282-295), encode_state (env.hpp:88-113) */
      double x[RS_MAX_WIDTH], q[RS_MAX_WIDTH];
      int k = 0;
      for (int i = 0; i < m; ++i) {
        x[k++] = (double)F[i].pending_prompt / (double)c->kv_capacity_tokens;
        for (int b = 0; b < c->n_state_edges; ++b)
          x[k++] = (double)F[i].dbc[b] / (double)c->max_batch_size;
        x[k++] = round2(F[i].capacity);
        x[k++] = round2(F[i].t_hat_c);
      }
      int64_t qlen = s->rq.size < 512 ? s->rq.size : 512;
      x[k++] = (double)qlen / 512.0;
      x[k++] = has_head ? (double)s->prompt[head] / 1024.0 : 0.0;
      x[k++] = (has_head && s->pred[head] >= 0) ? (double)s->pred[head] : 0.0;
      int na = c->rl_dims[c->rl_num_layers];
      if (c->rl_epsilon > 0.0 && rng_uniform(&P->rng) < c->rl_epsilon) /* dqn.hpp:92-99 */
        return (int)rng_uniform_below(&P->rng, (uint64_t)na);
      mlp_forward(c, x, q);
      return argmax_action(q, na);
    }
  }
  return -2;
}

/* MinMinPolicy::pick_queue_index, policies.hpp:179-191 */
static int64_t minmin_pick(const sim_t* s) {
  const rs_profile* pr = &s->c->profile;
  int64_t best = 0;
  double best_time = DBL_MAX;
  for (int64_t i = 0; i < s->rq.size; ++i) {
    uint32_t r = dq_at(&s->rq, i);
    double t = pr->prompt_time_per_token * (double)s->prompt[r] +
               pr->decode_time_base * (double)dec_est(s, r);
    if (t < best_time) { best_time = t; best = i; }
  }
  return best;
}

static int64_t heavy_decode_cutoff(const rs_profile* p, const rs_thresholds* t) { /* latency.hpp:132-138 */
  int64_t c = (int64_t)ceil(t->heavy_decode_seconds / p->decode_time_base - 1e-12);
  while (!(p->decode_time_base * (double)c >= t->heavy_decode_seconds)) ++c;
  return c;
}

/* ------------------------------------------------------------- reward */

/* mixing_for (impact.hpp:51-77) against InstanceLoad::token_sum (39-43). */
static double mixing_for(const rs_impact* im, int64_t p, int64_t d, int64_t token_sum) {
  double pi = (double)p;
  double lead = im->prompt_exponent == 2 ? pi * pi : pi;
  double t_p = im->grad1 * (lead + (double)token_sum);
  double r_p = t_p <= im->epsilon_s ? 1.0 : 1.0 - t_p / im->epsilon_s;
  double r_d = -im->grad2 * (double)(token_sum + p + d);
  return im->alpha * r_p + (1.0 - im->alpha) * r_d;
}

/* heuristic_h (impact.hpp:94-103) over instance_loads() (env.hpp:341-354). */
static double heuristic_h(const sim_t* s, int64_t p, int64_t d, int action) {
  int m = s->c->num_instances;
  double best = 0.0, chosen = 0.0;
  for (int i = 0; i < m; ++i) {
    const inst_t* I = &s->inst[i];
    int64_t ts = 0;
    for (int k = 0; k < I->n_run; ++k) ts += (int64_t)s->prompt[I->run[k].req] + s->emitted[I->run[k].req];
    for (int64_t k = 0; k < I->wait.size; ++k) {
      uint32_t r = dq_at(&I->wait, k);
      ts += (int64_t)s->prompt[r] + s->emitted[r];
    }
    double sc = mixing_for(&s->c->impact, p, d, ts);
    if (i == 0 || best < sc) best = sc; /* std::max(best, sc) */
    if (i == action) chosen = sc;
  }
  return chosen - best;
}

/* Eq. 3 queue penalty: the reward scan of ClusterSim::step (env.hpp:289-298). */
static double queue_penalty(const sim_t* s) {
  const rs_profile* p = &s->c->profile;
  double qp = 0.0;
  for (int64_t i = 0; i < s->n; ++i) {
    if (s->arrival[i] > s->clock || s->completion[i] >= 0.0) continue;
    double d_hat = (double)dec_est(s, (uint32_t)i);
    /* estimate_request_time, latency.hpp:87-92 */
    double t_hat = p->prompt_time_per_token * (double)s->prompt[i] + p->decode_time_base * d_hat;
    double f = (double)s->emitted[i] / d_hat;
    qp += (1.0 / t_hat) * (1.0 - f);
  }
  return qp;
}

/* RewardConfig::shaping_coefficient (env.hpp:55-63). */
static double shaping_coefficient(const rs_trajectory* t) {
  switch (t->shaping) {
    case RS_SHAPING_NONE: return 0.0;
    case RS_SHAPING_ADDITIVE: return 1.0;
    default: return t->gamma * exp(-t->beta_d * (double)t->episode_k);
  }
}

/* -------------------------------------------------------------- replay */

static int run_impl(const rs_batch_cfg* c, int64_t n, const double* arrival,
                    const int32_t* prompt, const int32_t* decode, const uint8_t* task,
                    const uint8_t* given, uint64_t predictor_seed, uint64_t policy_seed,
                    int32_t* o_instance, double* o_routed, double* o_first,
                    double* o_completion, int32_t* o_preempt, uint8_t* o_pred,
                    rs_replay_stats* st, int32_t* action_log, int64_t action_cap,
                    const rs_trajectory* traj) {
  if (c->num_instances < 1 || c->max_batch_size < 1 || c->kv_capacity_tokens < 1) return -1;
  if (c->policy < 0 || c->policy >= RS_POLICY_COUNT) return -1;
  int m = c->num_instances;
  sim_t S;
  memset(&S, 0, sizeof(S));
  S.c = c;
  S.n = n;
  S.arrival = arrival;
  S.prompt = prompt;
  S.decode = decode;
  size_t nn = (size_t)(n > 0 ? n : 1);
  S.pred = (int32_t*)calloc(nn, sizeof(int32_t));
  S.dest = (int32_t*)calloc(nn, sizeof(int32_t));
  S.routed = (double*)malloc(nn * sizeof(double));
  S.first = (double*)malloc(nn * sizeof(double));
  S.completion = (double*)malloc(nn * sizeof(double));
  S.emitted = (int32_t*)calloc(nn, sizeof(int32_t));
  S.preempt = (int32_t*)calloc(nn, sizeof(int32_t));
  S.assigned = (int32_t*)malloc(nn * sizeof(int32_t));
  S.inst = (inst_t*)calloc((size_t)m, sizeof(inst_t));
  S.rq.cap = (int64_t)nn;
  S.rq.buf = (uint32_t*)malloc(nn * sizeof(uint32_t));
  S.scratch = (int32_t*)malloc(sizeof(int32_t) * (size_t)c->max_batch_size);
  pol_t* P = (pol_t*)calloc(1, sizeof(pol_t));
  feat_t* F = (feat_t*)calloc((size_t)m, sizeof(feat_t));
  for (int64_t i = 0; i < n; ++i) {
    S.routed[i] = S.first[i] = S.completion[i] = -1.0;
    S.assigned[i] = -1;
  }
  int cap_run = c->max_batch_size;
  for (int i = 0; i < m; ++i) {
    S.inst[i].run = (run_entry*)malloc(sizeof(run_entry) * (size_t)cap_run);
    S.inst[i].wait.cap = (int64_t)nn + 1;
    S.inst[i].wait.buf = (uint32_t*)malloc(((size_t)nn + 1) * sizeof(uint32_t));
  }
  /* predictions are drawn in arrival-index order from one stream and are
   * policy independent (env.hpp:357-375), so they are resolved up front. */
  mt64* prng = (mt64*)malloc(sizeof(mt64));
  mt64_seed(prng, predictor_seed);
  for (int64_t i = 0; i < n; ++i)
    S.pred[i] = predict_one(c, prng, prompt[i], decode[i], task[i], given, i);
  free(prng);
  mt64_seed(&P->rng, policy_seed);
  P->dsl_cutoff = heavy_decode_cutoff(&c->profile, &c->thresholds);

  uint64_t hash = 0xcbf29ce484222325ULL;
  int64_t sum_q = 0, sum_w = 0, nlog = 0;
  int status = RS_REPLAY_FINISHED;
  S.error_instance = -1;
  inject_arrivals(&S); /* ctor, env.hpp:193 */
  while (S.completed != n && S.tick < c->max_ticks) { /* run_policy */
    for (int i = 0; i < m; ++i) snapshot(&S, &S.inst[i], &F[i]);
    if (c->policy == RS_POLICY_MIN_MIN) {
      int64_t pick = minmin_pick(&S);
      if (pick != 0 && pick < S.rq.size) { /* move_to_front, env.hpp:234-243 */
        uint32_t v = dq_at(&S.rq, pick);
        dq_erase(&S.rq, pick);
        dq_push_front(&S.rq, v);
      }
    }
    int action = decide(&S, P, F);
    hash = (hash ^ (uint64_t)(uint32_t)(action + 1)) * 0x100000001b3ULL;
    if (action_log && nlog < action_cap) action_log[nlog++] = action;
    /* ClusterSim::step, env.hpp:251-322 */
    if (action < 0 || action > m) { status = RS_REPLAY_BAD_ACTION; break; }
    double t1 = S.clock + c->delta_t;
    double bd_h = 0.0;
    int bd_infeasible = 0;
    if (action < m && S.rq.size > 0) {
      uint32_t h = dq_at(&S.rq, 0);
      if ((int64_t)prompt[h] + decode[h] > c->kv_capacity_tokens) {
        S.infeasible++;
        bd_infeasible = 1;
      } else {
        if (traj) bd_h = heuristic_h(&S, prompt[h], dec_est(&S, h), action);
        S.rq.head = (S.rq.head + 1) % S.rq.cap;
        S.rq.size--;
        S.routed[h] = S.clock;
        inst_t* I = &S.inst[action]; /* Instance::enqueue, instance.hpp:113-130 */
        S.assigned[h] = action;
        if (S.clock > I->clock) I->clock = S.clock;
        dq_push_back(&I->wait, h);
      }
    }
    int completions = 0, tokens = 0;
    for (int i = 0; i < m && !S.error; ++i) { /* run_until, instance.hpp:303-310 */
      inst_t* I = &S.inst[i];
      while (I->clock < t1 && (I->n_run > 0 || I->wait.size > 0)) {
        int d = inst_step(&S, I, &tokens);
        if (d < 0) { S.error = 1; S.error_instance = i; break; }
        completions += d;
      }
      if (!S.error && I->n_run == 0 && I->wait.size == 0 && I->clock < t1) I->clock = t1;
    }
    if (S.error) { status = RS_REPLAY_NOT_ADMISSIBLE; break; }
    S.completed += completions;
    S.clock = t1;
    inject_arrivals(&S);
    S.tick++;
    sum_q += S.rq.size;
    for (int i = 0; i < m; ++i) sum_w += S.inst[i].wait.size;
    if (traj && S.tick <= traj->capacity) { /* TickRecord, env.hpp:300-319 */
      int64_t k = S.tick - 1;
      double qp = queue_penalty(&S);
      double shaping = shaping_coefficient(traj) * bd_h;
      if (traj->time_s) traj->time_s[k] = S.clock;
      if (traj->action) traj->action[k] = action;
      if (traj->queue_penalty) traj->queue_penalty[k] = qp;
      if (traj->completions) traj->completions[k] = completions;
      if (traj->h) traj->h[k] = bd_h;
      if (traj->shaping_term) traj->shaping_term[k] = shaping;
      if (traj->reward) traj->reward[k] = -qp + traj->r_w * (double)completions + shaping;
      if (traj->infeasible_route) traj->infeasible_route[k] = (uint8_t)bd_infeasible;
      if (traj->router_queue) traj->router_queue[k] = (int32_t)S.rq.size;
      if (traj->tokens_emitted) traj->tokens_emitted[k] = tokens;
      for (int i = 0; i < m; ++i) {
        if (traj->instance_running) traj->instance_running[k * m + i] = S.inst[i].n_run;
        if (traj->instance_waiting) traj->instance_waiting[k * m + i] = (int32_t)S.inst[i].wait.size;
      }
    }
  }
  if (status == RS_REPLAY_FINISHED && S.completed != n) status = RS_REPLAY_MAX_TICKS;

  if (st) {
    memset(st, 0, sizeof(*st));
    st->ticks = S.tick;
    st->infeasible = S.infeasible;
    st->completed = S.completed;
    st->decision_hash = hash;
    st->sum_router_queue = sum_q;
    st->sum_instance_waiting = sum_w;
    st->clock = S.clock;
    st->status = status;
    st->error_instance = S.error_instance;
    st->injected = S.cursor;
    /* compute_metrics order, metrics.hpp:94-121 */
    double fa = DBL_MAX, lc = 0.0;
    double *e2e = (double*)malloc(nn * sizeof(double)), *ttft = (double*)malloc(nn * sizeof(double)),
           *tbt = (double*)malloc(nn * sizeof(double));
    int64_t ne = 0, nt = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (S.routed[i] >= 0.0) st->routed++;
      if (!(S.completion[i] >= 0.0)) continue;
      double e = S.completion[i] - arrival[i], f = S.first[i] - arrival[i];
      st->total_e2e_s += e;
      st->total_ttft_s += f;
      e2e[ne] = e;
      ttft[ne] = f;
      ne++;
      if (S.emitted[i] >= 2) {
        double b = (S.completion[i] - S.first[i]) / (double)(S.emitted[i] - 1);
        st->total_tbt_s += b;
        tbt[nt++] = b;
      }
      if (S.routed[i] >= 0.0) st->total_router_wait_s += S.routed[i] - arrival[i];
      st->total_preemptions += S.preempt[i];
      st->total_tokens += S.emitted[i];
      if (arrival[i] < fa) fa = arrival[i];
      if (S.completion[i] > lc) lc = S.completion[i];
    }
    st->tbt_count = nt;
    st->first_arrival_s = fa;
    st->last_completion_s = lc;
    st->makespan_s = lc - fa;
    if (ne > 0) {
      qsort(e2e, (size_t)ne, sizeof(double), ora_cmp_double);
      qsort(ttft, (size_t)ne, sizeof(double), ora_cmp_double);
      st->e2e_p50 = ora_nearest_rank(e2e, ne, 0.50);
      st->e2e_p90 = ora_nearest_rank(e2e, ne, 0.90);
      st->e2e_p99 = ora_nearest_rank(e2e, ne, 0.99);
      st->ttft_p50 = ora_nearest_rank(ttft, ne, 0.50);
      st->ttft_p90 = ora_nearest_rank(ttft, ne, 0.90);
      st->ttft_p99 = ora_nearest_rank(ttft, ne, 0.99);
      if (nt > 0) {
        qsort(tbt, (size_t)nt, sizeof(double), ora_cmp_double);
        st->tbt_p50 = ora_nearest_rank(tbt, nt, 0.50);
        st->tbt_p90 = ora_nearest_rank(tbt, nt, 0.90);
        st->tbt_p99 = ora_nearest_rank(tbt, nt, 0.99);
      }
      st->percentiles_valid = 1;
    }
    free(e2e);
    free(ttft);
    free(tbt);
  }
  for (int64_t i = 0; i < n; ++i) {
    if (o_instance) o_instance[i] = S.assigned[i];
    if (o_routed) o_routed[i] = S.routed[i];
    if (o_first) o_first[i] = S.first[i];
    if (o_completion) o_completion[i] = S.completion[i];
    if (o_preempt) o_preempt[i] = S.preempt[i];
    /* the reference only predicts requests that reached the router queue */
    if (o_pred) o_pred[i] = i < S.cursor ? (uint8_t)S.pred[i] : (uint8_t)255;
  }
  for (int i = 0; i < m; ++i) {
    free(S.inst[i].run);
    free(S.inst[i].wait.buf);
  }
  free(S.inst);
  free(S.rq.buf);
  free(S.scratch);
  free(S.pred);
  free(S.dest);
  free(S.routed);
  free(S.first);
  free(S.completion);
  free(S.emitted);
  free(S.preempt);
  free(S.assigned);
  free(P);
  free(F);
  return 0;
}

int ora_run_replay(const rs_batch_cfg* c, int64_t n, const double* arrival,
                   const int32_t* prompt, const int32_t* decode, const uint8_t* task,
                   const uint8_t* given, uint64_t predictor_seed, uint64_t policy_seed,
                   int32_t* o_instance, double* o_routed, double* o_first,
                   double* o_completion, int32_t* o_preempt, uint8_t* o_pred,
                   rs_replay_stats* st, int32_t* action_log, int64_t action_cap) {
  return run_impl(c, n, arrival, prompt, decode, task, given, predictor_seed, policy_seed,
                  o_instance, o_routed, o_first, o_completion, o_preempt, o_pred, st,
                  action_log, action_cap, NULL);
}

int ora_run_trajectory(const rs_batch_cfg* c, int64_t n, const double* arrival,
                       const int32_t* prompt, const int32_t* decode, const uint8_t* task,
                       const uint8_t* given, uint64_t predictor_seed, uint64_t policy_seed,
                       int32_t* o_instance, double* o_routed, double* o_first,
                       double* o_completion, int32_t* o_preempt, uint8_t* o_pred,
                       rs_replay_stats* st, const rs_trajectory* traj) {
  if (!traj) return -1;
  return run_impl(c, n, arrival, prompt, decode, task, given, predictor_seed, policy_seed,
                  o_instance, o_routed, o_first, o_completion, o_preempt, o_pred, st, NULL, 0,
                  traj);
}

int ora_cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

double ora_nearest_rank(const double* v, int64_t n, double q) { /* metrics.hpp:70-75 */
  size_t idx = (size_t)ceil(q * (double)n);
  if (idx > 0) --idx;
  if (idx > (size_t)(n - 1)) idx = (size_t)(n - 1);
  return v[idx];
}
