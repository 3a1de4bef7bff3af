// router.cuh — the per-replay tick loop: router decide() for every policy
// (policies.hpp:50-245 + workload_aware + RlPolicy), routing, the instance
// sweep, arrival injection and the end-of-replay statistics.
#pragma once

#include "replay.cuh"

namespace rs {

constexpr int kMaxTokens = 1 << 20;  // engine limit on prompt / decode tokens

struct Feat {  // InstanceFeatures subset, from the maintained aggregates
  long long res, pend, dleft, tleft, tok;
  int cnt, kv, nrun, mind;
};

__device__ __forceinline__ Feat load_feat(const Grp& G, int i) {
  const InstHot& h = G.inst[i];
  Feat f;
  f.res = h.res_run + h.res_wait;
  f.pend = h.pend_run + h.pend_wait;
  f.dleft = h.dleft_run + h.dleft_wait;
  f.tleft = h.tleft_run + h.tleft_wait;
  f.tok = h.tok_run + h.tok_wait;
  f.cnt = h.n_run + h.w_cnt + h.o_cnt;
  f.kv = h.kv_run;
  f.nrun = h.n_run;
  f.mind = h.min_dleft;
  return f;
}

// can_accept (policies.hpp:44-48)
__device__ __forceinline__ bool can_accept(const KParams& P, const Feat& f, int need) {
  return (long long)P.kv_cap - f.res >= need && f.cnt < P.max_batch;
}

// capacity_fraction (instance.hpp:138-142)
__device__ __forceinline__ double capacity_of(const KParams& P, int kv) {
  double v = __dsub_rn(1.0, div_exact((double)kv, (double)P.kv_cap, P.inv_kv, P.kv_pow2));
  return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
}

// mixing_for (impact.hpp:73-77): prompt_impact (51-59), decode_impact
// (63-67), mixing_penalty (69-71) against an instance's token mass
// InstanceLoad::token_sum (39-43), in the reference's operand order.
__device__ __forceinline__ double mixing_for(const KParams& P, long long p, long long d,
                                             long long token_sum) {
  const double pi = (double)p;
  const double lead = P.prompt_exp == 2 ? __dmul_rn(pi, pi) : pi;
  const double t_p = __dmul_rn(P.grad1, __dadd_rn(lead, (double)token_sum));
  const double r_p = t_p <= P.eps_s ? 1.0 : __dsub_rn(1.0, __ddiv_rn(t_p, P.eps_s));
  const double r_d = __dmul_rn(-P.grad2, (double)(token_sum + p + d));
  return __dadd_rn(__dmul_rn(P.alpha, r_p), __dmul_rn(__dsub_rn(1.0, P.alpha), r_d));
}

// round2 (env.hpp:82): std::round(x * 100.0) / 100.0.  The quotient of the
// integer k = round(x * 100) by 100 is formed without a division for
// 0 < k <= 2^22 (every state feature: capacity in [0, 1], T^_c up to ~4e4 s):
// q0 = k * RN(0.01), one exact FMA residual and one FMA correction give RN(k / 100)
// (Markstein; checked for every k in the range, tools/check_round2.py).  Zero
// keeps its sign (k / 100 = k); anything else divides.
constexpr double kRound2FastMax = 4194304.0;  // 2^22
__device__ __forceinline__ double round2(double x) {
  const double k = round(__dmul_rn(x, 100.0));
  if (k > 0.0 && k <= kRound2FastMax) {
    const double q0 = __dmul_rn(k, 0.01);
    const double r = __fma_rn(-q0, 100.0, k);
    return __fma_rn(r, 0.01, q0);
  }
  return k == 0.0 ? k : __ddiv_rn(k, 100.0);
}

__device__ __forceinline__ InstHot load_inst(const Grp& G, int i) { return G.inst[i]; }
__device__ __forceinline__ void store_inst(const Grp& G, int i, const InstHot& h) {
  if (lane_id() == 0) G.inst[i] = h;
  __syncwarp();
}

// Head-window: request data of the range head (prompt, true decode, bucket),
// one request per group lane.
template <int W>
__device__ __forceinline__ void head_window(const KParams& P, Replay& R, int q, const Lanes<W>& L) {
  if (q >= R.h_base && q < R.h_base + W) return;
  R.h_base = q & ~(W - 1);
  const int j = R.h_base + L.l;
  if (j < R.n) {
    R.h_prompt = P.prompt[R.off + j];
    R.h_true = P.decode[R.off + j];
    R.h_bucket = P.bucket[R.off + j];
  }
}

template <int W>
__device__ __forceinline__ Rec load_req(const KParams& P, long long off, int req, int* bucket,
                                       const Lanes<W>& L) {
  int v[3] = {0, 0, 0};
  if (L.l == 0) {
    v[0] = P.prompt[off + req];
    v[1] = P.decode[off + req];
    v[2] = P.bucket[off + req];
  }
  Rec r;
  r.req = req;
  r.prompt = L.shfl(v[0], 0);
  r.tru = L.shfl(v[1], 0);
  *bucket = L.shfl(v[2], 0);
  r.dhat = P.ub[*bucket];
  r.emit = 0;
  return r;
}

template <int POL, int W>
__device__ __forceinline__ Rec head_rec(const KParams& P, int* front, Replay& R, int* bucket,
                                       const Lanes<W>& L) {
  if (POL == RS_POLICY_MIN_MIN && R.nfront > 0) return load_req(P, R.off, front[0], bucket, L);
  head_window(P, R, R.qhead, L);
  const int s = R.qhead - R.h_base;
  Rec r;
  r.req = R.qhead;
  r.prompt = L.shfl(R.h_prompt, s);
  r.tru = L.shfl(R.h_true, s);
  *bucket = L.shfl(R.h_bucket, s);
  r.dhat = P.ub[*bucket];
  r.emit = 0;
  return r;
}
template <int POL>
__device__ __forceinline__ Rec head_rec(const KParams& P, int* front, Replay& R, int* bucket, int l) {
  return head_rec<POL>(P, front, R, bucket, warp_lanes(l));
}

// arrival window: one arrival time per group lane
template <int W>
__device__ __forceinline__ void load_arrival_window(const KParams& P, Replay& R, const Lanes<W>& L) {
  const int j = R.a_base + L.l;
  R.a_val = j < R.n ? P.arrival[R.off + j] : __longlong_as_double(0x7ff0000000000000ll);
}
__device__ __forceinline__ void load_arrival_window(const KParams& P, Replay& R, int l) {
  load_arrival_window(P, R, warp_lanes(l));
}

// ClusterSim::inject_arrivals (env.hpp:357-375): predictions were resolved
// by the predictor pre-pass, so injection is a cursor advance.
__device__ __forceinline__ void inject(const KParams& P, Replay& R, int l) {
  for (;;) {
    const int j = R.a_base + l;
    const bool ok = j >= R.cursor && j < R.n && R.a_val <= R.clock;
    R.cursor += __popc(__ballot_sync(kFull, ok));
    if (R.cursor == R.a_base + kWarp && R.cursor < R.n) {
      R.a_base += kWarp;
      load_arrival_window(P, R, l);
      continue;
    }
    break;
  }
}

template <int POL>
__device__ __forceinline__ int queue_len(const Replay& R) {
  if (POL == RS_POLICY_MIN_MIN) return R.nfront + (R.cursor - R.qhead) - R.n_removed;
  return R.cursor - R.qhead;
}

// Skip range entries that min_min moved to the front list.
template <int W>
__device__ __forceinline__ void mm_skip_removed(const KParams& P, Replay& R, const Lanes<W>& L) {
  while (R.qhead < R.cursor && R.n_removed > 0) {
    int rem = 0;
    if (L.l == 0) rem = P.mm_removed[R.off + R.qhead];
    rem = L.shfl(rem, 0);
    if (!rem) break;
    R.qhead++;
    R.n_removed--;
  }
}
__device__ __forceinline__ void mm_skip_removed(const KParams& P, Replay& R, int l) {
  mm_skip_removed(P, R, warp_lanes(l));
}

// MinMinPolicy::pick_queue_index (policies.hpp:179-191) + move_to_front
// (env.hpp:234-243).  Queue order = front list, then the range in index
// order minus removed entries.  Returns false on front-list overflow.
template <int W>
__device__ inline bool minmin_pick(const KParams& P, int* front, Replay& R, const Lanes<W>& L) {
  const int l = L.l;
  unsigned long long fk = ~0ull;
  int fpos = 0x7fffffff;
  for (int c = 0; c < R.nfront; c += W) {  // front list (<= kMaxFront entries)
    const int f = c + l;
    unsigned long long k = ~0ull;
    if (f < R.nfront) {
      const int req = front[f];
      const double est = __dadd_rn(__dmul_rn(P.tpp, (double)P.prompt[R.off + req]),
                                   __dmul_rn(P.dtb, (double)P.ub[P.bucket[R.off + req]]));
      k = ordered_key(est);
    }
    const unsigned long long mk = L.min_u64(k);
    if (mk < fk) {
      fk = mk;
      fpos = L.min((f < R.nfront && k == mk) ? f : 0x7fffffff);
    }
  }
  unsigned long long rk = ~0ull;
  int ridx = -1;
  for (int c = R.qhead; c < R.cursor; c += W) {
    const int j = c + l;
    unsigned long long k = ~0ull;
    if (j < R.cursor) {
      const long long g = R.off + j;
      if (!P.mm_removed[g]) {
        const double est = __dadd_rn(__dmul_rn(P.tpp, (double)P.prompt[g]),
                                     __dmul_rn(P.dtb, (double)P.ub[P.bucket[g]]));
        k = ordered_key(est);
      }
    }
    const unsigned long long mk = L.min_u64(k);
    if (mk < rk) {
      rk = mk;
      ridx = L.min((k == mk && j < R.cursor) ? j : 0x7fffffff);
    }
  }
  if (R.nfront > 0 && fk <= rk) {  // front entry (earlier queue positions win ties)
    if (fpos == 0) return true;
    const int v = front[fpos];
    L.sync();
    if (l == 0) {
      for (int k = fpos; k > 0; --k) front[k] = front[k - 1];
      front[0] = v;
    }
    L.sync();
    return true;
  }
  if (ridx < 0) return true;
  if (R.nfront == 0 && ridx == R.qhead) return true;  // already the head
  if (R.nfront >= kMaxFront) return false;
  if (l == 0) {
    P.mm_removed[R.off + ridx] = 1;
    for (int k = R.nfront; k > 0; --k) front[k] = front[k - 1];
    front[0] = ridx;
  }
  L.sync();
  R.nfront++;
  R.n_removed++;
  mm_skip_removed(P, R, L);
  return true;
}
__device__ inline bool minmin_pick(const KParams& P, int* front, Replay& R, int l) {
  return minmin_pick(P, front, R, warp_lanes(l));
}

// ε-greedy stream (DqnAgent::act, dqn.hpp:92-99) in shared memory.
template <int W>
__device__ __forceinline__ unsigned long long rng_draw(unsigned long long* rngbuf, Replay& R,
                                                       const Lanes<W>& L) {
  if (R.rng_pos == 312) {
    mt_twist(rngbuf, L);  // outputs are tempered as they are drawn
    R.rng_pos = 0;
  }
  return mt_temper(rngbuf[R.rng_pos++]);
}
__device__ __forceinline__ unsigned long long rng_draw(unsigned long long* rngbuf, Replay& R, int l) {
  return rng_draw(rngbuf, R, warp_lanes(l));
}

// Router decision for one tick.  `has_head` / `hr` / `hb` describe the head.
template <int POL>
__device__ inline int decide(const KParams& P, const Grp& G, const MlpView& M, Replay& R,
                             bool has_head, const Rec& hr, int hb) {
  const int m = P.m;
  const int l = lane_id();
  const int need = reserved_of(hr.prompt, hr.dhat, 0);
  if (POL == RS_POLICY_ROUND_ROBIN) {  // policies.hpp:50-69
    if (!has_head) return m;
    const int t = (int)(R.rr_next % (unsigned long long)m);
    if (!can_accept(P, load_feat(G, t), need)) return m;
    R.rr_next++;
    return t;
  } else if (POL == RS_POLICY_DEDICATED_SMALL_LARGE) {  // policies.hpp:73-104
    if (!has_head) return m;
    int t;
    if (m < 2 || hr.dhat >= P.dsl_cutoff) t = 0;
    else t = 1 + (int)(R.dsl_next % (unsigned long long)(m - 1));
    if (!can_accept(P, load_feat(G, t), need)) return m;
    if (m >= 2 && t >= 1) R.dsl_next++;
    return t;
  } else if (POL == RS_POLICY_MAX_CAPACITY) {  // policies.hpp:150-170
    if (!has_head || R.clock < R.mc_next) return m;
    unsigned long long bk = 0;
    int bi = -1;
    for (int g = 0; g < m; g += kWarp) {
      const int i = g + l;
      const bool v = i < m;
      const unsigned long long k = v ? ordered_key(capacity_of(P, G.inst[i].kv_run)) : 0ull;
      const int a = warp_argmax_key(k, v);
      const unsigned long long ka = __shfl_sync(kFull, k, a);
      if (bi < 0 || ka > bk) { bk = ka; bi = g + a; }
    }
    const Feat f = load_feat(G, bi);
    if ((long long)P.kv_cap - f.res < need) return m;
    R.mc_next = __dadd_rn(R.clock, 1.0);
    return bi;
  } else if (POL == RS_POLICY_EARLIEST_AVAILABLE) {  // policies.hpp:214-228
    if (!has_head) return m;
    for (int g = 0; g < m; g += kWarp) {
      const int i = g + l;
      bool ok = false;
      if (i < m) ok = (long long)P.kv_cap - load_feat(G, i).res >= need;
      const unsigned b = __ballot_sync(kFull, ok);
      if (b) return g + __ffs(b) - 1;
    }
    return m;
  } else if (POL == RS_POLICY_RL) {  // RlPolicy + encode_state (env.hpp:88-113)
    double* x = G.rlx;
    const int nsb = P.n_state_edges;
    const int per = 3 + nsb;
    for (int g = 0; g < m; g += kWarp) {
      const int i = g + l;
      if (i < m) {
        const Feat f = load_feat(G, i);
        double* xi = x + i * per;
        xi[0] = __ddiv_rn((double)f.pend, (double)P.kv_cap);
        for (int b = 0; b < nsb; ++b)
          xi[1 + b] = __ddiv_rn((double)G.dbc[i * RS_MAX_BUCKETS + b], (double)P.max_batch);
        xi[1 + nsb] = round2(capacity_of(P, f.kv));
        const double that = f.nrun == 0 ? 0.0 : __dmul_rn(P.dtb, (double)f.mind);
        xi[2 + nsb] = round2(that);
      }
    }
    if (l == 0) {
      const int q = queue_len<POL>(R);
      x[m * per] = __ddiv_rn((double)(q < 512 ? q : 512), 512.0);
      x[m * per + 1] = has_head ? __ddiv_rn((double)hr.prompt, 1024.0) : 0.0;
      x[m * per + 2] = has_head ? (double)hb : 0.0;
    }
    __syncwarp();
    const int na = P.rl_dims[P.rl_layers];
    if (P.rl_eps > 0.0) {
      const double u = u01(rng_draw(G.rng, R, l));
      if (u < P.rl_eps) {
        const double v = __dmul_rn(u01(rng_draw(G.rng, R, l)), (double)na);
        const unsigned long long k = (unsigned long long)v;  // static_cast<uint64_t>
        return (int)(k < (unsigned long long)na ? k : (unsigned long long)na - 1);
      }
    }
    double* h0 = x + M.dims[0];
    double* h1 = h0 + P.rl_maxw;
    return mlp_forward_warp(M, x, h0, h1, nullptr, warp_lanes(l), &R.qmacs);
  } else {
    // argmin policies: decode_balancer / jsq / min_min / workload_aware
    if (!has_head) return m;
    unsigned long long bk = ~0ull;
    int bi = -1;
    for (int g = 0; g < m; g += kWarp) {
      const int i = g + l;
      bool v = i < m;
      unsigned long long k = ~0ull;
      if (v) {
        const Feat f = load_feat(G, i);
        if (POL == RS_POLICY_DECODE_BALANCER) {  // policies.hpp:108-127
          v = can_accept(P, f, need);
          k = (unsigned long long)f.tleft;
        } else if (POL == RS_POLICY_JSQ) {  // policies.hpp:131-146
          k = (unsigned long long)(f.pend + f.dleft);
        } else if (POL == RS_POLICY_MIN_MIN) {  // policies.hpp:193-206
          k = ordered_key(__dadd_rn(__dmul_rn((double)f.pend, P.tpp),
                                    __dmul_rn((double)f.dleft, P.dtb)));
        } else {  // RS_POLICY_WORKLOAD_AWARE, SURVEY.md Appendix B
          v = can_accept(P, f, need);
          const long long p = hr.prompt, d = hr.dhat;
          const double avail = __dmul_rn(P.dtb, (double)f.dleft);
          const double pcost = __dmul_rn(P.tpp, (double)(f.pend + p));
          const double mix = mixing_for(P, p, d, f.tok);
          const double score = __dsub_rn(__dadd_rn(avail, pcost), __dmul_rn(P.eps_s, mix));
          k = ordered_key(score);
        }
      }
      const int a = warp_argmin_key(k, v);
      if (a >= 0) {
        const unsigned long long ka = __shfl_sync(kFull, k, a);
        if (bi < 0 || ka < bk) { bk = ka; bi = g + a; }
      }
    }
    if (POL == RS_POLICY_JSQ || POL == RS_POLICY_MIN_MIN) return bi;
    return bi < 0 ? m : bi;
  }
}

// Per-replay record: the replay-state fields (ClusterSim accessors, the
// decision hash, the time-average numerators).  The per-request aggregates
// of compute_metrics (metrics.hpp:84-162: sequential pool-index-order sums,
// nearest-rank percentiles) are filled by stats_kernel (stats.cuh), which
// runs right after the replay kernel.
template <int W>
__device__ inline void write_replay_stats(const KParams& P, const Replay& R, int r, const Lanes<W>& L) {
  if (L.l == 0) {
    rs_replay_stats& s = P.stats[r];
    s.ticks = R.tick;
    s.routed = R.routed;
    s.infeasible = R.infeasible;
    s.completed = R.completed;
    s.decision_hash = R.hash;
    s.sum_router_queue = R.sum_q;
    s.sum_instance_waiting = R.sum_w;
    s.clock = R.clock;
    s.status = R.status;
    s.error_instance = R.err_inst;
    s.injected = R.cursor;
    s.qnet_macs = R.qmacs;
  }
  L.sync();
}

__device__ inline void write_replay_stats(const KParams& P, const Replay& R, int r, int l) {
  write_replay_stats(P, R, r, warp_lanes(l));
}

// ---------------------------------------------------- trajectory mode
// ClusterConfig::record_trajectory: the reward of ClusterSim::step
// (env.hpp:257-303) and the TickRecord (env.hpp:305-319), per tick.

// heuristic_h (impact.hpp:94-103) of routing the head (p, d_hat) to
// `action`, over instance_loads() before the enqueue (env.hpp:268-269):
// the chosen instance's mixing score minus the best, std::max order.
__device__ inline double traj_heuristic_h(const KParams& P, const Grp& G, int p, int d,
                                          int action) {
  double best = 0.0, chosen = 0.0;
  for (int i = 0; i < P.m; ++i) {
    const InstHot& h = G.inst[i];
    const double sc = mixing_for(P, p, d, h.tok_run + h.tok_wait);
    if (i == 0 || best < sc) best = sc;  // best = std::max(best, sc)
    if (i == action) chosen = sc;
  }
  return __dsub_rn(chosen, best);
}

// Eq. 3 queue penalty (env.hpp:289-298): sum over the arrived, uncompleted
// requests in pool-index order of (1/T^)(1 - emitted/d^), T^ =
// estimate_request_time (latency.hpp:87-92).  Emitted counts come from
// ov_emit, refreshed here for every running and ring-resident request
// (overflow entries carry theirs; router-queue entries are 0).  `lo` is
// the first uncompleted index (monotone).  Sequential fp64 adds in index
// order, identical on every lane.
__device__ inline double traj_queue_penalty(const KParams& P, const Grp& G, const Replay& R,
                                            int& lo) {
  const int l = lane_id();
  const long long off = R.off;
  for (int i = 0; i < P.m; ++i) {
    const InstHot& h = G.inst[i];
    for (int j = l; j < h.n_run; j += kWarp)
      P.ov_emit[off + G.r_req[i * P.rcap + j]] = G.r_emit[i * P.rcap + j];
    for (int q = l; q < h.w_cnt; q += kWarp) {
      int sl = h.w_head + q;
      if (sl >= P.wcap) sl -= P.wcap;
      P.ov_emit[off + G.w_req[i * P.wcap + sl]] = G.w_emit[i * P.wcap + sl];
    }
  }
  __syncwarp();
  for (;;) {  // advance past the completed prefix
    const int j = lo + l;
    const bool open = j < R.cursor && !(P.o_completion[off + j] >= 0.0);
    const unsigned b = __ballot_sync(kFull, open || j >= R.cursor);
    if (b) { lo += __ffs(b) - 1; break; }
    lo += kWarp;
  }
  double acc = 0.0;
  for (int base = lo; base < R.cursor; base += kWarp) {
    const int j = base + l;
    double term = 0.0;
    bool v = false;
    if (j < R.cursor) {
      const long long g = off + j;
      v = !(P.o_completion[g] >= 0.0);
      if (v) {
        const double d_hat = (double)P.ub[P.bucket[g]];
        const double t_hat = __dadd_rn(__dmul_rn(P.tpp, (double)P.prompt[g]),
                                       __dmul_rn(P.dtb, d_hat));
        const double f = __ddiv_rn((double)P.ov_emit[g], d_hat);
        term = __dmul_rn(__ddiv_rn(1.0, t_hat), __dsub_rn(1.0, f));
      }
    }
    const unsigned vm = __ballot_sync(kFull, v);
    for (int k = 0; k < kWarp; ++k) {
      const double tk = __shfl_sync(kFull, term, k);
      if ((vm >> k) & 1u) acc = __dadd_rn(acc, tk);
    }
  }
  return acc;
}

// One TickRecord (after ++tick_, env.hpp:303-319) into the trajectory.
__device__ inline void traj_record(const KParams& P, const Grp& G, const Replay& R, int r,
                                   int action, int comps, double h, bool infeasible,
                                   int tokens, int qlen, int& lo) {
  const rs_trajectory& T = P.traj;
  double qp = 0.0;
  if (P.traj_scan) qp = traj_queue_penalty(P, G, R, lo);
  if (R.tick > T.capacity) return;
  const long long rec = (long long)r * T.capacity + (R.tick - 1);
  const int l = lane_id();
  if (l == 0) {
    const double shaping = __dmul_rn(P.c_k, h);
    if (T.time_s) T.time_s[rec] = R.clock;
    if (T.action) T.action[rec] = action;
    if (T.queue_penalty) T.queue_penalty[rec] = qp;
    if (T.completions) T.completions[rec] = comps;
    if (T.h) T.h[rec] = h;
    if (T.shaping_term) T.shaping_term[rec] = shaping;
    if (T.reward)  // env.hpp:300-302
      T.reward[rec] = __dadd_rn(__dadd_rn(-qp, __dmul_rn(P.r_w, (double)comps)), shaping);
    if (T.infeasible_route) T.infeasible_route[rec] = infeasible ? 1 : 0;
    if (T.router_queue) T.router_queue[rec] = qlen;
    if (T.tokens_emitted) T.tokens_emitted[rec] = tokens;
  }
  for (int i = l; i < P.m; i += kWarp) {
    const InstHot& hi = G.inst[i];
    if (T.instance_running) T.instance_running[rec * P.m + i] = hi.n_run;
    if (T.instance_waiting) T.instance_waiting[rec * P.m + i] = hi.w_cnt + hi.o_cnt;
  }
  __syncwarp();
}

template <int POL>
__device__ void run_replay(const KParams& P, const Grp& G, const MlpView& M, int r) {
  constexpr bool NEED_DBC = POL == RS_POLICY_RL;
  const int l = lane_id();
  Replay R;
  R.off = P.offsets[r];
  R.n = (int)(P.offsets[r + 1] - R.off);
  const int m = P.m;

  // outputs to the reference's "not yet" values; input checks
  bool bad = false;
  for (int j = l; j < R.n; j += kWarp) {
    const long long g = R.off + j;
    P.o_instance[g] = -1;
    P.o_routed[g] = -1.0;
    P.o_first[g] = -1.0;
    P.o_completion[g] = -1.0;
    P.o_preempt[g] = 0;
    if (POL == RS_POLICY_MIN_MIN) P.mm_removed[g] = 0;
    if (P.traj_on) P.ov_emit[g] = 0;  // tokens_emitted of never-routed requests
    const int p = P.prompt[g], d = P.decode[g];
    if (p < 1 || p > kMaxTokens || d < 1 || d > kMaxTokens) bad = true;
    if (j > 0 && P.arrival[g] < P.arrival[g - 1]) bad = true;
  }
  bad = __any_sync(kFull, bad);
  int traj_lo = 0;  // first uncompleted request (reward scan)
  for (int i = l; i < m; i += kWarp) {
    InstHot h;
    h.clock = 0.0;
    h.res_wait = h.pend_wait = h.dleft_wait = h.tleft_wait = h.tok_wait = 0;
    h.n_run = h.n_prefill = h.res_run = h.kv_run = h.pend_run = 0;
    h.dleft_run = h.tleft_run = h.tok_run = 0;
    h.min_dleft = 0x7fffffff;
    h.w_head = h.w_cnt = h.o_cnt = 0;
    h.o_head = h.o_tail = (int)kNil;
    h._pad0 = h._pad1 = 0;
    G.inst[i] = h;
    if (NEED_DBC)
      for (int b = 0; b < RS_MAX_BUCKETS; ++b) G.dbc[i * RS_MAX_BUCKETS + b] = 0;
  }
  R.clock = 0.0;
  R.tick = 0;
  R.qhead = R.cursor = 0;
  R.completed = 0;
  R.nfront = R.n_removed = 0;
  R.total_wait = 0;
  R.rr_next = R.dsl_next = 0;
  R.mc_next = 0.0;
  R.hash = 0xcbf29ce484222325ull;
  R.qmacs = 0;
  R.infeasible = R.routed = R.sum_q = R.sum_w = 0;
  R.status = RS_REPLAY_FINISHED;
  R.err_inst = -1;
  R.rng_pos = 312;
  R.a_base = 0;
  R.h_base = -2 * kWarp;
  R.h_prompt = R.h_true = R.h_bucket = 0;
  if (POL == RS_POLICY_RL && P.rl_eps > 0.0)
    mt_seed_warp(G.rng, P.policy_seed ? P.policy_seed[r] : 0ull, l);
  __syncwarp();
  load_arrival_window(P, R, l);
  if (bad) {
    R.status = RS_REPLAY_INVALID_TRACE;
  } else {
    inject(P, R, l);  // ctor (env.hpp:193)
  }

  // ---------------------------------------------------------- tick loop
  while (R.status == RS_REPLAY_FINISHED && R.completed != R.n && R.tick < P.max_ticks) {
    if (POL == RS_POLICY_MIN_MIN && queue_len<POL>(R) > 0) {
      if (!minmin_pick(P, G.front, R, l)) { R.status = RS_REPLAY_CAPACITY; break; }
    }
    const bool has_head = queue_len<POL>(R) > 0;
    Rec hr;
    int hb = 0;
    if (has_head) {
      hr = head_rec<POL>(P, G.front, R, &hb, l);
    } else {
      hr.req = hr.prompt = hr.dhat = hr.tru = hr.emit = 0;
    }
    const int action = decide<POL>(P, G, M, R, has_head, hr, hb);
    R.hash = hash_action(R.hash, action);
    if (action < 0 || action > m) { R.status = RS_REPLAY_BAD_ACTION; break; }
    const double t1 = __dadd_rn(R.clock, P.delta_t);
    double th = 0.0;  // RewardBreakdown::h
    bool infeasible = false;
    if (action < m && has_head) {
      if ((long long)hr.prompt + hr.tru > P.kv_cap) {
        R.infeasible++;  // env.hpp:262-267: flagged, stays queued
        infeasible = true;
      } else {
        if (P.traj_on && l == 0) th = traj_heuristic_h(P, G, hr.prompt, hr.dhat, action);
        if (POL == RS_POLICY_MIN_MIN && R.nfront > 0) {
          if (l == 0)
            for (int k = 0; k + 1 < R.nfront; ++k) G.front[k] = G.front[k + 1];
          __syncwarp();
          R.nfront--;
        } else {
          R.qhead++;
          if (POL == RS_POLICY_MIN_MIN) mm_skip_removed(P, R, l);
        }
        if (l == 0) {
          P.o_routed[R.off + hr.req] = R.clock;
          P.o_instance[R.off + hr.req] = action;
        }
        R.routed++;
        InstHot h = load_inst(G, action);  // Instance::enqueue
        if (h.clock < R.clock) h.clock = R.clock;
        wait_push_back(P, G, R.off, action, h, hr);
        store_inst(G, action, h);
        R.total_wait++;
      }
    }
    // run_until(t1) for every instance, index order (independent)
    int comps = 0, tokens = 0;
    for (int g = 0; g < m && R.status == RS_REPLAY_FINISHED; g += kWarp) {
      const int i = g + l;
      bool busy = false;
      if (i < m) {
        const InstHot& hi = G.inst[i];
        if (hi.clock < t1) {
          if (hi.n_run > 0 || hi.w_cnt > 0) busy = true;
          else G.inst[i].clock = t1;  // idle instance skips ahead
        }
      }
      unsigned mask = __ballot_sync(kFull, busy);
      __syncwarp();
      while (mask) {
        const int ii = g + __ffs(mask) - 1;
        mask &= mask - 1;
        InstHot h = load_inst(G, ii);
        const int w0 = h.w_cnt + h.o_cnt;
        while (h.clock < t1 && (h.n_run > 0 || h.w_cnt > 0)) {
          const int c = inst_step<NEED_DBC>(P, G, R.off, ii, h, tokens);
          if (c < 0) {
            R.status = RS_REPLAY_NOT_ADMISSIBLE;
            R.err_inst = ii;
            break;
          }
          comps += c;
        }
        if (h.n_run == 0 && h.w_cnt == 0 && h.clock < t1) h.clock = t1;
        R.total_wait += h.w_cnt + h.o_cnt - w0;
        store_inst(G, ii, h);
        if (R.status != RS_REPLAY_FINISHED) break;
      }
    }
    if (R.status != RS_REPLAY_FINISHED) break;
    R.completed += comps;
    R.clock = t1;
    inject(P, R, l);
    R.tick++;
    R.sum_q += queue_len<POL>(R);
    R.sum_w += R.total_wait;
    if (P.traj_on)
      traj_record(P, G, R, r, action, comps, th, infeasible, tokens, queue_len<POL>(R), traj_lo);
  }
  if (R.status == RS_REPLAY_FINISHED && R.completed != R.n) R.status = RS_REPLAY_MAX_TICKS;

  write_replay_stats(P, R, r, l);
}

template <int POL>
__global__ void __launch_bounds__(256) replay_kernel(const __grid_constant__ KParams P) {
  extern __shared__ __align__(16) char smem[];
  const int w = threadIdx.x / kWarp;
  MlpView M;
  M.layers = P.rl_layers;
  M.dims = P.rl_dims;
  M.woff = P.rl_woff;
  M.boff = P.rl_boff;
  M.w = reinterpret_cast<const double*>(smem);
  int groups_off = 0;
  if (POL == RS_POLICY_RL) {
    if (P.rl_wt_global) {  // too big for shared memory: transposed copy in L2
      M.w = P.rl_wt_global;
    } else {
      mlp_stage_weights(P.rl_w, P.rl_layers, P.rl_dims, P.rl_woff, P.rl_boff,
                        reinterpret_cast<double*>(smem));
      groups_off = P.smem_weights_bytes;
    }
  }
  char* gbase = smem + groups_off + (size_t)w * P.smem_group_bytes;
  const Grp G = make_grp(P, gbase);
  for (;;) {
    int r = 0;
    if (lane_id() == 0) r = atomicAdd(P.work_counter, 1);
    r = __shfl_sync(kFull, r, 0);
    if (r >= P.num_replays) break;
    run_replay<POL>(P, G, M, r);
  }
}

}  // namespace rs
