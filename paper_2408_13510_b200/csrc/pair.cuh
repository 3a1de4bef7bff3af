// pair.cuh — large fleets (32 < m <= 64): TWO warps per replay, one instance
// per lane (instances wid * 32 + lane), instead of one warp holding two
// instances per lane.
//
// Why.  With two instances per lane the tick loop is twice as long and its
// code twice as large; c5 (m = 64, 512 replays) runs one warp per scheduler,
// so every dependent latency and every instruction-fetch miss is exposed
// (ncu: issue active 13%, `no_instruction` 2.7 cycles per issue).  A warp
// pair runs the one-instance-per-lane loop of the m <= 32 kernel on each half
// of the fleet, two warps per scheduler.
//
// What the warps share.  Every replay-level quantity (router queue, clock,
// tick, hash, arrival windows, head record, counters) is computed by BOTH
// warps identically from the same inputs, so it never moves between them.
// Exchanges, through a few shared words and a 64-thread named barrier:
//   * the routing decision (per-warp argmin / argmax / first-fit, combined
//     with the lower instance index winning ties, exactly the whole-fleet
//     order of policies.hpp);
//   * the fused predictor's draws (warp 0 draws, the barrier publishes them);
//   * "nothing admissible" flags, carried by the decision exchanges (every
//     tick with a head) and by the barrier reductions (bar.red.or) of
//     run_policy's done() once every request has arrived and been routed —
//     between those the warps may be a few ticks apart, which nothing
//     observes (disjoint instances, replicated replay state);
//   * the final completion / waiting sums.
// Instance stepping and its events (admission, prefill, decode steps,
// completion scans, preemption) touch only the warp's own instances and run
// warp-locally between the barriers.  A replay that raises "nothing
// admissible" or ends unfinished is re-run by warp 0 alone on the
// two-instances-per-lane code (index-order stepping, output
// initialisation), bit-identical by construction.
#pragma once

#include "fast_kernel.cuh"

namespace rs {

struct Pair {
  int wid;    // 0 = instances 0..31, 1 = instances 32..63
  int bar;    // named barrier id of the pair (1..15)
  int* xw;    // shared exchange words of the pair (2 banks x 8, + the work word)
  int bank;   // exchange bank, alternating: a warp can rewrite its words only
              // after a second barrier, so the partner has read the last ones
};

__device__ __forceinline__ void pair_sync(const Pair& Q) {
  asm volatile("bar.sync %0, 64;" ::"r"(Q.bar) : "memory");
}
// OR of a predicate over the 64 threads of the pair (one barrier)
__device__ __forceinline__ bool pair_any(const Pair& Q, bool p) {
  unsigned r;
  asm volatile(
      "{ .reg .pred a, b; setp.ne.u32 a, %1, 0; bar.red.or.pred b, %2, 64, a; selp.u32 %0, 1, 0, b; }"
      : "=r"(r)
      : "r"((unsigned)p), "r"(Q.bar)
      : "memory");
  return r != 0;
}
// Each warp posts three words and its error flag (lane 0); the other
// warp's come back, the flags OR-ed into `err`.
__device__ __forceinline__ void pair_swap3(Pair& Q, int l, int a, int b, int c, int& oa, int& ob,
                                           int& oc, bool own_err, bool& err) {
  int* x = Q.xw + Q.bank * 8;
  Q.bank ^= 1;
  if (l == 0) {
    x[Q.wid * 4 + 0] = a;
    x[Q.wid * 4 + 1] = b;
    x[Q.wid * 4 + 2] = c;
    x[Q.wid * 4 + 3] = own_err;
  }
  pair_sync(Q);
  const int o = (Q.wid ^ 1) * 4;
  oa = x[o];
  ob = x[o + 1];
  oc = x[o + 2];
  err = err || own_err || x[o + 3] != 0;
}

// The routing decision of decide_fast for the whole fleet, from each warp's
// half: the same scores per instance, combined in index order.  The
// exchange also carries the warps' "nothing admissible" flags (`err`, in:
// this warp's; out: either's when an exchange took place, else false — a
// decision without an exchange is made by both warps alone); the caller
// re-runs the replay when it comes back set.
template <int POL>
__device__ __forceinline__ int decide_pair(const KParams& P, Replay& R, Inst& I, bool has_head,
                                           const Rec& hr, const Lanes<kWarp>& L, Pair& Q,
                                           bool& err) {
  const bool own_err = err;
  err = false;
  const int l = L.l;
  const int m = P.m;
  const int i = Q.wid * kWarp + l;
  const bool here = i < m;
  const int need = reserved_of(hr.prompt, hr.dhat, 0);
  if (!has_head) return m;
  if (POL == RS_POLICY_ROUND_ROBIN || POL == RS_POLICY_DEDICATED_SMALL_LARGE) {
    int t;
    if (POL == RS_POLICY_ROUND_ROBIN) {  // policies.hpp:50-69
      t = (int)(R.rr_next % (unsigned long long)m);
    } else {  // policies.hpp:73-104
      if (m < 2 || hr.dhat >= P.dsl_cutoff) t = 0;
      else t = 1 + (int)(R.dsl_next % (unsigned long long)(m - 1));
    }
    const bool mine = (t >> 5) == Q.wid;
    int ok = mine ? L.shfl((int)(i == t && can_accept(P, feat_of(I), need)), t & (kWarp - 1)) : 0;
    int ook, d1, d2;
    pair_swap3(Q, l, ok, 0, 0, ook, d1, d2, own_err, err);
    if (!mine) ok = ook;
    if (!ok) return m;
    if (POL == RS_POLICY_ROUND_ROBIN) R.rr_next++;
    else if (m >= 2 && t >= 1) R.dsl_next++;
    return t;
  } else if (POL == RS_POLICY_EARLIEST_AVAILABLE) {  // policies.hpp:214-228
    const bool ok = here && (long long)P.kv_cap - feat_of(I).res >= need;
    const int b = (int)L.ballot(ok);
    int ob, d1, d2;
    pair_swap3(Q, l, b, 0, 0, ob, d1, d2, own_err, err);
    const unsigned b0 = (unsigned)(Q.wid == 0 ? b : ob), b1 = (unsigned)(Q.wid == 0 ? ob : b);
    if (b0) return __ffs(b0) - 1;
    if (b1) return kWarp + __ffs(b1) - 1;
    return m;
  } else if (POL == RS_POLICY_MAX_CAPACITY) {  // policies.hpp:150-170
    if (R.clock < R.mc_next) return m;
    const unsigned long long k = here ? ordered_key(capacity_of(P, I.kv)) : 0ull;
    const int a = grp_argmax_key(L, k, here);
    const unsigned long long ka = a >= 0 ? L.shfl(k, a) : 0ull;
    int hi, lo, oi;
    pair_swap3(Q, l, (int)(ka >> 32), (int)ka, a >= 0 ? Q.wid * kWarp + a : -1, hi, lo, oi, own_err, err);
    const unsigned long long ko = ((unsigned long long)(unsigned)hi << 32) | (unsigned)lo;
    const int mi = a >= 0 ? Q.wid * kWarp + a : -1;
    // index order: warp 0's best, replaced only by a strictly larger key
    const int i0 = Q.wid == 0 ? mi : oi, i1 = Q.wid == 0 ? oi : mi;
    const unsigned long long k0 = Q.wid == 0 ? ka : ko, k1 = Q.wid == 0 ? ko : ka;
    int bi = i0;
    if (i1 >= 0 && (bi < 0 || k1 > k0)) bi = i1;
    const bool mine = bi >= 0 && (bi >> 5) == Q.wid;
    int ok = mine ? L.shfl((int)(i == bi && (long long)P.kv_cap - feat_of(I).res >= need),
                           bi & (kWarp - 1))
                  : 0;
    int ook, d1, d2;
    pair_swap3(Q, l, ok, 0, 0, ook, d1, d2, own_err, err);
    if (!mine) ok = ook;
    if (!ok) return m;
    R.mc_next = __dadd_rn(R.clock, 1.0);
    return bi;
  } else {  // argmin policies (decode_balancer, jsq, workload_aware)
    bool v = here;
    unsigned long long k = ~0ull;
    if (v) {
      const FeatI f = feat_of(I);
      if (POL == RS_POLICY_DECODE_BALANCER) {  // policies.hpp:108-127
        v = can_accept(P, f, need);
        k = (unsigned long long)f.tleft;
      } else if (POL == RS_POLICY_JSQ) {  // policies.hpp:131-146
        k = (unsigned long long)(f.pend + f.dleft);
      } else {  // workload_aware, SURVEY.md Appendix B
        v = can_accept(P, f, need);
        const int p = hr.prompt, d = hr.dhat;
        const double avail = __dmul_rn(P.dtb, (double)f.dleft);
        const double pcost = __dmul_rn(P.tpp, (double)(f.pend + p));
        const double pi = (double)p;
        const double lead = P.prompt_exp == 2 ? __dmul_rn(pi, pi) : pi;
        const double t_p = __dmul_rn(P.grad1, __dadd_rn(lead, (double)f.tok));
        const double r_p =
            t_p <= P.eps_s ? 1.0 : __dsub_rn(1.0, div_exact(t_p, P.eps_s, P.inv_eps, P.eps_pow2));
        const double r_d = __dmul_rn(-P.grad2, (double)(f.tok + p + d));
        const double mix = __dadd_rn(__dmul_rn(P.alpha, r_p),
                                     __dmul_rn(__dsub_rn(1.0, P.alpha), r_d));
        k = ordered_key(__dsub_rn(__dadd_rn(avail, pcost), __dmul_rn(P.eps_s, mix)));
      }
    }
    const int a = argmin_narrow(L, k, v, kWarp);
    const unsigned long long ka = a >= 0 ? L.shfl(k, a) : ~0ull;
    int hi, lo, oi;
    pair_swap3(Q, l, (int)(ka >> 32), (int)ka, a >= 0 ? Q.wid * kWarp + a : -1, hi, lo, oi, own_err, err);
    const unsigned long long ko = ((unsigned long long)(unsigned)hi << 32) | (unsigned)lo;
    const int mi = a >= 0 ? Q.wid * kWarp + a : -1;
    const int i0 = Q.wid == 0 ? mi : oi, i1 = Q.wid == 0 ? oi : mi;
    const unsigned long long k0 = Q.wid == 0 ? ka : ko, k1 = Q.wid == 0 ? ko : ka;
    int bi = i0;  // ties: the lower index (warp 0)
    if (i1 >= 0 && (bi < 0 || k1 < k0)) bi = i1;
    if (POL == RS_POLICY_JSQ) return bi;
    return bi < 0 ? m : bi;
  }
}

// One replay on a warp pair (run_replay_fast's tick loop, one instance per
// lane).  Returns kRerunSeq / kRerunInit like it; never re-runs itself.
template <int POL, int T>
__device__ __forceinline__ FastRun run_replay_pair(const KParams& P, int gw, char* gbase, int r,
                                                   const Lanes<kWarp>& L, Pair& Q) {
  constexpr int W = kWarp;
  const int l = L.l;
  const int i = Q.wid * W + l;  // this lane's instance
  Replay R;
  R.off = P.offsets[r];
  R.n = (int)(P.offsets[r + 1] - R.off);
  const int m = P.m;
  const long long off = R.off;
  int* front = reinterpret_cast<int*>(gbase + P.off_front);

  bool bad = false;
  if (P.vinfo) {  // validated and zeroed by the validate_kernel pre-pass
    bad = P.vinfo[r].x != 0;
  } else {
    for (int j = Q.wid * W + l; j < R.n; j += 2 * W) {
      const long long g = off + j;
      P.o_preempt[g] = 0;
      if (P.resident) continue;  // streamed inputs: validated per window on load
      const int p = P.prompt[g], d = P.decode[g];
      if (p < 1 || p > kMaxTokens || d < 1 || d > kMaxTokens) bad = true;
      if (j > 0 && P.arrival[g] < P.arrival[g - 1]) bad = true;
    }
    bad = pair_any(Q, bad);
  }
  Inst I;
  inst_init(I);
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
  R.h_base = -2 * W;
  R.h_prompt = R.h_true = R.h_bucket = 0;
  unsigned long long* pst = reinterpret_cast<unsigned long long*>(gbase + P.off_pred);
  R.pred_pos = 312;
  R.a_val = 0.0;
  R.resident_seen = 0;
  const bool draws = P.predict_inline && P.predictor_mode == RS_PREDICTOR_SIMULATED;
  if (draws && Q.wid == 0) mt_seed(pst, P.predictor_seed[r], L);  // Rng(predictor_seed), env.hpp:173
  L.sync();
  // arrival window (both warps) + its predictions (warp 0; the barrier
  // publishes them before either warp reads a head record)
  auto load_window = [&]() {
    if (P.resident) {
      // streamed inputs (load_window_fast): wait for the copy stream to land
      // this window; both warps poll, and give up together
      const int need = min(R.n, R.a_base + W);
      bool late = false;
      if (need > R.resident_seen) {
        int v = L.min(load_acquire(P.resident));
        const unsigned long long t0 = globaltimer_ns();
        while (v < need && !late) {
          __nanosleep(256);
          v = L.min(load_acquire(P.resident));
          late = v < need && L.any(globaltimer_ns() - t0 > kStreamTimeoutNs);
        }
        R.resident_seen = v;
      }
      if (pair_any(Q, late)) {
        R.status = RS_REPLAY_NOT_RUN;  // the copy stream never delivered
        return;
      }
      const double prev_last = L.shfl(R.a_val, W - 1);
      load_arrival_window(P, R, L);
      // the window's trace contract (the up-front pass cannot read inputs
      // still in flight): token ranges, non-decreasing arrivals
      const int j = R.a_base + l;
      const double up = L.shfl_up(R.a_val, 1);
      bool badw = false;
      if (j < R.n) {
        const long long g = R.off + j;
        const int p = P.prompt[g], d = P.decode[g];
        badw = p < 1 || p > kMaxTokens || d < 1 || d > kMaxTokens;
        if (j > 0 && R.a_val < (l == 0 ? prev_last : up)) badw = true;
      }
      if (L.any(badw)) {
        R.status = RS_REPLAY_INVALID_TRACE;
        return;
      }
    } else {
      load_arrival_window(P, R, L);
    }
    if (P.predict_inline) {
      if (Q.wid == 0) predict_window(P, R, pst, L);
      pair_sync(Q);
    }
  };
  auto inject = [&]() {  // inject_fast (env.hpp:357-375)
    for (;;) {
      const int j = R.a_base + l;
      const bool ok = j >= R.cursor && j < R.n && R.a_val <= R.clock;
      R.cursor += __popc(L.ballot(ok));
      if (R.cursor == R.a_base + W && R.cursor < R.n) {
        R.a_base += W;
        load_window();
        if (R.status != RS_REPLAY_FINISHED) break;  // a streamed window failed
        continue;
      }
      break;
    }
  };
  auto next_arrival = [&]() {
    const int k = R.cursor - R.a_base;
    const double a = L.shfl(R.a_val, k & (W - 1));
    R.next_arr = R.cursor < R.n ? a : __longlong_as_double(0x7ff0000000000000ll);
  };
  load_window();
  R.hr_q = -1;
  R.hr_prompt = R.hr_true = R.hr_bucket = 0;
  if (bad) R.status = RS_REPLAY_INVALID_TRACE;
  else if (R.status == RS_REPLAY_FINISHED) inject();
  next_arrival();

  int lcomp = 0;
  long long lsw = 0;
  bool perr = false;  // "nothing admissible" in this warp's half
  while (R.status == RS_REPLAY_FINISHED && R.tick < P.max_ticks) {
    if (R.cursor == R.n && queue_len<POL>(R) == 0) {  // run_policy's done()
      if (pair_any(Q, perr)) return kRerunSeq;
      if (!pair_any(Q, i < m && (I.n > 0 || I.w_cnt > 0))) break;
    }
    const bool has_head = queue_len<POL>(R) > 0;
    Rec hr;
    if (has_head) {
      if (R.hr_q == R.qhead) {  // same head as last tick
        hr.req = R.qhead;
        hr.prompt = R.hr_prompt;
        hr.tru = R.hr_true;
        hr.dhat = P.ub[R.hr_bucket];
        hr.emit = 0;
      } else {
        int hb = 0;
        hr = head_rec<POL>(P, front, R, &hb, L);
        R.hr_q = hr.req;
        R.hr_prompt = hr.prompt;
        R.hr_true = hr.tru;
        R.hr_bucket = hb;
      }
    } else {
      hr.req = hr.prompt = hr.dhat = hr.tru = hr.emit = 0;
    }
    bool err = perr;
    const int action = decide_pair<POL>(P, R, I, has_head, hr, L, Q, err);
    if (err) return kRerunSeq;  // (both warps: the flag came through the exchange)
    R.hash = hash_action(R.hash, action);
    const double t1 = __dadd_rn(R.clock, P.delta_t);
    if (action < m && has_head) {
      if ((long long)hr.prompt + hr.tru > P.kv_cap) {
        R.infeasible++;  // env.hpp:262-267: flagged, stays queued
      } else {
        R.qhead++;
        if (Q.wid == 0 && l == 0) {
          P.o_routed[off + hr.req] = R.clock;
          P.o_instance[off + hr.req] = action;
        }
        R.routed++;
        if (i == action) lane_enqueue(P, gw, off, action, I, hr, R.clock);
      }
    }

    // ---- run_until(t1) of this warp's instances (warp-local) ------------
    bool act = false;
    // (a warp that hit "nothing admissible" stops stepping; the replay is
    // re-run at the pair's next exchange)
    if (!perr && i < m && I.clock < t1) {
      if (I.n > 0 || I.w_cnt > 0) act = true;
      else I.clock = t1;  // idle instance skips ahead (instance.hpp:309)
    }
    bool again = L.any(act);
    while (again) {
      bool ev = false;
      if (act) {
        if (I.n == 0 && I.w_cnt == 0) {  // emptied by last iteration's events
          I.clock = t1;
          act = false;
        } else {
          bool prefill = false;
          bool skip = false;
          if (I.w_cnt > 0 && I.n < P.max_batch) {
            lane_admit<T>(P, gw, off, i, I);
            if (I.n == 0) {  // logic_error, instance.hpp:209-211
              ev = true;
              skip = true;
            }
            prefill = I.npf > 0;
          }
          if (skip) {
          } else if (prefill) {  // whole-prompt prefill; co-running decodes stall
            I.clock = __dadd_rn(I.clock, __dadd_rn(__dadd_rn(P.intercept,
                                                             __dmul_rn(P.tpp, (double)I.pend)),
                                                   __dmul_rn(P.dpt, (double)I.kv)));
            I.kv += I.pend;
            I.pend = 0;
            I.npf = 0;
            if (I.kv > P.kv_cap && I.n > 1) ev = true;
          } else {  // every running request emits one token
            const int n = I.n;
            if (n != I.el_n) {
              I.dec_el = __dadd_rn(P.dtb, __dmul_rn(P.dpt, (double)n));
              I.el_n = n;
            }
            I.clock = __dadd_rn(I.clock, I.dec_el);
            I.D++;
            I.kv += n;
            I.tleft -= n;
            I.dleft -= n - I.nge;
            if (I.ft < n) {  // first tokens of requests admitted since the last decode
              for (int j = I.ft; j < n; ++j) {
                const int q = rget<kFQ, T>(P, gw, i, j);
                if (q & kFresh) P.o_first[off + (q & kReqMask)] = I.clock;
              }
              I.ft = n;
            }
            if (I.D >= I.ev_at || I.kv > P.kv_cap) {
              ev = true;
            } else if (I.w_cnt == 0 && I.clock < t1) {  // a second pure decode step
              I.clock = __dadd_rn(I.clock, I.dec_el);
              I.D++;
              I.kv += n;
              I.tleft -= n;
              I.dleft -= n - I.nge;
              if (I.D >= I.ev_at || I.kv > P.kv_cap) ev = true;
            }
          }
        }
      }
      act = act && I.clock < t1;
      const bool any_ev = L.any(ev);
      again = L.any(act);
      if (!any_ev) continue;
      // ---- events (warp): errors, completion scans, preemption ----------
      if (L.any(ev && I.n == 0)) {  // nothing admissible: re-run in index order
        perr = true;
        break;
      }
      const bool sc = ev && (I.D >= I.next_done || I.D >= I.next_ge) && I.npf == 0 &&
                      I.el_n == I.n;
      unsigned sm = L.ballot(sc);
      while (sm) {
        const int owner = __ffs(sm) - 1;
        sm &= sm - 1;
        warp_scan_instance<W, false, T>(P, gw, off, Q.wid * W + owner, owner, I, L);
      }
      if (ev && I.kv > P.kv_cap && I.n > 1) lane_preempt<T>(P, gw, off, i, I);
    }
    lcomp += I.comps;
    I.comps = 0;
    lsw += I.w_cnt + I.o_cnt;
    R.clock = t1;
    if (R.clock >= R.next_arr) {  // inject_arrivals only when due
      inject();
      next_arrival();
    }
    R.tick++;
    R.sum_q += queue_len<POL>(R);
  }
  if (pair_any(Q, perr)) return kRerunSeq;
  // fleet totals: each warp's sums, exchanged
  const int c = L.sum(lcomp);
  const long long w = L.sum_ll(lsw);
  int oc, ohi, olo;
  bool nerr = false;
  pair_swap3(Q, l, c, (int)(w >> 32), (int)w, oc, ohi, olo, false, nerr);
  R.completed = c + oc;
  R.sum_w = w + (long long)(((unsigned long long)(unsigned)ohi << 32) | (unsigned)olo);
  if (R.status == RS_REPLAY_FINISHED && R.completed != R.n) R.status = RS_REPLAY_MAX_TICKS;
  if (R.status != RS_REPLAY_FINISHED) return kRerunInit;
  if (Q.wid == 0) write_replay_stats(P, R, r, L);
  return kDone;
}

// Warp pairs: block = 2 x pairs warps; pair p uses shared slot p and named
// barrier 1 + p.  A replay the pair cannot finish exactly (errors, max_ticks)
// is re-run by warp 0 on the two-instances-per-lane code.
template <int POL, int T>
__global__ void replay_pair_kernel(const __grid_constant__ KParams P) {
  extern __shared__ __align__(16) char smem[];
  const Lanes<kWarp> L = make_lanes<kWarp>();
  const int warp = threadIdx.x >> 5;
  Pair Q;
  Q.wid = warp & 1;
  Q.bar = 1 + (warp >> 1);
  int gbyte = (warp >> 1) * P.smem_group_bytes;
  asm volatile("" : "+r"(gbyte));
  char* gbase = smem + gbyte;
  const int gw = gbyte >> 2;
  Q.xw = reinterpret_cast<int*>(gbase + P.off_pair);
  Q.bank = 0;
  MlpView M{};
  for (;;) {
    int r = 0;
    if (Q.wid == 0 && L.l == 0) Q.xw[16] = atomicAdd(P.work_counter, 1);
    pair_sync(Q);
    r = Q.xw[16];
    pair_sync(Q);  // (the word is rewritten only after both read it)
    if (r >= P.num_replays) break;
    const FastRun o = run_replay_pair<POL, T>(P, gw, gbase, r, L, Q);
    if (o != kDone) {
      pair_sync(Q);  // warp 1 parks while warp 0 re-runs the replay alone
      if (Q.wid == 0) {
        int fin = 0, fch = 0;
        if (o == kRerunSeq)
          run_replay_fast<POL, 2, kWarp, true, T, 0>(P, gw, gbase, M, r, true, fin, fch, L);
        else
          run_replay_fast<POL, 2, kWarp, false, T, 0>(P, gw, gbase, M, r, true, fin, fch, L);
      }
      pair_sync(Q);
    }
  }
}

}  // namespace rs
