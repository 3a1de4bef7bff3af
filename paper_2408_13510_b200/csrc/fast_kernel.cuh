// fast_kernel.cuh — tick loop of the fast (lane = instance) replay kernel.
#pragma once

#include "fast.cuh"

namespace rs {

// InstanceFeatures (instance.hpp:317-360) of the lane's instance at a tick
// boundary, from the maintained aggregates.  At a step boundary every
// admitted prompt has been prefilled (whole-prompt prefill), so running
// prompt-bucket counts and pending running prompt tokens are zero.
struct FeatI {  // InstanceFeatures subset (fast kernel)
  long long res, pend, dleft, tleft, tok;  // running + waiting (queues grow with the trace)
  int cnt, kv, nrun, mind;
};

__device__ __forceinline__ bool can_accept(const KParams& P, const FeatI& f, int need) {
  return P.kv_cap - f.res >= need && f.cnt < P.max_batch;  // policies.hpp:44-48
}

__device__ __forceinline__ FeatI feat_of(const Inst& I) {
  FeatI f;
  f.res = (long long)res_run(I) + I.tokw + I.dlw;  // reserved = token mass + decode left
  f.pend = I.pend + I.pendw;
  f.dleft = I.dleft + I.dlw;
  f.tleft = I.tleft + I.tlw;
  f.tok = (long long)tok_run(I) + I.tokw;
  f.cnt = I.n + I.w_cnt + I.o_cnt;
  f.kv = I.kv;
  f.nrun = I.n;
  f.mind = I.n == 0 ? 0 : (I.nge > 0 ? 0 : I.next_ge - I.D);
  return f;
}

// Lowest lane (< width) holding the minimal key among valid lanes; all valid
// lanes lie below `width` (a power of two), so log2(width) butterfly rounds.
template <int W>
__device__ __forceinline__ int argmin_narrow(const Lanes<W>& L, unsigned long long key, bool valid,
                                             int width) {
  if (W == kWarp) {
    // whole warp: two 32-bit warp-minimum reductions (high word, then the low
    // word among the lanes tied on it) instead of log2(width) 64-bit shuffles
    const unsigned long long k = valid ? key : ~0ull;
    const unsigned hi = (unsigned)(k >> 32);
    const unsigned mh = __reduce_min_sync(kFull, hi);
    const bool tie = hi == mh;
    const unsigned ml = __reduce_min_sync(kFull, tie ? (unsigned)k : 0xffffffffu);
    const unsigned ok = L.ballot(valid && tie && (unsigned)k == ml);
    return ok ? __ffs(ok) - 1 : -1;
  }
  unsigned long long k = valid ? key : ~0ull;
  for (int o = width >> 1; o > 0; o >>= 1) {
    const unsigned long long w = L.shfl_xor(k, o);
    k = w < k ? w : k;
  }
  const unsigned ok = L.ballot(valid && key == k);
  return ok ? __ffs(ok) - 1 : -1;
}

// Lowest group lane whose key is minimal (maximal) among valid lanes; -1 if none.
template <int W>
__device__ __forceinline__ int grp_argmin_key(const Lanes<W>& L, unsigned long long key, bool valid) {
  const unsigned long long k = valid ? key : ~0ull;
  const unsigned long long mn = L.min_u64(k);
  const unsigned ok = L.ballot(valid && k == mn);
  return ok ? __ffs(ok) - 1 : -1;
}
template <int W>
__device__ __forceinline__ int grp_argmax_key(const Lanes<W>& L, unsigned long long key, bool valid) {
  const unsigned long long k = valid ? key : 0ull;
  const unsigned long long mx = L.max_u64(k);
  const unsigned ok = L.ballot(valid && k == mx);
  return ok ? __ffs(ok) - 1 : -1;
}

template <int POL, int G, int W, int T>
__device__ __forceinline__ int decide_fast(const KParams& P, int gw, const MlpView& M, Replay& R,
                                  Inst (&S)[G], bool has_head, const Rec& hr, int hb,
                                  char* gbase, const Lanes<W>& L) {
  const int l = L.l;
  const int m = P.m;
  const int need = reserved_of(hr.prompt, hr.dhat, 0);
  if (POL == RS_POLICY_ROUND_ROBIN || POL == RS_POLICY_DEDICATED_SMALL_LARGE) {
    if (!has_head) return m;
    int t;
    if (POL == RS_POLICY_ROUND_ROBIN) {  // policies.hpp:50-69
      t = (int)(R.rr_next % (unsigned long long)m);
    } else {  // policies.hpp:73-104
      if (m < 2 || hr.dhat >= P.dsl_cutoff) t = 0;
      else t = 1 + (int)(R.dsl_next % (unsigned long long)(m - 1));
    }
    bool ok = false;
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (g * W + l == t) ok = can_accept(P, feat_of(S[g]), need);
    ok = L.shfl(ok, t & (W - 1));
    if (!ok) return m;
    if (POL == RS_POLICY_ROUND_ROBIN) R.rr_next++;
    else if (m >= 2 && t >= 1) R.dsl_next++;
    return t;
  } else if (POL == RS_POLICY_EARLIEST_AVAILABLE) {  // policies.hpp:214-228
    if (!has_head) return m;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i = g * W + l;
      const bool ok = i < m && (long long)P.kv_cap - feat_of(S[g]).res >= need;
      const unsigned b = L.ballot(ok);
      if (b) return g * W + __ffs(b) - 1;
    }
    return m;
  } else if (POL == RS_POLICY_MAX_CAPACITY) {  // policies.hpp:150-170
    if (!has_head || R.clock < R.mc_next) return m;
    unsigned long long bk = 0;
    int bi = -1;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i = g * W + l;
      const bool v = i < m;
      const unsigned long long k = v ? ordered_key(capacity_of(P, S[g].kv)) : 0ull;
      const int a = grp_argmax_key(L, k, v);
      if (a >= 0) {
        const unsigned long long ka = L.shfl(k, a);
        if (bi < 0 || ka > bk) { bk = ka; bi = g * W + a; }
      }
    }
    bool ok = false;
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (g * W + l == bi) ok = (long long)P.kv_cap - feat_of(S[g]).res >= need;
    ok = L.shfl(ok, bi & (W - 1));
    if (!ok) return m;
    R.mc_next = __dadd_rn(R.clock, 1.0);
    return bi;
  } else if (POL == RS_POLICY_RL) {  // RlPolicy + encode_state (env.hpp:88-113)
    double* x = reinterpret_cast<double*>(gbase + P.off_rlx);
    const int nsb = P.n_state_edges;
    const int per = 3 + nsb;
    // The state is written over the previous tick's in place; a lane notes
    // whether any of its words changed bitwise.  An unchanged state has the
    // same greedy action (the forward is a function of x's bits): a third
    // to nearly half of all ticks repeat the previous state exactly
    // (c3 34%, c4's RL cells 42-45%, measured on the oracle).
    bool chg = false;
    auto put = [&](double* p, double v) {
      chg |= __double_as_longlong(*p) != __double_as_longlong(v);
      *p = v;
    };
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i = g * W + l;
      if (i < m) {
        const FeatI f = feat_of(S[g]);
        double* xi = x + i * per;
        put(xi, div_exact((double)f.pend, (double)P.kv_cap, P.inv_kv, P.kv_pow2));
        // decode-bucket counts of the running batch (every running request
        // is in its decode phase at a tick boundary), counted by the owner
        // lane: cge[b] = #requests with decode_left >= state edge b
        int cge[RS_MAX_BUCKETS + 1];
#pragma unroll
        for (int b = 0; b < RS_MAX_BUCKETS; ++b) cge[b] = 0;
        if (nsb == 3) {  // three state edges {0, e1, e2} (BucketScheme::state_default)
          // tracked counts, exact until decode_left of a tracked entry drops
          // below an edge (D reaches nx1 / nx2): then recount the batch
          Inst& I = S[g];
          if (I.D >= I.nx1 || I.D >= I.nx2) {
            I.sb1 = I.sb2 = 0;
            I.nx1 = I.nx2 = kBig;
            for (int j = 0; j < I.n; ++j)
              sb_add(P, I, rget<kFD, T>(P, gw, i, j) - (I.D + rget<kFK, T>(P, gw, i, j)));
          }
          cge[1] = I.sb1;
          cge[2] = I.sb2;
        } else {
          for (int j = 0; j < S[g].n; ++j) {
            int d = rget<kFD, T>(P, gw, i, j) - (S[g].D + rget<kFK, T>(P, gw, i, j));
            d = d > 0 ? d : 0;
#pragma unroll
            for (int b = 1; b < RS_MAX_BUCKETS; ++b)
              if (b < nsb) cge[b] += d >= P.state_edges[b];
          }
        }
#pragma unroll
        for (int b = 0; b < RS_MAX_BUCKETS; ++b) {
          if (b >= nsb) break;
          const int hi = b + 1 < nsb ? cge[b + 1] : 0;
          const int c = (b == 0 ? S[g].n : cge[b]) - hi;
          put(xi + 1 + b, div_exact((double)c, (double)P.max_batch, P.inv_mb, P.mb_pow2));
        }
        put(xi + 1 + nsb, round2(capacity_of(P, f.kv)));
        const double that = f.nrun == 0 ? 0.0 : __dmul_rn(P.dtb, (double)f.mind);
        put(xi + 2 + nsb, round2(that));
      }
    }
    if (l == 0) {
      const int q = queue_len<POL>(R);
      // min(Q, 512) / 512 and prompt / 1024: power-of-two divisors of small
      // integers, so the quotient is an exact multiply (no division sequence)
      put(x + m * per, __dmul_rn((double)(q < 512 ? q : 512), 0x1p-9));
      put(x + m * per + 1, has_head ? __dmul_rn((double)hr.prompt, 0x1p-10) : 0.0);
      put(x + m * per + 2, has_head ? (double)hb : 0.0);
    }
    L.sync();
    if (L.any(chg)) R.rl_prev = -1;
    const int na = P.rl_dims[P.rl_layers];
    if (P.rl_eps > 0.0) {  // DqnAgent::act (dqn.hpp:92-99)
      unsigned long long* rng = reinterpret_cast<unsigned long long*>(gbase + P.off_rng);
      const double u = u01(rng_draw(rng, R, L));
      if (u < P.rl_eps) {
        const double v = __dmul_rn(u01(rng_draw(rng, R, L)), (double)na);
        const unsigned long long k = (unsigned long long)v;
        return (int)(k < (unsigned long long)na ? k : (unsigned long long)na - 1);
      }
    }
    if (!P.rl_wt_global) {  // staged weights: LDS-only forward over nonzero inputs
      // x | h0 | h1 | nonzero list, each region an even number of doubles
      // (16-byte aligned: the list records and the paired weights load as
      // 16-byte vectors)
      const int xd = (gw >> 1) + (P.off_rlx >> 3);
      const int mw = (P.rl_maxw + 1) & ~1;
      const int h0d = xd + ((P.rl_dims[0] + 1) & ~1), h1d = h0d + mw, lvd = h1d + mw;
      if (R.rl_prev < 0)
        R.rl_prev = mlp_forward_list(P.rl_dims, P.rl_woff, P.rl_boff, P.rl_layers, xd, h0d, h1d,
                                     lvd, L, R.qmacs);
      return R.rl_prev;
    }
    double* h0 = x + M.dims[0];
    double* h1 = h0 + P.rl_maxw;
    if (R.rl_prev < 0) R.rl_prev = mlp_forward_warp(M, x, h0, h1, nullptr, L, &R.qmacs);
    return R.rl_prev;
  } else {  // argmin policies
    if (!has_head) return m;
    if (POL == RS_POLICY_DECODE_BALANCER || POL == RS_POLICY_WORKLOAD_AWARE) {
      // a saturated fleet defers most ticks: skip the scores when no
      // instance can take the head (the reference's result is `defer`)
      bool any_ok = false;
#pragma unroll
      for (int g = 0; g < G; ++g)
        any_ok |= (g * W + l < m) && can_accept(P, feat_of(S[g]), need);
      if (!L.any(any_ok)) return m;
    }
    unsigned long long bk = ~0ull;
    int bi = -1;
    // G > 1: each lane first keeps the best of its own instances (lower g
    // wins ties, i.e. the lower index), then ONE warp minimum; the lowest
    // index holding it is the lowest g, then the lowest lane, among the lanes
    // whose own best equals the minimum
    int lg = -1;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i = g * W + l;
      bool v = i < m;
      unsigned long long k = ~0ull;
      if (v) {
        const FeatI f = feat_of(S[g]);
        if (POL == RS_POLICY_DECODE_BALANCER) {  // policies.hpp:108-127
          v = can_accept(P, f, need);
          k = (unsigned long long)f.tleft;
        } else if (POL == RS_POLICY_JSQ) {  // policies.hpp:131-146
          k = (unsigned long long)(f.pend + f.dleft);
        } else if (POL == RS_POLICY_MIN_MIN) {  // policies.hpp:193-206
          k = ordered_key(__dadd_rn(__dmul_rn((double)f.pend, P.tpp),
                                    __dmul_rn((double)f.dleft, P.dtb)));
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
      if (G == 1) {
        bi = argmin_narrow(L, k, v, P.mwidth);
      } else if (v && (lg < 0 || k < bk)) {
        bk = k;
        lg = g;
      }
    }
    if (G > 1) {
      const bool lv = lg >= 0;
      const unsigned long long mn = L.min_u64(lv ? bk : ~0ull);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const unsigned b = L.ballot(lv && lg == g && bk == mn);
        if (bi < 0 && b) bi = g * W + __ffs(b) - 1;
      }
    }
    if (POL == RS_POLICY_JSQ || POL == RS_POLICY_MIN_MIN) return bi;
    return bi < 0 ? m : bi;
  }
}

// Fused predictor: the predictions of the 32 requests of the arrival window
// [a_base, a_base + 32), drawn in index order from the replay's own
// mt19937_64 stream exactly as inject_arrivals draws them (env.hpp:357-375,
// predict_simulated predictor.hpp:98-110: one draw, a second for a miss in a
// middle bucket).  The stream is policy independent, so drawing a window
// ahead of injection is equivalent.  Written to the predicted-bucket output.
// Out of line (once per 32 arrivals): inlined, the draw loop and its bucket
// searches sat in the tick loop's instruction footprint.  Returns the
// stream position after the window.
template <int W>
__device__ __noinline__ int predict_window_cold(const KParams& P, int a_base, int n, long long off,
                                                int pos, unsigned long long* pst, const Lanes<W> L) {
  const int l = L.l;
  const int j = a_base + l;
  const bool v = j < n;
  const long long g = off + j;
  int pred = 0;
  if (P.predictor_mode == RS_PREDICTOR_GIVEN) {
    if (v) pred = P.given_bucket[g];
  } else if (P.predictor_mode == RS_PREDICTOR_EMPIRICAL) {  // predictor.hpp:146-158
    if (v) pred = P.emp_table[P.task[g]][bucket_of(P.band_edges, P.n_band_edges, P.prompt[g])];
  } else {
    const int nb = P.n_pred_edges;
    int tb = 0;
    double acc = 1.0;
    if (v) {
      tb = bucket_of(P.pred_edges, nb, P.decode[g]);
      acc = P.accuracy[P.task[g]];
    }
    const int cnt = min(W, n - a_base);
    for (int k = 0; k < cnt; ++k) {
      const int tbk = L.shfl(tb, k);
      const double ak = L.shfl(acc, k);
      int pk = 0;
      if (nb > 1) {
        if (pos == 312) {
          mt_twist(pst, L);  // outputs are tempered as they are drawn
          pos = 0;
        }
        const double u = u01(mt_temper(pst[pos++]));
        if (u < ak) {
          pk = tbk;
        } else if (tbk == 0) {
          pk = 1;
        } else if (tbk == nb - 1) {
          pk = nb - 2;
        } else {
          if (pos == 312) {
            mt_twist(pst, L);
            pos = 0;
          }
          pk = u01(mt_temper(pst[pos++])) < 0.5 ? tbk - 1 : tbk + 1;
        }
      }
      if (l == k) pred = pk;
    }
  }
  if (v) P.o_pred[g] = (uint8_t)pred;
  L.sync();
  return pos;
}
template <int W>
__device__ __forceinline__ void predict_window(const KParams& P, Replay& R, unsigned long long* pst,
                                              const Lanes<W>& L) {
  R.pred_pos = predict_window_cold(P, R.a_base, R.n, R.off, R.pred_pos, pst, L);
}

template <int W>
__device__ __forceinline__ void load_window_fast(const KParams& P, Replay& R,
                                                 unsigned long long* pst, const Lanes<W>& L) {
  const int l = L.l;
  if (P.resident) {
    // streamed inputs: wait until the copy stream has landed this window
    const int need = min(R.n, R.a_base + W);
    if (need > R.resident_seen) {
      // every lane acquires; the warp minimum is visible to all of them
      int v = L.min(load_acquire(P.resident));
      if (v < need) {
        const unsigned long long t0 = globaltimer_ns();
        while (v < need) {
          __nanosleep(256);
          v = L.min(load_acquire(P.resident));
          if (v < need && L.any(globaltimer_ns() - t0 > kStreamTimeoutNs)) {
            R.status = RS_REPLAY_NOT_RUN;  // copy stream never delivered
            return;
          }
        }
      }
      R.resident_seen = v;
    }
    const double prev_last = L.shfl(R.a_val, W - 1);
    load_arrival_window(P, R, L);
    // lazy validation of the window (the up-front pass cannot read inputs
    // that are still in flight): arrivals non-decreasing, token ranges, and
    // the 32-bit aggregate bound over the requests seen so far
    const int j = R.a_base + l;
    const bool v = j < R.n;
    bool bad = false;
    if (v) {
      const long long g = R.off + j;
      const int p = P.prompt[g], d = P.decode[g];
      bad = p < 1 || p > kMaxTokens || d < 1 || d > kMaxTokens;
    }
    const double up = L.shfl_up(R.a_val, 1);
    const double prev = l == 0 ? prev_last : up;
    if (v && j > 0 && R.a_val < prev) bad = true;
    if (L.any(bad)) R.status = RS_REPLAY_INVALID_TRACE;
  } else {
    load_arrival_window(P, R, L);
  }
  if (P.predict_inline) predict_window(P, R, pst, L);
}

// ClusterSim::inject_arrivals (env.hpp:357-375): a cursor advance over the
// register window of arrival times; the next window is predicted on load.
template <int W>
__device__ __forceinline__ void inject_fast(const KParams& P, Replay& R, unsigned long long* pst,
                                            const Lanes<W>& L) {
  const int l = L.l;
  for (;;) {
    const int j = R.a_base + l;
    const bool ok = j >= R.cursor && j < R.n && R.a_val <= R.clock;
    R.cursor += __popc(L.ballot(ok));
    if (R.cursor == R.a_base + W && R.cursor < R.n) {
      R.a_base += W;
      load_window_fast(P, R, pst, L);
      if (R.status != RS_REPLAY_FINISHED) break;  // streamed window failed validation
      continue;
    }
    break;
  }
}

// Outcome of one pass over a replay.
enum FastRun { kDone = 0, kRerunSeq = 1, kRerunInit = 2 };

// `init` writes the reference's "not yet" values (-1) into the instance /
// routed / first-token / completion outputs up front.  A replay that
// finishes overwrites every one of them, so the first pass skips those
// writes (32 -> 4 B/request of initialisation traffic) and a replay that
// ends unfinished (livelock, max_ticks, errors: rare) is re-run with init.
// `seq` steps instances one at a time in index order (exact stop point of a
// "nothing admissible" error).
// Streamed outputs: advance the replay's final prefix `fin` (every request
// below it has completed: its outputs are final) and count the replay into
// every chunk mark it has passed.  Called after ticks that completed
// something and finished without error: a tick cut short by "nothing
// admissible" is re-run in index order and may end with fewer completions,
// so it publishes nothing.  The writes of the whole warp are fenced system
// wide before a mark moves (the copy engine reads them next).
template <int W>
__device__ __forceinline__ void publish_final(const KParams& P, long long off, int n, int upto,
                                           int& fin, int& fch, const Lanes<W>& L) {
  if (L.l == 0)
    while (fin < upto && P.o_completion[off + fin] >= 0.0) ++fin;
  fin = L.shfl(fin, 0);
  if (fch < P.n_out_bounds && fin >= min(P.out_bounds[fch], n)) {
    __threadfence_system();
    L.sync();
    if (L.l == 0)
      while (fch < P.n_out_bounds && fin >= min(P.out_bounds[fch], n))
        atomicAdd(P.out_marks + fch++, 1);
    fch = L.shfl(fch, 0);
  }
}

// SO: streamed outputs (publish_final) — 0 = not compiled in, 1 = on
// (the replay_fast_kernel_lat_so build), 2 = compiled in behind a runtime
// test of P.out_marks.  Which form each build uses is a measured choice
// (A/B on one box): the plain latency build is fastest with 0 (c2); the
// two-instance-per-lane and throughput builds run measurably faster with
// the runtime form (ptxas schedules the tick loop differently; c5 1.30 s
// with 0 against 1.00 s with 2).
template <int POL, int G, int W, bool SEQ, int T, int SO>
__device__ __forceinline__ FastRun run_replay_fast(const KParams& P, int gw, char* gbase, const MlpView& M, int r,
                                   bool init, int& fin, int& fch, const Lanes<W>& L) {
  constexpr bool seq = SEQ;  // compile-time: the index-order re-run is a separate instantiation
  const int l = L.l;
  Replay R;
  R.off = P.offsets[r];
  R.n = (int)(P.offsets[r + 1] - R.off);
  const int m = P.m;
  const long long off = R.off;
  int* front = reinterpret_cast<int*>(gbase + P.off_front);

  bool bad = false;
  if (!init && P.vinfo) {  // validated and zeroed by the validate_kernel pre-pass
    bad = P.vinfo[r].x != 0;
  } else for (int j = l; j < R.n; j += W) {
    const long long g = off + j;
    if (init && (SO == 0 || j >= fin)) {  // (streamed outputs: below fin already published, rewritten identically)
      P.o_instance[g] = -1;
      P.o_routed[g] = -1.0;
      P.o_first[g] = -1.0;
      P.o_completion[g] = -1.0;
    }
    P.o_preempt[g] = 0;
    if (POL == RS_POLICY_MIN_MIN) P.mm_removed[g] = 0;
    if ((SO == 1 || (SO == 2 && P.out_marks)) && !init)
      P.o_completion[g] = -1.0;  // not completed (publish_final)
    if (P.resident) continue;  // streamed inputs: validated per window on load
    const int p = P.prompt[g], d = P.decode[g];
    if (p < 1 || p > kMaxTokens || d < 1 || d > kMaxTokens) bad = true;
    if (j > 0 && P.arrival[g] < P.arrival[g - 1]) bad = true;
  }
  bad = L.any(bad);
  Inst S[G];
#pragma unroll
  for (int g = 0; g < G; ++g) inst_init(S[g]);
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
  if (POL == RS_POLICY_RL && P.rl_eps > 0.0)
    mt_seed(reinterpret_cast<unsigned long long*>(gbase + P.off_rng),
            P.policy_seed ? P.policy_seed[r] : 0ull, L);
  unsigned long long* pst = reinterpret_cast<unsigned long long*>(gbase + P.off_pred);
  R.pred_pos = 312;
  R.a_val = 0.0;
  R.resident_seen = 0;
  R.rl_prev = -1;
  if (P.predict_inline && P.predictor_mode == RS_PREDICTOR_SIMULATED)
    mt_seed(pst, P.predictor_seed[r], L);  // Rng(predictor_seed), env.hpp:173
  L.sync();
  load_window_fast(P, R, pst, L);
  // arrival time of the next request to inject (+inf when none is left)
  auto next_arrival = [&]() {
    const int k = R.cursor - R.a_base;
    const double a = L.shfl(R.a_val, k & (W - 1));
    R.next_arr = R.cursor < R.n ? a : __longlong_as_double(0x7ff0000000000000ll);
  };
  R.hr_q = -1;
  R.hr_prompt = R.hr_true = R.hr_bucket = 0;
  if (bad) R.status = RS_REPLAY_INVALID_TRACE;
  else if (R.status == RS_REPLAY_FINISHED) inject_fast(P, R, pst, L);
  next_arrival();

  // Per-lane tick accounting, reduced once at the end: completions of the
  // lane's instances, and the sum over ticks of their end-of-tick waiting
  // counts (the router's per-tick sum of instance waiting, env.hpp:326-337).
  int lcomp = 0;
  long long lsw = 0;
  while (R.status == RS_REPLAY_FINISHED && R.tick < P.max_ticks) {
    // run_policy's done() (every request completed) once every request has
    // arrived and been routed: no instance holds work
    if (R.cursor == R.n && queue_len<POL>(R) == 0) {
      bool busy = false;
#pragma unroll
      for (int g = 0; g < G; ++g) busy |= S[g].n > 0 || S[g].w_cnt > 0;
      if (!L.any(busy)) break;
    }
    if (POL == RS_POLICY_MIN_MIN && queue_len<POL>(R) > 0) {
      if (!minmin_pick(P, front, R, L)) { R.status = RS_REPLAY_CAPACITY; break; }
    }
    const bool has_head = queue_len<POL>(R) > 0;
    Rec hr;
    int hb = 0;
    if (has_head) {
      if (POL != RS_POLICY_MIN_MIN && R.hr_q == R.qhead) {  // same head as last tick
        hr.req = R.qhead;
        hr.prompt = R.hr_prompt;
        hr.tru = R.hr_true;
        hb = R.hr_bucket;
        hr.dhat = P.ub[hb];
        hr.emit = 0;
      } else {
        hr = head_rec<POL>(P, front, R, &hb, L);
        R.hr_q = hr.req;
        R.hr_prompt = hr.prompt;
        R.hr_true = hr.tru;
        R.hr_bucket = hb;
      }
    } else {
      hr.req = hr.prompt = hr.dhat = hr.tru = hr.emit = 0;
    }
    const int action = decide_fast<POL, G, W, T>(P, gw, M, R, S, has_head, hr, hb, gbase, L);
    R.hash = hash_action(R.hash, action);
    // env.hpp:252-254: only an agent can produce an out-of-range action (the
    // heuristics return 0..m by construction)
    if (POL == RS_POLICY_RL && (action < 0 || action > m)) {
      R.status = RS_REPLAY_BAD_ACTION;
      break;
    }
    const double t1 = __dadd_rn(R.clock, P.delta_t);
    if (action < m && has_head) {
      if ((long long)hr.prompt + hr.tru > P.kv_cap) {
        R.infeasible++;  // env.hpp:262-267: flagged, stays queued
      } else {
        if (POL == RS_POLICY_MIN_MIN && R.nfront > 0) {
          if (l == 0)
            for (int k = 0; k + 1 < R.nfront; ++k) front[k] = front[k + 1];
          L.sync();
          R.nfront--;
        } else {
          R.qhead++;
          if (POL == RS_POLICY_MIN_MIN) mm_skip_removed(P, R, L);
        }
        if (l == 0) {
          P.o_routed[off + hr.req] = R.clock;
          P.o_instance[off + hr.req] = action;
        }
        R.routed++;
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (g * W + l == action) {
            lane_enqueue(P, gw, off, action, S[g], hr, R.clock);
          }
      }
    }

    // ---- run_until(t1) for every instance (env.hpp:277-287) -----------
    // One warp collective per iteration: an OR-reduction of (event | again).
    bool act[G];
    bool again = false;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i = g * W + l;
      act[g] = false;
      if (i < m && S[g].clock < t1) {
        if (S[g].n > 0 || S[g].w_cnt > 0) act[g] = true;
        else S[g].clock = t1;  // idle instance skips ahead (instance.hpp:309)
      }
      again |= act[g];
    }
    unsigned fl = L.any(again) ? 2u : 0u;
    while (fl & 2u) {
      if (SEQ) {  // only the lowest-index instance that still has work
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int i = g * W + l;
          act[g] = false;
          if (i < m && S[g].clock < t1) {
            if (S[g].n > 0 || S[g].w_cnt > 0) act[g] = true;
            else S[g].clock = t1;
          }
        }
        int g0 = G;
#pragma unroll
        for (int g = G - 1; g >= 0; --g)
          if (L.ballot(act[g])) g0 = g;
        const unsigned lm = L.ballot(act[g0 < G ? g0 : 0]);
#pragma unroll
        for (int g = 0; g < G; ++g) act[g] = act[g] && g == g0 && l == __ffs(lm) - 1;
      }
      bool ev = false;
      unsigned evg = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (!act[g]) continue;
        Inst& I = S[g];
        const int i = g * W + l;
        if (I.n == 0 && I.w_cnt == 0) {  // emptied by last iteration's events
          I.clock = t1;
          act[g] = false;
          continue;
        }
        // a prefill is only ever pending right after an admission, and an
        // instance with an empty batch has waiting work (checked above), so
        // the common decode step skips both tests
        bool prefill = false;
        if (I.w_cnt > 0 && I.n < P.max_batch) {
          lane_admit<T>(P, gw, off, i, I);
          if (I.n == 0) {  // logic_error, instance.hpp:209-211
            ev = true;
            evg |= 1u << g;
            continue;
          }
          prefill = I.npf > 0;
        }
        if (prefill) {  // whole-prompt prefill; co-running decodes stall
          I.clock = __dadd_rn(I.clock, __dadd_rn(__dadd_rn(P.intercept,
                                                           __dmul_rn(P.tpp, (double)I.pend)),
                                                 __dmul_rn(P.dpt, (double)I.kv)));
          I.kv += I.pend;
          I.pend = 0;
          I.npf = 0;
          if (I.kv > P.kv_cap && I.n > 1) { ev = true; evg |= 1u << g; }
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
          // KV overflow needs n > 1, but a lone request never overflows: it
          // was routed only if prompt + true decode fit (env.hpp:262-267)
          if (I.D >= I.ev_at || I.kv > P.kv_cap) {
            ev = true;
            evg |= 1u << g;
          } else if (I.w_cnt == 0 && I.clock < t1) {
            // Nothing waits, so the next step of this instance is another
            // pure decode step (no admission can precede it): take it now
            // instead of in a further warp iteration (decode steps are
            // ~17 ms against the 20 ms tick, so this is the common case).
            I.clock = __dadd_rn(I.clock, I.dec_el);
            I.D++;
            I.kv += n;
            I.tleft -= n;
            I.dleft -= n - I.nge;
            if (I.D >= I.ev_at || I.kv > P.kv_cap) {
              ev = true;
              evg |= 1u << g;
            }
          }
        }
      }
      // a stepped instance steps again while its clock is behind t1 (it has
      // work: only events can empty it, and the next iteration checks that)
      again = false;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        act[g] = act[g] && S[g].clock < t1;
        // sequential mode keeps going while ANY instance still has a step
        again |= seq ? (g * W + l < m && S[g].clock < t1 &&
                        (S[g].n > 0 || S[g].w_cnt > 0))
                     : act[g];
      }
      fl = (L.any(again) ? 2u : 0u) | (L.any(ev) ? 1u : 0u);
      if (!(fl & 1u)) continue;
      // ---- events (whole warp): errors, completion scans, preemption ----
      {
        int err = kBig;
#pragma unroll
        for (int g = 0; g < G; ++g)
          if ((evg >> g) & 1u)
            if (S[g].n == 0) err = min(err, g * W + l);
        err = L.min(err);
        if (err != kBig) {
          if (!seq) return kRerunSeq;  // exact stop point needs index order: re-run
          R.status = RS_REPLAY_NOT_ADMISSIBLE;
          R.err_inst = err;
          break;
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const bool mine = (evg >> g) & 1u;
        const bool sc = mine && (S[g].D >= S[g].next_done || S[g].D >= S[g].next_ge) &&
                        S[g].npf == 0 && S[g].el_n == S[g].n;
        unsigned sm = L.ballot(sc);
        while (sm) {
          const int owner = __ffs(sm) - 1;
          sm &= sm - 1;
          warp_scan_instance<W, POL == RS_POLICY_RL, T>(P, gw, off, g * W + owner, owner, S[g], L);
        }
        if (mine && S[g].kv > P.kv_cap && S[g].n > 1) {
          lane_preempt<T>(P, gw, off, g * W + l, S[g]);
        }
      }
    }
    if (R.status != RS_REPLAY_FINISHED) break;
    int comps = 0, wn = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      comps += S[g].comps;
      S[g].comps = 0;
      wn += S[g].w_cnt + S[g].o_cnt;
      // An instance emptied by this tick's last events skips ahead to t1
      // (instance.hpp:309) lazily: nothing reads an idle instance's clock
      // before either the next run_until (which snaps it to that tick's t1)
      // or an enqueue (which raises it to the router clock, this t1).
    }
    lcomp += comps;
    lsw += wn;
    if ((SO == 1 || (SO == 2 && P.out_marks)) && L.any(comps != 0))
      publish_final(P, off, R.n, R.cursor, fin, fch, L);
    R.clock = t1;
    if (R.clock >= R.next_arr) {  // inject_arrivals (env.hpp:357-375) only when due
      inject_fast(P, R, pst, L);
      next_arrival();
    }
    R.tick++;
    R.sum_q += queue_len<POL>(R);
  }
  R.completed = L.sum(lcomp);
  R.sum_w = L.sum_ll(lsw);
  if (R.status == RS_REPLAY_FINISHED && R.completed != R.n) R.status = RS_REPLAY_MAX_TICKS;
  if (!init && R.status != RS_REPLAY_FINISHED) return kRerunInit;
  write_replay_stats(P, R, r, L);
  if (SO == 1 || (SO == 2 && P.out_marks)) {  // the replay is over: every output is final
    fin = R.n;
    if (fch < P.n_out_bounds) {
      __threadfence_system();
      L.sync();
      if (L.l == 0)
        while (fch < P.n_out_bounds) atomicAdd(P.out_marks + fch++, 1);
      fch = L.shfl(fch, 0);
    }
  }
  return kDone;
}

template <int POL, int G, int W, int T, int SO>
__device__ __forceinline__ void replay_fast_body(const KParams& P) {
  extern __shared__ __align__(16) char smem[];
  const Lanes<W> L = make_lanes<W>();
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
  // one shared-memory slot per lane group (32/W replays per warp)
  int gbyte = groups_off + (int)(threadIdx.x / W) * P.smem_group_bytes;
  asm volatile("" : "+r"(gbyte));  // keep the group base in a register
  char* gbase = smem + gbyte;
  const int gw = gbyte >> 2;
  for (;;) {
    int r = 0;
    if (L.l == 0) r = atomicAdd(P.work_counter, 1);
    r = L.shfl(r, 0);
    if (r >= P.num_replays) break;
    int fin = 0, fch = 0;  // streamed outputs: final prefix, next chunk mark
    const FastRun o =
        run_replay_fast<POL, G, W, false, T, SO>(P, gw, gbase, M, r, false, fin, fch, L);
    if (o == kRerunSeq)
      run_replay_fast<POL, G, W, true, T, SO>(P, gw, gbase, M, r, true, fin, fch, L);
    else if (o == kRerunInit)
      run_replay_fast<POL, G, W, false, T, SO>(P, gw, gbase, M, r, true, fin, fch, L);
  }
}

// Up to 8 replay warps per block, two blocks per SM (<= 128 registers: the
// throughput regime wants 16 resident replays per SM).
template <int POL, int G, int W, int T>
__global__ void __launch_bounds__(256, 2) replay_fast_kernel(const __grid_constant__ KParams P) {
  replay_fast_body<POL, G, W, T, 2>(P);
}

// Latency regime (every replay resident in one wave, <= 8 warps per SM):
// no launch bound, so ptxas keeps the whole tick loop in registers (158 for
// workload_aware, no spills) instead of capping at 128 with ~450 B of spill
// traffic on the tick chain; one such block per SM fits the register file.
template <int POL, int G, int W, int T>
__global__ void replay_fast_kernel_lat(const __grid_constant__ KParams P) {
  replay_fast_body<POL, G, W, T, G == 1 ? 0 : 2>(P);
}

// The latency-regime build with streamed outputs (rs_replay_batch_host with
// page-locked output buffers): replays publish finalised request chunks.
template <int POL, int G, int W, int T>
__global__ void replay_fast_kernel_lat_so(const __grid_constant__ KParams P) {
  replay_fast_body<POL, G, W, T, 1>(P);
}

// Up to 16 (the RL policy in the throughput regime): its Q-network is staged
// once per block, so one wide block per SM leaves the most shared memory for
// replay slots (512 threads x 128 registers = the register file).  A separate
// instantiation: the 512-thread bound changes the code ptxas generates, and
// blocks of <= 8 warps run faster with the 256-thread build (measured, c3).
template <int POL, int G, int W, int T>
__global__ void __launch_bounds__(512) replay_fast_kernel_wide(const __grid_constant__ KParams P) {
  replay_fast_body<POL, G, W, T, 2>(P);
}

}  // namespace rs
