// replay.cuh — kernels (a)+(b)+(c): the fused per-replay tick loop.
//
// One warp owns one replay (ClusterSim) at a time and pulls replay ids from
// an atomic work counter (persistent kernel, load balance across the mix of
// policies / rates / seeds).  Per tick (ClusterSim::step, env.hpp:251-322):
//   router   : decide() from the per-instance aggregates kept in shared
//              memory (lane i scores instance i; warp argmin / argmax with
//              lowest-index tie-break, policies.hpp:50-228);
//   route    : pop the router-queue head, Instance::enqueue (instance.hpp:
//              113-130) into the instance's shared-memory waiting ring;
//   simulate : only instances with work and clock < t1 are stepped
//              (ballot over lanes); Instance::step (instance.hpp:203-277) is
//              warp-parallel over the running batch (<= 4 entries per lane,
//              prefix scans for chunked prefill, ballot/popc compaction of
//              completions), fp64 clocks with explicit _rn operations;
//   arrivals : a 32-wide register window over arrival times (coalesced).
// The reference's per-tick O(N) reward scan (env.hpp:289-298) is off the
// decision path and is not performed.
#pragma once

#include "common.cuh"
#include "mlp.cuh"

namespace rs {

struct Rec {  // a request record in a waiting queue
  int req, prompt, dhat, tru, emit;
};

struct Grp {  // shared-memory view of one replay
  InstHot* inst;
  int *r_req, *r_prompt, *r_prem, *r_emit, *r_true, *r_dhat;
  int *w_req, *w_prompt, *w_dhat, *w_true, *w_emit;
  int* dbc;
  double* rlx;
  unsigned long long* rng;
  int* front;
};

struct Replay {  // per-replay registers (uniform across the warp)
  long long off;
  int n;
  double clock;
  long long tick;
  int qhead, cursor;
  int completed;
  int nfront, n_removed;
  int total_wait;
  unsigned long long rr_next, dsl_next;
  double mc_next;
  unsigned long long hash;
  long long infeasible, routed, sum_q, sum_w;
  int status, err_inst;
  int rng_pos;
  // windows (per-lane registers)
  int a_base;      // arrival window base (replay-local index)
  double a_val;    // arrival[a_base + lane]
  int h_base;      // head window base
  int h_prompt, h_true, h_bucket;
  // fast kernel: arrival time of request `cursor` (+inf when all arrived)
  // and the cached head record (valid while qhead == hr_q)
  double next_arr;
  int hr_q, hr_prompt, hr_true, hr_bucket;
  int pred_pos;  // fused predictor: next unread mt19937_64 output (312 = regenerate)
  int resident_seen;  // streamed inputs: watermark seen
  int rl_prev;  // fast kernel, RL: greedy action of the state held in x (-1: none)
  long long qmacs;  // RL: Q-network multiply-adds executed
};

__device__ __forceinline__ Grp make_grp(const KParams& P, char* base) {
  Grp G;
  G.inst = reinterpret_cast<InstHot*>(base);
  const int mr = P.m * P.rcap, mw = P.m * P.wcap;
  int* run = reinterpret_cast<int*>(base + P.off_run);
  G.r_req = run; G.r_prompt = run + mr; G.r_prem = run + 2 * mr;
  G.r_emit = run + 3 * mr; G.r_true = run + 4 * mr; G.r_dhat = run + 5 * mr;
  int* wt = reinterpret_cast<int*>(base + P.off_wait);
  G.w_req = wt; G.w_prompt = wt + mw; G.w_dhat = wt + 2 * mw; G.w_true = wt + 3 * mw;
  G.w_emit = wt + 4 * mw;
  G.dbc = reinterpret_cast<int*>(base + P.off_dbc);
  G.rlx = reinterpret_cast<double*>(base + P.off_rlx);
  G.rng = reinterpret_cast<unsigned long long*>(base + P.off_rng);
  G.front = reinterpret_cast<int*>(base + P.off_front);
  return G;
}

__device__ __forceinline__ int reserved_of(int prompt, int dhat, int emit) {
  return prompt + (dhat > emit ? dhat : emit);  // instance.hpp:365-368
}

// ------------------------------------------------------- waiting queue
// Logical queue = shared ring (front part, capacity wcap) ++ global
// doubly-linked overflow list (rest).  Invariant: o_cnt > 0 => ring full.

__device__ __forceinline__ void wait_add(InstHot& h, const Rec& r, int sign) {
  h.res_wait += sign * reserved_of(r.prompt, r.dhat, r.emit);
  h.pend_wait += sign * r.prompt;
  const int dl = r.dhat - r.emit;
  h.dleft_wait += sign * (dl > 0 ? dl : 0);
  const int tl = r.tru - r.emit;
  h.tleft_wait += sign * (tl > 0 ? tl : 0);
  h.tok_wait += sign * (r.prompt + r.emit);
}

__device__ __forceinline__ Rec ring_read(const Grp& G, int base, int slot) {
  Rec r;
  r.req = G.w_req[base + slot];
  r.prompt = G.w_prompt[base + slot];
  r.dhat = G.w_dhat[base + slot];
  r.tru = G.w_true[base + slot];
  r.emit = G.w_emit[base + slot];
  return r;
}
__device__ __forceinline__ void ring_write(const Grp& G, int base, int slot, const Rec& r) {
  if (lane_id() == 0) {
    G.w_req[base + slot] = r.req;
    G.w_prompt[base + slot] = r.prompt;
    G.w_dhat[base + slot] = r.dhat;
    G.w_true[base + slot] = r.tru;
    G.w_emit[base + slot] = r.emit;
  }
  __syncwarp();
}

__device__ __forceinline__ void ov_push_back(const KParams& P, long long off, InstHot& h,
                                             const Rec& r) {
  if (lane_id() == 0) {
    P.ov_emit[off + r.req] = r.emit;
    P.ov_next[off + r.req] = kNil;
    P.ov_prev[off + r.req] = h.o_cnt ? (uint32_t)h.o_tail : kNil;
    if (h.o_cnt) P.ov_next[off + h.o_tail] = (uint32_t)r.req;
  }
  if (h.o_cnt == 0) h.o_head = r.req;
  h.o_tail = r.req;
  h.o_cnt++;
}

__device__ __forceinline__ void ov_push_front(const KParams& P, long long off, InstHot& h,
                                              const Rec& r) {
  if (lane_id() == 0) {
    P.ov_emit[off + r.req] = r.emit;
    P.ov_prev[off + r.req] = kNil;
    P.ov_next[off + r.req] = h.o_cnt ? (uint32_t)h.o_head : kNil;
    if (h.o_cnt) P.ov_prev[off + h.o_head] = (uint32_t)r.req;
  }
  if (h.o_cnt == 0) h.o_tail = r.req;
  h.o_head = r.req;
  h.o_cnt++;
}

// Full record of a request held in the overflow list (lane 0 loads).
__device__ __forceinline__ Rec ov_record(const KParams& P, long long off, int req) {
  int v[4] = {0, 0, 0, 0};
  if (lane_id() == 0) {
    v[0] = P.prompt[off + req];
    v[1] = P.decode[off + req];
    v[2] = P.ub[P.bucket[off + req]];
    v[3] = P.ov_emit[off + req];
  }
  Rec r;
  r.req = req;
  r.prompt = __shfl_sync(kFull, v[0], 0);
  r.tru = __shfl_sync(kFull, v[1], 0);
  r.dhat = __shfl_sync(kFull, v[2], 0);
  r.emit = __shfl_sync(kFull, v[3], 0);
  return r;
}

__device__ __forceinline__ void ov_unlink(const KParams& P, long long off, InstHot& h, int req) {
  uint32_t nx = 0, pv = 0;
  if (lane_id() == 0) {
    nx = P.ov_next[off + req];
    pv = P.ov_prev[off + req];
  }
  nx = __shfl_sync(kFull, nx, 0);
  pv = __shfl_sync(kFull, pv, 0);
  if (lane_id() == 0) {
    if (pv != kNil) P.ov_next[off + pv] = nx;
    if (nx != kNil) P.ov_prev[off + nx] = pv;
  }
  if (pv == kNil) h.o_head = (int)nx;
  if (nx == kNil) h.o_tail = (int)pv;
  h.o_cnt--;
  __syncwarp();
}

// Move the overflow head into the ring tail (keeps queue order).
__device__ __forceinline__ void ring_refill(const KParams& P, const Grp& G, long long off,
                                            int i, InstHot& h) {
  if (h.o_cnt == 0 || h.w_cnt >= P.wcap) return;
  const int req = h.o_head;
  Rec r = ov_record(P, off, req);
  ov_unlink(P, off, h, req);
  int slot = h.w_head + h.w_cnt;
  if (slot >= P.wcap) slot -= P.wcap;
  ring_write(G, i * P.wcap, slot, r);
  h.w_cnt++;
}

__device__ __forceinline__ void wait_push_back(const KParams& P, const Grp& G, long long off,
                                               int i, InstHot& h, const Rec& r) {
  if (h.o_cnt == 0 && h.w_cnt < P.wcap) {
    int slot = h.w_head + h.w_cnt;
    if (slot >= P.wcap) slot -= P.wcap;
    ring_write(G, i * P.wcap, slot, r);
    h.w_cnt++;
  } else {
    ov_push_back(P, off, h, r);
    __syncwarp();
  }
  wait_add(h, r, +1);
}

__device__ __forceinline__ void wait_push_front(const KParams& P, const Grp& G, long long off,
                                                int i, InstHot& h, const Rec& r) {
  const int base = i * P.wcap;
  if (h.w_cnt == P.wcap) {  // spill the ring's back element to the overflow front
    int slot = h.w_head + h.w_cnt - 1;
    if (slot >= P.wcap) slot -= P.wcap;
    Rec back = ring_read(G, base, slot);
    ov_push_front(P, off, h, back);
    __syncwarp();
    h.w_cnt--;
  }
  h.w_head = h.w_head == 0 ? P.wcap - 1 : h.w_head - 1;
  ring_write(G, base, h.w_head, r);
  h.w_cnt++;
  wait_add(h, r, +1);
}

// Remove queue position `pos` (< w_cnt) from the ring, order kept.
__device__ inline void ring_erase(const KParams& P, const Grp& G, long long off, int i,
                                  InstHot& h, int pos) {
  const int base = i * P.wcap;
  const int l = lane_id();
  Rec tmp[4];
  // read entries pos+1 .. w_cnt-1 into registers, then write them one slot
  // toward the head
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int q = pos + 1 + l + 32 * k;
    if (q < h.w_cnt) {
      int s = h.w_head + q;
      if (s >= P.wcap) s -= P.wcap;
      tmp[k] = ring_read(G, base, s);
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int q = pos + 1 + l + 32 * k;
    if (q < h.w_cnt) {
      int s = h.w_head + q - 1;
      if (s >= P.wcap) s -= P.wcap;
      G.w_req[base + s] = tmp[k].req;
      G.w_prompt[base + s] = tmp[k].prompt;
      G.w_dhat[base + s] = tmp[k].dhat;
      G.w_true[base + s] = tmp[k].tru;
      G.w_emit[base + s] = tmp[k].emit;
    }
  }
  __syncwarp();
  h.w_cnt--;
  ring_refill(P, G, off, i, h);
}

// ------------------------------------------------------------ running

__device__ __forceinline__ void run_append(const KParams& P, const Grp& G, int i, InstHot& h,
                                           const Rec& r) {
  const int idx = i * P.rcap + h.n_run;
  if (lane_id() == 0) {
    G.r_req[idx] = r.req;
    G.r_prompt[idx] = r.prompt;
    G.r_prem[idx] = r.prompt;  // full prompt recompute, instance.hpp:190
    G.r_emit[idx] = r.emit;
    G.r_true[idx] = r.tru;
    G.r_dhat[idx] = r.dhat;
  }
  h.n_run++;
  h.n_prefill++;
  h.res_run += reserved_of(r.prompt, r.dhat, r.emit);
  h.kv_run += r.emit;
  h.pend_run += r.prompt;
  const int dl = r.dhat - r.emit > 0 ? r.dhat - r.emit : 0;
  h.dleft_run += dl;
  h.tleft_run += r.tru - r.emit;
  h.tok_run += r.prompt + r.emit;
  h.min_dleft = dl < h.min_dleft ? dl : h.min_dleft;
}

// Instance::admit_waiting (instance.hpp:149-195).
__device__ inline void admit(const KParams& P, const Grp& G, long long off, int i, InstHot& h) {
  const int base = i * P.wcap;
  const int l = lane_id();
  while (h.w_cnt > 0 && h.n_run < P.max_batch) {
    if (P.batching == RS_BATCHING_FCFS) {  // strict head of line
      Rec r = ring_read(G, base, h.w_head);
      if (h.res_run + reserved_of(r.prompt, r.dhat, r.emit) > P.kv_cap) break;
      h.w_head = h.w_head + 1 == P.wcap ? 0 : h.w_head + 1;
      h.w_cnt--;
      wait_add(h, r, -1);
      run_append(P, G, i, h, r);
      ring_refill(P, G, off, i, h);
      continue;
    }
    // BinPacking: largest reservation that fits (first on ties);
    // LeastWorkLeft: smallest decode_left that fits (first on ties).
    const bool bp = P.batching == RS_BATCHING_BIN_PACKING;
    unsigned long long best = ~0ull;  // (key << 32) | position, min wins
    for (int q0 = 0; q0 < h.w_cnt; q0 += kWarp) {
      const int q = q0 + l;
      unsigned long long k = ~0ull;
      if (q < h.w_cnt) {
        int s = h.w_head + q;
        if (s >= P.wcap) s -= P.wcap;
        Rec r = ring_read(G, base, s);
        const int need = reserved_of(r.prompt, r.dhat, r.emit);
        if (h.res_run + need <= P.kv_cap) {
          const int dl = r.dhat - r.emit > 0 ? r.dhat - r.emit : 0;
          const unsigned key = bp ? (unsigned)(0x7fffffff - need) : (unsigned)dl;
          k = ((unsigned long long)key << 32) | (unsigned)q;
        }
      }
      k = warp_min_u64(k);
      best = k < best ? k : best;
    }
    int pick = best == ~0ull ? -1 : (int)(best & 0xffffffffu);
    unsigned best_key = (unsigned)(best >> 32);
    int pick_req = -1;
    Rec pr;
    // overflow part (queue positions >= w_cnt), walked serially
    if (h.o_cnt > 0) {
      int cur = h.o_head;
      for (int q = 0; q < h.o_cnt; ++q) {
        Rec r = ov_record(P, off, cur);
        const int need = reserved_of(r.prompt, r.dhat, r.emit);
        if (h.res_run + need <= P.kv_cap) {
          const int dl = r.dhat - r.emit > 0 ? r.dhat - r.emit : 0;
          const unsigned key = bp ? (unsigned)(0x7fffffff - need) : (unsigned)dl;
          if (pick < 0 || key < best_key) {  // strictly better only
            best_key = key;
            pick = h.w_cnt + q;
            pick_req = cur;
            pr = r;
          }
        }
        uint32_t nx = 0;
        if (l == 0) nx = P.ov_next[off + cur];
        cur = (int)__shfl_sync(kFull, nx, 0);
      }
    }
    if (pick < 0) break;
    if (pick < h.w_cnt) {
      int s = h.w_head + pick;
      if (s >= P.wcap) s -= P.wcap;
      pr = ring_read(G, base, s);
      ring_erase(P, G, off, i, h, pick);
    } else {
      ov_unlink(P, off, h, pick_req);
    }
    wait_add(h, pr, -1);
    run_append(P, G, i, h, pr);
  }
  __syncwarp();
}

// Recompute every running aggregate from shared memory (after preemption).
template <bool NEED_DBC>
__device__ inline void running_aggregates(const KParams& P, const Grp& G, int i, InstHot& h) {
  const int base = i * P.rcap;
  const int l = lane_id();
  int res = 0, kv = 0, pend = 0, npf = 0, dl = 0, tl = 0, tok = 0, mn = 0x7fffffff;
  int cnt[RS_MAX_BUCKETS];
#pragma unroll
  for (int b = 0; b < RS_MAX_BUCKETS; ++b) cnt[b] = 0;
  for (int j = l; j < h.n_run; j += kWarp) {
    const int pr = G.r_prompt[base + j], pm = G.r_prem[base + j], em = G.r_emit[base + j];
    const int tr = G.r_true[base + j], dh = G.r_dhat[base + j];
    res += reserved_of(pr, dh, em);
    kv += pr - pm + em;
    pend += pm;
    npf += pm > 0;
    const int d = dh - em > 0 ? dh - em : 0;
    dl += d;
    tl += tr - em;
    tok += pr + em;
    mn = d < mn ? d : mn;
    if (NEED_DBC && pm <= 0) cnt[bucket_of(P.state_edges, P.n_state_edges, d)]++;
  }
  h.res_run = warp_sum(res);
  h.kv_run = warp_sum(kv);
  h.pend_run = warp_sum(pend);
  h.n_prefill = warp_sum(npf);
  h.dleft_run = warp_sum(dl);
  h.tleft_run = warp_sum(tl);
  h.tok_run = warp_sum(tok);
  h.min_dleft = warp_min(mn);
  if (NEED_DBC) {
#pragma unroll
    for (int b = 0; b < RS_MAX_BUCKETS; ++b) {
      const int c = warp_sum(cnt[b]);
      if (l == b) G.dbc[i * RS_MAX_BUCKETS + b] = c;
    }
    __syncwarp();
  }
}

// Instance::step (instance.hpp:203-277) + preempt_if_needed (282-299).
// Returns the number of completions, or -1 when nothing is admissible;
// adds the iteration's IterationOutcome::tokens_emitted to `tokens`.
template <bool NEED_DBC>
__device__ inline int inst_step(const KParams& P, const Grp& G, long long off, int i,
                                InstHot& h, int& tokens) {
  const int l = lane_id();
  if (h.w_cnt > 0 && h.n_run < P.max_batch) admit(P, G, off, i, h);
  if (h.n_run == 0) return -1;  // logic_error, instance.hpp:209-211
  const int base = i * P.rcap;
  const int n = h.n_run;

  int e_req[kMaxRunChunks], e_pr[kMaxRunChunks], e_pm[kMaxRunChunks], e_em[kMaxRunChunks],
      e_tr[kMaxRunChunks], e_dh[kMaxRunChunks];
  bool emits[kMaxRunChunks];
#pragma unroll
  for (int k = 0; k < kMaxRunChunks; ++k) {
    const int j = k * kWarp + l;
    const bool v = j < n;
    e_req[k] = v ? G.r_req[base + j] : 0;
    e_pr[k] = v ? G.r_prompt[base + j] : 0;
    e_pm[k] = v ? G.r_prem[base + j] : 0;
    e_em[k] = v ? G.r_emit[base + j] : 0;
    e_tr[k] = v ? G.r_true[base + j] : 0x7fffffff;
    e_dh[k] = v ? G.r_dhat[base + j] : 0;
    emits[k] = false;
  }

  double elapsed;
  const bool prefill = h.n_prefill > 0;
  if (prefill) {
    const int kv_before = h.kv_run;
    int processed;
    if (P.chunk <= 0) {  // whole prompts, co-running decodes stall
      processed = h.pend_run;
#pragma unroll
      for (int k = 0; k < kMaxRunChunks; ++k) e_pm[k] = 0;
    } else {  // chunked prefill: take_i = min(B, P_i) - min(B, P_{i-1})
      const int budget = P.chunk;
      int carry = 0;
#pragma unroll
      for (int k = 0; k < kMaxRunChunks; ++k) {
        if (k * kWarp < n) {
          const bool v = k * kWarp + l < n;
          const int x = v ? e_pm[k] : 0;
          const int incl = warp_incl_scan(x, l) + carry;
          const int excl = incl - x;
          const int take = min(budget, incl) - min(budget, excl);
          emits[k] = v && x == 0;  // co-decoders
          tokens += __popc(__ballot_sync(kFull, emits[k]));
          e_pm[k] = x - take;
          carry = __shfl_sync(kFull, incl, kWarp - 1);
        }
      }
      processed = min(budget, carry);
    }
    // prompt_batch_time (latency.hpp:68-74), reference operand order
    elapsed = __dadd_rn(__dadd_rn(P.intercept, __dmul_rn(P.tpp, (double)processed)),
                        __dmul_rn(P.dpt, (double)kv_before));
  } else {
    // decode_batch_time with the running count (instance.hpp:244-245)
    elapsed = __dadd_rn(P.dtb, __dmul_rn(P.dpt, (double)n));
    tokens += n;
#pragma unroll
    for (int k = 0; k < kMaxRunChunks; ++k) emits[k] = k * kWarp + l < n;
  }
  h.clock = __dadd_rn(h.clock, elapsed);

  // emission, first tokens, completions (instance.hpp:254-273)
  bool done[kMaxRunChunks];
  int ncomp = 0;
#pragma unroll
  for (int k = 0; k < kMaxRunChunks; ++k) {
    done[k] = false;
    if (emits[k]) {
      e_em[k] += 1;
      if (e_em[k] == 1) P.o_first[off + e_req[k]] = h.clock;
      if (e_em[k] >= e_tr[k]) {
        done[k] = true;
        P.o_completion[off + e_req[k]] = h.clock;
      }
    }
    if (k * kWarp < n) ncomp += __popc(__ballot_sync(kFull, done[k]));
  }

  // write back: compaction keeps running order
  int npos = 0;
  int res = 0, kv = 0, pend = 0, npf = 0, dl = 0, tl = 0, tok = 0, mn = 0x7fffffff;
  int cnt[RS_MAX_BUCKETS];
#pragma unroll
  for (int b = 0; b < RS_MAX_BUCKETS; ++b) cnt[b] = 0;
#pragma unroll
  for (int k = 0; k < kMaxRunChunks; ++k) {
    if (k * kWarp < n) {
      const bool v = k * kWarp + l < n;
      const bool keep = v && !done[k];
      if (ncomp) {
        const unsigned km = __ballot_sync(kFull, keep);
        const int pos = npos + __popc(km & lanemask_lt());
        if (keep) {
          const int d = base + pos;
          G.r_req[d] = e_req[k];
          G.r_prompt[d] = e_pr[k];
          G.r_prem[d] = e_pm[k];
          G.r_emit[d] = e_em[k];
          G.r_true[d] = e_tr[k];
          G.r_dhat[d] = e_dh[k];
        }
        npos += __popc(km);
      } else if (v) {
        G.r_emit[base + k * kWarp + l] = e_em[k];
        if (prefill) G.r_prem[base + k * kWarp + l] = e_pm[k];
      }
      if (keep) {
        res += reserved_of(e_pr[k], e_dh[k], e_em[k]);
        kv += e_pr[k] - e_pm[k] + e_em[k];
        pend += e_pm[k];
        npf += e_pm[k] > 0;
        const int d = e_dh[k] - e_em[k] > 0 ? e_dh[k] - e_em[k] : 0;
        dl += d;
        tl += e_tr[k] - e_em[k];
        tok += e_pr[k] + e_em[k];
        mn = d < mn ? d : mn;
        if (NEED_DBC && e_pm[k] <= 0) cnt[bucket_of(P.state_edges, P.n_state_edges, d)]++;
      }
    }
  }
  h.n_run = n - ncomp;
  h.res_run = warp_sum(res);
  h.kv_run = warp_sum(kv);
  h.pend_run = warp_sum(pend);
  h.n_prefill = warp_sum(npf);
  h.dleft_run = warp_sum(dl);
  h.tleft_run = warp_sum(tl);
  h.tok_run = warp_sum(tok);
  h.min_dleft = warp_min(mn);
  if (NEED_DBC) {
#pragma unroll
    for (int b = 0; b < RS_MAX_BUCKETS; ++b) {
      const int c = warp_sum(cnt[b]);
      if (l == b) G.dbc[i * RS_MAX_BUCKETS + b] = c;
    }
  }
  __syncwarp();

  // preempt_if_needed: evict the newest admission (running is sorted by
  // admit_seq, so the back) while KV overflows, front of the waiting queue.
  if (h.kv_run > P.kv_cap && h.n_run > 1) {
    while (h.kv_run > P.kv_cap && h.n_run > 1) {
      const int v = base + h.n_run - 1;
      Rec r;
      r.req = G.r_req[v];
      r.prompt = G.r_prompt[v];
      r.dhat = G.r_dhat[v];
      r.tru = G.r_true[v];
      r.emit = G.r_emit[v];
      const int pm = G.r_prem[v];
      h.kv_run -= r.prompt - pm + r.emit;
      h.n_run--;
      if (l == 0) P.o_preempt[off + r.req] += 1;
      wait_push_front(P, G, off, i, h, r);
    }
    running_aggregates<NEED_DBC>(P, G, i, h);
  }
  return ncomp;
}

}  // namespace rs
