// fast.cuh — the fast replay kernel for whole-prompt prefill (chunk_size
// off, the reference default): lane = instance, warp = replay.
//
// Why it is exact.  Without chunking, a step that admits anything is a
// prefill step that consumes EVERY pending prompt token and emits nothing
// (instance.hpp:219-242), and every other step is a decode step in which
// EVERY running request emits one token (instance.hpp:243-249).  So the
// tokens a running request has emitted are
//     emitted = emitted_at_admission + (decode steps since admission)
//             = D + key,   key = emitted_at_admission - D_at_admission,
// with D the instance's decode-step counter.  A decode step is then O(1):
// clock += dtb + dpt*n, D += 1, and the aggregates move by closed forms
// (kv += n, true-left -= n, token mass += n, reservations += #overrun,
// decode-left -= n - #overrun).  Per-entry work happens only at EVENTS:
//   * the first decode step after admission  -> first-token stores (lane),
//   * D == min(true - key)                    -> completions (warp scan),
//   * D == min(dhat - key) (emitted reaches the estimate) -> warp re-count,
//   * KV overflow                             -> preemption (lane).
// Each lane owns one instance (<= 32 per group, G groups per lane), so all
// instances of a replay advance in parallel.  A replay that raises "nothing
// admissible" is re-run with instances stepped one at a time in index order,
// reproducing exactly where the reference's exception stops a tick.
//
// Shared memory is addressed as one int array from a single per-warp word
// base (`gw`, laundered so the compiler keeps it in a register) plus the
// per-field word offsets of KParams (constant bank), and the lane id is
// likewise computed once: no pointer structs to rematerialize with S2R.
#pragma once

#include "router.cuh"

namespace rs {

extern __shared__ __align__(16) int rs_smw[];

constexpr int kFresh = 0x40000000;  // entry awaits its first token
constexpr int kReqMask = 0x3fffffff;
constexpr int kBig = 0x7fffffff;

struct Inst {  // one instance, held in its lane's registers
  double clock;
  double dec_el;  // decode_batch_time for el_n running (cached)
  int el_n;
  int D, n, npf, ft;
  // kv = sum prompt-done + emitted, pend = unprefilled prompt, dleft = sum
  // max(d_hat - emitted, 0), tleft = sum true - emitted over running.  The
  // reservation sum and token mass follow (instance.hpp:365-368): per entry
  // reserved = prompt + max(d_hat, emitted) = (prompt + emitted) + max(d_hat
  // - emitted, 0), so res = kv + pend + dleft and tok = kv + pend (res_run /
  // tok_run); neither is stored.
  int kv, pend, dleft, tleft, nge, next_ge, next_done;
  int w_head, w_cnt, o_cnt, o_head, o_tail;
  int comps;
  // waiting-queue aggregates: a queue can hold every request of the replay,
  // so these grow with the trace length (64-bit; updated only on enqueue,
  // admission and preemption).  The running ones are bounded by the batch.
  // (reserved over waiting = tokw + dlw, as for running)
  long long pendw, dlw, tlw, tokw;
  // RL state encoding (encode_state, env.hpp:88-113) with the default state
  // scheme {0, e1, e2}: running entries with decode_left >= e1 / >= e2, and
  // the decode-step count D at which the next of them drops below e1 / e2
  // (decode_left falls by one per decode step).  Exact between events.
  int sb1, sb2, nx1, nx2;
  int ev_at;  // min(next_done, next_ge): the decode step of the next scan event
};

// Running entry fields (admission order): request id | fresh bit, prompt,
// d_hat, true decode, key.  Entry j < rsm of instance i in the group's
// shared memory (odd per-instance stride: lane-owned rows hit distinct
// banks); entries j >= rsm in the warp's global tail.  T = 0: the launch
// has no tail (rsm = rcap) and every access is a shared-memory one; T = 1:
// tail accesses inline (fleets whose batches often outgrow the head: c5's
// heavy-decode m = 64); T = 2: tail accesses out of line (rare path, no
// register cost in the tick loop).
enum RunField { kFQ = 0, kFP = 1, kFD = 2, kFT = 3, kFK = 4 };

template <int F>
__device__ __forceinline__ int run_word(const KParams& P) {
  return F == kFQ ? P.f_rreq : F == kFP ? P.f_rprompt : F == kFD ? P.f_rdhat
       : F == kFT ? P.f_rtrue : P.f_rkey;
}
// The global tail, out of line: the rare path must not hold registers (or
// hoisted address arithmetic) in the tick loop.
static __device__ __noinline__ int* run_tail_ptr(const KParams& P, int f, int i, int j) {
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  return P.run_tail + ((gwarp * 5 + f) * P.m + i) * P.rtail + (j - P.rsm);
}
template <int F>
__device__ __forceinline__ int* run_tail_at(const KParams& P, int i, int j) {
  return run_tail_ptr(P, F, i, j);
}
static __device__ __noinline__ void run_tail_put5(const KParams& P, int i, int j, int q, int pr, int dh,
                                           int tr, int ky) {
  int* p = run_tail_ptr(P, 0, i, j);
  const long long fs = (long long)P.m * P.rtail;  // field stride
  p[0] = q;
  p[fs] = pr;
  p[2 * fs] = dh;
  p[3 * fs] = tr;
  p[4 * fs] = ky;
}
struct Ent5 {
  int q, pr, dh, tr, ky;
};
static __device__ __noinline__ Ent5 run_tail_get5(const KParams& P, int i, int j) {
  const int* p = run_tail_ptr(P, 0, i, j);
  const long long fs = (long long)P.m * P.rtail;
  return Ent5{p[0], p[fs], p[2 * fs], p[3 * fs], p[4 * fs]};
}
__device__ __forceinline__ int* run_tail_inl(const KParams& P, int f, int i, int j) {
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  return P.run_tail + ((gwarp * 5 + f) * P.m + i) * P.rtail + (j - P.rsm);
}
template <int F, int T>
__device__ __forceinline__ int rget(const KParams& P, int gw, int i, int j) {
  if (T == 0 || j < P.rsm) return rs_smw[gw + run_word<F>(P) + i * P.rstride + j];
  return T == 1 ? *run_tail_inl(P, F, i, j) : *run_tail_at<F>(P, i, j);
}
// all five fields of entry j
template <int T>
__device__ __forceinline__ void rput5(const KParams& P, int gw, int i, int j, int q, int pr,
                                      int dh, int tr, int ky) {
  if (T == 0 || j < P.rsm) {
    const int b = gw + i * P.rstride + j;
    rs_smw[b + P.f_rreq] = q;
    rs_smw[b + P.f_rprompt] = pr;
    rs_smw[b + P.f_rdhat] = dh;
    rs_smw[b + P.f_rtrue] = tr;
    rs_smw[b + P.f_rkey] = ky;
  } else if (T == 1) {
    int* p = run_tail_inl(P, 0, i, j);
    const long long fs = (long long)P.m * P.rtail;  // field stride
    p[0] = q;
    p[fs] = pr;
    p[2 * fs] = dh;
    p[3 * fs] = tr;
    p[4 * fs] = ky;
  } else {
    run_tail_put5(P, i, j, q, pr, dh, tr, ky);
  }
}
template <int T>
__device__ __forceinline__ void rget5(const KParams& P, int gw, int i, int j, int& q, int& pr,
                                      int& dh, int& tr, int& ky) {
  if (T == 0 || j < P.rsm) {
    const int b = gw + i * P.rstride + j;
    q = rs_smw[b + P.f_rreq];
    pr = rs_smw[b + P.f_rprompt];
    dh = rs_smw[b + P.f_rdhat];
    tr = rs_smw[b + P.f_rtrue];
    ky = rs_smw[b + P.f_rkey];
  } else if (T == 1) {
    const int* p = run_tail_inl(P, 0, i, j);
    const long long fs = (long long)P.m * P.rtail;
    q = p[0];
    pr = p[fs];
    dh = p[2 * fs];
    tr = p[3 * fs];
    ky = p[4 * fs];
  } else {
    const Ent5 e = run_tail_get5(P, i, j);
    q = e.q;
    pr = e.pr;
    dh = e.dh;
    tr = e.tr;
    ky = e.ky;
  }
}
__device__ __forceinline__ int& WQ(const KParams& P, int gw, int i, int s) {
  return rs_smw[gw + P.f_wreq + i * P.wcap + s];
}
__device__ __forceinline__ int& WP(const KParams& P, int gw, int i, int s) {
  return rs_smw[gw + P.f_wprompt + i * P.wcap + s];
}
__device__ __forceinline__ int& WD(const KParams& P, int gw, int i, int s) {
  return rs_smw[gw + P.f_wdhat + i * P.wcap + s];
}
__device__ __forceinline__ int& WT(const KParams& P, int gw, int i, int s) {
  return rs_smw[gw + P.f_wtrue + i * P.wcap + s];
}
__device__ __forceinline__ int& WE(const KParams& P, int gw, int i, int s) {
  return rs_smw[gw + P.f_wemit + i * P.wcap + s];
}

__device__ __forceinline__ void inst_init(Inst& I) {
  I.clock = 0.0;
  I.dec_el = 0.0;
  I.el_n = -1;
  I.D = I.n = I.npf = I.ft = 0;
  I.kv = I.pend = I.dleft = I.tleft = I.nge = 0;
  I.next_ge = I.next_done = kBig;
  I.w_head = I.w_cnt = I.o_cnt = 0;
  I.o_head = I.o_tail = (int)kNil;
  I.comps = 0;
  I.pendw = I.dlw = I.tlw = I.tokw = 0;
  I.sb1 = I.sb2 = 0;
  I.nx1 = I.nx2 = kBig;
  I.ev_at = kBig;
}

__device__ __forceinline__ int res_run(const Inst& I) { return I.kv + I.pend + I.dleft; }
__device__ __forceinline__ int tok_run(const Inst& I) { return I.kv + I.pend; }

// state-bucket tracking of one running entry with decode_left dl at step D
__device__ __forceinline__ void sb_add(const KParams& P, Inst& I, int dl) {
  const int e1 = P.state_edges[1], e2 = P.state_edges[2];
  if (dl >= e1) {
    I.sb1++;
    I.nx1 = min(I.nx1, I.D + dl - e1 + 1);
  }
  if (dl >= e2) {
    I.sb2++;
    I.nx2 = min(I.nx2, I.D + dl - e2 + 1);
  }
}

__device__ __forceinline__ void waitagg(Inst& I, int prompt, int dhat, int tru, int emit, int s) {
  I.pendw += (long long)(s * prompt);
  I.dlw += (long long)(s * (dhat > emit ? dhat - emit : 0));
  I.tlw += (long long)(s * (tru > emit ? tru - emit : 0));
  I.tokw += (long long)(s * (prompt + emit));
}

// ---- per-lane waiting queue (shared ring + global overflow list) --------

__device__ __forceinline__ void lane_ov_push_back(const KParams& P, long long off, Inst& I,
                                                  int req, int emit) {
  P.ov_emit[off + req] = emit;
  P.ov_next[off + req] = kNil;
  P.ov_prev[off + req] = I.o_cnt ? (uint32_t)I.o_tail : kNil;
  if (I.o_cnt) P.ov_next[off + I.o_tail] = (uint32_t)req;
  else I.o_head = req;
  I.o_tail = req;
  I.o_cnt++;
}

__device__ __forceinline__ void lane_ov_push_front(const KParams& P, long long off, Inst& I,
                                                   int req, int emit) {
  P.ov_emit[off + req] = emit;
  P.ov_prev[off + req] = kNil;
  P.ov_next[off + req] = I.o_cnt ? (uint32_t)I.o_head : kNil;
  if (I.o_cnt) P.ov_prev[off + I.o_head] = (uint32_t)req;
  else I.o_tail = req;
  I.o_head = req;
  I.o_cnt++;
}

__device__ __forceinline__ void lane_ov_unlink(const KParams& P, long long off, Inst& I, int req) {
  const uint32_t nx = P.ov_next[off + req], pv = P.ov_prev[off + req];
  if (pv != kNil) P.ov_next[off + pv] = nx;
  else I.o_head = (int)nx;
  if (nx != kNil) P.ov_prev[off + nx] = pv;
  else I.o_tail = (int)pv;
  I.o_cnt--;
}

__device__ __forceinline__ void ring_put(const KParams& P, int gw, int i, int s, int req, int prompt,
                                         int dhat, int tru, int emit) {
  WQ(P, gw, i, s) = req;
  WP(P, gw, i, s) = prompt;
  WD(P, gw, i, s) = dhat;
  WT(P, gw, i, s) = tru;
  WE(P, gw, i, s) = emit;
}

__device__ __forceinline__ void lane_refill(const KParams& P, int gw, long long off, int i, Inst& I) {
  if (I.o_cnt == 0 || I.w_cnt >= P.wcap) return;
  const int req = I.o_head;
  const int prompt = P.prompt[off + req], tru = P.decode[off + req];
  const int dhat = P.ub[P.bucket[off + req]], emit = P.ov_emit[off + req];
  lane_ov_unlink(P, off, I, req);
  int s = I.w_head + I.w_cnt;
  if (s >= P.wcap) s -= P.wcap;
  ring_put(P, gw, i, s, req, prompt, dhat, tru, emit);
  I.w_cnt++;
}

// Instance::enqueue (instance.hpp:113-130) by the owning lane.
__device__ __forceinline__ void lane_enqueue(const KParams& P, int gw, long long off, int i, Inst& I,
                                             const Rec& r, double now) {
  if (I.clock < now) I.clock = now;
  if (I.o_cnt == 0 && I.w_cnt < P.wcap) {
    int s = I.w_head + I.w_cnt;
    if (s >= P.wcap) s -= P.wcap;
    ring_put(P, gw, i, s, r.req, r.prompt, r.dhat, r.tru, 0);
    I.w_cnt++;
  } else {
    lane_ov_push_back(P, off, I, r.req, 0);
  }
  waitagg(I, r.prompt, r.dhat, r.tru, 0, +1);
}

__device__ __forceinline__ void lane_push_front(const KParams& P, int gw, long long off, int i,
                                                Inst& I, int req, int prompt, int dhat, int tru,
                                                int emit) {
  if (I.w_cnt == P.wcap) {  // spill the ring's back element to the overflow front
    int s = I.w_head + I.w_cnt - 1;
    if (s >= P.wcap) s -= P.wcap;
    lane_ov_push_front(P, off, I, WQ(P, gw, i, s), WE(P, gw, i, s));
    I.w_cnt--;
  }
  I.w_head = I.w_head == 0 ? P.wcap - 1 : I.w_head - 1;
  ring_put(P, gw, i, I.w_head, req, prompt, dhat, tru, emit);
  I.w_cnt++;
  waitagg(I, prompt, dhat, tru, emit, +1);
}

// Append an admitted request to the running batch (instance.hpp:187-192).
template <int T>
__device__ __forceinline__ void lane_admit_one(const KParams& P, int gw, int i, Inst& I, int req,
                                               int prompt, int dhat, int tru, int emit) {
  rput5<T>(P, gw, i, I.n, req | (emit == 0 ? kFresh : 0), prompt, dhat, tru, emit - I.D);
  I.n++;
  I.npf++;
  I.pend += prompt;
  I.kv += emit;
  I.dleft += dhat > emit ? dhat - emit : 0;
  I.tleft += tru - emit;
  const int ge_at = dhat - emit + I.D;
  if (ge_at <= I.D) I.nge++;
  else I.next_ge = ge_at < I.next_ge ? ge_at : I.next_ge;
  const int done_at = tru - emit + I.D;
  I.next_done = done_at < I.next_done ? done_at : I.next_done;
  sb_add(P, I, dhat - emit);
  I.ev_at = min(I.next_done, I.next_ge);
  waitagg(I, prompt, dhat, tru, emit, -1);
}

// Instance::admit_waiting (instance.hpp:149-195) by the owning lane.
template <int T>
__device__ __forceinline__ void lane_admit(const KParams& P, int gw, long long off, int i, Inst& I) {
  while (I.w_cnt > 0 && I.n < P.max_batch) {
    if (P.batching == RS_BATCHING_FCFS) {  // strict head of line
      const int s = I.w_head;
      const int prompt = WP(P, gw, i, s), dhat = WD(P, gw, i, s), emit = WE(P, gw, i, s);
      if (res_run(I) + reserved_of(prompt, dhat, emit) > P.kv_cap) break;
      const int req = WQ(P, gw, i, s), tru = WT(P, gw, i, s);
      I.w_head = s + 1 == P.wcap ? 0 : s + 1;
      I.w_cnt--;
      lane_admit_one<T>(P, gw, i, I, req, prompt, dhat, tru, emit);
      lane_refill(P, gw, off, i, I);
      continue;
    }
    // BinPacking (largest reservation that fits, first wins) or
    // LeastWorkLeft (smallest decode_left that fits, first wins).
    const bool bp = P.batching == RS_BATCHING_BIN_PACKING;
    bool found = false;
    int bkey = 0, pos = -1, preq = -1;
    for (int q = 0; q < I.w_cnt; ++q) {
      int s = I.w_head + q;
      if (s >= P.wcap) s -= P.wcap;
      const int prompt = WP(P, gw, i, s), dhat = WD(P, gw, i, s), emit = WE(P, gw, i, s);
      const int need = reserved_of(prompt, dhat, emit);
      if (res_run(I) + need > P.kv_cap) continue;
      const int key = bp ? -need : (dhat > emit ? dhat - emit : 0);
      if (!found || key < bkey) { found = true; bkey = key; pos = q; }
    }
    int cur = I.o_head;
    for (int q = 0; q < I.o_cnt; ++q) {
      const int prompt = P.prompt[off + cur], emit = P.ov_emit[off + cur];
      const int dhat = P.ub[P.bucket[off + cur]];
      const int need = reserved_of(prompt, dhat, emit);
      if (res_run(I) + need <= P.kv_cap) {
        const int key = bp ? -need : (dhat > emit ? dhat - emit : 0);
        if (!found || key < bkey) { found = true; bkey = key; pos = I.w_cnt + q; preq = cur; }
      }
      cur = (int)P.ov_next[off + cur];
    }
    if (!found) break;
    if (pos < I.w_cnt) {
      int s = I.w_head + pos;
      if (s >= P.wcap) s -= P.wcap;
      const int req = WQ(P, gw, i, s), prompt = WP(P, gw, i, s), dhat = WD(P, gw, i, s),
                tru = WT(P, gw, i, s), emit = WE(P, gw, i, s);
      for (int q = pos; q + 1 < I.w_cnt; ++q) {  // erase, order kept
        int s0 = I.w_head + q, s1 = s0 + 1;
        if (s0 >= P.wcap) s0 -= P.wcap;
        if (s1 >= P.wcap) s1 -= P.wcap;
        ring_put(P, gw, i, s0, WQ(P, gw, i, s1), WP(P, gw, i, s1), WD(P, gw, i, s1),
                 WT(P, gw, i, s1), WE(P, gw, i, s1));
      }
      I.w_cnt--;
      lane_admit_one<T>(P, gw, i, I, req, prompt, dhat, tru, emit);
      lane_refill(P, gw, off, i, I);
    } else {
      const int prompt = P.prompt[off + preq], tru = P.decode[off + preq];
      const int dhat = P.ub[P.bucket[off + preq]], emit = P.ov_emit[off + preq];
      lane_ov_unlink(P, off, I, preq);
      lane_admit_one<T>(P, gw, i, I, preq, prompt, dhat, tru, emit);
    }
  }
}

// Group-cooperative rescan of instance i's running batch after a decode
// step: completions (emitted >= true) are stored and compacted away, then
// every aggregate is recomputed exactly.  `owner` lane holds the instance.
// A whole warp keeps its <= 4 entries per lane in registers; a narrower
// group streams the batch in W-entry chunks, compacting as it goes (an
// entry only ever moves down, onto a slot already read).
// SB: also recount the RL state-bucket tracking (Inst::sb1..nx2).
template <int W, bool SB, int T>
__device__ __forceinline__ void warp_scan_instance(const KParams& P, int gw, long long off, int i,
                                          int owner, Inst& I, const Lanes<W>& L) {
  const int l = L.l;
  if (T) L.sync();  // the owner's global-tail writes before any lane reads them
  const int D = L.shfl(I.D, owner);
  const int n = L.shfl(I.n, owner);
  const double clock = L.shfl(I.clock, owner);
  int kv = 0, dl = 0, tl = 0, nge = 0, nxg = kBig, nxd = kBig;
  int s1 = 0, s2 = 0, x1 = kBig, x2 = kBig;
  int ncomp = 0;
  auto account = [&](int pr, int dh, int tr, int ky) {
    const int em = D + ky;
    kv += pr + em;
    const int d = dh - em;
    dl += d > 0 ? d : 0;
    tl += tr - em;
    if (em >= dh) nge++;
    else nxg = min(nxg, dh - ky);
    nxd = min(nxd, tr - ky);
    if (SB) {
      const int e1 = P.state_edges[1], e2 = P.state_edges[2];
      if (d >= e1) { s1++; x1 = min(x1, D + d - e1 + 1); }
      if (d >= e2) { s2++; x2 = min(x2, D + d - e2 + 1); }
    }
  };
  if (W == kWarp) {
    int rq[kMaxRunChunks], pr[kMaxRunChunks], dh[kMaxRunChunks], tr[kMaxRunChunks],
        ky[kMaxRunChunks];
    bool keep[kMaxRunChunks];
#pragma unroll
    for (int k = 0; k < kMaxRunChunks; ++k) {
      const int j = k * kWarp + l;
      keep[k] = false;
      rq[k] = pr[k] = dh[k] = tr[k] = ky[k] = 0;
      if (k * kWarp < n) {
        bool done = false;
        if (j < n) {
          rget5<T>(P, gw, i, j, rq[k], pr[k], dh[k], tr[k], ky[k]);
          done = D + ky[k] >= tr[k];
          if (done) P.o_completion[off + (rq[k] & kReqMask)] = clock;
          keep[k] = !done;
        }
        ncomp += __popc(L.ballot(done));
      }
    }
    int npos = 0;
#pragma unroll
    for (int k = 0; k < kMaxRunChunks; ++k) {
      if (k * kWarp < n) {
        if (ncomp) {
          const unsigned km = L.ballot(keep[k]);
          if (keep[k]) {
            const int d = npos + __popc(km & L.lt());
            rput5<T>(P, gw, i, d, rq[k], pr[k], dh[k], tr[k], ky[k]);
          }
          npos += __popc(km);
        }
        if (keep[k]) account(pr[k], dh[k], tr[k], ky[k]);
      }
    }
  } else {
    for (int c = 0; c < n; c += W) {
      const int j = c + l;
      int rq = 0, pr = 0, dh = 0, tr = 0, ky = 0;
      bool keep = false;
      if (j < n) {
        rget5<T>(P, gw, i, j, rq, pr, dh, tr, ky);
        const bool done = D + ky >= tr;
        if (done) P.o_completion[off + (rq & kReqMask)] = clock;
        keep = !done;
      }
      const unsigned km = L.ballot(keep);
      const int nv = c + W < n ? W : n - c;  // valid entries in this chunk
      const int before = ncomp;
      ncomp += nv - __popc(km);
      L.sync();  // every lane has read its entry before any slot is rewritten
      if (keep) {
        const int d = c - before + __popc(km & L.lt());
        if (d != j) {
          rput5<T>(P, gw, i, d, rq, pr, dh, tr, ky);
        }
      }
      if (keep) account(pr, dh, tr, ky);
      L.sync();
    }
  }
  kv = L.sum(kv);
  dl = L.sum(dl);
  tl = L.sum(tl);
  nge = L.sum(nge);
  nxg = L.min(nxg);
  nxd = L.min(nxd);
  if (SB) {
    s1 = L.sum(s1);
    s2 = L.sum(s2);
    x1 = L.min(x1);
    x2 = L.min(x2);
  }
  L.sync();
  if (l == owner) {
    if (SB) {
      I.sb1 = s1;
      I.sb2 = s2;
      I.nx1 = x1;
      I.nx2 = x2;
    }
    I.n = n - ncomp;
    I.comps += ncomp;
    I.kv = kv;
    I.pend = 0;
    I.npf = 0;
    I.dleft = dl;
    I.tleft = tl;
    I.nge = nge;
    I.next_ge = nxg;
    I.next_done = nxd;
    I.ft = I.n;  // every survivor has emitted
    I.ev_at = min(nxd, nxg);
  }
}

// Serial (owner lane) recount of every running aggregate after preemption.
// No request can complete here: completions were handled this step.
template <int T>
__device__ __forceinline__ void lane_recount(const KParams& P, int gw, int i, Inst& I) {
  int kv = 0, dl = 0, tl = 0, nge = 0, nxg = kBig, nxd = kBig;
  I.sb1 = I.sb2 = 0;
  I.nx1 = I.nx2 = kBig;
  for (int j = 0; j < I.n; ++j) {
    const int pr = rget<kFP, T>(P, gw, i, j), dh = rget<kFD, T>(P, gw, i, j),
              tr = rget<kFT, T>(P, gw, i, j), ky = rget<kFK, T>(P, gw, i, j);
    const int em = I.D + ky;
    kv += pr + em;
    dl += dh > em ? dh - em : 0;
    tl += tr - em;
    if (em >= dh) nge++;
    else nxg = min(nxg, dh - ky);
    nxd = min(nxd, tr - ky);
    sb_add(P, I, dh - em);
  }
  I.kv = kv;
  I.dleft = dl;
  I.tleft = tl;
  I.nge = nge;
  I.next_ge = nxg;
  I.next_done = nxd;
  I.ev_at = min(nxd, nxg);
}

// preempt_if_needed (instance.hpp:282-299) by the owning lane.  Running is
// in admission order, so the newest admission is last; all prompts are
// prefilled at a step boundary.
template <int T>
__device__ __forceinline__ void lane_preempt(const KParams& P, int gw, long long off, int i,
                                             Inst& I) {
  while (I.kv > P.kv_cap && I.n > 1) {
    const int j = I.n - 1;
    int req, prompt, dhat, tru, key;
    rget5<T>(P, gw, i, j, req, prompt, dhat, tru, key);
    req &= kReqMask;
    const int emit = I.D + key;
    I.kv -= prompt + emit;
    I.n--;
    P.o_preempt[off + req] += 1;
    lane_push_front(P, gw, off, i, I, req, prompt, dhat, tru, emit);
  }
  if (I.ft > I.n) I.ft = I.n;
  lane_recount<T>(P, gw, i, I);
}

}  // namespace rs
