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
//   * the first decode step after admission  -> first-token stores,
//   * D == min(true - key)                    -> completions (scan),
//   * D == min(dhat - key) (emitted reaches the estimate) -> re-count,
//   * KV overflow                             -> preemption.
// Each lane owns one instance (<= 32 per group, G groups per lane), so all
// instances of a replay advance in parallel; events are handled by the whole
// warp.  A replay that raises "nothing admissible" is re-run with
// instances stepped one at a time in index order, reproducing exactly where
// the reference's exception stops a tick.
#pragma once

#include "router.cuh"

namespace rs {

constexpr int kFresh = 0x40000000;       // entry awaits its first token
constexpr int kReqMask = 0x3fffffff;
constexpr int kBig = 0x7fffffff;

struct Inst {  // one instance, held in its lane's registers
  double clock;
  int D, n, npf, ft;
  int res, kv, pend, dleft, tleft, tok, nge, next_ge, next_done;
  int w_head, w_cnt, o_cnt, o_head, o_tail;
  int comps;
  long long resw, pendw, dlw, tlw, tokw;
};

struct FRun {  // running entries, admission order, stride per instance
  int *req, *prompt, *dhat, *tru, *key;
  int stride;
};

struct FastGrp {
  FRun R;
  int *w_req, *w_prompt, *w_dhat, *w_true, *w_emit;
  int wstride;
  double* rlx;
  unsigned long long* rng;
  int* front;
};

__device__ __forceinline__ FastGrp make_fast_grp(const KParams& P, char* base) {
  FastGrp G;
  const int rs_ = P.rcap | 1, ws_ = P.wcap;
  int* run = reinterpret_cast<int*>(base + P.off_run);
  const int mr = P.m * rs_;
  G.R.req = run; G.R.prompt = run + mr; G.R.dhat = run + 2 * mr; G.R.tru = run + 3 * mr;
  G.R.key = run + 4 * mr;
  G.R.stride = rs_;
  int* wt = reinterpret_cast<int*>(base + P.off_wait);
  const int mw = P.m * ws_;
  G.w_req = wt; G.w_prompt = wt + mw; G.w_dhat = wt + 2 * mw; G.w_true = wt + 3 * mw;
  G.w_emit = wt + 4 * mw;
  G.wstride = ws_;
  G.rlx = reinterpret_cast<double*>(base + P.off_rlx);
  G.rng = reinterpret_cast<unsigned long long*>(base + P.off_rng);
  G.front = reinterpret_cast<int*>(base + P.off_front);
  return G;
}

__device__ __forceinline__ void inst_init(Inst& I) {
  I.clock = 0.0;
  I.D = I.n = I.npf = I.ft = 0;
  I.res = I.kv = I.pend = I.dleft = I.tleft = I.tok = I.nge = 0;
  I.next_ge = I.next_done = kBig;
  I.w_head = I.w_cnt = I.o_cnt = 0;
  I.o_head = I.o_tail = (int)kNil;
  I.comps = 0;
  I.resw = I.pendw = I.dlw = I.tlw = I.tokw = 0;
}

__device__ __forceinline__ void waitagg(Inst& I, int prompt, int dhat, int tru, int emit, int s) {
  I.resw += s * reserved_of(prompt, dhat, emit);
  I.pendw += s * prompt;
  I.dlw += s * (dhat > emit ? dhat - emit : 0);
  I.tlw += s * (tru > emit ? tru - emit : 0);
  I.tokw += s * (prompt + emit);
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

__device__ __forceinline__ void lane_ring_put(const FastGrp& G, int i, int slot, int req, int prompt,
                                              int dhat, int tru, int emit) {
  const int b = i * G.wstride + slot;
  G.w_req[b] = req;
  G.w_prompt[b] = prompt;
  G.w_dhat[b] = dhat;
  G.w_true[b] = tru;
  G.w_emit[b] = emit;
}

__device__ __forceinline__ void lane_refill(const KParams& P, const FastGrp& G, long long off, int i,
                                            Inst& I) {
  if (I.o_cnt == 0 || I.w_cnt >= P.wcap) return;
  const int req = I.o_head;
  const int prompt = P.prompt[off + req], tru = P.decode[off + req];
  const int dhat = P.ub[P.bucket[off + req]], emit = P.ov_emit[off + req];
  lane_ov_unlink(P, off, I, req);
  int slot = I.w_head + I.w_cnt;
  if (slot >= P.wcap) slot -= P.wcap;
  lane_ring_put(G, i, slot, req, prompt, dhat, tru, emit);
  I.w_cnt++;
}

// Instance::enqueue (instance.hpp:113-130) by the owning lane.
__device__ __forceinline__ void lane_enqueue(const KParams& P, const FastGrp& G, long long off,
                                             int i, Inst& I, const Rec& r, double now) {
  if (I.clock < now) I.clock = now;
  if (I.o_cnt == 0 && I.w_cnt < P.wcap) {
    int slot = I.w_head + I.w_cnt;
    if (slot >= P.wcap) slot -= P.wcap;
    lane_ring_put(G, i, slot, r.req, r.prompt, r.dhat, r.tru, 0);
    I.w_cnt++;
  } else {
    lane_ov_push_back(P, off, I, r.req, 0);
  }
  waitagg(I, r.prompt, r.dhat, r.tru, 0, +1);
}

__device__ __forceinline__ void lane_push_front(const KParams& P, const FastGrp& G, long long off,
                                                int i, Inst& I, int req, int prompt, int dhat,
                                                int tru, int emit) {
  if (I.w_cnt == P.wcap) {  // spill the ring's back element to the overflow front
    int s = I.w_head + I.w_cnt - 1;
    if (s >= P.wcap) s -= P.wcap;
    const int b = i * G.wstride + s;
    lane_ov_push_front(P, off, I, G.w_req[b], G.w_emit[b]);
    I.w_cnt--;
  }
  I.w_head = I.w_head == 0 ? P.wcap - 1 : I.w_head - 1;
  lane_ring_put(G, i, I.w_head, req, prompt, dhat, tru, emit);
  I.w_cnt++;
  waitagg(I, prompt, dhat, tru, emit, +1);
}

// Append an admitted request to the running batch (instance.hpp:187-192).
__device__ __forceinline__ void lane_admit_one(const FastGrp& G, int i, Inst& I, int req,
                                               int prompt, int dhat, int tru, int emit) {
  const int b = i * G.R.stride + I.n;
  G.R.req[b] = req | (emit == 0 ? kFresh : 0);
  G.R.prompt[b] = prompt;
  G.R.dhat[b] = dhat;
  G.R.tru[b] = tru;
  G.R.key[b] = emit - I.D;
  I.n++;
  I.npf++;
  I.res += reserved_of(prompt, dhat, emit);
  I.pend += prompt;
  I.kv += emit;
  I.dleft += dhat > emit ? dhat - emit : 0;
  I.tleft += tru - emit;
  I.tok += prompt + emit;
  const int ge_at = dhat - emit + I.D;
  if (ge_at <= I.D) I.nge++;
  else I.next_ge = ge_at < I.next_ge ? ge_at : I.next_ge;
  const int done_at = tru - emit + I.D;
  I.next_done = done_at < I.next_done ? done_at : I.next_done;
  waitagg(I, prompt, dhat, tru, emit, -1);
}

// Instance::admit_waiting (instance.hpp:149-195) by the owning lane.
__device__ inline void lane_admit(const KParams& P, const FastGrp& G, long long off, int i,
                                  Inst& I) {
  while (I.w_cnt > 0 && I.n < P.max_batch) {
    if (P.batching == RS_BATCHING_FCFS) {
      const int b = i * G.wstride + I.w_head;
      const int prompt = G.w_prompt[b], dhat = G.w_dhat[b], emit = G.w_emit[b];
      if (I.res + reserved_of(prompt, dhat, emit) > P.kv_cap) break;
      const int req = G.w_req[b], tru = G.w_true[b];
      I.w_head = I.w_head + 1 == P.wcap ? 0 : I.w_head + 1;
      I.w_cnt--;
      lane_admit_one(G, i, I, req, prompt, dhat, tru, emit);
      lane_refill(P, G, off, i, I);
      continue;
    }
    // BinPacking (largest reservation that fits, first wins) or
    // LeastWorkLeft (smallest decode_left that fits, first wins).
    const bool bp = P.batching == RS_BATCHING_BIN_PACKING;
    int best = -1, bkey = 0, pos = -1, preq = -1;
    for (int q = 0; q < I.w_cnt; ++q) {
      int s = I.w_head + q;
      if (s >= P.wcap) s -= P.wcap;
      const int b = i * G.wstride + s;
      const int prompt = G.w_prompt[b], dhat = G.w_dhat[b], emit = G.w_emit[b];
      const int need = reserved_of(prompt, dhat, emit);
      if (I.res + need > P.kv_cap) continue;
      const int key = bp ? -need : (dhat > emit ? dhat - emit : 0);
      if (best < 0 || key < bkey) { best = 1; bkey = key; pos = q; }
    }
    int cur = I.o_head;
    for (int q = 0; q < I.o_cnt; ++q) {
      const int prompt = P.prompt[off + cur], emit = P.ov_emit[off + cur];
      const int dhat = P.ub[P.bucket[off + cur]];
      const int need = reserved_of(prompt, dhat, emit);
      if (I.res + need <= P.kv_cap) {
        const int key = bp ? -need : (dhat > emit ? dhat - emit : 0);
        if (best < 0 || key < bkey) { best = 1; bkey = key; pos = I.w_cnt + q; preq = cur; }
      }
      cur = (int)P.ov_next[off + cur];
    }
    if (best < 0) break;
    if (pos < I.w_cnt) {
      int s = I.w_head + pos;
      if (s >= P.wcap) s -= P.wcap;
      const int b = i * G.wstride + s;
      const int req = G.w_req[b], prompt = G.w_prompt[b], dhat = G.w_dhat[b], tru = G.w_true[b],
                emit = G.w_emit[b];
      for (int q = pos; q + 1 < I.w_cnt; ++q) {  // erase, order kept
        int s0 = I.w_head + q, s1 = s0 + 1;
        if (s0 >= P.wcap) s0 -= P.wcap;
        if (s1 >= P.wcap) s1 -= P.wcap;
        const int b0 = i * G.wstride + s0, b1 = i * G.wstride + s1;
        G.w_req[b0] = G.w_req[b1];
        G.w_prompt[b0] = G.w_prompt[b1];
        G.w_dhat[b0] = G.w_dhat[b1];
        G.w_true[b0] = G.w_true[b1];
        G.w_emit[b0] = G.w_emit[b1];
      }
      I.w_cnt--;
      lane_admit_one(G, i, I, req, prompt, dhat, tru, emit);
      lane_refill(P, G, off, i, I);
    } else {
      const int prompt = P.prompt[off + preq], tru = P.decode[off + preq];
      const int dhat = P.ub[P.bucket[off + preq]], emit = P.ov_emit[off + preq];
      lane_ov_unlink(P, off, I, preq);
      lane_admit_one(G, i, I, preq, prompt, dhat, tru, emit);
    }
  }
}

// Warp-cooperative rescan of instance i's running batch: completions
// (emitted >= true) are stored and compacted away, then every aggregate is
// recomputed exactly.  `owner` lane holds the instance; returns to it.
template <bool NEED_DBC>
__device__ inline void warp_scan_instance(const KParams& P, const FastGrp& G, long long off, int i,
                                          int owner, Inst& I, int* dbc_out) {
  const int l = lane_id();
  const int D = __shfl_sync(kFull, I.D, owner);
  const int n = __shfl_sync(kFull, I.n, owner);
  const double clock = __shfl_sync(kFull, I.clock, owner);
  const int base = i * G.R.stride;
  int rq[kMaxRunChunks], pr[kMaxRunChunks], dh[kMaxRunChunks], tr[kMaxRunChunks],
      ky[kMaxRunChunks];
  bool keep[kMaxRunChunks];
  int ncomp = 0;
#pragma unroll
  for (int k = 0; k < kMaxRunChunks; ++k) {
    const int j = k * kWarp + l;
    keep[k] = false;
    rq[k] = pr[k] = dh[k] = tr[k] = ky[k] = 0;
    if (k * kWarp < n) {
      bool done = false;
      if (j < n) {
        rq[k] = G.R.req[base + j];
        pr[k] = G.R.prompt[base + j];
        dh[k] = G.R.dhat[base + j];
        tr[k] = G.R.tru[base + j];
        ky[k] = G.R.key[base + j];
        done = D + ky[k] >= tr[k];
        if (done) P.o_completion[off + (rq[k] & kReqMask)] = clock;
        keep[k] = !done;
      }
      ncomp += __popc(__ballot_sync(kFull, done));
    }
  }
  int res = 0, kv = 0, dl = 0, tl = 0, tok = 0, nge = 0, nxg = kBig, nxd = kBig;
  int cnt[RS_MAX_BUCKETS];
#pragma unroll
  for (int b = 0; b < RS_MAX_BUCKETS; ++b) cnt[b] = 0;
  int npos = 0;
#pragma unroll
  for (int k = 0; k < kMaxRunChunks; ++k) {
    if (k * kWarp < n) {
      if (ncomp) {
        const unsigned km = __ballot_sync(kFull, keep[k]);
        if (keep[k]) {
          const int d = base + npos + __popc(km & lanemask_lt());
          G.R.req[d] = rq[k];
          G.R.prompt[d] = pr[k];
          G.R.dhat[d] = dh[k];
          G.R.tru[d] = tr[k];
          G.R.key[d] = ky[k];
        }
        npos += __popc(km);
      }
      if (keep[k]) {
        const int em = D + ky[k];
        res += reserved_of(pr[k], dh[k], em);
        kv += pr[k] + em;
        const int d = dh[k] - em;
        dl += d > 0 ? d : 0;
        tl += tr[k] - em;
        tok += pr[k] + em;
        if (em >= dh[k]) nge++;
        else nxg = min(nxg, dh[k] - ky[k]);
        nxd = min(nxd, tr[k] - ky[k]);
        if (NEED_DBC) cnt[bucket_of(P.state_edges, P.n_state_edges, d > 0 ? d : 0)]++;
      }
    }
  }
  res = warp_sum(res);
  kv = warp_sum(kv);
  dl = warp_sum(dl);
  tl = warp_sum(tl);
  tok = warp_sum(tok);
  nge = warp_sum(nge);
  nxg = warp_min(nxg);
  nxd = warp_min(nxd);
  if (NEED_DBC) {
#pragma unroll
    for (int b = 0; b < RS_MAX_BUCKETS; ++b) {
      const int c = warp_sum(cnt[b]);
      if (l == b) dbc_out[i * RS_MAX_BUCKETS + b] = c;
    }
  }
  __syncwarp();
  if (l == owner) {
    I.n = n - ncomp;
    I.comps += ncomp;
    I.res = res;
    I.kv = kv;
    I.pend = 0;
    I.npf = 0;
    I.dleft = dl;
    I.tleft = tl;
    I.tok = tok;
    I.nge = nge;
    I.next_ge = nxg;
    I.next_done = nxd;
    if (I.ft > I.n) I.ft = I.n;
  }
}

// preempt_if_needed (instance.hpp:282-299) by the owning lane; the caller
// rescans afterwards.  Running is in admission order, so the newest is last.
__device__ __forceinline__ bool lane_preempt(const KParams& P, const FastGrp& G, long long off,
                                             int i, Inst& I) {
  bool any = false;
  while (I.kv > P.kv_cap && I.n > 1) {
    const int b = i * G.R.stride + I.n - 1;
    const int req = G.R.req[b] & kReqMask, prompt = G.R.prompt[b], dhat = G.R.dhat[b],
              tru = G.R.tru[b];
    const int emit = I.D + G.R.key[b];
    I.kv -= prompt + emit;  // all prompts are prefilled at a step boundary
    I.n--;
    P.o_preempt[off + req] += 1;
    lane_push_front(P, G, off, i, I, req, prompt, dhat, tru, emit);
    any = true;
  }
  if (I.ft > I.n) I.ft = I.n;
  return any;
}

}  // namespace rs
