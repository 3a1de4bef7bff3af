// common.cuh — device-side shared definitions of the B200 replay engine.
//
// Numerics: every fp64 operation that the reference performs is issued here
// as an explicitly rounded __dadd_rn / __dmul_rn / __ddiv_rn in the
// reference's evaluation order, and the library is compiled with
// -fmad=false, so no DFMA contraction can change a clock.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rs_abi.h"

namespace rs {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxRunChunks = 4;                 // running entries per lane
constexpr int kMaxRunCap = kMaxRunChunks * kWarp;  // 128 running per instance
constexpr int kMaxInstances = 128;
constexpr int kMaxFront = 32;                    // min_min stuck-front list
constexpr uint32_t kNil = 0xffffffffu;

// Per-instance scalar block kept in shared memory (the router snapshot
// aggregates are maintained here so a tick never rescans a queue).
struct __align__(16) InstHot {
  double clock;           // Instance::clock_
  long long res_wait;     // sum reserved_tokens over waiting
  long long pend_wait;    // sum prompt over waiting
  long long dleft_wait;   // sum decode_left over waiting
  long long tleft_wait;   // sum max(0, true - emitted) over waiting
  long long tok_wait;     // sum prompt + emitted over waiting (token mass)
  int n_run;              // running_.size()
  int n_prefill;          // running entries with prompt_remaining > 0
  int res_run;            // sum reserved_tokens over running
  int kv_run;             // kv_tokens_in_use (sum footprint)
  int pend_run;           // sum prompt_remaining over running
  int dleft_run;          // sum decode_left over running
  int tleft_run;          // sum true - emitted over running
  int tok_run;            // sum prompt + emitted over running
  int min_dleft;          // min decode_left over running (INT_MAX if none)
  int w_head, w_cnt;      // shared-memory waiting ring
  int o_cnt;              // overflow (global doubly linked list)
  int o_head, o_tail;
  int _pad0, _pad1;
};
static_assert(sizeof(InstHot) == 112, "InstHot layout");

// Launch parameters (kernel argument block, read through the constant bank).
struct KParams {
  // HardwareProfile (latency.hpp:16-35)
  double tpp, intercept, dpt, dtb;
  double delta_t;
  // ImpactConfig (impact.hpp:14-32)
  double grad1, grad2, eps_s, alpha;
  double rl_eps;
  double accuracy[RS_NUM_TASKS];
  int prompt_exp;
  int kv_cap;
  int max_batch;
  int batching;
  int chunk;
  int m;
  int n_state_edges;
  int n_pred_edges;
  int state_edges[RS_MAX_BUCKETS];
  int pred_edges[RS_MAX_BUCKETS];
  int ub[RS_MAX_BUCKETS];          // upper_bound_tokens per predicted bucket
  int n_band_edges;
  int band_edges[RS_MAX_BANDS];
  uint8_t emp_table[RS_NUM_TASKS][RS_MAX_BANDS];
  int predictor_mode;
  int rcap, wcap;                  // running / waiting-ring capacity
  int dsl_cutoff;
  unsigned flags;
  long long max_ticks;
  // Q-network (transposed layout in workspace, see replay.cu)
  int rl_layers;
  int rl_dims[RS_MAX_LAYERS + 1];
  int rl_woff[RS_MAX_LAYERS];      // offset of W^T of layer l (doubles)
  int rl_boff[RS_MAX_LAYERS];      // offset of b of layer l
  const double* rl_w;               // reference flat layout (device)
  int rl_maxw;                     // widest hidden layer
  int smem_weights_bytes;          // staged W^T + b at the start of smem
  const double* rl_wt_global;      // W^T + b in global memory (nets too big for smem)
  // trace (CSR over replays)
  int num_replays;
  const long long* offsets;
  const double* arrival;
  const int* prompt;
  const int* decode;
  const uint8_t* task;
  const uint8_t* bucket;           // predicted buckets (rs_predict_buckets)
  const uint64_t* policy_seed;
  // outputs
  int* o_instance;
  double* o_routed;
  double* o_first;
  double* o_completion;
  int* o_preempt;
  uint8_t* o_pred;
  rs_replay_stats* stats;
  // workspace
  uint32_t* ov_next;
  uint32_t* ov_prev;
  int* ov_emit;
  uint8_t* mm_removed;
  int* work_counter;
  // shared-memory layout (bytes, per replay group)
  int smem_group_bytes;
  int off_run, off_wait, off_dbc, off_rlx, off_rng, off_front;
  int off_pair;  // warp-pair exchange words (pair.cuh), bytes
  // fast kernel: word offsets (relative to the group base) of the running
  // entry fields and waiting-ring fields, per-instance running stride, and
  // the power-of-two lane width covering the instances (argmin reductions)
  int f_rreq, f_rprompt, f_rdhat, f_rtrue, f_rkey;
  int f_wreq, f_wprompt, f_wdhat, f_wtrue, f_wemit;
  int rstride, mwidth;
  // Running entries j < rsm of an instance live in shared memory; entries
  // j >= rsm (a batch larger than the shared head: rare) in a per-warp
  // global tail of m x rtail slots per field (L2-resident), so large fleets
  // keep several replays resident per SM (rsm = rcap: no tail)
  int rsm, rtail;
  int* run_tail;
  // Divisors that are exact powers of two divide by an exact reciprocal
  // multiply (IEEE scaling: bit-identical to the division).
  double inv_eps, inv_kv, inv_mb;
  int eps_pow2, kv_pow2, mb_pow2;
  // fused predictor (fast kernel): predictions drawn at arrival injection
  int predict_inline;
  int off_pred;                    // mt19937_64 state + 312 outputs (bytes)
  const uint64_t* predictor_seed;
  const uint8_t* given_bucket;
  // streamed inputs (host entry point): requests [0, *resident) of every
  // replay are on the device; the copy stream raises it chunk by chunk while
  // the replay runs (nullptr = everything resident, validated up front)
  const int* resident;
  // streamed outputs (host entry point): per chunk of request indices, the
  // count of replays whose requests below out_bounds[c] are all final
  // (completed); nullptr = off (internal.h rs_internal_stream_out)
  int* out_marks;
  int n_out_bounds;
  int out_bounds[16];
  // ClusterConfig::record_trajectory (general kernel only): per-tick reward
  // (env.hpp:257-303) and TickRecords (env.hpp:305-319)
  const int2* vinfo;    // fast kernel: per-replay {bad, 0} from validate_kernel (null: walk the trace)
  rs_trajectory traj;   // device arrays (by value); traj_on = 0: off
  int traj_on;
  double r_w, c_k;      // RewardConfig::r_w, shaping_coefficient(episode_k)
  int traj_scan;        // evaluate the O(active) Eq. 3 queue-penalty scan
};

// acquire-load of the streamed-input watermark
constexpr unsigned long long kStreamTimeoutNs = 20000000000ull;  // 20 s

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int load_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// x / c, correctly rounded; a multiply when c is a power of two.
__device__ __forceinline__ double div_exact(double x, double c, double inv_c, int pow2) {
  return pow2 ? __dmul_rn(x, inv_c) : __ddiv_rn(x, c);
}

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ int lane_id() { return threadIdx.x & (kWarp - 1); }
// Lane id the compiler cannot rematerialize (no repeated S2R SR_TID.X).
__device__ __forceinline__ int opaque_lane() {
  int l = threadIdx.x & (kWarp - 1);
  asm volatile("" : "+r"(l));
  return l;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ int warp_sum(int v) {
  return (int)__reduce_add_sync(kFull, (unsigned)v);
}
__device__ __forceinline__ int warp_min(int v) { return __reduce_min_sync(kFull, v); }
__device__ __forceinline__ int warp_max(int v) { return __reduce_max_sync(kFull, v); }

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(kFull, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(kFull, v, o);
    v = w > v ? w : v;
  }
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// A lane group: W consecutive lanes of a warp that run one replay.  W = 32
// is the whole warp (every collective compiles to its full-mask form); for
// small fleets (m <= W < 32) a warp runs 32/W replays side by side, each
// group's collectives restricted to its own lanes (segmented shuffles,
// masked votes and reductions).  Control flow is uniform within a group and
// may diverge between the groups of a warp.
template <int W>
struct Lanes {
  static_assert(W == 4 || W == 8 || W == 16 || W == 32, "lane group width");
  int l;          // lane within the group, 0..W-1
  int base;       // first warp lane of the group
  unsigned mask;  // the group's lanes

  __device__ __forceinline__ unsigned m() const { return W == kWarp ? kFull : mask; }
  // group-local vote bits (bit k = group lane k)
  __device__ __forceinline__ unsigned ballot(bool p) const {
    return W == kWarp ? __ballot_sync(kFull, p) : (__ballot_sync(mask, p) >> base);
  }
  __device__ __forceinline__ bool any(bool p) const { return __any_sync(m(), p); }
  template <class T>
  __device__ __forceinline__ T shfl(T v, int src) const { return __shfl_sync(m(), v, src, W); }
  template <class T>
  __device__ __forceinline__ T shfl_up(T v, int d) const { return __shfl_up_sync(m(), v, d, W); }
  template <class T>
  __device__ __forceinline__ T shfl_xor(T v, int o) const { return __shfl_xor_sync(m(), v, o, W); }
  __device__ __forceinline__ int sum(int v) const {
    return (int)__reduce_add_sync(m(), (unsigned)v);
  }
  __device__ __forceinline__ int min(int v) const { return __reduce_min_sync(m(), v); }
  __device__ __forceinline__ int max(int v) const { return __reduce_max_sync(m(), v); }
  // 64-bit group min / max as two 32-bit redux.sync reductions: the high
  // word, then the low word over the lanes tied on it (exact; replaces
  // log2(W) rounds of paired 32-bit shuffles)
  __device__ __forceinline__ unsigned long long min_u64(unsigned long long v) const {
    const unsigned hi = (unsigned)(v >> 32);
    const unsigned mh = __reduce_min_sync(m(), hi);
    const unsigned ml = __reduce_min_sync(m(), hi == mh ? (unsigned)v : 0xffffffffu);
    return ((unsigned long long)mh << 32) | ml;
  }
  __device__ __forceinline__ unsigned long long max_u64(unsigned long long v) const {
    const unsigned hi = (unsigned)(v >> 32);
    const unsigned mh = __reduce_max_sync(m(), hi);
    const unsigned ml = __reduce_max_sync(m(), hi == mh ? (unsigned)v : 0u);
    return ((unsigned long long)mh << 32) | ml;
  }
  __device__ __forceinline__ long long sum_ll(long long v) const {
#pragma unroll
    for (int o = W >> 1; o > 0; o >>= 1) v += shfl_xor(v, o);
    return v;
  }
  __device__ __forceinline__ void sync() const { __syncwarp(m()); }
  // group-local mask of the lanes below this one
  __device__ __forceinline__ unsigned lt() const {
    unsigned b;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(b));
    return W == kWarp ? b : (b >> base);
  }
};

// The calling thread's group (lane id laundered so it is computed once).
template <int W>
__device__ __forceinline__ Lanes<W> make_lanes() {
  int t = threadIdx.x & (kWarp - 1);
  asm volatile("" : "+r"(t));
  Lanes<W> L;
  L.l = t & (W - 1);
  L.base = t & ~(W - 1);
  L.mask = W == kWarp ? kFull : (((1u << (W & 31)) - 1u) << L.base);
  return L;
}

// Whole-warp group for a known lane (the general kernel and predictor).
__device__ __forceinline__ Lanes<kWarp> warp_lanes(int l) {
  Lanes<kWarp> L;
  L.l = l;
  L.base = 0;
  L.mask = kFull;
  return L;
}

// Inclusive prefix sum across the warp.
__device__ __forceinline__ int warp_incl_scan(int v, int l) {
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    int t = __shfl_up_sync(kFull, v, o);
    if (l >= o) v += t;
  }
  return v;
}

// Total order on doubles matching operator< for non-NaN values, with -0
// folded onto +0 (the reference compares with < / >, where they are equal).
__device__ __forceinline__ unsigned long long ordered_key(double x) {
  if (x == 0.0) x = 0.0;
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// Lowest lane index whose value is minimal among `valid` lanes; -1 if none.
__device__ __forceinline__ int warp_argmin_key(unsigned long long key, bool valid) {
  unsigned long long k = valid ? key : ~0ull;
  unsigned long long mn = warp_min_u64(k);
  unsigned ok = __ballot_sync(kFull, valid && k == mn);
  return ok ? __ffs(ok) - 1 : -1;
}
__device__ __forceinline__ int warp_argmax_key(unsigned long long key, bool valid) {
  unsigned long long k = valid ? key : 0ull;
  unsigned long long mx = warp_max_u64(k);
  unsigned ok = __ballot_sync(kFull, valid && k == mx);
  return ok ? __ffs(ok) - 1 : -1;
}

// BucketScheme::bucket_of (predictor.hpp:34-40)
__device__ __forceinline__ int bucket_of(const int* edges, int n, long long tokens) {
  int b = 0;
  for (int i = 1; i < n; ++i)
    if (tokens >= edges[i]) b = i;
  return b;
}

// mix of a decision into the per-replay FNV-1a hash (same as the oracles)
__device__ __forceinline__ unsigned long long hash_action(unsigned long long h, int a) {
  return (h ^ (unsigned long long)(unsigned)(a + 1)) * 0x100000001b3ull;
}

// ----------------------------------------------------- std::mt19937_64
// Group-cooperative block generation of the next 312 state words.  Three
// dependency phases of the twist (i < 156 reads only old words; 156 <= i <
// 311 reads new s[i-156]; i = 311 reads new s[0]).  A whole warp holds its
// <= 5 new words per phase in registers; a narrower group walks each phase
// in ascending W-word chunks (a chunk reads s[i+1] of the next, still old,
// chunk before anything above it is written).
__device__ __forceinline__ unsigned long long mt_tw(unsigned long long a, unsigned long long b) {
  const unsigned long long x = (a & 0xFFFFFFFF80000000ull) | (b & 0x7FFFFFFFull);
  unsigned long long xa = x >> 1;
  if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
  return xa;
}

template <int W>
__device__ __forceinline__ void mt_twist_impl(unsigned long long* s, const Lanes<W>& L) {
  const int l = L.l;
  if (W == kWarp) {
    unsigned long long nv[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int i = l + 32 * k;
      if (i < 156) nv[k] = s[i + 156] ^ mt_tw(s[i], s[i + 1]);
    }
    L.sync();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int i = l + 32 * k;
      if (i < 156) s[i] = nv[k];
    }
    L.sync();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int i = 156 + l + 32 * k;
      if (i < 311) nv[k] = s[i - 156] ^ mt_tw(s[i], s[i + 1]);
    }
    L.sync();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int i = 156 + l + 32 * k;
      if (i < 311) s[i] = nv[k];
    }
  } else {
    for (int c = 0; c < 156; c += W) {
      const int i = c + l;
      unsigned long long v = 0;
      if (i < 156) v = s[i + 156] ^ mt_tw(s[i], s[i + 1]);
      L.sync();
      if (i < 156) s[i] = v;
      L.sync();
    }
    for (int c = 156; c < 311; c += W) {
      const int i = c + l;
      unsigned long long v = 0;
      if (i < 311) v = s[i - 156] ^ mt_tw(s[i], s[i + 1]);
      L.sync();
      if (i < 311) s[i] = v;
      L.sync();
    }
  }
  L.sync();
  if (l == 0) s[311] = s[155] ^ mt_tw(s[311], s[0]);
  L.sync();
}

// Out of line: a twist runs once per 312 draws, and inlined at every call
// site its unrolled phases would crowd the tick loop out of the instruction
// cache (the RL replay kernel was 37k instructions).
template <int W>
__device__ __noinline__ void mt_twist(unsigned long long* s, const Lanes<W> L) {
  mt_twist_impl(s, L);
}
__device__ inline void mt_twist_warp(unsigned long long* s, int l) { mt_twist(s, warp_lanes(l)); }

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// Seeding (std::mt19937_64 constructor); serial recurrence, group lane 0.
template <int W>
__device__ __noinline__ void mt_seed(unsigned long long* s, unsigned long long seed, const Lanes<W> L) {
  if (L.l == 0) {
    s[0] = seed;
    for (int i = 1; i < 312; ++i)
      s[i] = 6364136223846793005ull * (s[i - 1] ^ (s[i - 1] >> 62)) + (unsigned long long)i;
  }
  L.sync();
}

__device__ inline void mt_seed_warp(unsigned long long* s, unsigned long long seed, int l) {
  mt_seed(s, seed, warp_lanes(l));
}

// Rng::uniform (rng.hpp:29): (u64 >> 11) * 2^-53, exact.
__device__ __forceinline__ double u01(unsigned long long v) {
  return __dmul_rn((double)(v >> 11), 0x1.0p-53);
}

}  // namespace rs
