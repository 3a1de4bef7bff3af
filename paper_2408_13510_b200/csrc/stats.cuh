// stats.cuh — per-replay compute_metrics aggregates on the device
// (metrics.hpp:62-162), one CTA per replay,
// launched right after the replay kernel on the same stream.
//
//  * fp64 sums (E2E, TTFT, TBT, router wait): compute_metrics accumulates
//    them sequentially in pool-index order, so warp 0 walks the replay in
//    128-request blocks and one lane adds the staged terms in index order
//    (bit-identical; a tree reduction would not be), while warps 1..7 run
//    the order-free reductions and the selections below.
//  * counts, token / preemption totals, first arrival, last completion:
//    order-free integer / min / max reductions over all threads.
//  * nearest-rank p50/p90/p99 of E2E, TTFT, TBT (aggregate_of): no sort is
//    needed for three order statistics — an MSB-first radix select over the
//    order-preserving 64-bit keys of the doubles, the nine (metric, quantile)
//    selections sharing 8 passes of 8-bit digits (one 256-bin shared
//    histogram each).  The selected key IS the reference's value, bit for bit.
#pragma once

#include "common.cuh"

namespace rs {

struct StatsParams {
  int num_replays;
  const long long* offsets;
  const double* arrival;
  const int* decode;
  const double* routed;
  const double* first;
  const double* completion;
  const int* preempt;
  rs_replay_stats* stats;
};

constexpr int kStatsThreads = 256;
constexpr int kSel = 9;  // 3 metrics x 3 quantiles

__device__ __forceinline__ unsigned long long key_of(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double value_of(unsigned long long k) {
  const unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// nearest-rank index (metrics.hpp:70-75), in the reference's arithmetic
__device__ __forceinline__ int nearest_rank_index(double q, int n) {
  long long idx = (long long)ceil(__dmul_rn(q, (double)n));
  if (idx > 0) --idx;
  return (int)(idx < n - 1 ? idx : n - 1);
}

__global__ void __launch_bounds__(kStatsThreads, 3) stats_kernel(const __grid_constant__ StatsParams P) {
  __shared__ unsigned hist[kSel][256];
  __shared__ unsigned long long prefix[kSel];
  __shared__ int krem[kSel];
  __shared__ int counts[2];
  __shared__ unsigned long long red_ll[2];      // total preemptions, total tokens
  __shared__ unsigned long long red_key[2];     // min key(arrival), max key(completion)
  __shared__ double sums[4];                    // e2e, ttft, tbt, router wait
  __shared__ double stage[4][4 * kWarp];        // warp 0's staged sum terms
  const int t = threadIdx.x;
  const int lane = t & (kWarp - 1);
  for (int r = blockIdx.x; r < P.num_replays; r += gridDim.x) {
    const long long off = P.offsets[r];
    const int n = (int)(P.offsets[r + 1] - off);
    if (t < 2) {
      counts[t] = 0;
      red_ll[t] = 0;
    }
    if (t == 0) {
      red_key[0] = ~0ull;
      red_key[1] = 0ull;
    }
    __syncthreads();
    if (t < kWarp) {
      // compute_metrics order (metrics.hpp:94-121): sequential pool-order
      // sums.  Every term is >= +0 and the sums start at +0, so a skipped
      // term (not completed, single-token TBT) is an exact +0.0 add.  Per
      // block of 128 requests the lanes stage the four terms in shared
      // memory and lane 0 runs the four add chains; the next block's global
      // loads are in flight meanwhile.
      double se = 0.0, st = 0.0, sb = 0.0, sw = 0.0;
      constexpr int U = 4;
      double cc[U], ca[U], cf[U], cr[U];
      int cd[U];
      auto load = [&](int b0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = b0 + u * kWarp + lane;
          const long long g = off + j;
          cc[u] = j < n ? P.completion[g] : -1.0;
          ca[u] = j < n ? P.arrival[g] : 0.0;
          cf[u] = j < n ? P.first[g] : 0.0;
          cr[u] = j < n ? P.routed[g] : -1.0;
          cd[u] = j < n ? P.decode[g] : 0;
        }
      };
      if (n > 0) load(0);
      for (int b0 = 0; b0 < n; b0 += U * kWarp) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool c = cc[u] >= 0.0;
          const int k = u * kWarp + lane;
          stage[0][k] = c ? __dsub_rn(cc[u], ca[u]) : 0.0;
          stage[1][k] = c ? __dsub_rn(cf[u], ca[u]) : 0.0;
          stage[2][k] = c && cd[u] >= 2
                            ? __ddiv_rn(__dsub_rn(cc[u], cf[u]), (double)(cd[u] - 1)) : 0.0;
          stage[3][k] = c && cr[u] >= 0.0 ? __dsub_rn(cr[u], ca[u]) : 0.0;
        }
        __syncwarp();
        if (b0 + U * kWarp < n) load(b0 + U * kWarp);
        if (lane == 0) {
          const int cnt = min(U * kWarp, n - b0);
#pragma unroll 8
          for (int k = 0; k < cnt; ++k) {
            se = __dadd_rn(se, stage[0][k]);
            st = __dadd_rn(st, stage[1][k]);
            sb = __dadd_rn(sb, stage[2][k]);
            sw = __dadd_rn(sw, stage[3][k]);
          }
        }
        __syncwarp();
      }
      if (t == 0) {
        sums[0] = se;
        sums[1] = st;
        sums[2] = sb;
        sums[3] = sw;
      }
    }
    else {
      // warps 1..7, concurrently with warp 0's sums: order-free aggregates
      // and the radix select (named barrier 1 over these 224 threads)
      constexpr int NT = kStatsThreads - kWarp;
      const int tt = t - kWarp;
      auto bar = [] { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); };
      int c_done = 0, c_tbt = 0;
      long long pre = 0, tok = 0;
      unsigned long long kmin = ~0ull, kmax = 0ull;
      for (int i = tt; i < n; i += NT) {
        const double comp = P.completion[off + i];
        if (comp >= 0.0) {
          const int d = P.decode[off + i];
          c_done++;
          c_tbt += d >= 2;
          tok += d;
          pre += P.preempt[off + i];
          const unsigned long long ka = key_of(P.arrival[off + i]), kc = key_of(comp);
          kmin = ka < kmin ? ka : kmin;
          kmax = kc > kmax ? kc : kmax;
        }
      }
      atomicAdd(&counts[0], c_done);
      atomicAdd(&counts[1], c_tbt);
      atomicAdd(&red_ll[0], (unsigned long long)pre);
      atomicAdd(&red_ll[1], (unsigned long long)tok);
      atomicMin(&red_key[0], kmin);
      atomicMax(&red_key[1], kmax);
      bar();
      if (tt < kSel) {
        const int metric = tt / 3;
        const double q = (tt % 3) == 0 ? 0.50 : ((tt % 3) == 1 ? 0.90 : 0.99);
        const int cnt = metric == 2 ? counts[1] : counts[0];
        krem[tt] = cnt > 0 ? nearest_rank_index(q, cnt) : -1;
        prefix[tt] = 0;
      }
      for (int pass = 0; pass < 8; ++pass) {
        for (int k = tt; k < kSel * 256; k += NT) (&hist[0][0])[k] = 0;
        bar();
        const int sh = 56 - 8 * pass;
        constexpr int U = 2;  // 2 requests per thread per iteration: loads first
        for (int i0 = tt; i0 < n; i0 += U * NT) {
          double comp[U], arr[U], fst[U];
          int d[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = i0 + u * NT;
            comp[u] = i < n ? P.completion[off + i] : -1.0;
            arr[u] = i < n ? P.arrival[off + i] : 0.0;
            fst[u] = i < n ? P.first[off + i] : 0.0;
            d[u] = i < n ? P.decode[off + i] : 0;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (!(comp[u] >= 0.0)) continue;
            unsigned long long key[3];
            key[0] = key_of(__dsub_rn(comp[u], arr[u]));
            key[1] = key_of(__dsub_rn(fst[u], arr[u]));
            key[2] = d[u] >= 2 ? key_of(__ddiv_rn(__dsub_rn(comp[u], fst[u]), (double)(d[u] - 1)))
                               : 0ull;
#pragma unroll
            for (int s2 = 0; s2 < kSel; ++s2) {
              const int mtr = s2 / 3;
              if (mtr == 2 && d[u] < 2) continue;
              if (krem[s2] < 0) continue;
              const unsigned long long kk = key[mtr];
              if (pass > 0 && (kk >> (sh + 8)) != prefix[s2]) continue;
              atomicAdd(&hist[s2][(kk >> sh) & 0xffu], 1u);
            }
          }
        }
        bar();
        if (tt < kSel && krem[tt] >= 0) {  // bucket holding rank krem
          int below = 0, dig = 0;
          for (int b = 0; b < 256; ++b) {
            const int h = (int)hist[tt][b];
            if (below + h > krem[tt]) { dig = b; break; }
            below += h;
          }
          prefix[tt] = (prefix[tt] << 8) | (unsigned long long)dig;
          krem[tt] -= below;
        }
        bar();
      }
    }
    __syncthreads();  // join: sums (warp 0) + selections (warps 1..7)
    const int ne = counts[0], nt = counts[1];
    if (t == 0) {
      rs_replay_stats& s = P.stats[r];
      auto v = [&](int k) { return krem[k] >= 0 ? value_of(prefix[k]) : 0.0; };
      s.e2e_p50 = v(0); s.e2e_p90 = v(1); s.e2e_p99 = v(2);
      s.ttft_p50 = v(3); s.ttft_p90 = v(4); s.ttft_p99 = v(5);
      s.tbt_p50 = v(6); s.tbt_p90 = v(7); s.tbt_p99 = v(8);
      s.percentiles_valid = 1;
      s.total_preemptions = (long long)red_ll[0];
      s.total_tokens = (long long)red_ll[1];
      s.tbt_count = nt;
      s.total_e2e_s = sums[0];
      s.total_ttft_s = sums[1];
      s.total_tbt_s = sums[2];
      s.total_router_wait_s = sums[3];
      // metrics.hpp:91-92,119-120 initial values when nothing completed
      const double fa = ne ? value_of(red_key[0]) : __longlong_as_double(0x7fefffffffffffffll);
      const double lc = ne ? value_of(red_key[1]) : 0.0;
      s.first_arrival_s = fa;
      s.last_completion_s = lc;
      s.makespan_s = __dsub_rn(lc, fa);
      s._pad0 = 0;
      for (int k = 0; k < 2; ++k) s._pad[k] = 0;
    }
    __syncthreads();
  }
}

// Input validation + output initialisation pre-pass of the fast replay
// kernel (device-resident inputs), one CTA per replay, bandwidth-bound and
// coalesced: the trace checks of run_replay_fast (token ranges, arrivals
// non-decreasing — ClusterSim's trace contract — and the 32-bit aggregate
// bound N x max(prompt + max(decode, bucket bound))) and the zeroing of the
// preemption counters (and min_min's removed flags), so that a replay warp
// starts simulating at once instead of walking its whole trace serially.
struct ValidateParams {
  int num_replays;
  const long long* offsets;
  const double* arrival;
  const int* prompt;
  const int* decode;
  int* o_preempt;
  uint8_t* mm_removed;  // may be null
  double* o_completion; // may be null: set to -1 (not completed; streamed outputs)
  int2* vinfo;          // per replay: {bad, 0}
};

__global__ void __launch_bounds__(kStatsThreads) validate_kernel(const __grid_constant__ ValidateParams P) {
  __shared__ int s_bad;
  const int t = threadIdx.x;
  for (int r = blockIdx.x; r < P.num_replays; r += gridDim.x) {
    const long long off = P.offsets[r];
    const int n = (int)(P.offsets[r + 1] - off);
    if (t == 0) s_bad = 0;
    __syncthreads();
    int bad = 0;
    for (int j = t; j < n; j += kStatsThreads) {
      const long long g = off + j;
      const int p = P.prompt[g], d = P.decode[g];
      if (p < 1 || p > (1 << 20) || d < 1 || d > (1 << 20)) bad = 1;
      if (j > 0 && P.arrival[g] < P.arrival[g - 1]) bad = 1;
      P.o_preempt[g] = 0;
      if (P.mm_removed) P.mm_removed[g] = 0;
      if (P.o_completion) P.o_completion[g] = -1.0;
    }
    if (bad) atomicOr(&s_bad, 1);
    __syncthreads();
    if (t == 0) P.vinfo[r] = make_int2(s_bad, 0);
    __syncthreads();
  }
}

}  // namespace rs
