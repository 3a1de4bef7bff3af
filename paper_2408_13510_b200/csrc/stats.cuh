// stats.cuh — per-replay compute_metrics aggregates on the device
// (metrics.hpp:62-162), one CTA per replay,
// launched right after the replay kernel on the same stream.
//
//  * fp64 sums (E2E, TTFT, TBT, router wait): compute_metrics accumulates
//    them sequentially in pool-index order, so warp 0 walks the replay in
//    32-request chunks and adds the shuffled terms one by one in index order
//    (bit-identical; a tree reduction would not be).
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

__global__ void __launch_bounds__(kStatsThreads) stats_kernel(const __grid_constant__ StatsParams P) {
  __shared__ unsigned hist[kSel][256];
  __shared__ unsigned long long prefix[kSel];
  __shared__ int krem[kSel];
  __shared__ int counts[2];
  __shared__ unsigned long long red_ll[2];      // total preemptions, total tokens
  __shared__ unsigned long long red_key[2];     // min key(arrival), max key(completion)
  __shared__ double sums[4];                    // e2e, ttft, tbt, router wait
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
      // compute_metrics order (metrics.hpp:94-121): sequential pool-order sums
      double se = 0.0, st = 0.0, sb = 0.0, sw = 0.0;
      for (int b0 = 0; b0 < n; b0 += kWarp) {
        const int j = b0 + lane;
        const long long g = off + j;
        const double comp = j < n ? P.completion[g] : -1.0;
        const bool c = comp >= 0.0;
        double e = 0.0, f = 0.0, tb = 0.0, w = 0.0;
        bool htb = false, hw = false;
        if (c) {
          const double arr = P.arrival[g];
          const double fst = P.first[g];
          const double rt = P.routed[g];
          const int d = P.decode[g];  // tokens_emitted at completion
          e = __dsub_rn(comp, arr);
          f = __dsub_rn(fst, arr);
          if (d >= 2) {
            htb = true;
            tb = __ddiv_rn(__dsub_rn(comp, fst), (double)(d - 1));
          }
          if (rt >= 0.0) {
            hw = true;
            w = __dsub_rn(rt, arr);
          }
        }
        const unsigned cm = __ballot_sync(kFull, c), tm = __ballot_sync(kFull, htb),
                       wm = __ballot_sync(kFull, hw);
        for (int k = 0; k < kWarp; ++k) {
          const double ek = __shfl_sync(kFull, e, k), fk = __shfl_sync(kFull, f, k);
          const double bk = __shfl_sync(kFull, tb, k), wk = __shfl_sync(kFull, w, k);
          if ((cm >> k) & 1u) {
            se = __dadd_rn(se, ek);
            st = __dadd_rn(st, fk);
          }
          if ((tm >> k) & 1u) sb = __dadd_rn(sb, bk);
          if ((wm >> k) & 1u) sw = __dadd_rn(sw, wk);
        }
      }
      if (t == 0) {
        sums[0] = se;
        sums[1] = st;
        sums[2] = sb;
        sums[3] = sw;
      }
    }
    // order-free aggregates (every thread, warp 0 included)
    int c_done = 0, c_tbt = 0;
    long long pre = 0, tok = 0;
    unsigned long long kmin = ~0ull, kmax = 0ull;
    for (int i = t; i < n; i += kStatsThreads) {
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
    __syncthreads();
    const int ne = counts[0], nt = counts[1];
    if (t < kSel) {
      const int metric = t / 3;
      const double q = (t % 3) == 0 ? 0.50 : ((t % 3) == 1 ? 0.90 : 0.99);
      const int cnt = metric == 2 ? nt : ne;
      krem[t] = cnt > 0 ? nearest_rank_index(q, cnt) : -1;
      prefix[t] = 0;
    }
    for (int pass = 0; pass < 8; ++pass) {
      for (int k = t; k < kSel * 256; k += kStatsThreads) (&hist[0][0])[k] = 0;
      __syncthreads();
      const int sh = 56 - 8 * pass;
      for (int i = t; i < n; i += kStatsThreads) {
        const double comp = P.completion[off + i];
        if (!(comp >= 0.0)) continue;
        const double arr = P.arrival[off + i];
        const double fst = P.first[off + i];
        const int d = P.decode[off + i];
        unsigned long long key[3];
        key[0] = key_of(__dsub_rn(comp, arr));
        key[1] = key_of(__dsub_rn(fst, arr));
        key[2] = d >= 2 ? key_of(__ddiv_rn(__dsub_rn(comp, fst), (double)(d - 1))) : 0ull;
#pragma unroll
        for (int s = 0; s < kSel; ++s) {
          const int mtr = s / 3;
          if (mtr == 2 && d < 2) continue;
          if (krem[s] < 0) continue;
          const unsigned long long kk = key[mtr];
          if (pass > 0 && (kk >> (sh + 8)) != prefix[s]) continue;
          atomicAdd(&hist[s][(kk >> sh) & 0xffu], 1u);
        }
      }
      __syncthreads();
      if (t < kSel && krem[t] >= 0) {  // bucket holding rank krem
        int below = 0, dig = 0;
        for (int b = 0; b < 256; ++b) {
          const int h = (int)hist[t][b];
          if (below + h > krem[t]) { dig = b; break; }
          below += h;
        }
        prefix[t] = (prefix[t] << 8) | (unsigned long long)dig;
        krem[t] -= below;
      }
      __syncthreads();
    }
    if (t == 0) {
      rs_replay_stats& s = P.stats[r];
      double v[kSel];
      for (int k = 0; k < kSel; ++k) v[k] = krem[k] >= 0 ? value_of(prefix[k]) : 0.0;
      s.e2e_p50 = v[0]; s.e2e_p90 = v[1]; s.e2e_p99 = v[2];
      s.ttft_p50 = v[3]; s.ttft_p90 = v[4]; s.ttft_p99 = v[5];
      s.tbt_p50 = v[6]; s.tbt_p90 = v[7]; s.tbt_p99 = v[8];
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
      for (int k = 0; k < 4; ++k) s._pad[k] = 0;
    }
    __syncthreads();
  }
}

}  // namespace rs
