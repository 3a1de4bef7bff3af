// stats.cuh — per-replay nearest-rank percentiles on the device
// (aggregate_of, metrics.hpp:62-80).
//
// compute_metrics sorts E2E, TTFT and TBT over the completed requests and
// takes values[min(ceil(q*n) - 1, n - 1)] for q = 0.5, 0.9, 0.99.  A sort is
// not needed for three order statistics: one CTA per replay runs an MSB-first
// radix select over the order-preserving 64-bit keys of the doubles, all nine
// (metric, quantile) selections sharing the same 8 passes of 8-bit digits
// (one 256-bin shared histogram per selection).  The selected key IS the
// reference's value, bit for bit.  The fp64 means/sums stay those of the
// replay kernel (sequential, pool-index order).
#pragma once

#include "common.cuh"

namespace rs {

struct StatsParams {
  int num_replays;
  const long long* offsets;
  const double* arrival;
  const int* decode;
  const double* first;
  const double* completion;
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

__global__ void __launch_bounds__(kStatsThreads) percentile_kernel(const __grid_constant__ StatsParams P) {
  __shared__ unsigned hist[kSel][256];
  __shared__ unsigned long long prefix[kSel];
  __shared__ int krem[kSel];
  __shared__ int counts[3];
  const int t = threadIdx.x;
  for (int r = blockIdx.x; r < P.num_replays; r += gridDim.x) {
    const long long off = P.offsets[r];
    const int n = (int)(P.offsets[r + 1] - off);
    if (t < 3) counts[t] = 0;
    __syncthreads();
    int c_done = 0, c_tbt = 0;
    for (int i = t; i < n; i += kStatsThreads) {
      const double comp = P.completion[off + i];
      if (comp >= 0.0) {
        c_done++;
        c_tbt += P.decode[off + i] >= 2;  // tokens_emitted at completion
      }
    }
    atomicAdd(&counts[0], c_done);
    atomicAdd(&counts[2], c_tbt);
    __syncthreads();
    const int ne = counts[0], nt = counts[2];
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
    }
    __syncthreads();
  }
}

}  // namespace rs
