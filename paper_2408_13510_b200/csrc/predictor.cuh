// predictor.cuh — kernel (d): decode-length-predictor bucket lookup.
//
// Replaces the prediction half of ClusterSim::inject_arrivals
// (env.hpp:357-375).  The reference draws predictions from ONE Rng stream
// per replay, in arrival-index order, independently of the policy, so the
// whole replay's predictions are a pure function of (trace, predictor seed)
// and are computed here in a pre-pass, one warp per replay:
//  * the 32 lanes regenerate the mt19937_64 state block (312 words) and
//    temper it into shared memory (three dependency phases, common.cuh);
//  * the draws are consumed in request order (1 draw, 2 for a miss in a
//    middle bucket, predictor.hpp:105-109), the warp walking 32 requests at a
//    time with coalesced loads of decode/task and one coalesced byte store.
#pragma once

#include "common.cuh"

namespace rs {

struct PredParams {
  double accuracy[RS_NUM_TASKS];
  int n_pred_edges;
  int pred_edges[RS_MAX_BUCKETS];
  int n_band_edges;
  int band_edges[RS_MAX_BANDS];
  uint8_t emp_table[RS_NUM_TASKS][RS_MAX_BANDS];
  int mode;
  int num_replays;
  const long long* offsets;
  const int* prompt;
  const int* decode;
  const uint8_t* task;
  const uint8_t* given;
  const uint64_t* seeds;
  uint8_t* out;
};

constexpr int kPredWarpsPerBlock = 4;

__global__ void __launch_bounds__(kWarp * kPredWarpsPerBlock)
predict_kernel(const __grid_constant__ PredParams P) {
  __shared__ unsigned long long sm_state[kPredWarpsPerBlock][312];
  __shared__ unsigned long long sm_out[kPredWarpsPerBlock][312];
  const int w = threadIdx.x / kWarp;
  const int l = lane_id();
  unsigned long long* st = sm_state[w];
  unsigned long long* ob = sm_out[w];
  const int gw = blockIdx.x * kPredWarpsPerBlock + w;
  const int nw = gridDim.x * kPredWarpsPerBlock;
  for (int r = gw; r < P.num_replays; r += nw) {
    const long long off = P.offsets[r];
    const int n = (int)(P.offsets[r + 1] - off);
    if (P.mode == RS_PREDICTOR_GIVEN) {
      for (int i = l; i < n; i += kWarp) P.out[off + i] = P.given[off + i];
      continue;
    }
    if (P.mode == RS_PREDICTOR_EMPIRICAL) {  // EmpiricalPredictor::predict
      for (int i = l; i < n; i += kWarp) {
        int band = bucket_of(P.band_edges, P.n_band_edges, P.prompt[off + i]);
        P.out[off + i] = P.emp_table[P.task[off + i]][band];
      }
      continue;
    }
    // predict_simulated (predictor.hpp:98-110) over one mt19937_64 stream
    const int nb = P.n_pred_edges;
    mt_seed_warp(st, P.seeds[r], l);
    int pos = 312;  // next unread output in `ob`
    for (int base = 0; base < n; base += kWarp) {
      const int i = base + l;
      int tb = 0;
      double acc = 1.0;
      if (i < n) {
        tb = bucket_of(P.pred_edges, nb, P.decode[off + i]);
        acc = P.accuracy[P.task[off + i]];
      }
      const int cnt = min(kWarp, n - base);
      int mine = 0;
      for (int j = 0; j < cnt; ++j) {
        const int tbj = __shfl_sync(kFull, tb, j);
        const double aj = __shfl_sync(kFull, acc, j);
        int pj = 0;
        if (nb > 1) {
          if (pos == 312) {
            mt_twist_warp(st, l);
            for (int k = l; k < 312; k += kWarp) ob[k] = mt_temper(st[k]);
            __syncwarp();
            pos = 0;
          }
          const double u = u01(ob[pos++]);
          if (u < aj) {
            pj = tbj;
          } else if (tbj == 0) {
            pj = 1;
          } else if (tbj == nb - 1) {
            pj = nb - 2;
          } else {
            if (pos == 312) {
              mt_twist_warp(st, l);
              for (int k = l; k < 312; k += kWarp) ob[k] = mt_temper(st[k]);
              __syncwarp();
              pos = 0;
            }
            pj = u01(ob[pos++]) < 0.5 ? tbj - 1 : tbj + 1;
          }
        }
        if (l == j) mine = pj;
      }
      if (i < n) P.out[off + i] = (uint8_t)mine;
    }
  }
}

}  // namespace rs
