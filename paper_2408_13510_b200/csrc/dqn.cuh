// dqn.cuh — one double-DQN update step on the device:
// DqnAgent::update (dqn.hpp:107-127) on a sampled batch = double-DQN targets,
// Mlp::loss_and_gradient (mlp.hpp:78-136, Huber delta 1), AdamOptimizer::step
// (mlp.hpp:159-178), bit-identical to the reference.
//
// The reference accumulates every gradient element over the batch in sample
// order, skipping samples whose output delta is exactly 0, with one rounding
// per multiply and per add.  That order is kept by splitting the work:
//   dqn_sample_kernel : one warp per sample — targets (online argmax on s',
//                       target-net value), the forward on s with the layer
//                       inputs saved, the Huber term and clipped output
//                       delta, and the back-propagated deltas (each prev[i]
//                       is a sequential sum over o in index order).  Weights
//                       staged once per CTA in shared memory (W^T, lanes =
//                       outputs); back-propagation reads W row-major from L2
//                       (lanes = inputs, coalesced).
//   dqn_param_kernel  : one thread per parameter — its gradient as a
//                       sequential chain over the B samples, then the Adam
//                       update; thread 0 also sums the per-sample loss terms
//                       in sample order.
// Dense fp64 with per-step rounding, no reassociation: tensor cores (tcgen05 /
// DMMA) would change the rounding sequence, so the contraction stays on the
// FP64 pipe (it is 8k parameters x B samples — microseconds).
#pragma once

#include "common.cuh"
#include "mlp.cuh"

namespace rs {

struct DqnParams {
  int layers;
  int dims[RS_MAX_LAYERS + 1];
  int woff[RS_MAX_LAYERS], boff[RS_MAX_LAYERS];  // reference flat layout offsets
  int np;                                        // parameter count
  int maxw;                                      // widest layer
  int B;
  const double* state;       // [B][dims[0]]
  const int* action;         // [B]
  const double* reward;      // [B]
  const double* next_state;  // [B][dims[0]]
  const uint8_t* done;       // [B]
  const double* online;      // params (read by the sample kernel, updated by the param kernel)
  const double* target;
  double* online_out;        // == online (in place), written by dqn_param_kernel only
  double* adam_m;
  double* adam_v;
  double discount, inv_b;
  double lr, beta1, beta2, eps, bc1, bc2;
  // workspace: per sample the input of every layer and the delta at every
  // layer's output, plus the per-sample loss terms
  double* act;      // [B][act_stride]
  double* delta;    // [B][delta_stride]
  double* loss_terms;
  int act_off[RS_MAX_LAYERS], delta_off[RS_MAX_LAYERS];
  int act_stride, delta_stride;
  double* loss_out;
  int smem_w_bytes;  // one staged net (W^T + b)
};

constexpr int kDqnWarps = 8;

// Dense forward (affine, mlp.hpp:139-152: acc = b; acc += w*x in input
// order; ReLU on hidden layers) of shared-memory x by one warp, from staged
// W^T.  `save` (may be null) receives every layer's input; the output layer
// lands in `out` (shared).
__device__ inline void dqn_forward(const DqnParams& P, const double* WT, const double* x,
                                   double* h0, double* h1, double* out, double* save) {
  const int l = lane_id();
  const double* cur = x;
  for (int layer = 0; layer < P.layers; ++layer) {
    const int ni = P.dims[layer], no = P.dims[layer + 1];
    if (save)
      for (int i = l; i < ni; i += kWarp) save[P.act_off[layer] + i] = cur[i];
    const double* W = WT + P.woff[layer];
    const double* Bv = WT + P.boff[layer];
    const bool last = layer + 1 == P.layers;
    double* dst = last ? out : ((layer & 1) ? h1 : h0);
    for (int o = l; o < no; o += kWarp) {
      double acc = Bv[o];
      for (int i = 0; i < ni; ++i) acc = __dadd_rn(acc, __dmul_rn(W[i * no + o], cur[i]));
      dst[o] = (!last && !(acc > 0.0)) ? 0.0 : acc;
    }
    __syncwarp();
    cur = dst;
  }
}

__device__ __forceinline__ int dqn_argmax(const double* q, int n) {  // dqn.hpp:82-90
  int best = 0;
  for (int a = 1; a < n; ++a)
    if (q[a] > q[best]) best = a;
  return best;
}

__global__ void __launch_bounds__(kWarp * kDqnWarps) dqn_sample_kernel(const __grid_constant__ DqnParams P) {
  extern __shared__ __align__(16) double dsm[];
  const int nw = P.smem_w_bytes / 8;
  double* WTo = dsm;       // online W^T + b
  double* WTt = dsm + nw;  // target W^T + b
  mlp_stage_weights(P.online, P.layers, P.dims, P.woff, P.boff, WTo);
  mlp_stage_weights(P.target, P.layers, P.dims, P.woff, P.boff, WTt);
  const int w = threadIdx.x / kWarp, l = lane_id();
  const int d0 = P.dims[0], dout = P.dims[P.layers];
  double* scratch = dsm + 2 * nw + (size_t)w * (d0 + 4 * P.maxw);
  double* x = scratch;                 // [d0]
  double* h0 = x + d0;                 // [maxw]
  double* h1 = h0 + P.maxw;            // [maxw]
  double* q = h1 + P.maxw;             // [maxw] output layer
  double* dl = q + P.maxw;             // [maxw] delta
  for (int s = blockIdx.x * kDqnWarps + w; s < P.B; s += gridDim.x * kDqnWarps) {
    // ---- double-DQN target (dqn.hpp:113-119)
    double tgt = P.reward[s];
    if (!P.done[s]) {
      for (int i = l; i < d0; i += kWarp) x[i] = P.next_state[(size_t)s * d0 + i];
      __syncwarp();
      dqn_forward(P, WTo, x, h0, h1, q, nullptr);
      const int a_star = dqn_argmax(q, dout);
      __syncwarp();
      dqn_forward(P, WTt, x, h0, h1, q, nullptr);
      tgt = __dadd_rn(tgt, __dmul_rn(P.discount, q[a_star]));
      __syncwarp();
    }
    // ---- loss_and_gradient, one sample (mlp.hpp:88-135)
    double* save = P.act + (size_t)s * P.act_stride;
    double* dsave = P.delta + (size_t)s * P.delta_stride;
    for (int i = l; i < d0; i += kWarp) x[i] = P.state[(size_t)s * d0 + i];
    __syncwarp();
    dqn_forward(P, WTo, x, h0, h1, q, save);
    const int a = P.action[s];
    const double e = __dsub_rn(q[a], tgt);
    const double ae = fabs(e);
    if (l == 0) {
      const double h = ae <= 1.0 ? __dmul_rn(__dmul_rn(0.5, e), e) : __dsub_rn(ae, 0.5);
      P.loss_terms[s] = __dmul_rn(h, P.inv_b);
    }
    const double ec = e < -1.0 ? -1.0 : (e > 1.0 ? 1.0 : e);  // std::clamp
    for (int o = l; o < dout; o += kWarp) dl[o] = o == a ? __dmul_rn(ec, P.inv_b) : 0.0;
    __syncwarp();
    for (int layer = P.layers - 1; layer >= 0; --layer) {
      const int ni = P.dims[layer], no = P.dims[layer + 1];
      for (int o = l; o < no; o += kWarp) dsave[P.delta_off[layer] + o] = dl[o];
      if (layer == 0) break;
      const double* W = P.online + P.woff[layer];  // row-major [o][i], L2
      const double* ain = save + P.act_off[layer];
      double pd[RS_MAX_WIDTH / kWarp];
#pragma unroll
      for (int k = 0; k < RS_MAX_WIDTH / kWarp; ++k) pd[k] = 0.0;
      for (int o = 0; o < no; ++o) {
        const double d = dl[o];
        if (d == 0.0) continue;
#pragma unroll
        for (int k = 0; k < RS_MAX_WIDTH / kWarp; ++k) {
          const int i = k * kWarp + l;
          if (i < ni) pd[k] = __dadd_rn(pd[k], __dmul_rn(d, W[(size_t)o * ni + i]));
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < RS_MAX_WIDTH / kWarp; ++k) {
        const int i = k * kWarp + l;
        if (i < ni) dl[i] = ain[i] <= 0.0 ? 0.0 : pd[k];  // ReLU mask, mlp.hpp:124-130
      }
      __syncwarp();
    }
    __syncwarp();
  }
}

__global__ void dqn_param_kernel(const __grid_constant__ DqnParams P) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0) {  // loss: sequential in sample order (mlp.hpp:103)
    double loss = 0.0;
    for (int s = 0; s < P.B; ++s) loss = __dadd_rn(loss, P.loss_terms[s]);
    *P.loss_out = loss;
  }
  if (p >= P.np) return;
  // which layer / row / column this parameter is
  int layer = 0;
  while (layer + 1 < P.layers && p >= P.woff[layer + 1]) ++layer;
  const int ni = P.dims[layer], no = P.dims[layer + 1];
  const int local = p - P.woff[layer];
  const bool bias = local >= ni * no;
  const int o = bias ? local - ni * no : local / ni;
  const int i = bias ? 0 : local - o * ni;
  // gradient: sequential over samples, samples with d == 0 skipped
  double g = 0.0;
  for (int s = 0; s < P.B; ++s) {
    const double d = P.delta[(size_t)s * P.delta_stride + P.delta_off[layer] + o];
    if (d == 0.0) continue;
    g = bias ? __dadd_rn(g, d)
             : __dadd_rn(g, __dmul_rn(d, P.act[(size_t)s * P.act_stride + P.act_off[layer] + i]));
  }
  // AdamOptimizer::step (mlp.hpp:163-177)
  const double m = __dadd_rn(__dmul_rn(P.beta1, P.adam_m[p]),
                             __dmul_rn(__dsub_rn(1.0, P.beta1), g));
  const double v = __dadd_rn(__dmul_rn(P.beta2, P.adam_v[p]),
                             __dmul_rn(__dmul_rn(__dsub_rn(1.0, P.beta2), g), g));
  P.adam_m[p] = m;
  P.adam_v[p] = v;
  const double mhat = __ddiv_rn(m, P.bc1);
  const double vhat = __ddiv_rn(v, P.bc2);
  P.online_out[p] = __dsub_rn(P.online_out[p],
                              __ddiv_rn(__dmul_rn(P.lr, mhat), __dadd_rn(__dsqrt_rn(vhat), P.eps)));
}

}  // namespace rs
