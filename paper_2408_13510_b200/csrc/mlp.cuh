// mlp.cuh — kernel (c): the RL router's Q-network forward + action selection.
//
// Mlp::forward (mlp.hpp:54-68 / affine mlp.hpp:139-152) computes, per output,
//     acc = b[o]; for i in 0..ni-1: acc += w[o][i] * x[i]
// with one rounding after every multiply and every add.  Bit-exact parity
// forbids reassociation (no split-K, no tensor-core accumulation: tcgen05 /
// DMMA accumulate with a different rounding sequence), so each output is a
// sequential fp64 chain; the parallelism is across outputs (one lane per
// output, two chains per lane for ILP) and across replays (one warp each).
//
// The weights are staged ONCE per CTA in shared memory, transposed to
// W^T[i][o] so that the 32 lanes of a warp read 32 consecutive doubles per
// input (conflict-free), and x[i] is a shared-memory broadcast.
//
// Exact-zero inputs are skipped: w*(+-0) = +-0 and acc + (+-0) == acc for
// every acc != 0; for acc == +-0 only the sign of a zero can differ, which no
// ReLU (v > 0 ? v : 0) or argmax (strict >) can observe.  Decisions and
// non-zero Q values are therefore bit-identical to the reference.
#pragma once

#include "common.cuh"

namespace rs {

struct MlpView {
  int layers;
  const int* dims;   // layers + 1
  const int* woff;   // per layer: offset of W^T (doubles) in `w`
  const int* boff;   // per layer: offset of b
  const double* w;   // shared memory
};

// Forward of one state vector `x` (shared memory, dims[0] doubles) by one
// warp.  h0/h1: shared scratch of max width.  Writes the final layer to
// `q_out` (may be nullptr) and returns argmax_action (dqn.hpp:82-90).
template <int W>
__device__ __forceinline__ int mlp_forward_warp_impl(const MlpView& M, const double* x, double* h0,
                                                     double* h1, double* q_out, const Lanes<W>& L,
                                                     long long* macs) {
  const int l = L.l;
  const double* cur = x;
  unsigned long long best_key = 0;
  int best_idx = 0x7fffffff;
  bool have = false;
  for (int layer = 0; layer < M.layers; ++layer) {
    const int ni = M.dims[layer], no = M.dims[layer + 1];
    const double* WT = M.w + M.woff[layer];
    const double* B = M.w + M.boff[layer];
    const bool last = (layer + 1 == M.layers);
    double* dst = (layer & 1) ? h1 : h0;
    int nz = 0;  // nonzero inputs (uniform)
    for (int ob = 0; ob < no; ob += 2 * W) {
      const int o0 = ob + l, o1 = ob + W + l;
      const bool v0 = o0 < no, v1 = o1 < no;
      double a0 = v0 ? B[o0] : 0.0;
      double a1 = v1 ? B[o1] : 0.0;
#pragma unroll 4
      for (int i = 0; i < ni; ++i) {
        const double xi = cur[i];
        if (xi != 0.0) {
          nz += ob == 0;
          const double* row = WT + (size_t)i * no;
          const double w0 = v0 ? row[o0] : 0.0;
          const double w1 = v1 ? row[o1] : 0.0;
          a0 = __dadd_rn(a0, __dmul_rn(w0, xi));
          a1 = __dadd_rn(a1, __dmul_rn(w1, xi));
        }
      }
      if (!last) {
        if (v0) dst[o0] = a0 > 0.0 ? a0 : 0.0;
        if (v1) dst[o1] = a1 > 0.0 ? a1 : 0.0;
      } else {
        if (q_out) {
          if (v0) q_out[o0] = a0;
          if (v1) q_out[o1] = a1;
        }
        // running argmax, strict >: lower indices win ties
        if (v0) {
          unsigned long long k = ordered_key(a0);
          if (!have || k > best_key) { best_key = k; best_idx = o0; have = true; }
        }
        if (v1) {
          unsigned long long k = ordered_key(a1);
          if (!have || k > best_key) { best_key = k; best_idx = o1; have = true; }
        }
      }
    }
    L.sync();
    cur = dst;
    if (macs) *macs += (long long)nz * no;
  }
  const unsigned long long gmax = L.max_u64(have ? best_key : 0ull);
  const int cand = (have && best_key == gmax) ? best_idx : 0x7fffffff;
  return L.min(cand);
}

// Out of line in the replay kernels: they call it only for Q-networks too
// big for the staged forward (and the general kernel once per tick); inlined,
// it doubled the tick loop's instruction footprint.
template <int W>
__device__ __noinline__ int mlp_forward_warp(const MlpView M, const double* x, double* h0,
                                             double* h1, double* q_out, const Lanes<W> L,
                                             long long* macs = nullptr) {
  return mlp_forward_warp_impl(M, x, h0, h1, q_out, L, macs);
}

// The batched forward kernel (rs_mlp_forward): inline.
__device__ inline int mlp_forward_warp(const MlpView& M, const double* x, double* h0,
                                       double* h1, double* q_out, int l) {
  return mlp_forward_warp_impl(M, x, h0, h1, q_out, warp_lanes(l), nullptr);
}

extern __shared__ __align__(16) double rs_smd[];

// widest layer the shared-memory forward handles (wider nets: global path)
constexpr int kMlpMaskWords = 4;
constexpr int kMlpSmemMaxWidth = kMlpMaskWords * kWarp;

// Forward with weights staged in shared memory (double index 0, W^T rows
// [i][o]), x at double index xd, and per warp two lists of a layer's nonzero
// inputs in ascending index order as 16-byte records {value, W^T row offset}:
// A at double index lvd + 2k, B over the h0 | h1 area from h0d (both even).
// The accumulation is a counted loop over the nonzero terms only: each output
// still adds w*x for i = 0..ni-1 in order, zero terms omitted exactly as in
// mlp_forward_warp.  Layers with an even width and an even weight offset give
// each lane two ADJACENT outputs, so one 16-byte load fetches both weights
// (and one fetches the list record): 7 instructions per term pair instead of
// 10; other layers (the m+1-wide output layer) run one accumulator per lane.
template <int W>
__device__ inline int mlp_forward_list(const int* dims, const int* woff, const int* boff,
                                       int layers, int xd, int h0d, int h1d, int lvd,
                                       const Lanes<W>& L, long long& macs) {
  (void)h1d;  // h0 | h1 (contiguous, 2 x maxw doubles) hold the second record list
  const int l = L.l;
  const unsigned lt = L.lt();
  unsigned long long best_key = 0;
  int best_idx = 0x7fffffff;
  bool have = false;
  // the input layer's nonzero entries, compacted from x into list A
  int nnz = 0;
  {
    const int ni = dims[0], no = dims[1], wt = woff[0];
    for (int c = 0; c < ni; c += W) {
      const int i = c + l;
      const double v = i < ni ? rs_smd[xd + i] : 0.0;
      const bool nz = v != 0.0;
      const unsigned msk = L.ballot(nz);
      if (nz) {
        const int p = nnz + __popc(msk & lt);
        rs_smd[lvd + 2 * p] = v;
        rs_smd[lvd + 2 * p + 1] = __longlong_as_double((long long)(wt + i * no));
      }
      nnz += __popc(msk);
    }
    L.sync();
  }
  for (int layer = 0; layer < layers; ++layer) {
    const int no = dims[layer + 1];
    const int wt = woff[layer], bs = boff[layer];
    const bool last = layer + 1 == layers;
    // ping-pong: even layers read list A (lvd) and write B (h0d), odd ones
    // the reverse.  A hidden layer's ReLU outputs go straight into the next
    // layer's list: only the nonzero ones, in ascending output order, as
    // {value, next layer's W^T row} records (the list the compaction of a
    // stored h would build, without the store and re-read).
    const int ind = (layer & 1) ? h0d : lvd;
    const int outd = (layer & 1) ? lvd : h0d;
    const double2* rec = reinterpret_cast<const double2*>(rs_smd + ind);
    const int nwt = last ? 0 : woff[layer + 1];
    const int nno = last ? 0 : dims[layer + 2];
    int nout = 0;
    auto put = [&](int p, int o, double a) {
      rs_smd[outd + 2 * p] = a;
      rs_smd[outd + 2 * p + 1] = __longlong_as_double((long long)(nwt + o * nno));
    };
    auto arg = [&](int o, double a) {  // running argmax, strict >: lower indices win ties
      const unsigned long long k = ordered_key(a);
      if (!have || k > best_key) { best_key = k; best_idx = o; have = true; }
    };
    if (((no | wt) & 1) == 0) {  // paired adjacent outputs
      for (int ob = 0; ob < no; ob += 2 * W) {
        const int o0 = ob + 2 * l;
        const bool v = o0 < no;
        const int c0 = v ? o0 : 0;
        double a0 = v ? rs_smd[bs + o0] : 0.0;
        double a1 = v ? rs_smd[bs + o0 + 1] : 0.0;
#pragma unroll 4
        for (int k = 0; k < nnz; ++k) {
          const double2 r = rec[k];
          const int row = (int)__double_as_longlong(r.y);
          const double2 w = *reinterpret_cast<const double2*>(rs_smd + row + c0);
          a0 = __dadd_rn(a0, __dmul_rn(w.x, r.x));
          a1 = __dadd_rn(a1, __dmul_rn(w.y, r.x));
        }
        if (!last) {  // ReLU: a > 0 keeps a, anything else is an exact zero
          const bool nz0 = v && a0 > 0.0, nz1 = v && a1 > 0.0;
          const unsigned b0 = L.ballot(nz0), b1 = L.ballot(nz1);
          const int p = nout + __popc(b0 & lt) + __popc(b1 & lt);
          if (nz0) put(p, o0, a0);
          if (nz1) put(p + (nz0 ? 1 : 0), o0 + 1, a1);
          nout += __popc(b0) + __popc(b1);
        } else if (v) {
          arg(o0, a0);
          arg(o0 + 1, a1);
        }
      }
    } else {  // one output per lane
      for (int ob = 0; ob < no; ob += W) {
        const int o0 = ob + l;
        const bool v = o0 < no;
        const int c0 = v ? o0 : 0;
        double a0 = v ? rs_smd[bs + o0] : 0.0;
#pragma unroll 4
        for (int k = 0; k < nnz; ++k) {
          const double2 r = rec[k];
          const int row = (int)__double_as_longlong(r.y);
          a0 = __dadd_rn(a0, __dmul_rn(rs_smd[row + c0], r.x));
        }
        if (!last) {
          const bool nz0 = v && a0 > 0.0;
          const unsigned b0 = L.ballot(nz0);
          if (nz0) put(nout + __popc(b0 & lt), o0, a0);
          nout += __popc(b0);
        } else if (v) {
          arg(o0, a0);
        }
      }
    }
    L.sync();
    macs += (long long)nnz * no;
    nnz = nout;
  }
  const unsigned long long gmax = L.max_u64(have ? best_key : 0ull);
  const int cand = (have && best_key == gmax) ? best_idx : 0x7fffffff;
  return L.min(cand);
}

// Element k of the reference flat vector -> its slot in the transposed layout.
__device__ __forceinline__ void mlp_transpose_elem(const double* __restrict__ params, int layers,
                                                   const int* dims, const int* woff,
                                                   const int* boff, double* out, size_t k) {
  size_t src = 0;
  for (int layer = 0; layer < layers; ++layer) {
    const int ni = dims[layer], no = dims[layer + 1];
    const size_t nw = (size_t)ni * no;
    if (k < src + nw) {
      const size_t e = k - src;
      const int o = (int)(e / ni), i = (int)(e - (size_t)o * ni);
      out[woff[layer] + (size_t)i * no + o] = params[k];
      return;
    }
    if (k < src + nw + no) {
      out[boff[layer] + (k - src - nw)] = params[k];
      return;
    }
    src += nw + no;
  }
}

struct MlpTransposeArgs {
  const double* params;
  int layers;
  int dims[RS_MAX_LAYERS + 1];
  int woff[RS_MAX_LAYERS], boff[RS_MAX_LAYERS];
  double* out;
  size_t count;
};

// Global-memory transposed copy for Q-networks too large to stage in smem.
template <int Unused = 0>
__global__ void mlp_transpose_kernel(const __grid_constant__ MlpTransposeArgs A) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < A.count) mlp_transpose_elem(A.params, A.layers, A.dims, A.woff, A.boff, A.out, k);
}

// Cooperative (whole CTA) copy of the reference flat parameter vector
// (per layer W[o][i] row-major, then b) into the transposed shared layout.
__device__ inline void mlp_stage_weights(const double* __restrict__ params, int layers,
                                         const int* dims, const int* woff, const int* boff,
                                         double* smem_w) {
  size_t src = 0;
  for (int layer = 0; layer < layers; ++layer) {
    const int ni = dims[layer], no = dims[layer + 1];
    const int nw = ni * no;
    for (int k = threadIdx.x; k < nw; k += blockDim.x) {
      const int o = k / ni, i = k - o * ni;
      smem_w[woff[layer] + i * no + o] = params[src + k];
    }
    for (int k = threadIdx.x; k < no; k += blockDim.x) smem_w[boff[layer] + k] = params[src + nw + k];
    src += (size_t)nw + no;
  }
  __syncthreads();
}

}  // namespace rs
