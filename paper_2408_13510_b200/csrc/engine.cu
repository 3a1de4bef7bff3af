// engine.cu — host side of the C ABI (include/rs_abi.h): configuration
// validation, workspace layout, launch sizing and the device / host entry
// points.  All compute happens in the sm_100a kernels of predictor.cuh,
// replay.cuh, router.cuh and mlp.cuh; there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/rs_abi.h"
#include "common.cuh"
#include "mlp.cuh"
#include "predictor.cuh"
#include "router.cuh"
#include "fast_kernel.cuh"
#include "stats.cuh"
#include "internal.h"

namespace {

thread_local std::string g_err;

rs_status fail(rs_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define RS_CUDA(call)                                                             \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      return fail(e_ == cudaErrorMemoryAllocation ? RS_ERR_OUT_OF_MEMORY          \
                                                  : RS_ERR_CUDA,                  \
                  std::string(#call) + ": " + cudaGetErrorString(e_));            \
    }                                                                             \
  } while (0)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// upper_bound_tokens (predictor.hpp:44-51) for every predicted bucket.
int64_t ub_of(const rs_batch_cfg& c, int b) {
  return b + 1 < c.n_predictor_edges ? c.predictor_edges[b + 1] : c.predictor_top_cap;
}

bool device_ok(int dev) {
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return false;
  return p.major == 10;  // sm_100 family (the library carries sm_100a code)
}

rs_status require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail(RS_ERR_NO_DEVICE, "no CUDA device (the engine has no CPU fallback)");
  int dev = 0;
  cudaGetDevice(&dev);
  if (!device_ok(dev)) return fail(RS_ERR_NO_DEVICE, "current device is not sm_100");
  return RS_OK;
}

// Smem layout of one replay group (one warp) for this config.
struct Layout {
  int rcap, rsm, wcap;
  int off_run, off_wait, off_dbc, off_rlx, off_rng, off_front, off_pred, off_pair, group_bytes;
  int weights_bytes;
  int woff[RS_MAX_LAYERS], boff[RS_MAX_LAYERS];
  int maxw;
};

int min_reservation(const rs_batch_cfg& c) {
  int64_t mn = c.predictor_top_cap;
  for (int b = 0; b < c.n_predictor_edges; ++b) mn = std::min<int64_t>(mn, ub_of(c, b));
  return (int)std::max<int64_t>(2, 1 + mn);
}

int run_cap(const rs_batch_cfg& c) {
  const int rcap =
      (int)std::min<int64_t>(c.max_batch_size, c.kv_capacity_tokens / min_reservation(c));
  return std::max(rcap, 1);
}

// fast = the lane-per-instance kernel (no InstHot block, 5 running fields
// with an odd per-instance stride so lane-owned rows hit distinct banks;
// the first rsm entries of each instance in shared memory, the rest in the
// warp's global tail).
// fused = the simulated predictor draws inside the replay kernel (its
// mt19937_64 block lives in the replay's shared slot).
Layout make_layout(const rs_batch_cfg& c, int wcap, bool fast, int rsm = 0, bool fused = true) {
  Layout L{};
  const int m = c.num_instances;
  L.rcap = run_cap(c);
  L.rsm = fast ? std::max(1, std::min(rsm > 0 ? rsm : L.rcap, L.rcap)) : L.rcap;
  L.wcap = wcap;
  size_t off = fast ? 0 : (size_t)m * sizeof(rs::InstHot);
  L.off_run = (int)off;
  off = fast ? align_up(off + 5ull * m * (L.rsm | 1) * sizeof(int), 16)
             : align_up(off + 6ull * m * L.rcap * sizeof(int), 16);
  L.off_wait = (int)off;
  off = align_up(off + 5ull * m * L.wcap * sizeof(int), 16);
  L.off_dbc = (int)off;
  const bool rl = c.policy == RS_POLICY_RL;
  if (rl) off = align_up(off + (size_t)m * RS_MAX_BUCKETS * sizeof(int), 16);
  L.off_rlx = (int)off;
  L.maxw = 0;
  if (rl) {
    for (int l = 1; l < c.rl_num_layers; ++l) L.maxw = std::max(L.maxw, c.rl_dims[l]);
    L.maxw = std::max(L.maxw, 1);
    // x, h0, h1 (each rounded up to an even number of doubles), then the
    // nonzero-input list of 16-byte {value, row} records
    const size_t lmax = (size_t)std::max(c.rl_dims[0], L.maxw);
    const size_t ev = ((size_t)c.rl_dims[0] + 1) & ~(size_t)1;
    const size_t mw = ((size_t)L.maxw + 1) & ~(size_t)1;
    off = align_up(off + (ev + 2 * mw + 2 * lmax) * sizeof(double), 16);
  }
  L.off_rng = (int)off;
  if (rl && c.rl_epsilon > 0.0) off = align_up(off + 312 * sizeof(unsigned long long), 16);
  L.off_front = (int)off;
  if (c.policy == RS_POLICY_MIN_MIN) off = align_up(off + rs::kMaxFront * sizeof(int), 16);
  L.off_pred = (int)off;  // fused predictor's mt19937_64 state + outputs
  if (fast && fused && (c.flags & RS_FLAG_PREDICT_INLINE) &&
      c.predictor_mode == RS_PREDICTOR_SIMULATED)
    off = align_up(off + 312 * sizeof(unsigned long long), 16);
  L.off_pair = (int)off;  // warp-pair exchange words (m > 32: pair.cuh)
  if (fast && m > 32) off = align_up(off + 32 * sizeof(int), 16);
  L.group_bytes = (int)align_up(off, 128);
  L.weights_bytes = 0;
  if (rl) {
    size_t w = 0;
    for (int l = 0; l < c.rl_num_layers; ++l) {
      L.woff[l] = (int)w;
      w += (size_t)c.rl_dims[l] * c.rl_dims[l + 1];
      L.boff[l] = (int)w;
      w += (size_t)c.rl_dims[l + 1];
    }
    L.weights_bytes = (int)align_up(w * sizeof(double), 128);
  }
  return L;
}

rs_status validate(const rs_batch_cfg* c) {
  if (!c) return fail(RS_ERR_INVALID_ARGUMENT, "null config");
  if (c->abi_version != RS_ABI_VERSION) return fail(RS_ERR_INVALID_ARGUMENT, "abi_version mismatch");
  const rs_profile& p = c->profile;  // HardwareProfile::validate, latency.hpp:25-34
  if (!(p.prompt_time_per_token > 0.0) || !(p.prompt_time_intercept > 0.0) ||
      !(p.decode_time_per_token > 0.0) || !(p.decode_time_base > 0.0))
    return fail(RS_ERR_INVALID_ARGUMENT, "profile: all fields must be > 0");
  if (p.prompt_time_per_token <= p.decode_time_per_token)
    return fail(RS_ERR_INVALID_ARGUMENT,
                "profile: prompt_time_per_token must exceed decode_time_per_token");
  const rs_thresholds& t = c->thresholds;  // latency.hpp:42-50
  if (!(t.heavy_prompt_seconds > 0.0) || !(t.heavy_decode_seconds > 0.0))
    return fail(RS_ERR_INVALID_ARGUMENT, "thresholds: values must be > 0");
  if (t.heavy_decode_seconds <= t.heavy_prompt_seconds)
    return fail(RS_ERR_INVALID_ARGUMENT,
                "thresholds: heavy_decode_seconds must exceed heavy_prompt_seconds");
  const rs_impact& im = c->impact;  // impact.hpp:21-31
  if (!(im.grad1 > 0.0) || !(im.grad2 > 0.0) || !(im.epsilon_s > 0.0))
    return fail(RS_ERR_INVALID_ARGUMENT, "impact: grad1, grad2, epsilon_s must be > 0");
  if (im.alpha < 0.0 || im.alpha > 1.0) return fail(RS_ERR_INVALID_ARGUMENT, "impact: alpha outside [0, 1]");
  if (im.prompt_exponent != 1 && im.prompt_exponent != 2)
    return fail(RS_ERR_INVALID_ARGUMENT, "impact: prompt_exponent must be 1 or 2");
  if (c->kv_capacity_tokens < 1) return fail(RS_ERR_INVALID_ARGUMENT, "kv_capacity_tokens must be >= 1");
  if (c->max_batch_size < 1) return fail(RS_ERR_INVALID_ARGUMENT, "max_batch_size must be >= 1");
  if (c->chunk_size < 0) return fail(RS_ERR_INVALID_ARGUMENT, "chunk_size must be >= 1 (or 0 = off)");
  if (c->batching < 0 || c->batching > 2) return fail(RS_ERR_INVALID_ARGUMENT, "unknown batching policy");
  if (c->num_instances < 1) return fail(RS_ERR_INVALID_ARGUMENT, "cluster: num_instances must be >= 1");
  if (!(c->delta_t > 0.0)) return fail(RS_ERR_INVALID_ARGUMENT, "cluster: delta_t must be > 0");
  if (c->policy < 0 || c->policy >= RS_POLICY_COUNT) return fail(RS_ERR_INVALID_ARGUMENT, "unknown routing policy");
  auto check_edges = [](const int64_t* e, int n, const char* what) -> rs_status {
    if (n < 1 || n > RS_MAX_BUCKETS) return fail(RS_ERR_UNSUPPORTED, std::string(what) + ": 1..8 edges supported");
    if (e[0] != 0) return fail(RS_ERR_INVALID_ARGUMENT, std::string(what) + ": first edge must be 0");
    for (int i = 1; i < n; ++i)
      if (e[i] <= e[i - 1]) return fail(RS_ERR_INVALID_ARGUMENT, std::string(what) + ": edges must ascend");
    if (e[n - 1] > rs::kMaxTokens) return fail(RS_ERR_UNSUPPORTED, std::string(what) + ": edge above 2^20");
    return RS_OK;
  };
  rs_status s;
  if ((s = check_edges(c->predictor_edges, c->n_predictor_edges, "predictor scheme")) != RS_OK) return s;
  if ((s = check_edges(c->state_edges, c->n_state_edges, "state scheme")) != RS_OK) return s;
  if (c->predictor_top_cap < 1 || c->predictor_top_cap > rs::kMaxTokens)
    return fail(RS_ERR_UNSUPPORTED, "predictor_top_cap outside [1, 2^20]");
  for (int k = 0; k < RS_NUM_TASKS; ++k)
    if (c->accuracy[k] < 0.0 || c->accuracy[k] > 1.0)
      return fail(RS_ERR_INVALID_ARGUMENT, "accuracy outside [0,1]");
  if (c->predictor_mode < 0 || c->predictor_mode > 2) return fail(RS_ERR_INVALID_ARGUMENT, "unknown predictor mode");
  if (c->predictor_mode == RS_PREDICTOR_EMPIRICAL) {
    if ((s = check_edges(c->band_edges, c->n_band_edges, "band scheme")) != RS_OK) return s;
    for (int t2 = 0; t2 < RS_NUM_TASKS; ++t2)
      for (int b = 0; b < c->n_band_edges; ++b)
        if (c->empirical_table[t2][b] >= c->n_predictor_edges)
          return fail(RS_ERR_INVALID_ARGUMENT, "empirical_table bucket out of range");
  }
  // engine limits: 32-bit token arithmetic on device
  if (c->kv_capacity_tokens > (1ll << 30)) return fail(RS_ERR_UNSUPPORTED, "kv_capacity_tokens above 2^30");
  if (c->num_instances > rs::kMaxInstances) return fail(RS_ERR_UNSUPPORTED, "more than 128 instances");
  const int rcap = (int)std::min<int64_t>(c->max_batch_size, c->kv_capacity_tokens / min_reservation(*c));
  if (rcap > rs::kMaxRunCap) return fail(RS_ERR_UNSUPPORTED, "more than 128 concurrently running requests per instance");
  if (c->policy == RS_POLICY_RL) {
    if (c->rl_num_layers < 1 || c->rl_num_layers > RS_MAX_LAYERS)
      return fail(RS_ERR_INVALID_ARGUMENT, "rl: 1..4 layers");
    for (int l = 0; l <= c->rl_num_layers; ++l)
      if (c->rl_dims[l] < 1 || c->rl_dims[l] > RS_MAX_WIDTH)
        return fail(RS_ERR_UNSUPPORTED, "rl: layer width outside [1, 512]");
    if (c->rl_dims[0] != c->num_instances * (3 + c->n_state_edges) + 3)
      return fail(RS_ERR_INVALID_ARGUMENT, "rl: input width != state_dimension (env.hpp:78-80)");
    if (c->rl_dims[c->rl_num_layers] != c->num_instances + 1)
      return fail(RS_ERR_INVALID_ARGUMENT, "rl: output width != num_instances + 1");
    if (!c->rl_params) return fail(RS_ERR_INVALID_ARGUMENT, "rl: null parameters");
    if (c->rl_epsilon < 0.0 || c->rl_epsilon > 1.0) return fail(RS_ERR_INVALID_ARGUMENT, "rl: epsilon outside [0,1]");
  }
  if (c->max_ticks < 0) return fail(RS_ERR_INVALID_ARGUMENT, "max_ticks must be >= 0");
  return RS_OK;
}

// heavy_decode_token_cutoff (latency.hpp:132-138)
int64_t heavy_cutoff(const rs_profile& p, const rs_thresholds& t) {
  int64_t c = (int64_t)std::ceil(t.heavy_decode_seconds / p.decode_time_base - 1e-12);
  while (!(p.decode_time_base * (double)c >= t.heavy_decode_seconds)) ++c;
  return c;
}

struct WsLayout {
  size_t counter, next, prev, emit, removed, wt, vinfo, tail, total;
};

int sm_count() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) {
    cudaGetLastError();
    return 148;  // B200
  }
  return sms;
}

// Global tails of the fast kernel's running entries: every warp that can be
// resident (<= 64 per SM) owns 5 fields x m instances x
// (rcap - 1) slots (the smallest shared head is one entry).
size_t run_tail_ints(const rs_batch_cfg& c, int64_t num_replays) {
  const int rcap = run_cap(c);
  if (c.chunk_size != 0 || c.num_instances > 64 || rcap <= 1) return 0;
  // (a launch may round the replay count up to whole blocks of <= 16 warps,
  // and any warp can take any replay from the work counter)
  // (two warps per replay for m > 32: pair.cuh)
  const int64_t warps = std::min<int64_t>(2 * num_replays + 32, (int64_t)sm_count() * 64);
  return (size_t)warps * 5 * c.num_instances * (rcap - 1);
}

size_t rl_param_count(const rs_batch_cfg& c) {
  if (c.policy != RS_POLICY_RL) return 0;
  size_t w = 0;
  for (int l = 0; l < c.rl_num_layers; ++l)
    w += (size_t)c.rl_dims[l] * c.rl_dims[l + 1] + c.rl_dims[l + 1];
  return w;
}

WsLayout ws_layout(int64_t total_requests, int64_t num_replays, size_t rl_params = 0,
                   size_t tail_ints = 0) {
  WsLayout w;
  size_t off = 0;
  w.wt = off;  // transposed Q-network (global-weights mode), may be empty
  off = align_up(off + rl_params * sizeof(double), 256);
  w.counter = off;
  off = align_up(off + 256, 256);
  w.next = off;
  off = align_up(off + 4ull * total_requests, 256);
  w.prev = off;
  off = align_up(off + 4ull * total_requests, 256);
  w.emit = off;
  off = align_up(off + 4ull * total_requests, 256);
  w.removed = off;
  off = align_up(off + (size_t)total_requests, 256);
  w.vinfo = off;
  off = align_up(off + 8ull * (size_t)num_replays, 256);
  w.tail = off;
  off = align_up(off + 4ull * tail_ints, 256);
  w.total = off;
  return w;
}

// Per-device caches of the planner's kernel queries: the dynamic shared-memory
// opt-in of a kernel only ever rises, and the occupancy of (kernel, block,
// bytes) is fixed, so repeated calls do not repeat the driver round trips.
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, int> g_smem_set;
std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;

cudaError_t set_smem(const void* k, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(g_attr_mu);
  int& cur = g_smem_set[{dev, k}];
  if (cur >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

cudaError_t occ_blocks(int* out, const void* k, int threads, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(g_attr_mu);
  const auto key = std::make_tuple(dev, k, threads, bytes);
  const auto it = g_occ.find(key);
  if (it != g_occ.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, threads, bytes);
  if (e == cudaSuccess) g_occ[key] = *out;
  return e;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <typename K>
rs_status launch_kernel(K kern, const rs::KParams& kp, int wpb, int groups_per_warp,
                        int block_smem, int num_replays, cudaStream_t st) {
  RS_CUDA(set_smem((const void*)kern, block_smem));
  int dev = 0, sms = 0, per_sm = 0;
  RS_CUDA(cudaGetDevice(&dev));
  RS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RS_CUDA(occ_blocks(&per_sm, (const void*)kern, wpb * rs::kWarp, block_smem));
  if (per_sm < 1) return fail(RS_ERR_UNSUPPORTED, "replay kernel does not fit on an SM");
  const int per_block = wpb * groups_per_warp;
  const int want = (num_replays + per_block - 1) / per_block;
  const int grid = std::max(1, std::min(want, sms * per_sm));
  kern<<<grid, wpb * rs::kWarp, block_smem, st>>>(kp);
  RS_CUDA(cudaGetLastError());
  return RS_OK;
}

using KernelFn = void (*)(rs::KParams);

}  // namespace

// One translation unit per policy (generated by build.py, compiled in
// parallel) instantiates that policy's general and fast replay kernels.
namespace rs {
using KernelFn = void (*)(KParams);
KernelFn kernel_for_0_0(bool fast, int groups, int width, int variant);
KernelFn kernel_for_0_1(bool fast, int groups, int width, int variant);
KernelFn kernel_for_1_0(bool fast, int groups, int width, int variant);
KernelFn kernel_for_1_1(bool fast, int groups, int width, int variant);
KernelFn kernel_for_2_0(bool fast, int groups, int width, int variant);
KernelFn kernel_for_2_1(bool fast, int groups, int width, int variant);
KernelFn kernel_for_3_0(bool fast, int groups, int width, int variant);
KernelFn kernel_for_3_1(bool fast, int groups, int width, int variant);
KernelFn kernel_for_4_0(bool fast, int groups, int width, int variant);
KernelFn kernel_for_4_1(bool fast, int groups, int width, int variant);
KernelFn kernel_for_5_0(bool fast, int groups, int width, int variant);
KernelFn kernel_for_5_1(bool fast, int groups, int width, int variant);
KernelFn kernel_for_6_0(bool fast, int groups, int width, int variant);
KernelFn kernel_for_6_1(bool fast, int groups, int width, int variant);
KernelFn kernel_for_7_0(bool fast, int groups, int width, int variant);
KernelFn kernel_for_7_1(bool fast, int groups, int width, int variant);
KernelFn kernel_for_8_0(bool fast, int groups, int width, int variant);
KernelFn kernel_for_8_1(bool fast, int groups, int width, int variant);
}  // namespace rs

namespace {

KernelFn kernel_for(int policy, bool fast, int groups, int width, int variant = 0,
                    bool tail = false) {
  switch (policy * 2 + (tail ? 1 : 0)) {
    case 0: return rs::kernel_for_0_0(fast, groups, width, variant);
    case 1: return rs::kernel_for_0_1(fast, groups, width, variant);
    case 2: return rs::kernel_for_1_0(fast, groups, width, variant);
    case 3: return rs::kernel_for_1_1(fast, groups, width, variant);
    case 4: return rs::kernel_for_2_0(fast, groups, width, variant);
    case 5: return rs::kernel_for_2_1(fast, groups, width, variant);
    case 6: return rs::kernel_for_3_0(fast, groups, width, variant);
    case 7: return rs::kernel_for_3_1(fast, groups, width, variant);
    case 8: return rs::kernel_for_4_0(fast, groups, width, variant);
    case 9: return rs::kernel_for_4_1(fast, groups, width, variant);
    case 10: return rs::kernel_for_5_0(fast, groups, width, variant);
    case 11: return rs::kernel_for_5_1(fast, groups, width, variant);
    case 12: return rs::kernel_for_6_0(fast, groups, width, variant);
    case 13: return rs::kernel_for_6_1(fast, groups, width, variant);
    case 14: return rs::kernel_for_7_0(fast, groups, width, variant);
    case 15: return rs::kernel_for_7_1(fast, groups, width, variant);
    case 16: return rs::kernel_for_8_0(fast, groups, width, variant);
    case 17: return rs::kernel_for_8_1(fast, groups, width, variant);
  }
  return nullptr;
}

}  // namespace

namespace rs {
void set_error(const std::string& m) { g_err = m; }
}  // namespace rs

extern "C" {

uint32_t rs_abi_version(void) { return RS_ABI_VERSION; }

int32_t rs_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int ok = 0;
  for (int d = 0; d < n; ++d) ok += device_ok(d) ? 1 : 0;
  return ok;
}

rs_status rs_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return RS_ERR_INVALID_ARGUMENT;
  std::snprintf(buf, len, "%s", g_err.c_str());
  return RS_OK;
}

uint64_t rs_mix_seed(uint64_t seed, uint64_t stream) {  // rng.hpp:11-16
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

int64_t rs_heavy_decode_cutoff(const rs_profile* p, const rs_thresholds* t) {
  if (!p || !t) return -1;
  return heavy_cutoff(*p, *t);
}

rs_status rs_default_config(rs_batch_cfg* c) {
  if (!c) return fail(RS_ERR_INVALID_ARGUMENT, "null config");
  std::memset(c, 0, sizeof(*c));
  c->abi_version = RS_ABI_VERSION;
  c->policy = RS_POLICY_ROUND_ROBIN;
  c->profile = rs_profile{3.2e-4, 0.026, 3.3e-5, 0.0167};   // latency.hpp:17-20
  c->thresholds = rs_thresholds{0.5, 5.0};                  // latency.hpp:39-40
  c->impact = rs_impact{3.2e-4, 3.3e-5, 0.5, 0.5, 2, 0};    // impact.hpp:15-19
  c->kv_capacity_tokens = 16384;                            // instance.hpp:38-41
  c->max_batch_size = 128;
  c->batching = RS_BATCHING_FCFS;
  c->chunk_size = 0;
  c->num_instances = 4;                                     // experiment.hpp:52-53
  c->delta_t = 0.02;
  c->n_predictor_edges = 4;                                 // predictor.hpp:55
  const int64_t pe[4] = {0, 250, 1000, 4000};
  std::memcpy(c->predictor_edges, pe, sizeof(pe));
  c->n_state_edges = 3;                                     // predictor.hpp:59
  const int64_t se[3] = {0, 256, 2048};
  std::memcpy(c->state_edges, se, sizeof(se));
  c->predictor_top_cap = 4096;                              // workload.hpp:23
  c->predictor_mode = RS_PREDICTOR_SIMULATED;
  const double acc[5] = {0.9310, 0.7036, 0.7992, 0.6527, 0.9506};  // workload.hpp:165-174
  std::memcpy(c->accuracy, acc, sizeof(acc));
  c->n_band_edges = 7;                                      // predictor.hpp:162-164
  const int64_t be[7] = {0, 32, 64, 128, 256, 512, 1024};
  std::memcpy(c->band_edges, be, sizeof(be));
  c->max_ticks = 10000000;                                  // env.hpp:326
  return RS_OK;
}

rs_status rs_validate_config(const rs_batch_cfg* cfg) { return validate(cfg); }

rs_status rs_workspace_size(const rs_batch_cfg* cfg, int32_t num_replays,
                            int64_t total_requests, size_t* bytes) {
  rs_status s = validate(cfg);
  if (s != RS_OK) return s;
  if (!bytes || num_replays < 0 || total_requests < 0)
    return fail(RS_ERR_INVALID_ARGUMENT, "bad workspace query");
  *bytes = ws_layout(total_requests, num_replays, rl_param_count(*cfg),
                     run_tail_ints(*cfg, num_replays)).total;
  return RS_OK;
}

void* rs_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    g_err = "cudaHostAlloc failed";
    return nullptr;
  }
  return p;
}

void rs_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

rs_status rs_predict_buckets(const rs_batch_cfg* cfg, const rs_trace_soa* tr,
                             uint8_t* predicted_bucket, void* stream) {
  rs_status s = validate(cfg);
  if (s != RS_OK) return s;
  if ((s = require_device()) != RS_OK) return s;
  if (!tr || !predicted_bucket) return fail(RS_ERR_INVALID_ARGUMENT, "null trace/output");
  if (tr->num_replays == 0) return RS_OK;
  if (cfg->predictor_mode == RS_PREDICTOR_GIVEN && !tr->given_bucket)
    return fail(RS_ERR_INVALID_ARGUMENT, "GIVEN predictor mode needs trace->given_bucket");
  if (cfg->predictor_mode == RS_PREDICTOR_SIMULATED && !tr->predictor_seed)
    return fail(RS_ERR_INVALID_ARGUMENT, "simulated predictor needs trace->predictor_seed");
  rs::PredParams pp;
  std::memset(&pp, 0, sizeof(pp));
  std::memcpy(pp.accuracy, cfg->accuracy, sizeof(pp.accuracy));
  pp.n_pred_edges = cfg->n_predictor_edges;
  for (int i = 0; i < cfg->n_predictor_edges; ++i) pp.pred_edges[i] = (int)cfg->predictor_edges[i];
  pp.n_band_edges = cfg->n_band_edges;
  for (int i = 0; i < cfg->n_band_edges && i < RS_MAX_BANDS; ++i) pp.band_edges[i] = (int)cfg->band_edges[i];
  std::memcpy(pp.emp_table, cfg->empirical_table, sizeof(pp.emp_table));
  pp.mode = cfg->predictor_mode;
  pp.num_replays = tr->num_replays;
  pp.offsets = reinterpret_cast<const long long*>(tr->offsets);
  pp.prompt = tr->prompt_tokens;
  pp.decode = tr->decode_tokens;
  pp.task = tr->task;
  pp.given = tr->given_bucket;
  pp.seeds = tr->predictor_seed;
  pp.out = predicted_bucket;
  int dev = 0, sms = 0;
  RS_CUDA(cudaGetDevice(&dev));
  RS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks_needed = (tr->num_replays + rs::kPredWarpsPerBlock - 1) / rs::kPredWarpsPerBlock;
  const int grid = std::max(1, std::min(blocks_needed, sms * 8));
  rs::predict_kernel<<<grid, rs::kWarp * rs::kPredWarpsPerBlock, 0, (cudaStream_t)stream>>>(pp);
  RS_CUDA(cudaGetLastError());
  return RS_OK;
}

rs_status rs_replay_batch(const rs_batch_cfg* cfg, const rs_trace_soa* tr, rs_req_out* out,
                          rs_replay_stats* stats, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (cfg && (cfg->flags & RS_FLAG_RECORD_TRAJECTORY))
    return fail(RS_ERR_INVALID_ARGUMENT, "record_trajectory: use rs_replay_trajectory");
  return rs_internal_replay_batch(cfg, tr, out, stats, workspace, workspace_bytes, stream,
                                  nullptr, nullptr, nullptr);
}

rs_status rs_replay_trajectory(const rs_batch_cfg* cfg, const rs_trace_soa* tr, rs_req_out* out,
                               rs_replay_stats* stats, const rs_trajectory* traj,
                               void* workspace, size_t workspace_bytes, void* stream) {
  if (!cfg || !traj) return fail(RS_ERR_INVALID_ARGUMENT, "null config/trajectory");
  if (traj->capacity < 0) return fail(RS_ERR_INVALID_ARGUMENT, "trajectory capacity < 0");
  // RewardConfig::validate (env.hpp:46-52)
  if (!(traj->r_w > 0.0)) return fail(RS_ERR_INVALID_ARGUMENT, "reward: r_w must be > 0");
  if (!(traj->gamma >= 0.0 && traj->gamma < 1.0))
    return fail(RS_ERR_INVALID_ARGUMENT, "reward: gamma outside [0, 1)");
  if (!(traj->beta_d > 0.0)) return fail(RS_ERR_INVALID_ARGUMENT, "reward: beta_d must be > 0");
  if (traj->shaping < RS_SHAPING_NONE || traj->shaping > RS_SHAPING_GUIDED)
    return fail(RS_ERR_INVALID_ARGUMENT, "unknown shaping mode");
  rs_batch_cfg c = *cfg;
  c.flags |= RS_FLAG_RECORD_TRAJECTORY;
  return rs_internal_replay_batch(&c, tr, out, stats, workspace, workspace_bytes, stream,
                                  nullptr, nullptr, traj);
}

}  // extern "C"

// Streamed-input variant (used by rs_replay_batch_host): requests
// [0, *resident) of every replay are on the device, the rest still in flight
// on a copy stream that bumps *resident; the lane-per-instance kernel gates
// each 32-request arrival window on it. `inputs_done` (recorded by the copy
// stream after its last chunk) orders the percentile pass after the copies.
bool rs_internal_fast_path(const rs_batch_cfg* cfg) {
  return cfg->chunk_size == 0 && cfg->num_instances <= 64 &&
         env_int("RS_FORCE_GENERAL", 0) == 0;
}

rs_status rs_internal_replay_batch(const rs_batch_cfg* cfg, const rs_trace_soa* tr,
                                   rs_req_out* out, rs_replay_stats* stats, void* workspace,
                                   size_t workspace_bytes, void* stream, const int* resident,
                                   void* inputs_done, const rs_trajectory* traj,
                                   rs_internal_stream_out* sout) {
  rs_status s = validate(cfg);
  if (s != RS_OK) return s;
  if ((s = require_device()) != RS_OK) return s;
  if (!tr || !out || !stats) return fail(RS_ERR_INVALID_ARGUMENT, "null trace/out/stats");
  if (tr->num_replays < 0) return fail(RS_ERR_INVALID_ARGUMENT, "num_replays < 0");
  if (tr->num_replays == 0) return RS_OK;
  if (!out->instance || !out->routed_s || !out->first_token_s || !out->completion_s ||
      !out->preemptions || !out->predicted_bucket)
    return fail(RS_ERR_INVALID_ARGUMENT, "rs_replay_batch needs every per-request output array");
  if (cfg->policy == RS_POLICY_RL && cfg->rl_epsilon > 0.0 && !tr->policy_seed)
    return fail(RS_ERR_INVALID_ARGUMENT, "epsilon-greedy needs trace->policy_seed");
  const WsLayout wl = ws_layout(tr->total_requests, tr->num_replays, rl_param_count(*cfg),
                                run_tail_ints(*cfg, tr->num_replays));
  if (!workspace || workspace_bytes < wl.total)
    return fail(RS_ERR_INVALID_ARGUMENT, "workspace too small (rs_workspace_size)");
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = static_cast<char*>(workspace);

  // shared waiting-ring slots per instance (the rest of a long queue lives
  // in the global overflow list): smaller rings for larger fleets keep
  // several replays resident per SM
  const int m_inst = cfg->num_instances;
  const int wdef = m_inst <= 16 ? 64 : (m_inst <= 32 ? 32 : 16);
  int wcap = std::max(8, std::min(128, env_int("RS_WAIT_RING", wdef)));
  // whole-prompt prefill (no chunking, m <= 64) takes the lane-per-instance
  // kernel; chunked prefill and larger fleets take the general kernel
  const bool fast = rs_internal_fast_path(cfg) && !traj;
  if ((resident || sout) && !fast)
    return fail(RS_ERR_INVALID_ARGUMENT, "streamed inputs / outputs need the lane-per-instance kernel");
  if (sout && (sout->nbounds < 1 || sout->nbounds > 16 || !sout->marks))
    return fail(RS_ERR_INVALID_ARGUMENT, "streamed outputs: 1..16 chunks");
  const int groups = m_inst <= 32 ? 1 : 2;
  bool fused = true;  // the simulated predictor inside the replay kernel
  Layout L = make_layout(*cfg, wcap, fast);
  {
    // Throughput regime (more replays than ~16 per SM, the register limit):
    // resident replays per SM are bounded by shared memory, so shrink the
    // waiting ring (longer queues spill to the global overflow list) until
    // 16 replays fit per SM, or the ring is down to 8 slots.
    int dev0 = 0, sms0 = 0;
    RS_CUDA(cudaGetDevice(&dev0));
    RS_CUDA(cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0));
    const int target = std::min<long long>(16, ((long long)tr->num_replays + sms0 - 1) / sms0);
    auto per_sm = [&](const Layout& Lx) {
      int best = 0;
      const int wmax = cfg->policy == RS_POLICY_RL ? 16 : 8;
      for (int wpb = 1; wpb <= wmax; ++wpb) {
        const long long bytes = (long long)Lx.weights_bytes + (long long)wpb * Lx.group_bytes;
        const int blocks = std::min<long long>(32 / wpb, (228 * 1024) / (bytes + 1024));
        best = std::max(best, blocks * wpb);
      }
      return std::min(best, 16);
    };
    // Shrink the per-replay shared state until `target` replays fit per SM:
    // first the waiting ring (longer queues continue in the global overflow
    // list), then the running head to 32 entries (typical batches are 8-12,
    // measured max 27: the global tail is rarely touched; the tail build of
    // the kernel is used), then the fused predictor's 2.5 KB mt19937_64
    // block (the predictions are drawn by the predict_kernel pre-pass
    // instead; resident inputs only), then the head to 16.  RS_RUN_SMEM /
    // RS_WAIT_RING pin either (tests).
    const int rsm_env = env_int("RS_RUN_SMEM", 0);
    const bool ring_env = getenv("RS_WAIT_RING") != nullptr;
    const bool can_unfuse = !resident && (cfg->flags & RS_FLAG_PREDICT_INLINE) &&
                            cfg->predictor_mode == RS_PREDICTOR_SIMULATED;
    int rsm = rsm_env > 0 ? rsm_env : L.rcap;
    L = make_layout(*cfg, wcap, fast, rsm, fused);
    // RL: the waiting ring stops at 16 slots (a saturated fleet under an
    // untrained agent queues deep; measured c3 675 -> 642 ms against 8 slots
    // and a 32-entry running head, same box)
    const int wmin = cfg->policy == RS_POLICY_RL ? 16 : 8;
    while (fast && per_sm(L) < target) {
      if (!ring_env && wcap > wmin) wcap >>= 1;
      else if (!rsm_env && rsm > 32) rsm = 32;
      else if (can_unfuse && fused) fused = false;
      else if (!rsm_env && rsm > 16) rsm = 16;
      else break;
      L = make_layout(*cfg, wcap, fast, rsm, fused);
    }
  }
  rs::KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  const rs_profile& p = cfg->profile;
  kp.tpp = p.prompt_time_per_token;
  kp.intercept = p.prompt_time_intercept;
  kp.dpt = p.decode_time_per_token;
  kp.dtb = p.decode_time_base;
  kp.delta_t = cfg->delta_t;
  kp.grad1 = cfg->impact.grad1;
  kp.grad2 = cfg->impact.grad2;
  kp.eps_s = cfg->impact.epsilon_s;
  kp.alpha = cfg->impact.alpha;
  kp.rl_eps = cfg->rl_epsilon;
  std::memcpy(kp.accuracy, cfg->accuracy, sizeof(kp.accuracy));
  kp.prompt_exp = cfg->impact.prompt_exponent;
  kp.kv_cap = (int)cfg->kv_capacity_tokens;
  kp.max_batch = cfg->max_batch_size;
  kp.batching = cfg->batching;
  kp.chunk = cfg->chunk_size;
  kp.m = cfg->num_instances;
  kp.n_state_edges = cfg->n_state_edges;
  kp.n_pred_edges = cfg->n_predictor_edges;
  for (int i = 0; i < cfg->n_state_edges; ++i) kp.state_edges[i] = (int)cfg->state_edges[i];
  for (int i = 0; i < cfg->n_predictor_edges; ++i) {
    kp.pred_edges[i] = (int)cfg->predictor_edges[i];
    kp.ub[i] = (int)ub_of(*cfg, i);
  }
  kp.n_band_edges = cfg->n_band_edges;
  for (int i = 0; i < cfg->n_band_edges && i < RS_MAX_BANDS; ++i)
    kp.band_edges[i] = (int)cfg->band_edges[i];
  std::memcpy(kp.emp_table, cfg->empirical_table, sizeof(kp.emp_table));  // fused predictor
  kp.predictor_mode = cfg->predictor_mode;
  kp.rcap = L.rcap;
  kp.wcap = L.wcap;
  kp.dsl_cutoff = (int)std::min<int64_t>(INT_MAX, heavy_cutoff(cfg->profile, cfg->thresholds));
  kp.flags = cfg->flags;
  kp.max_ticks = cfg->max_ticks;
  kp.rl_layers = cfg->policy == RS_POLICY_RL ? cfg->rl_num_layers : 0;
  for (int i = 0; i <= RS_MAX_LAYERS; ++i) kp.rl_dims[i] = cfg->rl_dims[i];
  for (int i = 0; i < RS_MAX_LAYERS; ++i) {
    kp.rl_woff[i] = L.woff[i];
    kp.rl_boff[i] = L.boff[i];
  }
  kp.rl_w = cfg->rl_params;
  kp.rl_maxw = L.maxw;
  kp.smem_weights_bytes = L.weights_bytes;
  kp.num_replays = tr->num_replays;
  kp.offsets = reinterpret_cast<const long long*>(tr->offsets);
  kp.arrival = tr->arrival_s;
  kp.prompt = tr->prompt_tokens;
  kp.decode = tr->decode_tokens;
  kp.task = tr->task;
  kp.bucket = out->predicted_bucket;
  kp.policy_seed = tr->policy_seed;
  kp.o_instance = out->instance;
  kp.o_routed = out->routed_s;
  kp.o_first = out->first_token_s;
  kp.o_completion = out->completion_s;
  kp.o_preempt = out->preemptions;
  kp.o_pred = out->predicted_bucket;
  kp.stats = stats;
  kp.ov_next = reinterpret_cast<uint32_t*>(ws + wl.next);
  kp.ov_prev = reinterpret_cast<uint32_t*>(ws + wl.prev);
  kp.ov_emit = reinterpret_cast<int*>(ws + wl.emit);
  kp.mm_removed = reinterpret_cast<uint8_t*>(ws + wl.removed);
  kp.work_counter = reinterpret_cast<int*>(ws + wl.counter);
  kp.smem_group_bytes = L.group_bytes;
  kp.off_run = L.off_run;
  kp.off_wait = L.off_wait;
  kp.off_dbc = L.off_dbc;
  kp.off_rlx = L.off_rlx;
  kp.off_rng = L.off_rng;
  kp.off_front = L.off_front;
  kp.off_pred = L.off_pred;
  kp.off_pair = L.off_pair;
  kp.predictor_seed = tr->predictor_seed;
  kp.given_bucket = tr->given_bucket;
  kp.resident = resident;
  if (sout) sout->used = 0;
  if (traj) {  // ClusterConfig::record_trajectory (general kernel)
    kp.traj = *traj;
    kp.traj_on = 1;
    kp.traj_scan = (traj->queue_penalty || traj->reward) ? 1 : 0;
    kp.r_w = traj->r_w;
    // RewardConfig::shaping_coefficient(episode_k) (env.hpp:55-63), host libm
    kp.c_k = traj->shaping == RS_SHAPING_NONE       ? 0.0
             : traj->shaping == RS_SHAPING_ADDITIVE ? 1.0
                                                    : traj->gamma * std::exp(-traj->beta_d *
                                                                             static_cast<double>(
                                                                                 traj->episode_k));
  }
  if (cfg->flags & RS_FLAG_PREDICT_INLINE) {
    if (cfg->predictor_mode == RS_PREDICTOR_SIMULATED && !tr->predictor_seed)
      return fail(RS_ERR_INVALID_ARGUMENT, "simulated predictor needs trace->predictor_seed");
    if (cfg->predictor_mode == RS_PREDICTOR_GIVEN && !tr->given_bucket)
      return fail(RS_ERR_INVALID_ARGUMENT, "GIVEN predictor mode needs trace->given_bucket");
    if (fast && fused) {
      kp.predict_inline = 1;  // drawn at injection inside the replay kernel
    } else {  // a pre-pass kernel writes every prediction
      rs_status sp = rs_predict_buckets(cfg, tr, out->predicted_bucket, stream);
      if (sp != RS_OK) return sp;
    }
  }
  {  // fast-kernel word offsets (fast.cuh RQ/RP/.../WE accessors)
    const int m = cfg->num_instances;
    kp.rsm = L.rsm;
    kp.rtail = L.rcap - L.rsm;
    kp.run_tail = kp.rtail > 0 ? reinterpret_cast<int*>(ws + wl.tail) : nullptr;
    kp.rstride = L.rsm | 1;
    kp.f_rreq = L.off_run / 4;
    kp.f_rprompt = kp.f_rreq + m * kp.rstride;
    kp.f_rdhat = kp.f_rprompt + m * kp.rstride;
    kp.f_rtrue = kp.f_rdhat + m * kp.rstride;
    kp.f_rkey = kp.f_rtrue + m * kp.rstride;
    kp.f_wreq = L.off_wait / 4;
    kp.f_wprompt = kp.f_wreq + m * L.wcap;
    kp.f_wdhat = kp.f_wprompt + m * L.wcap;
    kp.f_wtrue = kp.f_wdhat + m * L.wcap;
    kp.f_wemit = kp.f_wtrue + m * L.wcap;
    kp.mwidth = 1;
    while (kp.mwidth < m && kp.mwidth < rs::kWarp) kp.mwidth <<= 1;
  }
  {  // power-of-two divisors -> exact reciprocal multiplies
    auto pow2 = [](double c, double* inv) {
      int e = 0;
      const double f = std::frexp(c, &e);
      *inv = 1.0 / c;
      return (f == 0.5 && e > -1000 && e < 1000) ? 1 : 0;
    };
    kp.eps_pow2 = pow2(cfg->impact.epsilon_s, &kp.inv_eps);
    kp.kv_pow2 = pow2((double)cfg->kv_capacity_tokens, &kp.inv_kv);
    kp.mb_pow2 = pow2((double)cfg->max_batch_size, &kp.inv_mb);
  }

  // warps (replays) per block: maximise resident warps per SM; the RL
  // weights are staged once per block, which favours wider blocks.
  int dev = 0;
  RS_CUDA(cudaGetDevice(&dev));
  int smem_optin = 0;
  RS_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int smem_sm = 228 * 1024;
  // Q-networks that leave fewer than 4 replay slots per SM next to their
  // staged weights, or with a layer wider than the shared-memory forward's
  // masks, run from a transposed copy in global memory (L2-resident).
  int max_dim = 0;
  for (int l = 0; l <= cfg->rl_num_layers && cfg->policy == RS_POLICY_RL; ++l)
    max_dim = std::max(max_dim, cfg->rl_dims[l]);
  const bool rl_global = cfg->policy == RS_POLICY_RL &&
                         (env_int("RS_RL_GLOBAL", 0) != 0 || max_dim > rs::kMlpSmemMaxWidth ||
                          L.weights_bytes + 4 * L.group_bytes > smem_optin);
  if (rl_global) {
    double* wt = reinterpret_cast<double*>(ws + wl.wt);
    const size_t np = rl_param_count(*cfg);
    rs::MlpTransposeArgs ta;
    ta.params = cfg->rl_params;
    ta.layers = cfg->rl_num_layers;
    for (int l = 0; l <= RS_MAX_LAYERS; ++l) ta.dims[l] = cfg->rl_dims[l];
    for (int l = 0; l < RS_MAX_LAYERS; ++l) {
      ta.woff[l] = L.woff[l];
      ta.boff[l] = L.boff[l];
    }
    ta.out = wt;
    ta.count = np;
    rs::mlp_transpose_kernel<0><<<(unsigned)((np + 255) / 256), 256, 0, st>>>(ta);
    RS_CUDA(cudaGetLastError());
    kp.rl_wt_global = wt;
    kp.smem_weights_bytes = 0;
    L.weights_bytes = 0;
  }
  // Launch plan for a lane-group width W (32/W replays per warp): warps
  // per block maximising resident replays per SM (registers via the
  // occupancy calculator, shared memory per replay slot; the RL weights are
  // staged once per block, which favours wider blocks).
  int sms = 0;
  RS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const bool tail = fast && L.rsm < L.rcap;  // the build with the global running tail
  const int wpb_env = env_int("RS_WARPS_PER_BLOCK", 0);
  struct Plan {
    int width = 0, wpb = 0, per_sm = 0, block_smem = 0;
    long long capacity = 0;  // resident replays on the device
    KernelFn kern = nullptr;
  };
  auto plan_for = [&](int width) -> Plan {
    Plan pl;
    pl.width = width;
    pl.kern = kernel_for(cfg->policy, fast, groups, width, 0, tail);
    if (!pl.kern) return pl;
    KernelFn wide = kernel_for(cfg->policy, fast, groups, width, 1, tail);
    const int gpw = rs::kWarp / width;
    // the wide RL instantiation takes blocks of up to 16 warps
    const int max_wpb = wide ? 16 : 8;
    KernelFn narrow = pl.kern;
    for (int wpb = max_wpb; wpb >= 1; --wpb) {
      if (wpb_env && wpb > wpb_env) continue;  // RS_WARPS_PER_BLOCK: an upper bound
      // wide RL blocks only in whole multiples of the 4 SM sub-partitions:
      // 9 warps would put 3 replays on one scheduler and 2 on the others,
      // and the slowest scheduler's replays set the tail (measured on c3)
      if (wpb > 8 && (wpb & 3)) continue;
      const long long bytes = L.weights_bytes + (long long)wpb * gpw * L.group_bytes;
      if (bytes > smem_optin) continue;
      KernelFn k = wpb > 8 ? wide : narrow;
      if (set_smem((const void*)k, (int)bytes) !=
          cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      int per_sm = 0;
      if (occ_blocks(&per_sm, (const void*)k, wpb * rs::kWarp,
                                                        (size_t)bytes) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      per_sm = std::min(per_sm, (int)(smem_sm / (bytes + 1024)));
      const long long cap = (long long)sms * per_sm * wpb * gpw;
      if (cap > pl.capacity) {
        pl.kern = k;
        pl.capacity = cap;
        pl.wpb = wpb;
        pl.per_sm = per_sm;
        pl.block_smem = (int)bytes;
      }
    }
    return pl;
  };
  const int width = rs::kWarp;  // one replay per warp
  Plan pl = plan_for(width);
  if (!pl.kern) return fail(RS_ERR_INVALID_ARGUMENT, "unknown policy");
  if (pl.wpb == 0)
    return fail(RS_ERR_UNSUPPORTED, "per-replay shared-memory state exceeds one SM (" +
                                        std::to_string(L.weights_bytes + L.group_bytes) + " B)");
  // When every replay fits in one wave of whole-warp groups, the kernel time
  // is the slowest warp's: spread the replays evenly, ceil(R / #SMs) warps
  // per SM (one block per SM when that is <= 8 warps), instead of packing
  // some SMs.
  if (pl.width == rs::kWarp && !wpb_env) {
    const int need = (tr->num_replays + sms - 1) / std::max(1, sms);
    if (need <= pl.per_sm * pl.wpb && need <= 8) {
      for (int wpb = need; wpb >= 1; --wpb) {
        if (L.weights_bytes + wpb * L.group_bytes <= smem_optin) {
          pl.wpb = wpb;
          pl.block_smem = L.weights_bytes + wpb * L.group_bytes;
          pl.kern = kernel_for(cfg->policy, fast, groups, pl.width, 0, tail);  // <= 8 warps
          // one block per SM: the uncapped-register build, when it fits
          KernelFn lat = env_int("RS_NO_LAT_KERNEL", 0) ? nullptr
                                                         : kernel_for(cfg->policy, fast, groups,
                                                                      pl.width, 2, tail);
          int lat_blocks = 0;
          if (lat &&
              set_smem((const void*)lat, pl.block_smem) == cudaSuccess &&
              occ_blocks(&lat_blocks, (const void*)lat, wpb * rs::kWarp,
                                                            (size_t)pl.block_smem) == cudaSuccess &&
              lat_blocks >= 1)
            pl.kern = lat;
          cudaGetLastError();
          break;
        }
      }
    }
  }
  // Shared memory already limits the plan to one block of <= 8 warps per SM
  // (e.g. the RL kernel with its staged Q-network): the register file is
  // not the constraint, so take the uncapped-register build there too.
  if (pl.width == rs::kWarp && pl.per_sm == 1 && pl.wpb <= 8 && pl.kern ==
      kernel_for(cfg->policy, fast, groups, pl.width, 0, tail) && !env_int("RS_NO_LAT_KERNEL", 0)) {
    KernelFn lat = kernel_for(cfg->policy, fast, groups, pl.width, 2, tail);
    int lat_blocks = 0;
    if (lat &&
        set_smem((const void*)lat, pl.block_smem) ==
            cudaSuccess &&
        occ_blocks(&lat_blocks, (const void*)lat, pl.wpb * rs::kWarp,
                                                      (size_t)pl.block_smem) == cudaSuccess &&
        lat_blocks >= 1)
      pl.kern = lat;
    cudaGetLastError();
  }
  // Streamed outputs: the latency-regime plan has a publishing build
  // (replay_fast_kernel_lat_so); other plans copy the outputs after the kernel.
  if (sout && !tail) {
    KernelFn lat = kernel_for(cfg->policy, fast, groups, pl.width, 2, tail);
    KernelFn lso = kernel_for(cfg->policy, fast, groups, pl.width, 3, tail);
    int blocks = 0;
    if (lat && lso && pl.kern == lat &&
        set_smem((const void*)lso, pl.block_smem) ==
            cudaSuccess &&
        occ_blocks(&blocks, (const void*)lso, pl.wpb * rs::kWarp,
                                                      (size_t)pl.block_smem) == cudaSuccess &&
        blocks >= 1) {
      pl.kern = lso;
      kp.out_marks = sout->marks;
      kp.n_out_bounds = sout->nbounds;
      for (int c = 0; c < sout->nbounds; ++c) kp.out_bounds[c] = sout->bounds[c];
      sout->used = 1;
    }
    cudaGetLastError();
  }
  if (env_int("RS_DEBUG_PLAN", 0)) {
    const char* variant = !fast                                                ? "general"
                          : pl.kern == kernel_for(cfg->policy, fast, groups, pl.width, 2, tail) ? "lat"
                          : pl.kern == kernel_for(cfg->policy, fast, groups, pl.width, 1, tail) ? "wide"
                          : (sout && sout->used)                                          ? "lat_so"
                                                                                        : "bounded";
    fprintf(stderr,
            "rs plan: policy %d fast %d kernel %s groups %d width %d wpb %d blocks/SM %d "
            "block_smem %d group_bytes %d weights %d wcap %d rsm %d fused_pred %d rl_global %d "
            "resident replays %lld\n",
            cfg->policy, (int)fast, variant, groups, pl.width, pl.wpb, pl.per_sm, pl.block_smem,
            L.group_bytes, L.weights_bytes, L.wcap, L.rsm, (int)fused, (int)rl_global,
            pl.capacity);
  }
  RS_CUDA(cudaMemsetAsync(kp.work_counter, 0, sizeof(int), st));
  if (fast && !resident && env_int("RS_NO_VALIDATE_PASS", 0) == 0) {
    // resident inputs: validation + preemption-counter zeroing as one
    // parallel pass instead of a serial walk per replay warp
    rs::ValidateParams vp;
    vp.num_replays = tr->num_replays;
    vp.offsets = kp.offsets;
    vp.arrival = kp.arrival;
    vp.prompt = kp.prompt;
    vp.decode = kp.decode;
    vp.o_preempt = kp.o_preempt;
    vp.mm_removed = cfg->policy == RS_POLICY_MIN_MIN ? kp.mm_removed : nullptr;
    vp.o_completion = nullptr;
    vp.vinfo = reinterpret_cast<int2*>(ws + wl.vinfo);
    const int vgrid = std::max(1, std::min(tr->num_replays, sms * 8));
    rs::validate_kernel<<<vgrid, rs::kStatsThreads, 0, st>>>(vp);
    RS_CUDA(cudaGetLastError());
    kp.vinfo = vp.vinfo;
  }
  // Fleets of 33..64 instances: two warps per replay, one instance per lane
  // (pair.cuh), when the heuristic has a pair build.  Pairs per block: all
  // replays resident in one wave when they fit, <= 8 pairs (16 warps) per
  // block.
  KernelFn pk = nullptr;
  int ppb = 0, pair_blocks = 0;
  if (fast && groups == 2 && !(sout && sout->used) && !traj &&
      env_int("RS_NO_PAIR", 0) == 0)
    pk = kernel_for(cfg->policy, fast, groups, rs::kWarp, 4, tail);
  if (pk) {
    const int want = std::max(1, std::min(8, (tr->num_replays + sms - 1) / sms));
    for (ppb = want; ppb >= 1; --ppb) {
      const int bytes = ppb * L.group_bytes;
      if (bytes > smem_optin) continue;
      if (set_smem((const void*)pk, bytes) !=
              cudaSuccess ||
          occ_blocks(&pair_blocks, (const void*)pk, 64 * ppb,
                                                        (size_t)bytes) != cudaSuccess) {
        cudaGetLastError();
        pair_blocks = 0;
        continue;
      }
      if (pair_blocks >= 1) break;
    }
    if (ppb < 1 || pair_blocks < 1) pk = nullptr;
  }
  if (pk) {
    if (env_int("RS_DEBUG_PLAN", 0))
      fprintf(stderr, "rs plan: policy %d fast 1 kernel pair pairs/block %d blocks/SM %d "
              "group_bytes %d wcap %d rsm %d\n", cfg->policy, ppb, pair_blocks, L.group_bytes,
              L.wcap, L.rsm);
    const int grid = std::max(1, std::min((tr->num_replays + ppb - 1) / ppb, sms * pair_blocks));
    pk<<<grid, 64 * ppb, ppb * L.group_bytes, st>>>(kp);
    RS_CUDA(cudaGetLastError());
  } else {
    rs_status s2 = launch_kernel(pl.kern, kp, pl.wpb, rs::kWarp / pl.width, pl.block_smem,
                                 tr->num_replays, st);
    if (s2 != RS_OK) return s2;
  }
  // compute_metrics aggregates (metrics.hpp:62-162), one CTA per replay;
  // the streamed-input caller launches them itself once its copies are queued
  if (inputs_done == kDeferStats) return RS_OK;
  return rs_internal_stats(tr, out, stats, stream, inputs_done);
}

rs_status rs_internal_check_weights(const double* params, size_t count) {
  if (!params) return fail(RS_ERR_INVALID_ARGUMENT, "rl: null parameters");
  for (size_t k = 0; k < count; ++k)
    if (!std::isfinite(params[k]))
      return fail(RS_ERR_UNSUPPORTED,
                  "rl: non-finite Q-network weight " + std::to_string(k) +
                      " (the forward skips exact-zero inputs, exact only for finite weights)");
  return RS_OK;
}

rs_status rs_internal_stats(const rs_trace_soa* tr, const rs_req_out* out, rs_replay_stats* stats,
                            void* stream, void* wait_event) {
  cudaStream_t st = (cudaStream_t)stream;
  if (wait_event) RS_CUDA(cudaStreamWaitEvent(st, (cudaEvent_t)wait_event, 0));
  rs::StatsParams sp;
  sp.num_replays = tr->num_replays;
  sp.offsets = reinterpret_cast<const long long*>(tr->offsets);
  sp.arrival = tr->arrival_s;
  sp.decode = tr->decode_tokens;
  sp.routed = out->routed_s;
  sp.first = out->first_token_s;
  sp.completion = out->completion_s;
  sp.preempt = out->preemptions;
  sp.stats = stats;
  int dev = 0, sms = 0;
  RS_CUDA(cudaGetDevice(&dev));
  RS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::max(1, std::min(tr->num_replays, sms * 8));
  rs::stats_kernel<<<grid, rs::kStatsThreads, 0, st>>>(sp);
  RS_CUDA(cudaGetLastError());
  return RS_OK;
}

