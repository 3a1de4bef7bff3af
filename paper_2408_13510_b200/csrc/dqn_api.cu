// dqn_api.cu — C-ABI entry points of the device double-DQN update
// (rs_dqn_update / rs_dqn_update_host / rs_dqn_workspace_size), the kernels
// are in dqn.cuh.  Replaces DqnAgent::update (dqn.hpp:107-127) after the
// batch has been drawn (ReplayBuffer::sample, replay.hpp:44-58, stays with
// the caller, like the rest of train_agent's host loop).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/rs_abi.h"
#include "dqn.cuh"

namespace rs {
void set_error(const std::string& m);
}

namespace {

rs_status fail3(rs_status s, const std::string& m) {
  rs::set_error(m);
  return s;
}

#define RS_CUDA3(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      return fail3(e_ == cudaErrorMemoryAllocation ? RS_ERR_OUT_OF_MEMORY       \
                                                   : RS_ERR_CUDA,               \
                   std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)

size_t al3(size_t v) { return (v + 255) / 256 * 256; }

struct DqnLayout {
  rs::DqnParams p;  // shape fields only
  size_t act_bytes, delta_bytes, loss_bytes, total;
  int smem;
};

rs_status dqn_layout(const rs_batch_cfg* cfg, int B, DqnLayout* L) {
  if (!cfg) return fail3(RS_ERR_INVALID_ARGUMENT, "null config");
  const int layers = cfg->rl_num_layers;
  if (layers < 1 || layers > RS_MAX_LAYERS) return fail3(RS_ERR_INVALID_ARGUMENT, "dqn: 1..4 layers");
  if (B < 1) return fail3(RS_ERR_INVALID_ARGUMENT, "mlp: empty batch");  // mlp.hpp:81
  std::memset(L, 0, sizeof(*L));
  rs::DqnParams& P = L->p;
  P.layers = layers;
  int w = 0, a = 0, d = 0;
  P.maxw = 1;
  for (int l = 0; l <= layers; ++l) {
    if (cfg->rl_dims[l] < 1 || cfg->rl_dims[l] > RS_MAX_WIDTH)
      return fail3(RS_ERR_UNSUPPORTED, "dqn: layer width outside [1, 512]");
    P.dims[l] = cfg->rl_dims[l];
  }
  for (int l = 0; l < layers; ++l) {
    P.woff[l] = w;
    w += P.dims[l] * P.dims[l + 1];
    P.boff[l] = w;
    w += P.dims[l + 1];
    P.act_off[l] = a;
    a += P.dims[l];
    P.delta_off[l] = d;
    d += P.dims[l + 1];
    P.maxw = std::max(P.maxw, P.dims[l + 1]);
  }
  P.np = w;
  P.act_stride = a;
  P.delta_stride = d;
  P.B = B;
  P.smem_w_bytes = (int)(al3((size_t)w * 8));
  L->smem = 2 * P.smem_w_bytes + rs::kDqnWarps * (P.dims[0] + 4 * P.maxw) * 8;
  L->act_bytes = al3((size_t)B * a * 8);
  L->delta_bytes = al3((size_t)B * d * 8);
  L->loss_bytes = al3((size_t)B * 8);
  L->total = L->act_bytes + L->delta_bytes + L->loss_bytes;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess &&
      optin > 0 && L->smem > optin)
    return fail3(RS_ERR_UNSUPPORTED, "dqn: online + target networks exceed shared memory");
  return RS_OK;
}

std::mutex g_mu;
void* g_base = nullptr;
size_t g_bytes = 0;
cudaStream_t g_stream = nullptr;

}  // namespace

extern "C" {

rs_status rs_dqn_workspace_size(const rs_batch_cfg* cfg, int32_t batch, size_t* bytes) {
  if (!bytes) return fail3(RS_ERR_INVALID_ARGUMENT, "null size");
  DqnLayout L;
  rs_status s = dqn_layout(cfg, batch, &L);
  if (s != RS_OK) return s;
  *bytes = L.total;
  return RS_OK;
}

rs_status rs_dqn_update(const rs_batch_cfg* cfg, const rs_dqn_batch* b, rs_dqn_state* st,
                        double discount, double* loss_out, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (!b || !st || !loss_out) return fail3(RS_ERR_INVALID_ARGUMENT, "null batch/state/loss");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail3(RS_ERR_NO_DEVICE, "no CUDA device (the engine has no CPU fallback)");
  }
  DqnLayout L;
  rs_status s = dqn_layout(cfg, b->batch, &L);
  if (s != RS_OK) return s;
  if (!workspace || workspace_bytes < L.total)
    return fail3(RS_ERR_INVALID_ARGUMENT, "workspace too small (rs_dqn_workspace_size)");
  if (!b->state || !b->action || !b->reward || !b->next_state || !b->done || !st->online ||
      !st->target || !st->adam_m || !st->adam_v)
    return fail3(RS_ERR_INVALID_ARGUMENT, "null batch / parameter array");
  if (!(st->learning_rate > 0.0)) return fail3(RS_ERR_INVALID_ARGUMENT, "agent: lr must be > 0");
  if (st->target_sync_interval < 1)
    return fail3(RS_ERR_INVALID_ARGUMENT, "agent: target_sync_interval must be >= 1");
  rs::DqnParams P = L.p;
  P.state = b->state;
  P.action = b->action;
  P.reward = b->reward;
  P.next_state = b->next_state;
  P.done = b->done;
  P.online = st->online;
  P.target = st->target;
  P.online_out = st->online;
  P.adam_m = st->adam_m;
  P.adam_v = st->adam_v;
  P.discount = discount;
  P.inv_b = 1.0 / static_cast<double>(b->batch);  // mlp.hpp:84
  // AdamOptimizer (mlp.hpp:159-189): ++t_, bias corrections with host libm pow
  const long long t = st->adam_t + 1;
  P.lr = st->learning_rate;
  P.beta1 = 0.9;
  P.beta2 = 0.999;
  P.eps = 1e-8;
  P.bc1 = 1.0 - std::pow(P.beta1, static_cast<double>(t));
  P.bc2 = 1.0 - std::pow(P.beta2, static_cast<double>(t));
  char* ws = static_cast<char*>(workspace);
  P.act = reinterpret_cast<double*>(ws);
  P.delta = reinterpret_cast<double*>(ws + L.act_bytes);
  P.loss_terms = reinterpret_cast<double*>(ws + L.act_bytes + L.delta_bytes);
  P.loss_out = loss_out;
  cudaStream_t cs = (cudaStream_t)stream;
  RS_CUDA3(cudaFuncSetAttribute(rs::dqn_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                L.smem));
  int dev = 0, sms = 0;
  RS_CUDA3(cudaGetDevice(&dev));
  RS_CUDA3(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = std::max(1, std::min(sms, (b->batch + rs::kDqnWarps - 1) / rs::kDqnWarps));
  rs::dqn_sample_kernel<<<blocks, rs::kWarp * rs::kDqnWarps, L.smem, cs>>>(P);
  RS_CUDA3(cudaGetLastError());
  rs::dqn_param_kernel<<<(P.np + 127) / 128, 128, 0, cs>>>(P);
  RS_CUDA3(cudaGetLastError());
  st->adam_t = t;
  st->updates += 1;
  if (st->updates % st->target_sync_interval == 0)  // sync_target (dqn.hpp:125-130)
    RS_CUDA3(cudaMemcpyAsync(st->target, st->online, (size_t)P.np * 8,
                             cudaMemcpyDeviceToDevice, cs));
  return RS_OK;
}

rs_status rs_dqn_update_host(const rs_batch_cfg* cfg, const rs_dqn_batch* b, rs_dqn_state* st,
                             double discount, double* loss_out, int32_t device) {
  if (!b || !st || !loss_out) return fail3(RS_ERR_INVALID_ARGUMENT, "null batch/state/loss");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail3(RS_ERR_NO_DEVICE, "no CUDA device (the engine has no CPU fallback)");
  }
  if (device < 0 || device >= ndev) return fail3(RS_ERR_INVALID_ARGUMENT, "bad device");
  RS_CUDA3(cudaSetDevice(device));
  DqnLayout L;
  rs_status s = dqn_layout(cfg, b->batch, &L);
  if (s != RS_OK) return s;
  const int B = b->batch, d0 = L.p.dims[0];
  const size_t np = (size_t)L.p.np;
  size_t o = 0;
  const size_t o_s = o; o += al3((size_t)B * d0 * 8);
  const size_t o_a = o; o += al3((size_t)B * 4);
  const size_t o_r = o; o += al3((size_t)B * 8);
  const size_t o_n = o; o += al3((size_t)B * d0 * 8);
  const size_t o_d = o; o += al3((size_t)B);
  const size_t o_on = o; o += al3(np * 8);
  const size_t o_tg = o; o += al3(np * 8);
  const size_t o_m = o; o += al3(np * 8);
  const size_t o_v = o; o += al3(np * 8);
  const size_t o_l = o; o += al3(8);
  const size_t o_ws = o; o += L.total;
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_stream) RS_CUDA3(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking));
  if (g_bytes < o) {
    if (g_base) cudaFree(g_base);
    g_base = nullptr;
    g_bytes = 0;
    RS_CUDA3(cudaMalloc(&g_base, o));
    g_bytes = o;
  }
  char* d = static_cast<char*>(g_base);
  cudaStream_t cs = g_stream;
  if (!b->state || !b->action || !b->reward || !b->next_state || !b->done || !st->online ||
      !st->target || !st->adam_m || !st->adam_v)
    return fail3(RS_ERR_INVALID_ARGUMENT, "null batch / parameter array");
  RS_CUDA3(cudaMemcpyAsync(d + o_s, b->state, (size_t)B * d0 * 8, cudaMemcpyHostToDevice, cs));
  RS_CUDA3(cudaMemcpyAsync(d + o_a, b->action, (size_t)B * 4, cudaMemcpyHostToDevice, cs));
  RS_CUDA3(cudaMemcpyAsync(d + o_r, b->reward, (size_t)B * 8, cudaMemcpyHostToDevice, cs));
  RS_CUDA3(cudaMemcpyAsync(d + o_n, b->next_state, (size_t)B * d0 * 8, cudaMemcpyHostToDevice, cs));
  RS_CUDA3(cudaMemcpyAsync(d + o_d, b->done, (size_t)B, cudaMemcpyHostToDevice, cs));
  RS_CUDA3(cudaMemcpyAsync(d + o_on, st->online, np * 8, cudaMemcpyHostToDevice, cs));
  RS_CUDA3(cudaMemcpyAsync(d + o_tg, st->target, np * 8, cudaMemcpyHostToDevice, cs));
  RS_CUDA3(cudaMemcpyAsync(d + o_m, st->adam_m, np * 8, cudaMemcpyHostToDevice, cs));
  RS_CUDA3(cudaMemcpyAsync(d + o_v, st->adam_v, np * 8, cudaMemcpyHostToDevice, cs));
  rs_dqn_batch db = *b;
  db.state = reinterpret_cast<const double*>(d + o_s);
  db.action = reinterpret_cast<const int32_t*>(d + o_a);
  db.reward = reinterpret_cast<const double*>(d + o_r);
  db.next_state = reinterpret_cast<const double*>(d + o_n);
  db.done = reinterpret_cast<const uint8_t*>(d + o_d);
  rs_dqn_state ds = *st;
  ds.online = reinterpret_cast<double*>(d + o_on);
  ds.target = reinterpret_cast<double*>(d + o_tg);
  ds.adam_m = reinterpret_cast<double*>(d + o_m);
  ds.adam_v = reinterpret_cast<double*>(d + o_v);
  s = rs_dqn_update(cfg, &db, &ds, discount, reinterpret_cast<double*>(d + o_l), d + o_ws, L.total,
                    cs);
  if (s != RS_OK) return s;
  RS_CUDA3(cudaMemcpyAsync(st->online, d + o_on, np * 8, cudaMemcpyDeviceToHost, cs));
  RS_CUDA3(cudaMemcpyAsync(st->target, d + o_tg, np * 8, cudaMemcpyDeviceToHost, cs));
  RS_CUDA3(cudaMemcpyAsync(st->adam_m, d + o_m, np * 8, cudaMemcpyDeviceToHost, cs));
  RS_CUDA3(cudaMemcpyAsync(st->adam_v, d + o_v, np * 8, cudaMemcpyDeviceToHost, cs));
  RS_CUDA3(cudaMemcpyAsync(loss_out, d + o_l, 8, cudaMemcpyDeviceToHost, cs));
  RS_CUDA3(cudaStreamSynchronize(cs));
  st->adam_t = ds.adam_t;
  st->updates = ds.updates;
  return RS_OK;
}

}  // extern "C"
