// multi.cu — rs_replay_batch_multi: one process driving several devices
// (SURVEY.md §8(e)).  Replays are independent (evaluate_policy's seed loop,
// experiment.hpp:648-670; SPEC.md:523-524 allows concurrent environments), so
// the batch is cut into contiguous replay shards, one per device; each device
// runs its shard through the same kernels as rs_replay_batch on its own
// stream, driven by its own host thread, with no collective on the data path.
// The only exchange is the final gather of the 256-byte per-replay
// statistics: ncclAllGather over a communicator set from ncclCommInitAll,
// after which device 0 holds every replay's record and copies them out.
//
// NCCL is opened with dlopen("libnccl.so.2") on first use, so the library has
// no link-time NCCL dependency and, inside a process that already loaded
// torch's NCCL, binds to that same copy (the SONAME is shared).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rs_abi.h"
#include "internal.h"

namespace rs {
void set_error(const std::string& m);  // engine.cu
}

namespace {

rs_status failm(rs_status s, const std::string& m) {
  rs::set_error(m);
  return s;
}

#define RS_CUDAM(call)                                                         \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess)                                                     \
      return failm(e_ == cudaErrorMemoryAllocation ? RS_ERR_OUT_OF_MEMORY      \
                                                   : RS_ERR_CUDA,              \
                   std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

struct Nccl {
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("dlopen libnccl.so.2: ") + dlerror();
      return;
    }
    n.comm_init_all = reinterpret_cast<decltype(n.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(h, "ncclGroupEnd"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.comm_init_all && n.all_gather && n.group_start && n.group_end && n.comm_destroy &&
           n.error_string;
    if (!n.ok) n.why = "libnccl.so.2 lacks a needed symbol";
  });
  return n;
}

size_t al(size_t v) { return (v + 255) / 256 * 256; }

// Per-device state of the multi-device path (own arena + stream), and the
// communicator set of the last device list.
struct Shard {
  void* base = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
};
struct MultiCache {
  std::mutex mu;
  Shard shard[16];
  std::vector<int> comm_devs;
  std::vector<ncclComm_t> comms;
};
MultiCache g_multi;

rs_status shard_arena(int dev, size_t need, char** out, cudaStream_t* st) {
  Shard& s = g_multi.shard[dev];
  if (!s.stream) RS_CUDAM(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  if (s.bytes < need) {
    if (s.base) cudaFree(s.base);
    s.base = nullptr;
    s.bytes = 0;
    RS_CUDAM(cudaMalloc(&s.base, need));
    s.bytes = need;
  }
  *out = static_cast<char*>(s.base);
  *st = s.stream;
  return RS_OK;
}

struct ShardJob {
  int dev;
  int r0, r1;            // replays [r0, r1)
  int64_t q0, q1;        // their requests [q0, q1) in the host arrays
  rs_replay_stats* dstats = nullptr;  // this shard's records (device)
  rs_replay_stats* gathered = nullptr;  // every shard's records (device)
  cudaStream_t st = nullptr;
  rs_status status = RS_OK;
  std::string err;
};

// One shard on its device: inputs up, the replay kernels, per-request
// results down (async on the shard stream).  Leaves dstats on the device.
void run_shard(const rs_batch_cfg* cfg, const rs_trace_soa* tr, rs_req_out* out, int shard_cap,
               int nshards, ShardJob& J) {
  auto fail = [&](rs_status s) {
    J.status = s;
    char buf[512];
    rs_last_error(buf, sizeof(buf));
    J.err = buf;
  };
  if (cudaSetDevice(J.dev) != cudaSuccess) {
    cudaGetLastError();
    J.status = RS_ERR_CUDA;
    J.err = "cudaSetDevice failed";
    return;
  }
  const int R = J.r1 - J.r0;
  const int64_t N = J.q1 - J.q0;
  const bool rl = cfg->policy == RS_POLICY_RL;
  size_t rl_bytes = 0;
  if (rl)
    for (int l = 0; l < cfg->rl_num_layers; ++l)
      rl_bytes += ((size_t)cfg->rl_dims[l] * cfg->rl_dims[l + 1] + cfg->rl_dims[l + 1]) * 8;
  size_t ws_bytes = 0;
  rs_status s = rs_workspace_size(cfg, R, N, &ws_bytes);
  if (s != RS_OK) return fail(s);
  size_t o = 0;
  const size_t o_off = o; o += al(8ull * (R + 1));
  const size_t o_arr = o; o += al(8ull * N);
  const size_t o_pr = o; o += al(4ull * N);
  const size_t o_de = o; o += al(4ull * N);
  const size_t o_tk = o; o += al(1ull * N);
  const size_t o_gv = o; o += al(1ull * N);
  const size_t o_ps = o; o += al(8ull * R);
  const size_t o_qs = o; o += al(8ull * R);
  const size_t o_rl = o; o += al(rl_bytes);
  const size_t o_in = o; o += al(4ull * N);
  const size_t o_ro = o; o += al(8ull * N);
  const size_t o_fi = o; o += al(8ull * N);
  const size_t o_co = o; o += al(8ull * N);
  const size_t o_pe = o; o += al(4ull * N);
  const size_t o_pb = o; o += al(1ull * N);
  const size_t o_st = o; o += al(sizeof(rs_replay_stats) * (size_t)shard_cap);
  const size_t o_ga = o; o += al(sizeof(rs_replay_stats) * (size_t)shard_cap * nshards);
  const size_t o_ws = o; o += al(ws_bytes);
  char* b = nullptr;
  if ((s = shard_arena(J.dev, o, &b, &J.st)) != RS_OK) return fail(s);
  const cudaStream_t st = J.st;
  // the shard's offsets, rebased to start at 0
  std::vector<int64_t> off(R + 1);
  for (int r = 0; r <= R; ++r) off[r] = tr->offsets[J.r0 + r] - J.q0;
  auto up = [&](size_t dst, const void* src, size_t n) {
    return (src && n) ? cudaMemcpyAsync(b + dst, src, n, cudaMemcpyHostToDevice, st)
                      : cudaSuccess;
  };
  auto at = [](const void* p, int64_t i, size_t es) -> const void* {
    return p ? static_cast<const char*>(p) + (size_t)i * es : nullptr;
  };
  cudaError_t e = up(o_off, off.data(), 8ull * (R + 1));
  if (e == cudaSuccess) e = up(o_arr, at(tr->arrival_s, J.q0, 8), 8ull * N);
  if (e == cudaSuccess) e = up(o_pr, at(tr->prompt_tokens, J.q0, 4), 4ull * N);
  if (e == cudaSuccess) e = up(o_de, at(tr->decode_tokens, J.q0, 4), 4ull * N);
  if (e == cudaSuccess) e = up(o_tk, at(tr->task, J.q0, 1), 1ull * N);
  if (e == cudaSuccess) e = up(o_gv, at(tr->given_bucket, J.q0, 1), 1ull * N);
  if (e == cudaSuccess) e = up(o_ps, at(tr->predictor_seed, J.r0, 8), 8ull * R);
  if (e == cudaSuccess) e = up(o_qs, at(tr->policy_seed, J.r0, 8), 8ull * R);
  if (e == cudaSuccess && rl) e = up(o_rl, cfg->rl_params, rl_bytes);
  // records beyond the shard's replays (the gather moves shard_cap per
  // device) are zero
  if (e == cudaSuccess)
    e = cudaMemsetAsync(b + o_st, 0, sizeof(rs_replay_stats) * (size_t)shard_cap, st);
  if (e != cudaSuccess) {
    J.status = RS_ERR_CUDA;
    J.err = std::string("shard input copy: ") + cudaGetErrorString(e);
    return;
  }
  rs_batch_cfg dcfg = *cfg;
  dcfg.flags |= RS_FLAG_PREDICT_INLINE;
  if (rl) dcfg.rl_params = reinterpret_cast<const double*>(b + o_rl);
  rs_trace_soa dt = *tr;
  dt.num_replays = R;
  dt.total_requests = N;
  dt.offsets = reinterpret_cast<const int64_t*>(b + o_off);
  dt.arrival_s = reinterpret_cast<const double*>(b + o_arr);
  dt.prompt_tokens = reinterpret_cast<const int32_t*>(b + o_pr);
  dt.decode_tokens = reinterpret_cast<const int32_t*>(b + o_de);
  dt.task = reinterpret_cast<const uint8_t*>(b + o_tk);
  dt.given_bucket = tr->given_bucket ? reinterpret_cast<const uint8_t*>(b + o_gv) : nullptr;
  dt.predictor_seed =
      tr->predictor_seed ? reinterpret_cast<const uint64_t*>(b + o_ps) : nullptr;
  dt.policy_seed = tr->policy_seed ? reinterpret_cast<const uint64_t*>(b + o_qs) : nullptr;
  rs_req_out dout;
  dout.instance = reinterpret_cast<int32_t*>(b + o_in);
  dout.routed_s = reinterpret_cast<double*>(b + o_ro);
  dout.first_token_s = reinterpret_cast<double*>(b + o_fi);
  dout.completion_s = reinterpret_cast<double*>(b + o_co);
  dout.preemptions = reinterpret_cast<int32_t*>(b + o_pe);
  dout.predicted_bucket = reinterpret_cast<uint8_t*>(b + o_pb);
  J.dstats = reinterpret_cast<rs_replay_stats*>(b + o_st);
  J.gathered = reinterpret_cast<rs_replay_stats*>(b + o_ga);
  if (R > 0) {
    s = rs_replay_batch(&dcfg, &dt, &dout, J.dstats, b + o_ws, ws_bytes, st);
    if (s != RS_OK) return fail(s);
  }
  if (out) {
    auto down = [&](void* dst, size_t src, size_t es) {
      return (dst && N) ? cudaMemcpyAsync(static_cast<char*>(dst) + (size_t)J.q0 * es, b + src,
                                          (size_t)N * es, cudaMemcpyDeviceToHost, st)
                        : cudaSuccess;
    };
    e = down(out->instance, o_in, 4);
    if (e == cudaSuccess) e = down(out->routed_s, o_ro, 8);
    if (e == cudaSuccess) e = down(out->first_token_s, o_fi, 8);
    if (e == cudaSuccess) e = down(out->completion_s, o_co, 8);
    if (e == cudaSuccess) e = down(out->preemptions, o_pe, 4);
    if (e == cudaSuccess) e = down(out->predicted_bucket, o_pb, 1);
    if (e != cudaSuccess) {
      J.status = RS_ERR_CUDA;
      J.err = std::string("shard output copy: ") + cudaGetErrorString(e);
    }
  }
}

}  // namespace

extern "C" rs_status rs_replay_batch_multi(const rs_batch_cfg* cfg, const rs_trace_soa* tr,
                                           rs_req_out* out, rs_replay_stats* stats,
                                           const int32_t* devices, int32_t ndev) {
  rs_status s = rs_validate_config(cfg);
  if (s != RS_OK) return s;
  if (!tr || !stats) return failm(RS_ERR_INVALID_ARGUMENT, "null trace/stats");
  if (!devices || ndev < 1 || ndev > 16)
    return failm(RS_ERR_INVALID_ARGUMENT, "devices: 1..16 device ids");
  int have = 0;
  if (cudaGetDeviceCount(&have) != cudaSuccess || have == 0) {
    cudaGetLastError();
    return failm(RS_ERR_NO_DEVICE, "no CUDA device (the engine has no CPU fallback)");
  }
  for (int d = 0; d < ndev; ++d) {
    if (devices[d] < 0 || devices[d] >= have || devices[d] >= 16)
      return failm(RS_ERR_INVALID_ARGUMENT, "bad device id");
    for (int k = 0; k < d; ++k)
      if (devices[k] == devices[d])
        return failm(RS_ERR_INVALID_ARGUMENT, "devices must be distinct (one shard each)");
  }
  const int R = tr->num_replays;
  if (R < 0) return failm(RS_ERR_INVALID_ARGUMENT, "num_replays < 0");
  if (R == 0) return RS_OK;
  if (!tr->offsets || tr->offsets[0] != 0 || tr->offsets[R] != tr->total_requests)
    return failm(RS_ERR_INVALID_ARGUMENT, "offsets must start at 0 and end at total_requests");
  for (int r = 0; r < R; ++r)
    if (tr->offsets[r + 1] < tr->offsets[r])
      return failm(RS_ERR_INVALID_ARGUMENT, "offsets must be non-decreasing");
  if (cfg->policy == RS_POLICY_RL) {
    size_t np = 0;
    for (int l = 0; l < cfg->rl_num_layers; ++l)
      np += (size_t)cfg->rl_dims[l] * cfg->rl_dims[l + 1] + cfg->rl_dims[l + 1];
    if ((s = rs_internal_check_weights(cfg->rl_params, np)) != RS_OK) return s;
  }
  Nccl& nc = nccl();
  if (!nc.ok) return failm(RS_ERR_UNSUPPORTED, "NCCL unavailable: " + nc.why);

  std::lock_guard<std::mutex> lock(g_multi.mu);
  // communicators for this device list (ncclCommInitAll: one per device,
  // ranks in list order); rebuilt only when the list changes
  const std::vector<int> devs(devices, devices + ndev);
  if (g_multi.comm_devs != devs) {
    for (ncclComm_t c : g_multi.comms) nc.comm_destroy(c);
    g_multi.comms.assign(ndev, nullptr);
    g_multi.comm_devs.clear();
    const ncclResult_t r = nc.comm_init_all(g_multi.comms.data(), ndev, devs.data());
    if (r != ncclSuccess) {
      g_multi.comms.clear();
      return failm(RS_ERR_CUDA, std::string("ncclCommInitAll: ") + nc.error_string(r));
    }
    g_multi.comm_devs = devs;
  }
  // contiguous shards of ceil(R / ndev) replays (the last may be short or
  // empty); every device gathers shard_cap records
  const int cap = (R + ndev - 1) / ndev;
  std::vector<ShardJob> jobs(ndev);
  for (int d = 0; d < ndev; ++d) {
    ShardJob& J = jobs[d];
    J.dev = devs[d];
    J.r0 = std::min(R, d * cap);
    J.r1 = std::min(R, (d + 1) * cap);
    J.q0 = tr->offsets[J.r0];
    J.q1 = tr->offsets[J.r1];
  }
  {
    std::vector<std::thread> th;
    for (int d = 0; d < ndev; ++d)
      th.emplace_back(run_shard, cfg, tr, out, cap, ndev, std::ref(jobs[d]));
    for (auto& t : th) t.join();
  }
  for (const ShardJob& J : jobs)
    if (J.status != RS_OK) {
      for (const ShardJob& K : jobs)
        if (K.st) {
          cudaSetDevice(K.dev);
          cudaStreamSynchronize(K.st);
        }
      return failm(J.status, "device " + std::to_string(J.dev) + ": " + J.err);
    }
  // the final gather of the per-replay statistics
  const size_t rec = sizeof(rs_replay_stats) * (size_t)cap;
  nc.group_start();
  ncclResult_t gr = ncclSuccess;
  for (int d = 0; d < ndev && gr == ncclSuccess; ++d) {
    RS_CUDAM(cudaSetDevice(jobs[d].dev));
    gr = nc.all_gather(jobs[d].dstats, jobs[d].gathered, rec, ncclUint8, g_multi.comms[d],
                       jobs[d].st);
  }
  const ncclResult_t ge = nc.group_end();
  if (gr != ncclSuccess || ge != ncclSuccess)
    return failm(RS_ERR_CUDA, std::string("ncclAllGather: ") +
                                  nc.error_string(gr != ncclSuccess ? gr : ge));
  RS_CUDAM(cudaSetDevice(jobs[0].dev));
  RS_CUDAM(cudaMemcpyAsync(stats, jobs[0].gathered, sizeof(rs_replay_stats) * (size_t)R,
                           cudaMemcpyDeviceToHost, jobs[0].st));
  for (const ShardJob& J : jobs) {
    RS_CUDAM(cudaSetDevice(J.dev));
    RS_CUDAM(cudaStreamSynchronize(J.st));
  }
  // as rs_replay_batch_host: requests that never reached the router queue
  // have no prediction (the reference leaves it unset)
  if (out && out->predicted_bucket)
    for (int r = 0; r < R; ++r)
      for (int64_t i = tr->offsets[r] + stats[r].injected; i < tr->offsets[r + 1]; ++i)
        out->predicted_bucket[i] = 255;
  return RS_OK;
}
