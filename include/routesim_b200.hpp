// routesim_b200.hpp — C++17 host mirror of the reference router/simulator API
// (routesim, /root/reference/proj/include/routesim) over the engine's C ABI
// (rs_abi.h).  Header-only; link against librs_b200.so.
//
// Same names, argument meaning and error behaviour as the reference where the
// semantics carry over:
//   HardwareProfile / Thresholds / ImpactConfig   latency.hpp:16-51, impact.hpp:14-32
//   InstanceConfig / BatchingPolicy                instance.hpp:19-54
//   ClusterConfig                                  env.hpp:117-147
//   make_policy(name)  -> invalid_argument on an unknown name (policies.hpp:230-245)
//   ClusterSim(cfg, trace).run_policy(policy, max_ticks)      env.hpp:174-194, 326-337
//     becomes BatchSim(cfg, traces, seeds).run_policy(policy, max_ticks) for a
//     whole batch of independent replays (evaluate_policy's seed loop,
//     experiment.hpp:648-670), one launch on one B200.
// Configuration errors throw std::invalid_argument (as ClusterConfig::validate);
// device / CUDA failures throw std::runtime_error.  A replay that the
// reference would abort (logic_error "nothing admissible", or run_policy
// returning false at max_ticks) is reported per replay in ReplayResult.status.
#pragma once

#include <algorithm>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "rs_abi.h"

namespace routesim_b200 {

struct HardwareProfile {
  double prompt_time_per_token = 3.2e-4;
  double prompt_time_intercept = 0.026;
  double decode_time_per_token = 3.3e-5;
  double decode_time_base = 0.0167;
};

struct Thresholds {
  double heavy_prompt_seconds = 0.5;
  double heavy_decode_seconds = 5.0;
};

struct ImpactConfig {
  double grad1 = 3.2e-4;
  double grad2 = 3.3e-5;
  double epsilon_s = 0.5;
  double alpha = 0.5;
  int prompt_exponent = 2;
};

enum class BatchingPolicy { FCFS, BinPacking, LeastWorkLeft };

struct InstanceConfig {
  long long kv_capacity_tokens = 16384;
  int max_batch_size = 128;
  BatchingPolicy batching = BatchingPolicy::FCFS;
  std::optional<int> chunk_size;
};

struct ClusterConfig {
  HardwareProfile profile;
  Thresholds thresholds;
  ImpactConfig impact;
  InstanceConfig instance;
  int num_instances = 4;
  double delta_t = 0.02;
  std::vector<long long> predictor_edges{0, 250, 1000, 4000};
  std::vector<long long> state_edges{0, 256, 2048};
  // AccuracyTable per TaskKind (Translation, QnA, SentimentAnalysis,
  // InContextQnA, EntityRecognition); ExperimentConfig's dataset default.
  double accuracy[RS_NUM_TASKS] = {0.9310, 0.7036, 0.7992, 0.6527, 0.9506};
};

// One arrival trace (ArrivalTrace, workload.hpp:205-207) in SoA form.
struct ArrivalTrace {
  std::vector<double> arrival_time_s;
  std::vector<int32_t> prompt_tokens;
  std::vector<int32_t> decode_tokens;
  std::vector<uint8_t> task;
  size_t size() const { return arrival_time_s.size(); }
};

// Request's mutable fields after the replay + the per-replay statistics.
struct ReplayResult {
  std::vector<int32_t> assigned_instance;
  std::vector<double> routed_time_s, first_token_time_s, completion_time_s;
  std::vector<int32_t> preemption_count;
  rs_replay_stats stats;
  bool finished() const { return stats.status == RS_REPLAY_FINISHED; }
};

// make_policy's registry (policies.hpp:230-245) + workload_aware + rl.
inline rs_policy make_policy(const std::string& name) {
  static const char* names[RS_POLICY_COUNT] = {
      "round_robin", "dedicated_small_large", "decode_balancer", "jsq", "max_capacity",
      "min_min", "earliest_available", "workload_aware", "rl"};
  for (int i = 0; i < RS_POLICY_COUNT; ++i)
    if (name == names[i]) return static_cast<rs_policy>(i);
  throw std::invalid_argument("unknown routing policy: " + name);
}

// rs_mix_seed: the reference's seed derivation (rng.hpp:11-16).
inline uint64_t mix_seed(uint64_t seed, uint64_t stream) { return rs_mix_seed(seed, stream); }

inline void check(rs_status s) {
  if (s == RS_OK) return;
  char buf[512];
  rs_last_error(buf, sizeof(buf));
  if (s == RS_ERR_INVALID_ARGUMENT) throw std::invalid_argument(buf);
  throw std::runtime_error(std::string("routesim_b200: ") + buf);
}

inline rs_batch_cfg to_abi(const ClusterConfig& c, rs_policy policy) {
  rs_batch_cfg a;
  check(rs_default_config(&a));
  a.policy = policy;
  a.profile = rs_profile{c.profile.prompt_time_per_token, c.profile.prompt_time_intercept,
                         c.profile.decode_time_per_token, c.profile.decode_time_base};
  a.thresholds = rs_thresholds{c.thresholds.heavy_prompt_seconds, c.thresholds.heavy_decode_seconds};
  a.impact = rs_impact{c.impact.grad1, c.impact.grad2, c.impact.epsilon_s, c.impact.alpha,
                       c.impact.prompt_exponent, 0};
  a.kv_capacity_tokens = c.instance.kv_capacity_tokens;
  a.max_batch_size = c.instance.max_batch_size;
  a.batching = static_cast<int32_t>(c.instance.batching);
  a.chunk_size = c.instance.chunk_size ? *c.instance.chunk_size : 0;
  a.num_instances = c.num_instances;
  a.delta_t = c.delta_t;
  if (c.predictor_edges.size() > RS_MAX_BUCKETS || c.state_edges.size() > RS_MAX_BUCKETS)
    throw std::invalid_argument("bucket scheme: at most 8 edges");
  a.n_predictor_edges = static_cast<int32_t>(c.predictor_edges.size());
  for (size_t i = 0; i < c.predictor_edges.size(); ++i) a.predictor_edges[i] = c.predictor_edges[i];
  a.n_state_edges = static_cast<int32_t>(c.state_edges.size());
  for (size_t i = 0; i < c.state_edges.size(); ++i) a.state_edges[i] = c.state_edges[i];
  for (int t = 0; t < RS_NUM_TASKS; ++t) a.accuracy[t] = c.accuracy[t];
  check(rs_validate_config(&a));
  return a;
}

// A batch of independent ClusterSims (one per trace) replayed on one device.
class BatchSim {
 public:
  BatchSim(ClusterConfig cfg, std::vector<ArrivalTrace> traces,
           std::vector<uint64_t> predictor_seeds, int device = 0)
      : cfg_(std::move(cfg)), traces_(std::move(traces)), seeds_(std::move(predictor_seeds)),
        device_(device) {
    if (seeds_.size() != traces_.size())
      throw std::invalid_argument("BatchSim: one predictor seed per trace");
    to_abi(cfg_, RS_POLICY_ROUND_ROBIN);  // validate early, like ClusterConfig::validate
  }

  // ClusterSim::run_policy for every replay.  The Q-network (rl) takes the
  // reference flat parameter layout (mlp.hpp:19-30) and its layer dims.
  std::vector<ReplayResult> run_policy(const std::string& policy,
                                       long long max_ticks = 10'000'000,
                                       const std::vector<int>& rl_dims = {},
                                       const std::vector<double>& rl_params = {},
                                       double epsilon = 0.0,
                                       const std::vector<uint64_t>& policy_seeds = {}) const {
    rs_batch_cfg a = to_abi(cfg_, make_policy(policy));
    a.max_ticks = max_ticks;
    if (a.policy == RS_POLICY_RL) {
      if (rl_dims.size() < 2 || rl_dims.size() > RS_MAX_LAYERS + 1)
        throw std::invalid_argument("rl: 2..5 layer dims required");
      a.rl_num_layers = static_cast<int32_t>(rl_dims.size() - 1);
      for (size_t i = 0; i < rl_dims.size(); ++i) a.rl_dims[i] = rl_dims[i];
      a.rl_params = rl_params.data();
      a.rl_epsilon = epsilon;
    }
    const size_t R = traces_.size();
    std::vector<int64_t> off(R + 1, 0);
    for (size_t r = 0; r < R; ++r) off[r + 1] = off[r] + static_cast<int64_t>(traces_[r].size());
    const int64_t N = off[R];
    std::vector<double> arr(static_cast<size_t>(N));
    std::vector<int32_t> pr(static_cast<size_t>(N)), de(static_cast<size_t>(N));
    std::vector<uint8_t> tk(static_cast<size_t>(N));
    for (size_t r = 0; r < R; ++r) {
      const ArrivalTrace& t = traces_[r];
      if (t.prompt_tokens.size() != t.size() || t.decode_tokens.size() != t.size() ||
          t.task.size() != t.size())
        throw std::invalid_argument("ArrivalTrace: ragged fields");
      std::copy(t.arrival_time_s.begin(), t.arrival_time_s.end(), arr.begin() + off[r]);
      std::copy(t.prompt_tokens.begin(), t.prompt_tokens.end(), pr.begin() + off[r]);
      std::copy(t.decode_tokens.begin(), t.decode_tokens.end(), de.begin() + off[r]);
      std::copy(t.task.begin(), t.task.end(), tk.begin() + off[r]);
    }
    rs_trace_soa tr{};
    tr.num_replays = static_cast<int32_t>(R);
    tr.total_requests = N;
    tr.offsets = off.data();
    tr.arrival_s = arr.data();
    tr.prompt_tokens = pr.data();
    tr.decode_tokens = de.data();
    tr.task = tk.data();
    tr.predictor_seed = seeds_.data();
    tr.policy_seed = policy_seeds.empty() ? nullptr : policy_seeds.data();
    std::vector<int32_t> inst(static_cast<size_t>(N)), pre(static_cast<size_t>(N));
    std::vector<double> ro(static_cast<size_t>(N)), fi(static_cast<size_t>(N)),
        co(static_cast<size_t>(N));
    std::vector<uint8_t> pb(static_cast<size_t>(N));
    std::vector<rs_replay_stats> st(R);
    rs_req_out out{inst.data(), ro.data(), fi.data(), co.data(), pre.data(), pb.data()};
    check(rs_replay_batch_host(&a, &tr, &out, st.data(), device_));
    std::vector<ReplayResult> res(R);
    for (size_t r = 0; r < R; ++r) {
      const auto b = off[r], e = off[r + 1];
      res[r].assigned_instance.assign(inst.begin() + b, inst.begin() + e);
      res[r].routed_time_s.assign(ro.begin() + b, ro.begin() + e);
      res[r].first_token_time_s.assign(fi.begin() + b, fi.begin() + e);
      res[r].completion_time_s.assign(co.begin() + b, co.begin() + e);
      res[r].preemption_count.assign(pre.begin() + b, pre.begin() + e);
      res[r].stats = st[r];
    }
    return res;
  }

 private:
  ClusterConfig cfg_;
  std::vector<ArrivalTrace> traces_;
  std::vector<uint64_t> seeds_;
  int device_;
};

// build_workload for a seed (experiment.hpp:291-305): Table-1 mixture.
inline ArrivalTrace build_workload(uint64_t seed, int64_t n, double rate_per_s = 20.0,
                                   const HardwareProfile& p = {}, const Thresholds& t = {}) {
  ArrivalTrace tr;
  tr.arrival_time_s.resize(static_cast<size_t>(n));
  tr.prompt_tokens.resize(static_cast<size_t>(n));
  tr.decode_tokens.resize(static_cast<size_t>(n));
  tr.task.resize(static_cast<size_t>(n));
  const rs_profile rp{p.prompt_time_per_token, p.prompt_time_intercept, p.decode_time_per_token,
                      p.decode_time_base};
  const rs_thresholds rt{t.heavy_prompt_seconds, t.heavy_decode_seconds};
  check(rs_generate_mixture(&rp, &rt, nullptr, seed, n, rate_per_s, 0, tr.arrival_time_s.data(),
                            tr.prompt_tokens.data(), tr.decode_tokens.data(), tr.task.data()));
  return tr;
}

}  // namespace routesim_b200
