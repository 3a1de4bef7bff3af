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
//   ClusterConfig::record_trajectory + trajectory()  env.hpp:131, 203, 251-319
//     becomes BatchSim::run_trajectory(policy, capacity, RewardConfig, episode_k)
//   compute_metrics + emit_report(dir)              metrics.hpp:84-238 -> emit_report(...)
//   DqnAgent::update after ReplayBuffer::sample     dqn.hpp:107-127 -> DqnTrainer::update
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

// RewardConfig (env.hpp:40-71).
enum class ShapingMode { None, Additive, Guided };
struct RewardConfig {
  double r_w = 60.0;
  double gamma = 0.99;
  double beta_d = 0.5;
  ShapingMode shaping = ShapingMode::Guided;
};

// TickRecord (env.hpp:150-168) with its RewardBreakdown (env.hpp:148-158).
struct TickRecord {
  long long tick = 0;
  double time = 0.0;
  int action = 0;
  double queue_penalty = 0.0, h = 0.0, shaping = 0.0, total = 0.0;
  int completions = 0;
  bool infeasible_route = false;
  int router_queue_len = 0;
  std::vector<int> instance_running, instance_waiting;
  int tokens_emitted = 0;
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
    return run(policy, max_ticks, rl_dims, rl_params, epsilon, policy_seeds, nullptr, 0,
               RewardConfig{}, 0);
  }

  // run_policy with the replays sharded over several devices of this process
  // (rs_replay_batch_multi: one shard per device, NCCL all-gather of the
  // per-replay statistics); results identical to run_policy.
  std::vector<ReplayResult> run_policy_multi(const std::string& policy,
                                             const std::vector<int32_t>& devices,
                                             long long max_ticks = 10'000'000,
                                             const std::vector<int>& rl_dims = {},
                                             const std::vector<double>& rl_params = {},
                                             double epsilon = 0.0,
                                             const std::vector<uint64_t>& policy_seeds = {}) const {
    if (devices.empty()) throw std::invalid_argument("run_policy_multi: no devices");
    return run(policy, max_ticks, rl_dims, rl_params, epsilon, policy_seeds, nullptr, 0,
               RewardConfig{}, 0, &devices);
  }

  // run_policy with record_trajectory: every replay's ClusterSim::trajectory()
  // (the first `capacity` ticks) into `trajectories`.
  std::vector<ReplayResult> run_trajectory(const std::string& policy, long long capacity,
                                           std::vector<std::vector<TickRecord>>& trajectories,
                                           const RewardConfig& reward = {}, int episode_k = 0,
                                           long long max_ticks = 10'000'000,
                                           const std::vector<int>& rl_dims = {},
                                           const std::vector<double>& rl_params = {},
                                           double epsilon = 0.0,
                                           const std::vector<uint64_t>& policy_seeds = {}) const {
    return run(policy, max_ticks, rl_dims, rl_params, epsilon, policy_seeds, &trajectories,
               capacity, reward, episode_k);
  }

 private:
  std::vector<ReplayResult> run(const std::string& policy, long long max_ticks,
                                const std::vector<int>& rl_dims,
                                const std::vector<double>& rl_params, double epsilon,
                                const std::vector<uint64_t>& policy_seeds,
                                std::vector<std::vector<TickRecord>>* trajectories,
                                long long capacity, const RewardConfig& reward,
                                int episode_k,
                                const std::vector<int32_t>* devices = nullptr) const {
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
    if (devices) {
      check(rs_replay_batch_multi(&a, &tr, &out, st.data(), devices->data(),
                                  static_cast<int32_t>(devices->size())));
    } else if (!trajectories) {
      check(rs_replay_batch_host(&a, &tr, &out, st.data(), device_));
    } else {
      if (capacity < 0) throw std::invalid_argument("trajectory capacity < 0");
      const size_t K = static_cast<size_t>(capacity) * R, m = static_cast<size_t>(a.num_instances);
      std::vector<double> t_time(K), t_qp(K), t_h(K), t_sh(K), t_tot(K);
      std::vector<int32_t> t_act(K), t_comp(K), t_rq(K), t_tok(K), t_run(K * m), t_wait(K * m);
      std::vector<uint8_t> t_inf(K);
      rs_trajectory tj{};
      tj.capacity = capacity;
      tj.r_w = reward.r_w;
      tj.gamma = reward.gamma;
      tj.beta_d = reward.beta_d;
      tj.shaping = static_cast<int32_t>(reward.shaping);
      tj.episode_k = episode_k;
      tj.time_s = t_time.data();
      tj.action = t_act.data();
      tj.queue_penalty = t_qp.data();
      tj.completions = t_comp.data();
      tj.h = t_h.data();
      tj.shaping_term = t_sh.data();
      tj.reward = t_tot.data();
      tj.infeasible_route = t_inf.data();
      tj.router_queue = t_rq.data();
      tj.tokens_emitted = t_tok.data();
      tj.instance_running = t_run.data();
      tj.instance_waiting = t_wait.data();
      check(rs_replay_trajectory_host(&a, &tr, &out, st.data(), &tj, device_));
      trajectories->assign(R, {});
      for (size_t r = 0; r < R; ++r) {
        const size_t k = static_cast<size_t>(std::min<long long>(st[r].ticks, capacity));
        auto& v = (*trajectories)[r];
        v.resize(k);
        for (size_t t = 0; t < k; ++t) {
          const size_t i = r * static_cast<size_t>(capacity) + t;
          TickRecord& x = v[t];
          x.tick = static_cast<long long>(t + 1);
          x.time = t_time[i];
          x.action = t_act[i];
          x.queue_penalty = t_qp[i];
          x.completions = t_comp[i];
          x.h = t_h[i];
          x.shaping = t_sh[i];
          x.total = t_tot[i];
          x.infeasible_route = t_inf[i] != 0;
          x.router_queue_len = t_rq[i];
          x.tokens_emitted = t_tok[i];
          x.instance_running.assign(t_run.begin() + i * m, t_run.begin() + (i + 1) * m);
          x.instance_waiting.assign(t_wait.begin() + i * m, t_wait.begin() + (i + 1) * m);
        }
      }
    }
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

// compute_metrics + emit_report (metrics.hpp:84-238) of one replay into
// `dir`: summary.json, requests.csv, timeseries.csv, byte-identical to the
// reference's.  `trajectory` null = a record_trajectory = false run.
inline void emit_report(const std::string& dir, const ClusterConfig& cfg,
                        const ArrivalTrace& trace, const ReplayResult& res,
                        const std::vector<TickRecord>* trajectory = nullptr) {
  const rs_batch_cfg a = to_abi(cfg, RS_POLICY_ROUND_ROBIN);
  const size_t k = trajectory ? trajectory->size() : 0, m = static_cast<size_t>(cfg.num_instances);
  std::vector<double> tt(k), tr(k);
  std::vector<int32_t> ta(k), tq(k), tk(k), trn(k * m), tw(k * m);
  for (size_t t = 0; t < k; ++t) {
    const TickRecord& x = (*trajectory)[t];
    tt[t] = x.time;
    tr[t] = x.total;
    ta[t] = x.action;
    tq[t] = x.router_queue_len;
    tk[t] = x.tokens_emitted;
    for (size_t i = 0; i < m; ++i) {
      trn[t * m + i] = x.instance_running.at(i);
      tw[t * m + i] = x.instance_waiting.at(i);
    }
  }
  rs_trajectory tj{};
  tj.time_s = tt.data();
  tj.action = ta.data();
  tj.reward = tr.data();
  tj.router_queue = tq.data();
  tj.tokens_emitted = tk.data();
  tj.instance_running = trn.data();
  tj.instance_waiting = tw.data();
  check(rs_emit_report(dir.c_str(), &a, static_cast<int64_t>(trace.size()),
                       trace.arrival_time_s.data(), trace.prompt_tokens.data(),
                       trace.decode_tokens.data(), trace.task.data(),
                       res.assigned_instance.data(), res.routed_time_s.data(),
                       res.first_token_time_s.data(), res.completion_time_s.data(),
                       res.preemption_count.data(), &res.stats, trajectory ? &tj : nullptr,
                       static_cast<int64_t>(k)));
}

// One transition of the replay buffer (replay.hpp:12-18).
struct Transition {
  std::vector<double> state;
  int action = 0;
  double reward = 0.0;
  std::vector<double> next_state;
  bool done = false;
};

// DqnAgent's trainable state (dqn.hpp:52-140): online / target networks in
// the flat layout, Adam moments.  update() = DqnAgent::update on a batch the
// caller sampled (ReplayBuffer::sample), executed on the device.
class DqnTrainer {
 public:
  DqnTrainer(std::vector<int> dims, std::vector<double> params, double learning_rate = 1e-3,
             long long target_sync_interval = 1000, int device = 0)
      : dims_(std::move(dims)), online_(std::move(params)), target_(online_),
        m_(online_.size(), 0.0), v_(online_.size(), 0.0), lr_(learning_rate),
        sync_(target_sync_interval), device_(device) {
    if (dims_.size() < 2 || dims_.size() > RS_MAX_LAYERS + 1)
      throw std::invalid_argument("dqn: 2..5 layer dims required");
  }

  double update(const std::vector<const Transition*>& batch, double discount) {
    const size_t B = batch.size(), d0 = static_cast<size_t>(dims_.front());
    std::vector<double> s(B * d0), ns(B * d0), r(B);
    std::vector<int32_t> a(B);
    std::vector<uint8_t> d(B);
    for (size_t i = 0; i < B; ++i) {
      const Transition& t = *batch[i];
      if (t.state.size() != d0 || t.next_state.size() != d0)
        throw std::invalid_argument("mlp: input dimension mismatch");
      std::copy(t.state.begin(), t.state.end(), s.begin() + i * d0);
      std::copy(t.next_state.begin(), t.next_state.end(), ns.begin() + i * d0);
      a[i] = t.action;
      r[i] = t.reward;
      d[i] = t.done ? 1 : 0;
    }
    rs_batch_cfg c;
    check(rs_default_config(&c));
    c.rl_num_layers = static_cast<int32_t>(dims_.size() - 1);
    for (size_t i = 0; i < dims_.size(); ++i) c.rl_dims[i] = dims_[i];
    rs_dqn_batch b{static_cast<int32_t>(B), 0, s.data(), a.data(), r.data(), ns.data(), d.data()};
    rs_dqn_state st{online_.data(), target_.data(), m_.data(), v_.data(), t_, updates_, sync_, lr_};
    double loss = 0.0;
    check(rs_dqn_update_host(&c, &b, &st, discount, &loss, device_));
    t_ = st.adam_t;
    updates_ = st.updates;
    return loss;
  }

  const std::vector<double>& online() const { return online_; }
  const std::vector<double>& target() const { return target_; }
  long long updates() const { return updates_; }

 private:
  std::vector<int> dims_;
  std::vector<double> online_, target_, m_, v_;
  double lr_;
  long long sync_;
  int device_;
  long long t_ = 0, updates_ = 0;
};

}  // namespace routesim_b200
