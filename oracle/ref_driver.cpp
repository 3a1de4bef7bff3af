// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never linked into the
// product).  A thin extern "C" harness around the UNMODIFIED reference
// headers at $(REF)/proj/include (compiled in place by oracle/Makefile into
// oracle/_ref/librs_ref.so).  Used by tests/ as the differential oracle, by
// tests/golden/make_golden.py to freeze fixtures, and by bench.py's
// `cpu_baseline` / `--impl reference` legs to time the reference's own CPU
// path on the host cores.
//
// The only policy added here is `workload_aware`: the
// reference has no workload-aware heuristic router (policies.hpp:230-245), so
// it is defined as a RoutingPolicy plugin written purely from reference
// primitives: can_accept (policies.hpp:44-48), estimate_instance_available
// (latency.hpp:96-99), mixing_for (impact.hpp:73-77) and
// ClusterSim::instance_loads (env.hpp:341-354).
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "routesim/dqn.hpp"
#include "routesim/env.hpp"
#include "routesim/experiment.hpp"
#include "routesim/metrics.hpp"
#include "routesim/policies.hpp"
#include "routesim/workload.hpp"

#include "../include/rs_abi.h"

using namespace routesim;

namespace {

thread_local std::string g_err;

// Workload-aware route() scoring, SURVEY.md Appendix B.  Lower score wins,
// lowest index on ties, defer when no instance can accept the head.
class WorkloadAwarePolicy final : public RoutingPolicy {
 public:
  WorkloadAwarePolicy(const ClusterSim& sim, HardwareProfile prof,
                      ImpactConfig impact)
      : sim_(sim), prof_(prof), impact_(impact) {}
  int decide(const SystemState& s) override {
    const Request* head = s.head();
    if (!head) return s.defer_action();
    const long long p = head->prompt_tokens;
    const long long d = head->decode_estimate();
    auto loads = sim_.instance_loads();
    int best = -1;
    double best_score = 0.0;
    for (int l = 0; l < s.num_instances(); ++l) {
      const auto& f = s.instances[static_cast<std::size_t>(l)];
      if (!can_accept(f, *head, s.max_batch_size)) continue;
      double avail = estimate_instance_available(prof_, f.outstanding_decode_estimate);
      double pcost = prof_.prompt_time_per_token *
                     static_cast<double>(f.pending_prompt_tokens + p);
      double mix = mixing_for(impact_, p, d, loads[static_cast<std::size_t>(l)]);
      double score = (avail + pcost) - impact_.epsilon_s * mix;
      if (best < 0 || score < best_score) {
        best = l;
        best_score = score;
      }
    }
    return best < 0 ? s.defer_action() : best;
  }
  std::string name() const override { return "workload_aware"; }

 private:
  const ClusterSim& sim_;
  HardwareProfile prof_;
  ImpactConfig impact_;
};

// epsilon-greedy adapter: DqnAgent::act (dqn.hpp:92-99) with a per-replay Rng.
class ActPolicy final : public RoutingPolicy {
 public:
  ActPolicy(const DqnAgent& agent, BucketScheme scheme, std::uint64_t seed)
      : agent_(agent), scheme_(std::move(scheme)), rng_(seed) {}
  int decide(const SystemState& s) override {
    return agent_.act(encode_state(s, scheme_), 0, rng_);
  }
  std::string name() const override { return "rl_act"; }

 private:
  const DqnAgent& agent_;
  BucketScheme scheme_;
  Rng rng_;
};

// Records every decision (exactly one decide() per tick in run_policy,
// env.hpp:326-337) into an FNV-1a hash and an optional action log.
class Recorder final : public RoutingPolicy {
 public:
  Recorder(RoutingPolicy& inner, std::vector<int32_t>* log)
      : inner_(inner), log_(log) {}
  int decide(const SystemState& s) override {
    int a = inner_.decide(s);
    hash_ = (hash_ ^ static_cast<std::uint64_t>(static_cast<std::uint32_t>(a + 1))) *
            0x100000001b3ULL;
    if (log_) log_->push_back(a);
    return a;
  }
  std::size_t pick_queue_index(const SystemState& s) override {
    return inner_.pick_queue_index(s);
  }
  std::string name() const override { return inner_.name(); }
  std::uint64_t hash() const { return hash_; }

 private:
  RoutingPolicy& inner_;
  std::vector<int32_t>* log_;
  std::uint64_t hash_ = 0xcbf29ce484222325ULL;
};

HardwareProfile to_profile(const rs_profile& p) {
  HardwareProfile h;
  h.prompt_time_per_token = p.prompt_time_per_token;
  h.prompt_time_intercept = p.prompt_time_intercept;
  h.decode_time_per_token = p.decode_time_per_token;
  h.decode_time_base = p.decode_time_base;
  return h;
}

Thresholds to_thresholds(const rs_thresholds& t) {
  Thresholds th;
  th.heavy_prompt_seconds = t.heavy_prompt_seconds;
  th.heavy_decode_seconds = t.heavy_decode_seconds;
  return th;
}

ClusterConfig to_cluster(const rs_batch_cfg& c, std::uint64_t predictor_seed) {
  ClusterConfig cc;
  cc.profile = to_profile(c.profile);
  cc.thresholds = to_thresholds(c.thresholds);
  cc.impact.grad1 = c.impact.grad1;
  cc.impact.grad2 = c.impact.grad2;
  cc.impact.epsilon_s = c.impact.epsilon_s;
  cc.impact.alpha = c.impact.alpha;
  cc.impact.prompt_exponent = c.impact.prompt_exponent;
  cc.reward.shaping = ShapingMode::None;
  cc.instance.kv_capacity_tokens = c.kv_capacity_tokens;
  cc.instance.max_batch_size = c.max_batch_size;
  cc.instance.batching = static_cast<BatchingPolicy>(c.batching);
  if (c.chunk_size > 0) cc.instance.chunk_size = c.chunk_size;
  cc.num_instances = c.num_instances;
  cc.delta_t = c.delta_t;
  cc.predictor_scheme.edges.assign(c.predictor_edges,
                                   c.predictor_edges + c.n_predictor_edges);
  cc.state_scheme.edges.assign(c.state_edges, c.state_edges + c.n_state_edges);
  cc.predictor_mode = PredictorMode::Simulated;
  AccuracyTable acc;
  for (int t = 0; t < kTaskKindCount; ++t) {
    acc.accuracy[static_cast<TaskKind>(t)] = c.accuracy[t];
  }
  cc.accuracy = acc;
  cc.predictor_seed = predictor_seed;
  cc.episode_k = 0;
  cc.record_trajectory = false;
  return cc;
}

// The reference top cap is fixed (kMaxDecodeTokens); refuse anything else.
bool check_cfg(const rs_batch_cfg& c) {
  if (c.predictor_top_cap != kMaxDecodeTokens) {
    g_err = "reference driver: predictor_top_cap must be kMaxDecodeTokens";
    return false;
  }
  if (c.predictor_mode == RS_PREDICTOR_EMPIRICAL) {
    g_err = "reference driver: use RS_PREDICTOR_GIVEN with precomputed buckets";
    return false;
  }
  return true;
}

std::unique_ptr<DqnAgent> make_agent(const rs_batch_cfg& c) {
  AgentConfig ac;
  ac.hidden = c.rl_dims[1];
  // act() uses epsilon_for(0) == epsilon_start exactly (dqn.hpp:73-80)
  if (c.rl_epsilon > 0.0) ac.epsilon_start = c.rl_epsilon;
  auto agent = std::make_unique<DqnAgent>(c.rl_dims[0], c.rl_dims[c.rl_num_layers],
                                          ac, 0);
  std::vector<int> dims(c.rl_dims, c.rl_dims + c.rl_num_layers + 1);
  if (agent->online().dims() != dims) agent->online() = Mlp(dims);
  auto& p = agent->online().params();
  std::memcpy(p.data(), c.rl_params, p.size() * sizeof(double));
  agent->sync_target();
  return agent;
}

struct ReplayIO {
  int64_t n;
  const double* arrival;
  const int32_t* prompt;
  const int32_t* decode;
  const uint8_t* task;
  uint64_t predictor_seed;
  uint64_t policy_seed;
  int32_t* instance;
  double* routed;
  double* first;
  double* completion;
  int32_t* preemptions;
  uint8_t* predicted;
  int32_t* action_log;      // optional, capacity action_cap
  int64_t action_cap;
};

int run_one(const rs_batch_cfg& c, const ReplayIO& io, rs_replay_stats* st,
            const DqnAgent* agent, bool record, const rs_trajectory* traj = nullptr) {
  ArrivalTrace trace;
  trace.requests.resize(static_cast<std::size_t>(io.n));
  for (int64_t i = 0; i < io.n; ++i) {
    Request& r = trace.requests[static_cast<std::size_t>(i)];
    r.id = static_cast<std::uint64_t>(i);
    r.arrival_time_s = io.arrival[i];
    r.prompt_tokens = io.prompt[i];
    r.true_decode_tokens = io.decode[i];
    r.task = static_cast<TaskKind>(io.task[i]);
  }
  ClusterConfig cc = to_cluster(c, io.predictor_seed);
  cc.record_trajectory = record;  // TickRecords feed the queue-length sums
  if (traj) {  // RewardConfig + episode_k of the trajectory request
    cc.reward.r_w = traj->r_w;
    cc.reward.gamma = traj->gamma;
    cc.reward.beta_d = traj->beta_d;
    cc.reward.shaping = static_cast<ShapingMode>(traj->shaping);
    cc.episode_k = traj->episode_k;
    cc.record_trajectory = true;
  }
  ClusterSim sim(cc, std::move(trace));
  std::unique_ptr<RoutingPolicy> pol;
  HardwareProfile prof = cc.profile;
  switch (c.policy) {
    case RS_POLICY_ROUND_ROBIN: pol = make_policy("round_robin", prof, cc.thresholds); break;
    case RS_POLICY_DEDICATED_SMALL_LARGE:
      pol = make_policy("dedicated_small_large", prof, cc.thresholds); break;
    case RS_POLICY_DECODE_BALANCER: pol = make_policy("decode_balancer", prof, cc.thresholds); break;
    case RS_POLICY_JSQ: pol = make_policy("jsq", prof, cc.thresholds); break;
    case RS_POLICY_MAX_CAPACITY: pol = make_policy("max_capacity", prof, cc.thresholds); break;
    case RS_POLICY_MIN_MIN: pol = make_policy("min_min", prof, cc.thresholds); break;
    case RS_POLICY_EARLIEST_AVAILABLE:
      pol = make_policy("earliest_available", prof, cc.thresholds); break;
    case RS_POLICY_WORKLOAD_AWARE:
      pol = std::make_unique<WorkloadAwarePolicy>(sim, prof, cc.impact); break;
    case RS_POLICY_RL:
      if (c.rl_epsilon > 0.0) {
        pol = std::make_unique<ActPolicy>(*agent, cc.state_scheme, io.policy_seed);
      } else {
        pol = std::make_unique<RlPolicy>(*agent, cc.state_scheme);
      }
      break;
    default: g_err = "unknown policy"; return -1;
  }
  std::vector<int32_t> log;
  Recorder rec(*pol, io.action_log ? &log : nullptr);
  int status = RS_REPLAY_FINISHED;
  try {
    bool ok = sim.run_policy(rec, c.max_ticks);
    status = ok ? RS_REPLAY_FINISHED : RS_REPLAY_MAX_TICKS;
  } catch (const std::logic_error& e) {
    // invalid_argument derives from logic_error; Instance::step throws the
    // plain logic_error.
    status = dynamic_cast<const std::invalid_argument*>(&e) ? RS_REPLAY_BAD_ACTION
                                                           : RS_REPLAY_NOT_ADMISSIBLE;
  }
  const RequestPool& pool = sim.pool();
  std::memset(st, 0, sizeof(*st));
  st->ticks = sim.tick();
  st->infeasible = sim.infeasible_routes();
  st->completed = static_cast<int64_t>(sim.completed_count());
  st->decision_hash = rec.hash();
  st->clock = sim.clock();
  st->status = status;
  st->error_instance = -1;
  double first_arrival = std::numeric_limits<double>::max();
  double last_completion = 0.0;
  for (int64_t i = 0; i < io.n; ++i) {
    const Request& r = pool[static_cast<std::size_t>(i)];
    if (io.instance) io.instance[i] = r.assigned_instance;
    if (io.routed) io.routed[i] = r.routed_time_s;
    if (io.first) io.first[i] = r.first_token_time_s;
    if (io.completion) io.completion[i] = r.completion_time_s;
    if (io.preemptions) io.preemptions[i] = r.preemption_count;
    if (io.predicted) io.predicted[i] = static_cast<uint8_t>(r.predicted_bucket < 0 ? 255 : r.predicted_bucket);
    if (r.routed_time_s >= 0.0) st->routed += 1;
    if (r.predicted_bucket >= 0) st->injected += 1;
    if (!r.completed()) continue;
    // compute_metrics order (metrics.hpp:94-121)
    st->total_e2e_s += r.completion_time_s - r.arrival_time_s;
    st->total_ttft_s += r.first_token_time_s - r.arrival_time_s;
    if (r.tokens_emitted >= 2) {
      st->total_tbt_s += (r.completion_time_s - r.first_token_time_s) /
                         static_cast<double>(r.tokens_emitted - 1);
      st->tbt_count += 1;
    }
    if (r.routed_time_s >= 0.0) st->total_router_wait_s += r.routed_time_s - r.arrival_time_s;
    st->total_preemptions += r.preemption_count;
    st->total_tokens += r.tokens_emitted;
    first_arrival = std::min(first_arrival, r.arrival_time_s);
    last_completion = std::max(last_completion, r.completion_time_s);
  }
  for (const auto& t : sim.trajectory()) {  // metrics.hpp:140-155 numerators
    st->sum_router_queue += t.router_queue_len;
    for (int w : t.instance_waiting) st->sum_instance_waiting += w;
  }
  st->first_arrival_s = first_arrival;
  st->last_completion_s = last_completion;
  st->makespan_s = last_completion - first_arrival;
  if (traj) {  // ClusterSim::trajectory() into the rs_trajectory arrays (record 0)
    const auto& tv = sim.trajectory();
    const int m = c.num_instances;
    int64_t k = 0;
    for (const auto& t : tv) {
      if (k >= traj->capacity) break;
      if (traj->time_s) traj->time_s[k] = t.time;
      if (traj->action) traj->action[k] = t.action;
      if (traj->queue_penalty) traj->queue_penalty[k] = t.reward.queue_penalty;
      if (traj->completions) traj->completions[k] = t.reward.completions;
      if (traj->h) traj->h[k] = t.reward.h;
      if (traj->shaping_term) traj->shaping_term[k] = t.reward.shaping;
      if (traj->reward) traj->reward[k] = t.reward.total;
      if (traj->infeasible_route) traj->infeasible_route[k] = t.reward.infeasible_route ? 1 : 0;
      if (traj->router_queue) traj->router_queue[k] = t.router_queue_len;
      if (traj->tokens_emitted) traj->tokens_emitted[k] = t.tokens_emitted;
      for (int i = 0; i < m; ++i) {
        if (traj->instance_running) traj->instance_running[k * m + i] = t.instance_running[i];
        if (traj->instance_waiting) traj->instance_waiting[k * m + i] = t.instance_waiting[i];
      }
      ++k;
    }
  }
  if (io.action_log) {
    int64_t k = std::min<int64_t>(io.action_cap, static_cast<int64_t>(log.size()));
    std::memcpy(io.action_log, log.data(), static_cast<std::size_t>(k) * sizeof(int32_t));
  }
  return 0;
}

}  // namespace

extern "C" {

int ref_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return -1;
  std::snprintf(buf, len, "%s", g_err.c_str());
  return 0;
}

uint64_t ref_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

// build_workload (experiment.hpp:291-305) for WorkloadKind::Mixture with an
// optional custom weight vector (generate_mixture, workload.hpp:220-245).
int ref_generate_mixture(const rs_profile* prof, const rs_thresholds* th,
                         const double* weights, uint64_t seed, int64_t n,
                         double rate, int32_t process, double* arrival,
                         int32_t* prompt, int32_t* decode, uint8_t* task) {
  try {
    HardwareProfile hp = to_profile(*prof);
    Thresholds tt = to_thresholds(*th);
    Rng rng(mix_seed(seed, 0xB00C));
    ArrivalSpec spec{process == 0 ? ArrivalProcess::Poisson : ArrivalProcess::FixedInterval,
                     rate};
    ArrivalTrace t;
    if (weights) {
      std::vector<double> w(weights, weights + kTaskKindCount);
      t = generate_mixture(dataset_task_specs(hp, tt), w, static_cast<std::size_t>(n), spec, rng);
    } else {
      t = generate_dataset_mixture(hp, tt, static_cast<std::size_t>(n), spec, rng);
    }
    for (int64_t i = 0; i < n; ++i) {
      const Request& r = t.requests[static_cast<std::size_t>(i)];
      arrival[i] = r.arrival_time_s;
      prompt[i] = r.prompt_tokens;
      decode[i] = r.true_decode_tokens;
      task[i] = static_cast<uint8_t>(r.task);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// DqnAgent(state_dim, actions, AgentConfig{hidden}, seed) online parameters
// (dqn.hpp:60-65 via Mlp::random, mlp.hpp:32-45).
int64_t ref_agent_init(int32_t state_dim, int32_t actions, int32_t hidden,
                       uint64_t seed, double* params_out, int64_t cap) {
  AgentConfig ac;
  ac.hidden = hidden;
  DqnAgent agent(state_dim, actions, ac, seed);
  const auto& p = agent.online().params();
  if (params_out && cap >= static_cast<int64_t>(p.size())) {
    std::memcpy(params_out, p.data(), p.size() * sizeof(double));
  }
  return static_cast<int64_t>(p.size());
}

// Mlp::forward + DqnAgent::argmax_action for `batch` states.
int ref_mlp_forward(const rs_batch_cfg* cfg, const double* states, int32_t batch,
                    double* q_out, int32_t* greedy_out) {
  try {
    auto agent = make_agent(*cfg);
    int din = cfg->rl_dims[0];
    int dout = cfg->rl_dims[cfg->rl_num_layers];
    for (int b = 0; b < batch; ++b) {
      std::vector<double> x(states + static_cast<std::size_t>(b) * din,
                            states + static_cast<std::size_t>(b + 1) * din);
      auto q = agent->online().forward(x);
      std::memcpy(q_out + static_cast<std::size_t>(b) * dout, q.data(),
                  static_cast<std::size_t>(dout) * sizeof(double));
      greedy_out[b] = agent->greedy(x);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// One replay through the unmodified ClusterSim::run_policy.
int ref_run_replay(const rs_batch_cfg* cfg, int64_t n, const double* arrival,
                   const int32_t* prompt, const int32_t* decode, const uint8_t* task,
                   uint64_t predictor_seed, uint64_t policy_seed,
                   int32_t* instance, double* routed, double* first,
                   double* completion, int32_t* preemptions, uint8_t* predicted,
                   rs_replay_stats* stats, int32_t* action_log, int64_t action_cap) {
  try {
    if (!check_cfg(*cfg)) return -1;
    std::unique_ptr<DqnAgent> agent;
    if (cfg->policy == RS_POLICY_RL) agent = make_agent(*cfg);
    ReplayIO io{n, arrival, prompt, decode, task, predictor_seed, policy_seed,
                instance, routed, first, completion, preemptions, predicted,
                action_log, action_cap};
    return run_one(*cfg, io, stats, agent.get(), true);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// One replay with record_trajectory on: TickRecords (env.hpp:305-319) into
// `traj` (host arrays, replay-local: record t-1 for tick t).
int ref_run_trajectory(const rs_batch_cfg* cfg, int64_t n, const double* arrival,
                       const int32_t* prompt, const int32_t* decode, const uint8_t* task,
                       uint64_t predictor_seed, uint64_t policy_seed, int32_t* instance,
                       double* routed, double* first, double* completion,
                       int32_t* preemptions, uint8_t* predicted, rs_replay_stats* stats,
                       const rs_trajectory* traj) {
  try {
    if (!check_cfg(*cfg)) return -1;
    std::unique_ptr<DqnAgent> agent;
    if (cfg->policy == RS_POLICY_RL) agent = make_agent(*cfg);
    ReplayIO io{n, arrival, prompt, decode, task, predictor_seed, policy_seed,
                instance, routed, first, completion, preemptions, predicted, nullptr, 0};
    return run_one(*cfg, io, stats, agent.get(), true, traj);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// One replay (record_trajectory as given) through run_policy, then the
// reference's own compute_metrics + emit_report (metrics.hpp:84-238) into
// `dir`, as cmd_run does (routesim_cli.cpp:28-40).  Returns 0, or -1 (error
// text in ref_last_error; "no completed requests" included).
int ref_emit_report(const rs_batch_cfg* cfg, int64_t n, const double* arrival,
                    const int32_t* prompt, const int32_t* decode, const uint8_t* task,
                    uint64_t predictor_seed, uint64_t policy_seed, int32_t record_trajectory,
                    const rs_trajectory* reward, const char* dir) {
  try {
    if (!check_cfg(*cfg)) return -1;
    std::unique_ptr<DqnAgent> agent;
    if (cfg->policy == RS_POLICY_RL) agent = make_agent(*cfg);
    ArrivalTrace trace;
    trace.requests.resize(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      Request& r = trace.requests[static_cast<std::size_t>(i)];
      r.id = static_cast<std::uint64_t>(i);
      r.arrival_time_s = arrival[i];
      r.prompt_tokens = prompt[i];
      r.true_decode_tokens = decode[i];
      r.task = static_cast<TaskKind>(task[i]);
    }
    ClusterConfig cc = to_cluster(*cfg, predictor_seed);
    cc.record_trajectory = record_trajectory != 0;
    if (reward) {
      cc.reward.r_w = reward->r_w;
      cc.reward.gamma = reward->gamma;
      cc.reward.beta_d = reward->beta_d;
      cc.reward.shaping = static_cast<ShapingMode>(reward->shaping);
      cc.episode_k = reward->episode_k;
    }
    ClusterSim sim(cc, std::move(trace));
    std::unique_ptr<RoutingPolicy> pol;
    HardwareProfile prof = cc.profile;
    static const char* names[] = {"round_robin", "dedicated_small_large", "decode_balancer",
                                  "jsq", "max_capacity", "min_min", "earliest_available"};
    if (cfg->policy >= 0 && cfg->policy < 7) {
      pol = make_policy(names[cfg->policy], prof, cc.thresholds);
    } else if (cfg->policy == RS_POLICY_WORKLOAD_AWARE) {
      pol = std::make_unique<WorkloadAwarePolicy>(sim, prof, cc.impact);
    } else if (cfg->rl_epsilon > 0.0) {
      pol = std::make_unique<ActPolicy>(*agent, cc.state_scheme, policy_seed);
    } else {
      pol = std::make_unique<RlPolicy>(*agent, cc.state_scheme);
    }
    sim.run_policy(*pol, cfg->max_ticks);
    auto rep = compute_metrics(sim.pool(), cc.profile, cc.thresholds, sim.trajectory(),
                               sim.tokens_per_second());
    emit_report(rep, sim.trajectory(), dir);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// `steps` DqnAgent::update calls (dqn.hpp:107-127) on a ReplayBuffer holding
// the n given transitions, sampling with Rng(sample_seed) (replay.hpp:44-58).
// The agent is DqnAgent(state_dim, actions, {hidden, lr, batch, sync}, 0) with
// its online (and target) parameters replaced by params_in.  Per step: the
// sampled transition indices (a copy of the Rng replays sample()'s draws),
// the loss, and the online parameters after the step.
int ref_dqn_train(int32_t state_dim, int32_t actions, int32_t hidden, const double* params_in,
                  int64_t n, const double* states, const int32_t* acts, const double* rewards,
                  const double* next_states, const uint8_t* dones, int32_t batch, int32_t steps,
                  uint64_t sample_seed, double discount, double lr, int64_t sync_interval,
                  int64_t* sampled_out, double* losses_out, double* online_out,
                  double* target_out) {
  try {
    AgentConfig ac;
    ac.hidden = hidden;
    ac.learning_rate = lr;
    ac.batch_size = static_cast<std::size_t>(batch);
    ac.replay_capacity = static_cast<std::size_t>(std::max<int64_t>(n, batch));
    ac.target_sync_interval = sync_interval;
    DqnAgent agent(state_dim, actions, ac, 0);
    auto& p = agent.online().params();
    std::memcpy(p.data(), params_in, p.size() * sizeof(double));
    agent.sync_target();
    ReplayBuffer replay(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      Transition t;
      t.state.assign(states + i * state_dim, states + (i + 1) * state_dim);
      t.action = acts[i];
      t.reward = rewards[i];
      t.next_state.assign(next_states + i * state_dim, next_states + (i + 1) * state_dim);
      t.done = dones[i] != 0;
      replay.push(std::move(t));
    }
    Rng rng(sample_seed);
    const std::size_t np = p.size();
    for (int32_t k = 0; k < steps; ++k) {
      Rng peek = rng;  // the draws update() is about to make
      auto smp = replay.sample(static_cast<std::size_t>(batch), peek);
      for (int32_t b = 0; b < batch; ++b)
        sampled_out[static_cast<int64_t>(k) * batch + b] = smp[static_cast<std::size_t>(b)] - &replay.at(0);
      auto loss = agent.update(replay, rng, discount);
      losses_out[k] = loss ? *loss : -1.0;
      std::memcpy(online_out + static_cast<std::size_t>(k) * np, agent.online().params().data(),
                  np * sizeof(double));
    }
    std::memcpy(target_out, agent.target().params().data(), np * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// run_experiment's empirical predictor (experiment.hpp:341-351) with the
// reference's own EmpiricalPredictor: fit on n_train Table-1 requests from
// Rng(mix_seed(seed, 0xF17)), then predict() for every (task, band) at the
// band's lowest prompt length.  table_out: [5][8] (bands < n_band_edges).
int ref_empirical_table(const rs_batch_cfg* cfg, uint64_t seed, int64_t n_train,
                        uint8_t* table_out) {
  try {
    HardwareProfile hp = to_profile(cfg->profile);
    Thresholds th = to_thresholds(cfg->thresholds);
    Rng rng(mix_seed(seed, 0xF17));
    ArrivalSpec spec{ArrivalProcess::Poisson, 1.0};
    auto training = generate_dataset_mixture(hp, th, static_cast<std::size_t>(n_train), spec, rng);
    BucketScheme scheme;
    scheme.edges.assign(cfg->predictor_edges, cfg->predictor_edges + cfg->n_predictor_edges);
    std::vector<long long> bands(cfg->band_edges, cfg->band_edges + cfg->n_band_edges);
    auto emp = EmpiricalPredictor::fit(training.requests, scheme, bands);
    for (int t = 0; t < kTaskKindCount; ++t)
      for (int b = 0; b < cfg->n_band_edges; ++b)
        table_out[t * RS_MAX_BANDS + b] = static_cast<uint8_t>(
            emp.predict(static_cast<TaskKind>(t),
                        static_cast<int>(std::max<long long>(1, cfg->band_edges[b]))));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CPU baseline: replays r in [0, R) of a CSR batch on `threads` host threads
// (atomic work counter), outputs per replay stats only.  Returns wall seconds
// (excluding nothing but thread start) or -1 on error.
double ref_run_batch(const rs_batch_cfg* cfg, int32_t num_replays,
                     const int64_t* offsets, const double* arrival,
                     const int32_t* prompt, const int32_t* decode,
                     const uint8_t* task, const uint64_t* predictor_seed,
                     const uint64_t* policy_seed, int32_t threads,
                     rs_replay_stats* stats) {
  try {
    if (!check_cfg(*cfg)) return -1.0;
    std::unique_ptr<DqnAgent> agent;
    if (cfg->policy == RS_POLICY_RL) agent = make_agent(*cfg);
    if (threads <= 0) threads = static_cast<int32_t>(std::thread::hardware_concurrency());
    std::atomic<int32_t> next{0};
    std::atomic<bool> failed{false};
    auto t0 = std::chrono::steady_clock::now();
    auto worker = [&]() {
      for (;;) {
        int32_t r = next.fetch_add(1);
        if (r >= num_replays) break;
        int64_t b = offsets[r], e = offsets[r + 1];
        ReplayIO io{e - b, arrival + b, prompt + b, decode + b, task + b,
                    predictor_seed[r], policy_seed ? policy_seed[r] : 0,
                    nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
        try {
          run_one(*cfg, io, &stats[r], agent.get(), false);
        } catch (...) {
          failed = true;
        }
      }
    };
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (failed) {
      g_err = "replay threw";
      return -1.0;
    }
    return wall;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// The golden run of test_harness.cpp:212-231 (JSQ, m=2, n=12, lambda=12,
// seed 777, shaping none): summary.json text into buf.
int ref_golden_summary(char* buf, size_t len, int32_t policy_is_jsq) {
  try {
    ExperimentConfig cfg;
    cfg.num_instances = 2;
    cfg.n_requests = 12;
    cfg.arrival.rate_per_s = 12.0;
    cfg.seed = 777;
    cfg.reward.shaping = ShapingMode::None;
    cfg.routing_policy = policy_is_jsq ? "jsq" : "round_robin";
    auto out = run_experiment(cfg);
    std::string s = report_to_json(out.report).dump(2) + "\n";
    if (s.size() + 1 > len) return -1;
    std::memcpy(buf, s.data(), s.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// summary.json of run_experiment for a mixture config (record_trajectory on),
// for fixture generation of arbitrary small cases.
int ref_experiment_summary(int32_t m, int64_t n, double rate, uint64_t seed,
                           const char* policy, char* buf, size_t len) {
  try {
    ExperimentConfig cfg;
    cfg.num_instances = m;
    cfg.n_requests = static_cast<std::size_t>(n);
    cfg.arrival.rate_per_s = rate;
    cfg.seed = seed;
    cfg.reward.shaping = ShapingMode::None;
    cfg.routing_policy = policy;
    auto out = run_experiment(cfg);
    std::string s = report_to_json(out.report).dump(2) + "\n";
    if (s.size() + 1 > len) return -1;
    std::memcpy(buf, s.data(), s.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int64_t ref_heavy_decode_cutoff(const rs_profile* p, const rs_thresholds* t) {
  return heavy_decode_token_cutoff(to_profile(*p), to_thresholds(*t));
}

}  // extern "C"
