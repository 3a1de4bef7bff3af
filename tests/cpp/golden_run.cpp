// C++ user of the engine through include/routesim_b200.hpp, written the way
// the reference's own golden test is (test_harness.cpp:212-231): JSQ, m=2,
// n=12, lambda=12, seed 777.  Prints the replay's statistics as JSON; with a
// directory argument also replays it with record_trajectory (shaping none, as
// the golden run) and writes the reference-format report there, then runs
// one DqnTrainer update.
#include <cstdio>
#include <cstring>

#include "routesim_b200.hpp"

int main(int argc, char** argv) {
  using namespace routesim_b200;
  ClusterConfig cfg;
  cfg.num_instances = 2;
  try {
    make_policy("not_a_policy");
    std::printf("{\"error\": \"make_policy accepted an unknown name\"}\n");
    return 1;
  } catch (const std::invalid_argument&) {
  }
  std::vector<ArrivalTrace> traces{build_workload(777, 12, 12.0)};
  BatchSim sim(cfg, traces, {mix_seed(777, 0x9Ded)});
  auto res = sim.run_policy("jsq");
  const rs_replay_stats& s = res[0].stats;
  // the same batch sharded over this process's devices (device 0 here):
  // rs_replay_batch_multi, identical results
  auto resm = sim.run_policy_multi("jsq", {0});
  if (std::memcmp(&resm[0].stats, &s, sizeof(rs_replay_stats)) != 0 ||
      resm[0].completion_time_s != res[0].completion_time_s) {
    std::printf("{\"error\": \"run_policy_multi differs from run_policy\"}\n");
    return 4;
  }
  if (argc > 1) {
    std::vector<std::vector<TickRecord>> traj;
    RewardConfig rw;
    rw.shaping = ShapingMode::None;
    auto rt = sim.run_trajectory("jsq", 100000, traj, rw);
    emit_report(argv[1], cfg, traces[0], rt[0], &traj[0]);
    // one DqnAgent::update on transitions built from the trajectory's ticks
    const int d0 = 6 * cfg.num_instances + 3;
    std::vector<int> dims{d0, 16, 16, cfg.num_instances + 1};
    std::vector<double> params(static_cast<size_t>(d0 * 16 + 16 + 16 * 16 + 16 + 16 * 3 + 3), 0.01);
    DqnTrainer tr(dims, params);
    std::vector<Transition> buf;
    for (size_t t = 0; t + 1 < traj[0].size() && buf.size() < 32; ++t) {
      Transition x;
      x.state.assign(static_cast<size_t>(d0), 0.1 * static_cast<double>(t % 7));
      x.next_state.assign(static_cast<size_t>(d0), 0.1 * static_cast<double>((t + 1) % 7));
      x.action = traj[0][t].action;
      x.reward = traj[0][t].total;
      buf.push_back(x);
    }
    std::vector<const Transition*> batch;
    for (auto& x : buf) batch.push_back(&x);
    const double loss = tr.update(batch, 0.9);
    if (!(loss >= 0.0) || tr.updates() != 1) {
      std::printf("{\"error\": \"dqn update\"}\n");
      return 3;
    }
  }
  std::printf("{\"status\": %d, \"completed\": %lld, \"ticks\": %lld, \"total_e2e_s\": %.17g, "
              "\"total_ttft_s\": %.17g, \"makespan_s\": %.17g, \"total_tokens\": %lld}\n",
              s.status, (long long)s.completed, (long long)s.ticks, s.total_e2e_s,
              s.total_ttft_s, s.makespan_s, (long long)s.total_tokens);
  return s.status == RS_REPLAY_FINISHED ? 0 : 2;
}
