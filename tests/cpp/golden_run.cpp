// C++ user of the engine through include/routesim_b200.hpp, written the way
// the reference's own golden test is (test_harness.cpp:212-231): JSQ, m=2,
// n=12, lambda=12, seed 777.  Prints the replay's statistics as JSON.
#include <cstdio>

#include "routesim_b200.hpp"

int main() {
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
  std::printf("{\"status\": %d, \"completed\": %lld, \"ticks\": %lld, \"total_e2e_s\": %.17g, "
              "\"total_ttft_s\": %.17g, \"makespan_s\": %.17g, \"total_tokens\": %lld}\n",
              s.status, (long long)s.completed, (long long)s.ticks, s.total_e2e_s,
              s.total_ttft_s, s.makespan_s, (long long)s.total_tokens);
  return s.status == RS_REPLAY_FINISHED ? 0 : 2;
}
