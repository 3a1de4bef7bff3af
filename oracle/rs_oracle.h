/* oracle/rs_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference routesim hot path (ClusterSim
 * tick loop, Instance continuous-batching step, the seven make_policy
 * heuristics, the workload-aware router of SURVEY.md Appendix B, the RL
 * greedy / epsilon-greedy adapter, the decode-length predictor) used ONLY by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker.  The product (paper_2408_13510_b200/) never links or calls it.
 *
 * Parity pinned: every function is checked against the compiled reference
 * (oracle/_ref/librs_ref.so, differential tests in tests/test_oracle.py) and
 * against the frozen fixtures in tests/golden/ (mini_summary.json
 * reproduction, per-request dumps made by tests/golden/make_golden.py).
 */
#ifndef RS_ORACLE_H_
#define RS_ORACLE_H_

#include <stdint.h>

#include "../include/rs_abi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One replay, ClusterSim::run_policy (env.hpp:326-337).  Any output pointer
 * may be NULL.  Returns 0, or -1 on an invalid configuration. */
int ora_run_replay(const rs_batch_cfg* cfg, int64_t n, const double* arrival,
                   const int32_t* prompt, const int32_t* decode,
                   const uint8_t* task, const uint8_t* given_bucket,
                   uint64_t predictor_seed, uint64_t policy_seed,
                   int32_t* instance, double* routed, double* first,
                   double* completion, int32_t* preemptions,
                   uint8_t* predicted, rs_replay_stats* stats,
                   int32_t* action_log, int64_t action_cap);

/* ora_run_replay with record_trajectory: the Eq. 3 reward and TickRecords
 * (env.hpp:257-319) of every tick into `traj` (host arrays; record t-1 for
 * tick t, m-wide fields at (t-1)*m + i). */
int ora_run_trajectory(const rs_batch_cfg* cfg, int64_t n, const double* arrival,
                       const int32_t* prompt, const int32_t* decode,
                       const uint8_t* task, const uint8_t* given_bucket,
                       uint64_t predictor_seed, uint64_t policy_seed,
                       int32_t* instance, double* routed, double* first,
                       double* completion, int32_t* preemptions,
                       uint8_t* predicted, rs_replay_stats* stats,
                       const rs_trajectory* traj);

/* inject_arrivals' prediction for every request in index order
 * (env.hpp:357-375). */
int ora_predict_buckets(const rs_batch_cfg* cfg, int64_t n,
                        const int32_t* prompt, const int32_t* decode,
                        const uint8_t* task, const uint8_t* given_bucket,
                        uint64_t predictor_seed, uint8_t* predicted);

/* Mlp::forward + argmax_action (mlp.hpp:54-68, dqn.hpp:82-90). */
int ora_mlp_forward(const rs_batch_cfg* cfg, const double* states,
                    int32_t batch, double* q_out, int32_t* greedy_out);

/* std::mt19937_64 outputs (rng.hpp:21-27). */
void ora_mt19937_64(uint64_t seed, int64_t count, uint64_t* out);

/* mix_seed (rng.hpp:11-16). */
uint64_t ora_mix_seed(uint64_t seed, uint64_t stream);

/* Nearest-rank percentile as aggregate_of (metrics.hpp:62-80). */
double ora_nearest_rank(const double* sorted_values, int64_t n, double q);

#ifdef __cplusplus
}
#endif

#endif
