/*
 * rs_abi.h — C ABI of the B200 batched trace-replay engine for the routesim
 * router/simulator hot path (arXiv 2408.13510 reference, /root/reference/proj).
 *
 * One call replays a whole batch of independent (trace x policy x seed)
 * episodes.  A per-tick `decide()` across the ABI would cost one launch per
 * tick, so the boundary is batch level: it replaces the reference's
 * sequential loop of
 *     ClusterSim sim(cfg, trace);                 env.hpp:174-194
 *     auto policy = make_policy(name, ...);       policies.hpp:230-245
 *     sim.run_policy(*policy, max_ticks);         env.hpp:326-337
 * over seeds, as done by evaluate_policy()  (experiment.hpp:648-670) and
 * run_matrix() (experiment.hpp:389-413).  Each entry point below cites the
 * reference interface it replaces.
 *
 * Conventions
 *  - Plain C types only; every struct is fixed-size with explicit padding so
 *    that ctypes / cgo / JNI bindings can mirror it byte for byte.
 *  - Device entry points take caller-owned device buffers and a cudaStream_t
 *    passed as void*; they never allocate inside the hot call.
 *  - Errors: an rs_status code; the message of the last failure on the
 *    calling thread is available from rs_last_error().  Per-replay failures
 *    of the reference (exceptions thrown inside one episode) are reported as
 *    per-replay status codes in rs_replay_stats.status, never as a call
 *    failure.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns RS_ERR_NO_DEVICE.
 */
#ifndef RS_ABI_H_
#define RS_ABI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 1u

#define RS_MAX_BUCKETS 8   /* predictor / state bucket edges            */
#define RS_MAX_BANDS 8     /* empirical-predictor prompt bands          */
#define RS_NUM_TASKS 5     /* TaskKind, request.hpp:11-17               */
#define RS_MAX_LAYERS 4    /* Q-network affine layers (dqn uses 3)      */
#define RS_MAX_WIDTH 512   /* widest Q-network layer supported on device */

typedef enum rs_status {
  RS_OK = 0,
  RS_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  RS_ERR_CUDA = 2,
  RS_ERR_UNSUPPORTED = 3,      /* valid for the reference, outside engine limits */
  RS_ERR_NO_DEVICE = 4,
  RS_ERR_OUT_OF_MEMORY = 5,
  RS_ERR_INTERNAL = 6
} rs_status;

/* make_policy names (policies.hpp:230-245) + the workload-aware router and
 * the RL adapter RlPolicy (dqn.hpp:282-295). */
typedef enum rs_policy {
  RS_POLICY_ROUND_ROBIN = 0,
  RS_POLICY_DEDICATED_SMALL_LARGE = 1,
  RS_POLICY_DECODE_BALANCER = 2,
  RS_POLICY_JSQ = 3,
  RS_POLICY_MAX_CAPACITY = 4,
  RS_POLICY_MIN_MIN = 5,
  RS_POLICY_EARLIEST_AVAILABLE = 6,
  RS_POLICY_WORKLOAD_AWARE = 7,
  RS_POLICY_RL = 8,
  RS_POLICY_COUNT = 9
} rs_policy;

/* BatchingPolicy, instance.hpp:19 */
typedef enum rs_batching {
  RS_BATCHING_FCFS = 0,
  RS_BATCHING_BIN_PACKING = 1,
  RS_BATCHING_LEAST_WORK_LEFT = 2
} rs_batching;

/* PredictorMode, env.hpp:115; GIVEN = buckets supplied in the trace. */
typedef enum rs_predictor_mode {
  RS_PREDICTOR_SIMULATED = 0,
  RS_PREDICTOR_EMPIRICAL = 1,
  RS_PREDICTOR_GIVEN = 2
} rs_predictor_mode;

/* Per-replay outcome; the reference's exceptions inside one episode. */
typedef enum rs_replay_status {
  RS_REPLAY_FINISHED = 0,        /* run_policy() returned true               */
  RS_REPLAY_MAX_TICKS = 1,       /* run_policy() returned false (starvation) */
  RS_REPLAY_NOT_ADMISSIBLE = 2,  /* logic_error, instance.hpp:209-211        */
  RS_REPLAY_BAD_ACTION = 3,      /* invalid_argument, env.hpp:252-254        */
  RS_REPLAY_CAPACITY = 4,        /* engine limit exceeded    */
  RS_REPLAY_NOT_RUN = 5,
  RS_REPLAY_INVALID_TRACE = 6    /* decreasing arrivals / tokens out of range */
} rs_replay_status;

/* HardwareProfile, latency.hpp:16-35 */
typedef struct rs_profile {
  double prompt_time_per_token;
  double prompt_time_intercept;
  double decode_time_per_token;
  double decode_time_base;
} rs_profile;

/* Thresholds, latency.hpp:38-51 */
typedef struct rs_thresholds {
  double heavy_prompt_seconds;
  double heavy_decode_seconds;
} rs_thresholds;

/* ImpactConfig, impact.hpp:14-32 */
typedef struct rs_impact {
  double grad1;
  double grad2;
  double epsilon_s;
  double alpha;
  int32_t prompt_exponent;
  int32_t _pad;
} rs_impact;

/* Everything ClusterConfig (env.hpp:117-147) + InstanceConfig
 * (instance.hpp:37-54) + the policy choice carry for one batch. */
typedef struct rs_batch_cfg {
  uint32_t abi_version;      /* = RS_ABI_VERSION */
  int32_t policy;            /* rs_policy */

  rs_profile profile;
  rs_thresholds thresholds;
  rs_impact impact;

  int64_t kv_capacity_tokens;   /* InstanceConfig */
  int32_t max_batch_size;
  int32_t batching;             /* rs_batching */
  int32_t chunk_size;           /* 0 = std::nullopt (no chunked prefill) */
  int32_t num_instances;        /* m */
  double delta_t;               /* router tick, seconds */

  int32_t n_predictor_edges;    /* BucketScheme::predictor_default {0,250,1000,4000} */
  int32_t n_state_edges;        /* BucketScheme::state_default {0,256,2048} */
  int64_t predictor_edges[RS_MAX_BUCKETS];
  int64_t state_edges[RS_MAX_BUCKETS];
  int64_t predictor_top_cap;    /* kMaxDecodeTokens = 4096, workload.hpp:23 */

  int32_t predictor_mode;       /* rs_predictor_mode */
  int32_t n_band_edges;         /* EmpiricalPredictor bands, predictor.hpp:162-164 */
  double accuracy[RS_NUM_TASKS];/* AccuracyTable per TaskKind (simulated mode) */
  int64_t band_edges[RS_MAX_BANDS];
  /* EmpiricalPredictor::predict() resolved per (task, band) on the host,
   * fallbacks included (predictor.hpp:146-158). */
  uint8_t empirical_table[RS_NUM_TASKS][RS_MAX_BANDS];

  /* RL router: Mlp dims (mlp.hpp:19-30) and the flat parameter vector in the
   * reference layout (per layer: W row-major [out][in], then b[out]).
   * Device pointer for rs_replay_batch, host pointer for the _host variant. */
  int32_t rl_num_layers;        /* number of affine layers (dims - 1) */
  int32_t rl_dims[RS_MAX_LAYERS + 1];
  /* Every weight finite: the device forward skips exact-zero inputs, which
   * equals the reference's w * 0 only for finite w (the _host entry points
   * reject non-finite weights with RS_ERR_UNSUPPORTED). */
  const double* rl_params;
  double rl_epsilon;            /* 0 => DqnAgent::greedy; >0 => DqnAgent::act */

  int64_t max_ticks;            /* run_policy(policy, max_ticks), default 10'000'000 */
  uint32_t flags;               /* RS_FLAG_* */
  int32_t _pad1;
} rs_batch_cfg;

#define RS_FLAG_NONE 0u
/* rs_replay_batch draws the decode-length predictions itself, at arrival
 * injection as the reference does (env.hpp:357-375), writing them to
 * out->predicted_bucket; rs_predict_buckets is then not needed.  Needs
 * trace->predictor_seed (simulated) or trace->given_bucket (given). */
#define RS_FLAG_PREDICT_INLINE 1u
/* ClusterConfig::record_trajectory (env.hpp:131, 305-319): set by
 * rs_replay_trajectory, which also evaluates the Eq. 3 reward per tick and
 * records TickRecords; rs_replay_batch rejects it. */
#define RS_FLAG_RECORD_TRAJECTORY 2u

/* ShapingMode, env.hpp:22-38 */
typedef enum rs_shaping {
  RS_SHAPING_NONE = 0,
  RS_SHAPING_ADDITIVE = 1,
  RS_SHAPING_GUIDED = 2
} rs_shaping;

/* RewardConfig (env.hpp:40-71) + episode_k, and the TickRecord trajectory
 * (env.hpp:150-168) of every replay, device buffers.  Replay r's tick t
 * (TickRecord::tick, 1-based) is record r*capacity + (t-1); the m-wide
 * fields hold instance i of that record at (r*capacity + t-1)*m + i.  Ticks
 * past `capacity` are simulated but not recorded (rs_replay_stats.ticks has
 * the true count).  Any array may be NULL (not recorded); when both
 * queue_penalty and reward are NULL the O(active) Eq. 3 scan is skipped. */
typedef struct rs_trajectory {
  int64_t capacity;           /* records per replay */
  double r_w;                 /* RewardConfig::r_w = 60 */
  double gamma;               /* RewardConfig::gamma = 0.99 */
  double beta_d;              /* RewardConfig::beta_d = 0.5 */
  int32_t shaping;            /* rs_shaping, default GUIDED */
  int32_t episode_k;          /* ClusterConfig::episode_k (c_k = shaping_coefficient(k)) */
  double* time_s;             /* TickRecord::time (router clock after the tick) */
  int32_t* action;            /* TickRecord::action */
  double* queue_penalty;      /* RewardBreakdown::queue_penalty (Eq. 3 scan) */
  int32_t* completions;       /* RewardBreakdown::completions */
  double* h;                  /* RewardBreakdown::h (heuristic_h, impact.hpp:94-103) */
  double* shaping_term;       /* RewardBreakdown::shaping = c_k * h */
  double* reward;             /* RewardBreakdown::total */
  uint8_t* infeasible_route;  /* RewardBreakdown::infeasible_route */
  int32_t* router_queue;      /* TickRecord::router_queue_len */
  int32_t* tokens_emitted;    /* TickRecord::tokens_emitted */
  int32_t* instance_running;  /* [.. x m] TickRecord::instance_running */
  int32_t* instance_waiting;  /* [.. x m] TickRecord::instance_waiting */
} rs_trajectory;

/* Struct-of-arrays trace batch, CSR over replays.  Request i of replay r is
 * element offsets[r] + i.  Field meaning follows Request (request.hpp:42-69). */
typedef struct rs_trace_soa {
  int32_t num_replays;
  int32_t _pad;
  int64_t total_requests;
  const int64_t* offsets;         /* [R+1] */
  const double* arrival_s;        /* non-decreasing within each replay */
  const int32_t* prompt_tokens;   /* >= 1 */
  const int32_t* decode_tokens;   /* true decode length, >= 1 */
  const uint8_t* task;            /* TaskKind */
  const uint8_t* given_bucket;    /* RS_PREDICTOR_GIVEN only, else NULL */
  const uint64_t* predictor_seed; /* [R] Rng seed of the simulated predictor */
  const uint64_t* policy_seed;    /* [R] Rng seed for epsilon-greedy, or NULL */
} rs_trace_soa;

/* Per-request results (Request's mutable fields), same CSR indexing. */
typedef struct rs_req_out {
  int32_t* instance;        /* assigned_instance, -1 if never routed */
  double* routed_s;         /* routed_time_s, -1 if never routed */
  double* first_token_s;    /* first_token_time_s, -1 if none */
  double* completion_s;     /* completion_time_s, -1 if not completed */
  int32_t* preemptions;     /* preemption_count */
  uint8_t* predicted_bucket;/* predicted_bucket written by inject_arrivals */
} rs_req_out;

/* Per-replay statistics (one record per replay, 256 bytes).  Sums follow
 * compute_metrics (metrics.hpp:84-162): sequential in pool-index order over
 * completed requests, so means are bit-identical to the reference. */
typedef struct rs_replay_stats {
  int64_t ticks;                /* decisions == ClusterSim::tick() */
  int64_t routed;
  int64_t infeasible;           /* ClusterSim::infeasible_routes() */
  int64_t completed;
  uint64_t decision_hash;       /* FNV-1a over the per-tick actions */
  int64_t sum_router_queue;     /* sum over ticks of router queue length */
  int64_t sum_instance_waiting; /* sum over ticks and instances of waiting size */
  int64_t total_preemptions;
  int64_t total_tokens;
  int64_t tbt_count;
  double clock;                 /* router clock at exit */
  double total_e2e_s;
  double total_ttft_s;
  double total_tbt_s;
  double total_router_wait_s;
  double first_arrival_s;
  double last_completion_s;
  double makespan_s;
  double e2e_p50, e2e_p90, e2e_p99;
  double ttft_p50, ttft_p90, ttft_p99;
  double tbt_p50, tbt_p90, tbt_p99;
  int32_t status;               /* rs_replay_status */
  int32_t error_instance;       /* instance that raised, or -1 */
  int32_t percentiles_valid;
  int32_t _pad0;
  int64_t injected;             /* requests that reached the router queue */
  int64_t qnet_macs;            /* RL: multiply-adds the Q-network forwards executed
                                   (exact-zero inputs skipped, a repeated state's
                                   action reused); 0 for the heuristics */
  int32_t _pad[2];
} rs_replay_stats;

/* ---- identity / device ------------------------------------------------ */
uint32_t rs_abi_version(void);
/* Number of usable sm_100 devices (0 on a host without one). */
int32_t rs_device_count(void);
/* Copies the calling thread's last error message (NUL-terminated). */
rs_status rs_last_error(char* buf, size_t len);

/* Fills a config with the reference defaults (ExperimentConfig/ClusterConfig
 * field initialisers, experiment.hpp:45-76, env.hpp:117-130): profile,
 * thresholds, impact, KV 16384, batch 128, FCFS, m = 4, dt = 0.02, default
 * bucket schemes, dataset_default accuracy, max_ticks 10M. */
rs_status rs_default_config(rs_batch_cfg* cfg);
/* Same validation as ClusterConfig::validate (env.hpp:133-146) plus engine
 * limits.  Returns RS_ERR_INVALID_ARGUMENT / RS_ERR_UNSUPPORTED. */
rs_status rs_validate_config(const rs_batch_cfg* cfg);

/* ---- device entry points (caller-owned device memory) ------------------ */

/* Scratch bytes rs_replay_batch needs for this batch shape. */
rs_status rs_workspace_size(const rs_batch_cfg* cfg, int32_t num_replays,
                            int64_t total_requests, size_t* bytes);

/* Kernel (d): decode-length-predictor bucket lookup for every request of
 * every replay, in arrival order per replay.  Replaces the prediction part of
 * ClusterSim::inject_arrivals (env.hpp:357-375): BucketScheme::bucket_of
 * (predictor.hpp:34-40), predict_simulated (predictor.hpp:98-110) or
 * EmpiricalPredictor::predict (predictor.hpp:146-158). */
rs_status rs_predict_buckets(const rs_batch_cfg* cfg, const rs_trace_soa* trace,
                             uint8_t* predicted_bucket, void* cuda_stream);

/* Kernels (a)+(b)+(c): replay every episode of the batch to completion (or
 * max_ticks) under cfg->policy.  Replaces ClusterSim::run_policy
 * (env.hpp:326-337) over a batch of independent ClusterSims.  Requires
 * predicted buckets in out->predicted_bucket (rs_predict_buckets, or a copy
 * of trace->given_bucket).  Per-replay statistics go to `stats` (device). */
rs_status rs_replay_batch(const rs_batch_cfg* cfg, const rs_trace_soa* trace,
                          rs_req_out* out, rs_replay_stats* stats,
                          void* workspace, size_t workspace_bytes,
                          void* cuda_stream);

/* rs_replay_batch with ClusterConfig::record_trajectory (cfg->flags must
 * carry RS_FLAG_RECORD_TRAJECTORY): additionally evaluates, per tick, the
 * reward of ClusterSim::step (env.hpp:257-303: Eq. 3 queue penalty over the
 * arrived, uncompleted requests in pool-index order, completions, the
 * shaping term c_k * heuristic_h of the routed head) and writes the
 * TickRecords (env.hpp:305-319) into `traj` (device buffers).  Always runs
 * the general (warp-per-replay) kernel. */
rs_status rs_replay_trajectory(const rs_batch_cfg* cfg, const rs_trace_soa* trace,
                               rs_req_out* out, rs_replay_stats* stats,
                               const rs_trajectory* traj, void* workspace,
                               size_t workspace_bytes, void* cuda_stream);

/* Pinned host memory for the _host entry points (cudaHostAlloc). */
void* rs_host_alloc(size_t bytes);
void rs_host_free(void* p);

/* Host-buffer convenience: H2D, predictor, replay, stats, D2H on `device`.
 * This is the reference-facing call (evaluate_policy over seeds).  Any of the
 * out arrays may be NULL to skip its copy-back. */
rs_status rs_replay_batch_host(const rs_batch_cfg* cfg, const rs_trace_soa* trace,
                               rs_req_out* out, rs_replay_stats* stats,
                               int32_t device);

/* rs_replay_batch_host sharded over several devices of this process
 * (evaluate_policy's independent seed loop,
 * experiment.hpp:648-670, run concurrently as SPEC.md:523-524 allows):
 * replays [k*S, (k+1)*S), S = ceil(num_replays / ndev), run on devices[k],
 * each device on its own stream and host thread with no collective on the
 * data path; the per-replay statistics are then all-gathered over NCCL
 * (ncclCommInitAll over `devices`, libnccl.so.2 opened at first use) and
 * copied to `stats` from devices[0].  Results are identical to one
 * rs_replay_batch_host call over the whole batch.  `devices` must be
 * distinct; RS_ERR_UNSUPPORTED when NCCL cannot be loaded. */
rs_status rs_replay_batch_multi(const rs_batch_cfg* cfg, const rs_trace_soa* trace,
                                rs_req_out* out, rs_replay_stats* stats,
                                const int32_t* devices, int32_t ndev);

/* rs_replay_trajectory with host buffers (trace, outputs and the
 * trajectory arrays in `traj`), on `device`; the reference-facing form of
 * ClusterSim::trajectory() (env.hpp:203) for a batch. */
rs_status rs_replay_trajectory_host(const rs_batch_cfg* cfg, const rs_trace_soa* trace,
                                    rs_req_out* out, rs_replay_stats* stats,
                                    const rs_trajectory* traj, int32_t device);

/* Standalone stage kernels for per-stage parity (host buffers in/out). */
/* Mlp::forward over `batch` state vectors (mlp.hpp:54-68). */
rs_status rs_mlp_forward_host(const rs_batch_cfg* cfg, const double* states,
                              int32_t batch, double* q_out, int32_t* greedy_out,
                              int32_t device);

/* ---- host-side workload generation (not on the hot path) --------------- */

/* generate_mixture (workload.hpp:220-245) over dataset_task_specs
 * (workload.hpp:176-186) with the given task weights (NULL = Table 1 sample
 * counts, i.e. generate_dataset_mixture, workload.hpp:247-258), seeded as
 * build_workload does: Rng(mix_seed(seed, 0xB00C)) (experiment.hpp:291-305).
 * process: 0 = Poisson, 1 = fixed interval. */
rs_status rs_generate_mixture(const rs_profile* profile,
                              const rs_thresholds* thresholds,
                              const double* task_weights, uint64_t seed,
                              int64_t n, double rate_per_s, int32_t process,
                              double* arrival_s, int32_t* prompt_tokens,
                              int32_t* decode_tokens, uint8_t* task);

/* Same, for many seeds at once on host threads (threads <= 0: all cores). */
rs_status rs_generate_mixture_batch(const rs_profile* profile,
                                    const rs_thresholds* thresholds,
                                    const double* task_weights,
                                    const uint64_t* seeds, int32_t num_seeds,
                                    int64_t n, double rate_per_s,
                                    int32_t process, int32_t threads,
                                    double* arrival_s, int32_t* prompt_tokens,
                                    int32_t* decode_tokens, uint8_t* task);

/* EmpiricalPredictor::fit (predictor.hpp:119-142) on a training trace and
 * predict() (predictor.hpp:146-158) resolved per (task, prompt band) into
 * cfg->empirical_table, using cfg's predictor and band edges; sets
 * cfg->predictor_mode = RS_PREDICTOR_EMPIRICAL. */
rs_status rs_empirical_fit_trace(rs_batch_cfg* cfg, int64_t n, const int32_t* prompt_tokens,
                                 const int32_t* decode_tokens, const uint8_t* task);

/* run_experiment's empirical predictor (experiment.hpp:341-351): the fit on
 * n_train (the reference uses 20000) Table-1-mixture requests drawn from
 * Rng(mix_seed(seed, 0xF17)). */
rs_status rs_empirical_fit(rs_batch_cfg* cfg, uint64_t seed, int64_t n_train);

/* Mlp::random (mlp.hpp:32-45) as DqnAgent's constructor uses it
 * (dqn.hpp:60-65): Rng(seed), w = (2u - 1) * sqrt(2 / fan_in), b = 0. */
rs_status rs_mlp_random_init(const int32_t* dims, int32_t num_layers, uint64_t seed,
                             double* params_out);

/* ---- DQN training step ------------------------ */

/* A sampled batch of transitions (Transition, replay.hpp:12-18), struct of
 * arrays: state / next_state are [batch x state_dim] row-major. */
typedef struct rs_dqn_batch {
  int32_t batch;
  int32_t _pad;
  const double* state;
  const int32_t* action;
  const double* reward;
  const double* next_state;
  const uint8_t* done;
} rs_dqn_batch;

/* DqnAgent's trainable state: online / target networks (reference flat
 * layout, as rs_batch_cfg.rl_params), AdamOptimizer moments and step count
 * (mlp.hpp:159-189), updates_ and AgentConfig's learning rate / target sync
 * interval (dqn.hpp:22-30).  Array pointers are device memory for
 * rs_dqn_update, host memory for rs_dqn_update_host; the counters are
 * advanced by the call. */
typedef struct rs_dqn_state {
  double* online;
  double* target;
  double* adam_m;
  double* adam_v;
  int64_t adam_t;                /* AdamOptimizer::t_ before the step */
  int64_t updates;               /* DqnAgent::updates_ before the step */
  int64_t target_sync_interval;  /* AgentConfig, default 1000 */
  double learning_rate;          /* AgentConfig, default 1e-3 */
} rs_dqn_state;

/* Scratch bytes rs_dqn_update needs (per-sample activations and deltas). */
rs_status rs_dqn_workspace_size(const rs_batch_cfg* cfg, int32_t batch, size_t* bytes);

/* DqnAgent::update (dqn.hpp:107-127) after ReplayBuffer::sample: double-DQN
 * targets (online argmax on s', target-net value, reward + discount * Q),
 * Mlp::loss_and_gradient (mean Huber, mlp.hpp:78-136), AdamOptimizer::step
 * (mlp.hpp:163-177), ++updates_ and sync_target every target_sync_interval
 * updates — bit-identical to the reference.  Network shape from
 * cfg->rl_num_layers / rl_dims.  *loss_out (device) receives the batch loss. */
rs_status rs_dqn_update(const rs_batch_cfg* cfg, const rs_dqn_batch* batch, rs_dqn_state* state,
                        double discount, double* loss_out, void* workspace,
                        size_t workspace_bytes, void* cuda_stream);

/* Same with host buffers (copied in and out every call) on `device`. */
rs_status rs_dqn_update_host(const rs_batch_cfg* cfg, const rs_dqn_batch* batch,
                             rs_dqn_state* state, double discount, double* loss_out,
                             int32_t device);

/* ---- host-side report layer (one replay) ------------------------------- */

/* compute_metrics + emit_report (metrics.hpp:84-238) for one replay of a
 * finished batch: writes `dir`/summary.json (report_to_json(...).dump(2),
 * byte-identical to the reference's nlohmann serialisation), requests.csv and
 * timeseries.csv ("%.17g" doubles, format_double).  Inputs are the replay's
 * slice of the trace and of the per-request outputs (host arrays), its
 * rs_replay_stats record (the device's sums and percentiles are used), and
 * optionally its trajectory (host arrays, record t-1 for tick t, traj_len
 * records): with traj == NULL the report is that of record_trajectory =
 * false (mean_router_queue / mean_instance_waiting 0, timeseries.csv
 * header only), as run_matrix / evaluate_policy produce.
 * RS_ERR_INVALID_ARGUMENT when no request completed (compute_metrics'
 * invalid_argument) or a file cannot be written (emit_report's
 * runtime_error). */
rs_status rs_emit_report(const char* dir, const rs_batch_cfg* cfg, int64_t n,
                         const double* arrival_s, const int32_t* prompt_tokens,
                         const int32_t* decode_tokens, const uint8_t* task,
                         const int32_t* instance, const double* routed_s,
                         const double* first_token_s, const double* completion_s,
                         const int32_t* preemptions, const rs_replay_stats* stats,
                         const rs_trajectory* traj, int64_t traj_len);

/* mix_seed (rng.hpp:11-16). */
uint64_t rs_mix_seed(uint64_t seed, uint64_t stream);

/* heavy_decode_token_cutoff (latency.hpp:132-138), used by
 * dedicated_small_large. */
int64_t rs_heavy_decode_cutoff(const rs_profile* profile,
                               const rs_thresholds* thresholds);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* RS_ABI_H_ */
