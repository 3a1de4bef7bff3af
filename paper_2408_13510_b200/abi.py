"""ctypes mirror of include/rs_abi.h (the engine's C ABI).

Struct layouts are byte-for-byte those of the header; tests/test_abi.py checks
the sizes and every exported symbol.  Nothing here computes: the product path
is the CUDA library `_lib/librs_b200.so`; this module only loads it and
builds argument structs.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
# RS_B200_LIB: load another build of the library (A/B timing of kernel variants)
LIB_PATH = Path(os.environ.get("RS_B200_LIB", PKG_DIR / "_lib" / "librs_b200.so"))

RS_ABI_VERSION = 1
RS_MAX_BUCKETS = 8
RS_MAX_BANDS = 8
RS_NUM_TASKS = 5
RS_MAX_LAYERS = 4
RS_MAX_WIDTH = 512

# rs_status
RS_OK = 0
RS_ERR_INVALID_ARGUMENT = 1
RS_ERR_CUDA = 2
RS_ERR_UNSUPPORTED = 3
RS_ERR_NO_DEVICE = 4
RS_ERR_OUT_OF_MEMORY = 5
RS_ERR_INTERNAL = 6

# rs_policy — make_policy names (policies.hpp:230-245) + workload_aware + rl
POLICIES = {
    "round_robin": 0,
    "dedicated_small_large": 1,
    "decode_balancer": 2,
    "jsq": 3,
    "max_capacity": 4,
    "min_min": 5,
    "earliest_available": 6,
    "workload_aware": 7,
    "rl": 8,
}
POLICY_NAMES = {v: k for k, v in POLICIES.items()}
BATCHING = {"fcfs": 0, "bin_packing": 1, "least_work_left": 2}
PRED_SIMULATED, PRED_EMPIRICAL, PRED_GIVEN = 0, 1, 2
RS_FLAG_PREDICT_INLINE = 1  # rs_replay_batch draws predictions at injection
RS_FLAG_RECORD_TRAJECTORY = 2  # ClusterConfig::record_trajectory (rs_replay_trajectory)
SHAPING = {"none": 0, "additive": 1, "guided": 2}  # ShapingMode (env.hpp:22)

# rs_replay_status
REPLAY_FINISHED = 0
REPLAY_MAX_TICKS = 1
REPLAY_NOT_ADMISSIBLE = 2
REPLAY_BAD_ACTION = 3
REPLAY_CAPACITY = 4
REPLAY_NOT_RUN = 5
REPLAY_INVALID_TRACE = 6

# Table 1 predictor accuracies (workload.hpp:165-174), TaskKind order.
DATASET_ACCURACY = (0.9310, 0.7036, 0.7992, 0.6527, 0.9506)
DATASET_SAMPLES = (7351.0, 6988.0, 6564.0, 7122.0, 3304.0)


class Profile(C.Structure):
    _fields_ = [("prompt_time_per_token", C.c_double),
                ("prompt_time_intercept", C.c_double),
                ("decode_time_per_token", C.c_double),
                ("decode_time_base", C.c_double)]


class Thresholds(C.Structure):
    _fields_ = [("heavy_prompt_seconds", C.c_double),
                ("heavy_decode_seconds", C.c_double)]


class Impact(C.Structure):
    _fields_ = [("grad1", C.c_double), ("grad2", C.c_double),
                ("epsilon_s", C.c_double), ("alpha", C.c_double),
                ("prompt_exponent", C.c_int32), ("_pad", C.c_int32)]


class BatchCfg(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32),
        ("policy", C.c_int32),
        ("profile", Profile),
        ("thresholds", Thresholds),
        ("impact", Impact),
        ("kv_capacity_tokens", C.c_int64),
        ("max_batch_size", C.c_int32),
        ("batching", C.c_int32),
        ("chunk_size", C.c_int32),
        ("num_instances", C.c_int32),
        ("delta_t", C.c_double),
        ("n_predictor_edges", C.c_int32),
        ("n_state_edges", C.c_int32),
        ("predictor_edges", C.c_int64 * RS_MAX_BUCKETS),
        ("state_edges", C.c_int64 * RS_MAX_BUCKETS),
        ("predictor_top_cap", C.c_int64),
        ("predictor_mode", C.c_int32),
        ("n_band_edges", C.c_int32),
        ("accuracy", C.c_double * RS_NUM_TASKS),
        ("band_edges", C.c_int64 * RS_MAX_BANDS),
        ("empirical_table", (C.c_uint8 * RS_MAX_BANDS) * RS_NUM_TASKS),
        ("rl_num_layers", C.c_int32),
        ("rl_dims", C.c_int32 * (RS_MAX_LAYERS + 1)),
        ("rl_params", C.POINTER(C.c_double)),
        ("rl_epsilon", C.c_double),
        ("max_ticks", C.c_int64),
        ("flags", C.c_uint32),
        ("_pad1", C.c_int32),
    ]


class TraceSoA(C.Structure):
    _fields_ = [
        ("num_replays", C.c_int32),
        ("_pad", C.c_int32),
        ("total_requests", C.c_int64),
        ("offsets", C.c_void_p),
        ("arrival_s", C.c_void_p),
        ("prompt_tokens", C.c_void_p),
        ("decode_tokens", C.c_void_p),
        ("task", C.c_void_p),
        ("given_bucket", C.c_void_p),
        ("predictor_seed", C.c_void_p),
        ("policy_seed", C.c_void_p),
    ]


class ReqOut(C.Structure):
    _fields_ = [
        ("instance", C.c_void_p),
        ("routed_s", C.c_void_p),
        ("first_token_s", C.c_void_p),
        ("completion_s", C.c_void_p),
        ("preemptions", C.c_void_p),
        ("predicted_bucket", C.c_void_p),
    ]


class ReplayStats(C.Structure):
    _fields_ = [
        ("ticks", C.c_int64),
        ("routed", C.c_int64),
        ("infeasible", C.c_int64),
        ("completed", C.c_int64),
        ("decision_hash", C.c_uint64),
        ("sum_router_queue", C.c_int64),
        ("sum_instance_waiting", C.c_int64),
        ("total_preemptions", C.c_int64),
        ("total_tokens", C.c_int64),
        ("tbt_count", C.c_int64),
        ("clock", C.c_double),
        ("total_e2e_s", C.c_double),
        ("total_ttft_s", C.c_double),
        ("total_tbt_s", C.c_double),
        ("total_router_wait_s", C.c_double),
        ("first_arrival_s", C.c_double),
        ("last_completion_s", C.c_double),
        ("makespan_s", C.c_double),
        ("e2e_p50", C.c_double), ("e2e_p90", C.c_double), ("e2e_p99", C.c_double),
        ("ttft_p50", C.c_double), ("ttft_p90", C.c_double), ("ttft_p99", C.c_double),
        ("tbt_p50", C.c_double), ("tbt_p90", C.c_double), ("tbt_p99", C.c_double),
        ("status", C.c_int32),
        ("error_instance", C.c_int32),
        ("percentiles_valid", C.c_int32),
        ("_pad0", C.c_int32),
        ("injected", C.c_int64),
        ("qnet_macs", C.c_int64),
        ("_pad", C.c_int32 * 2),
    ]


assert C.sizeof(ReplayStats) == 256, C.sizeof(ReplayStats)

# TickRecord fields of rs_trajectory: (name, numpy dtype, m-wide)
TRAJ_FIELDS = (("time_s", np.float64, False), ("action", np.int32, False),
               ("queue_penalty", np.float64, False), ("completions", np.int32, False),
               ("h", np.float64, False), ("shaping_term", np.float64, False),
               ("reward", np.float64, False), ("infeasible_route", np.uint8, False),
               ("router_queue", np.int32, False), ("tokens_emitted", np.int32, False),
               ("instance_running", np.int32, True), ("instance_waiting", np.int32, True))


class Trajectory(C.Structure):
    """rs_trajectory: RewardConfig (env.hpp:40-71) + episode_k and the
    TickRecord arrays (env.hpp:150-168)."""
    _fields_ = [("capacity", C.c_int64), ("r_w", C.c_double), ("gamma", C.c_double),
                ("beta_d", C.c_double), ("shaping", C.c_int32), ("episode_k", C.c_int32)] + [
                   (name, C.c_void_p) for name, _, _ in TRAJ_FIELDS]


class DqnBatch(C.Structure):
    """rs_dqn_batch: a sampled batch of transitions (replay.hpp:12-18)."""
    _fields_ = [("batch", C.c_int32), ("_pad", C.c_int32), ("state", C.c_void_p),
                ("action", C.c_void_p), ("reward", C.c_void_p), ("next_state", C.c_void_p),
                ("done", C.c_void_p)]


class DqnState(C.Structure):
    """rs_dqn_state: online / target nets, Adam moments and counters."""
    _fields_ = [("online", C.c_void_p), ("target", C.c_void_p), ("adam_m", C.c_void_p),
                ("adam_v", C.c_void_p), ("adam_t", C.c_int64), ("updates", C.c_int64),
                ("target_sync_interval", C.c_int64), ("learning_rate", C.c_double)]


def make_trajectory(capacity: int, replays: int, m: int, r_w: float = 60.0,
                    gamma: float = 0.99, beta_d: float = 0.5, shaping: str = "guided",
                    episode_k: int = 0, fields=None):
    """A host rs_trajectory with numpy arrays for `fields` (default all):
    returns (struct, {name: array shaped [replays, capacity(, m)]})."""
    arrays = {}
    t = Trajectory(int(capacity), r_w, gamma, beta_d, SHAPING[shaping], int(episode_k))
    for name, dt, wide in TRAJ_FIELDS:
        if fields is not None and name not in fields:
            continue
        shape = (replays, capacity, m) if wide else (replays, capacity)
        a = np.zeros(shape, dt)
        arrays[name] = a
        setattr(t, name, a.ctypes.data)
    return t, arrays

# numpy view of rs_replay_stats for arrays of records
_I64 = ("ticks", "routed", "infeasible", "completed")
STATS_DTYPE = np.dtype(
    [(n, np.int64) for n in _I64] + [("decision_hash", np.uint64)]
    + [(n, np.int64) for n in ("sum_router_queue", "sum_instance_waiting",
                               "total_preemptions", "total_tokens", "tbt_count")]
    + [(n, np.float64) for n in ("clock", "total_e2e_s", "total_ttft_s", "total_tbt_s",
                                 "total_router_wait_s", "first_arrival_s",
                                 "last_completion_s", "makespan_s", "e2e_p50", "e2e_p90",
                                 "e2e_p99", "ttft_p50", "ttft_p90", "ttft_p99", "tbt_p50",
                                 "tbt_p90", "tbt_p99")]
    + [("status", np.int32), ("error_instance", np.int32), ("percentiles_valid", np.int32),
       ("_pad0", np.int32), ("injected", np.int64), ("qnet_macs", np.int64),
       ("_pad", np.int32, (2,))])
assert STATS_DTYPE.itemsize == 256


def default_config(policy: str = "round_robin", num_instances: int = 4) -> BatchCfg:
    """ExperimentConfig defaults (experiment.hpp:45-76) as an rs_batch_cfg.

    Mirrors rs_default_config() in the C library (checked equal in tests)."""
    c = BatchCfg()
    c.abi_version = RS_ABI_VERSION
    c.policy = POLICIES[policy]
    c.profile = Profile(3.2e-4, 0.026, 3.3e-5, 0.0167)       # latency.hpp:17-20
    c.thresholds = Thresholds(0.5, 5.0)                        # latency.hpp:39-40
    c.impact = Impact(3.2e-4, 3.3e-5, 0.5, 0.5, 2, 0)          # impact.hpp:15-19
    c.kv_capacity_tokens = 16384                               # instance.hpp:38
    c.max_batch_size = 128
    c.batching = BATCHING["fcfs"]
    c.chunk_size = 0
    c.num_instances = num_instances
    c.delta_t = 0.02                                           # env.hpp:124
    c.n_predictor_edges = 4
    for i, e in enumerate((0, 250, 1000, 4000)):               # predictor.hpp:55
        c.predictor_edges[i] = e
    c.n_state_edges = 3
    for i, e in enumerate((0, 256, 2048)):                     # predictor.hpp:59
        c.state_edges[i] = e
    c.predictor_top_cap = 4096                                 # workload.hpp:23
    c.predictor_mode = PRED_SIMULATED
    for i, a in enumerate(DATASET_ACCURACY):                   # experiment.hpp:62
        c.accuracy[i] = a
    c.n_band_edges = 7
    for i, e in enumerate((0, 32, 64, 128, 256, 512, 1024)):   # predictor.hpp:162-164
        c.band_edges[i] = e
    c.rl_num_layers = 0
    c.rl_epsilon = 0.0
    c.max_ticks = 10_000_000                                   # env.hpp:326
    c.flags = 0
    return c


def set_rl(cfg: BatchCfg, dims, params: np.ndarray) -> np.ndarray:
    """Attach a Q-network (reference flat layout).  Returns the contiguous
    fp64 array that must outlive every call using `cfg`."""
    p = np.ascontiguousarray(params, dtype=np.float64)
    cfg.rl_num_layers = len(dims) - 1
    for i, d in enumerate(dims):
        cfg.rl_dims[i] = int(d)
    cfg.rl_params = p.ctypes.data_as(C.POINTER(C.c_double))
    return p


def mlp_param_count(dims) -> int:
    return sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 1))


def state_dimension(m: int, n_state_edges: int = 3) -> int:
    """state_dimension (env.hpp:78-80)."""
    return m * (3 + n_state_edges) + 3


def mix_seed(seed: int, stream: int) -> int:
    """mix_seed (rng.hpp:11-16) in pure Python (host-side seed derivation)."""
    M = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (stream + 1)) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


_LIB = None


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load the engine's C-ABI library (fails loudly if it is not built)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(f"engine library missing: {p} (run __graft_entry__.build())")
    if path is None:
        try:  # a library older than its sources is almost always a mistake
            from . import build as _build
            stamp = p.parent / ".stamp"
            if stamp.exists() and stamp.read_text() != _build._digest():
                import warnings
                warnings.warn(f"{p} is older than its sources (run __graft_entry__.build())")
        except OSError:
            pass
    lib = C.CDLL(str(p))
    _declare(lib)
    if path is None:
        _LIB = lib
    return lib


EXPORTED_SYMBOLS = (
    "rs_abi_version", "rs_device_count", "rs_last_error", "rs_default_config",
    "rs_validate_config", "rs_workspace_size", "rs_predict_buckets",
    "rs_replay_batch", "rs_replay_batch_host", "rs_mlp_forward_host",
    "rs_generate_mixture", "rs_generate_mixture_batch", "rs_mix_seed",
    "rs_heavy_decode_cutoff", "rs_host_alloc", "rs_host_free", "rs_mlp_random_init",
    "rs_replay_trajectory", "rs_replay_trajectory_host", "rs_emit_report",
    "rs_dqn_workspace_size", "rs_dqn_update", "rs_dqn_update_host",
    "rs_empirical_fit", "rs_empirical_fit_trace", "rs_replay_batch_multi",
)


def _declare(lib: C.CDLL) -> None:
    P = C.POINTER
    lib.rs_abi_version.restype = C.c_uint32
    lib.rs_device_count.restype = C.c_int32
    lib.rs_last_error.argtypes = [C.c_char_p, C.c_size_t]
    lib.rs_default_config.argtypes = [P(BatchCfg)]
    lib.rs_validate_config.argtypes = [P(BatchCfg)]
    lib.rs_workspace_size.argtypes = [P(BatchCfg), C.c_int32, C.c_int64, P(C.c_size_t)]
    lib.rs_predict_buckets.argtypes = [P(BatchCfg), P(TraceSoA), C.c_void_p, C.c_void_p]
    lib.rs_replay_batch.argtypes = [P(BatchCfg), P(TraceSoA), P(ReqOut), C.c_void_p,
                                    C.c_void_p, C.c_size_t, C.c_void_p]
    lib.rs_replay_batch_host.argtypes = [P(BatchCfg), P(TraceSoA), P(ReqOut), C.c_void_p,
                                         C.c_int32]
    if hasattr(lib, "rs_replay_batch_multi"):  # (older builds loaded for A/B timing lack it)
        lib.rs_replay_batch_multi.argtypes = [P(BatchCfg), P(TraceSoA), P(ReqOut), C.c_void_p,
                                              C.c_void_p, C.c_int32]
    lib.rs_replay_trajectory.argtypes = [P(BatchCfg), P(TraceSoA), P(ReqOut), C.c_void_p,
                                         P(Trajectory), C.c_void_p, C.c_size_t, C.c_void_p]
    lib.rs_replay_trajectory_host.argtypes = [P(BatchCfg), P(TraceSoA), P(ReqOut), C.c_void_p,
                                              P(Trajectory), C.c_int32]
    lib.rs_emit_report.argtypes = [C.c_char_p, P(BatchCfg), C.c_int64] + [C.c_void_p] * 10 + [
        P(Trajectory), C.c_int64]
    lib.rs_dqn_workspace_size.argtypes = [P(BatchCfg), C.c_int32, P(C.c_size_t)]
    lib.rs_dqn_update.argtypes = [P(BatchCfg), P(DqnBatch), P(DqnState), C.c_double, C.c_void_p,
                                  C.c_void_p, C.c_size_t, C.c_void_p]
    lib.rs_dqn_update_host.argtypes = [P(BatchCfg), P(DqnBatch), P(DqnState), C.c_double,
                                       C.c_void_p, C.c_int32]
    lib.rs_mlp_forward_host.argtypes = [P(BatchCfg), C.c_void_p, C.c_int32, C.c_void_p,
                                        C.c_void_p, C.c_int32]
    lib.rs_generate_mixture.argtypes = [P(Profile), P(Thresholds), C.c_void_p, C.c_uint64,
                                        C.c_int64, C.c_double, C.c_int32, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
    lib.rs_generate_mixture_batch.argtypes = [P(Profile), P(Thresholds), C.c_void_p,
                                              C.c_void_p, C.c_int32, C.c_int64, C.c_double,
                                              C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p]
    lib.rs_mix_seed.restype = C.c_uint64
    lib.rs_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
    lib.rs_heavy_decode_cutoff.restype = C.c_int64
    lib.rs_heavy_decode_cutoff.argtypes = [P(Profile), P(Thresholds)]
    lib.rs_empirical_fit.argtypes = [P(BatchCfg), C.c_uint64, C.c_int64]
    lib.rs_empirical_fit_trace.argtypes = [P(BatchCfg), C.c_int64, C.c_void_p, C.c_void_p,
                                           C.c_void_p]
    lib.rs_mlp_random_init.argtypes = [C.c_void_p, C.c_int32, C.c_uint64, C.c_void_p]
    lib.rs_host_alloc.restype = C.c_void_p
    lib.rs_host_alloc.argtypes = [C.c_size_t]
    lib.rs_host_free.argtypes = [C.c_void_p]


def last_error(lib: C.CDLL) -> str:
    buf = C.create_string_buffer(1024)
    lib.rs_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


class EngineError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rs_status={status}: {msg}")
        self.status = status


def check(lib: C.CDLL, status: int) -> None:
    if status != RS_OK:
        raise EngineError(status, last_error(lib))
