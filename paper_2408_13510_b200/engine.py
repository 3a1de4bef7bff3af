"""Host-side mirror of the reference's router/simulator API over the C ABI.

Reference names are kept so harness code reads the same:

  reference (routesim, C++)                      here
  ---------------------------------------------  ------------------------------------------
  ClusterConfig (env.hpp:117-147)                ClusterConfig
  make_policy(name, ...) (policies.hpp:230-245)  make_policy(name) -> policy id (ValueError
                                                 on an unknown name, as invalid_argument)
  ClusterSim(cfg, trace) + run_policy(policy,    BatchSim(cfg, traces, seeds).run_policy(
    max_ticks) (env.hpp:174-194, 326-337)          policy, max_ticks) for a whole batch
  record_trajectory + trajectory()               BatchSim.run_trajectory(policy, capacity,
    (env.hpp:131, 203, 305-319)                    reward, episode_k)
  RewardConfig (env.hpp:40-71)                   RewardConfig
  DqnAgent::update (dqn.hpp:107-127) after      DqnTrainer.update(batch, discount)
    ReplayBuffer::sample
  evaluate_policy over seeds                     BatchSim over the seed batch
    (experiment.hpp:648-670)
  build_workload (experiment.hpp:291-305)        build_workload(seed, n, rate, ...)

Every replay runs in the sm_100a kernels of the engine library; there is no
CPU fallback (a missing library or device raises).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi


def make_policy(name: str) -> int:
    """make_policy's name registry (+ workload_aware, rl)."""
    try:
        return abi.POLICIES[name]
    except KeyError:
        raise ValueError(f"unknown routing policy: {name}") from None


@dataclass
class ClusterConfig:
    """ClusterConfig + InstanceConfig with the reference defaults."""
    num_instances: int = 4
    kv_capacity_tokens: int = 16384
    max_batch_size: int = 128
    batching: str = "fcfs"
    chunk_size: int | None = None
    delta_t: float = 0.02
    prompt_time_per_token: float = 3.2e-4
    prompt_time_intercept: float = 0.026
    decode_time_per_token: float = 3.3e-5
    decode_time_base: float = 0.0167
    heavy_prompt_seconds: float = 0.5
    heavy_decode_seconds: float = 5.0
    grad1: float = 3.2e-4
    grad2: float = 3.3e-5
    epsilon_s: float = 0.5
    alpha: float = 0.5
    prompt_exponent: int = 2
    predictor_edges: tuple = (0, 250, 1000, 4000)
    state_edges: tuple = (0, 256, 2048)
    accuracy: tuple = abi.DATASET_ACCURACY  # ExperimentConfig default
    predictor_mode: str = "simulated"

    def to_abi(self, policy: str) -> abi.BatchCfg:
        c = abi.default_config(policy, self.num_instances)
        c.kv_capacity_tokens = self.kv_capacity_tokens
        c.max_batch_size = self.max_batch_size
        c.batching = abi.BATCHING[self.batching]
        c.chunk_size = self.chunk_size or 0
        c.delta_t = self.delta_t
        c.profile = abi.Profile(self.prompt_time_per_token, self.prompt_time_intercept,
                                self.decode_time_per_token, self.decode_time_base)
        c.thresholds = abi.Thresholds(self.heavy_prompt_seconds, self.heavy_decode_seconds)
        c.impact = abi.Impact(self.grad1, self.grad2, self.epsilon_s, self.alpha,
                              self.prompt_exponent, 0)
        c.n_predictor_edges = len(self.predictor_edges)
        for i, e in enumerate(self.predictor_edges):
            c.predictor_edges[i] = e
        c.n_state_edges = len(self.state_edges)
        for i, e in enumerate(self.state_edges):
            c.state_edges[i] = e
        for i, a in enumerate(self.accuracy):
            c.accuracy[i] = a
        c.predictor_mode = {"simulated": abi.PRED_SIMULATED, "empirical": abi.PRED_EMPIRICAL,
                            "given": abi.PRED_GIVEN}[self.predictor_mode]
        return c


@dataclass
class RewardConfig:
    """RewardConfig (env.hpp:40-71) with the reference defaults."""
    r_w: float = 60.0
    gamma: float = 0.99
    beta_d: float = 0.5
    shaping: str = "guided"   # ShapingMode: none | additive | guided


@dataclass
class TraceBatch:
    """CSR batch of arrival traces (struct of arrays)."""
    offsets: np.ndarray            # int64 [R+1]
    arrival: np.ndarray            # float64
    prompt: np.ndarray             # int32
    decode: np.ndarray             # int32
    task: np.ndarray               # uint8
    given_bucket: np.ndarray | None = None

    @property
    def num_replays(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def total(self) -> int:
        return int(self.offsets[-1])

    @staticmethod
    def from_traces(traces) -> "TraceBatch":
        n = [len(t.arrival) for t in traces]
        off = np.zeros(len(traces) + 1, np.int64)
        off[1:] = np.cumsum(n)
        cat = lambda f, dt: np.ascontiguousarray(np.concatenate([getattr(t, f) for t in traces])
                                                 if traces else np.zeros(0, dt), dtype=dt)
        return TraceBatch(off, cat("arrival", np.float64), cat("prompt", np.int32),
                          cat("decode", np.int32), cat("task", np.uint8))

    def replay(self, r: int):
        s = slice(int(self.offsets[r]), int(self.offsets[r + 1]))
        return s


@dataclass
class BatchResult:
    instance: np.ndarray
    routed: np.ndarray
    first: np.ndarray
    completion: np.ndarray
    preemptions: np.ndarray
    predicted: np.ndarray
    stats: np.ndarray   # STATS_DTYPE [R]
    offsets: np.ndarray

    def replay(self, r: int) -> dict:
        s = slice(int(self.offsets[r]), int(self.offsets[r + 1]))
        return {k: getattr(self, k)[s] for k in ("instance", "routed", "first", "completion",
                                                 "preemptions", "predicted")}


def build_workload(seeds, n: int, rate: float = 20.0, weights=None, process: int = 0,
                   cfg: ClusterConfig | None = None, threads: int = 0) -> TraceBatch:
    """build_workload (experiment.hpp:291-305) for many seeds (host threads)."""
    lib = abi.load_library()
    cfg = cfg or ClusterConfig()
    c = cfg.to_abi("round_robin")
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    R = int(seeds.shape[0])
    arr = np.empty(R * n, np.float64)
    pr = np.empty(R * n, np.int32)
    de = np.empty(R * n, np.int32)
    tk = np.empty(R * n, np.uint8)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    abi.check(lib, lib.rs_generate_mixture_batch(C.byref(c.profile), C.byref(c.thresholds),
                                                 abi.ptr(w), seeds.ctypes.data, R, n, rate,
                                                 process, threads, arr.ctypes.data,
                                                 pr.ctypes.data, de.ctypes.data, tk.ctypes.data))
    off = np.arange(R + 1, dtype=np.int64) * n
    return TraceBatch(off, arr, pr, de, tk)


class BatchSim:
    """A batch of independent ClusterSims replayed on one B200.

    predictor_seeds[r] seeds replay r's simulated predictor stream (the
    reference derives it as mix_seed(seed, 0x9Ded), experiment.hpp:320)."""

    def __init__(self, cfg: ClusterConfig, traces: TraceBatch, predictor_seeds,
                 policy_seeds=None, device: int = 0):
        self.cfg = cfg
        self.traces = traces
        self.predictor_seeds = np.ascontiguousarray(predictor_seeds, dtype=np.uint64)
        self.policy_seeds = (None if policy_seeds is None
                             else np.ascontiguousarray(policy_seeds, dtype=np.uint64))
        self.device = device
        self.lib = abi.load_library()

    def run_policy(self, policy: str, max_ticks: int = 10_000_000, agent=None,
                   epsilon: float = 0.0) -> BatchResult:
        return self._run(policy, max_ticks, agent, epsilon, None)

    def run_trajectory(self, policy: str, capacity: int, reward: RewardConfig | None = None,
                       episode_k: int = 0, max_ticks: int = 10_000_000, agent=None,
                       epsilon: float = 0.0, fields=None):
        """run_policy with ClusterConfig::record_trajectory (env.hpp:131): also
        returns every replay's ClusterSim::trajectory() (env.hpp:203) as
        {TickRecord field: array [R, capacity(, m)]}; replay r's tick t is
        row t-1 (ticks past `capacity` run but are not recorded)."""
        reward = reward or RewardConfig()
        t, arrays = abi.make_trajectory(capacity, self.traces.num_replays,
                                        self.cfg.num_instances, r_w=reward.r_w,
                                        gamma=reward.gamma, beta_d=reward.beta_d,
                                        shaping=reward.shaping, episode_k=episode_k,
                                        fields=fields)
        res = self._run(policy, max_ticks, agent, epsilon, t)
        return res, arrays

    def _run(self, policy, max_ticks, agent, epsilon, traj) -> BatchResult:
        pid = make_policy(policy)
        c = self.cfg.to_abi(policy)
        c.policy = pid
        c.max_ticks = int(max_ticks)
        keep = None
        if pid == abi.POLICIES["rl"]:
            if agent is None:
                raise ValueError("rl policy needs agent=(dims, params)")
            dims, params = agent
            keep = abi.set_rl(c, dims, params)
            c.rl_epsilon = float(epsilon)
        t = self.traces
        N, R = t.total, t.num_replays
        tr = abi.TraceSoA(R, 0, N, t.offsets.ctypes.data, t.arrival.ctypes.data,
                          t.prompt.ctypes.data, t.decode.ctypes.data, t.task.ctypes.data,
                          abi.ptr(t.given_bucket), self.predictor_seeds.ctypes.data,
                          abi.ptr(self.policy_seeds))
        res = BatchResult(np.empty(N, np.int32), np.empty(N, np.float64), np.empty(N, np.float64),
                          np.empty(N, np.float64), np.empty(N, np.int32), np.empty(N, np.uint8),
                          np.zeros(R, abi.STATS_DTYPE), t.offsets)
        out = abi.ReqOut(res.instance.ctypes.data, res.routed.ctypes.data, res.first.ctypes.data,
                         res.completion.ctypes.data, res.preemptions.ctypes.data,
                         res.predicted.ctypes.data)
        if traj is None:
            abi.check(self.lib, self.lib.rs_replay_batch_host(
                C.byref(c), C.byref(tr), C.byref(out), res.stats.ctypes.data, self.device))
        else:
            abi.check(self.lib, self.lib.rs_replay_trajectory_host(
                C.byref(c), C.byref(tr), C.byref(out), res.stats.ctypes.data, C.byref(traj),
                self.device))
        del keep
        return res


def mlp_forward(dims, params, states: np.ndarray, device: int = 0):
    """Mlp::forward + greedy argmax on the device for a batch of states."""
    lib = abi.load_library()
    c = abi.default_config("rl", max(1, dims[-1] - 1))
    keep = abi.set_rl(c, dims, params)
    x = np.ascontiguousarray(states, dtype=np.float64)
    B = int(x.shape[0])
    q = np.empty((B, dims[-1]), np.float64)
    g = np.empty(B, np.int32)
    abi.check(lib, lib.rs_mlp_forward_host(C.byref(c), x.ctypes.data, B, q.ctypes.data,
                                           g.ctypes.data, device))
    del keep
    return q, g


def mlp_random_init(dims, seed: int) -> np.ndarray:
    """DqnAgent(state_dim, actions, {hidden}, seed)'s online network weights
    (Mlp::random, mlp.hpp:32-45), reference flat layout."""
    lib = abi.load_library()
    d = np.ascontiguousarray(dims, dtype=np.int32)
    p = np.empty(abi.mlp_param_count(list(dims)), np.float64)
    abi.check(lib, lib.rs_mlp_random_init(d.ctypes.data, len(dims) - 1, int(seed), p.ctypes.data))
    return p


class DqnTrainer:
    """The trainable state of a DqnAgent (dqn.hpp:52-140) on the host: online
    and target networks, Adam moments and counters.  `update` runs one
    DqnAgent::update step on the device (rs_dqn_update_host) for a batch the
    caller has sampled (ReplayBuffer::sample, replay.hpp:44-58)."""

    def __init__(self, dims, params, learning_rate: float = 1e-3,
                 target_sync_interval: int = 1000, device: int = 0):
        self.dims = list(dims)
        self.online = np.ascontiguousarray(params, dtype=np.float64).copy()
        self.target = self.online.copy()
        self.adam_m = np.zeros_like(self.online)
        self.adam_v = np.zeros_like(self.online)
        self.adam_t = 0
        self.updates = 0
        self.lr = float(learning_rate)
        self.sync = int(target_sync_interval)
        self.device = device
        self.lib = abi.load_library()
        self.cfg = abi.default_config("rl", max(1, self.dims[-1] - 1))
        self.cfg.rl_num_layers = len(self.dims) - 1
        for i, d in enumerate(self.dims):
            self.cfg.rl_dims[i] = int(d)

    def update(self, state, action, reward, next_state, done, discount: float) -> float:
        c = lambda a, dt: np.ascontiguousarray(a, dtype=dt)
        s, a, r = c(state, np.float64), c(action, np.int32), c(reward, np.float64)
        ns, d = c(next_state, np.float64), c(done, np.uint8)
        b = abi.DqnBatch(int(a.shape[0]), 0, s.ctypes.data, a.ctypes.data, r.ctypes.data,
                         ns.ctypes.data, d.ctypes.data)
        st = abi.DqnState(self.online.ctypes.data, self.target.ctypes.data,
                          self.adam_m.ctypes.data, self.adam_v.ctypes.data, self.adam_t,
                          self.updates, self.sync, self.lr)
        loss = np.zeros(1, np.float64)
        abi.check(self.lib, self.lib.rs_dqn_update_host(C.byref(self.cfg), C.byref(b),
                                                        C.byref(st), float(discount),
                                                        loss.ctypes.data, self.device))
        self.adam_t, self.updates = int(st.adam_t), int(st.updates)
        return float(loss[0])
