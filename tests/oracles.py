"""Bindings to the two CPU checkers (TEST INFRASTRUCTURE ONLY).

 * `ora_*`  — oracle/rs_oracle.c, the plain-C restatement (oracle/build/).
 * `ref_*`  — oracle/_ref/librs_ref.so, the UNMODIFIED reference headers
             compiled in place behind oracle/ref_driver.cpp.  Built only where
             /root/reference exists; the built .so travels to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use
these, and only as checkers / baselines.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from paper_2408_13510_b200 import abi

ROOT = Path(__file__).resolve().parents[1]
ORA_PATH = ROOT / "oracle" / "build" / "librs_oracle.so"
REF_PATH = ROOT / "oracle" / "_ref" / "librs_ref.so"
REF_NOSCAN_PATH = ROOT / "oracle" / "_ref" / "librs_ref_noscan.so"
REFERENCE_DIR = Path(os.environ.get("RS_REFERENCE_DIR", "/root/reference"))


def _make(target: str) -> None:
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), target], check=True)


_ora = None
_ref = None
_ref_noscan = None


def ora_lib() -> C.CDLL:
    global _ora
    if _ora is None:
        _make("oracle")  # no-op when up to date; rebuilds after header changes
        lib = C.CDLL(str(ORA_PATH))
        P = C.POINTER
        lib.ora_run_replay.argtypes = [P(abi.BatchCfg), C.c_int64] + [C.c_void_p] * 5 + [
            C.c_uint64, C.c_uint64] + [C.c_void_p] * 8 + [C.c_int64]
        lib.ora_predict_buckets.argtypes = [P(abi.BatchCfg), C.c_int64] + [C.c_void_p] * 4 + [
            C.c_uint64, C.c_void_p]
        lib.ora_mlp_forward.argtypes = [P(abi.BatchCfg), C.c_void_p, C.c_int32, C.c_void_p,
                                        C.c_void_p]
        lib.ora_run_trajectory.argtypes = [P(abi.BatchCfg), C.c_int64] + [C.c_void_p] * 5 + [
            C.c_uint64, C.c_uint64] + [C.c_void_p] * 7 + [P(abi.Trajectory)]
        lib.ora_mt19937_64.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        lib.ora_mix_seed.restype = C.c_uint64
        lib.ora_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        _ora = lib
    return _ora


def have_ref() -> bool:
    return REF_PATH.exists() or (REFERENCE_DIR / "proj" / "include" / "routesim").exists()


def ref_lib(noscan: bool = False) -> C.CDLL:
    """oracle/_ref/librs_ref.so (the unmodified reference); noscan=True: the
    same with the reward-only queue-penalty scan compiled out (Makefile)."""
    global _ref, _ref_noscan
    if noscan:
        if _ref_noscan is None:
            if not REF_NOSCAN_PATH.exists():
                _make("ref")
            _ref_noscan = _declare_ref(C.CDLL(str(REF_NOSCAN_PATH)))
        return _ref_noscan
    if _ref is None:
        if not REF_PATH.exists():
            _make("ref")
        _ref = _declare_ref(C.CDLL(str(REF_PATH)))
    return _ref


def _declare_ref(lib: C.CDLL) -> C.CDLL:
    P = C.POINTER
    lib.ref_generate_mixture.argtypes = [P(abi.Profile), P(abi.Thresholds), C.c_void_p,
                                         C.c_uint64, C.c_int64, C.c_double, C.c_int32,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.ref_run_replay.argtypes = [P(abi.BatchCfg), C.c_int64] + [C.c_void_p] * 4 + [
        C.c_uint64, C.c_uint64] + [C.c_void_p] * 8 + [C.c_int64]
    lib.ref_run_trajectory.argtypes = [P(abi.BatchCfg), C.c_int64] + [C.c_void_p] * 4 + [
        C.c_uint64, C.c_uint64] + [C.c_void_p] * 7 + [P(abi.Trajectory)]
    lib.ref_run_batch.restype = C.c_double
    lib.ref_run_batch.argtypes = [P(abi.BatchCfg), C.c_int32] + [C.c_void_p] * 7 + [
        C.c_int32, C.c_void_p]
    lib.ref_agent_init.restype = C.c_int64
    lib.ref_agent_init.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p,
                                   C.c_int64]
    lib.ref_mlp_forward.argtypes = [P(abi.BatchCfg), C.c_void_p, C.c_int32, C.c_void_p,
                                    C.c_void_p]
    lib.ref_golden_summary.argtypes = [C.c_char_p, C.c_size_t, C.c_int32]
    lib.ref_experiment_summary.argtypes = [C.c_int32, C.c_int64, C.c_double, C.c_uint64,
                                           C.c_char_p, C.c_char_p, C.c_size_t]
    lib.ref_mix_seed.restype = C.c_uint64
    lib.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
    lib.ref_heavy_decode_cutoff.restype = C.c_int64
    lib.ref_heavy_decode_cutoff.argtypes = [P(abi.Profile), P(abi.Thresholds)]
    lib.ref_last_error.argtypes = [C.c_char_p, C.c_size_t]
    return lib


def ref_error() -> str:
    buf = C.create_string_buffer(1024)
    ref_lib().ref_last_error(buf, len(buf))
    return buf.value.decode()


@dataclass
class Trace:
    arrival: np.ndarray
    prompt: np.ndarray
    decode: np.ndarray
    task: np.ndarray

    @property
    def n(self) -> int:
        return int(self.arrival.shape[0])


@dataclass
class ReplayResult:
    instance: np.ndarray
    routed: np.ndarray
    first: np.ndarray
    completion: np.ndarray
    preemptions: np.ndarray
    predicted: np.ndarray
    stats: np.ndarray  # one STATS_DTYPE record
    actions: np.ndarray | None = None


def make_trace(rows) -> Trace:
    """(arrival, prompt, decode[, task]) rows, as test_env.cpp's trace_of."""
    a = np.array([r[0] for r in rows], dtype=np.float64)
    p = np.array([r[1] for r in rows], dtype=np.int32)
    d = np.array([r[2] for r in rows], dtype=np.int32)
    t = np.array([r[3] if len(r) > 3 else 1 for r in rows], dtype=np.uint8)  # QnA
    return Trace(a, p, d, t)


def ref_generate(seed: int, n: int, rate: float = 20.0, weights=None, process: int = 0,
                 cfg: abi.BatchCfg | None = None) -> Trace:
    cfg = cfg or abi.default_config()
    a = np.empty(n, np.float64)
    p = np.empty(n, np.int32)
    d = np.empty(n, np.int32)
    t = np.empty(n, np.uint8)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    rc = ref_lib().ref_generate_mixture(C.byref(cfg.profile), C.byref(cfg.thresholds),
                                        abi.ptr(w), seed, n, rate, process, a.ctypes.data,
                                        p.ctypes.data, d.ctypes.data, t.ctypes.data)
    assert rc == 0, ref_error()
    return Trace(a, p, d, t)


def _alloc(n):
    return ReplayResult(np.empty(n, np.int32), np.empty(n, np.float64),
                        np.empty(n, np.float64), np.empty(n, np.float64),
                        np.empty(n, np.int32), np.empty(n, np.uint8),
                        np.zeros(1, abi.STATS_DTYPE))


def _run(fn, cfg, tr: Trace, predictor_seed, policy_seed, log_actions, given=None):
    n = tr.n
    out = _alloc(max(n, 1))
    cap = int(min(cfg.max_ticks, 4_000_000)) if log_actions else 0
    log = np.empty(max(cap, 1), np.int32) if log_actions else None
    args = [C.byref(cfg), n, tr.arrival.ctypes.data, tr.prompt.ctypes.data,
            tr.decode.ctypes.data, tr.task.ctypes.data]
    if given is not None:
        args.append(abi.ptr(given))
    args += [predictor_seed, policy_seed, out.instance.ctypes.data, out.routed.ctypes.data,
             out.first.ctypes.data, out.completion.ctypes.data, out.preemptions.ctypes.data,
             out.predicted.ctypes.data, out.stats.ctypes.data, abi.ptr(log), cap]
    rc = fn(*args)
    if rc != 0:
        raise RuntimeError(f"checker failed rc={rc}")
    if log_actions:
        out.actions = log[: int(min(out.stats["ticks"][0], cap))].copy()
    for f in ("instance", "routed", "first", "completion", "preemptions", "predicted"):
        setattr(out, f, getattr(out, f)[:n])
    return out


def ora_run(cfg, tr: Trace, predictor_seed=1, policy_seed=0, log_actions=False,
            given=None) -> ReplayResult:
    return _run(ora_lib().ora_run_replay, cfg, tr, predictor_seed, policy_seed, log_actions,
                given=given if given is not None else np.zeros(max(tr.n, 1), np.uint8))


def ref_run(cfg, tr: Trace, predictor_seed=1, policy_seed=0, log_actions=False) -> ReplayResult:
    lib = ref_lib()
    try:
        return _run(lib.ref_run_replay, cfg, tr, predictor_seed, policy_seed, log_actions)
    except RuntimeError as e:
        raise RuntimeError(f"{e}: {ref_error()}") from None


def ref_agent_params(state_dim: int, actions: int, hidden: int, seed: int) -> np.ndarray:
    lib = ref_lib()
    n = lib.ref_agent_init(state_dim, actions, hidden, seed, None, 0)
    p = np.empty(n, np.float64)
    lib.ref_agent_init(state_dim, actions, hidden, seed, p.ctypes.data, n)
    return p


def compare(a: ReplayResult, b: ReplayResult, exact_times: bool = True) -> list[str]:
    """Differences between two replay results ([] when identical)."""
    errs = []
    for f in ("instance", "preemptions", "predicted"):
        x, y = getattr(a, f), getattr(b, f)
        if not np.array_equal(x, y):
            i = int(np.flatnonzero(x != y)[0])
            errs.append(f"{f} differs at {i}: {x[i]} vs {y[i]} ({int((x != y).sum())} total)")
    for f in ("routed", "first", "completion"):
        x, y = getattr(a, f), getattr(b, f)
        if exact_times:
            bad = x.view(np.uint64) != y.view(np.uint64)
        else:
            bad = ~np.isclose(x, y, rtol=1e-6, atol=0)
        if bad.any():
            i = int(np.flatnonzero(bad)[0])
            errs.append(f"{f} differs at {i}: {x[i]!r} vs {y[i]!r} ({int(bad.sum())} total)")
    sa, sb = a.stats[0], b.stats[0]
    for f in ("ticks", "routed", "infeasible", "completed", "decision_hash", "status",
              "total_preemptions", "total_tokens", "tbt_count", "sum_router_queue",
              "sum_instance_waiting"):
        if sa[f] != sb[f]:
            errs.append(f"stats.{f}: {sa[f]} vs {sb[f]}")
    pct = ("e2e_p50", "e2e_p90", "e2e_p99", "ttft_p50", "ttft_p90", "ttft_p99", "tbt_p50",
           "tbt_p90", "tbt_p99")
    both_pct = sa["percentiles_valid"] and sb["percentiles_valid"]
    for f in ("clock", "total_e2e_s", "total_ttft_s", "total_tbt_s", "total_router_wait_s",
              "makespan_s") + (pct if both_pct else ()):
        x, y = float(sa[f]), float(sb[f])
        if exact_times and not (x == y or (np.isnan(x) and np.isnan(y))):
            errs.append(f"stats.{f}: {x!r} vs {y!r}")
        elif not exact_times and not np.isclose(x, y, rtol=1e-6):
            errs.append(f"stats.{f}: {x!r} vs {y!r}")
    if a.actions is not None and b.actions is not None and not np.array_equal(a.actions,
                                                                               b.actions):
        i = int(np.flatnonzero(a.actions[: min(len(a.actions), len(b.actions))] !=
                               b.actions[: min(len(a.actions), len(b.actions))])[0]) \
            if min(len(a.actions), len(b.actions)) else 0
        errs.append(f"actions differ first at tick {i}")
    return errs


def _run_traj(fn, cfg, tr: Trace, predictor_seed, policy_seed, capacity, reward, given=None):
    """One replay with record_trajectory: (ReplayResult, {field: [capacity(, m)]})."""
    n = tr.n
    out = _alloc(max(n, 1))
    t, arrays = abi.make_trajectory(capacity, 1, cfg.num_instances, **(reward or {}))
    args = [C.byref(cfg), n, tr.arrival.ctypes.data, tr.prompt.ctypes.data,
            tr.decode.ctypes.data, tr.task.ctypes.data]
    if given is not None:
        args.append(abi.ptr(given))
    args += [predictor_seed, policy_seed, out.instance.ctypes.data, out.routed.ctypes.data,
             out.first.ctypes.data, out.completion.ctypes.data, out.preemptions.ctypes.data,
             out.predicted.ctypes.data, out.stats.ctypes.data, C.byref(t)]
    if fn(*args) != 0:
        raise RuntimeError("checker failed")
    for f in ("instance", "routed", "first", "completion", "preemptions", "predicted"):
        setattr(out, f, getattr(out, f)[:n])
    k = int(min(out.stats["ticks"][0], capacity))
    return out, {name: a[0, :k] for name, a in arrays.items()}


def ora_trajectory(cfg, tr: Trace, predictor_seed=1, policy_seed=0, capacity=200_000,
                   reward=None):
    return _run_traj(ora_lib().ora_run_trajectory, cfg, tr, predictor_seed, policy_seed,
                     capacity, reward, given=np.zeros(max(tr.n, 1), np.uint8))


def ref_trajectory(cfg, tr: Trace, predictor_seed=1, policy_seed=0, capacity=200_000,
                   reward=None):
    try:
        return _run_traj(ref_lib().ref_run_trajectory, cfg, tr, predictor_seed, policy_seed,
                         capacity, reward)
    except RuntimeError as e:
        raise RuntimeError(f"{e}: {ref_error()}") from None


def compare_trajectory(a: dict, b: dict) -> list[str]:
    """Bitwise differences between two trajectories ([] when identical)."""
    errs = []
    for name in a:
        x, y = a[name], b[name]
        if x.shape != y.shape:
            errs.append(f"{name}: shape {x.shape} vs {y.shape}")
            continue
        bad = (x.view(np.uint64) != y.view(np.uint64)) if x.dtype == np.float64 else (x != y)
        if bad.any():
            i = np.argwhere(bad)[0]
            errs.append(f"{name} differs at {tuple(i)}: {x[tuple(i)]!r} vs {y[tuple(i)]!r} "
                        f"({int(bad.sum())} total)")
    return errs


def ref_emit_report(cfg, tr: Trace, directory, predictor_seed=1, policy_seed=0,
                    record_trajectory=True, reward=None):
    """The reference's compute_metrics + emit_report of one replay into `directory`."""
    lib = ref_lib()
    lib.ref_emit_report.argtypes = [C.POINTER(abi.BatchCfg), C.c_int64] + [C.c_void_p] * 4 + [
        C.c_uint64, C.c_uint64, C.c_int32, C.POINTER(abi.Trajectory), C.c_char_p]
    t = None  # None: to_cluster's RewardConfig (shaping none)
    if reward is not None:
        t, _ = abi.make_trajectory(0, 1, cfg.num_instances, fields=(), **reward)
    rc = lib.ref_emit_report(C.byref(cfg), tr.n, tr.arrival.ctypes.data, tr.prompt.ctypes.data,
                             tr.decode.ctypes.data, tr.task.ctypes.data, predictor_seed,
                             policy_seed, 1 if record_trajectory else 0,
                             C.byref(t) if t is not None else None,
                             os.fsencode(str(directory)))
    if rc != 0:
        raise RuntimeError(ref_error())


def ref_dqn_train(dims, params, states, actions, rewards, next_states, dones, batch, steps,
                  sample_seed, discount, lr=1e-3, sync_interval=1000):
    """`steps` reference DqnAgent::update calls; returns (sampled index
    [steps, batch], losses [steps], online params after each step
    [steps, np], final target params)."""
    lib = ref_lib()
    lib.ref_dqn_train.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64] + [
        C.c_void_p] * 5 + [C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_double, C.c_int64] + [
        C.c_void_p] * 4
    c = lambda a, dt: np.ascontiguousarray(a, dtype=dt)
    params, states, next_states = c(params, np.float64), c(states, np.float64), c(next_states,
                                                                                  np.float64)
    actions, rewards, dones = c(actions, np.int32), c(rewards, np.float64), c(dones, np.uint8)
    n, np_ = int(actions.shape[0]), int(params.shape[0])
    idx = np.zeros((steps, batch), np.int64)
    losses = np.zeros(steps, np.float64)
    online = np.zeros((steps, np_), np.float64)
    target = np.zeros(np_, np.float64)
    rc = lib.ref_dqn_train(dims[0], dims[-1], dims[1], params.ctypes.data, n,
                           states.ctypes.data, actions.ctypes.data, rewards.ctypes.data,
                           next_states.ctypes.data, dones.ctypes.data, batch, steps, sample_seed,
                           discount, lr, sync_interval, idx.ctypes.data, losses.ctypes.data,
                           online.ctypes.data, target.ctypes.data)
    if rc != 0:
        raise RuntimeError(ref_error())
    return idx, losses, online, target


def ref_empirical_table(cfg, seed, n_train=20000):
    """The reference's EmpiricalPredictor fit + predict table ([5, 8] uint8)."""
    lib = ref_lib()
    lib.ref_empirical_table.argtypes = [C.POINTER(abi.BatchCfg), C.c_uint64, C.c_int64,
                                        C.c_void_p]
    out = np.zeros((abi.RS_NUM_TASKS, abi.RS_MAX_BANDS), np.uint8)
    if lib.ref_empirical_table(C.byref(cfg), seed, n_train, out.ctypes.data) != 0:
        raise RuntimeError(ref_error())
    return out
