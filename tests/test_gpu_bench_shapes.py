"""GPU parity at the BASELINE bench shapes and launch plans.

The parity suite elsewhere launches <= 24 replays, so the planner always
takes the latency-regime kernel.  These tests launch the batch sizes bench.py
launches, so the same kernel instantiation, waiting-ring size and block
shape run (asserted from the planner's RS_DEBUG_PLAN line), and check a
sample of the replays against the compiled reference (oracle/_ref) and the
pinned C oracle:

  c3  RL 51-64-64-9 (Mlp::random seed 42, the bench's agent), 4,096 replays
      x 4,000 requests at lambda = 40, m = 8
  c4  round_robin / jsq / workload_aware / rl (27-64-64-5, seed 42), m = 4,
      16,384 replays x 2,000 requests at lambda 55 and 80 (saturated queues;
      more replays than resident slots: the 256-thread-bound / wide RL builds)
  c5  workload_aware, m = 64, two 200k-request replays of the heavy-decode
      mixture (weights 0/3/1/2/0, lambda = 40) inside a 512-replay launch
"""
import ctypes as C
import re
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine

pytestmark = pytest.mark.gpu

HEAVY_DECODE = (0.0, 3.0, 1.0, 2.0, 0.0)


def trace_of(tb, r):
    s = tb.replay(r)
    return O.Trace(tb.arrival[s], tb.prompt[s], tb.decode[s], tb.task[s])


def run_batch(lib, cfg, tb, pseeds, capfd):
    """rs_replay_batch_host over the whole batch (pageable buffers, no
    input streaming: the device-resident path the bench's device leg takes) with
    the simulated predictor drawn inline, as bench.py runs it.  Returns the
    per-request arrays, the stats and the planner's line."""
    N, R = tb.total, tb.num_replays
    ps = np.ascontiguousarray(pseeds, np.uint64)
    tr = abi.TraceSoA(R, 0, N, tb.offsets.ctypes.data, tb.arrival.ctypes.data,
                      tb.prompt.ctypes.data, tb.decode.ctypes.data, tb.task.ctypes.data, None,
                      ps.ctypes.data, None)
    arrs = [np.empty(N, np.int32), np.empty(N, np.float64), np.empty(N, np.float64),
            np.empty(N, np.float64), np.empty(N, np.int32), np.empty(N, np.uint8)]
    stats = np.zeros(R, abi.STATS_DTYPE)
    out = abi.ReqOut(*[a.ctypes.data for a in arrs])
    c = abi.BatchCfg.from_buffer_copy(bytes(cfg))
    c.flags |= abi.RS_FLAG_PREDICT_INLINE
    capfd.readouterr()
    abi.check(lib, lib.rs_replay_batch_host(C.byref(c), C.byref(tr), C.byref(out),
                                            stats.ctypes.data, 0))
    plan = [ln for ln in capfd.readouterr().err.splitlines() if ln.startswith("rs plan:")]
    return arrs, stats, (plan[-1] if plan else "")


def result_of(tb, arrs, stats, r):
    s = tb.replay(r)
    return O.ReplayResult(*[a[s] for a in arrs], stats[r:r + 1])


def plan_field(plan, key):
    m = re.search(rf"{key} (\S+)", plan)
    return m.group(1) if m else None


@pytest.fixture
def debug_plan(monkeypatch):
    monkeypatch.setenv("RS_DEBUG_PLAN", "1")
    # the bench's device leg: inputs resident before the launch (no streaming)
    monkeypatch.setenv("RS_STREAM_INPUTS", "0")
    for k in ("RS_FORCE_GENERAL", "RS_RUN_SMEM", "RS_WAIT_RING", "RS_WARPS_PER_BLOCK",
              "RS_RL_GLOBAL"):
        monkeypatch.delenv(k, raising=False)


def check_sample(cfg, tb, pseeds, arrs, stats, picks, ref_picks, agent=None):
    """Every replay: finished and conserving requests.  `picks`: bitwise vs
    the C oracle (threads); `ref_picks`: bitwise vs the compiled reference."""
    assert np.all(stats["status"] == abi.REPLAY_FINISHED)
    n_req = np.diff(tb.offsets)
    assert np.array_equal(stats["completed"], n_req)
    with ThreadPoolExecutor(8) as ex:  # ctypes releases the GIL
        want = list(ex.map(lambda r: O.ora_run(cfg, trace_of(tb, r), int(pseeds[r])), picks))
    for r, w in zip(picks, want):
        assert O.compare(result_of(tb, arrs, stats, r), w) == [], f"replay {r} vs C oracle"
    if O.have_ref():
        with ThreadPoolExecutor(8) as ex:
            want = list(ex.map(lambda r: O.ref_run(cfg, trace_of(tb, r), int(pseeds[r])),
                               ref_picks))
        for r, w in zip(ref_picks, want):
            assert O.compare(result_of(tb, arrs, stats, r), w) == [], f"replay {r} vs oracle/_ref"


def seed_batch(seeds, n, rate, weights=None):
    tb = engine.build_workload(seeds, n, rate, weights)
    ps = np.array([abi.mix_seed(int(s), 0x9DED) for s in seeds], np.uint64)
    return tb, ps


def bench_agent(m):
    """bench.py's agent_for(m): DqnAgent(state_dim, m + 1, 64, seed 42)
    initial weights, which equal the compiled reference's own constructor's."""
    sd = abi.state_dimension(m)
    dims = [sd, 64, 64, m + 1]
    params = engine.mlp_random_init(dims, 42)
    if O.have_ref():
        assert np.array_equal(params, O.ref_agent_params(sd, m + 1, 64, 42))
    return dims, params


def test_c3_shape_rl_agent(gpu, debug_plan, capfd):
    R, n, m = 4096, 4000, 8
    tb, ps = seed_batch(np.arange(1, R + 1), n, 40.0)
    dims, params = bench_agent(m)
    cfg = abi.default_config("rl", m)
    keep = abi.set_rl(cfg, dims, params)
    arrs, stats, plan = run_batch(gpu, cfg, tb, ps, capfd)
    # 16 replays per SM next to the staged Q-network: the running head and
    # the waiting ring shrink and the predictions come from the pre-pass
    assert plan_field(plan, "kernel") == "wide", plan
    assert plan_field(plan, "fused_pred") == "0", plan
    picks = [0, 1, 777, 2048, 4095]
    check_sample(cfg, tb, ps, arrs, stats, picks, picks[:3])
    del keep


@pytest.mark.parametrize("policy", ["round_robin", "jsq", "workload_aware", "rl"])
def test_c4_shape_saturated_sweep(gpu, debug_plan, capfd, policy):
    R, n, m = 16384, 2000, 4
    half = R // 2
    tb55, ps55 = seed_batch(np.arange(1, half + 1), n, 55.0)
    tb80, ps80 = seed_batch(np.arange(1, half + 1), n, 80.0)
    cat = lambda f: np.ascontiguousarray(np.concatenate([getattr(tb55, f), getattr(tb80, f)]))
    tb = engine.TraceBatch(np.arange(R + 1, dtype=np.int64) * n, cat("arrival"), cat("prompt"),
                           cat("decode"), cat("task"))
    ps = np.concatenate([ps55, ps80])
    cfg = abi.default_config(policy, m)
    keep = None
    if policy == "rl":
        dims, params = bench_agent(m)
        keep = abi.set_rl(cfg, dims, params)
    arrs, stats, plan = run_batch(gpu, cfg, tb, ps, capfd)
    # the throughput regime: more replays than resident slots, the
    # register-bounded (or wide RL) build
    assert plan_field(plan, "kernel") == ("wide" if policy == "rl" else "bounded"), plan
    assert int(plan.rsplit(" ", 1)[1]) < R, plan
    # saturated queues at lambda = 80: routing waits in the router queue
    assert np.mean(stats["sum_router_queue"][half:] / stats["ticks"][half:]) > 1.0
    picks = [0, 5, half - 1, half, half + 3, R - 1]
    check_sample(cfg, tb, ps, arrs, stats, picks, [0, half, R - 1])
    del keep


def test_c5_shape_large_fleet(gpu, debug_plan, capfd):
    # two full 200k-request replays inside a 512-replay launch (the plan
    # depends on the replay count and config, not on replay lengths; the
    # other 510 replays are 4,000 requests to bound host memory)
    R, m = 512, 64
    big, bps = seed_batch([1, 2], 200_000, 40.0, HEAVY_DECODE)
    small, sps = seed_batch(np.arange(3, R + 1), 4000, 40.0, HEAVY_DECODE)
    cat = lambda f: np.ascontiguousarray(np.concatenate([getattr(big, f), getattr(small, f)]))
    off = np.concatenate([big.offsets[:-1], big.total + small.offsets]).astype(np.int64)
    tb = engine.TraceBatch(off, cat("arrival"), cat("prompt"), cat("decode"), cat("task"))
    ps = np.concatenate([bps, sps])
    cfg = abi.default_config("workload_aware", m)
    arrs, stats, plan = run_batch(gpu, cfg, tb, ps, capfd)
    assert plan_field(plan, "kernel") == "pair", plan  # two warps per replay (pair.cuh)
    check_sample(cfg, tb, ps, arrs, stats, [0, 1, 2, 300, R - 1], [2, R - 1])


def test_300k_request_replay(gpu, debug_plan, capfd):
    # Beyond the round-1 32-bit aggregate guard (N x max(prompt + max(decode,
    # 4096)) <= 2^30, i.e. about 210k requests): the waiting-queue aggregates
    # are 64-bit, so a 300k-request replay runs, bit-exact (c2's fleet and
    # arrival rate, ~750k ticks).
    tb, ps = seed_batch([9, 10], 300_000, 20.0)
    cfg = abi.default_config("workload_aware", 8)
    arrs, stats, plan = run_batch(gpu, cfg, tb, ps, capfd)
    assert np.all(stats["status"] == abi.REPLAY_FINISHED)
    check_sample(cfg, tb, ps, arrs, stats, [0, 1], [])
