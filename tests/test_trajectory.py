"""record_trajectory: the Eq. 3 reward and the TickRecords of every tick
(ClusterSim::step, env.hpp:251-319) — SURVEY.md §8(f) rank 2.

CPU: the C restatement against the frozen reference trajectories
(tests/golden/trajectories.npz, made from oracle/_ref by make_golden.py) and
against the live compiled reference.  GPU: rs_replay_trajectory(_host)
against the same fixtures and the oracle, every field bitwise (fp64 reward
terms included: the scan is sequential in pool-index order, as the
reference's)."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine

GOLDEN = Path(__file__).resolve().parent / "golden"


def traj_cases():
    return sorted(json.loads((GOLDEN / "trajectories.json").read_text()))


@pytest.fixture(scope="module")
def golden():
    z = np.load(GOLDEN / "trajectories.npz")
    return {k: z[k] for k in z.files}, json.loads((GOLDEN / "trajectories.json").read_text())


def golden_case(golden, name):
    arr, meta = golden
    m = meta[name]
    cfg = abi.BatchCfg.from_buffer_copy(arr[f"{name}.cfg"].tobytes())
    cfg.rl_params = None
    keep = None
    if m["dims"]:
        eps = cfg.rl_epsilon
        keep = abi.set_rl(cfg, m["dims"], arr[f"{name}.params"])
        cfg.rl_epsilon = eps
    tr = O.Trace(arr[f"{name}.arrival"], arr[f"{name}.prompt"], arr[f"{name}.decode"],
                 arr[f"{name}.task"])
    want = {k.split(".traj.")[1]: v for k, v in arr.items() if k.startswith(f"{name}.traj.")}
    return cfg, tr, m, want, arr[f"{name}.stats"], keep


@pytest.mark.parametrize("name", traj_cases())
def test_oracle_reproduces_golden_trajectory(golden, name):
    cfg, tr, m, want, stats, keep = golden_case(golden, name)
    res, got = O.ora_trajectory(cfg, tr, m["predictor_seed"], m["policy_seed"],
                                reward=m["reward"])
    assert int(res.stats["ticks"][0]) == m["ticks"]
    assert O.compare_trajectory(got, want) == []
    del keep


@pytest.mark.skipif(not O.have_ref(), reason="compiled reference unavailable")
@pytest.mark.parametrize("policy,m,n,rate,seed,reward", [
    ("jsq", 4, 200, 20.0, 31, {}),
    ("earliest_available", 3, 200, 35.0, 32, {"shaping": "additive"}),
    ("max_capacity", 4, 150, 10.0, 33, {"episode_k": 4}),
    ("dedicated_small_large", 4, 200, 25.0, 34, {"shaping": "none", "r_w": 10.0}),
    ("workload_aware", 8, 300, 45.0, 35, {"gamma": 0.5, "beta_d": 2.0, "episode_k": 1}),
])
def test_oracle_trajectory_matches_live_reference(policy, m, n, rate, seed, reward):
    cfg = abi.default_config(policy, m)
    tr = O.ref_generate(seed, n, rate)
    ps = abi.mix_seed(seed, 0x9DED)
    ra, ta = O.ref_trajectory(cfg, tr, ps, reward=reward)
    oa, to = O.ora_trajectory(cfg, tr, ps, reward=reward)
    assert O.compare(oa, ra) == []
    assert O.compare_trajectory(to, ta) == []


def test_trajectory_struct_layout():
    assert C.sizeof(abi.Trajectory) == 8 * 4 + 4 * 2 + 8 * len(abi.TRAJ_FIELDS)


# ------------------------------------------------------------------ GPU


def engine_trajectory(lib, cfg, traces, pseeds, qseeds, capacity, reward, fields=None):
    tb = engine.TraceBatch.from_traces(traces)
    N, R = tb.total, tb.num_replays
    ps = np.ascontiguousarray(pseeds, np.uint64)
    qs = np.ascontiguousarray(qseeds, np.uint64)
    tr = abi.TraceSoA(R, 0, N, tb.offsets.ctypes.data, tb.arrival.ctypes.data,
                      tb.prompt.ctypes.data, tb.decode.ctypes.data, tb.task.ctypes.data, None,
                      ps.ctypes.data, qs.ctypes.data)
    arrs = [np.empty(N, np.int32), np.empty(N, np.float64), np.empty(N, np.float64),
            np.empty(N, np.float64), np.empty(N, np.int32), np.empty(N, np.uint8)]
    stats = np.zeros(R, abi.STATS_DTYPE)
    out = abi.ReqOut(*[a.ctypes.data for a in arrs])
    t, tarr = abi.make_trajectory(capacity, R, cfg.num_instances, fields=fields, **(reward or {}))
    abi.check(lib, lib.rs_replay_trajectory_host(C.byref(cfg), C.byref(tr), C.byref(out),
                                                 stats.ctypes.data, C.byref(t), 0))
    res = []
    for r in range(R):
        s = tb.replay(r)
        res.append(O.ReplayResult(*[a[s] for a in arrs], stats[r:r + 1]))
    return res, tarr


@pytest.mark.gpu
@pytest.mark.parametrize("name", traj_cases())
def test_gpu_trajectory_golden(golden, name):
    lib = abi.load_library()
    cfg, tr, m, want, stats, keep = golden_case(golden, name)
    cap = m["ticks"] + 5
    res, got = engine_trajectory(lib, cfg, [tr], [m["predictor_seed"]], [m["policy_seed"]], cap,
                                 m["reward"])
    assert int(res[0].stats["ticks"][0]) == m["ticks"]
    assert int(res[0].stats["decision_hash"][0]) == int(stats["decision_hash"][0])
    k = m["ticks"]
    assert O.compare_trajectory({f: a[0, :k] for f, a in got.items()}, want) == []
    del keep


@pytest.mark.gpu
@pytest.mark.parametrize("policy,m", [("jsq", 4), ("workload_aware", 8), ("round_robin", 2),
                                      ("min_min", 4), ("rl", 4)])
def test_gpu_trajectory_ragged_batch_vs_oracle(policy, m):
    """A ragged batch (1..400 requests) in one call: every replay's
    trajectory equals the oracle's, bitwise; capacity truncation keeps the
    first `capacity` ticks and the full tick count."""
    lib = abi.load_library()
    cfg = abi.default_config(policy, m)
    keep = None
    if policy == "rl":
        dims = [abi.state_dimension(m), 32, 32, m + 1]
        keep = abi.set_rl(cfg, dims, engine.mlp_random_init(dims, 5))
        cfg.rl_epsilon = 0.1
    sizes = [1, 7, 120, 400, 33, 250]
    seeds = list(range(40, 40 + len(sizes)))
    traces = []
    for s, n in zip(seeds, sizes):
        b = engine.build_workload([s], n, 30.0)
        traces.append(O.Trace(b.arrival, b.prompt, b.decode, b.task))
    ps = [abi.mix_seed(s, 0x9DED) for s in seeds]
    qs = [s * 3 + 1 for s in seeds]
    reward = {"shaping": "guided", "episode_k": 2}
    for cap in (100_000, 500):
        res, got = engine_trajectory(lib, cfg, traces, ps, qs, cap, reward)
        for r, tr in enumerate(traces):
            wres, want = O.ora_trajectory(cfg, tr, ps[r], qs[r], capacity=cap, reward=reward)
            assert O.compare(res[r], wres) == [], (cap, r)
            k = int(min(wres.stats["ticks"][0], cap))
            assert O.compare_trajectory({f: a[r, :k] for f, a in got.items()}, want) == [], (cap, r)
    del keep


@pytest.mark.gpu
def test_gpu_trajectory_subset_without_scan():
    """Only action / router_queue / running requested: the Eq. 3 scan is
    skipped and the recorded fields are unchanged."""
    lib = abi.load_library()
    cfg = abi.default_config("jsq", 4)
    b = engine.build_workload([3], 300, 25.0)
    tr = O.Trace(b.arrival, b.prompt, b.decode, b.task)
    ps = abi.mix_seed(3, 0x9DED)
    fields = ("action", "router_queue", "instance_running")
    res, got = engine_trajectory(lib, cfg, [tr], [ps], [0], 50_000, {}, fields=fields)
    wres, want = O.ora_trajectory(cfg, tr, ps)
    k = int(wres.stats["ticks"][0])
    assert set(got) == set(fields)
    assert O.compare_trajectory({f: a[0, :k] for f, a in got.items()},
                                {f: want[f] for f in fields}) == []


@pytest.mark.gpu
def test_gpu_replay_batch_rejects_trajectory_flag():
    lib = abi.load_library()
    cfg = abi.default_config("jsq", 4)
    cfg.flags |= abi.RS_FLAG_RECORD_TRAJECTORY
    b = engine.build_workload([3], 10, 25.0)
    ps = np.array([1], np.uint64)
    tr = abi.TraceSoA(1, 0, 10, b.offsets.ctypes.data, b.arrival.ctypes.data,
                      b.prompt.ctypes.data, b.decode.ctypes.data, b.task.ctypes.data, None,
                      ps.ctypes.data, None)
    stats = np.zeros(1, abi.STATS_DTYPE)
    out = abi.ReqOut(None, None, None, None, None, None)
    assert lib.rs_replay_batch_host(C.byref(cfg), C.byref(tr), C.byref(out),
                                    stats.ctypes.data, 0) == abi.RS_ERR_INVALID_ARGUMENT


@pytest.mark.gpu
def test_gpu_engine_run_trajectory_mirror():
    """BatchSim.run_trajectory (the host mirror) on a seed batch."""
    seeds = [1, 2, 3]
    tb = engine.build_workload(seeds, 200, 30.0)
    ps = [abi.mix_seed(s, 0x9DED) for s in seeds]
    sim = engine.BatchSim(engine.ClusterConfig(num_instances=4), tb, ps)
    res, traj = sim.run_trajectory("workload_aware", 20_000, engine.RewardConfig(shaping="additive"))
    cfg = abi.default_config("workload_aware", 4)
    for r in range(3):
        s = tb.replay(r)
        tr = O.Trace(tb.arrival[s], tb.prompt[s], tb.decode[s], tb.task[s])
        wres, want = O.ora_trajectory(cfg, tr, ps[r], reward={"shaping": "additive"})
        k = int(wres.stats["ticks"][0])
        assert int(res.stats["ticks"][r]) == k
        assert O.compare_trajectory({f: a[r, :k] for f, a in traj.items()}, want) == []
