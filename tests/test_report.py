"""Report layer: compute_metrics + emit_report
(metrics.hpp:84-238) through rs_emit_report must write summary.json,
requests.csv and timeseries.csv BYTE-identical to the reference's own
emit_report on the same replay.

CPU: fed with the oracle's per-request outputs, stats and trajectory (the
oracle is pinned bit-exact to the reference, so any byte difference is a
formatting defect: nlohmann's Grisu2 digits, %.17g, column order).  GPU: fed
with the engine's outputs (rs_replay_trajectory_host), i.e. the device
sums / percentiles end to end."""
from pathlib import Path

import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine, report

FILES = ("summary.json", "requests.csv", "timeseries.csv")
CASES = [
    # policy, m, n, rate, seed, reward, record_trajectory
    ("jsq", 2, 12, 12.0, 777, {"shaping": "none"}, True),     # test_harness.cpp:212-231 golden run
    ("workload_aware", 4, 300, 20.0, 1, {}, True),
    ("round_robin", 4, 250, 40.0, 2, {"shaping": "additive"}, True),
    ("min_min", 3, 200, 30.0, 3, {"episode_k": 3}, False),
    ("decode_balancer", 8, 400, 45.0, 4, {}, True),
    ("max_capacity", 4, 60, 5.0, 5, {}, False),
]


def same_files(a: Path, b: Path):
    diffs = []
    for f in FILES:
        x, y = (a / f).read_bytes(), (b / f).read_bytes()
        if x != y:
            xl, yl = x.decode().splitlines(), y.decode().splitlines()
            i = next((k for k in range(min(len(xl), len(yl))) if xl[k] != yl[k]),
                     min(len(xl), len(yl)))
            diffs.append(f"{f} line {i}: {xl[i] if i < len(xl) else None!r} vs "
                         f"{yl[i] if i < len(yl) else None!r}")
    return diffs


def trace_for(seed, n, rate):
    b = engine.build_workload([seed], n, rate)
    return O.Trace(b.arrival, b.prompt, b.decode, b.task)


@pytest.mark.skipif(not O.have_ref(), reason="compiled reference unavailable")
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_emit_report_bytes_match_reference(tmp_path, case):
    policy, m, n, rate, seed, reward, record = case
    cfg = abi.default_config(policy, m)
    tr = trace_for(seed, n, rate)
    ps = abi.mix_seed(seed, 0x9DED)
    O.ref_emit_report(cfg, tr, tmp_path / "ref", ps, 0, record, reward)
    res, traj = O.ora_trajectory(cfg, tr, ps, reward=reward)
    report.emit_report(tmp_path / "ours", cfg, tr.arrival, tr.prompt, tr.decode, tr.task,
                       res.instance, res.routed, res.first, res.completion, res.preemptions,
                       res.stats, traj if record else None)
    assert same_files(tmp_path / "ref", tmp_path / "ours") == []


def test_emit_report_golden_summary(tmp_path):
    """The reference's own golden (proj/tests/golden/mini_summary.json,
    frozen in tests/golden/) reproduced byte for byte from the oracle's
    replay of its configuration (JSQ, m=2, n=12, lambda=12, seed 777)."""
    cfg = abi.default_config("jsq", 2)
    tr = trace_for(777, 12, 12.0)
    ps = abi.mix_seed(777, 0x9DED)
    res, traj = O.ora_trajectory(cfg, tr, ps, reward={"shaping": "none"})
    report.emit_report(tmp_path, cfg, tr.arrival, tr.prompt, tr.decode, tr.task, res.instance,
                       res.routed, res.first, res.completion, res.preemptions, res.stats, traj)
    golden = Path(__file__).resolve().parent / "golden" / "mini_summary.json"
    assert (tmp_path / "summary.json").read_bytes() == golden.read_bytes()


def test_emit_report_no_completions_raises(tmp_path):
    cfg = abi.default_config("jsq", 2)
    tr = trace_for(1, 5, 10.0)
    st = np.zeros(1, abi.STATS_DTYPE)
    neg = np.full(5, -1.0)
    with pytest.raises(abi.EngineError, match="no completed requests"):
        report.emit_report(tmp_path, cfg, tr.arrival, tr.prompt, tr.decode, tr.task,
                           np.full(5, -1), neg, neg, neg, np.zeros(5), st)


@pytest.mark.gpu
@pytest.mark.skipif(not O.have_ref(), reason="compiled reference unavailable")
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_gpu_emit_report_bytes_match_reference(tmp_path, case):
    """Engine outputs (device sums + device percentiles + device trajectory)
    -> rs_emit_report == the reference's emit_report, byte for byte."""
    policy, m, n, rate, seed, reward, record = case
    cfg = abi.default_config(policy, m)
    tr = trace_for(seed, n, rate)
    ps = abi.mix_seed(seed, 0x9DED)
    O.ref_emit_report(cfg, tr, tmp_path / "ref", ps, 0, record, reward)
    tb = engine.TraceBatch.from_traces([tr])
    sim = engine.BatchSim(engine.ClusterConfig(num_instances=m), tb, [ps])
    rc = engine.RewardConfig(**{k: v for k, v in reward.items() if k != "episode_k"})
    res, traj = sim.run_trajectory(policy, 100_000, rc, episode_k=reward.get("episode_k", 0))
    assert int(res.stats["percentiles_valid"][0]) == 1
    k = int(res.stats["ticks"][0])
    report.emit_report(tmp_path / "ours", cfg, tr.arrival, tr.prompt, tr.decode, tr.task,
                       res.instance, res.routed, res.first, res.completion, res.preemptions,
                       res.stats[0:1], {f: a[0, :k] for f, a in traj.items()} if record else None)
    assert same_files(tmp_path / "ref", tmp_path / "ours") == []
