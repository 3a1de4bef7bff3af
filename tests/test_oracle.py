"""Pinning the CPU checker (CPU only).

The C restatement (oracle/rs_oracle.c) must reproduce
 * every frozen golden replay of the compiled reference (tests/golden/),
 * the reference's own golden summary (proj/tests/golden/mini_summary.json,
   test_harness.cpp:212-231) through report.summary,
 * the live compiled reference on randomised configurations,
bit for bit, before it is trusted as the GPU engine's parity oracle."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine, report

GOLDEN = Path(__file__).resolve().parent / "golden"


def golden_cases():
    meta = json.loads((GOLDEN / "replays.json").read_text())
    return sorted(meta)


@pytest.fixture(scope="module")
def golden():
    z = np.load(GOLDEN / "replays.npz")
    return {k: z[k] for k in z.files}, json.loads((GOLDEN / "replays.json").read_text())


def golden_case(golden, name):
    arr, meta = golden
    cfg = abi.BatchCfg.from_buffer_copy(arr[f"{name}.cfg"].tobytes())
    cfg.rl_params = None
    keep = None
    if meta[name]["dims"]:
        keep = abi.set_rl(cfg, meta[name]["dims"], arr[f"{name}.params"])
    tr = O.Trace(arr[f"{name}.arrival"], arr[f"{name}.prompt"], arr[f"{name}.decode"],
                 arr[f"{name}.task"])
    want = O.ReplayResult(arr[f"{name}.instance"], arr[f"{name}.routed"], arr[f"{name}.first"],
                          arr[f"{name}.completion"], arr[f"{name}.preemptions"],
                          arr[f"{name}.predicted"], arr[f"{name}.stats"])
    return cfg, tr, meta[name], want, keep


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_reproduces_golden_replay(golden, name):
    cfg, tr, meta, want, keep = golden_case(golden, name)
    got = O.ora_run(cfg, tr, meta["predictor_seed"], meta["policy_seed"])
    assert O.compare(got, want) == []
    del keep


def test_mt19937_64_known_answer():
    out = np.empty(10000, np.uint64)
    O.ora_lib().ora_mt19937_64(5489, 10000, out.ctypes.data)
    assert int(out[-1]) == 9981545732273789042  # C++ [rand.predef] requirement


def test_golden_summary_via_oracle(lib):
    # test_harness.cpp:212-231: JSQ, m=2, n=12, lambda=12, seed 777.
    tb = engine.build_workload([777], 12, 12.0)
    tr = O.Trace(tb.arrival, tb.prompt, tb.decode, tb.task)
    cfg = abi.default_config("jsq", 2)
    res = O.ora_run(cfg, tr, abi.mix_seed(777, 0x9DED))
    got = report.summary(tr.arrival, tr.decode, res.routed, res.first, res.completion,
                         res.preemptions, res.stats[0], 2)
    want = json.loads((GOLDEN / "mini_summary.json").read_text())
    assert got == want  # exact float equality, field by field


@pytest.mark.skipif(not O.have_ref(), reason="reference driver unavailable")
@pytest.mark.parametrize("case", range(24))
def test_oracle_matches_live_reference(case):
    rng = np.random.default_rng(1000 + case)
    pol = list(abi.POLICIES)[case % len(abi.POLICIES)]
    m = int(rng.choice([1, 2, 3, 4, 8]))
    cfg = abi.default_config(pol, m)
    cfg.batching = int(rng.choice([0, 0, 1, 2]))
    cfg.chunk_size = int(rng.choice([0, 0, 64, 300]))
    cfg.kv_capacity_tokens = int(rng.choice([16384, 16384, 8000, 5000]))
    cfg.max_batch_size = int(rng.choice([128, 128, 16, 4]))
    cfg.max_ticks = 60000
    if rng.random() < 0.3:
        for t in range(5):
            cfg.accuracy[t] = float(rng.random())
    n = int(rng.integers(50, 400))
    tr = O.ref_generate(int(rng.integers(1, 1 << 40)), n, float(rng.choice([10.0, 20.0, 45.0])),
                        None if rng.random() < 0.7 else rng.random(5) + 0.01)
    keep = None
    qs = 0
    if pol == "rl":
        sd = abi.state_dimension(m)
        keep = abi.set_rl(cfg, [sd, 32, 32, m + 1],
                          O.ref_agent_params(sd, m + 1, 32, int(rng.integers(1, 1000))))
        if rng.random() < 0.5:
            cfg.rl_epsilon = 0.2
            qs = int(rng.integers(1, 1 << 30))
    ps = int(rng.integers(0, 1 << 62))
    a = O.ref_run(cfg, tr, ps, qs, log_actions=True)
    b = O.ora_run(cfg, tr, ps, qs, log_actions=True)
    assert O.compare(a, b) == []
    del keep


@pytest.mark.skipif(not O.have_ref(), reason="reference driver unavailable")
def test_mlp_forward_matches_reference():
    rng = np.random.default_rng(5)
    for dims in ([27, 64, 64, 5], [51, 64, 64, 9], [9, 3, 2]):
        cfg = abi.default_config("rl", dims[-1] - 1)
        p = rng.standard_normal(abi.mlp_param_count(dims))
        keep = abi.set_rl(cfg, dims, p)
        x = rng.standard_normal((64, dims[0]))
        x[rng.random(x.shape) < 0.4] = 0.0
        q1, g1 = np.empty((64, dims[-1])), np.empty(64, np.int32)
        q2, g2 = np.empty((64, dims[-1])), np.empty(64, np.int32)
        assert O.ref_lib().ref_mlp_forward(C.byref(cfg), x.ctypes.data, 64, q1.ctypes.data,
                                            g1.ctypes.data) == 0
        assert O.ora_lib().ora_mlp_forward(C.byref(cfg), x.ctypes.data, 64, q2.ctypes.data,
                                            g2.ctypes.data) == 0
        assert np.array_equal(q1.view(np.uint64), q2.view(np.uint64))
        assert np.array_equal(g1, g2)
        del keep


def test_patched_reference_without_reward_scan_matches():
    """oracle/_ref/librs_ref_noscan.so (the reference with the reward-only
    queue-penalty scan compiled out) replays to the same
    statistics as the unmodified reference: the scan feeds no decision."""
    if not O.have_ref():
        pytest.skip("reference sources not available")
    for pol, m, seed in (("workload_aware", 4, 3), ("jsq", 8, 4), ("round_robin", 2, 5)):
        tr = O.ref_generate(seed, 1500, 25.0)
        cfg = abi.default_config(pol, m)
        ps = abi.mix_seed(seed, 0x9DED)
        stats = []
        for noscan in (False, True):
            lib = O.ref_lib(noscan=noscan)
            off = np.array([0, tr.arrival.size], np.int64)
            st = np.zeros(1, abi.STATS_DTYPE)
            psa = np.array([ps], np.uint64)
            w = lib.ref_run_batch(C.byref(cfg), 1, off.ctypes.data, tr.arrival.ctypes.data,
                                  tr.prompt.ctypes.data, tr.decode.ctypes.data,
                                  tr.task.ctypes.data, psa.ctypes.data, None, 1,
                                  st.ctypes.data)
            assert w > 0
            stats.append(st)
        assert stats[0].tobytes() == stats[1].tobytes(), pol
