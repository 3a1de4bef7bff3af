"""GPU parity: the sm_100a engine against the pinned oracle and the frozen
reference fixtures, called through the C ABI (rs_replay_batch_host).

Bar: bit-exact routing decisions (per-tick action hash), per-request
instance, predicted bucket, preemption count and fp64 routed / first-token /
completion times, and the per-replay stats."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine, report

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(params=["fast", "general", "streamed", "tail"], autouse=True)
def kernel_path(request, monkeypatch):
    """Every parity test runs on both replay kernels: the lane-per-instance
    fast kernel (whole-prompt prefill) and the general warp-per-instance one;
    "streamed" forces rs_replay_batch_host's chunked input copies overlapping
    the fast kernel (taken whenever the replays have equal lengths);
    "tail" keeps only 2 running entries per instance in shared memory, so
    every larger running batch continues in the warp's global tail."""
    if request.param == "general":
        monkeypatch.setenv("RS_FORCE_GENERAL", "1")
    else:
        monkeypatch.delenv("RS_FORCE_GENERAL", raising=False)
    monkeypatch.setenv("RS_STREAM_INPUTS", "1" if request.param == "streamed" else "0")
    if request.param == "tail":
        monkeypatch.setenv("RS_RUN_SMEM", "2")
    else:
        monkeypatch.delenv("RS_RUN_SMEM", raising=False)
    return request.param


def run_engine(lib, cfg, traces, pseeds, qseeds=None):
    tb = engine.TraceBatch.from_traces(traces)
    N, R = tb.total, tb.num_replays
    ps = np.ascontiguousarray(pseeds, np.uint64)
    qs = None if qseeds is None else np.ascontiguousarray(qseeds, np.uint64)
    tr = abi.TraceSoA(R, 0, N, tb.offsets.ctypes.data, tb.arrival.ctypes.data,
                      tb.prompt.ctypes.data, tb.decode.ctypes.data, tb.task.ctypes.data, None,
                      ps.ctypes.data, abi.ptr(qs))
    arrs = [np.empty(N, np.int32), np.empty(N, np.float64), np.empty(N, np.float64),
            np.empty(N, np.float64), np.empty(N, np.int32), np.empty(N, np.uint8)]
    stats = np.zeros(R, abi.STATS_DTYPE)
    out = abi.ReqOut(*[a.ctypes.data for a in arrs])
    abi.check(lib, lib.rs_replay_batch_host(C.byref(cfg), C.byref(tr), C.byref(out),
                                            stats.ctypes.data, 0))
    res = []
    for r in range(R):
        s = tb.replay(r)
        res.append(O.ReplayResult(*[a[s] for a in arrs], stats[r:r + 1]))
    return res


def load_golden():
    z = np.load(GOLDEN / "replays.npz")
    return {k: z[k] for k in z.files}, json.loads((GOLDEN / "replays.json").read_text())


GOLD = None


def golden_case(name):
    global GOLD
    if GOLD is None:
        GOLD = load_golden()
    arr, meta = GOLD
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


@pytest.mark.parametrize("name", sorted(json.loads((GOLDEN / "replays.json").read_text())))
def test_engine_reproduces_reference_golden(gpu, name):
    cfg, tr, meta, want, keep = golden_case(name)
    got = run_engine(gpu, cfg, [tr], [meta["predictor_seed"]], [meta["policy_seed"]])[0]
    assert O.compare(got, want) == []
    del keep


@pytest.mark.parametrize("pol", [p for p in abi.POLICIES if p != "rl"])
def test_batched_replays_match_oracle(gpu, pol):
    # 24 seeds of the c1 shape plus ragged sizes (incl. a 1-request replay)
    sizes = [2000] * 20 + [1, 7, 333, 1200]
    seeds = list(range(1, len(sizes) + 1))
    tb = engine.build_workload(seeds[:20], 2000, 20.0)
    traces = [O.Trace(tb.arrival[tb.replay(r)], tb.prompt[tb.replay(r)], tb.decode[tb.replay(r)],
                      tb.task[tb.replay(r)]) for r in range(20)]
    for s, n in zip(seeds[20:], sizes[20:]):
        t = engine.build_workload([s], n, 20.0)
        traces.append(O.Trace(t.arrival, t.prompt, t.decode, t.task))
    m = 4 if pol != "max_capacity" else 3
    cfg = abi.default_config(pol, m)
    ps = [abi.mix_seed(s, 0x9DED) for s in seeds]
    got = run_engine(gpu, cfg, traces, ps)
    for r, tr in enumerate(traces):
        want = O.ora_run(cfg, tr, ps[r])
        assert O.compare(got[r], want) == [], f"replay {r}"


@pytest.mark.parametrize("m,eps,glob", [(4, 0.0, 0), (8, 0.0, 0), (4, 0.3, 0), (2, 0.0, 0),
                                        (8, 0.0, 1), (64, 0.0, 0), (4, 0.0, "wide"),
                                        (4, 0.3, "wide")])
def test_rl_router_matches_oracle(gpu, m, eps, glob, monkeypatch):
    # glob=1 forces the global-memory (L2) weights path; m=64 needs it anyway;
    # "wide" forces 16-warp blocks (the 512-thread RL instantiation)
    if glob == "wide":
        monkeypatch.setenv("RS_WARPS_PER_BLOCK", "16")
        monkeypatch.setenv("RS_WAIT_RING", "8")  # small replay slots: 16 fit next to the net
    elif glob:
        monkeypatch.setenv("RS_RL_GLOBAL", "1")
    sd = abi.state_dimension(m)
    rng = np.random.default_rng(m)
    dims = [sd, 64, 64, m + 1]
    params = rng.uniform(-1, 1, abi.mlp_param_count(dims)) * 0.3
    cfg = abi.default_config("rl", m)
    keep = abi.set_rl(cfg, dims, params)
    cfg.rl_epsilon = eps
    cfg.max_ticks = 200000
    tb = engine.build_workload(range(1, 9), 600, 40.0)
    traces = [O.Trace(tb.arrival[tb.replay(r)], tb.prompt[tb.replay(r)], tb.decode[tb.replay(r)],
                      tb.task[tb.replay(r)]) for r in range(8)]
    ps = [abi.mix_seed(s, 0x9DED) for s in range(1, 9)]
    qs = [1000 + s for s in range(8)]
    got = run_engine(gpu, cfg, traces, ps, qs)
    for r, tr in enumerate(traces):
        want = O.ora_run(cfg, tr, ps[r], qs[r])
        assert O.compare(got[r], want) == [], f"replay {r}"
    del keep


@pytest.mark.parametrize("variant", ["chunk64", "chunk512", "bin_packing", "lwl", "kv5000",
                                     "batch8", "m1", "m32", "m40", "m64", "ring_overflow"])
def test_instance_variants_match_oracle(gpu, variant, monkeypatch):
    pols = ["jsq", "round_robin", "workload_aware", "min_min", "decode_balancer"]
    m = {"m1": 1, "m32": 32, "m40": 40, "m64": 64}.get(variant, 3)
    if m > 32:  # two instances per lane (c5's fleet shape): every heuristic
        pols = sorted(abi.POLICIES.keys() - {"rl"})
    for pol in pols:
        cfg = abi.default_config(pol, m)
        if variant.startswith("chunk"):
            cfg.chunk_size = int(variant[5:])
        elif variant == "bin_packing":
            cfg.batching = 1
        elif variant == "lwl":
            cfg.batching = 2
        elif variant == "kv5000":
            cfg.kv_capacity_tokens = 5000
            for t in range(5):
                cfg.accuracy[t] = 0.2
        elif variant == "batch8":
            cfg.max_batch_size = 8
        elif variant == "ring_overflow":
            monkeypatch.setenv("RS_WAIT_RING", "8")
        cfg.max_ticks = 100000
        tb = engine.build_workload(range(40, 46), 700 if m <= 32 else 2500,
                                   35.0 if m > 1 else 8.0)
        traces = [O.Trace(tb.arrival[tb.replay(r)], tb.prompt[tb.replay(r)],
                          tb.decode[tb.replay(r)], tb.task[tb.replay(r)]) for r in range(6)]
        ps = [abi.mix_seed(s, 0x9DED) for s in range(40, 46)]
        got = run_engine(gpu, cfg, traces, ps)
        for r, tr in enumerate(traces):
            want = O.ora_run(cfg, tr, ps[r])
            assert O.compare(got[r], want) == [], f"{variant} {pol} replay {r}"


def test_preemption_paths_match_oracle(gpu, monkeypatch):
    rng = np.random.default_rng(3)
    for ring in ("64", "8"):
        monkeypatch.setenv("RS_WAIT_RING", ring)
        for pol in ("jsq", "round_robin", "workload_aware", "min_min"):
            for bat in (0, 1, 2):
                rows = [(i * 0.05, int(rng.integers(100, 600)), int(rng.integers(600, 999)),
                         int(rng.integers(0, 5))) for i in range(150)]
                tr = O.make_trace(rows)
                cfg = abi.default_config(pol, 2)
                cfg.kv_capacity_tokens = 6000
                cfg.batching = bat
                cfg.max_ticks = 200000
                for t in range(5):
                    cfg.accuracy[t] = 0.0
                got = run_engine(gpu, cfg, [tr], [5])[0]
                want = O.ora_run(cfg, tr, 5)
                assert O.compare(got, want) == [], (ring, pol, bat)


def test_golden_summary_on_gpu(gpu):
    sim = engine.BatchSim(engine.ClusterConfig(num_instances=2),
                          engine.build_workload([777], 12, 12.0), [abi.mix_seed(777, 0x9DED)])
    res = sim.run_policy("jsq")
    r = res.replay(0)
    got = report.summary(sim.traces.arrival, sim.traces.decode, r["routed"], r["first"],
                         r["completion"], r["preemptions"], res.stats[0], 2)
    assert got == json.loads((GOLDEN / "mini_summary.json").read_text())


def test_mlp_forward_kernel_matches_oracle(gpu):
    rng = np.random.default_rng(9)
    for dims in ([27, 64, 64, 5], [51, 64, 64, 9], [387, 128, 128, 65], [9, 3, 2]):  # m=64: 387 wide
        p = rng.standard_normal(abi.mlp_param_count(dims))
        x = rng.standard_normal((257, dims[0]))
        x[rng.random(x.shape) < 0.5] = 0.0
        q, g = engine.mlp_forward(dims, p, x)
        cfg = abi.default_config("rl", dims[-1] - 1)
        keep = abi.set_rl(cfg, dims, p)
        q2, g2 = np.empty_like(q), np.empty(257, np.int32)
        assert O.ora_lib().ora_mlp_forward(C.byref(cfg), x.ctypes.data, 257, q2.ctypes.data,
                                            g2.ctypes.data) == 0
        assert np.array_equal(g, g2)
        assert np.array_equal(q, q2)  # == (only the sign of an exact zero may differ)
        del keep


def test_full_size_c2_shape_matches_oracle(gpu):
    # BASELINE config 2 shape: 31,329 requests, 8 instances, workload-aware.
    seeds = [1, 2]
    tb = engine.build_workload(seeds, 31329, 20.0)
    traces = [O.Trace(tb.arrival[tb.replay(r)], tb.prompt[tb.replay(r)], tb.decode[tb.replay(r)],
                      tb.task[tb.replay(r)]) for r in range(2)]
    ps = [abi.mix_seed(s, 0x9DED) for s in seeds]
    for pol in ("workload_aware", "jsq"):
        cfg = abi.default_config(pol, 8)
        got = run_engine(gpu, cfg, traces, ps)
        for r, tr in enumerate(traces):
            want = O.ora_run(cfg, tr, ps[r])
            assert O.compare(got[r], want) == [], (pol, r)


def test_conservation_properties_at_scale(gpu):
    # Size-independent invariants on a 256-replay batch (no oracle needed).
    seeds = np.arange(100, 356)
    tb = engine.build_workload(seeds, 4000, 40.0)
    sim = engine.BatchSim(engine.ClusterConfig(num_instances=8), tb,
                          [abi.mix_seed(int(s), 0x9DED) for s in seeds])
    res = sim.run_policy("workload_aware")
    st = res.stats
    assert np.all(st["status"] == abi.REPLAY_FINISHED)
    assert np.all(st["completed"] == 4000)
    assert np.all(st["routed"] == 4000)
    assert np.all(st["total_tokens"] == np.add.reduceat(tb.decode.astype(np.int64), tb.offsets[:-1]))
    assert np.all(res.completion >= res.first)
    assert np.all(res.first > res.routed)
    assert np.all(res.routed >= tb.arrival)
    assert np.all((res.instance >= 0) & (res.instance < 8))
    # determinism: identical inputs, identical decisions
    res2 = sim.run_policy("workload_aware")
    assert np.array_equal(res.stats["decision_hash"], res2.stats["decision_hash"])
    assert np.array_equal(res.completion.view(np.uint64), res2.completion.view(np.uint64))


def test_streamed_inputs_validate_per_window(gpu, kernel_path):
    # Streamed inputs are validated as each 32-request window lands: a bad
    # request deep in one replay fails that replay only.
    if kernel_path != "streamed":
        pytest.skip("streamed-input path only")
    tb = engine.build_workload([5, 6, 7], 3000, 20.0)
    traces = [O.Trace(tb.arrival[tb.replay(r)].copy(), tb.prompt[tb.replay(r)].copy(),
                      tb.decode[tb.replay(r)].copy(), tb.task[tb.replay(r)].copy())
              for r in range(3)]
    traces[1].arrival[2500] = traces[1].arrival[2499] - 1.0  # arrivals out of order
    traces[2].prompt[1700] = 0                                # empty prompt
    ps = [abi.mix_seed(s, 0x9DED) for s in (5, 6, 7)]
    cfg = abi.default_config("workload_aware", 4)
    got = run_engine(gpu, cfg, traces, ps)
    assert O.compare(got[0], O.ora_run(cfg, traces[0], ps[0])) == []
    assert got[1].stats["status"][0] == abi.REPLAY_INVALID_TRACE
    assert got[2].stats["status"][0] == abi.REPLAY_INVALID_TRACE



@pytest.mark.parametrize("m", [40, 64])
def test_large_fleets_warp_pairs_and_reruns(gpu, kernel_path, m, monkeypatch):
    """33..64 instances: the warp-pair kernel (pair.cuh; "fast" and "tail"
    paths), the two-instances-per-lane kernel (RS_NO_PAIR, and the streamed
    path), every heuristic pair build, and the pair kernel's re-runs on the
    single-warp code: "nothing admissible" (index-order re-run) and
    max_ticks (re-run with output initialisation)."""
    if kernel_path == "general":
        pytest.skip("fast-kernel plans only")
    for no_pair in ("0", "1"):
        monkeypatch.setenv("RS_NO_PAIR", no_pair)
        tb = engine.build_workload(range(60, 64), 1800, 30.0)
        traces = [O.Trace(tb.arrival[tb.replay(r)], tb.prompt[tb.replay(r)],
                          tb.decode[tb.replay(r)], tb.task[tb.replay(r)]) for r in range(4)]
        ps = [abi.mix_seed(s, 0x9DED) for s in range(60, 64)]
        cases = [(pol, {}) for pol in sorted(abi.POLICIES.keys() - {"rl", "min_min"})]
        cases += [("jsq", {"kv_capacity_tokens": 4096}),            # nothing admissible
                  ("round_robin", {"kv_capacity_tokens": 4096, "max_ticks": 20000})]  # unfinished
        for pol, over in cases:
            cfg = abi.default_config(pol, m)
            for k, v in over.items():
                setattr(cfg, k, v)
            got = run_engine(gpu, cfg, traces, ps)
            for r, tr in enumerate(traces):
                want = O.ora_run(cfg, tr, ps[r])
                assert O.compare(got[r], want) == [], (no_pair, pol, over, r)


@pytest.mark.parametrize("m", [4, 8, 40])
def test_no_head_windows_match_oracle(gpu, kernel_path, m, monkeypatch):
    """No-head windows (fast_kernel.cuh / pair.cuh): the ticks between an
    empty router queue and the next arrival run as one run_until.  Sparse
    arrivals (long windows), tick lengths below and above a decode step (one
    step crossing several boundaries: each must add the waiting count of the
    state before the next step), max_ticks falling inside a window, and
    bin-packing admission (waiting queues that persist through a window)."""
    if kernel_path == "general" and m > 32:
        pytest.skip("general kernel: covered at m <= 32")
    monkeypatch.setenv("RS_NO_PAIR", "0")
    tb = engine.build_workload(range(80, 84), 700, 3.0 if m <= 8 else 12.0)
    traces = [O.Trace(tb.arrival[tb.replay(r)], tb.prompt[tb.replay(r)],
                      tb.decode[tb.replay(r)], tb.task[tb.replay(r)]) for r in range(4)]
    ps = [abi.mix_seed(s, 0x9DED) for s in range(80, 84)]
    cases = [("workload_aware", {}), ("jsq", {"delta_t": 0.005}),
             ("round_robin", {"delta_t": 0.0931}), ("earliest_available", {"delta_t": 0.3}),
             ("decode_balancer", {"max_ticks": 5003}),
             ("workload_aware", {"delta_t": 0.05, "max_ticks": 1777}),
             ("max_capacity", {"batching": abi.BATCHING["bin_packing"], "kv_capacity_tokens": 6000}),
             ("dedicated_small_large", {"kv_capacity_tokens": 5000, "delta_t": 0.011})]
    for pol, over in cases:
        cfg = abi.default_config(pol, m)
        for k, v in over.items():
            setattr(cfg, k, v)
        got = run_engine(gpu, cfg, traces, ps)
        for r, tr in enumerate(traces):
            want = O.ora_run(cfg, tr, ps[r])
            assert O.compare(got[r], want) == [], (pol, over, r)


def test_qnet_mac_counter(gpu, kernel_path):
    """rs_replay_stats.qnet_macs: the Q-network multiply-adds the replay's
    forwards executed — positive for the RL router, at most the dense count
    per decision (zero inputs skipped, repeated states memoised), 0 for the
    heuristics; the decisions themselves stay bit-exact."""
    m = 4
    tb = engine.build_workload(range(90, 93), 500, 25.0)
    traces = [O.Trace(tb.arrival[tb.replay(r)], tb.prompt[tb.replay(r)],
                      tb.decode[tb.replay(r)], tb.task[tb.replay(r)]) for r in range(3)]
    ps = [abi.mix_seed(s, 0x9DED) for s in range(90, 93)]
    sd = abi.state_dimension(m)
    dims = [sd, 64, 64, m + 1]
    params = engine.mlp_random_init(dims, 42)
    cfg = abi.default_config("rl", m)
    keep = abi.set_rl(cfg, dims, params)  # noqa: F841 (keeps the weights alive)
    dense = sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))
    got = run_engine(gpu, cfg, traces, ps)
    for r, tr in enumerate(traces):
        assert O.compare(got[r], O.ora_run(cfg, tr, ps[r])) == []
        st = got[r].stats[0]
        assert 0 < int(st["qnet_macs"]) < dense * int(st["ticks"])
    got = run_engine(gpu, abi.default_config("jsq", m), traces, ps)
    assert all(int(g.stats[0]["qnet_macs"]) == 0 for g in got)
