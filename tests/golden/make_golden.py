"""Freeze golden fixtures from the COMPILED REFERENCE (oracle/_ref, built from
the unmodified /root/reference headers).  Run here, where /root/reference
exists; the outputs are committed and the GPU box only reads them.

    python tests/golden/make_golden.py

 * mini_summary.json  — run_experiment for test_harness.cpp:212-231 (JSQ, m=2,
                        n=12, lambda=12, seed 777), report_to_json().dump(2):
                        byte-identical to proj/tests/golden/mini_summary.json.
 * replays.npz        — per-request outputs + per-replay stats of the
                        reference ClusterSim::run_policy for the cases below.
 * trajectories.npz   — ClusterSim::trajectory() (record_trajectory on: the
                        Eq. 3 reward breakdown + TickRecords, env.hpp:251-319)
                        for traj_cases(), under several RewardConfigs.

    python tests/golden/make_golden.py [--traj-only]
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))

import oracles as O  # noqa: E402
from paper_2408_13510_b200 import abi  # noqa: E402


def cases():
    """(name, cfg, trace, predictor_seed, policy_seed, agent) tuples."""
    out = []
    tr = O.ref_generate(1, 2000, 20.0)  # BASELINE c1: 2,000 req, lambda 20, seed 1
    ps = abi.mix_seed(1, 0x9DED)
    for pol in abi.POLICIES:
        if pol == "rl":
            continue
        out.append((f"c1_{pol}", abi.default_config(pol, 4), tr, ps, 0, None))
    params = O.ref_agent_params(27, 5, 64, 42)
    out.append(("c1_rl_seed42", abi.default_config("rl", 4), tr, ps, 0, ([27, 64, 64, 5], params)))
    out.append(("c1_rl_eps", abi.default_config("rl", 4), tr, ps, 99,
                ([27, 64, 64, 5], params)))
    tr8 = O.ref_generate(3, 1500, 40.0)
    p8 = O.ref_agent_params(51, 9, 64, 7)
    out.append(("m8_rl_seed7", abi.default_config("rl", 8), tr8, abi.mix_seed(3, 0x9DED), 0,
                ([51, 64, 64, 9], p8)))
    c = abi.default_config("jsq", 3)
    c.chunk_size = 128
    out.append(("chunk128_jsq", c, O.ref_generate(9, 800, 30.0), abi.mix_seed(9, 0x9DED), 0, None))
    c = abi.default_config("workload_aware", 2)
    c.batching = abi.BATCHING["bin_packing"]
    out.append(("binpack_wa", c, O.ref_generate(10, 600, 25.0), abi.mix_seed(10, 0x9DED), 0, None))
    c = abi.default_config("round_robin", 2)
    c.batching = abi.BATCHING["least_work_left"]
    out.append(("lwl_rr", c, O.ref_generate(11, 600, 25.0), abi.mix_seed(11, 0x9DED), 0, None))
    # overrun-heavy synthetic trace: preemptions
    rng = np.random.default_rng(3)
    rows = [(i * 0.05, int(rng.integers(100, 600)), int(rng.integers(600, 999)),
             int(rng.integers(0, 5))) for i in range(150)]
    c = abi.default_config("jsq", 2)
    c.kv_capacity_tokens = 6000
    for t in range(5):
        c.accuracy[t] = 0.0
    out.append(("preempt_jsq", c, O.make_trace(rows), 5, 0, None))
    # starvation (test_env.cpp:359-380 defect): round robin livelocks
    c = abi.default_config("round_robin", 2)
    c.kv_capacity_tokens = 4096
    c.max_ticks = 30000
    out.append(("livelock_rr", c, O.ref_generate(5, 120, 30.0), abi.mix_seed(5, 0x9DED), 0, None))
    # logic_error: nothing admissible
    c = abi.default_config("jsq", 2)
    c.kv_capacity_tokens = 4096
    out.append(("not_admissible_jsq", c, O.ref_generate(5, 300, 30.0), abi.mix_seed(5, 0x9DED), 0,
                None))
    return out


def traj_cases():
    """(name, cfg, trace, predictor_seed, policy_seed, agent, reward) tuples."""
    out = []
    tr = O.ref_generate(21, 300, 20.0)
    ps = abi.mix_seed(21, 0x9DED)
    out.append(("jsq_default", abi.default_config("jsq", 4), tr, ps, 0, None, {}))
    out.append(("wa_guided_k2", abi.default_config("workload_aware", 4), tr, ps, 0, None,
                {"shaping": "guided", "episode_k": 2}))
    out.append(("rr_additive_rw30", abi.default_config("round_robin", 4),
                O.ref_generate(22, 250, 45.0), abi.mix_seed(22, 0x9DED), 0, None,
                {"shaping": "additive", "r_w": 30.0}))
    out.append(("minmin_none", abi.default_config("min_min", 3), O.ref_generate(23, 250, 60.0),
                abi.mix_seed(23, 0x9DED), 0, None, {"shaping": "none"}))
    c = abi.default_config("decode_balancer", 3)
    c.chunk_size = 96
    out.append(("chunk96_db", c, O.ref_generate(24, 250, 30.0), abi.mix_seed(24, 0x9DED), 0, None,
                {"episode_k": 5}))
    rng = np.random.default_rng(4)
    rows = [(i * 0.05, int(rng.integers(100, 600)), int(rng.integers(600, 999)),
             int(rng.integers(0, 5))) for i in range(120)]
    c = abi.default_config("jsq", 2)
    c.kv_capacity_tokens = 6000
    for t in range(5):
        c.accuracy[t] = 0.0
    out.append(("preempt_jsq", c, O.make_trace(rows), 6, 0, None, {"shaping": "additive"}))
    params = O.ref_agent_params(27, 5, 64, 42)
    out.append(("rl_eps", abi.default_config("rl", 4), O.ref_generate(25, 200, 30.0),
                abi.mix_seed(25, 0x9DED), 77, ([27, 64, 64, 5], params), {"episode_k": 1}))
    return out


def main_traj():
    arrays = {}
    meta = {}
    for name, cfg, tr, ps, qs, agent, reward in traj_cases():
        keep = None
        if agent is not None:
            keep = abi.set_rl(cfg, agent[0], agent[1])
            arrays[f"{name}.params"] = agent[1]
            cfg.rl_epsilon = 0.2
        res, traj = O.ref_trajectory(cfg, tr, ps, qs, reward=reward)
        arrays.update({f"{name}.arrival": tr.arrival, f"{name}.prompt": tr.prompt,
                       f"{name}.decode": tr.decode, f"{name}.task": tr.task,
                       f"{name}.stats": res.stats, f"{name}.completion": res.completion,
                       f"{name}.cfg": np.frombuffer(bytes(cfg), np.uint8)})
        for k, v in traj.items():
            arrays[f"{name}.traj.{k}"] = v
        meta[name] = {"predictor_seed": ps, "policy_seed": qs, "reward": reward,
                      "dims": agent[0] if agent else None,
                      "ticks": int(res.stats["ticks"][0])}
        del keep
        print(f"traj {name:20s} ticks={meta[name]['ticks']:8d}")
    np.savez_compressed(HERE / "trajectories.npz", **arrays)
    (HERE / "trajectories.json").write_text(json.dumps(meta, indent=1) + "\n")


def main():
    main_traj()
    if "--traj-only" in sys.argv:
        return
    lib = O.ref_lib()
    buf = C.create_string_buffer(1 << 16)
    assert lib.ref_golden_summary(buf, len(buf), 1) == 0
    (HERE / "mini_summary.json").write_text(buf.value.decode())
    arrays = {}
    meta = {}
    for name, cfg, tr, ps, qs, agent in cases():
        keep = None
        if agent is not None:
            keep = abi.set_rl(cfg, agent[0], agent[1])
            arrays[f"{name}.params"] = agent[1]
        if name == "c1_rl_eps":
            cfg.rl_epsilon = 0.1
        res = O.ref_run(cfg, tr, ps, qs)
        arrays.update({f"{name}.arrival": tr.arrival, f"{name}.prompt": tr.prompt,
                       f"{name}.decode": tr.decode, f"{name}.task": tr.task,
                       f"{name}.instance": res.instance, f"{name}.routed": res.routed,
                       f"{name}.first": res.first, f"{name}.completion": res.completion,
                       f"{name}.preemptions": res.preemptions, f"{name}.predicted": res.predicted,
                       f"{name}.stats": res.stats, f"{name}.cfg": np.frombuffer(bytes(cfg), np.uint8)})
        meta[name] = {"predictor_seed": ps, "policy_seed": qs,
                      "dims": agent[0] if agent else None,
                      "ticks": int(res.stats["ticks"][0]), "status": int(res.stats["status"][0])}
        del keep
        print(f"{name:24s} ticks={meta[name]['ticks']:8d} status={meta[name]['status']}")
    np.savez_compressed(HERE / "replays.npz", **arrays)
    (HERE / "replays.json").write_text(json.dumps(meta, indent=1) + "\n")


if __name__ == "__main__":
    main()
