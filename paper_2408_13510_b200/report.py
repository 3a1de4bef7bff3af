"""Per-replay report in the reference's summary.json shape (metrics.hpp:84-194),
and emit_report (metrics.hpp:197-238) through the engine library's C ABI
(rs_emit_report: byte-identical summary.json / requests.csv / timeseries.csv).

The fp64 sums are the engine's own sequential, pool-index-order sums
(rs_replay_stats), so means are bit-identical to compute_metrics; the
nearest-rank percentiles are taken here on the host from the per-request
outputs (aggregate_of, metrics.hpp:62-80).
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from . import abi


def nearest_rank(sorted_values: np.ndarray, q: float) -> float:
    n = sorted_values.shape[0]
    idx = int(math.ceil(q * n))
    if idx > 0:
        idx -= 1
    return float(sorted_values[min(idx, n - 1)])


def _agg(values: np.ndarray, total: float) -> dict:
    n = int(values.shape[0])
    if n == 0:
        return {"mean": 0.0, "p50": 0.0, "p90": 0.0, "p99": 0.0, "count": 0}
    v = np.sort(values)
    return {"mean": total / n, "p50": nearest_rank(v, 0.50), "p90": nearest_rank(v, 0.90),
            "p99": nearest_rank(v, 0.99), "count": n}


def summary(arrival, decode, routed, first, completion, preemptions, stats, num_instances) -> dict:
    """report_to_json(compute_metrics(...)) for one replay (metrics.hpp:172-194)."""
    done = completion >= 0.0
    e2e = completion[done] - arrival[done]
    ttft = first[done] - arrival[done]
    dd = decode[done]
    has_tbt = dd >= 2
    tbt = (completion[done][has_tbt] - first[done][has_tbt]) / (dd[has_tbt] - 1).astype(np.float64)
    ticks = int(stats["ticks"])
    if int(stats["percentiles_valid"]):
        # device nearest-rank selections (stats_kernel, stats.cuh)
        def _dev(name, n, total):
            return {"mean": total / n if n else 0.0, "p50": float(stats[f"{name}_p50"]),
                    "p90": float(stats[f"{name}_p90"]), "p99": float(stats[f"{name}_p99"]),
                    "count": int(n)}
        e2e_agg = _dev("e2e", e2e.shape[0], float(stats["total_e2e_s"]))
        ttft_agg = _dev("ttft", ttft.shape[0], float(stats["total_ttft_s"]))
        tbt_agg = _dev("tbt", tbt.shape[0], float(stats["total_tbt_s"]))
    else:
        e2e_agg = _agg(e2e, float(stats["total_e2e_s"]))
        ttft_agg = _agg(ttft, float(stats["total_ttft_s"]))
        tbt_agg = _agg(tbt, float(stats["total_tbt_s"]))
    out = {
        "completed": int(stats["completed"]),
        "total_tokens": int(stats["total_tokens"]),
        "total_e2e_s": float(stats["total_e2e_s"]),
        "makespan_s": float(stats["makespan_s"]),
        "e2e_s": e2e_agg,
        "ttft_s": ttft_agg,
        "tbt_s": tbt_agg,
        "mean_router_wait_s": (float(stats["total_router_wait_s"]) / int(done.sum())
                               if done.any() else 0.0),
        "mean_router_queue": float(stats["sum_router_queue"]) / ticks if ticks else 0.0,
        "mean_instance_waiting": (float(stats["sum_instance_waiting"]) / (ticks * num_instances)
                                  if ticks else 0.0),
        "mean_throughput_tokens_s": (float(stats["total_tokens"]) / float(stats["makespan_s"])
                                     if float(stats["makespan_s"]) > 0.0 else 0.0),
        "total_preemptions": int(stats["total_preemptions"]),
    }
    return out


def emit_report(directory, cfg: abi.BatchCfg, arrival, prompt, decode, task, instance, routed,
                first, completion, preemptions, stats, trajectory: dict | None = None) -> None:
    """emit_report(compute_metrics(...), trajectory, dir) for ONE replay
    (metrics.hpp:84-238), through rs_emit_report.  `stats` is the replay's
    STATS_DTYPE record; `trajectory` its {TickRecord field: array} (the
    replay's row of BatchSim.run_trajectory, trimmed to its tick count) or
    None for a record_trajectory = false report."""
    lib = abi.load_library()
    c = lambda a, dt: np.ascontiguousarray(a, dtype=dt)
    arrs = [c(arrival, np.float64), c(prompt, np.int32), c(decode, np.int32), c(task, np.uint8),
            c(instance, np.int32), c(routed, np.float64), c(first, np.float64),
            c(completion, np.float64), c(preemptions, np.int32)]
    st = np.ascontiguousarray(np.asarray(stats).reshape(-1)[:1], dtype=abi.STATS_DTYPE)
    t = None
    k = 0
    keep = []
    if trajectory is not None:
        t = abi.Trajectory()
        for name, dt, _ in abi.TRAJ_FIELDS:
            if name in trajectory:
                a = np.ascontiguousarray(trajectory[name], dtype=dt)
                keep.append(a)
                setattr(t, name, a.ctypes.data)
                k = int(a.shape[0])
    abi.check(lib, lib.rs_emit_report(os.fsencode(str(directory)), C.byref(cfg), len(arrs[0]),
                                      *[a.ctypes.data for a in arrs], st.ctypes.data,
                                      C.byref(t) if t is not None else None, k))
