#!/usr/bin/env python
"""Benchmark: routing decisions/s over batched trace replays (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl engine|reference]

Default workload (config c2 of BASELINE.json): 31,329-request 5-task-mix
traces (Poisson lambda = 20/s), 1,024 seeds per GPU, 8 instances, the
workload-aware router.  One step = one pass of the hot path over the whole
batch: predictor kernel (d) + fused replay kernel (a+b+c) with the inputs
resident in HBM, then a final NCCL all-gather of the per-replay statistics.

 * value : decisions (ClusterSim ticks) of all replays of all ranks / max-over-
           ranks device time of the step (CUDA events on the launch stream).
 * e2e   : the same metric through the reference-facing C-ABI host call
           rs_replay_batch_host with pinned host buffers (H2D + kernels + D2H
           of every per-request result inside the timed region).
 * cpu_baseline (rank 0, N = 1): the compiled UNMODIFIED reference
           (oracle/_ref) on the host cores over a bounded seed sample.
 * --impl reference: the reference's own CPU path on all host cores.
Multi-GPU: one process per GPU (torchrun), replays sharded by seed (weak
scaling, no data-path collective), stats gathered over NCCL at the end.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "routing decisions/sec over batched trace replays (whole box) at 1/2/4/8 B200"
UNIT = "decisions/s"
REPLAY_BYTES_PER_REQUEST = 8 + 4 + 4 + 1 + (4 + 8 + 8 + 8 + 4)  # in: arrival, prompt, decode, bucket; out
REPLAY_BYTES_PER_REPLAY = 8 + 256  # offsets + stats record
PREWARM_S = float(os.environ.get("RS_BENCH_PREWARM_S", "2.0"))  # 0 under ncu (tools/profile.sh)
GATE_S = 0.3  # device spin ahead of the timed region's start event (see the timed loop)
E2E_WINDOWS = 3  # e2e: median of this many timed windows of K steps (see timed_e2e)

CONFIGS = {
    # name: (requests, seeds per GPU, instances, rate(s), policy (or policies), weights, description)
    "c1": (2000, 1, 4, 20.0, "workload_aware", None,
           "c1: single 2,000-request 5-task-mix trace (lambda=20), 4 instances, workload_aware"),
    "c2": (31329, 1024, 8, 20.0, "workload_aware", None,
           "c2: 31,329-request 5-task-mix trace (Poisson lambda=20) x 1,024 seeds per GPU, "
           "8 instances, workload_aware router"),
    "c3": (4000, 4096, 8, 40.0, "rl", None,
           "c3: RL Q-network (51-64-64-9, random init seed 42) greedy rollouts, 4,096 replays x "
           "4,000 requests (lambda=40), 8 instances"),
    "c4": (2000, 1024, 4, tuple(5.0 * k for k in range(1, 17)),
           ("round_robin", "jsq", "workload_aware", "rl"), None,
           "c4: policy sweep {round_robin, jsq, workload_aware, rl (27-64-64-5, random init "
           "seed 42)} x 16 arrival rates (lambda=5..80) x 1,024 seeds per GPU, 2,000-request "
           "traces, 4 instances (65,536 replays per GPU per step)"),
    "c5": (200000, 512, 64, 40.0, "workload_aware", (0.0, 3.0, 1.0, 2.0, 0.0),
           "c5: 64 instances, 200k-request heavy-decode mixture (weights 0/3/1/2/0, lambda=40) "
           "x 512 seeds per GPU"),
}


def cfg_shape(cfgname):
    """(requests, seeds per GPU, instances, rates, policies, weights, description)."""
    n, R, m, rate, pol, w, desc = CONFIGS[cfgname]
    rates = tuple(rate) if isinstance(rate, tuple) else (rate,)
    pols = tuple(pol) if isinstance(pol, tuple) else (pol,)
    return n, R, m, rates, pols, w, desc


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region.

    Started before the warm-up (nvidia-smi's own start-up disturbs the GPU for
    tens of ms: measured as a slow first timed step when it was started at
    the timed region), stopped after it; only the samples whose timestamps
    fall inside the timed window (`mark`) are summarised."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.out = b""
        self.window = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        import datetime
        rows = []
        for line in self.out.decode(errors="replace").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or not f[1].isdigit() or int(f[1]) not in self.gpus:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            try:
                rows.append((ts, int(f[2]), int(f[3]), f[5:9]))
            except ValueError:
                continue
        if self.window and rows:
            t0, t1 = self.window
            inside = [r for r in rows if r[0] is not None and t0 - 0.05 <= r[0] <= t1 + 0.25]
            rows = inside or rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [r for r in rows if r[1] > 500] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": float(np.median([r[1] for r in load])),
                "sm_max_mhz": max(r[2] for r in rows), "reasons": reasons, "samples": len(load)}


def make_workload(cfgname, rank, threads=0):
    """The config's traces on this rank: for every arrival rate, seeds
    rank*R+1..(rank+1)*R (one replay each), rate-major.  Every policy of a
    sweep replays the same traces."""
    from paper_2408_13510_b200 import abi, engine
    n, R, m, rates, pols, weights, desc = cfg_shape(cfgname)
    seeds = np.arange(rank * R + 1, rank * R + R + 1, dtype=np.uint64)
    parts = [engine.build_workload(seeds, n, rate, weights, threads=threads) for rate in rates]
    if len(parts) == 1:
        tb = parts[0]
    else:
        cat = lambda f: np.ascontiguousarray(np.concatenate([getattr(t, f) for t in parts]))
        off = np.arange(len(parts) * R + 1, dtype=np.int64) * n
        tb = engine.TraceBatch(off, cat("arrival"), cat("prompt"), cat("decode"), cat("task"))
    all_seeds = np.tile(seeds, len(rates))
    pseeds = np.array([abi.mix_seed(int(s), 0x9DED) for s in all_seeds], np.uint64)
    return tb, pseeds, all_seeds


def agent_for(m):
    """DqnAgent(state_dim, m+1, hidden 64, seed 42) initial weights (Mlp::random)."""
    from paper_2408_13510_b200 import abi, engine
    sd = abi.state_dimension(m)
    dims = [sd, 64, 64, m + 1]
    return dims, engine.mlp_random_init(dims, 42)


def ref_agent_for(m):
    """The same agent from the compiled reference (DqnAgent ctor, dqn.hpp:60-65)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles as O  # baseline infrastructure
    from paper_2408_13510_b200 import abi
    sd = abi.state_dimension(m)
    return [sd, 64, 64, m + 1], O.ref_agent_params(sd, m + 1, 64, 42)


def sample_plan(cfgname, per):
    """The bounded CPU sample of a config: per policy, `per` replays with
    seeds 1..per and the sweep's arrival rates spread over them.  Returns
    [(policy, [(rate_index, seed), ...])]; replay (rate_index, seed) is the
    engine's replay rate_index * R + seed - 1 on rank 0 (make_workload)."""
    n, R, m, rates, pols, weights, desc = cfg_shape(cfgname)
    step = max(1, len(rates) // per)
    return [(policy, [((pi + k * step) % len(rates), k + 1) for k in range(per)])
            for pi, policy in enumerate(pols)]


def cpu_reference(cfgname, sample_replays, threads, noscan=False):
    """Compiled unmodified reference (oracle/_ref) on host threads over the
    bounded sample of sample_plan: traces from the reference's own generator
    (build_workload, experiment.hpp:291-305, via ref_generate_mixture), the
    agent from its own DqnAgent constructor, replays through its own
    ClusterSim::run_policy.  Nothing of the engine is loaded on this path.
    Returns (decisions/s, decisions, wall s, description, samples) with
    samples = [(policy, rate_index, seed, rs_replay_stats record)].
    noscan: the reference with its reward-only per-tick queue-penalty scan
    (env.hpp:289-298) compiled out (oracle/Makefile, librs_ref_noscan.so)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles as O  # baseline infrastructure
    from paper_2408_13510_b200 import abi  # ctypes structs only (no library load)
    n, R, m, rates, pols, weights, desc = cfg_shape(cfgname)
    lib = O.ref_lib(noscan=noscan)
    per = max(1, sample_replays)  # one replay per host thread, per policy
    ticks = 0
    wall = 0.0
    samples = []
    for policy, picks in sample_plan(cfgname, per):
        traces = [O.ref_generate(seed, n, rates[ri], weights) for ri, seed in picks]
        off = np.arange(per + 1, dtype=np.int64) * n
        cat = lambda f: np.ascontiguousarray(np.concatenate([getattr(t, f) for t in traces]))
        arr, pr, de, tk = cat("arrival"), cat("prompt"), cat("decode"), cat("task")
        ps = np.array([O.ref_lib().ref_mix_seed(seed, 0x9DED) for _, seed in picks], np.uint64)
        cfg = abi.default_config(policy, m)
        keep = None
        if policy == "rl":
            dims, params = ref_agent_for(m)
            keep = abi.set_rl(cfg, dims, params)
        stats = np.zeros(per, abi.STATS_DTYPE)
        w = lib.ref_run_batch(C.byref(cfg), per, off.ctypes.data, arr.ctypes.data,
                              pr.ctypes.data, de.ctypes.data, tk.ctypes.data,
                              ps.ctypes.data, None, threads, stats.ctypes.data)
        del keep
        if w <= 0:
            raise RuntimeError("reference batch failed: " + O.ref_error())
        ticks += int(stats["ticks"].sum())
        wall += w
        samples += [(policy, ri, seed, stats[k]) for k, (ri, seed) in enumerate(picks)]
    what = (f"{per} replays (seeds 1..{per}) per policy x {len(pols)} "
            f"{'policies' if len(pols) > 1 else 'policy'} of the {cfgname} workload")
    return ticks / wall, ticks, wall, what, samples


# rs_replay_stats fields the reference's run_policy + compute_metrics sums
# define without a trajectory (ref_run_batch records none): compared exactly
PARITY_FIELDS = ("decision_hash", "ticks", "routed", "infeasible", "completed", "status",
                 "total_preemptions", "total_tokens", "tbt_count", "clock", "total_e2e_s",
                 "total_ttft_s", "total_tbt_s", "total_router_wait_s", "makespan_s")


def parity_sample(cfgname, samples, cell_stats, pols, R):
    """The engine's own answers for the replays the reference just ran on the
    host, field by field (bitwise for the fp64 sums): the bench checks itself."""
    bad = []
    for policy, ri, seed, want in samples:
        got = cell_stats[pols.index(policy)][ri * R + seed - 1]
        diff = [f for f in PARITY_FIELDS
                if np.asarray(got[f]).tobytes() != np.asarray(want[f]).tobytes()]
        if diff:
            bad.append({"policy": policy, "rate_index": ri, "seed": seed, "fields": diff})
    return {"checked": len(samples), "bit_exact": len(samples) - len(bad),
            "against": "oracle/_ref (compiled unmodified reference, same seeds)",
            "fields": list(PARITY_FIELDS), "mismatches": bad[:8]}


def cpu_port_scan_free(cfgname, sample_replays, threads):
    """The plain-C restatement (oracle/rs_oracle.c: the same tick loop without
    the reference's O(N) per-tick reward scan, env.hpp:289-298 — the work the
    GPU engine does) on host threads over the same bounded sample as
    cpu_reference: the like-for-like CPU figure."""
    from concurrent.futures import ThreadPoolExecutor
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles as O  # baseline infrastructure
    from paper_2408_13510_b200 import abi
    n, R, m, rates, pols, weights, desc = cfg_shape(cfgname)
    per = max(1, sample_replays)
    ticks = 0
    wall = 0.0
    for policy, picks in sample_plan(cfgname, per):
        traces = [O.ref_generate(seed, n, rates[ri], weights) for ri, seed in picks]
        cfg = abi.default_config(policy, m)
        keep = None
        if policy == "rl":
            dims, params = ref_agent_for(m)
            keep = abi.set_rl(cfg, dims, params)
        O.ora_lib()
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:  # ctypes releases the GIL
            res = list(ex.map(lambda k: O.ora_run(cfg, traces[k],
                                                  abi.mix_seed(picks[k][1], 0x9DED)),
                              range(per)))
        wall += time.perf_counter() - t0
        ticks += sum(int(r.stats["ticks"][0]) for r in res)
        del keep
    return ticks / wall, ticks, wall


def config_dict(cfgname, world):
    """The workload description both arms print (same keys, same values)."""
    n, R, m, rates, pols, weights, desc = cfg_shape(cfgname)
    rate_s = (f"{rates[0]:g}" if len(rates) == 1 else f"{rates[0]:g}..{rates[-1]:g} "
              f"({len(rates)} rates)")
    return {"workload": desc, "policy": "+".join(pols), "instances": m,
            "requests_per_replay": n, "replays_per_gpu": R * len(rates) * len(pols),
            "arrival_rate": rate_s, "predictor": "simulated, Table-1 accuracy",
            "l2": f"inputs {(8 + 4 + 4 + 1) * n * R * len(rates) / 1e6:.0f} MB per GPU "
                  f"{'>' if (8 + 4 + 4 + 1) * n * R * len(rates) > 126e6 else '<='} 126 MB L2 "
                  "(no flush between steps)",
            "parallelism": f"replay shards x{world} (weak)"}


def run_reference_impl(args, cfgname):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = min(threads, 64, cfg_shape(cfgname)[1])
    runs = []
    for i in range(args.warmup + args.steps):
        v, ticks, wall, what, _ = cpu_reference(cfgname, sample, threads)
        if i >= args.warmup:
            runs.append((v, wall))
    value = float(np.mean([r[0] for r in runs]))
    config = config_dict(cfgname, args.gpus)
    config["sample_replays"] = f"{what} per step (bounded sample, same seeds every step)"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean([r[1] for r in runs]) * 1e3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference workload generator, oracle/_ref)",
            "config": config,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{what}, on {threads} host threads, per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) on
    this node the way the driver does, and return their exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--replays", type=int, default=0, help="override seeds per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dump-stats", default="",
                    help="rank 0 saves every rank's per-replay stats (the gathered records) "
                         "of the first cell as .npy (tests)")
    args = ap.parse_args()
    if args.replays:
        n, R, m, rate, pol, w, desc = CONFIGS[args.config]
        CONFIGS[args.config] = (n, args.replays, m, rate, pol, w,
                                desc.replace(f"{R:,}", f"{args.replays:,}"))
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.impl == "reference":
        run_reference_impl(args, args.config)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))

    import torch
    import torch.distributed as dist
    from paper_2408_13510_b200 import abi, engine
    from paper_2408_13510_b200 import dist as rdist

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: one rank per GPU")
    if not os.environ.get("RS_BENCH_SAME_DEVICE") and torch.cuda.device_count() < world:
        raise SystemExit(f"--gpus {world}: only {torch.cuda.device_count()} visible GPUs")
    # RS_BENCH_SAME_DEVICE / RS_DIST_BACKEND=gloo exist only to exercise the
    # multi-rank path on a one-GPU box; the real run is one rank per GPU on NCCL.
    if os.environ.get("RS_BENCH_SAME_DEVICE"):
        local = 0
    backend = os.environ.get("RS_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    lib = abi.load_library()
    if lib.rs_device_count() < 1:
        raise RuntimeError("no sm_100 device")
    n, R_seeds, m, rates, pols, weights, desc = cfg_shape(args.config)
    t_gen = time.time()
    tb, pseeds, seeds = make_workload(args.config, rank)
    t_gen = time.time() - t_gen
    N, R = tb.total, tb.num_replays
    dev = torch.device("cuda", local)
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    d_off, d_arr, d_pr, d_de, d_tk = (tt(tb.offsets), tt(tb.arrival), tt(tb.prompt),
                                      tt(tb.decode), tt(tb.task))
    d_ps = tt(pseeds.view(np.int64))
    o_in = torch.empty(N, dtype=torch.int32, device=dev)
    o_ro = torch.empty(N, dtype=torch.float64, device=dev)
    o_fi = torch.empty(N, dtype=torch.float64, device=dev)
    o_co = torch.empty(N, dtype=torch.float64, device=dev)
    o_pe = torch.empty(N, dtype=torch.int32, device=dev)
    o_pb = torch.empty(N, dtype=torch.uint8, device=dev)
    tr = abi.TraceSoA(R, 0, N, d_off.data_ptr(), d_arr.data_ptr(), d_pr.data_ptr(),
                      d_de.data_ptr(), d_tk.data_ptr(), None, d_ps.data_ptr(), None)
    out = abi.ReqOut(o_in.data_ptr(), o_ro.data_ptr(), o_fi.data_ptr(), o_co.data_ptr(),
                     o_pe.data_ptr(), o_pb.data_ptr())

    # one cell per policy: the same traces, the policy's config, its own stats
    keep = []
    cells = []
    ws_max = 0
    for policy in pols:
        cfg = abi.default_config(policy, m)
        if policy == "rl":
            dims, params = agent_for(m)
            d_params = tt(params)
            keep += [abi.set_rl(cfg, dims, params), d_params]  # host copy for the e2e call
            dcfg = abi.BatchCfg.from_buffer_copy(bytes(cfg))
            dcfg.rl_params = C.cast(C.c_void_p(d_params.data_ptr()), C.POINTER(C.c_double))
        else:
            dcfg = abi.BatchCfg.from_buffer_copy(bytes(cfg))
        dcfg.flags |= abi.RS_FLAG_PREDICT_INLINE  # predictor fused into the replay kernel
        wsz = C.c_size_t(0)
        abi.check(lib, lib.rs_workspace_size(C.byref(dcfg), R, N, C.byref(wsz)))
        ws_max = max(ws_max, wsz.value)
        cells.append({"policy": policy, "cfg": cfg, "dcfg": dcfg,
                      "st": torch.zeros(R * 256, dtype=torch.uint8, device=dev)})
    d_ws = torch.empty(ws_max, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    gathered = torch.empty(world * R * 256, dtype=torch.uint8, device=dev) if world > 1 else None

    def step(ev=None):
        # per cell one rs_replay_batch = the validation pre-pass, the replay
        # kernel (predictions drawn at injection) and the per-replay stats
        # kernel, on torch's stream
        for k, c in enumerate(cells):
            if ev is not None:
                ev[k].record(stream)
            abi.check(lib, lib.rs_replay_batch(C.byref(c["dcfg"]), C.byref(tr), C.byref(out),
                                               c["st"].data_ptr(), d_ws.data_ptr(), ws_max, sh))
        if ev is not None:
            ev[len(cells)].record(stream)
        if world > 1:  # final gather of the per-replay statistics (NCCL)
            for c in cells:
                if backend == "nccl":
                    dist.all_gather_into_tensor(gathered, c["st"])
                else:  # gloo gathers host tensors
                    gathered.copy_(rdist.gather_stats(c["st"].cpu(), world))

    # clock sampler first: its start-up must not land in the timed region
    clk = ClockSampler(list(range(world)) if world > 1 else [local]).start()
    # Pre-warm: a fresh box's first seconds of work run ~35% slower (clock /
    # power ramp; measured), so repeat untimed full steps for >= PREWARM_S
    # before the W warm-up steps.  Reported in config.prewarm_s.
    t_pw = time.perf_counter()
    while time.perf_counter() - t_pw < PREWARM_S:
        step()
        torch.cuda.synchronize(dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    cell_stats = [np.frombuffer(c["st"].cpu().numpy().tobytes(), dtype=abi.STATS_DTYPE)
                  for c in cells]
    ticks_local = int(sum(int(st["ticks"].sum()) for st in cell_stats))
    unfinished = int(sum(int((st["status"] != abi.REPLAY_FINISHED).sum()) for st in cell_stats))

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(cells) + 1)]
           for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_win0 = time.time()
    # Launch gate: a ~0.3 s spin on the stream ahead of the start event, so all
    # K steps are enqueued while the GPU is still busy.  Host-side stalls of
    # 50-180 ms inside CUDA API calls on the shared box otherwise land between
    # the start event and the first replay launch (measured: first timed step
    # 164 ms vs 106 ms for the others).  The spin is outside the timed region.
    torch.cuda._sleep(int(GATE_S * 1.965e9))
    start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    stop.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk.mark(t_win0, time.time())
    clk.stop()
    elapsed = start.elapsed_time(stop) / 1e3
    replay_s = sum(e[0].elapsed_time(e[-1]) for e in evs) / 1e3 / args.steps
    step_ms = [round(e[0].elapsed_time(e[-1]), 3) for e in evs]
    cell_ms = [sum(e[k].elapsed_time(e[k + 1]) for e in evs) / args.steps
               for k in range(len(cells))]
    red_dev = dev if backend == "nccl" else "cpu"
    elapsed = rdist.max_over_ranks(elapsed, red_dev)          # slowest rank's device time
    ticks_total = rdist.sum_over_ranks(float(ticks_local), red_dev)
    value = ticks_total * args.steps / elapsed

    # ------------------------------------------------------------ e2e (C ABI)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        h_off, h_arr, h_pr, h_de, h_tk, h_ps = (pin(tb.offsets), pin(tb.arrival), pin(tb.prompt),
                                                pin(tb.decode), pin(tb.task),
                                                pin(pseeds.view(np.int64)))
        hout = [torch.empty(N, dtype=d, pin_memory=True) for d in
                (torch.int32, torch.float64, torch.float64, torch.float64, torch.int32,
                 torch.uint8)]
        h_st = [torch.zeros(R * 256, dtype=torch.uint8, pin_memory=True) for _ in cells]
        htr = abi.TraceSoA(R, 0, N, h_off.data_ptr(), h_arr.data_ptr(), h_pr.data_ptr(),
                           h_de.data_ptr(), h_tk.data_ptr(), None, h_ps.data_ptr(), None)
        hro_full = abi.ReqOut(*[x.data_ptr() for x in hout])
        hro_stats = abi.ReqOut(None, None, None, None, None, None)
        # per cell (one rs_replay_batch_host call each) the inputs go up again
        h2d = len(cells) * (8 * (R + 1) + 8 * N + 4 * N + 4 * N + N + 8 * R)
        for c in cells:
            if c["policy"] == "rl":
                h2d += 8 * abi.mlp_param_count(agent_for(m)[0])
        d2h_stats = 256 * R * len(cells)
        d2h_full = (N * (4 + 8 + 8 + 8 + 4 + 1) + 256 * R) * len(cells)

        def timed_e2e(hro):
            def e2e_step():
                for c, hs in zip(cells, h_st):
                    abi.check(lib, lib.rs_replay_batch_host(C.byref(c["cfg"]), C.byref(htr),
                                                            C.byref(hro), hs.data_ptr(), local))
            e2e_step()  # warm the arena
            # E2E_WINDOWS timed windows of K steps each, the median window
            # reported: a wall-clock window absorbs the shared box's host-side
            # stalls (50-180 ms inside CUDA API calls, measured), which one
            # window of K ~100 ms steps cannot average out
            wins = []
            for _ in range(E2E_WINDOWS):
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                for _ in range(args.steps):
                    e2e_step()
                torch.cuda.synchronize(dev)
                wins.append(rdist.max_over_ranks(time.perf_counter() - t0, red_dev))
            return float(np.median(wins)), wins

        # headline e2e: the reference-facing result of evaluate_policy
        # (experiment.hpp:648-670) is the per-replay statistics, so the D2H
        # per step is the rs_replay_stats records; the variant that also
        # copies every per-request array back is reported beside it
        t_stats, w_stats = timed_e2e(hro_stats)
        t_full, _ = timed_e2e(hro_full)
        e2e = {"value": ticks_total * args.steps / t_stats, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h_stats),
               "ms_per_step": t_stats * 1e3 / args.steps,
               "window_ms_per_step": [round(w * 1e3 / args.steps, 3) for w in w_stats],
               "timing": f"median of {E2E_WINDOWS} wall-clock windows of {args.steps} steps",
               "path": "rs_replay_batch_host (C ABI, pinned host buffers, wall clock)",
               "with_per_request_d2h": {"value": ticks_total * args.steps / t_full,
                                        "d2h_bytes_per_step": int(d2h_full),
                                        "ms_per_step": t_full * 1e3 / args.steps,
                                        "outputs": "every per-request array, copied back in 8 "
                                                   "request-index chunks as the replays "
                                                   "finalise them (streamed outputs)"}}
        for hs, st in zip(h_st, cell_stats):
            h_stats = np.frombuffer(hs.numpy().tobytes(), dtype=abi.STATS_DTYPE)
            if not np.array_equal(h_stats["decision_hash"], st["decision_hash"]):
                raise RuntimeError("e2e path decisions differ from the device path")

    if args.dump_stats:  # every rank's records of the first cell, in rank order
        src = cells[0]["st"] if backend == "nccl" else cells[0]["st"].cpu()
        allst = rdist.gather_stats(src, world) if world > 1 else src
        if rank == 0:
            np.save(args.dump_stats, rdist.stats_view(allst))
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = load_peaks()
    alg_bytes = (REPLAY_BYTES_PER_REQUEST * N + REPLAY_BYTES_PER_REPLAY * R) * len(cells)
    achieved = alg_bytes / replay_s / 1e9
    traffic = None
    prof = ROOT / "profiles" / "r2" / f"ncu_replay_{args.config}.json"
    if not prof.exists():
        prof = ROOT / "profiles" / f"ncu_replay_{args.config}.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            # only when the profiled launch had this exact shape
            if pj.get("algorithmic_bytes_per_launch") == alg_bytes:
                traffic = pj.get("dram_bytes_per_launch")
        except (ValueError, OSError):
            traffic = None
    config = config_dict(args.config, world)
    config["prewarm_s"] = PREWARM_S
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: reference workload generator, seeds 1..{R_seeds * world} "
                f"(rank r takes seeds r*{R_seeds}+1..(r+1)*{R_seeds})",
        "config": config,
        "decisions_per_step": ticks_total, "unfinished_replays": unfinished,
        "gpu_launches": 3 * len(cells) * args.steps * world,  # validate + replay + stats
        "kernel_ms": {"replay_batch": replay_s * 1e3, "per_step": step_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "rs::replay_fast_kernel (+ validate_kernel and stats_kernel, timed together)",
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "peak_source": peak_src},
        # the binding constraint: a replay is a serial tick chain, so the step
        # time is ~ (ticks of the longest replay) x (latency of one tick)
        "tick_chain": {
            "longest_replay_ticks": int(max(int(st["ticks"].max()) for st in cell_stats)),
            "ns_per_tick_longest_replay": replay_s * 1e9 / max(
                1, max(int(st["ticks"].max()) for st in cell_stats)),
            "note": "kernel time / ticks of the longest replay; the HBM roofline "
                    "fraction is small because the work is latency-bound, not bandwidth-bound"},
        "clocks": clk.summary(),
        "trace_gen_s": t_gen,
    }
    rl_cells = [(c, st, ms) for c, st, ms in zip(cells, cell_stats, cell_ms) if c["policy"] == "rl"]
    if rl_cells:
        # Q-network forward (mlp.hpp:54-68) once per decision (RlPolicy::decide
        # runs every tick): 2 FLOP per MAC of the dense (6m+3)-64-64-(m+1) net,
        # issued as separately rounded DMUL + DADD (bit-exact, -fmad=false);
        # peak = the measured DMUL+DADD rate (profiles/fp64_peak.json).
        dims = agent_for(m)[0]
        macs = sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))
        dense = sum(2.0 * macs * float(st["ticks"].sum()) for _, st, _ in rl_cells)
        # executed: the kernels count the multiply-adds their forwards issued
        # (rs_replay_stats.qnet_macs: exact-zero inputs skipped, a repeated
        # state's action reused without a forward)
        flop = sum(2.0 * float(st["qnet_macs"].sum()) for _, st, _ in rl_cells)
        dec = sum(float(st["ticks"].sum()) for _, st, _ in rl_cells)
        sec = sum(ms for _, _, ms in rl_cells) / 1e3
        fp = ROOT / "profiles" / "fp64_peak.json"
        fpeak = json.loads(fp.read_text())["fp64_tflops_mul_add"] if fp.exists() else None
        line["roofline_fp64_qnet"] = {
            "bound": "fp64", "achieved": flop / sec / 1e12, "peak": fpeak, "unit": "TFLOP/s",
            "frac": (flop / sec / 1e12 / fpeak) if fpeak else None,
            "flop_per_decision_executed": flop / max(1.0, dec),
            "flop_per_decision_dense": 2 * macs, "dims": dims,
            "dense_equivalent_tflops": dense / sec / 1e12,
            "note": "EXECUTED FLOPs of the Q-net forwards (DMUL + DADD issued: exact-zero "
                    "inputs skipped, repeated states memoised) over the RL cells' kernel time "
                    "(the whole fused tick, not the forward alone)",
            "peak_source": "measured DMUL+DADD (profiles/fp64_peak.json, tools/fp64_peak.cu)"}
    if len(cells) > 1:
        line["per_policy"] = {c["policy"]: {"decisions": int(st["ticks"].sum()),
                                            "kernel_ms": ms,
                                            "decisions_per_s": int(st["ticks"].sum()) / ms * 1e3}
                              for c, st, ms in zip(cells, cell_stats, cell_ms)}
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = min(threads, 64, R_seeds)
        try:
            cv, cticks, cwall, what, samples = cpu_reference(args.config, sample, threads)
            # the bench checks its own answers: the engine's stats for the
            # replays the reference just ran, compared field by field
            line["parity_sample"] = parity_sample(args.config, samples, cell_stats, list(pols),
                                                  R_seeds)
            if world == 1:  # the reported CPU baseline: rank 0 at N = 1 only
                line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": threads,
                                        "kind": "reference",
                                        "sample": f"{what} on {threads} host threads, "
                                                  f"{cwall:.1f} s wall, {cticks} decisions"}
        except Exception as e:  # baseline is reported, never the target
            line["parity_sample"] = {"checked": 0, "bit_exact": 0, "error": str(e)}
            if world == 1:
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0,
                                        "kind": "reference", "sample": f"unavailable: {e}"}
        if world == 1:
            try:
                # like for like: the same reference with its reward-only
                # per-tick scan (env.hpp:289-298) compiled out, the work the
                # engine does
                pv, pticks, pwall, _, _ = cpu_reference(args.config, sample, threads,
                                                        noscan=True)
                line["cpu_baseline_scan_free"] = {
                    "value": pv, "unit": UNIT, "cores": threads,
                    "kind": "reference (patched: env.hpp:289-298 reward scan compiled out)",
                    "sample": f"same sample, oracle/_ref/librs_ref_noscan.so, "
                              f"{pwall:.1f} s wall, {pticks} decisions"}
            except Exception as e:
                line["cpu_baseline_scan_free"] = {"value": None, "sample": f"unavailable: {e}"}
            try:  # the plain-C restatement of the same scan-free tick loop
                cv2, cticks2, cwall2 = cpu_port_scan_free(args.config, sample, threads)
                line["cpu_baseline_c_port"] = {
                    "value": cv2, "unit": UNIT, "cores": threads, "kind": "port",
                    "sample": f"same sample, oracle/rs_oracle.c (no per-tick reward scan), "
                              f"{cwall2:.1f} s wall, {cticks2} decisions"}
            except Exception as e:
                line["cpu_baseline_c_port"] = {"value": None, "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    del keep
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
