"""Multi-device paths on the GPU box.

* rs_replay_batch_multi (one process, one shard per device, NCCL all-gather
  of the per-replay statistics) equals one rs_replay_batch_host call over the
  whole batch, bit for bit, on every device this box has (1 on the driver's
  box: the NCCL path still runs, over a one-device communicator).
* bench.py's engine arm with 2 ranks (torchrun) equals the 1-rank run of the
  same seeds: sharded + gathered records identical.  Two ranks share the one
  device here (RS_BENCH_SAME_DEVICE, gloo: NCCL refuses two ranks on one GPU);
  with >= 2 devices the same check runs on NCCL, one rank per GPU.
"""
import ctypes as C
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2408_13510_b200 import abi, engine

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _batch(seeds, n, rate=20.0):
    tb = engine.build_workload(seeds, n, rate)
    ps = np.array([abi.mix_seed(int(s), 0x9DED) for s in seeds], np.uint64)
    return tb, ps


def _call(lib, fn, cfg, tb, ps, *extra):
    N, R = tb.total, tb.num_replays
    tr = abi.TraceSoA(R, 0, N, tb.offsets.ctypes.data, tb.arrival.ctypes.data,
                      tb.prompt.ctypes.data, tb.decode.ctypes.data, tb.task.ctypes.data, None,
                      ps.ctypes.data, None)
    arrs = [np.full(N, 7, d) for d in (np.int32, np.float64, np.float64, np.float64, np.int32,
                                        np.uint8)]
    stats = np.zeros(R, abi.STATS_DTYPE)
    out = abi.ReqOut(*[a.ctypes.data for a in arrs])
    abi.check(lib, fn(C.byref(cfg), C.byref(tr), C.byref(out), stats.ctypes.data, *extra))
    return arrs, stats


@pytest.mark.parametrize("policy,R", [("workload_aware", 24), ("jsq", 7), ("rl", 9)])
def test_multi_device_api_matches_single_call(gpu, policy, R):
    ndev = min(gpu.rs_device_count(), 8)
    tb, ps = _batch(range(1, R + 1), 1500, 30.0)
    cfg = abi.default_config(policy, 4)
    keep = None
    if policy == "rl":
        dims = [abi.state_dimension(4), 64, 64, 5]
        keep = abi.set_rl(cfg, dims, engine.mlp_random_init(dims, 42))
    want_a, want_s = _call(gpu, gpu.rs_replay_batch_host, cfg, tb, ps, 0)
    for nd in sorted({1, ndev}):
        devs = (C.c_int32 * nd)(*range(nd))
        got_a, got_s = _call(gpu, gpu.rs_replay_batch_multi, cfg, tb, ps, devs, nd)
        assert got_s.tobytes() == want_s.tobytes(), nd
        for g, w in zip(got_a, want_a):
            assert g.tobytes() == w.tobytes(), nd
    del keep


def test_multi_device_rejects_duplicates(gpu):
    tb, ps = _batch([1, 2], 100)
    cfg = abi.default_config("jsq", 4)
    devs = (C.c_int32 * 2)(0, 0)
    with pytest.raises(abi.EngineError):
        _call(gpu, gpu.rs_replay_batch_multi, cfg, tb, ps, devs, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(tmp_path, name, world, per_rank, env_extra):
    out = tmp_path / f"{name}.npy"
    env = dict(os.environ, RS_BENCH_PREWARM_S="0", **env_extra)
    args = [str(ROOT / "bench.py"), "--gpus", str(world), "--replays", str(per_rank),
            "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu-baseline",
            "--dump-stats", str(out)]
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port())] + args
    else:
        cmd = [sys.executable] + args
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return np.load(out), r.stdout


def test_bench_two_ranks_equal_one_rank(gpu, tmp_path):
    one, _ = _bench(tmp_path, "one", 1, 64, {})
    if gpu.rs_device_count() >= 2:
        env = {"RS_DIST_BACKEND": "nccl"}
    else:
        env = {"RS_BENCH_SAME_DEVICE": "1", "RS_DIST_BACKEND": "gloo"}
    two, line = _bench(tmp_path, "two", 2, 32, env)
    assert len(one) == len(two) == 64
    assert one.tobytes() == two.tobytes()
    assert '"n_gpus": 2' in line


def test_host_entry_points_reject_non_finite_weights(gpu):
    # the device forward skips exact-zero inputs, which equals the
    # reference's w * 0 only for finite weights
    tb, ps = _batch([1, 2], 200)
    cfg = abi.default_config("rl", 4)
    dims = [abi.state_dimension(4), 64, 64, 5]
    params = engine.mlp_random_init(dims, 42)
    params[17] = np.inf
    keep = abi.set_rl(cfg, dims, params)
    for fn, extra in ((gpu.rs_replay_batch_host, (0,)),
                      (gpu.rs_replay_batch_multi, ((C.c_int32 * 1)(0), 1))):
        with pytest.raises(abi.EngineError) as e:
            _call(gpu, fn, cfg, tb, ps, *extra)
        assert e.value.status == abi.RS_ERR_UNSUPPORTED
    del keep
