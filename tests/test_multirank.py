"""The N>1 path on CPU (gloo, world size 2): replay sharding by seed and the
final all-gather of per-replay statistics reproduce a single-rank run.  The
per-replay work here is done by the CPU oracle standing in for the device
(the point is the host-side sharding / gather / max-over-ranks logic)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracles as O
from paper_2408_13510_b200 import abi, dist as rdist, engine


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _replay_stats(seeds, n=300, m=3, policy="jsq"):
    tb = engine.build_workload(seeds, n, 25.0)
    cfg = abi.default_config(policy, m)
    recs = np.zeros(len(seeds), abi.STATS_DTYPE)
    for r, s in enumerate(seeds):
        sl = tb.replay(r)
        tr = O.Trace(tb.arrival[sl], tb.prompt[sl], tb.decode[sl], tb.task[sl])
        recs[r] = O.ora_run(cfg, tr, abi.mix_seed(int(s), 0x9DED)).stats[0]
    return recs


def _worker(rank, world, port, per_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seeds = rdist.shard_seeds(per_rank, rank)
        recs = _replay_stats(seeds)
        u8 = torch.from_numpy(recs.view(np.uint8).copy())
        gathered = rdist.gather_stats(u8, world)
        slowest = rdist.max_over_ranks(float(rank + 1), "cpu")
        total = rdist.sum_over_ranks(float(recs["ticks"].sum()), "cpu")
        if rank == 0:
            q.put((gathered.numpy().tobytes(), slowest, total))
    finally:
        dist.destroy_process_group()


def test_weak_scaling_shards_and_gather_match_single_rank(lib):
    world, per_rank = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, slowest, total = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    gathered = np.frombuffer(got, dtype=abi.STATS_DTYPE)
    single = _replay_stats(np.arange(1, world * per_rank + 1, dtype=np.uint64))
    assert gathered.tobytes() == single.tobytes()   # rank-ordered, bit-identical records
    assert slowest == 2.0                            # max over ranks
    assert total == float(single["ticks"].sum())     # decisions of the whole job


def test_seed_partitions_cover_exactly_once():
    for world in (1, 2, 4, 8):
        w = [rdist.shard_seeds(5, r) for r in range(world)]
        assert np.array_equal(np.concatenate(w), np.arange(1, 5 * world + 1))
        s = [rdist.split_seeds(np.arange(1, 1025), r, world) for r in range(world)]
        assert np.array_equal(np.concatenate(s), np.arange(1, 1025))
        assert max(len(x) for x in s) - min(len(x) for x in s) <= 1
