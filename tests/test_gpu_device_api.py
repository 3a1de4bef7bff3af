"""Device-buffer entry points (rs_predict_buckets, rs_replay_batch on a caller
stream) with torch-allocated device memory: the standalone predictor kernel
against the oracle, and the separate-predictor and fused-predictor
(RS_FLAG_PREDICT_INLINE) replay paths against each other and the oracle."""
import ctypes as C

import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine

pytestmark = pytest.mark.gpu


def _dev_batch(torch, tb, pseeds, given=None):
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    bufs = dict(off=t(tb.offsets), arr=t(tb.arrival), pr=t(tb.prompt), de=t(tb.decode),
                tk=t(tb.task), ps=t(np.asarray(pseeds, np.uint64).view(np.int64)))
    if given is not None:
        bufs["gv"] = t(given)
    tr = abi.TraceSoA(tb.num_replays, 0, tb.total, bufs["off"].data_ptr(),
                      bufs["arr"].data_ptr(), bufs["pr"].data_ptr(), bufs["de"].data_ptr(),
                      bufs["tk"].data_ptr(), bufs["gv"].data_ptr() if given is not None else None,
                      bufs["ps"].data_ptr(), None)
    return bufs, tr


def _replay(torch, lib, cfg, tr, N, R, separate_predict):
    dev = torch.device("cuda", 0)
    outs = [torch.empty(N, dtype=d, device=dev) for d in
            (torch.int32, torch.float64, torch.float64, torch.float64, torch.int32, torch.uint8)]
    st = torch.zeros(R * 256, dtype=torch.uint8, device=dev)
    ro = abi.ReqOut(*[o.data_ptr() for o in outs])
    ws = C.c_size_t(0)
    abi.check(lib, lib.rs_workspace_size(C.byref(cfg), R, N, C.byref(ws)))
    wsb = torch.empty(ws.value, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    c = abi.BatchCfg.from_buffer_copy(bytes(cfg))
    if separate_predict:
        abi.check(lib, lib.rs_predict_buckets(C.byref(c), C.byref(tr), outs[5].data_ptr(), s))
    else:
        c.flags |= abi.RS_FLAG_PREDICT_INLINE
    abi.check(lib, lib.rs_replay_batch(C.byref(c), C.byref(tr), C.byref(ro), st.data_ptr(),
                                       wsb.data_ptr(), ws.value, s))
    torch.cuda.synchronize()
    host = [o.cpu().numpy() for o in outs]
    stats = np.frombuffer(st.cpu().numpy().tobytes(), dtype=abi.STATS_DTYPE)
    return host, stats


@pytest.mark.parametrize("mode", ["simulated", "given", "empirical"])
def test_predict_kernel_matches_oracle(gpu, mode):
    import torch
    seeds = list(range(1, 9))
    tb = engine.build_workload(seeds, 1500, 20.0)
    cfg = abi.default_config("jsq", 4)
    given = None
    if mode == "given":
        cfg.predictor_mode = abi.PRED_GIVEN
        given = np.random.default_rng(1).integers(0, 4, tb.total).astype(np.uint8)
    elif mode == "empirical":
        cfg.predictor_mode = abi.PRED_EMPIRICAL
        tab = np.random.default_rng(2).integers(0, 4, (5, 8)).astype(np.uint8)
        for t in range(5):
            for b in range(8):
                cfg.empirical_table[t][b] = int(tab[t, b])
    ps = [abi.mix_seed(s, 0x9DED) for s in seeds]
    bufs, tr = _dev_batch(torch, tb, ps, given)
    out = torch.empty(tb.total, dtype=torch.uint8, device="cuda")
    abi.check(gpu, gpu.rs_predict_buckets(C.byref(cfg), C.byref(tr), out.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
    got = out.cpu().numpy()
    g = np.zeros(max(tb.total, 1), np.uint8) if given is None else given
    for r in range(tb.num_replays):
        sl = tb.replay(r)
        want = np.empty(sl.stop - sl.start, np.uint8)
        assert O.ora_lib().ora_predict_buckets(C.byref(cfg), want.shape[0],
                                               tb.prompt[sl].ctypes.data,
                                               tb.decode[sl].ctypes.data, tb.task[sl].ctypes.data,
                                               g[sl].ctypes.data, ps[r], want.ctypes.data) == 0
        assert np.array_equal(got[sl], want), r


@pytest.mark.parametrize("pol", ["workload_aware", "min_min", "round_robin"])
def test_fused_and_separate_predictor_paths_agree(gpu, pol):
    import torch
    seeds = list(range(20, 36))
    tb = engine.build_workload(seeds, 1200, 25.0)
    ps = [abi.mix_seed(s, 0x9DED) for s in seeds]
    bufs, tr = _dev_batch(torch, tb, ps)
    cfg = abi.default_config(pol, 4)
    a, sa = _replay(torch, gpu, cfg, tr, tb.total, tb.num_replays, True)
    b, sb = _replay(torch, gpu, cfg, tr, tb.total, tb.num_replays, False)
    for x, y in zip(a[:5], b[:5]):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))
    assert sa.tobytes() == sb.tobytes()
    for r in range(tb.num_replays):  # and both equal the oracle
        sl = tb.replay(r)
        tr1 = O.Trace(tb.arrival[sl], tb.prompt[sl], tb.decode[sl], tb.task[sl])
        want = O.ora_run(cfg, tr1, ps[r])
        got = O.ReplayResult(b[0][sl], b[1][sl], b[2][sl], b[3][sl], b[4][sl], b[5][sl],
                             sb[r:r + 1])
        got.predicted = np.where(np.arange(sl.stop - sl.start) < sb[r]["injected"],
                                 got.predicted, 255).astype(np.uint8)
        assert O.compare(got, want) == [], r


@pytest.mark.parametrize("streamed", [0, 1])
def test_host_entry_graph_replay_matches_oracle(gpu, monkeypatch, streamed):
    """rs_replay_batch_host with PINNED host buffers: the first call runs
    directly, the second identical call is captured into a CUDA graph, later
    calls replay it.  Every call's per-request outputs equal the oracle's,
    with and without streamed input copies; fresh inputs in the same pinned
    buffers flow through the replayed graph."""
    import torch
    monkeypatch.setenv("RS_STREAM_INPUTS", "1" if streamed else "0")
    lib = gpu
    R, n = 6, 400
    cfg = abi.default_config("workload_aware", 4)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    outs = [torch.empty(R * n, dtype=d, pin_memory=True) for d in
            (torch.int32, torch.float64, torch.float64, torch.float64, torch.int32, torch.uint8)]
    stats = torch.zeros(R * 256, dtype=torch.uint8, pin_memory=True)
    tb = engine.build_workload(range(1, R + 1), n, 30.0)
    h = [pin(tb.offsets), pin(tb.arrival), pin(tb.prompt), pin(tb.decode), pin(tb.task)]
    ps = pin(np.array([abi.mix_seed(s, 0x9DED) for s in range(1, R + 1)], np.uint64).view(np.int64))
    tr = abi.TraceSoA(R, 0, R * n, *[x.data_ptr() for x in h], None, ps.data_ptr(), None)
    ro = abi.ReqOut(*[o.data_ptr() for o in outs])
    for call in range(4):
        if call == 3:  # new trace contents in the same buffers
            tb = engine.build_workload(range(11, 11 + R), n, 30.0)
            for dst, src in zip(h[1:], (tb.arrival, tb.prompt, tb.decode, tb.task)):
                dst.copy_(torch.from_numpy(src))
        abi.check(lib, lib.rs_replay_batch_host(C.byref(cfg), C.byref(tr), C.byref(ro),
                                                stats.data_ptr(), 0))
        st = np.frombuffer(stats.numpy().tobytes(), dtype=abi.STATS_DTYPE)
        arrs = [o.numpy() for o in outs]
        for r in range(R):
            s = slice(r * n, (r + 1) * n)
            trr = O.Trace(tb.arrival[s], tb.prompt[s], tb.decode[s], tb.task[s])
            want = O.ora_run(cfg, trr, int(ps.numpy().view(np.uint64)[r]))
            got = O.ReplayResult(*[a[s] for a in arrs], st[r:r + 1])
            assert O.compare(got, want) == [], (call, r)


@pytest.mark.parametrize("mode", ["given", "empirical"])
def test_fused_predictor_modes_match_separate_kernel(gpu, mode):
    """The at-injection predictor in GIVEN and EMPIRICAL mode against the
    standalone predict kernel (itself checked against the oracle above):
    identical buckets and identical replays."""
    import torch
    seeds = list(range(40, 52))
    tb = engine.build_workload(seeds, 900, 25.0)
    ps = [abi.mix_seed(s, 0x9DED) for s in seeds]
    cfg = abi.default_config("workload_aware", 4)
    given = None
    if mode == "given":
        cfg.predictor_mode = abi.PRED_GIVEN
        given = np.random.default_rng(3).integers(0, 4, tb.total).astype(np.uint8)
    else:
        abi.check(gpu, gpu.rs_empirical_fit(C.byref(cfg), 9, 20000))
    bufs, tr = _dev_batch(torch, tb, ps, given)
    a, sa = _replay(torch, gpu, cfg, tr, tb.total, tb.num_replays, True)
    b, sb = _replay(torch, gpu, cfg, tr, tb.total, tb.num_replays, False)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))
    assert sa.tobytes() == sb.tobytes()
