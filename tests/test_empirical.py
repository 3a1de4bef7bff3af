"""Empirical decode-length predictor: the host-side fit
(rs_empirical_fit / rs_empirical_fit_trace, EmpiricalPredictor::fit +
predict, predictor.hpp:119-158) against the reference's own EmpiricalPredictor
(oracle/_ref), and the device lookup in a full replay against the oracle fed
with the same per-request buckets."""
import ctypes as C

import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine


@pytest.mark.skipif(not O.have_ref(), reason="compiled reference unavailable")
@pytest.mark.parametrize("seed,edges", [(1, None), (7, None), (42, (0, 100, 300, 900, 2000)),
                                        (3, (0, 500))])
def test_empirical_fit_matches_reference(lib, seed, edges):
    cfg = abi.default_config("jsq", 4)
    if edges:
        cfg.n_predictor_edges = len(edges)
        for i, e in enumerate(edges):
            cfg.predictor_edges[i] = e
    abi.check(lib, lib.rs_empirical_fit(C.byref(cfg), seed, 20000))
    assert cfg.predictor_mode == abi.PRED_EMPIRICAL
    got = np.array([[cfg.empirical_table[t][b] for b in range(cfg.n_band_edges)]
                    for t in range(abi.RS_NUM_TASKS)])
    want = O.ref_empirical_table(cfg, seed)[:, :cfg.n_band_edges]
    assert np.array_equal(got, want)


def test_empirical_fit_fallbacks(lib):
    """Unseen cells fall back to the task marginal, unseen tasks to the global
    marginal; ties resolve to the lowest bucket (predictor.hpp:146-170)."""
    cfg = abi.default_config("jsq", 4)
    # task 0: prompt 10 (band 0) decodes 300, 300 (bucket 1); prompt 200 (band 3) decode 50
    # task 1: one request, decode 5000 (bucket 3); tasks 2-4 unseen
    prompt = np.array([10, 10, 200, 40], np.int32)
    decode = np.array([300, 300, 50, 4096], np.int32)
    task = np.array([0, 0, 0, 1], np.uint8)
    abi.check(lib, lib.rs_empirical_fit_trace(C.byref(cfg), 4, prompt.ctypes.data,
                                              decode.ctypes.data, task.ctypes.data))
    tab = np.array([[cfg.empirical_table[t][b] for b in range(7)] for t in range(5)])
    assert tab[0, 0] == 1 and tab[0, 3] == 0      # seen cells
    assert tab[0, 5] == 1                         # task-0 marginal {0:1, 1:2}
    assert tab[1, 0] == 3                         # task-1 marginal
    assert tab[2, 0] == 1                         # global {0:1, 1:2, 3:1}


@pytest.mark.gpu
def test_gpu_empirical_replay_matches_oracle(gpu):
    """A replay batch in EMPIRICAL mode (device table lookup at injection)
    equals the oracle run with the same buckets given per request."""
    cfg = abi.default_config("workload_aware", 4)
    abi.check(gpu, gpu.rs_empirical_fit(C.byref(cfg), 5, 20000))
    seeds = [1, 2, 3]
    tb = engine.build_workload(seeds, 400, 25.0)
    ps = np.array([abi.mix_seed(s, 0x9DED) for s in seeds], np.uint64)
    N, R = tb.total, tb.num_replays
    tr = abi.TraceSoA(R, 0, N, tb.offsets.ctypes.data, tb.arrival.ctypes.data,
                      tb.prompt.ctypes.data, tb.decode.ctypes.data, tb.task.ctypes.data, None,
                      ps.ctypes.data, None)
    arrs = [np.empty(N, np.int32), np.empty(N, np.float64), np.empty(N, np.float64),
            np.empty(N, np.float64), np.empty(N, np.int32), np.empty(N, np.uint8)]
    st = np.zeros(R, abi.STATS_DTYPE)
    abi.check(gpu, gpu.rs_replay_batch_host(C.byref(cfg), C.byref(tr),
                                            C.byref(abi.ReqOut(*[a.ctypes.data for a in arrs])),
                                            st.ctypes.data, 0))
    bands = np.array([cfg.band_edges[b] for b in range(cfg.n_band_edges)])
    table = np.array([[cfg.empirical_table[t][b] for b in range(8)] for t in range(5)])
    given_cfg = abi.BatchCfg.from_buffer_copy(bytes(cfg))
    given_cfg.predictor_mode = abi.PRED_GIVEN
    for r in range(R):
        s = tb.replay(r)
        band = np.searchsorted(bands, tb.prompt[s], side="right") - 1
        given = table[tb.task[s], band].astype(np.uint8)
        trr = O.Trace(tb.arrival[s], tb.prompt[s], tb.decode[s], tb.task[s])
        want = O.ora_run(given_cfg, trr, int(ps[r]), given=given)
        got = O.ReplayResult(*[a[s] for a in arrs], st[r:r + 1])
        assert O.compare(got, want) == [], r
