"""rs_replay_batch_host with PINNED host buffers: the path that captures a
repeated call into a CUDA graph and replays it (a replayed graph
must not read watermark values a later call of another shape rewrote).

Sequence A, A (captured), B (direct, other shape: rewrites the direct-call
watermarks), A (graph replay), B, B (captured), A, B — every result equal
to the first run of its shape and to the oracle."""
import ctypes as C

import numpy as np
import pytest

import oracles as O
from paper_2408_13510_b200 import abi, engine

pytestmark = pytest.mark.gpu


class Pinned:
    """numpy arrays over rs_host_alloc (page-locked) memory."""

    def __init__(self, lib):
        self.lib = lib
        self.ptrs = []

    def array(self, n, dtype):
        dtype = np.dtype(dtype)
        p = self.lib.rs_host_alloc(max(1, n * dtype.itemsize))
        assert p
        self.ptrs.append(p)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)),
                                     shape=(max(1, n * dtype.itemsize),)).view(dtype)[:n]

    def free(self):
        for p in self.ptrs:
            self.lib.rs_host_free(C.c_void_p(p))
        self.ptrs = []


class Call:
    """One pinned-buffer call shape (inputs + outputs live across calls)."""

    def __init__(self, lib, pin, seeds, n):
        tb = engine.build_workload(seeds, n, 20.0)
        self.tb = tb
        self.pseeds = [abi.mix_seed(int(s), 0x9DED) for s in seeds]
        N, R = tb.total, tb.num_replays
        self.R = R

        def put(a):
            h = pin.array(a.size, a.dtype)
            h[:] = a
            return h
        self.h_in = [put(tb.offsets), put(tb.arrival), put(tb.prompt), put(tb.decode),
                     put(tb.task),
                     put(np.array(self.pseeds, np.uint64))]
        self.outs = [pin.array(N, d) for d in (np.int32, np.float64, np.float64, np.float64,
                                                np.int32, np.uint8)]
        self.stats = pin.array(R, abi.STATS_DTYPE)
        o, a, p, d, t, ps = self.h_in
        self.tr = abi.TraceSoA(R, 0, N, o.ctypes.data, a.ctypes.data, p.ctypes.data,
                               d.ctypes.data, t.ctypes.data, None, ps.ctypes.data, None)
        self.out = abi.ReqOut(*[x.ctypes.data for x in self.outs])
        self.cfg = abi.default_config("workload_aware", 4)

    def run(self, lib):
        for x in self.outs:
            x[:] = 0
        self.stats[:] = np.zeros(1, abi.STATS_DTYPE)
        abi.check(lib, lib.rs_replay_batch_host(C.byref(self.cfg), C.byref(self.tr),
                                                C.byref(self.out), self.stats.ctypes.data, 0))
        return [x.copy() for x in self.outs], self.stats.copy()


def test_graph_replay_after_other_shape(gpu, monkeypatch):
    monkeypatch.setenv("RS_STREAM_INPUTS", "1")  # stream (watermarked) even small inputs
    for k in ("RS_NO_GRAPH", "RS_DEBUG_TIMING", "RS_FORCE_GENERAL", "RS_RUN_SMEM"):
        monkeypatch.delenv(k, raising=False)
    pin = Pinned(gpu)
    try:
        A = Call(gpu, pin, [11, 12, 13], 3000)  # chunks 256 / 2048 / 3000
        B = Call(gpu, pin, [21, 22], 2500)      # chunks 256 / 2048 / 2500: same count
        first = {}
        for name in ("A", "A", "B", "A", "B", "B", "A", "B"):
            c = A if name == "A" else B
            arrs, st = c.run(gpu)
            assert np.all(st["status"] == abi.REPLAY_FINISHED), name
            if name not in first:
                first[name] = (arrs, st)
                for r in range(c.R):
                    s = c.tb.replay(r)
                    tr = O.Trace(c.tb.arrival[s], c.tb.prompt[s], c.tb.decode[s], c.tb.task[s])
                    want = O.ora_run(c.cfg, tr, c.pseeds[r])
                    got = O.ReplayResult(*[a[s] for a in arrs], st[r:r + 1])
                    assert O.compare(got, want) == [], (name, r)
            else:
                a0, s0 = first[name]
                assert st.tobytes() == s0.tobytes(), name
                for x, y in zip(arrs, a0):
                    assert x.tobytes() == y.tobytes(), name
    finally:
        pin.free()
