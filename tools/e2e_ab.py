#!/usr/bin/env python
"""A/B of the host-buffer entry point rs_replay_batch_host (bench.py's e2e
leg) in ONE process: streamed inputs (chunked H2D overlapping the replay
kernel) vs a full H2D before the kernel, stats-only D2H, interleaved rounds,
wall clock per call.  Also the device-resident kernel time for reference.

    python tools/e2e_ab.py [--config c2] [--rounds 4]
"""
import argparse
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2408_13510_b200 import abi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rounds", type=int, default=4)
    a = ap.parse_args()
    lib = abi.load_library()
    n, R, m, rates, pols, weights, desc = bench.cfg_shape(a.config)
    tb, pseeds, _ = bench.make_workload(a.config, 0)
    N, R = tb.total, tb.num_replays
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
    h = [pin(tb.offsets), pin(tb.arrival), pin(tb.prompt), pin(tb.decode), pin(tb.task),
         pin(pseeds.view(np.int64))]
    tr = abi.TraceSoA(R, 0, N, *[x.data_ptr() for x in h[:5]], None, h[5].data_ptr(), None)
    out = abi.ReqOut(None, None, None, None, None, None)
    st = torch.zeros(R * 256, dtype=torch.uint8, pin_memory=True)
    cfg = abi.default_config(pols[0], m)

    def call(stream_inputs):
        os.environ["RS_STREAM_INPUTS"] = "1" if stream_inputs else "0"
        t0 = time.perf_counter()
        abi.check(lib, lib.rs_replay_batch_host(C.byref(cfg), C.byref(tr), C.byref(out),
                                                st.data_ptr(), 0))
        return (time.perf_counter() - t0) * 1e3

    t0 = time.time()
    while time.time() - t0 < 3.0:
        call(True)
    for r in range(a.rounds):
        s = [call(True) for _ in range(3)]
        f = [call(False) for _ in range(3)]
        print(f"round {r}: streamed {' '.join(f'{x:7.1f}' for x in s)} ms | "
              f"full-H2D {' '.join(f'{x:7.1f}' for x in f)} ms", flush=True)


if __name__ == "__main__":
    main()
