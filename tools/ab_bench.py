#!/usr/bin/env python
"""A/B timing of replay-path variants in ONE process (same box, same inputs,
interleaved), to separate real effects from box-to-box / ramp-up noise.

    python tools/ab_bench.py [--config c2] [--rounds 3]

Variants: fused predictor (RS_FLAG_PREDICT_INLINE) vs separate predictor
kernel + replay.  Prints the CUDA-event time of each, per round.
"""
import argparse
import ctypes as C
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
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--replays", type=int, default=0)
    a = ap.parse_args()
    if a.replays:
        n, R, m, rate, pol, w, desc = bench.CONFIGS[a.config]
        bench.CONFIGS[a.config] = (n, a.replays, m, rate, pol, w, desc)
    lib = abi.load_library()
    n, R, m, rate, policy, weights, desc = bench.CONFIGS[a.config]
    tb, pseeds, _ = bench.make_workload(a.config, 0)
    dev = torch.device("cuda", 0)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    N = tb.total
    bufs = [t(tb.offsets), t(tb.arrival), t(tb.prompt), t(tb.decode), t(tb.task),
            t(pseeds.view(np.int64))]
    tr = abi.TraceSoA(R, 0, N, *[b.data_ptr() for b in bufs[:5]], None, bufs[5].data_ptr(), None)
    outs = [torch.empty(N, dtype=d, device=dev) for d in
            (torch.int32, torch.float64, torch.float64, torch.float64, torch.int32, torch.uint8)]
    out = abi.ReqOut(*[o.data_ptr() for o in outs])
    st = torch.zeros(R * 256, dtype=torch.uint8, device=dev)
    cfg = abi.default_config(policy, m)
    keep = None
    if policy == "rl":
        dims, params = bench.agent_for(m)
        dp = t(params)
        keep = abi.set_rl(cfg, dims, params)
        cfg = abi.BatchCfg.from_buffer_copy(bytes(cfg))
        cfg.rl_params = C.cast(C.c_void_p(dp.data_ptr()), C.POINTER(C.c_double))
    ws = C.c_size_t(0)
    abi.check(lib, lib.rs_workspace_size(C.byref(cfg), R, N, C.byref(ws)))
    wsb = torch.empty(ws.value, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)
    fused = abi.BatchCfg.from_buffer_copy(bytes(cfg))
    fused.flags |= abi.RS_FLAG_PREDICT_INLINE

    def run(c, separate):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        if separate:
            abi.check(lib, lib.rs_predict_buckets(C.byref(c), C.byref(tr), outs[5].data_ptr(),
                                                  s.cuda_stream))
        abi.check(lib, lib.rs_replay_batch(C.byref(c), C.byref(tr), C.byref(out), st.data_ptr(),
                                           wsb.data_ptr(), ws.value, s.cuda_stream))
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    t0 = time.time()
    while time.time() - t0 < 2.0:
        run(fused, False)
    for r in range(a.rounds):
        print(f"round {r}: fused {run(fused, False):8.2f} ms   separate {run(cfg, True):8.2f} ms",
              flush=True)
    del keep


if __name__ == "__main__":
    main()
