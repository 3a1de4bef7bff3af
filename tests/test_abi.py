"""The C-ABI boundary (CPU): the library loads, exports every symbol the
header declares, the ctypes mirror matches the C layout, config validation
mirrors ClusterConfig::validate (env.hpp:133-146), and compute entry points
refuse to run without a device (no CPU fallback)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2408_13510_b200 import abi

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "rs_abi.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(abi.EXPORTED_SYMBOLS)


def test_abi_version(lib):
    assert lib.rs_abi_version() == abi.RS_ABI_VERSION


STRUCTS = {
    "rs_batch_cfg": abi.BatchCfg,
    "rs_trace_soa": abi.TraceSoA,
    "rs_req_out": abi.ReqOut,
    "rs_replay_stats": abi.ReplayStats,
    "rs_profile": abi.Profile,
    "rs_impact": abi.Impact,
    "rs_trajectory": abi.Trajectory,
    "rs_dqn_batch": abi.DqnBatch,
    "rs_dqn_state": abi.DqnState,
}


def test_struct_layout_matches_c(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, cls in STRUCTS.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(src)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.splitlines())
    for cname, cls in STRUCTS.items():
        assert int(got[cname]) == C.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, f"{cname}.{f}"
    assert abi.STATS_DTYPE.itemsize == C.sizeof(abi.ReplayStats)
    for f, _ in abi.ReplayStats._fields_:
        assert abi.STATS_DTYPE.fields[f][1] == getattr(abi.ReplayStats, f).offset, f


def test_default_config_matches_library(lib):
    c = abi.BatchCfg()
    assert lib.rs_default_config(C.byref(c)) == abi.RS_OK
    py = abi.default_config("round_robin", 4)
    assert bytes(c) == bytes(py)
    assert lib.rs_validate_config(C.byref(c)) == abi.RS_OK


@pytest.mark.parametrize("mutate,code", [
    (lambda c: setattr(c, "num_instances", 0), abi.RS_ERR_INVALID_ARGUMENT),
    (lambda c: setattr(c, "delta_t", 0.0), abi.RS_ERR_INVALID_ARGUMENT),
    (lambda c: setattr(c, "kv_capacity_tokens", 0), abi.RS_ERR_INVALID_ARGUMENT),
    (lambda c: setattr(c, "max_batch_size", 0), abi.RS_ERR_INVALID_ARGUMENT),
    (lambda c: setattr(c, "policy", 99), abi.RS_ERR_INVALID_ARGUMENT),
    (lambda c: setattr(c.profile, "decode_time_per_token", 1.0), abi.RS_ERR_INVALID_ARGUMENT),
    (lambda c: setattr(c.impact, "alpha", 1.5), abi.RS_ERR_INVALID_ARGUMENT),
    (lambda c: setattr(c.impact, "prompt_exponent", 3), abi.RS_ERR_INVALID_ARGUMENT),
    (lambda c: c.predictor_edges.__setitem__(1, 0), abi.RS_ERR_INVALID_ARGUMENT),
    (lambda c: setattr(c, "kv_capacity_tokens", 1 << 31), abi.RS_ERR_UNSUPPORTED),
    (lambda c: setattr(c, "num_instances", 129), abi.RS_ERR_UNSUPPORTED),
    (lambda c: (setattr(c, "kv_capacity_tokens", 1 << 20), setattr(c, "max_batch_size", 512)),
     abi.RS_ERR_UNSUPPORTED),
])
def test_validation_mirrors_reference(lib, mutate, code):
    c = abi.default_config("jsq", 4)
    mutate(c)
    assert lib.rs_validate_config(C.byref(c)) == code
    assert abi.last_error(lib)


def test_rl_config_validation(lib):
    c = abi.default_config("rl", 4)
    assert lib.rs_validate_config(C.byref(c)) == abi.RS_ERR_INVALID_ARGUMENT  # no agent
    dims = [27, 64, 64, 5]
    p = np.zeros(abi.mlp_param_count(dims))
    keep = abi.set_rl(c, dims, p)
    assert lib.rs_validate_config(C.byref(c)) == abi.RS_OK
    c.rl_dims[0] = 26  # != state_dimension(4)
    assert lib.rs_validate_config(C.byref(c)) == abi.RS_ERR_INVALID_ARGUMENT
    del keep


def test_mix_seed_and_cutoff(lib):
    for s, k in [(1, 0xB00C), (777, 0x9DED), (2**63 + 5, 3)]:
        assert lib.rs_mix_seed(s, k) == abi.mix_seed(s, k)
    c = abi.default_config()
    assert lib.rs_heavy_decode_cutoff(C.byref(c.profile), C.byref(c.thresholds)) == 300


def test_no_cpu_fallback_without_device(lib):
    if lib.rs_device_count() > 0:
        pytest.skip("a device is present")
    from paper_2408_13510_b200 import engine
    tb = engine.TraceBatch.from_traces([])
    tb = engine.TraceBatch(np.array([0, 1], np.int64), np.array([0.0]), np.array([5], np.int32),
                           np.array([5], np.int32), np.array([1], np.uint8))
    sim = engine.BatchSim(engine.ClusterConfig(), tb, [1])
    with pytest.raises(abi.EngineError) as e:
        sim.run_policy("jsq")
    assert e.value.status == abi.RS_ERR_NO_DEVICE


def test_unknown_policy_name():
    from paper_2408_13510_b200 import engine
    with pytest.raises(ValueError, match="unknown routing policy"):
        engine.make_policy("shortest_job_first")
