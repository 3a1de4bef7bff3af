"""The C++ host mirror (include/routesim_b200.hpp) over the C ABI.

CPU: it compiles against rs_abi.h and links librs_b200.so, and without a
device it fails loudly (no CPU fallback).  GPU: the reference's golden run
(test_harness.cpp:212-231) through BatchSim reproduces mini_summary.json."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden" / "mini_summary.json"


@pytest.fixture(scope="module")
def exe(lib, tmp_path_factory):
    out = tmp_path_factory.mktemp("cpp") / "golden_run"
    libdir = ROOT / "paper_2408_13510_b200" / "_lib"
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "golden_run.cpp"), "-o", str(out),
                    f"-L{libdir}", "-lrs_b200", f"-Wl,-rpath,{libdir}"], check=True)
    return out


def test_cpp_host_builds_and_refuses_without_device(exe, lib):
    if lib.rs_device_count() > 0:
        pytest.skip("a device is present")
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode != 0
    assert "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_cpp_host_golden_run(exe, gpu):
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    # (NCCL may print its version line first: run_policy_multi initialises it)
    got = json.loads(r.stdout.strip().splitlines()[-1])
    want = json.loads(GOLDEN.read_text())
    assert got["completed"] == want["completed"]
    assert got["total_tokens"] == want["total_tokens"]
    assert got["total_e2e_s"] == want["total_e2e_s"]
    assert got["makespan_s"] == want["makespan_s"]
    assert got["total_ttft_s"] / got["completed"] == want["ttft_s"]["mean"]


@pytest.mark.gpu
def test_cpp_host_report_and_dqn(exe, gpu, tmp_path):
    """BatchSim::run_trajectory + emit_report (C++ mirror) write the reference's
    golden summary.json byte for byte; DqnTrainer::update runs."""
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert (tmp_path / "summary.json").read_bytes() == GOLDEN.read_bytes()
    assert (tmp_path / "timeseries.csv").read_text().startswith(
        "tick,time_s,action,reward,router_queue,inst0_waiting")
