"""bench.py's reference arm on CPU: `--impl reference` needs no GPU (it times
the compiled, unmodified reference on the host cores) and prints ONE JSON
line with the driver's contract keys; under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(extra_env=None, *args):
    env = dict(os.environ)
    env.update(extra_env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                           "--config", "c1", "--steps", "1", "--warmup", "0", *args],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)


def test_reference_arm_prints_one_contract_line(lib):
    p = _run()
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["unit"] == "decisions/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent(lib):
    p = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--gpus", "2")
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.strip() == ""


def test_reference_arm_loads_only_the_reference(lib):
    """The reference arm generates its traces and agent with oracle/_ref and
    replays them there: the engine library is never loaded on that path."""
    code = ("import bench, sys; v = bench.cpu_reference('c4', 1, 1); "
            "maps = open('/proc/self/maps').read(); "
            "print('ENGINE' if 'librs_b200' in maps else 'CLEAN', "
            "'REF' if 'librs_ref' in maps else 'NOREF', len(v[4]))")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.split() == ["CLEAN", "REF", "4"]


def test_reference_arm_config_matches_engine_arm_keys():
    sys.path.insert(0, str(ROOT))
    import bench
    for name in bench.CONFIGS:
        c1, c2 = bench.config_dict(name, 1), bench.config_dict(name, 1)
        assert c1 == c2 and {"workload", "policy", "instances", "requests_per_replay",
                             "replays_per_gpu", "arrival_rate"} <= set(c1)
    plan = bench.sample_plan("c4", 16)
    assert [p for p, _ in plan] == ["round_robin", "jsq", "workload_aware", "rl"]
    for _, picks in plan:  # every rate of the sweep is sampled, seeds 1..16
        assert sorted(ri for ri, _ in picks) == list(range(16))
        assert [s for _, s in picks] == list(range(1, 17))


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """--gpus N outside torchrun launches N ranks itself (never a silent 1-GPU line)."""
    sys.path.insert(0, str(ROOT))
    import bench
    seen = {}

    def fake_run(cmd, *a, **k):
        seen["cmd"] = cmd
        return subprocess.CompletedProcess(cmd, 0)

    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])

    class A:
        gpus = 4
    assert bench.relaunch_under_torchrun(A()) == 0
    cmd = seen["cmd"]
    assert "torch.distributed.run" in cmd and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
