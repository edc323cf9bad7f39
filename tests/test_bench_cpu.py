"""bench.py's launch contract on a CPU box: --gpus N never silently measures fewer GPUs."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_gpus_without_enough_devices_fails_loudly():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert "--gpus 2 requested" in r.stderr


def test_spawn_builds_one_rank_per_gpu(monkeypatch):
    seen = {}
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])

    class FakeCuda:
        @staticmethod
        def device_count():
            return 8

    import torch
    monkeypatch.setattr(torch, "cuda", FakeCuda)
    monkeypatch.setattr(os, "execv", lambda exe, cmd: seen.update(cmd=cmd))
    args = type("A", (), {"gpus": 4})()
    bench.spawn_ranks(args)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_world_size_mismatch_is_refused(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "1")
    args = type("A", (), {"gpus": 2})()
    with pytest.raises(SystemExit, match="WORLD_SIZE=1"):
        bench.run_ours(args, bench.CONFIGS["c1"])


def test_reference_arm_loads_no_product_code():
    """The reference arm generates A with the oracle and never imports the product package."""
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--config','c1','--steps','1','--warmup','0'];"
            "import bench; bench.main(); print('LOADED', 'paper_2501_15964_b200' in sys.modules)")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "LOADED False" in r.stdout
    import json
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["host_cores"] >= 1
