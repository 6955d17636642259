"""bench.py contract on CPU: the reference arm (the CPU oracle) prints one JSON
line on rank 0 and nothing on other ranks (torchrun launches every rank)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(rank):
    env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK=str(rank))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                           "--steps", "1", "--warmup", "3"], capture_output=True, text=True, env=env, timeout=600)


def test_reference_arm_rank0_line():
    r = _run(0)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "updates/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["steps"] == 1 and d["warmup"] == 3


def test_reference_arm_other_ranks_silent():
    r = _run(1)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""
