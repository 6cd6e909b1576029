"""bench.py's driver contract on CPU: the reference arm (`--impl reference`)
runs the compiled reference (or the oracle port) on the host and prints ONE
JSON line with the keys the driver reads; non-zero ranks print nothing."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None):
    e = dict(os.environ, **(env or {}))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=e)
    assert r.returncode == 0, r.stderr
    return [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    lines = run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--n", "3000",
                 "--batch", "512"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_other_ranks_silent():
    assert run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--n", "1000"],
               env={"RANK": "1", "WORLD_SIZE": "2"}) == []


def test_reference_arm_same_config_as_ours():
    """The reference arm reports the same config dict our arm does (records,
    global batch, lr), and --gpus N without a launcher stands for N ranks."""
    lines = run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                 "--n", "3000", "--batch", "256"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    import bench
    import argparse
    a = argparse.Namespace(n=3000, batch=256, lr=0.01, dp="fused")
    assert d["config"] == bench.workload_config(a, 2)
    assert d["n_gpus"] == 2 and d["cpu_baseline"]["host"]["nproc"] >= 1


def test_gpus_mismatch_fails_loudly():
    e = dict(os.environ, RANK="0", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=120, env=e)
    assert r.returncode != 0 and "--gpus 4" in r.stderr
