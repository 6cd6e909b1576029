"""bench.py's N>1 path end to end (the driver's scaling runs use it across
GPUs over NCCL): here two ranks share the one GPU over gloo
(GBX_BENCH_BACKEND=gloo test mode) — peer export/attach, fused steps, e2e,
the sharded C5 secondary, the detach before rank 0's single-GPU secondaries,
and exactly one JSON line. Timings in this mode are meaningless (the two
ranks' contexts time-slice)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_bench_two_ranks_one_json_line():
    env = dict(os.environ, GBX_BENCH_BACKEND="gloo")
    r = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
         "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--records", "20000",
         "--c5-apps", "100", "--c5-shaders-per-app", "200", "--qt-tuples", "20000",
         "--wide-records", "65536",
         "--no-cpu-baseline"],
        cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and "dp_fallback" not in d
    assert d["aggregation_sharded"]["rows_gathered"] == 100
    for k in ("inference", "qtable", "batch_sweep", "variants", "algorithm1", "wide_mlp"):
        assert k in d, k


def test_bench_gpus_flag_spawns_ranks():
    """`python bench.py --gpus 2` with no launcher starts the two ranks itself
    (the driver may call it that way); still one JSON line with n_gpus 2."""
    env = dict(os.environ, GBX_BENCH_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run(
        [sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
         "--records", "20000", "--no-secondary", "--no-cpu-baseline"],
        cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["records"] == 40000
