"""The real multi-process peer-set path (CUDA IPC exchange regions,
system-scope arrival counter and LL parameter words: the fused kernel's
SYS=true instantiation that `bench.py --gpus N` runs across GPUs), driven by
separate processes on ONE GPU whose contexts time-slice. Parameters must be
identical across ranks and within 2 fp32 ulp (observed 0) of a single-process
fit with the same global batch."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n,batch,ranks,opt", [(20_000, 2048, 2, "sgd"), (12_000, 3000, 3, "sgd"),
                                             (30_000, 8192, 4, "sgd"), (20_000, 4096, 2, "adam")])
def test_ipc_peer_set_matches_single_process(n, batch, ranks, opt):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ipc_peer_probe.py"), str(n),
                        str(batch), str(ranks), opt], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
