"""Per-call overhead of a 1-epoch fit_dev at the bench's headline config:
wall time vs CUDA-event time around the call vs the kernels' own time."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx  # noqa: E402
from bench import synthetic_log  # noqa: E402

n, batch = 1_000_000, 8192
feat, tgt = synthetic_log(n)
dev = gbx.Device(0)
st = torch.cuda.ExternalStream(dev.stream)
fd, td = torch.from_numpy(feat).cuda(), torch.from_numpy(tgt).cuda()
pd = torch.from_numpy(dev.policy_init(7)).cuda()
torch.cuda.synchronize()
for _ in range(3):
    dev.fit_dev(pd.data_ptr(), fd.data_ptr(), td.data_ptr(), n, 0.01, 1, batch, 99, stream=dev.stream)
K = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ksum = 0.0
torch.cuda.synchronize()
t0 = time.perf_counter()
e0.record(st)
for _ in range(K):
    dev.fit_dev(pd.data_ptr(), fd.data_ptr(), td.data_ptr(), n, 0.01, 1, batch, 99, stream=dev.stream)
    sh, tr = dev.last_fit_timing()
    ksum += sh + tr
e1.record(st)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K * 1e3
print(f"wall {wall:.3f} ms/call, events {e0.elapsed_time(e1) / K:.3f} ms/call, kernels {ksum / K:.3f} ms/call")
