"""Inference timing breakdown with bench-like trained parameters:
forward_dev FAST over 1M states, per-kernel durations from an ncu launch list
(run under ncu) or CUDA-event totals (run plain)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx
from bench import synthetic_log

n = 1_000_000
feat, tgt = synthetic_log(n)
dev = gbx.Device(0)
p0 = dev.policy_init(7)
trained, _ = dev.fit(p0, feat, tgt, 0.01, 8, 8192, 99)
fd = torch.from_numpy(feat).cuda()
act = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, p in (("init", p0), ("trained", trained)):
    pd = torch.from_numpy(p).cuda()
    for _ in range(3):
        dev.forward_dev(pd.data_ptr(), fd.data_ptr(), n, None, act.data_ptr(), gbx.FWD_FAST, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dev.forward_dev(pd.data_ptr(), fd.data_ptr(), n, None, act.data_ptr(), gbx.FWD_FAST, torch.cuda.current_stream().cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    print(name, "FAST ms/call", e0.elapsed_time(e1) / 10, "recheck", dev.last_recheck_count())
