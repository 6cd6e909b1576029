"""Experience-store fold + snapshot at 10M tuples: host wall time vs the
stream's device time (CUDA events) per rep — equal when the path is
device-bound (including the gaps its size read-backs leave)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2111_12055_b200 as gbx
from bench import qtable_tuples_torch
n = 10_000_000
dev = gbx.Device(0)
keys, act, rew, now = qtable_tuples_torch(torch, n, 5)
feat = torch.empty((n, 44), dtype=torch.float32, device="cuda")
tgt = torch.empty((n, 2), dtype=torch.float64, device="cuda")
qt = gbx.DeviceQTable(dev)
s = torch.cuda.ExternalStream(dev.stream)
for rep in range(4):
    e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    qt.clear()
    t0 = time.perf_counter()
    e0.record(s)
    qt.update_batch_dev(keys.data_ptr(), act.data_ptr(), rew.data_ptr(), now.data_ptr(), n)
    e1.record(s)
    t1 = time.perf_counter()
    rows = qt.snapshot_dev(0.1, feat.data_ptr(), tgt.data_ptr(), n)
    e2.record(s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"fold host {1e3*(t1-t0):.2f} ms dev {e0.elapsed_time(e1):.2f} ms | snapshot host {1e3*(t2-t1):.2f} dev {e1.elapsed_time(e2):.2f}")
