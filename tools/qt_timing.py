"""Per-rep timing of the experience-store fold (variance triage)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2111_12055_b200 as gbx
from bench import qtable_tuples_torch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
dev = gbx.Device(0)
keys, act, rew, now = qtable_tuples_torch(torch, n, 5)
feat = torch.empty((n, 44), dtype=torch.float32, device="cuda")
tgt = torch.empty((n, 2), dtype=torch.float64, device="cuda")
qt = gbx.DeviceQTable(dev)
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    qt.clear()
    qt.update_batch_dev(keys.data_ptr(), act.data_ptr(), rew.data_ptr(), now.data_ptr(), n)
    t1 = time.perf_counter()
    rows = qt.snapshot_dev(0.1, feat.data_ptr(), tgt.data_ptr(), n)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: fold {1e3*(t1-t0):.1f} ms, snapshot {1e3*(t2-t1):.1f} ms, rows {rows}", flush=True)
