"""Driver for ncu launch lists of the experience-store fold (row f1)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2111_12055_b200 as gbx
from bench import qtable_tuples_torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
keys, act, rew, now = qtable_tuples_torch(torch, n, 5)
feat = torch.empty((n, 44), dtype=torch.float32, device="cuda")
tgt = torch.empty((n, 2), dtype=torch.float64, device="cuda")
dev = gbx.Device(0)
qt = gbx.DeviceQTable(dev)
for _ in range(2):
    qt.clear()
    qt.update_batch_dev(keys.data_ptr(), act.data_ptr(), rew.data_ptr(), now.data_ptr(), n)
    qt.snapshot_dev(0.1, feat.data_ptr(), tgt.data_ptr(), n)
torch.cuda.synchronize()
