import sys, numpy as np
sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx
import torch
n, H = int(sys.argv[1]), 512
dev = gbx.Device(0)
f = np.random.default_rng(3).random((n, 44), dtype=np.float32) * 7
t = np.empty((n, 2)); t[:, 0] = np.random.default_rng(4).uniform(0.02, 0.98, n); t[:, 1] = 1 - t[:, 0]
fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda()
pd = torch.from_numpy(dev.wide_init(H, 7)).cuda()
for _ in range(2):
    dev.wide_fit_dev(H, pd.data_ptr(), fd.data_ptr(), td.data_ptr(), n, 0.01, 1, 8192, 1)
torch.cuda.synchronize()
