"""ncu driver: a few BF16 wide steps (C4 shape, B = 8192, H = 512)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx
dev = gbx.Device(0)
n, b, H = 8192 * 4, 8192, 512
feat = torch.rand((n, 44), device="cuda") * 7
tgt = torch.rand((n, 2), device="cuda", dtype=torch.float64)
p = torch.from_numpy(dev.wide_init(H, 7)).cuda()
torch.cuda.synchronize()
dev.wide_fit_dev(H, p.data_ptr(), feat.data_ptr(), tgt.data_ptr(), n, 0.01, 1, b, 5, dev.stream,
                 precision=sys.argv[1] if len(sys.argv) > 1 else "bf16")
torch.cuda.synchronize()
