"""C5 timing probe: 1e8 shaders / 1e4 apps generated on the device; evaluate
(inference + aggregation) vs greedy inference alone, CUDA events."""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2111_12055_b200 as gbx

dev = gbx.Device(0)
apps, per = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (10_000, 10_000)
s, feat = bench.synthetic_suite_torch(torch, apps, per)
ds = dev.suite_upload_dev(s, feat)
n = ds.n_shaders
p = torch.from_numpy(dev.policy_init(7)).cuda()
act = torch.empty(n, dtype=torch.uint8, device="cuda")
rows = torch.empty((apps, 5), dtype=torch.float64, device="cuda")
st = torch.cuda.ExternalStream(dev.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("evaluate", lambda: ds.evaluate_dev(p.data_ptr(), 10, 77, act.data_ptr(), rows.data_ptr(), dev.stream)),
                 ("forward", lambda: dev.forward_dev(p.data_ptr(), feat.data_ptr(), n, None, act.data_ptr(), gbx.FWD_FAST, dev.stream))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(5):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 5:.3f} ms")
