"""BF16 wide-MLP probe: GEMM vs the bf16 model, one step / short fits vs
oracle/wide_emul.py, and the C4 epoch time (CUDA events) for TF32 and BF16."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle
from oracle import wide_emul as W
import paper_2111_12055_b200 as gbx

dev = gbx.Device(0)
orc = oracle.Restatement()
rng = np.random.default_rng(1)
for (M, N, K) in [(128, 256, 64), (300, 200, 100), (8192, 512, 512), (512, 512, 8192), (77, 33, 8)]:
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    D = dev.bf16_gemm(A, B).astype(np.float64)
    ref = W.bf16(A).astype(np.float64) @ W.bf16(B).astype(np.float64).T
    sc = np.abs(W.bf16(A)).astype(np.float64) @ np.abs(W.bf16(B)).astype(np.float64).T
    print(f"gemm {M}x{N}x{K}: max err/scale {np.max(np.abs(D - ref) / sc):.3e}")

for H, n, b, ep in [(512, 2048, 2048, 1), (512, 4096, 1024, 2), (128, 777, 100, 1), (512, 8192, 8192, 1)]:
    dims = (44, H, H, 2)
    feat, tgt = orc.g1(42, n)
    p0 = orc.policy_init(7, dims)
    orders = [orc.fit_order(n, 5, e + 1) for e in range(ep)]
    pe, le = W.fit(p0, feat, tgt, orders, 0.01, ep, b, H, emulate=True)
    pg, lg = dev.wide_fit(H, p0, feat, tgt, 0.01, ep, b, 5, precision="bf16")
    pg2, _ = dev.wide_fit(H, p0, feat, tgt, 0.01, ep, b, 5, precision="bf16")
    ue, ug = pe.astype(np.float64) - p0, pg.astype(np.float64) - p0
    d = np.abs(ug - ue)
    print(f"fit H={H} n={n} B={b} ep={ep}: max|du| {d.max():.3e} max|u| {np.abs(ue).max():.3e} "
          f"ratio {d.max() / np.abs(ue).max():.3e} median rel {np.median(d / (np.abs(ue) + 1e-30)):.3e} "
          f"loss gpu {lg} emu {le} rel {np.abs(np.array(lg) - le).max() / abs(le[0]):.2e} det {np.array_equal(pg, pg2)}")

import torch
for prec in ("tf32", "bf16"):
    n, b, H = 262144, 8192, 512
    feat = torch.rand((n, 44), device="cuda") * 7
    tgt = torch.rand((n, 2), device="cuda", dtype=torch.float64)
    p = torch.from_numpy(dev.wide_init(H, 7)).cuda()
    st = torch.cuda.ExternalStream(dev.stream)
    dev.wide_fit_dev(H, p.data_ptr(), feat.data_ptr(), tgt.data_ptr(), n, 0.01, 1, b, 5, dev.stream, precision=prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(3):
        dev.wide_fit_dev(H, p.data_ptr(), feat.data_ptr(), tgt.data_ptr(), n, 0.01, 1, b, 5, dev.stream, precision=prec)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    steps = n // b
    print(f"{prec}: epoch {ms:.3f} ms, {ms / steps * 1000:.1f} us/step, {n * 1669120 / (ms * 1e-3) / 1e12:.1f} TFLOP/s")
