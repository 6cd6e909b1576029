"""Exploration on the GPU box: tcgen05 GEMM + wide-MLP path vs numpy/oracle."""
import sys, time, numpy as np
sys.path.insert(0, ".")
import oracle, paper_2111_12055_b200 as gbx
orc = oracle.Restatement(); dev = gbx.Device(0)
def trunc(x): return (np.ascontiguousarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
rng = np.random.default_rng(1)
for (M, N, K) in [(128, 128, 32), (300, 200, 100), (1000, 512, 44), (512, 48, 1000), (77, 33, 8)]:
    A = rng.standard_normal((M, K)).astype(np.float32); B = rng.standard_normal((N, K)).astype(np.float32)
    D = dev.tf32_gemm(A, B).astype(np.float64)
    ref = trunc(A).astype(np.float64) @ trunc(B).astype(np.float64).T
    sc = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    print(f"gemm {M}x{N}x{K}: max|D-trunc_ref|/sum|ab| = {np.max(np.abs(D-ref)/sc):.2e}  max|D-exact|/sum|ab| = {np.max(np.abs(D - A.astype(np.float64)@B.astype(np.float64).T)/sc):.2e}")
H = 512; dims = (44, H, H, 2)
p_dev = dev.wide_init(H, 7); p_orc = orc.policy_init(7, dims)
print("wide init bit-exact:", np.array_equal(p_dev, p_orc))
feat, tgt = orc.g1(42, 4096)
pr = dev.wide_forward(H, p_orc, feat); po, _ = orc.forward(p_orc, feat, dims)
print(f"wide forward: max|dp| = {np.abs(pr-po).max():.2e}")
for (n, b, ep) in [(2048, 256, 1), (4096, 512, 2)]:
    t0 = time.time(); rc, pref, elref, _ = orc.fit(p_orc, feat[:n], tgt[:n], 0.01, ep, b, 5, dims=dims); t1 = time.time()
    pg, elg = dev.wide_fit(H, p_orc, feat[:n], tgt[:n], 0.01, ep, b, 5)
    d = np.abs(pg.astype(np.float64) - pref); upd = np.abs(pref - p_orc.astype(np.float64))
    print(f"wide fit n={n} b={b} ep={ep}: oracle {t1-t0:.1f}s; max|dw|={d.max():.2e} (max update {upd.max():.2e}, rel {d.max()/upd.max():.2e}); loss {elg} vs {elref}")
# throughput: 1M records, batch 8192, 1 epoch, device-resident
import torch  # after libgbxcu: both resolve the same libnccl via RUNPATH
n = 1_000_000
f = np.random.default_rng(3).random((n, 44), dtype=np.float32) * 7
t = np.full((n, 2), 0.5); t[:, 0] = np.random.default_rng(4).uniform(0.02, 0.98, n); t[:, 1] = 1 - t[:, 0]
fd, td = torch.from_numpy(f).cuda(), torch.from_numpy(t).cuda(); pd = torch.from_numpy(p_dev).cuda()
dev.wide_fit_dev(H, pd.data_ptr(), fd.data_ptr(), td.data_ptr(), n, 0.01, 1, 8192, 1)
torch.cuda.synchronize(); t0 = time.time()
for _ in range(3): dev.wide_fit_dev(H, pd.data_ptr(), fd.data_ptr(), td.data_ptr(), n, 0.01, 1, 8192, 1)
torch.cuda.synchronize(); dt = (time.time() - t0) / 3
print(f"wide fit 1M x 1 epoch @8192: {dt*1e3:.1f} ms -> {n/dt:.3e} records/s, {n*1669120/dt/1e12:.1f} TFLOP/s")
