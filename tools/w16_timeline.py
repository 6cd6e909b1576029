"""In-graph timeline of the BF16 wide-MLP step (C4 shape: B = 8192, H = 512),
from the GBX_PHASE_TIMING build of tools/phase_timing.sh: per launch, when its
first CTA entered, when its inputs were ready (griddepcontrol.wait), when the
last CTA finished its main loop and when the last CTA exited, relative to the
step's first entry (ns). Steps 1..7 of an 8-step epoch are averaged."""
import ctypes as C, os, sys, numpy as np
sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx
lib = gbx.load_library(os.path.abspath("tools/timing/libgbxcu.so"))
lib.gbxcu_debug_w16_trace.argtypes = [C.c_void_p, C.c_int]
lib.gbxcu_debug_w16_steps.argtypes = [C.c_void_p, C.c_int]
import torch
H = int(sys.argv[1]) if len(sys.argv) > 1 else 512
b = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
dev = gbx.Device(0)
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8 * b  # records (steps past the 8th are not traced)
feat = torch.rand((n, 44), device="cuda") * 7
tgt = torch.rand((n, 2), device="cuda", dtype=torch.float64)
tgt = tgt / tgt.sum(1, keepdim=True)
p = torch.from_numpy(dev.wide_init(H, 7)).cuda()
torch.cuda.synchronize()
run = lambda: dev.wide_fit_dev(H, p.data_ptr(), feat.data_ptr(), tgt.data_ptr(), n, 1e-3, 1, b, 5, dev.stream,
                               precision="bf16")
import time
t0 = time.perf_counter(); run(); torch.cuda.synchronize()  # graph capture + warm-up
print(f"first call (capture + instantiate + run): {(time.perf_counter() - t0) * 1e3:.1f} ms host")
t0 = time.perf_counter(); run(); torch.cuda.synchronize()
print(f"second call: {(time.perf_counter() - t0) * 1e3:.1f} ms host")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
lib.gbxcu_debug_w16_steps(None, 1)
e0.record(torch.cuda.ExternalStream(dev.stream))
run()
e1.record(torch.cuda.ExternalStream(dev.stream))
torch.cuda.synchronize()
st = np.zeros(4096, np.uint64)
lib.gbxcu_debug_w16_steps(st.ctypes.data, 0)
ns = min(4096, (n + b - 1) // b)
d = np.diff(st[:ns].astype(np.float64)) / 1e3
print("per-step us (gather entry to next): first 12", np.round(d[:12], 1), "median", np.median(d),
      "p90", np.percentile(d, 90), "max", d.max(), "sum", d.sum())
print(f"epoch of {n} records: {e0.elapsed_time(e1):.3f} ms = {e0.elapsed_time(e1) * 1e3 / ((n + b - 1) // b):.1f} us/step")
res = []
for rep in range(5):
    lib.gbxcu_debug_w16_trace(None, 1)
    run()
    torch.cuda.synchronize()
    buf = np.zeros((64, 8, 2), np.uint64)
    lib.gbxcu_debug_w16_trace(buf.ctypes.data, 0)
    res.append(buf.astype(np.float64))
names = ["gather", "G1 (X W0^T)", "G2 (H1 W1^T + head)", "G3 (D2 W1)", "G4 (gW1 split-K)", "G5 (gW0 split-K)",
         "update"]
rows = []
for buf in res:
    for s in range(1, 8):
        t0 = buf[8 * s, 0, 0]
        nxt = buf[8 * (s + 1), 0, 0] if s < 7 else np.nan
        rows.append([[buf[8 * s + k, 0, 0] - t0, buf[8 * s + k, 1, 0] - t0, buf[8 * s + k, 2, 1] - t0,
                      buf[8 * s + k, 3, 1] - t0, buf[8 * s + k, 1, 1] - t0, buf[8 * s + k, 2, 0] - t0,
                      buf[8 * s + k, 3, 0] - t0] for k in range(7)] + [[nxt - t0] * 7])
a = np.nanmedian(np.array(rows), axis=0)
ph = []
for buf in res:
    for s in range(1, 7):
        t0 = buf[8 * s, 0, 0]
        ph.append([[buf[8 * s + k, q, 0] - t0, buf[8 * s + k, q, 1] - t0] for k in (2, 4) for q in range(4, 8)])
ph = np.nanmedian(np.array(ph), axis=0) / 1e3
print(f"H={H} B={b}: step (gather entry to next gather entry) {a[7][0] / 1e3:.2f} us  (median of steps 1-6)")
print(f"{'launch':24s} {'1st entry':>10s} {'ready':>13s} {'main loop':>13s} {'exit':>13s}   (us from step start;"
      " min-max over CTAs)")
for k in range(7):
    e, r, m, x, r1, m0, x0 = a[k] / 1e3
    print(f"{names[k]:24s} {e:10.2f} {r:6.2f}-{r1:6.2f} {m0:6.2f}-{m:6.2f} {x0:6.2f}-{x:6.2f}")
print("G2 head phases (min-max over CTAs): logits done, softmax done, pass 2 done, sums written:")
print("   " + "  ".join(f"{x:6.2f}-{y:6.2f}" for x, y in ph[0:4]))
print("G4/G5 SGD phases: partial dumped, barrier 1 passed, epilogue entry, TMEM dumped:")
print("   " + "  ".join(f"{x:6.2f}-{y:6.2f}" for x, y in ph[4:8]))
