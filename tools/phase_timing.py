import ctypes as C, os, sys, numpy as np
sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx
lib = gbx.load_library(os.path.abspath("tools/timing/libgbxcu.so"))
lib.gbxcu_debug_phase_cycles.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
lib.gbxcu_debug_phase_cycles_tc.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
names_tc = ["P0 convert", "F1", "F2", "F3 B1 tail", "B2+G1+scalars", "G0", "tile top (wait+prefetch)",
            "partial store+flag", "flag wait", "reduce+SGD+publish", "LL all-gather", "F3 logits", "F3 softmax", "", "", ""]
from bench import synthetic_log
names = ["P0 convert", "F1", "F2", "F3+B1", "B2(+gw1,extras)", "G0", "tile loop top", "wait+prefetch",
         "partials write", "grid barrier 1", "loss+param reduce", "grid barrier 2", "reload", "", "", ""]
dev = gbx.Device(0)
for n, b in [(20000, 32), (1000000, 4096), (1000000, 8192), (1000000, 65536)]:
    f, t = synthetic_log(n)
    p = dev.policy_init(7)
    dev.fit(p, f, t, 0.01, 1, b, 99)
    buf = (C.c_ulonglong * 16)()
    fn = lib.gbxcu_debug_phase_cycles if b <= 32 else lib.gbxcu_debug_phase_cycles_tc
    if b > 32: names = names_tc
    fn(buf, 1)
    dev.fit(p, f, t, 0.01, 1, b, 99)
    fn(buf, 1)
    v = np.array(buf[:], np.float64); steps = (n + b - 1) // b
    print(f"batch {b}: {v.sum()/steps:.0f} cycles/step (CTA 0)")
    for i in np.argsort(-v):
        if v[i] > 0: print(f"   {names[i]:22s} {v[i]/steps:9.0f} cyc/step {v[i]/v.sum():6.1%}")

# per-CTA globaltimer trace (steps 8..15) of the last fit (batch 65536 above -> rerun 8192)
f, t = synthetic_log(1000000)
p = dev.policy_init(7)
dev.fit(p, f, t, 0.01, 1, 8192, 99)
tr = (C.c_ulonglong * (8 * 160 * 6))()
lib.gbxcu_debug_trace_tc(tr)
T = np.array(tr[:], np.float64).reshape(8, 160, 6)[:, :148, :5]
for s in range(8):
    base = T[s, :, 0].min()
    rel = (T[s] - base)
    print(f"step {8+s}: start spread {np.ptp(T[s,:,0]):.0f} ns | publish min/med/max "
          f"{rel[:,1].min():.0f}/{np.median(rel[:,1]):.0f}/{rel[:,1].max():.0f} | waitdone "
          f"{rel[:,2].min():.0f}/{rel[:,2].max():.0f} | slice pub {rel[:,3].min():.0f}/{rel[:,3].max():.0f}"
          f" | gathered {rel[:,4].min():.0f}/{rel[:,4].max():.0f} ns; slowest publisher CTA {int(rel[:,1].argmax())}")
np.save("gpurun_out/tc_trace.npy", T)
