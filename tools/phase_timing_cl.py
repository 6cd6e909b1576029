"""Phase cycles of the batch-32 cluster train kernel (CTA 0, thread 0), from
the GBX_PHASE_TIMING build of tools/phase_timing.sh."""
import ctypes as C, os, sys, numpy as np
sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx
lib = gbx.load_library(os.path.abspath("tools/timing/libgbxcu.so"))
lib.gbxcu_debug_phase_cycles_cl.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
from bench import synthetic_log
names = ["step top", "P0", "F1", "cluster barrier 1", "gather h1", "F2 + barrier 2 + gather h2",
         "F3 + B1 + barrier 3 + gather d2", "B2", "G + flag", "SGD + pushes"]
dev = gbx.Device(0)
f, t = synthetic_log(100000)
p = dev.policy_init(7)
dev.fit(p, f, t, 0.01, 1, 32, 99)
buf = (C.c_ulonglong * 16)()
lib.gbxcu_debug_phase_cycles_cl(buf, 1)
dev.fit(p, f, t, 0.01, 1, 32, 99)
lib.gbxcu_debug_phase_cycles_cl(buf, 1)
v = np.array(buf[:10], np.float64); steps = 100000 // 32
print(f"{v.sum() / steps:.0f} cycles/step")
for i in np.argsort(-v):
    print(f"  {names[i]:34s} {v[i] / steps:7.0f} {v[i] / v.sum():6.1%}")
