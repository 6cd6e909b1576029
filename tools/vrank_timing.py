"""Train-kernel time per 1M-record epoch at B = 8192 with the peer-set
exchange run over R virtual ranks in one launch (R = 1: the plain kernel).
The reduce reads R partial arrays: this shows how the exchange scales with R."""
import sys

sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx  # noqa: E402
from bench import synthetic_log  # noqa: E402

n = 1_000_000
feat, tgt = synthetic_log(n)
dev = gbx.Device(0)
p0 = dev.policy_init(7)
for R in (1, 2, 4, 8):
    ms = []
    for rep in range(3):
        dev.fit(p0, feat, tgt, 0.01, 1, 8192, 99, virtual_ranks=R if R > 1 else 0)
        ms.append(dev.last_fit_timing()[1])
    print(f"R={R}: train kernel {min(ms):.3f} ms per epoch")
