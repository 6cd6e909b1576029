"""update_batch latency on a small experience store that grows every call
(Algorithm 1's regime) and on one that does not."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2111_12055_b200 as gbx  # noqa: E402

dev = gbx.Device(0)
rng = np.random.default_rng(1)
n = 10_000
for grow in (True, False):
    qt = gbx.DeviceQTable(dev)
    keys = rng.integers(0, 50, (n, 30)).astype(np.uint32)
    keys[:, 0] %= 8
    ms = []
    for it in range(6):
        if grow:
            keys = rng.integers(0, 50, (n, 30)).astype(np.uint32)
            keys[:, 0] %= 8
        act = rng.integers(0, 2, n).astype(np.uint8)
        t0 = time.perf_counter()
        qt.update_batch(keys, act, rng.random(n), np.full(n, 10 * it, np.uint64))
        ms.append((time.perf_counter() - t0) * 1e3)
    print("growing" if grow else "fixed  ", " ".join(f"{m:.2f}" for m in ms), "ms; states", qt.size())
    qt.close()
