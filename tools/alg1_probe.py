"""Phase timing of DeviceTuner.run_iteration (bench `algorithm1`)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2111_12055_b200 as gbx  # noqa: E402
from paper_2111_12055_b200 import tuner as T  # noqa: E402

R = oracle.Reference()
dev = gbx.Device(0)
h = R.suite_generate(benchmark_count=44, seed=7)
tu = T.DeviceTuner(dev, T.TunerConfig(num_iterations=3, checkins_per_iteration=50, seed=5))
orig = {k: getattr(dev, k) for k in ("collect", "aggregate", "fit", "forward")}
acc = {}


def wrap(name, fn):
    def f(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
        return r
    return f


for k, fn in orig.items():
    setattr(dev, k, wrap(k, fn))
for k in ("update_batch", "snapshot", "export"):
    setattr(tu.table, k, wrap(k, getattr(tu.table, k)))
for i in range(4):
    R.suite_advance(h, 50)
    s = R.suite_export(h)
    keys = R.suite_keys(h, len(s["features"]))
    now = R.suite_checkin(h)
    acc.clear()
    t0 = time.perf_counter()
    log = tu.run_iteration(i, s, keys, now)
    tot = time.perf_counter() - t0
    print(f"iter {i}: {tot * 1e3:.1f} ms", {k: round(v * 1e3, 1) for k, v in acc.items()}, "rows", log["table_size"])
