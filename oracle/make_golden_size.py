"""Goldens AT THE BENCHMARKED SIZES from the COMPILED REFERENCE
(oracle/_ref/libgbxref.so = the unmodified proj/src/*.cpp).

Run here (where /root/reference exists; ~4 min of single-threaded fit):
    python -m oracle.make_golden_size
Writes tests/golden/at_size.npz (outputs + input checksums only; the GPU
tests regenerate the inputs from the same seeds).

Cases (fit = proj/src/policy.cpp:297-337, forward = :29-55 / select_greedy
:339-342):
  c2     the bench headline epoch: bench.synthetic_log(1_000_000) (numpy
         PCG64 seed 42), PolicyNet::init(7), lr 0.01, batch 8192, seed 99, 1 epoch
  c2b32  the same log and init at the reference default batch 32 (31,250
         dependent steps; the bit-exact 1-CTA kernel's regime)
  c2inf  greedy actions over the 1M headline states under c2's trained net
  c3     G1 (SplitMix64, proj/tests/test_policy.cpp:15-28) 10M records, init 7,
         lr 0.01, global batch 65,536 (C3 at 8 GPUs = 8 x 8,192), seed 5, 1 epoch
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Reference, Restatement, build  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "at_size.npz")


def main() -> None:
    import bench

    build(ref=True)
    ref, orc = Reference(), Restatement()
    out = {}

    def fnv(a):
        return np.uint64(orc.fnv1a(np.ascontiguousarray(a)))

    feat, tgt = bench.synthetic_log(1_000_000)
    out["c2_feat_fnv"], out["c2_tgt_fnv"] = fnv(feat), fnv(tgt)
    p7 = ref.policy_init(7)
    for name, batch in (("c2", 8192), ("c2b32", 32)):
        t0 = time.perf_counter()
        rc, p, el, _ = ref.fit(p7, feat, tgt, 0.01, 1, batch, 99)
        assert rc == 0, ref.err()
        out[f"{name}_params"], out[f"{name}_loss"] = p, el
        out[f"{name}_cfg"] = np.array([1_000_000, 7, 1, batch, 99], np.int64)
        print(f"{name}: fit 1M records batch {batch}: {time.perf_counter() - t0:.1f} s, "
              f"loss {el[0]!r}", flush=True)
    act = ref.select_greedy(out["c2_params"], feat)
    out["c2inf_act_fnv"], out["c2inf_wave64"] = fnv(act), np.int64(act.sum())
    out["c2inf_act_head"] = act[:4096].copy()
    del feat, tgt

    n3 = 10_000_000
    feat, tgt = ref.g1(3, n3)
    out["c3_feat_fnv"], out["c3_tgt_fnv"] = fnv(feat), fnv(tgt)
    t0 = time.perf_counter()
    rc, p, el, _ = ref.fit(p7, feat, tgt, 0.01, 1, 65536, 5)
    assert rc == 0, ref.err()
    out["c3_params"], out["c3_loss"] = p, el
    out["c3_cfg"] = np.array([n3, 7, 1, 65536, 5, 3], np.int64)
    print(f"c3: fit 10M records batch 65536: {time.perf_counter() - t0:.1f} s, loss {el[0]!r}")
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "B")


if __name__ == "__main__":
    main()
