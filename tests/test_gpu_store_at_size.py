"""Experience store AT THE BENCHMARKED SIZE: bench.py's
`qtable` workload — 10M tuples over ~5.7M distinct StateKeys (351 varying
key bits, so the MSD digit covers only the first six words and every
duplicate group goes through the device tail check) — folded into a fresh
device table and snapshotted.

The fold is independent per key, so exact parity at size is checked on a
sample: 2,000 of the table's keys, every tuple that carries one of them (in
sequence order), folded by the compiled reference (QTable::update,
proj/src/qtable.cpp:76-92; snapshot_policy_dataset, :143-155) must give
exactly the device table's entries and snapshot rows for those keys. The
whole table is checked through size-independent properties: keys strictly
increasing, update counts summing to the number of tuples, one state per
distinct key. Tolerances as test_gpu_qtable.py: bit-exact except targets
(rel 1e-15, CUDA vs glibc exp)."""
import numpy as np
import pytest

import oracle
import paper_2111_12055_b200 as gbx

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not oracle.ref_available():
        pytest.skip("compiled reference not available")
    return oracle.Reference()


def row_hash(k):
    """64-bit polynomial hash of each 30-word row (wrapping uint64)."""
    h = np.zeros(len(k), np.uint64)
    p = np.uint64(0x9E3779B97F4A7C15)
    for w in range(k.shape[1]):
        h = h * p + k[:, w].astype(np.uint64)
    return h


def test_store_fold_and_snapshot_at_bench_size(dev, ref):
    import torch
    import bench
    n = 10_000_000
    keys, act, rew, now = bench.qtable_tuples_torch(torch, n, 5)   # bench.py's qtable inputs
    torch.cuda.synchronize()
    qt = gbx.DeviceQTable(dev, 0.3, 1.0)
    qt.update_batch_dev(keys.data_ptr(), act.data_ptr(), rew.data_ptr(), now.data_ptr(), n)
    t = qt.export()
    feat, tgt = qt.snapshot(0.1)
    qt.close()
    K = np.ascontiguousarray(keys.cpu().numpy()).view(np.uint32)
    A = act.cpu().numpy()
    R = rew.cpu().numpy()
    T = now.cpu().numpy().astype(np.uint64)
    del keys, act, rew, now

    # whole table: strictly increasing keys, counts sum to n, one state per distinct key
    tk = t["keys"]
    diff = tk[1:] != tk[:-1]
    assert diff.any(axis=1).all()
    first = diff.argmax(axis=1)
    i = np.arange(len(first))
    assert (tk[1:][i, first] > tk[:-1][i, first]).all()
    has = t["has"].astype(bool)
    assert int(t["cnt"][has].sum()) == n
    hv = row_hash(K)
    assert len(np.unique(hv)) == len(tk)
    both = has.all(axis=1)
    assert len(feat) == int(both.sum())

    # sampled exact parity against the reference
    rng = np.random.default_rng(2024)
    pick = np.sort(rng.choice(len(tk), 2000, replace=False))
    sel = tk[pick]
    mask = np.isin(hv, row_hash(sel))
    sub = K[mask]
    o = ref.qtable_fold(sub, A[mask], R[mask], T[mask], alpha=0.3, omega=1.0, rho=0.1)
    np.testing.assert_array_equal(o["keys"], sel)          # (no hash collision let a stranger in)
    np.testing.assert_array_equal(t["has"][pick], o["has"])
    h = o["has"].astype(bool)
    for f in ("t", "cnt", "q"):
        np.testing.assert_array_equal(t[f][pick][h], o[f][h])
    rows = (np.cumsum(both) - 1)[pick[both[pick]]]
    np.testing.assert_array_equal(feat[rows], o["feat"])
    np.testing.assert_allclose(tgt[rows], o["tgt"], rtol=1e-15, atol=1e-300)
