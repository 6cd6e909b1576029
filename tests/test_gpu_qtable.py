"""GPU parity of the device experience store: batched
QTable::update (proj/src/qtable.cpp:76-92) and snapshot_policy_dataset
(:143-155) against the compiled reference (oracle/_ref, unmodified sources).

Tolerances: keys, key order, entry presence, timestamps, update counts and
snapshot features bit-exact; Q values bit-exact for omega == 1 (the
reference default) and rel 1e-14 otherwise (pow); Boltzmann targets rel 1e-15
(CUDA exp vs glibc exp, last ulp)."""
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


def tuples(seed, n, n_distinct, wide=False):
    """n tuples over ~n_distinct keys: stage in [0, 8), counters small (or full
    u32 range when wide), some words constant, check-ins non-decreasing."""
    rng = np.random.default_rng(seed)
    base = np.zeros((n_distinct, 30), np.uint32)
    base[:, 0] = rng.integers(0, 8, n_distinct)
    hi = 2**32 if wide else 40
    base[:, 1:] = rng.integers(0, hi, (n_distinct, 29), dtype=np.uint64).astype(np.uint32)
    base[:, 25] = 7                       # a constant word (skipped radix pass)
    keys = base[rng.integers(0, n_distinct, n)]
    act = rng.integers(0, 2, n).astype(np.uint8)
    rew = rng.random(n) * 0.4 + 0.8
    now = np.sort(rng.integers(0, 1000, n)).astype(np.uint64)
    return keys, act, rew, now


def check_table(t, o, q_rtol=0.0):
    np.testing.assert_array_equal(t["keys"], o["keys"])
    np.testing.assert_array_equal(t["has"], o["has"])
    h = o["has"].astype(bool)
    np.testing.assert_array_equal(t["t"][h], o["t"][h])
    np.testing.assert_array_equal(t["cnt"][h], o["cnt"][h])
    if q_rtol == 0.0:
        np.testing.assert_array_equal(t["q"][h], o["q"][h])
    else:
        np.testing.assert_allclose(t["q"][h], o["q"][h], rtol=q_rtol)


@pytest.mark.parametrize("n,n_distinct,wide", [(1, 1, False), (5000, 1200, False),
                                               (60_000, 20_000, True), (200_000, 3000, False)])
def test_fold_and_snapshot_match_reference(dev, ref, n, n_distinct, wide):
    keys, act, rew, now = tuples(n + n_distinct, n, n_distinct, wide)
    o = ref.qtable_fold(keys, act, rew, now, alpha=0.3, omega=1.0, rho=0.1)
    qt = gbx.DeviceQTable(dev, 0.3, 1.0)
    qt.update_batch(keys, act, rew, now)
    check_table(qt.export(), o)
    feat, tgt = qt.snapshot(0.1)
    np.testing.assert_array_equal(feat, o["feat"])            # glibc log1pf restated
    np.testing.assert_allclose(tgt, o["tgt"], rtol=1e-15, atol=1e-300)
    assert qt.size()[0] == len(o["keys"])
    qt.close()


def test_fold_omega_below_one(dev, ref):
    keys, act, rew, now = tuples(3, 40_000, 2000)
    o = ref.qtable_fold(keys, act, rew, now, alpha=0.25, omega=0.97, rho=0.05)
    qt = gbx.DeviceQTable(dev, 0.25, 0.97)
    qt.update_batch(keys, act, rew, now)
    check_table(qt.export(), o, q_rtol=1e-14)


def test_incremental_batches_equal_one_fold(dev, ref):
    keys, act, rew, now = tuples(11, 30_000, 4000)
    o = ref.qtable_fold(keys, act, rew, now)
    qt = gbx.DeviceQTable(dev)
    for lo, hi in [(0, 7000), (7000, 7001), (7001, 22_000), (22_000, 30_000)]:
        qt.update_batch(keys[lo:hi], act[lo:hi], rew[lo:hi], now[lo:hi])
    check_table(qt.export(), o)
    feat, tgt = qt.snapshot(0.1)
    np.testing.assert_array_equal(feat, o["feat"])


def test_clock_regression_matches_reference(dev, ref):
    keys, act, rew, now = tuples(5, 10_000, 500)
    now = now.copy()
    now[6000:] = now[6000:] - now[6000] // 2 - 1           # time goes backwards mid-stream
    o = ref.qtable_fold(keys, act, rew, now)
    assert o["bad"] >= 0
    qt = gbx.DeviceQTable(dev)
    with pytest.raises(gbx.ClockRegressionError) as ei:
        qt.update_batch(keys, act, rew, now)
    assert ei.value.index == o["bad"]
    check_table(qt.export(), o)                             # prefix applied, as the reference


def test_snapshot_validation(dev):
    qt = gbx.DeviceQTable(dev)
    with pytest.raises(gbx.InvalidTemperatureError):
        qt.snapshot(0.0)
    keys = np.zeros((2, 30), np.uint32)
    keys[:, 0] = 9                                           # invalid stage index
    qt.update_batch(keys, np.array([0, 1], np.uint8), np.array([1.0, 1.0]), np.array([0, 0], np.uint64))
    with pytest.raises(gbx.ValidationError):
        qt.snapshot(0.1)
    with pytest.raises(gbx.ValidationError):
        gbx.DeviceQTable(dev, 0.0, 1.0)
    with pytest.raises(gbx.ValidationError):
        qt.update_batch(keys[:1], np.array([2], np.uint8), np.array([1.0]), np.array([0], np.uint64))


def test_snapshot_feeds_fit_on_device(dev, ref):
    """Experience store -> training records stay on the device (fit_dev)."""
    import torch
    keys, act, rew, now = tuples(21, 50_000, 9000)
    qt = gbx.DeviceQTable(dev)
    qt.update_batch(keys, act, rew, now)
    feat_h, tgt_h = qt.snapshot(0.1)
    d_feat = torch.empty((len(feat_h), 44), dtype=torch.float32, device="cuda")
    d_tgt = torch.empty((len(feat_h), 2), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    r = qt.snapshot_dev(0.1, d_feat.data_ptr(), d_tgt.data_ptr(), len(feat_h))
    torch.cuda.synchronize()
    assert r == len(feat_h)
    np.testing.assert_array_equal(d_feat.cpu().numpy(), feat_h)
    np.testing.assert_array_equal(d_tgt.cpu().numpy(), tgt_h)


def test_load_text_then_snapshot_matches_reference(dev, ref):
    """Experience-log load (row f2): the reference's persisted Q-table text
    (QTable::save format) -> device table -> device snapshot, against the
    reference's QTable::load + snapshot_policy_dataset."""
    keys, act, rew, now = tuples(17, 20_000, 3000, wide=True)
    o = ref.qtable_fold(keys, act, rew, now)
    h = ["gbx-qtable 1 0.3 1"]
    for r in range(len(o["keys"])):
        for a in (0, 1):
            if o["has"][r, a]:
                h.append(" ".join(str(int(v)) for v in o["keys"][r]) +
                         f" {a} {float(o['q'][r, a])!r} {int(o['t'][r, a])} {int(o['cnt'][r, a])}")
    text = "\n".join(h) + "\n"
    qt = gbx.DeviceQTable.load(dev, text)
    check_table(qt.export(), o)
    feat, tgt = qt.snapshot(0.1)
    f_ref, t_ref = ref.qtable_snapshot(text, 0.1)            # QTable::load in the reference
    np.testing.assert_array_equal(feat, f_ref)
    np.testing.assert_allclose(tgt, t_ref, rtol=1e-15, atol=1e-300)
    with pytest.raises(gbx.ValidationError):
        gbx.DeviceQTable.load(dev, "gbx-qtable 2 0.3 1\n")
    with pytest.raises(gbx.ValidationError):
        gbx.DeviceQTable.load(dev, "gbx-qtable 1 0.3 1\n1 2 3\n")


def test_hot_key_long_segment(dev, ref):
    """One (key, action) updated 200k times in a row: a single long segment
    folded sequentially (the Eq.-5 chain), plus a handful of cold keys."""
    n = 200_000
    keys = np.zeros((n, 30), np.uint32)
    keys[:, 0] = 3
    keys[:, 5] = 17
    keys[::1000, 7] = np.arange(0, n, 1000, dtype=np.uint32) % 5  # a few other keys
    act = np.zeros(n, np.uint8)
    act[1::2] = 1
    rew = np.random.default_rng(2).random(n) + 0.5
    now = np.arange(n, dtype=np.uint64) // 7
    o = ref.qtable_fold(keys, act, rew, now, alpha=0.3, omega=0.999)
    qt = gbx.DeviceQTable(dev, 0.3, 0.999)
    qt.update_batch(keys, act, rew, now)
    check_table(qt.export(), o, q_rtol=1e-12)


@pytest.mark.parametrize("case", ["shared_prefix", "few_varying_words", "bench_shape", "digit_edge",
                                  "one_action", "rare_word", "rare_action"])
def test_sort_paths_match_reference(dev, ref, case):
    """The fold's MSD fast path (one sort by the top varying key bits above
    the action bit) and its fallback to the full LSD sort when neighbours
    share those bits but not the key (shared_prefix: keys differ only far
    down, in word 27); few_varying_words: every varying bit fits the digit;
    bench_shape: the benchmark's keys (3 + 5 x 12 key bits + the action fill
    the 64-bit digit exactly, words 6.. checked on the device); digit_edge:
    two 32-bit words, only the first fits beside the action bit; one_action:
    every tuple has action 1 (no action bit in the digit); rare_word /
    rare_action: a bit that varies in one tuple only, off the sample the
    packing is chosen from (200k tuples: every 3rd is sampled) — the first
    pass's exact spread must trigger the re-run."""
    rng = np.random.default_rng(17)
    n_distinct, n = 3000, (200_000 if case.startswith("rare") else 40_000)
    base = np.zeros((n_distinct, 30), np.uint32)
    if case == "shared_prefix":
        prefix = rng.integers(0, 4096, (40, 27)).astype(np.uint32)
        prefix[:, 0] %= 8                                   # stage < 8 (encode_state)
        base[:, :27] = prefix[rng.integers(0, 40, n_distinct)]
        base[:, 27] = rng.integers(0, 1 << 20, n_distinct).astype(np.uint32)
    elif case == "few_varying_words":
        base[:, 0] = rng.integers(0, 8, n_distinct)
        base[:, 3] = rng.integers(0, 1 << 16, n_distinct).astype(np.uint32)
    elif case == "bench_shape":
        base[:] = rng.integers(0, 4096, (n_distinct, 30)).astype(np.uint32)
        base[:, 0] %= 8
        base[:, 0] |= 4                                     # word 0 spans exactly 3 bits
        base[:, 1:6] |= 2048                                # words 1..5 exactly 12 bits
    elif case == "digit_edge":
        base[:, 0] = 5
        base[:, 2] = rng.integers(0, 2**32, n_distinct, dtype=np.uint64).astype(np.uint32) | 2**31
        base[:, 4] = rng.integers(0, 2**32, n_distinct, dtype=np.uint64).astype(np.uint32) | 2**31
    elif case.startswith("rare"):
        base[:, 0] = rng.integers(0, 8, n_distinct)
        base[:, 4] = rng.integers(0, 1 << 12, n_distinct).astype(np.uint32)
    else:  # one_action
        base[:, 0] = rng.integers(0, 8, n_distinct)
        base[:, 1:5] = rng.integers(0, 1 << 20, (n_distinct, 4)).astype(np.uint32)
    keys = base[rng.integers(0, n_distinct, n)]
    act = rng.integers(0, 2, n).astype(np.uint8)
    if case == "one_action":
        act[:] = 1
    if case == "rare_word":
        keys = keys.copy()
        keys[100_000, 2] = 5                                # word 2 constant elsewhere; 100000 % 3 == 1
    if case == "rare_action":
        act[:] = 0
        act[100_001] = 1
    rew = rng.random(n) * 0.4 + 0.8
    now = np.sort(rng.integers(0, 1000, n)).astype(np.uint64)
    o = ref.qtable_fold(keys, act, rew, now, alpha=0.3, omega=1.0, rho=0.1)
    qt = gbx.DeviceQTable(dev, 0.3, 1.0)
    qt.update_batch(keys, act, rew, now)
    check_table(qt.export(), o)
    feat, tgt = qt.snapshot(0.1)
    np.testing.assert_array_equal(feat, o["feat"])
    np.testing.assert_allclose(tgt, o["tgt"], rtol=1e-15, atol=1e-300)


def test_columnar_file_round_trip(dev, ref, tmp_path):
    """Binary columnar table file (row f2): device table -> file -> a fresh
    device table, identical contents and hyperparameters, same snapshot as the
    reference; corrupted / truncated / foreign files are rejected."""
    keys, act, rew, now = tuples(23, 30_000, 4000, wide=True)
    o = ref.qtable_fold(keys, act, rew, now, alpha=0.25, omega=0.9, rho=0.1)
    qt = gbx.DeviceQTable(dev, 0.25, 0.9)
    qt.update_batch(keys, act, rew, now)
    path = str(tmp_path / "table.gbxq")
    qt.save_columnar(path)
    qt2 = gbx.DeviceQTable.load_columnar(dev, path)
    a, b = qt.export(), qt2.export()
    hv = a["has"].astype(bool)
    for k in ("keys", "has"):
        np.testing.assert_array_equal(a[k], b[k])
    for k in ("q", "t", "cnt"):
        np.testing.assert_array_equal(a[k][hv], b[k][hv])   # absent entries carry no state
    check_table(b, o, q_rtol=1e-14)
    feat, tgt = qt2.snapshot(0.1)
    np.testing.assert_array_equal(feat, o["feat"])
    np.testing.assert_allclose(tgt, o["tgt"], rtol=1e-13, atol=1e-300)
    # alpha/omega travel with the file: one more fold agrees with the original
    k2, a2, r2, n2 = keys[:100], act[:100], rew[:100], now[:100] + 5000
    qt.update_batch(k2, a2, r2, n2)
    qt2.update_batch(k2, a2, r2, n2)
    a, b = qt.export(), qt2.export()
    np.testing.assert_array_equal(a["has"], b["has"])
    hv = a["has"].astype(bool)
    np.testing.assert_array_equal(a["q"][hv], b["q"][hv])
    raw = bytearray(open(path, "rb").read())
    bad = str(tmp_path / "bad.gbxq")
    for mutate in (lambda r: r.__setitem__(100, r[100] ^ 1),      # payload bit flip
                   lambda r: r.__delitem__(slice(len(r) - 8, None)),  # truncated
                   lambda r: r.__setitem__(0, ord("X"))):           # magic
        r = bytearray(raw)
        mutate(r)
        open(bad, "wb").write(bytes(r))
        with pytest.raises(gbx.ValidationError):
            gbx.DeviceQTable.load_columnar(dev, bad)
    with pytest.raises(gbx.ValidationError):
        gbx.DeviceQTable.load_columnar(dev, str(tmp_path / "missing.gbxq"))
