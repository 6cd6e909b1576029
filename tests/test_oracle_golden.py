"""CPU tests: the oracle restatement (oracle/gbx_oracle.c) against the golden
vectors generated from the compiled reference (oracle/make_golden.py), the
reference's own known-answer tests, and — when oracle/_ref is present — the
compiled reference directly."""
import numpy as np
import pytest

import oracle
from conftest import golden


def test_kats(orc):
    k = golden("kat")
    # proj/tests/test_policy.cpp:85-94
    assert orc.kl_loss((0.5, 0.5), (0.75, 0.25)) == pytest.approx(0.14384103622589042, abs=1e-9)
    assert orc.kl_loss((0.5, 0.5), (0.75, 0.25)) == float(k["kl_half_vs_075"])
    assert orc.kl_loss((0.73, 0.27), (0.73, 0.27)) == float(k["kl_identity"])
    zt = orc.kl_loss((0.5, 0.5), (1.0, 0.0))
    assert np.isfinite(zt) and zt >= 0 and zt == float(k["kl_zero_target"])
    # proj/tests/test_qtable.cpp:114-131
    b = orc.boltzmann_pair(1.0, 0.9, 0.1)
    assert b[0] == pytest.approx(0.7310585786300049, rel=1e-12)
    np.testing.assert_array_equal(b, k["boltzmann_1_09_rho01"])


def test_param_count_and_init(orc):
    # proj/tests/test_policy.cpp:32-46
    p = orc.policy_init(1)
    assert p.size == 5026 and p.nbytes == 20104
    np.testing.assert_array_equal(orc.policy_init(1234), orc.policy_init(1234))
    assert not np.array_equal(orc.policy_init(1234), orc.policy_init(1235))
    np.testing.assert_array_equal(orc.policy_init(7), golden("forward_g1")["params_init"])


def test_zero_net_uniform_and_tie(orc):
    # proj/tests/test_policy.cpp:58-76, 197-202
    feat, _ = orc.g1(12, 5)
    probs, act = orc.forward(np.zeros(5026, np.float32), feat)
    assert (probs == 0.5).all() and (act == 1).all()


def test_forward_matches_golden(orc):
    g = golden("forward_g1")
    feat, _ = orc.g1(int(g["seed"]), int(g["n"]))
    assert orc.fnv1a(feat) == int(g["feat_fnv"])
    for tag in ("init", "trained"):
        probs, act = orc.forward(g[f"params_{tag}"], feat)
        np.testing.assert_array_equal(probs, g[f"probs_{tag}"])
        np.testing.assert_array_equal(act, g[f"act_{tag}"])


def test_gradient_matches_golden(orc):
    g = golden("gradient")
    for inst in range(3):
        f, t = orc.g1(2024 + inst, 3)
        p = orc.policy_init(1000 + inst)
        np.testing.assert_array_equal(orc.batch_kl_gradient(p, f, t), g[f"g{inst}"])
        assert orc.batch_kl_loss(p, f, t) == float(g[f"l{inst}"])
    f, t = orc.g1(77, 32)
    np.testing.assert_array_equal(orc.batch_kl_gradient(orc.policy_init(7), f, t), g["g32"])


@pytest.mark.parametrize("name", ["c1", "b4096", "det40", "b1", "bigger_than_n"])
def test_fit_matches_golden(orc, name):
    g = golden("fit")
    ds, n, isd, ep, b, sd = (int(x) for x in g[f"{name}_cfg"])
    f, t = orc.g1(ds, n)
    rc, p, el, _ = orc.fit(orc.policy_init(isd), f, t, float(g[f"{name}_lr"]), ep, b, sd)
    assert rc == 0
    np.testing.assert_array_equal(p, g[f"{name}_params"])
    np.testing.assert_array_equal(el, g[f"{name}_loss"])


def test_overfit_single_sample(orc):
    # proj/tests/test_policy.cpp:139-153
    g = golden("fit")
    f, _ = orc.g1(8, 1)
    rc, p, el, _ = orc.fit(orc.policy_init(42), f, np.array([[0.99, 0.01]]), 0.05, 200, 32, 7)
    assert rc == 0 and el[-1] < 0.01 and el[-1] <= el[0]
    np.testing.assert_array_equal(p, g["overfit_params"])


def test_fit_validation(orc):
    f, t = orc.g1(1, 4)
    assert orc.fit(orc.policy_init(1), f, t, lr=-1.0)[0] == 1
    assert orc.fit(orc.policy_init(1), f[:0], t[:0])[0] == 1


def test_fit_order_matches_golden(orc):
    g = golden("order")
    o = orc.fit_order(int(g["n"]), int(g["seed"]), int(g["epochs"]))
    np.testing.assert_array_equal(o.astype(np.uint32), g["order"])
    big = orc.fit_order(int(g["big_n"]), int(g["big_seed"]), int(g["big_epochs"])).astype(np.uint32)
    assert orc.fnv1a(big) == int(g["big_fnv"])
    np.testing.assert_array_equal(big[:512], g["big_head"])


@pytest.mark.parametrize("name", ["suite_free", "suite_contended"])
def test_aggregate_matches_golden(orc, name):
    s = dict(golden(name))
    nb = len(s["app_pipe_off"]) - 1
    act = orc.forward(s["eval_params"], s["features"])[1]
    rs = np.array([orc.derive_seed(int(s["eval_seed"]), 0x45564C, b) for b in range(nb)], np.uint64)
    rows = orc.aggregate(s, act, rs, 10)
    np.testing.assert_array_equal(rows[:, 0 + 2], s["eval_rows"][:, 1])   # tuned fps
    np.testing.assert_array_equal(rows[:, 3], s["eval_rows"][:, 2])       # uplift %
    lo, cnt = orc.histogram(rows[:, 3])
    np.testing.assert_array_equal(lo, s["hist_lower"])
    np.testing.assert_array_equal(cnt, s["hist_count"])
    # baseline fps is the all-wave64 noise-free rate (simenv.cpp:378-381)
    base = orc.aggregate(s, np.ones(s["shader_lat"].shape[0], np.uint8), rs, 1)
    np.testing.assert_array_equal(base[:, 1], s["app_f64"][:, 0])
    # run_benchmark samples under an arbitrary assignment
    _, smp = orc.aggregate(s, s["rand_actions"], s["rand_run_seed"], 10, want_samples=True)
    np.testing.assert_array_equal(smp, s["rand_samples"])


def test_collect_semantics(orc):
    # epsilon = 1 -> uniform coin on u_action; epsilon = 0 -> select_sample
    feat, _ = orc.g1(3, 300)
    p = orc.policy_init(9)
    off = np.array([0, 100, 250, 300], np.uint64)
    seeds = np.array([11, 22, 33], np.uint64)
    a1 = orc.collect(p, feat, off, seeds, 1.0)
    a0 = orc.collect(p, feat, off, seeds, 0.0)
    assert 0.3 < a1.mean() < 0.7 and a0.dtype == np.uint8
    assert not np.array_equal(a0, orc.collect(p, feat, off, np.array([12, 22, 33], np.uint64), 0.0))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_restatement_vs_compiled_reference(orc):
    ref = oracle.Reference()
    feat, tgt = ref.g1(42, 2000)
    np.testing.assert_array_equal(feat, orc.g1(42, 2000)[0])
    p = ref.policy_init(7)
    np.testing.assert_array_equal(orc.forward(p, feat)[0], ref.forward(p, feat)[0])
    for (n, b, ep) in [(2000, 32, 2), (999, 100, 3), (37, 5, 4)]:
        r1 = orc.fit(p, feat[:n], tgt[:n], 0.01, ep, b, 99)
        r2 = ref.fit(p, feat[:n], tgt[:n], 0.01, ep, b, 99)
        np.testing.assert_array_equal(r1[1], r2[1])
        np.testing.assert_array_equal(r1[2], r2[2])
    np.testing.assert_array_equal(orc.fit_order(777, 3, 2), ref.fit_order(777, 3, 2))
    h = ref.suite_generate(benchmark_count=5, bandwidth_capacity=1.2, seed=9)
    s = ref.suite_export(h)
    rows_ref, lo_ref, cnt_ref = ref.evaluate(h, p, 7, 5)
    ref.suite_free(h)
    nb = len(s["app_pipe_off"]) - 1
    rs = np.array([orc.derive_seed(5, 0x45564C, b) for b in range(nb)], np.uint64)
    rows = orc.aggregate(s, orc.forward(p, s["features"])[1], rs, 7)
    np.testing.assert_array_equal(rows[:, 3], rows_ref[:, 2])


def test_qtable_snapshot_golden_shape():
    q = golden("qtable")
    # 3 keys carry both actions (stage 0, 5, 7); the one-sided key is dropped
    assert q["feat"].shape == (3, 44) and np.allclose(q["tgt"].sum(1), 1.0)


def test_log1pf_restatement_matches_host_glibc():
    """encode_state's log1pf (proj/src/core.cpp:50) restated (oracle C, mirrored
    by the device kernel) equals the host glibc log1pf on integer counts."""
    import ctypes as C

    import oracle

    libm = C.CDLL("libm.so.6")
    libm.log1pf.restype = C.c_float
    libm.log1pf.argtypes = [C.c_float]
    r = oracle.Restatement().lib
    rng = np.random.default_rng(0)
    counts = np.concatenate([np.arange(0, 20000), rng.integers(0, 2**32, 20000, dtype=np.uint64)])
    for c in counts:
        x = float(np.float32(c))
        a = np.float32(libm.log1pf(x))
        b = np.float32(r.orc_log1pf_counts(x))
        assert a.view(np.uint32) == b.view(np.uint32), c
