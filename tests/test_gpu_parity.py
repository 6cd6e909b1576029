"""GPU parity tests: the CUDA path (through the C ABI) against the oracle
restatement and the golden vectors from the compiled reference.

Tolerances (stated per BASELINE.json north_star):
  * actions, permutation indices, per-app aggregation rows, histograms: bit-exact;
  * EXACT-mode probabilities: <= 4 ulp of fp64 (CUDA exp vs glibc exp);
  * FAST-mode probabilities: relative 1e-5;
  * gradients: relative 1e-12 per component (log/exp ulps propagate);
  * weights after N SGD steps: <= 1 fp32 ulp per weight (1-CTA steps,
    expected 0), <= 2 ulp for multi-CTA steps (fp64 re-association);
  * epoch losses: relative 1e-12.
"""
import numpy as np
import pytest

import paper_2111_12055_b200 as gbx
from conftest import golden

pytestmark = pytest.mark.gpu


def ulps32(a, b):
    a = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64)
    return np.abs(a - b)


def ulps64(a, b):
    a = np.ascontiguousarray(a, np.float64).view(np.int64)
    b = np.ascontiguousarray(b, np.float64).view(np.int64)
    return np.abs(a.astype(object) - b.astype(object)).astype(np.float64)


# ----------------------------------------------------------------- policy
@pytest.mark.parametrize("seed", [0, 1, 7, 1234, 2**63 + 5])
def test_policy_init_bit_exact(dev, orc, seed):
    np.testing.assert_array_equal(dev.policy_init(seed), orc.policy_init(seed))


@pytest.mark.parametrize("tag", ["init", "trained"])
def test_forward_matches_golden(dev, orc, tag):
    g = golden("forward_g1")
    feat, _ = orc.g1(int(g["seed"]), int(g["n"]))
    p = g[f"params_{tag}"]
    probs, act = dev.forward(p, feat, gbx.FWD_EXACT)
    np.testing.assert_array_equal(act, g[f"act_{tag}"])
    assert ulps64(probs, g[f"probs_{tag}"]).max() <= 4
    probs_f, act_f = dev.forward(p, feat, gbx.FWD_FAST)
    np.testing.assert_array_equal(act_f, g[f"act_{tag}"])
    np.testing.assert_allclose(probs_f, g[f"probs_{tag}"], rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("n", [1, 31, 33, 1000, 200_003])
def test_forward_ragged_sizes(dev, orc, n):
    g = golden("forward_g1")
    feat, _ = orc.g1(1000 + n, n)
    p = g["params_trained"]
    probs_o, act_o = orc.forward(p, feat)
    probs, act = dev.forward(p, feat, gbx.FWD_FAST)
    np.testing.assert_array_equal(act, act_o)
    np.testing.assert_allclose(probs, probs_o, rtol=1e-5, atol=1e-7)
    act_g = dev.select_greedy(p, feat)
    np.testing.assert_array_equal(act_g, act_o)


def test_forward_exact_ties_and_zero_net(dev, orc):
    feat, _ = orc.g1(12, 777)
    for mode in (gbx.FWD_EXACT, gbx.FWD_FAST):
        probs, act = dev.forward(np.zeros(5026, np.float32), feat, mode)
        assert (probs == 0.5).all() and (act == 1).all()   # test_policy.cpp:58-76,197-202
    # identical output rows -> l0 == l1 exactly for every state -> Wave64
    p = orc.policy_init(3)
    p[4960:4992] = p[4992:5024]
    p[5024] = p[5025] = 0.25
    _, act = dev.forward(p, feat, gbx.FWD_FAST)
    assert (act == 1).all()
    np.testing.assert_array_equal(act, orc.forward(p, feat)[1])


def test_forward_near_ties_are_exact(dev, orc):
    # Shrink the logit gap so that a large share of states falls inside the
    # fp32 guard band; actions must still equal the fp64 reference.
    p = golden("forward_g1")["params_trained"].copy()
    p[4960:4992] = p[4992:5024] + np.float32(1e-7) * np.sign(p[4992:5024])
    feat, _ = orc.g1(99, 50_000)
    _, act = dev.forward(p, feat, gbx.FWD_FAST)
    np.testing.assert_array_equal(act, orc.forward(p, feat)[1])


def test_forward_recheck_path_is_bit_exact(dev, orc):
    """A net trained on noise targets (small logit gaps): many states fall in
    the guard band and go through the warp-per-state exact re-check, whose
    probabilities must equal the fp64 reference bit for bit."""
    p = golden("forward_g1")["params_trained"]
    feat, _ = orc.g1(2024, 100_000)
    probs_o, act_o = orc.forward(p, feat)
    probs, act = dev.forward(p, feat, gbx.FWD_FAST)
    n_re = dev.last_recheck_count()
    assert 1000 < n_re < len(feat)
    np.testing.assert_array_equal(act, act_o)
    probs_x, _ = dev.forward(p, feat, gbx.FWD_EXACT)
    same = (probs == probs_x).all(1)
    assert same.sum() >= n_re          # re-checked rows carry the exact probabilities
    seg = np.array([0, 40_000, 100_000], np.uint64)
    seeds = np.array([11, 12], np.uint64)
    np.testing.assert_array_equal(dev.collect(p, feat, seg, seeds, 0.1),
                                  orc.collect(p, feat, seg, seeds, 0.1))


def _splitmix_units(state: int, n: int) -> np.ndarray:
    """The first n next_unit() of SplitMix64(state) (proj/include/gbx/rng.hpp)."""
    with np.errstate(over="ignore"):
        k = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(state) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


@pytest.mark.parametrize("tag", ["init", "trained"])
def test_sample_batch_is_sequential_select_sample(dev, orc, tag):
    """select_sample over a batch from one stream (SURVEY §8b gbxcu_sample_batch):
    state j uses the (j+1)-th draw; Wave32 iff u < p0 of the fp64 reference."""
    p = golden("forward_g1")[f"params_{tag}"]
    feat, _ = orc.g1(77, 60_000)
    probs_o, _ = orc.forward(p, feat)
    for state in (0, 12345, 2**64 - 3):
        u = _splitmix_units(state, len(feat))
        want = np.where(u < probs_o[:, 0], 0, 1).astype(np.uint8)
        np.testing.assert_array_equal(dev.sample_batch(p, feat, state), want)
    # near-ties: u drawn right at p0 go through the exact re-check
    np.testing.assert_array_equal(dev.sample_batch(p, feat[:1000], 99),
                                  np.where(_splitmix_units(99, 1000) < probs_o[:1000, 0], 0, 1))


def test_forward_rejects_non_finite(dev, orc):
    feat, _ = orc.g1(5, 64)
    feat[17, 10] = np.nan
    with pytest.raises(gbx.ValidationError):
        dev.forward(orc.policy_init(3), feat)
    feat[17, 10] = np.inf
    with pytest.raises(gbx.ValidationError):
        dev.forward(orc.policy_init(3), feat, gbx.FWD_FAST)


def test_forward_empty(dev):
    probs, act = dev.forward(np.zeros(5026, np.float32), np.zeros((0, 44), np.float32))
    assert probs.shape == (0, 2) and act.shape == (0,)


# ------------------------------------------------------- loss / gradient
def test_gradient_matches_golden(dev, orc):
    g = golden("gradient")
    for inst in range(3):
        f, t = orc.g1(2024 + inst, 3)
        p = orc.policy_init(1000 + inst)
        np.testing.assert_allclose(dev.batch_kl_gradient(p, f, t), g[f"g{inst}"], rtol=1e-12,
                                   atol=1e-300)
        assert dev.batch_kl_loss(p, f, t) == pytest.approx(float(g[f"l{inst}"]), rel=1e-13)
    f, t = orc.g1(77, 32)
    np.testing.assert_allclose(dev.batch_kl_gradient(orc.policy_init(7), f, t), g["g32"],
                               rtol=1e-12, atol=1e-300)


def test_gradient_large_batch(dev, orc):
    f, t = orc.g1(31, 3001)
    p = golden("forward_g1")["params_trained"]
    np.testing.assert_allclose(dev.batch_kl_gradient(p, f, t), orc.batch_kl_gradient(p, f, t),
                               rtol=1e-11, atol=1e-300)


# -------------------------------------------------------------------- fit
@pytest.mark.parametrize("name", ["c1", "b4096", "det40", "b1", "bigger_than_n"])
def test_fit_matches_golden(dev, orc, name):
    g = golden("fit")
    ds, n, isd, ep, b, sd = (int(x) for x in g[f"{name}_cfg"])
    f, t = orc.g1(ds, n)
    p, el = dev.fit(orc.policy_init(isd), f, t, float(g[f"{name}_lr"]), ep, b, sd)
    tol = 1 if b <= 64 else 2
    assert ulps32(p, g[f"{name}_params"]).max() <= tol
    np.testing.assert_allclose(el, g[f"{name}_loss"], rtol=1e-12)


def test_fit_overfit_single_sample(dev, orc):
    g = golden("fit")
    f, _ = orc.g1(8, 1)
    p, el = dev.fit(orc.policy_init(42), f, np.array([[0.99, 0.01]]), 0.05, 200, 32, 7)
    assert el[-1] < 0.01 and el[-1] <= el[0]
    assert ulps32(p, g["overfit_params"]).max() <= 1


def test_fit_uniform_targets_keep_zero_net(dev, orc):
    # proj/tests/test_policy.cpp:155-166
    f, _ = orc.g1(9, 16)
    t = np.full((16, 2), 0.5)
    p, el = dev.fit(np.zeros(5026, np.float32), f, t, 0.01, 20, 32, 0)
    assert (el < 1e-6).all()


@pytest.mark.parametrize("batch,max_ctas", [(4096, 0), (4096, 7), (1000, 3), (65536, 0)])
def test_fit_multi_cta_within_tolerance(dev, orc, batch, max_ctas):
    n = 70_001
    f, t = orc.g1(17, n)
    p0 = orc.policy_init(21)
    rc, p_ref, el_ref, _ = orc.fit(p0, f, t, 0.02, 2, batch, 4)
    p, el = dev.fit(p0, f, t, 0.02, 2, batch, 4, max_ctas=max_ctas)
    assert ulps32(p, p_ref).max() <= 2
    np.testing.assert_allclose(el, el_ref, rtol=1e-12)
    p2, el2 = dev.fit(p0, f, t, 0.02, 2, batch, 4, max_ctas=max_ctas)
    np.testing.assert_array_equal(p, p2)          # deterministic (test_policy.cpp:168-184)
    np.testing.assert_array_equal(el, el2)


def test_fit_c1_many_epochs_bit_stable(dev, orc):
    f, t = orc.g1(42, 3000)
    p0 = orc.policy_init(7)
    rc, p_ref, el_ref, _ = orc.fit(p0, f, t, 0.01, 5, 32, 99)
    p, el = dev.fit(p0, f, t, 0.01, 5, 32, 99)
    assert ulps32(p, p_ref).max() <= 1
    np.testing.assert_allclose(el, el_ref, rtol=1e-12)


def test_fit_divergence_matches_reference(dev, orc):
    f, t = orc.g1(6, 256)
    f[:, 8:] *= np.float32(1e3)
    p0 = orc.policy_init(5)
    rc, p_ref, el_ref, ep_ref = orc.fit(p0, f, t, 1e12, 4, 32, 1)
    assert rc == 2
    with pytest.raises(gbx.TrainingDivergedError) as ei:
        dev.fit(p0, f, t, 1e12, 4, 32, 1)
    assert ei.value.epoch == ep_ref
    same = (ei.value.params == p_ref) | (np.isnan(ei.value.params) & np.isnan(p_ref))
    assert same.mean() > 0.99


def test_fit_validation(dev, orc):
    f, t = orc.g1(1, 8)
    p = orc.policy_init(1)
    with pytest.raises(gbx.ValidationError):
        dev.fit(p, f, t, lr=0.0)
    with pytest.raises(gbx.ValidationError):
        dev.fit(p, f, t, epochs=0)
    with pytest.raises(gbx.ValidationError):
        dev.fit(p, f, t, batch=0)
    with pytest.raises(gbx.ValidationError):
        dev.fit(p, f[:0], t[:0])


def test_fit_order_matches_golden(dev, orc):
    g = golden("order")
    np.testing.assert_array_equal(dev.fit_order(int(g["n"]), int(g["seed"]), int(g["epochs"])),
                                  g["order"])
    big = dev.fit_order(int(g["big_n"]), int(g["big_seed"]), int(g["big_epochs"]))
    assert orc.fnv1a(big) == int(g["big_fnv"])
    for n in (1, 2, 3, 5, 64, 4097):
        np.testing.assert_array_equal(dev.fit_order(n, 3, 3), orc.fit_order(n, 3, 3).astype(np.uint32))


def test_fit_order_full_size_is_permutation(dev, orc):
    n = 1_000_000
    o = dev.fit_order(n, 99, 1)
    assert np.array_equal(np.sort(o), np.arange(n, dtype=np.uint32))
    ref = orc.fit_order(n, 99, 1).astype(np.uint32)
    assert orc.fnv1a(o) == orc.fnv1a(ref)


def test_c3_size_fit_properties(dev, orc):
    """C3 at its full size (10M records, one epoch, global batch 65,536): the
    reference cannot be run to completion here, so size-independent
    properties — a valid permutation (the oracle's own, by checksum),
    determinism of the whole epoch, finite and decreasing loss on a
    learnable target, weights changed everywhere the gradient reaches."""
    import torch
    n = 10_000_000
    o = dev.fit_order(n, 5, 1)
    assert orc.fnv1a(o) == orc.fnv1a(orc.fit_order(n, 5, 1).astype(np.uint32))
    g = torch.Generator(device="cuda").manual_seed(3)
    feat = torch.rand((n, 44), generator=g, device="cuda", dtype=torch.float32) * 7.0
    feat[:, :8] = 0.0
    feat[torch.arange(n, device="cuda"), torch.randint(0, 8, (n,), generator=g, device="cuda")] = 1.0
    p = torch.sigmoid(feat[:, 8].double() - 3.5)        # learnable target
    tgt = torch.stack([p, 1.0 - p], 1).contiguous()
    p0 = torch.from_numpy(orc.policy_init(9)).cuda()
    outs = []
    for _ in range(2):
        w = p0.clone()
        el = dev.fit_dev(w.data_ptr(), feat.data_ptr(), tgt.data_ptr(), n, 0.05, 2, 65536, 5)
        outs.append((w.cpu().numpy(), el))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    el = outs[0][1]
    assert np.isfinite(el).all() and el[1] < el[0]
    assert np.mean(outs[0][0] != p0.cpu().numpy()) > 0.9


def test_c5_size_evaluate_properties(dev, orc):
    """C5 at its nominal size (1e8 shaders across 1e4 apps, generated on the
    device): FAST actions equal the exact fp64 path on a 200k-shader sample,
    and three app-range shards reassemble the full rows bit for bit."""
    import torch
    import bench
    s, feat = bench.synthetic_suite_torch(torch, 10_000, 10_000)
    ds = dev.suite_upload_dev(s, feat)
    params = orc.policy_init(7)
    pd = torch.from_numpy(params).cuda()
    act = torch.empty(ds.n_shaders, dtype=torch.uint8, device="cuda")
    rows = torch.empty((ds.n_apps, 5), dtype=torch.float64, device="cuda")
    ds.evaluate_dev(pd.data_ptr(), 10, 77, act.data_ptr(), rows.data_ptr())
    torch.cuda.synchronize()
    rows = rows.cpu().numpy()
    assert np.isfinite(rows).all()
    idx = torch.randint(0, ds.n_shaders, (200_000,), device="cuda")
    sample = feat[idx].cpu().numpy()
    _, exact = dev.forward(params, sample, gbx.FWD_EXACT)
    np.testing.assert_array_equal(act[idx].cpu().numpy(), exact)
    cuts = [0, 3_333, 6_666, ds.n_apps]
    parts = [ds.evaluate_shard(params, 10, 77, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    np.testing.assert_array_equal(np.concatenate(parts), rows)
    ds.close()
    del s, feat
    torch.cuda.empty_cache()


# ------------------------------------------------------------- collection
@pytest.mark.parametrize("eps", [0.0, 0.3, 1.0])
def test_collect_matches_oracle(dev, orc, eps):
    feat, _ = orc.g1(8, 20_000)
    p = golden("forward_g1")["params_trained"]
    off = np.array([0, 1, 5000, 5001, 12_345, 20_000], np.uint64)
    seeds = np.array([orc.derive_seed(3, 0x414354, 0, b) for b in range(5)], np.uint64)
    np.testing.assert_array_equal(dev.collect(p, feat, off, seeds, eps),
                                  orc.collect(p, feat, off, seeds, eps))


# ------------------------------------------------------------ aggregation
@pytest.mark.parametrize("name", ["suite_free", "suite_contended"])
def test_aggregate_and_evaluate_match_golden(dev, orc, name):
    s = dict(golden(name))
    nb = len(s["app_pipe_off"]) - 1
    rows_o, smp_o = orc.aggregate(s, s["rand_actions"], s["rand_run_seed"], 10, want_samples=True)
    rows, smp = dev.aggregate(s, s["rand_actions"], s["rand_run_seed"], 10, want_samples=True)
    np.testing.assert_array_equal(rows, rows_o)
    np.testing.assert_array_equal(smp, s["rand_samples"])
    ds = dev.suite_upload(s, s["features"])
    rows_e, (lo, cnt), act = ds.evaluate(s["eval_params"], 10, int(s["eval_seed"]),
                                         want_actions=True)
    np.testing.assert_array_equal(act, orc.forward(s["eval_params"], s["features"])[1])
    np.testing.assert_array_equal(rows_e[:, 2], s["eval_rows"][:, 1])
    np.testing.assert_array_equal(rows_e[:, 3], s["eval_rows"][:, 2])
    np.testing.assert_array_equal(lo, s["hist_lower"])
    np.testing.assert_array_equal(cnt, s["hist_count"])
    ds.close()


def _ragged_suite(seed, n_apps):
    """Random CSR suite with the shapes the reference never guarantees away:
    apps without pipelines, pipelines without slots, long and 1-slot
    pipelines, shared shaders, and caps that throttle about half the apps."""
    rng = np.random.default_rng(seed)
    pipes = rng.integers(1, 5, n_apps)
    pipes[rng.random(n_apps) < 0.05] = 0
    npipe = int(pipes.sum())
    sizes = rng.integers(0, 120, npipe)
    sizes[rng.random(npipe) < 0.1] = 0
    sizes[rng.random(npipe) < 0.05] = 1
    sizes[rng.random(npipe) < 0.05] = 700
    n_slots = int(sizes.sum())
    n_sh = max(1, n_slots // 2)
    lat = rng.random((n_sh, 3))
    lat[:, 1] *= 1.6
    lat[:, 2] *= 0.6
    frac = rng.random(n_slots) * 0.06 + 0.01
    app_f64 = np.stack([rng.random(n_apps) + 0.5,                         # baseline fps
                        np.where(rng.random(n_apps) < 0.6, rng.random(n_apps) * 8.0, np.inf),  # cap
                        rng.random(n_apps) * 0.01,                       # sigma
                        rng.random(n_apps) * 1.2], 1)                    # throttle threshold
    return dict(app_pipe_off=np.concatenate([[0], np.cumsum(pipes)]).astype(np.uint64),
                pipe_slot_off=np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64),
                slot_shader=rng.integers(0, n_sh, n_slots).astype(np.uint32),
                slot_frac=frac,
                pipe_wt=np.stack([rng.random(npipe) * 1.5 + 0.5, (rng.random(npipe) * 6 + 2) * 1e-3], 1),
                shader_lat=lat, app_f64=app_f64), rng.integers(0, 2, n_sh).astype(np.uint8)


@pytest.mark.parametrize("seed,n_apps", [(1, 1), (2, 3), (3, 97), (4, 1030)])
def test_aggregate_ragged_suites_match_oracle(dev, orc, seed, n_apps):
    """K3 (several apps folded per warp, speculative single pass per pipeline,
    re-run for throttled apps) against the oracle's frame_time / run_benchmark
    / evaluate rows (simenv.cpp:439-510, tuner.cpp:276-291), bit for bit."""
    s, act = _ragged_suite(seed, n_apps)
    run_seed = np.array([orc.derive_seed(seed, 0x45564C, b) for b in range(n_apps)], np.uint64)
    rows_o, smp_o = orc.aggregate(s, act, run_seed, 10, want_samples=True)
    rows, smp = dev.aggregate(s, act, run_seed, 10, want_samples=True)
    throttled = np.isfinite(s["app_f64"][:, 1])
    assert n_apps < 50 or throttled.any()
    np.testing.assert_array_equal(rows, rows_o)
    np.testing.assert_array_equal(smp, smp_o)


@pytest.mark.parametrize("uplift", [[3.0], [-2.5, -2.5], [0.0, 1.0, 2.0], [-7.3, 0.2, 12.9, 12.0]])
def test_histogram_edges(dev, orc, uplift):
    lo, cnt = dev.histogram(uplift)
    lo_o, cnt_o = orc.histogram(uplift)
    np.testing.assert_array_equal(lo, lo_o)
    np.testing.assert_array_equal(cnt, cnt_o)


# ------------------------------------------------------- data-parallel path
@pytest.mark.parametrize("batch", [64, 4096])
def test_fit_data_parallel_step_path(orc, batch):
    """One-rank NCCL communicator: fit runs the DP step sequence (per-CTA
    partials -> fixed-tree reduce -> ncclAllReduce -> SGD update kernel)."""
    d = gbx.Device(0)
    d.comm_init(gbx.Device.comm_unique_id(), 1, 0)
    f, t = orc.g1(23, 20_000)
    p0 = orc.policy_init(4)
    rc, p_ref, el_ref, _ = orc.fit(p0, f, t, 0.01, 2, batch, 8)
    p, el = d.fit(p0, f, t, 0.01, 2, batch, 8)
    assert ulps32(p, p_ref).max() <= 2
    np.testing.assert_allclose(el, el_ref, rtol=1e-12)
    d.comm_destroy()
    d.close()


# ------------------------------------------- fused peer-set (multi-GPU) path
@pytest.mark.parametrize("vranks,batch", [(2, 4096), (4, 8192), (8, 8192), (3, 1000)])
def test_fit_peer_set_virtual_ranks(dev, orc, vranks, batch):
    """The multi-GPU kernel path (reduce-scatter over every rank's CTAs through
    peer-memory partials, arrival counters on every rank, LL parameter words
    written to every rank) run with `vranks` virtual ranks inside one launch:
    same tolerance against the reference as the 1-GPU path, deterministic."""
    n = 50_003
    f, t = orc.g1(19, n)
    p0 = orc.policy_init(13)
    rc, p_ref, el_ref, _ = orc.fit(p0, f, t, 0.02, 2, batch, 6)
    p, el = dev.fit(p0, f, t, 0.02, 2, batch, 6, virtual_ranks=vranks)
    assert ulps32(p, p_ref).max() <= 2
    np.testing.assert_allclose(el, el_ref, rtol=1e-12)
    p2, el2 = dev.fit(p0, f, t, 0.02, 2, batch, 6, virtual_ranks=vranks)
    np.testing.assert_array_equal(p, p2)
    np.testing.assert_array_equal(el, el2)


def test_fit_peer_set_divergence_agrees(dev, orc):
    f, t = orc.g1(6, 4096)
    f[:, 8:] *= np.float32(1e3)
    p0 = orc.policy_init(5)
    rc, p_ref, el_ref, ep_ref = orc.fit(p0, f, t, 1e12, 4, 512, 1)
    assert rc == 2
    with pytest.raises(gbx.TrainingDivergedError) as ei:
        dev.fit(p0, f, t, 1e12, 4, 512, 1, virtual_ranks=4)
    assert ei.value.epoch == ep_ref
    # the net holds the weights after the last finite step, as the reference's
    # does when fit throws (policy.cpp:321-325) — not the start of the epoch
    pe = ei.value.params
    both = np.isfinite(pe) & np.isfinite(p_ref)
    same = (np.isnan(pe) & np.isnan(p_ref)) | (pe == p_ref)
    same[both] |= ulps32(pe[both], p_ref[both]) <= 2
    assert same.mean() > 0.99
    assert not np.array_equal(p_ref, p0) or np.array_equal(pe, p0)
    # the context stays usable (monotonic counters / tags resynchronised)
    f2, t2 = orc.g1(7, 20_000)
    rc, p_ref2, _, _ = orc.fit(p0, f2, t2, 0.01, 1, 2048, 3)
    p2, _ = dev.fit(p0, f2, t2, 0.01, 1, 2048, 3, virtual_ranks=4)
    assert ulps32(p2, p_ref2).max() <= 2


def test_suite_upload_from_device_memory(dev, orc):
    """gbxcu_suite_upload accepts device-resident arrays (unified addressing):
    same evaluate rows as the host upload of the same suite."""
    import torch
    s = dict(golden("suite_free"))
    keys = ("app_pipe_off", "pipe_slot_off", "slot_shader", "slot_frac", "pipe_wt", "shader_lat",
            "app_f64")
    ds_h = dev.suite_upload(s, s["features"])
    rows_h, hist_h, act_h = ds_h.evaluate(s["eval_params"], 10, int(s["eval_seed"]), want_actions=True)
    t = {k: torch.from_numpy(np.ascontiguousarray(s[k])).cuda() for k in keys}
    ds_d = dev.suite_upload_dev(t, torch.from_numpy(np.ascontiguousarray(s["features"], np.float32)).cuda())
    rows_d, hist_d, act_d = ds_d.evaluate(s["eval_params"], 10, int(s["eval_seed"]), want_actions=True)
    np.testing.assert_array_equal(rows_d, rows_h)
    np.testing.assert_array_equal(act_d, act_h)
    ds_h.close()
    ds_d.close()


@pytest.mark.parametrize("vranks", [2, 5])
def test_fit_peer_set_multi_epoch_many_tiles(dev, orc, vranks):
    """Virtual-rank peer set with several tiles per CTA per step and several
    epochs (tags and counters continue across epoch launches)."""
    n = 40_003
    f, t = orc.g1(29, n)
    p0 = orc.policy_init(3)
    rc, p_ref, el_ref, _ = orc.fit(p0, f, t, 0.02, 3, 20_000, 12)
    p, el = dev.fit(p0, f, t, 0.02, 3, 20_000, 12, virtual_ranks=vranks)
    assert ulps32(p, p_ref).max() <= 2
    np.testing.assert_allclose(el, el_ref, rtol=1e-12)


@pytest.mark.parametrize("name", ["suite_free", "suite_contended"])
def test_evaluate_shards_reassemble_bit_exact(dev, orc, name):
    """aggregation sharded by app range — concatenated shard rows
    equal evaluate()'s, and so does the histogram built from them."""
    s = dict(golden(name))
    ds = dev.suite_upload(s, s["features"])
    rows, (lo, cnt) = ds.evaluate(s["eval_params"], 10, int(s["eval_seed"]))
    na = ds.n_apps
    for cuts in ([0, na], [0, na // 3, na], [0, 1, na // 2, na - 1, na]):
        parts = [ds.evaluate_shard(s["eval_params"], 10, int(s["eval_seed"]), a, b)
                 for a, b in zip(cuts[:-1], cuts[1:])]
        got = np.concatenate(parts)
        np.testing.assert_array_equal(got, rows)
        lo2, cnt2 = dev.histogram(got[:, 3])
        np.testing.assert_array_equal(lo2, lo)
        np.testing.assert_array_equal(cnt2, cnt)
    assert ds.evaluate_shard(s["eval_params"], 10, 1, 2, 2).shape == (0, 5)
    with pytest.raises(gbx.ValidationError):
        ds.evaluate_shard(s["eval_params"], 10, 1, 0, na + 1)
    ds.close()


@pytest.mark.parametrize("world", [2, 3])
def test_evaluate_distributed_across_processes(world):
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "shard_eval_probe.py"),
                        str(world)], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


def test_bench_c5_sharded_collectives():
    """bench.py's sharded-C5 secondary (run on N>1 ranks) driven by 2 processes
    over gloo on one GPU: collectives complete and every app's row is gathered."""
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "c5_sharded_probe.py"), "2"],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
