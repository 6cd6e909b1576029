"""Parity AT THE BENCHMARKED SIZES, against the compiled reference.

tests/golden/at_size.npz was written by oracle/make_golden_size.py from the
unmodified reference library (fit, proj/src/policy.cpp:297-337;
select_greedy, :339-342). The inputs are regenerated here from the same seeds
and checked by checksum first, so a data mismatch can never pass as parity.

Tolerances (module docstring of test_gpu_parity.py): weights <= 2 fp32 ulp
for multi-CTA steps (fp64 re-association; <= 1 for the 1-CTA batch-32 kernel),
epoch loss relative 1e-12, actions bit-exact, per-app rows bit-exact.
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


@pytest.fixture(scope="module")
def g():
    return golden("at_size")


@pytest.fixture(scope="module")
def c2_log(g, orc):
    import bench
    feat, tgt = bench.synthetic_log(1_000_000)
    assert orc.fnv1a(feat) == int(g["c2_feat_fnv"]) and orc.fnv1a(tgt) == int(g["c2_tgt_fnv"])
    return feat, tgt


def test_c2_headline_epoch_matches_reference(dev, orc, g, c2_log):
    """The bench's step (1M records, batch 8192, one epoch) through the host
    API and through the device-pointer call the bench times."""
    import torch
    feat, tgt = c2_log
    p0 = orc.policy_init(7)
    p, el = dev.fit(p0, feat, tgt, 0.01, 1, 8192, 99)
    assert ulps32(p, g["c2_params"]).max() <= 2
    np.testing.assert_allclose(el, g["c2_loss"], rtol=1e-12)
    fd, td = torch.from_numpy(feat).cuda(), torch.from_numpy(tgt).cuda()
    pd = torch.from_numpy(p0).cuda()
    torch.cuda.synchronize()
    el2 = dev.fit_dev(pd.data_ptr(), fd.data_ptr(), td.data_ptr(), feat.shape[0], 0.01, 1, 8192, 99,
                      stream=dev.stream)
    assert ulps32(pd.cpu().numpy(), g["c2_params"]).max() <= 2
    np.testing.assert_allclose(el2, g["c2_loss"], rtol=1e-12)


def test_c2_batch32_epoch_matches_reference(dev, orc, g, c2_log):
    """The reference default batch at C2's size: 31,250 dependent SGD steps on
    the 1-CTA kernel in the reference's summation order."""
    feat, tgt = c2_log
    p, el = dev.fit(orc.policy_init(7), feat, tgt, 0.01, 1, 32, 99)
    assert ulps32(p, g["c2b32_params"]).max() <= 1
    np.testing.assert_allclose(el, g["c2b32_loss"], rtol=1e-12)


@pytest.mark.parametrize("mode", [gbx.FWD_FAST, gbx.FWD_EXACT])
def test_c2_inference_at_size_matches_reference(dev, orc, g, c2_log, mode):
    """Greedy decisions over all 1M headline states under the trained net:
    bit-exact against the reference's select_greedy (checksum of all 1M)."""
    feat, _ = c2_log
    _, act = dev.forward(g["c2_params"], feat, mode, want_probs=False)
    np.testing.assert_array_equal(act[:4096], g["c2inf_act_head"])
    assert int(act.sum()) == int(g["c2inf_wave64"])
    assert orc.fnv1a(act) == int(g["c2inf_act_fnv"])


@pytest.fixture(scope="module")
def c3_log(g, orc):
    feat, tgt = orc.g1(3, 10_000_000)
    assert orc.fnv1a(feat) == int(g["c3_feat_fnv"]) and orc.fnv1a(tgt) == int(g["c3_tgt_fnv"])
    return feat, tgt


@pytest.mark.parametrize("vranks", [1, 8])
def test_c3_epoch_matches_reference(dev, orc, g, c3_log, vranks):
    """C3 at its full size: 10M records, global batch 65,536, one epoch —
    on one GPU (148 CTAs) and as the 8-GPU decomposition (8 virtual ranks x
    8,192 records per step, each rank's own exchange region)."""
    import torch
    feat, tgt = c3_log
    fd, td = torch.from_numpy(feat).cuda(), torch.from_numpy(tgt).cuda()
    pd = torch.from_numpy(orc.policy_init(7)).cuda()
    torch.cuda.synchronize()
    el = dev.fit_dev(pd.data_ptr(), fd.data_ptr(), td.data_ptr(), feat.shape[0], 0.01, 1, 65536, 5,
                     stream=dev.stream, virtual_ranks=vranks if vranks > 1 else 0)
    assert ulps32(pd.cpu().numpy(), g["c3_params"]).max() <= 2
    np.testing.assert_allclose(el, g["c3_loss"], rtol=1e-12)
    del fd, td
    torch.cuda.empty_cache()


def _sub_suite(s, apps, seed):
    """The CSR slices of `apps` (host numpy), re-based, with their shaders
    compacted, plus evaluate's per-app run seeds (tuner.cpp:280-281)."""
    apo, pso = s["app_pipe_off"], s["pipe_slot_off"]
    a_off, p_off, slots, pipes = [0], [0], [], []
    for b in apps:
        p_lo, p_hi = int(apo[b]), int(apo[b + 1])
        for p in range(p_lo, p_hi):
            slots.append(np.arange(int(pso[p]), int(pso[p + 1])))
            p_off.append(p_off[-1] + int(pso[p + 1] - pso[p]))
            pipes.append(p)
        a_off.append(a_off[-1] + (p_hi - p_lo))
    slots = np.concatenate(slots)
    shaders = s["slot_shader"][slots].astype(np.int64)
    uniq, inv = np.unique(shaders, return_inverse=True)
    sub = dict(app_pipe_off=np.array(a_off, np.uint64), pipe_slot_off=np.array(p_off, np.uint64),
               slot_shader=inv.astype(np.uint32), slot_frac=s["slot_frac"][slots],
               pipe_wt=s["pipe_wt"][pipes], shader_lat=s["shader_lat"][uniq],
               app_f64=s["app_f64"][apps])
    return sub, uniq


def test_c5_sampled_apps_match_oracle(dev, orc):
    """C5 at its nominal size (1e8 shaders / 1e4 apps, generated on the
    device): for 128 apps (first, last and a random sample) the device's
    greedy actions equal the oracle's fp64 select_greedy on every shader of
    the app, and the device's per-app rows equal the oracle's frame_time /
    run_benchmark / evaluate rows (simenv.cpp:439-510, tuner.cpp:276-291)
    bit for bit, computed from the app's own CSR slice."""
    import torch
    import bench
    n_apps, per_app, seed = 10_000, 10_000, 77
    s, feat = bench.synthetic_suite_torch(torch, n_apps, per_app)
    ds = dev.suite_upload_dev(s, feat)
    params = golden("forward_g1")["params_trained"]
    pd = torch.from_numpy(params).cuda()
    act = torch.empty(ds.n_shaders, dtype=torch.uint8, device="cuda")
    rows = torch.empty((ds.n_apps, 5), dtype=torch.float64, device="cuda")
    ds.evaluate_dev(pd.data_ptr(), 10, seed, act.data_ptr(), rows.data_ptr())
    torch.cuda.synchronize()
    rows = rows.cpu().numpy()
    rng = np.random.default_rng(11)
    apps = np.unique(np.concatenate([[0, n_apps - 1], rng.choice(n_apps, 126, replace=False)]))
    host = {k: v.cpu().numpy() for k, v in s.items()}
    sub, shaders = _sub_suite(host, apps, seed)
    f_sub = feat[torch.from_numpy(shaders).cuda()].cpu().numpy()
    _, act_o = orc.forward(params, f_sub)
    np.testing.assert_array_equal(act[torch.from_numpy(shaders).cuda()].cpu().numpy(), act_o)
    run_seed = np.array([orc.derive_seed(seed, 0x45564C, int(b)) for b in apps], np.uint64)
    rows_o = orc.aggregate(sub, act_o, run_seed, 10, app_ids=apps)
    np.testing.assert_array_equal(rows[apps], rows_o)
    ds.close()
    del s, feat, host
    torch.cuda.empty_cache()
