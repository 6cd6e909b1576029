"""GPU parity of the TD-regression loss and the Adam update on the fused
tensor-core train kernel (k_train_tc.cu) against the oracle restatement
(oracle/gbx_oracle.c:orc_fit_variant, pinned in test_oracle_variants.py).

The variants always run on the fused kernel (DMMA partial sums, fixed
cross-CTA association), never on the bit-exact 1-CTA kernel, so the tolerance
is the multi-CTA one: <= 2 fp32 ulp per weight after the fit; epoch losses
relative 1e-12. Adam's bias corrections use the device pow (<= 1 ulp fp64 of
glibc's), covered by the same bound.
"""
import numpy as np
import pytest

import paper_2111_12055_b200 as gbx
from test_oracle_variants import td_data, ulps32

pytestmark = pytest.mark.gpu

CASES = [("td", "sgd"), ("kl", "adam"), ("td", "adam")]


def data(orc, loss, seed, n):
    return td_data(orc, seed, n) if loss == "td" else orc.g1(seed, n)


@pytest.mark.parametrize("loss,opt", CASES)
@pytest.mark.parametrize("batch,max_ctas", [(32, 0), (1000, 3), (4096, 0)])
def test_variant_fit_matches_oracle(dev, orc, loss, opt, batch, max_ctas):
    n = 20_011
    f, t = data(orc, loss, 17, n)
    p0 = orc.policy_init(21)
    lr = 1e-3 if opt == "adam" else 0.01
    epochs = 2
    rc, p_ref, el_ref, _ = orc.fit_variant(p0, f, t, lr, epochs, batch, 4, loss=loss, optimizer=opt)
    assert rc == 0
    p, el = dev.fit(p0, f, t, lr, epochs, batch, 4, max_ctas=max_ctas, loss=loss, optimizer=opt)
    u = ulps32(p, p_ref)
    assert u.max() <= 2, (u.max(), int((u > 0).sum()))
    np.testing.assert_allclose(el, el_ref, rtol=1e-12)
    p2, el2 = dev.fit(p0, f, t, lr, epochs, batch, 4, max_ctas=max_ctas, loss=loss, optimizer=opt)
    np.testing.assert_array_equal(p, p2)  # deterministic
    np.testing.assert_array_equal(el, el2)


@pytest.mark.parametrize("loss,opt", [("td", "adam"), ("kl", "adam")])
def test_variant_peer_set_virtual_ranks(dev, orc, loss, opt):
    """Adam moments owned slice-wise by the CTAs of every rank of the set."""
    f, t = data(orc, loss, 5, 30_000)
    p0 = orc.policy_init(3)
    rc, p_ref, el_ref, _ = orc.fit_variant(p0, f, t, 1e-3, 2, 8192, 9, loss=loss, optimizer=opt)
    p, el = dev.fit(p0, f, t, 1e-3, 2, 8192, 9, virtual_ranks=4, loss=loss, optimizer=opt)
    assert ulps32(p, p_ref).max() <= 2
    np.testing.assert_allclose(el, el_ref, rtol=1e-12)


def test_variant_adam_moments_reset_per_fit(dev, orc):
    f, t = data(orc, "td", 8, 3000)
    p0 = orc.policy_init(2)
    a, _ = dev.fit(p0, f, t, 1e-3, 1, 256, 1, loss="td", optimizer="adam")
    dev.fit(p0, f, t, 1e-3, 3, 256, 7, loss="td", optimizer="adam")
    b, _ = dev.fit(p0, f, t, 1e-3, 1, 256, 1, loss="td", optimizer="adam")
    np.testing.assert_array_equal(a, b)


def test_variant_td_learns(dev, orc):
    f, t = data(orc, "td", 2, 50_000)
    p, el = dev.fit(orc.policy_init(1), f, t, 1e-3, 5, 1024, 3, loss="td", optimizer="adam")
    assert el[-1] < 0.7 * el[0]


def test_variant_divergence(dev, orc):
    f, t = data(orc, "td", 6, 512)
    t[:, 1] *= 1e300
    p0 = orc.policy_init(5)
    rc, _, _, ep_ref = orc.fit_variant(p0, f, t, 0.5, 3, 64, 1, loss="td")
    assert rc == 2
    with pytest.raises(gbx.TrainingDivergedError) as ei:
        dev.fit(p0, f, t, 0.5, 3, 64, 1, loss="td")
    assert ei.value.epoch == ep_ref


def test_variant_validation(dev, orc):
    f, t = orc.g1(1, 64)
    p = orc.policy_init(1)
    with pytest.raises(ValueError):
        dev.fit(p, f, t, loss="huber")
    with pytest.raises(gbx.ValidationError):
        dev.fit(p, f, t, optimizer="adam", betas=(1.0, 0.999))


@pytest.mark.parametrize("n,batch", [(1, 32), (7, 32), (33, 32), (100, 1000), (1500, 64)])
def test_variant_ragged_sizes(dev, orc, n, batch):
    """Edge sizes through the lone-CTA and multi-CTA variant paths: a single
    record, a partial last batch, n below the batch size."""
    for loss, opt in CASES:
        f, t = data(orc, loss, 40 + n, n)
        p0 = orc.policy_init(6)
        lr = 1e-3 if opt == "adam" else 0.01
        rc, p_ref, el_ref, _ = orc.fit_variant(p0, f, t, lr, 3, batch, 2, loss=loss, optimizer=opt)
        assert rc == 0
        p, el = dev.fit(p0, f, t, lr, 3, batch, 2, loss=loss, optimizer=opt)
        assert ulps32(p, p_ref).max() <= 2, (loss, opt)
        np.testing.assert_allclose(el, el_ref, rtol=1e-12)
