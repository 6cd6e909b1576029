"""The north star's TD-regression loss and Adam update (absent from the
reference: parity unpinned by it). The oracle restatement
(oracle/gbx_oracle.c:orc_fit_variant) is pinned here against
  * its own KL + SGD mode == the reference's fit restatement (bit-exact);
  * an independent fp64 torch autograd computation of one full-batch step
    (TD + SGD, KL + Adam, TD + Adam): <= 1 fp32 ulp per weight (summation
    order of the gradient differs, ~1e-16 relative).
"""
import numpy as np
import pytest
import torch

DIMS = (44, 64, 32, 2)


def ulps32(a, b):
    a = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64)
    return np.abs(a - b)


def td_data(orc, seed, n):
    f, _ = orc.g1(seed, n)
    rng = np.random.default_rng(seed)
    act = rng.integers(0, 2, n).astype(np.float64)
    rew = rng.normal(0.5, 1.0, n) + 0.3 * f[:, 0].astype(np.float64) * (2 * act - 1)
    return f, np.stack([act, rew], 1)


def torch_grad(params, feat, tgt, loss):
    """Full-batch gradient in fp64 (param layout: per layer W[out][in] then b)."""
    w = torch.tensor(params.astype(np.float64), requires_grad=True)
    x = torch.tensor(feat.astype(np.float64))
    h, o = x, 0
    for li in range(3):
        i, j = DIMS[li], DIMS[li + 1]
        W = w[o:o + i * j].view(j, i)
        o += i * j
        b = w[o:o + j]
        o += j
        h = h @ W.T + b
        if li < 2:
            h = torch.relu(h)
    t = torch.tensor(tgt)
    if loss == "td":
        a = t[:, 0].long()
        q = h.gather(1, a[:, None])[:, 0]
        L = ((q - t[:, 1]) ** 2).mean()
    else:
        lp = torch.log_softmax(h, 1).clamp(np.log(1e-7), np.log1p(-1e-7))
        p = lp.exp()
        L = (p * (lp - torch.log(t.clamp(1e-7, 1 - 1e-7)))).sum(1).mean()
    L.backward()
    return w.grad.numpy(), float(L.detach())


def test_kl_sgd_mode_is_fit(orc):
    f, t = orc.g1(3, 700)
    p0 = orc.policy_init(9)
    rc, p_ref, el_ref, _ = orc.fit(p0, f, t, 0.02, 3, 32, 5)
    rc2, p, el, _ = orc.fit_variant(p0, f, t, 0.02, 3, 32, 5)
    assert rc == rc2 == 0
    np.testing.assert_array_equal(p, p_ref)
    np.testing.assert_array_equal(el, el_ref)


@pytest.mark.parametrize("loss,opt", [("td", "sgd"), ("kl", "adam"), ("td", "adam")])
def test_one_full_batch_step_vs_autograd(orc, loss, opt):
    n = 300
    if loss == "td":
        f, t = td_data(orc, 11, n)
    else:
        f, t = orc.g1(11, n)
    p0 = orc.policy_init(4)
    lr = 0.01
    rc, p, el, _ = orc.fit_variant(p0, f, t, lr, 1, n, 2, loss=loss, optimizer=opt)
    assert rc == 0
    g, L = torch_grad(p0, f, t, loss)
    w0 = p0.astype(np.float64)
    if opt == "sgd":
        want = (w0 - lr * g).astype(np.float32)
    else:
        b1, b2, eps = 0.9, 0.999, 1e-8
        m, v = (1 - b1) * g, (1 - b2) * g * g
        want = (w0 - lr * (m / (1 - b1)) / (np.sqrt(v / (1 - b2)) + eps)).astype(np.float32)
    assert ulps32(p, want).max() <= 1
    np.testing.assert_allclose(el[0], L, rtol=1e-12)


def test_adam_first_step_is_signed_lr(orc):
    """Adam's first update is lr * g / (|g| + eps): every weight with a
    non-negligible gradient moves by ~lr."""
    f, t = orc.g1(5, 256)
    p0 = orc.policy_init(8)
    rc, p, _, _ = orc.fit_variant(p0, f, t, 1e-3, 1, 256, 0, optimizer="adam")
    g, _ = torch_grad(p0, f, t, "kl")
    big = np.abs(g) > 1e-4
    d = p.astype(np.float64) - p0.astype(np.float64)
    np.testing.assert_allclose(np.abs(d[big]), 1e-3, rtol=1e-3)
    assert (np.sign(d[big]) == -np.sign(g[big])).all()


def test_td_adam_learns(orc):
    f, t = td_data(orc, 2, 4000)
    p0 = orc.policy_init(1)
    rc, p, el, _ = orc.fit_variant(p0, f, t, 1e-3, 4, 64, 3, loss="td", optimizer="adam")
    assert rc == 0 and el[-1] < 0.7 * el[0]
