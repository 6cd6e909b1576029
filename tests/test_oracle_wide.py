"""CPU: the wide-MLP numerics model (oracle/wide_emul.py) with its BF16
rounding points switched off is the reference's fp64 fit (the C restatement
generalised over widths, oracle/gbx_oracle.c), bit for bit — so the model
adds only the rounding points the GPU tests grade against."""
import numpy as np

from oracle import wide_emul as W


def test_wide_model_without_rounding_is_the_restatement(orc):
    h, n, batch, epochs = 64, 900, 128, 2
    dims = (44, h, h, 2)
    feat, tgt = orc.g1(42, n)
    p0 = orc.policy_init(7, dims)
    rc, p_ref, el_ref, _ = orc.fit(p0, feat, tgt, 0.01, epochs, batch, 5, dims=dims)
    assert rc == 0
    orders = [orc.fit_order(n, 5, e + 1) for e in range(epochs)]
    p, el = W.fit(p0, feat, tgt, orders, 0.01, epochs, batch, h, emulate=False)
    np.testing.assert_array_equal(p, p_ref)
    np.testing.assert_allclose(el, el_ref, rtol=1e-15)


def test_bf16_rounding_is_round_to_nearest_even():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 2 ** -7 + 2 ** -8, -3.5, 0.0, 1.0 + 2 ** -8 + 2 ** -20],
                 np.float32)
    np.testing.assert_array_equal(W.bf16(x), np.array([1.0, 1.0, 1.0 + 2 ** -6, -3.5, 0.0, 1.0 + 2 ** -7],
                                                      np.float32))
