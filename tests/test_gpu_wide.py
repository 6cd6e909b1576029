"""GPU tests of the wide-MLP variant (BASELINE.json C4: 44 -> 512 -> 512 -> 2)
on the tcgen05 TF32 path, against numpy (GEMM) and the generic-dims oracle
restatement (forward, fit). The reference hard-codes 44-64-32-2, so this is
"parity unpinned" by the reference; the oracle follows the reference's
algorithm generalised over widths (oracle/gbx_oracle.c).

Tolerances (TF32 operands are truncated to 10 mantissa bits, fp32 accumulation):
  * GEMM: |D - trunc(A) trunc(B)^T| <= 2e-6 * sum|a||b| (accumulation only);
  * init: bit-exact;
  * forward probabilities: |dp| <= 3e-3;
  * fit: max |dw| <= 3% of the largest weight change the oracle makes over the
    run; epoch losses within 1% relative.
"""
import numpy as np
import pytest

from conftest import golden  # noqa: F401

pytestmark = pytest.mark.gpu
H = 512
DIMS = (44, H, H, 2)


def trunc(x):
    return (np.ascontiguousarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (300, 200, 100), (1000, 512, 44), (512, 48, 1000),
                                   (77, 33, 8), (4100, 130, 516)])
def test_tf32_gemm_matches_truncated_model(dev, M, N, K):
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    D = dev.tf32_gemm(A, B).astype(np.float64)
    ref = trunc(A).astype(np.float64) @ trunc(B).astype(np.float64).T
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    assert np.max(np.abs(D - ref) / scale) <= 2e-6


def test_wide_init_bit_exact(dev, orc):
    for seed in (0, 7, 99):
        np.testing.assert_array_equal(dev.wide_init(H, seed), orc.policy_init(seed, DIMS))


def test_wide_forward_within_tf32_tolerance(dev, orc):
    feat, _ = orc.g1(42, 3000)
    p = orc.policy_init(7, DIMS)
    probs = dev.wide_forward(H, p, feat)
    ref, _ = orc.forward(p, feat, DIMS)
    assert np.abs(probs - ref).max() <= 3e-3
    np.testing.assert_allclose(probs.sum(1), 1.0, atol=1e-12)


@pytest.mark.parametrize("n,batch,epochs", [(2048, 256, 1), (3000, 512, 2), (777, 100, 1)])
def test_wide_fit_tracks_oracle(dev, orc, n, batch, epochs):
    feat, tgt = orc.g1(42, n)
    p0 = orc.policy_init(7, DIMS)
    rc, p_ref, el_ref, _ = orc.fit(p0, feat, tgt, 0.01, epochs, batch, 5, dims=DIMS)
    assert rc == 0
    p, el = dev.wide_fit(H, p0, feat, tgt, 0.01, epochs, batch, 5)
    change = np.abs(p_ref.astype(np.float64) - p0).max()
    assert np.abs(p.astype(np.float64) - p_ref).max() <= 0.03 * change
    np.testing.assert_allclose(el, el_ref, rtol=1e-2)
    p2, el2 = dev.wide_fit(H, p0, feat, tgt, 0.01, epochs, batch, 5)
    np.testing.assert_array_equal(p, p2)   # deterministic
    np.testing.assert_array_equal(el, el2)


def test_wide_data_parallel_path(orc):
    import paper_2111_12055_b200 as gbx

    d = gbx.Device(0)
    d.comm_init(gbx.Device.comm_unique_id(), 1, 0)
    feat, tgt = orc.g1(3, 1024)
    p0 = orc.policy_init(11, DIMS)
    rc, p_ref, el_ref, _ = orc.fit(p0, feat, tgt, 0.01, 1, 256, 2, dims=DIMS)
    p, el = d.wide_fit(H, p0, feat, tgt, 0.01, 1, 256, 2)
    change = np.abs(p_ref.astype(np.float64) - p0).max()
    assert np.abs(p.astype(np.float64) - p_ref).max() <= 0.03 * change
    d.comm_destroy()
    d.close()
