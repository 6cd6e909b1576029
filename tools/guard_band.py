"""Share of states a rigorous guard sends to the exact re-check, for the fp32
FFMA bound (as in k_forward.cu) and for hypothetical TF32 / 3xTF32 tensor-core
forwards, on the init net and a bench-trained net (CPU, numpy + the oracle).

The 3xTF32 bound assumes exact tf32 products, split error 2^-20 per term and
fp32 accumulation with <= 2^-22 relative error per add over 3K terms; plain
TF32 assumes operand truncation (2^-10 each). Usage: python tools/guard_band.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
from bench import synthetic_log  # noqa: E402


def layers(p):
    p = p.astype(np.float64)
    return (p[:2816].reshape(64, 44), p[2816:2880], p[2880:4928].reshape(32, 64), p[4928:4960],
            p[4960:5024].reshape(2, 32), p[5024:])


def main():
    o = oracle.Restatement()
    f, t = synthetic_log(200_000)
    p0 = o.policy_init(7)
    _, p1, _, _ = o.fit(p0, f, t, 0.01, 2, 8192, 99)
    u = 2.0 ** -24
    for name, p in (("init", p0), ("trained", p1)):
        W0, b0, W1, b1, W2, b2 = layers(p)
        x = f.astype(np.float64)
        h1 = np.maximum(x @ W0.T + b0, 0)
        h2 = np.maximum(h1 @ W1.T + b1, 0)
        l = h2 @ W2.T + b2
        d = np.abs(l[:, 1] - l[:, 0])
        R0, R1, R2 = (np.abs(W).sum(1).max() for W in (W0, W1, W2))
        B0, B1, B2 = (np.abs(b).max() for b in (b0, b1, b2))
        Rd = np.abs(W2[1] - W2[0]).sum()
        X, H1, H2 = np.abs(x).max(1), h1.max(1), h2.max(1)
        X1, H1s = np.abs(x).sum(1), h1.sum(1)
        W0m, W1m = np.abs(W0).max(), np.abs(W1).max()

        def band(g1, g2, g3):  # k_forward.cu guard_threshold's form
            D1 = g1 * (B0 + np.minimum(R0 * X, W0m * X1))
            D2 = g2 * (B1 + np.minimum(R1 * H1, W1m * H1s)) + R1 * D1
            return 1.02 * (2 * g3 * (B2 + R2 * H2) + Rd * D2)

        rows = {"fp32 FFMA (k_forward.cu)": band(14 * u, 65 * u, 33 * u),
                "3xTF32 tensor cores": band(146 * 2.0 ** -22, 194 * 2.0 ** -22, 33 * u),
                "TF32 tensor cores": band(2.0 ** -9, 2.0 ** -9, 33 * u)}
        print(f"{name}: median |l1 - l0| = {np.median(d):.4g}")
        for k, T in rows.items():
            print(f"   {k:28s} re-checked {np.mean(d <= T):8.4%}")


if __name__ == "__main__":
    main()
