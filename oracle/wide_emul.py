"""Wide-MLP (C4) numerics model — TEST INFRASTRUCTURE ONLY.

A numpy restatement of one fit step of the 44 -> H -> H -> 2 policy (fit,
run_forward, accumulate_gradient generalised over widths: proj/src/policy.cpp
:29-55 forward, :209-279 gradient, :297-337 fit's SGD step, the same
algorithm oracle/gbx_oracle.c restates for any dims) that places the device's
BF16 rounding points explicitly (paper_2111_12055_b200/csrc/k_wide16.cu):

  * GEMM operands rounded to bf16 (round to nearest even): the gathered
    features, W0, W1, and the activations H1, D2, D1 between the GEMMs;
  * GEMM accumulators rounded to fp32 once (the tensor core's fp32
    accumulation order is not modelled: that difference is what the tests'
    tolerance covers), biases added in fp32, relu;
  * the head (logits, softmax, KL, d3) in fp64 like the reference; D2 =
    (fp32(d3_0) w2_0 + fp32(d3_1) w2_1) [h2 > 0] in fp32; gW2, gb1, gb2, the
    loss and the split-K gradient sums in fp64 (the device's fp32 partial
    column sums are inside the tests' tolerance);
  * SGD w = float(double(w) - lr g).

With emulate=False every rounding point is the identity and the model is the
reference's fp64 algorithm: tests pin it there against the C restatement
(orc.fit with dims), so the rounding points are the only thing it adds.
"""
from __future__ import annotations

import numpy as np

F = 44


def bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as fp32 (finite inputs)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def unpack(params, H):
    p = np.asarray(params, np.float32)
    o = 0
    w0 = p[o:o + H * F].reshape(H, F); o += H * F
    b0 = p[o:o + H]; o += H
    w1 = p[o:o + H * H].reshape(H, H); o += H * H
    b1 = p[o:o + H]; o += H
    w2 = p[o:o + 2 * H].reshape(2, H); o += 2 * H
    b2 = p[o:o + 2]
    return w0, b0, w1, b1, w2, b2


def step(params, feat, tgt, rows, nb, lr, H, emulate=True):
    """One SGD step on records `rows` of a global batch of nb. Returns
    (new params fp32, KL sum over the rows, gradient fp64)."""
    r16 = bf16 if emulate else (lambda a: np.asarray(a, np.float64))
    f32 = (lambda a: np.asarray(a, np.float32)) if emulate else (lambda a: np.asarray(a, np.float64))
    w0, b0, w1, b1, w2, b2 = unpack(params, H)
    X = np.asarray(feat, np.float32)[rows]
    Xb = r16(X).astype(np.float64)
    acc1 = f32(Xb @ r16(w0).astype(np.float64).T)
    h1 = np.maximum(f32(acc1 + (b0 if emulate else b0.astype(np.float64))), 0)
    H1 = r16(h1).astype(np.float64)
    acc2 = f32(H1 @ r16(w1).astype(np.float64).T)
    h2 = np.maximum(f32(acc2 + (b1 if emulate else b1.astype(np.float64))), 0).astype(np.float64)
    z = b2.astype(np.float64)[None, :] + h2 @ w2.astype(np.float64).T
    m = z.max(1, keepdims=True)
    e = np.exp(z - m)
    p = e / e.sum(1, keepdims=True)
    t = np.asarray(tgt, np.float64)[rows]
    pc, tc = np.clip(p, 1e-7, 1 - 1e-7), np.clip(t, 1e-7, 1 - 1e-7)
    lr_ = np.log(pc / tc)
    loss = (pc * lr_).sum(1)
    d3 = p * (lr_ - loss[:, None]) / nb
    if emulate:  # fp32: fp32(d3_0) w2_0 + fp32(d3_1) w2_1, products and sum each rounded
        d3f = d3.astype(np.float32)
        d2 = np.where(h2 > 0, d3f[:, :1] * w2[0][None, :] + d3f[:, 1:] * w2[1][None, :], 0).astype(np.float64)
    else:
        d2 = np.where(h2 > 0, d3 @ w2.astype(np.float64), 0)
    D2 = r16(d2).astype(np.float64)
    acc3 = f32(D2 @ r16(w1).astype(np.float64))
    d1 = np.where(H1 > 0, acc3, 0)
    D1 = r16(d1).astype(np.float64)
    g_w0 = D1.T @ Xb
    g_b0 = D1.sum(0)
    g_w1 = D2.T @ H1
    g_b1 = d2.sum(0)
    g_w2 = d3.T @ h2
    g_b2 = d3.sum(0)
    g = np.concatenate([g_w0.ravel(), g_b0, g_w1.ravel(), g_b1, g_w2.ravel(), g_b2])
    new = (np.asarray(params, np.float32).astype(np.float64) - lr * g).astype(np.float32)
    return new, float(loss.sum()), g


def fit(params, feat, tgt, order, lr, epochs, batch, H, emulate=True, max_steps=None):
    """fit's epoch loop over a given permutation per epoch (orc.fit_order).
    Returns (params, epoch mean losses)."""
    n = len(feat)
    p = np.asarray(params, np.float32).copy()
    losses = []
    steps = 0
    for e in range(epochs):
        total = 0.0
        for s0 in range(0, n, batch):
            rows = np.asarray(order[e][s0:s0 + batch], np.int64)
            nb = len(rows)
            p, kl, _ = step(p, feat, tgt, rows, nb, lr, H, emulate)
            total += kl
            steps += 1
            if max_steps is not None and steps >= max_steps:
                return p, losses + [total / n]
        losses.append(total / n)
    return p, losses
