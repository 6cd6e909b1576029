"""CPU, world_size 2 (gloo): the data-parallel decomposition of a fit step.

Each global minibatch is split into equal contiguous rank slices (the same
rule gbxcu's step_slice uses); every rank computes the gradient contributions
of its slice scaled by the GLOBAL 1/|b| plus its KL sum, one all-reduce sums
them, and every rank applies the identical SGD update. The result must match
the single-process oracle fit (fp64 re-association only)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def rank_slice(start, stop, rank, nranks):
    nb = stop - start
    per = (nb + nranks - 1) // nranks
    lo = min(stop, start + rank * per)
    return lo, min(stop, lo + per)


def _worker(rank, world, port, n, batch, epochs, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle

    orc = oracle.Restatement()
    feat, tgt = orc.g1(42, n)
    p = orc.policy_init(7)
    order = np.arange(n, dtype=np.uint64)
    losses = []
    for e in range(epochs):
        order = orc.fit_order(n, 99, e + 1)  # order after e+1 in-place passes
        total = 0.0
        for start in range(0, n, batch):
            stop = min(n, start + batch)
            lo, hi = rank_slice(start, stop, rank, world)
            g, ls = orc.partial_gradient(p, feat, tgt, order[lo:hi], 1.0 / (stop - start))
            buf = torch.from_numpy(np.concatenate([g, [ls]]))
            dist.all_reduce(buf)
            red = buf.numpy()
            loss = red[-1] / (stop - start)
            assert np.isfinite(loss)
            total += loss * (stop - start)
            p = (p.astype(np.float64) - 0.01 * red[:-1]).astype(np.float32)
        losses.append(total / n)
    if rank == 0:
        np.save(out, np.concatenate([p.astype(np.float64), losses]))
    dist.destroy_process_group()


@pytest.mark.parametrize("batch", [64, 250])
def test_two_rank_fit_matches_single_process(tmp_path, batch):
    import oracle

    n, epochs, world = 600, 2, 2
    out = str(tmp_path / "p.npy")
    port = 29500 + (os.getpid() % 1000) + batch
    mp.spawn(_worker, args=(world, port, n, batch, epochs, out), nprocs=world, join=True)
    res = np.load(out)
    p_dp, loss_dp = res[:5026].astype(np.float32), res[5026:]
    orc = oracle.Restatement()
    feat, tgt = orc.g1(42, n)
    rc, p_ref, loss_ref, _ = orc.fit(orc.policy_init(7), feat, tgt, 0.01, epochs, batch, 99)
    assert rc == 0
    # fp32 weights: at most 1 ulp apart (fp64 re-association of the gradient sum)
    ulp = np.abs(p_dp.view(np.int32).astype(np.int64) - p_ref.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1, ulp.max()
    np.testing.assert_allclose(loss_dp, loss_ref, rtol=1e-12)


def test_rank_slices_partition_every_batch():
    for nb in (1, 2, 7, 64, 65, 4096):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                lo, hi = rank_slice(100, 100 + nb, r, world)
                covered.extend(range(lo, hi))
            assert covered == list(range(100, 100 + nb))
