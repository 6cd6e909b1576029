"""The REAL multi-process peer-set path (CUDA IPC exchange regions, system-scope
counters and LL words — what `bench.py --gpus N` runs across GPUs) exercised
with two processes on ONE GPU. Their contexts time-slice instead of running
concurrently, so every step waits for the other process's slice: slow, but it
is the same code path end to end (export / attach / fused kernel<SYS=true>).

Usage: python tools/ipc_peer_probe.py [n_records] [global_batch] [ranks] [sgd|adam]
Prints the max fp32-ulp difference of the ranks' parameters against a
single-process fit with the same global batch, and between the ranks."""
import multiprocessing as mp
import sys

import numpy as np

sys.path.insert(0, ".")


def worker(rank, n, batch, q_handles, q_peers, q_out, opt="sgd"):
    import paper_2111_12055_b200 as gbx
    from bench import synthetic_log

    dev = gbx.Device(0)
    q_handles.put((rank, dev.peer_export()))
    handles = q_peers.get()
    dev.peer_attach(handles, rank)
    feat, tgt = synthetic_log(n)
    p0 = dev.policy_init(7)
    try:
        p, el = dev.fit(p0, feat, tgt, 0.01 if opt == "sgd" else 1e-3, 2, batch, 99, optimizer=opt)
        q_out.put((rank, p, el, None))
    except Exception as e:  # noqa: BLE001
        q_out.put((rank, None, None, repr(e)))


def ulps(a, b):
    a = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64)
    return int(np.abs(a - b).max())


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    R = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    opt = sys.argv[4] if len(sys.argv) > 4 else "sgd"
    ctx = mp.get_context("spawn")
    qh, qo = ctx.Queue(), ctx.Queue()
    qp = [ctx.Queue() for _ in range(R)]
    procs = [ctx.Process(target=worker, args=(r, n, batch, qh, qp[r], qo, opt)) for r in range(R)]
    for p in procs:
        p.start()
    got = dict(qh.get(timeout=120) for _ in range(R))
    for r in range(R):
        qp[r].put([got[k] for k in range(R)])
    res = {}
    for _ in range(R):
        r, p, el, err = qo.get(timeout=600)
        res[r] = (p, el, err)
    for p in procs:
        p.join(timeout=60)
    for r in range(R):
        if res[r][2]:
            print(f"rank {r} failed: {res[r][2]}")
            return 1
    import paper_2111_12055_b200 as gbx
    from bench import synthetic_log
    feat, tgt = synthetic_log(n)
    dev = gbx.Device(0)
    p1, el1 = dev.fit(dev.policy_init(7), feat, tgt, 0.01 if opt == "sgd" else 1e-3, 2, batch, 99,
                      optimizer=opt)
    across = max(ulps(res[0][0], res[r][0]) for r in range(R))
    print(f"peer set of {R} processes on one GPU, n={n}, global batch {batch}: "
          f"max across ranks {across} ulp, rank0 vs single process "
          f"{ulps(res[0][0], p1)} ulp; losses {res[0][1]} vs {el1}")
    ok = across == 0 and ulps(res[0][0], p1) <= 2 and np.allclose(res[0][1], el1, rtol=1e-12)
    print("OK" if ok else "MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
