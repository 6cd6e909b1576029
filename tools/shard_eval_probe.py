"""evaluate() sharded by app range across processes (SURVEY §8e aggregation
sharding), gloo for the row gather, all ranks on one GPU: the gathered rows
and histogram must equal a single-process evaluate bit for bit.
Usage: python tools/shard_eval_probe.py [ranks] [golden suite name]"""
import multiprocessing as mp
import os
import sys

import numpy as np

sys.path.insert(0, ".")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def golden(name):
    return np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))


def worker(rank, world, name, port, q):
    import torch.distributed as dist

    import paper_2111_12055_b200 as gbx

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = dict(golden(name))
    dev = gbx.Device(0)
    ds = dev.suite_upload(s, s["features"])
    rows, hist = ds.evaluate_distributed(s["eval_params"], 10, int(s["eval_seed"]), rank, world)
    if rank == 0:
        q.put((rows, hist))
    dist.barrier()
    dist.destroy_process_group()


def free_port() -> int:
    """A currently unused local TCP port for the rendezvous."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    name = sys.argv[2] if len(sys.argv) > 2 else "suite_contended"
    port = free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, world, name, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    rows, (lo, cnt) = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    import paper_2111_12055_b200 as gbx
    s = dict(golden(name))
    dev = gbx.Device(0)
    ds = dev.suite_upload(s, s["features"])
    rows1, (lo1, cnt1) = ds.evaluate(s["eval_params"], 10, int(s["eval_seed"]))
    ok = (np.array_equal(rows, rows1) and np.array_equal(lo, lo1) and np.array_equal(cnt, cnt1)
          and all(p.exitcode == 0 for p in procs))
    print(f"{world} ranks, {name}: {len(rows)} apps, rows identical {np.array_equal(rows, rows1)}, "
          f"histogram identical {np.array_equal(lo, lo1) and np.array_equal(cnt, cnt1)}")
    print("OK" if ok else "MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
