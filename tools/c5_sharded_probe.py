"""bench.run_c5_sharded driven by N processes on one GPU over gloo (the
bench itself uses NCCL across GPUs): checks the sharded C5 secondary's
collectives and that the gathered rows cover every app. Small suite."""
import multiprocessing as mp
import os
import sys

sys.path.insert(0, ".")


def worker(rank, world, port, q):
    import argparse

    import torch
    import torch.distributed as dist

    import bench
    import paper_2111_12055_b200 as gbx

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = gbx.Device(0)
    args = argparse.Namespace(c5_apps=300, c5_shaders_per_app=200)
    out = bench.run_c5_sharded(args, dev, torch, dist, rank, world)
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def free_port() -> int:
    """A currently unused local TCP port for the rendezvous."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
    ok = out["rows_gathered"] == 300 and out["value"] > 0 and all(p.exitcode == 0 for p in ps)
    print(out)
    print("OK" if ok else "MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
