#!/usr/bin/env python3
"""bench.py — driver contract for the gbx-b200 hot path.

Workload (BASELINE.json configs[1], the single-GPU config the metric is quoted
on): a synthetic 1M-tuple experience log (44 fp32 features + fp64 Boltzmann
target pair per record), default 44->64->32->2 policy MLP. One STEP = one
epoch of `fit` (device Fisher-Yates replay + fused fp64-parity train-step
kernel + SGD) over the whole log at global batch B. The secondary numbers
(`inference`, `aggregation`) time the full-suite greedy inference over the
same 1M states and a C5-style aggregation sweep.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--n N]
  python bench.py --impl reference ...   # the reference's own CPU fit

Multi-GPU (torchrun): weak scaling — every rank holds an N*1M-record log (the
global permutation needs the whole log), the global batch is N*B, and each
step's gradient is all-reduced once over NCCL inside libgbxcu.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "experience samples/sec trained; shader decisions/sec inferred, at 1/2/4/8 GPU"
HBM_PEAK_FALLBACK = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--records", dest="n", type=int, default=1_000_000,
                    help="records per GPU (weak scaling)")
    ap.add_argument("--batch", type=int, default=8192,
                    help="minibatch per GPU (global = N x this; 65,536 at 8 GPUs, SURVEY C3)")
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--dp", default="fused", choices=["fused", "nccl"],
                    help="N>1 gradient exchange: fused = in-kernel reduce-scatter/all-gather over "
                         "NVLink peer memory (one launch per epoch); nccl = per-step ncclAllReduce")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--c5-apps", type=int, default=10_000)
    ap.add_argument("--qt-tuples", type=int, default=10_000_000,
                    help="experience-store secondary: tuples folded into a fresh device Q-table")
    ap.add_argument("--c5-shaders-per-app", type=int, default=10_000)
    ap.add_argument("--wide-records", type=int, default=10_000_000,
                    help="C4 secondary: records of the wide-MLP (hidden 512) epoch")
    return ap.parse_args()


# ------------------------------------------------------------------ inputs
def synthetic_log(n: int, seed: int = 42):
    """G1-shaped synthetic records: stage one-hot + 36 counter features in
    [0, 7), target p ~ U[0.02, 0.98) -> (p, 1-p) (proj/tests/test_policy.cpp:15-28)."""
    rng = np.random.default_rng(seed)
    feat = np.zeros((n, 44), np.float32)
    feat[np.arange(n), rng.integers(0, 8, n)] = 1.0
    feat[:, 8:] = rng.random((n, 36), dtype=np.float32) * np.float32(7.0)
    p = rng.uniform(0.02, 0.98, n)
    tgt = np.stack([p, 1.0 - p], 1)
    return feat, tgt


def synthetic_suite(n_apps: int, per_app: int, seed: int = 5, cap: float = np.inf):
    """C5-style suite: per_app distinct shaders per app, 2-4 pipelines,
    exec_fraction U[0.03,0.09) scaled to a 0.85 cap per pipeline."""
    rng = np.random.default_rng(seed)
    n_sh = n_apps * per_app
    lat = np.stack([rng.random(n_sh), rng.random(n_sh) * 1.6, rng.random(n_sh) * 0.6], 1)
    pipes = rng.integers(2, 5, n_apps)
    app_pipe_off = np.concatenate([[0], np.cumsum(pipes)]).astype(np.uint64)
    sizes = []
    for a in range(n_apps):
        k = int(pipes[a])
        base, extra = divmod(per_app, k)
        sizes.extend([base + (1 if i < extra else 0) for i in range(k)])
    pipe_slot_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    frac = rng.uniform(0.03, 0.09, n_sh)
    tot = np.add.reduceat(frac, pipe_slot_off[:-1].astype(np.int64))
    scale = np.where(tot > 0.85, 0.85 / tot, 1.0)
    frac = frac * np.repeat(scale, np.diff(pipe_slot_off).astype(np.int64))
    npipe = len(sizes)
    wt = np.stack([rng.uniform(0.5, 2.0, npipe), rng.uniform(2.0, 8.0, npipe) * 1e-3], 1)
    app = np.stack([np.ones(n_apps), np.full(n_apps, cap), np.full(n_apps, 0.005),
                    np.ones(n_apps)], 1)
    s = dict(app_pipe_off=app_pipe_off, pipe_slot_off=pipe_slot_off,
             slot_shader=np.arange(n_sh, dtype=np.uint32), slot_frac=frac, pipe_wt=wt,
             shader_lat=lat, app_f64=app)
    feat, _ = synthetic_log(n_sh, seed + 1)
    return s, feat


def synthetic_suite_torch(torch, n_apps: int, per_app: int, seed: int = 5, cap: float = float("inf")):
    """synthetic_suite generated on the device (C5 at its nominal 1e8 scale):
    same distributions; G1-shaped features."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    dev = "cuda"
    n_sh = n_apps * per_app
    lat = torch.rand((n_sh, 3), generator=g, device=dev, dtype=torch.float64)
    lat[:, 1] *= 1.6
    lat[:, 2] *= 0.6
    pipes = torch.randint(2, 5, (n_apps,), generator=g, device=dev)
    app_pipe_off = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(pipes, 0)])
    npipe = int(app_pipe_off[-1])
    app_of_pipe = torch.repeat_interleave(torch.arange(n_apps, device=dev), pipes)
    idx_in_app = torch.arange(npipe, device=dev) - app_pipe_off[app_of_pipe]
    k = pipes[app_of_pipe]
    sizes = per_app // k + (idx_in_app < per_app % k).to(torch.int64)
    pipe_slot_off = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(sizes, 0)])
    frac = torch.rand(n_sh, generator=g, device=dev, dtype=torch.float64) * 0.06 + 0.03
    tot = torch.segment_reduce(frac, "sum", lengths=sizes)
    scale = torch.where(tot > 0.85, 0.85 / tot, torch.ones_like(tot))
    frac *= torch.repeat_interleave(scale, sizes)
    wt = torch.stack([torch.rand(npipe, generator=g, device=dev, dtype=torch.float64) * 1.5 + 0.5,
                      (torch.rand(npipe, generator=g, device=dev, dtype=torch.float64) * 6 + 2) * 1e-3], 1)
    app = torch.stack([torch.ones(n_apps, dtype=torch.float64, device=dev),
                       torch.full((n_apps,), cap, dtype=torch.float64, device=dev),
                       torch.full((n_apps,), 0.005, dtype=torch.float64, device=dev),
                       torch.ones(n_apps, dtype=torch.float64, device=dev)], 1)
    feat = torch.rand((n_sh, 44), generator=g, device=dev, dtype=torch.float32) * 7.0
    feat[:, :8] = 0.0
    stage = torch.randint(0, 8, (n_sh,), generator=g, device=dev)
    feat[torch.arange(n_sh, device=dev), stage] = 1.0
    s = dict(app_pipe_off=app_pipe_off, pipe_slot_off=pipe_slot_off,
             slot_shader=torch.arange(n_sh, dtype=torch.int32, device=dev), slot_frac=frac,
             pipe_wt=wt, shader_lat=lat, app_f64=app)
    return s, feat


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: a background thread polls NVML every 5 ms (nvidia-smi -lms through
    a pipe lost its block-buffered output when terminated, so a short region
    reported no samples). Falls back to one-shot nvidia-smi queries."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.sm, self.reasons, self.max_mhz, self.source = [], set(), None, None

    def _poll_nvml(self):
        import pynvml as N
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        get_r = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            N.nvmlDeviceGetCurrentClocksThrottleReasons
        masks = [(nm, getattr(N, attr, 0)) for nm, attr in self.REASONS]
        while True:  # at least one sample, and one after the region ends
            self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
            r = get_r(h)
            for nm, m in masks:
                if m and (r & m):
                    self.reasons.add(nm)
            self._ready.set()
            if self._stop.is_set():
                break
            self._stop.wait(self.period)

    def _poll_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout
                f = [x.strip() for x in out.split(",")]
                self.sm.append(float(f[0]))
                self.max_mhz = float(f[1])
                for nm, v in zip(names, f[2:6]):
                    if v.lower().startswith("active"):
                        self.reasons.add(nm)
                self._ready.set()
            except (OSError, ValueError, IndexError, subprocess.SubprocessError):
                self._ready.set()
                return

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            try:
                self.source = "nvml"
                self._poll_nvml()
            finally:
                N.nvmlShutdown()
        except Exception:  # no NVML binding / library: nvidia-smi one-shots
            self.source = "nvidia-smi"
            self._poll_smi()
        self._ready.set()

    def __enter__(self):
        import threading
        self._stop = threading.Event()
        self._ready = threading.Event()
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        # NVML start-up can outlast a short timed region: the region begins
        # only once the sampler is polling (first sample taken)
        self._ready.wait(timeout=10)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": self.source}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def pipe_peaks(device: int):
    import ctypes as C

    path = os.path.join(ROOT, "tools", "libpeaks.so")
    if not os.path.exists(path):
        return None, None
    L = C.CDLL(path)
    L.peak_fp64_tflops.restype = C.c_double
    L.peak_fp32_tflops.restype = C.c_double
    L.peak_fp64_tensor_tflops.restype = C.c_double
    return (L.peak_fp64_tflops(device), L.peak_fp64_tensor_tflops(device),
            L.peak_fp32_tflops(device))


def host_info():
    """nproc and the CPU model of the host the CPU baselines run on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model,
            "affinity_cpus": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None}


def workload_config(args, world):
    """The config both arms report (the driver compares them)."""
    return {"workload": "C2: 1M-tuple experience log per GPU, default MLP 44-64-32-2, "
                        "1 fit epoch per step (fp64 parity mode)",
            "records": args.n * world, "global_batch": args.batch * world, "lr": args.lr,
            "parallelism": f"dp{world}" + (f" ({args.dp} gradient exchange)" if world > 1 else ""),
            "l2": "inputs (196 MB/GPU) larger than L2"}


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: re-run this script under
    torch.distributed.run with one rank per GPU (rank 0 prints the line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


# ------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The reference's own CPU fit (oracle/_ref: the unmodified reference
    library; the restatement when it is not built) on the SAME workload as
    our arm: the same synthetic log, init, lr, seed and global batch. fit is
    single-threaded by contract. Each step is one epoch over
    the full log when the run fits the time budget, else over the log's
    first `sample` records (the per-record cost of fit does not depend on n)."""
    if rank != 0:
        return
    import oracle

    if not oracle.ref_available():
        kind, impl = "port", oracle.Restatement()
    else:
        kind, impl = "reference", oracle.Reference()
    n_total, batch = args.n * world, args.batch * world
    feat, tgt = synthetic_log(n_total)
    p0 = impl.policy_init(7)
    # rate probe on a 50k-record prefix, then size the per-step sample so the
    # whole --warmup W --steps K run stays within ~3 minutes
    m0 = min(n_total, 50_000)
    t0 = time.perf_counter()
    assert impl.fit(p0, feat[:m0], tgt[:m0], args.lr, 1, batch, 99)[0] == 0
    rate = m0 / (time.perf_counter() - t0)
    budget_s = float(os.environ.get("GBX_REF_BUDGET_S", "180"))
    sample = int(min(n_total, max(m0, budget_s * rate / max(1, args.steps + args.warmup))))
    fs, ts = (feat, tgt) if sample == n_total else (feat[:sample], tgt[:sample])
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        rc = impl.fit(p0, fs, ts, args.lr, 1, batch, 99)[0]
        dt = time.perf_counter() - t0
        assert rc == 0
        if it >= args.warmup:
            times.append(dt)
    v = sample / statistics.mean(times)
    what = ("the full log" if sample == n_total else f"the first {sample} records of the log")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": 1, "kind": kind,
                         "sample": f"fit, 1 epoch over {what} per step ({sample} records), "
                                   f"batch {batch}, lr {args.lr}, seed 99, init 7; fit is "
                                   "single-threaded by contract (SPEC.md:301)",
                         "host": host_info()},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args):
    import oracle

    kind, impl = ("reference", oracle.Reference()) if oracle.ref_available() else (
        "port", oracle.Restatement())
    # the N=1 workload itself: one epoch over the same 1M-record log, same batch
    sample = args.n
    feat, tgt = synthetic_log(sample)
    t0 = time.perf_counter()
    rc = impl.fit(impl.policy_init(7), feat, tgt, args.lr, 1, args.batch, 99)[0]
    dt = time.perf_counter() - t0
    assert rc == 0
    return {"value": sample / dt, "unit": "samples/s", "cores": 1, "kind": kind,
            "sample": f"fit, 1 epoch over the headline's {sample}-record log, batch {args.batch}, "
                      f"{dt:.1f} s on 1 host core (fit is single-threaded, SPEC.md:301)"}


# ----------------------------------------------------------------- our arm
def main():
    args = parse()
    launched = "WORLD_SIZE" in os.environ
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if launched and args.gpus > 1 and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    if args.impl == "reference":
        # only rank 0 works; without a launcher it stands for all N ranks
        run_reference(args, rank, world if launched else args.gpus)
        return
    if not launched and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))

    import torch
    import torch.distributed as dist

    import paper_2111_12055_b200 as gbx

    # one process per GPU; GBX_BENCH_BACKEND=gloo + more ranks than GPUs is a
    # test mode only (all ranks share GPU 0: exercises the N>1 code path)
    backend = os.environ.get("GBX_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = gbx.Device(local)
    dp_note = None
    if world > 1 and args.dp == "fused":
        # the fused peer set needs CUDA IPC between the ranks' GPUs; if any rank
        # cannot export/attach, every rank falls back to the NCCL path together
        ok_attach = 1
        handles = [None] * world
        try:
            h = dev.peer_export()
        except (gbx.CudaError, gbx.ValidationError) as e:
            h, dp_note = None, f"peer export failed: {e}"
        dist.all_gather_object(handles, h)
        if any(x is None for x in handles):
            ok_attach = 0
        else:
            try:
                dev.peer_attach(handles, rank)
            except (gbx.CudaError, gbx.ValidationError) as e:
                ok_attach, dp_note = 0, f"peer attach failed: {e}"
        flags = [None] * world
        dist.all_gather_object(flags, ok_attach)
        if not all(flags):
            dp_note = dp_note or "a peer rank could not attach the exchange regions"
            if ok_attach:
                dev.peer_detach()
            args.dp = "nccl"
        dist.barrier()
    if world > 1 and args.dp == "nccl":
        uid = [gbx.Device.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        dev.comm_init(uid[0], world, rank)
    stream = torch.cuda.ExternalStream(dev.stream)

    n_total = args.n * world
    batch = args.batch * world
    feat_h, tgt_h = synthetic_log(n_total)
    feat_h = np.ascontiguousarray(feat_h)
    params0 = dev.policy_init(7)
    feat_d = torch.from_numpy(feat_h).cuda()
    tgt_d = torch.from_numpy(tgt_h).cuda()
    params_d = torch.from_numpy(params0).cuda()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    kernel_ms = {"shuffle": 0.0, "train": 0.0}

    def step():
        dev.fit_dev(params_d.data_ptr(), feat_d.data_ptr(), tgt_d.data_ptr(), n_total, args.lr, 1,
                    batch, 99, stream=dev.stream)
        sh, tr = dev.last_fit_timing()  # CUDA events around the launches (fit syncs at its end)
        kernel_ms["shuffle"] += sh
        kernel_ms["train"] += tr

    try:
        step()
        ok = torch.tensor([1], device="cuda")
    except gbx.CudaError as e:  # the peer exchange failed on some rank
        ok, dp_note = torch.tensor([0], device="cuda"), str(e)
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if world > 1 and args.dp == "fused" and int(ok.item()) == 0:
        # fall back to the per-step NCCL all-reduce path (recorded in the JSON)
        dp_note = dp_note or "a peer rank failed"
        dev.peer_detach()
        uid = [gbx.Device.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        dev.comm_init(uid[0], world, rank)
        args.dp = "nccl"
        step()
    for _ in range(max(0, args.warmup - 1)):
        step()
    barrier()
    kernel_ms = {"shuffle": 0.0, "train": 0.0}
    l0 = dev.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = dev.launches - l0
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = n_total * args.steps / (ms_max * 1e-3)

    # ---- e2e: public host API, host buffers, H2D + D2H inside the region.
    #      N = 1: gbxcu_fit (uploads the whole log). N > 1: fit_sharded — each
    #      rank uploads only its 1/N of the log from pinned memory and the
    #      shards are all-gathered over NVLink before the fused fit.
    lo, hi = rank * args.n, (rank + 1) * args.n
    pinned_feat_t = torch.from_numpy(feat_h[lo:hi] if world > 1 else feat_h).pin_memory()
    pinned_tgt_t = torch.from_numpy(tgt_h[lo:hi] if world > 1 else tgt_h).pin_memory()
    pinned_feat, pinned_tgt = pinned_feat_t.numpy(), pinned_tgt_t.numpy()

    def e2e_step():
        if world > 1:
            dev.fit_sharded(params0, pinned_feat, pinned_tgt, args.lr, 1, batch, 99)
        else:
            dev.fit(params0, pinned_feat, pinned_tgt, args.lr, 1, batch, 99)

    e2e_step()  # warm
    barrier()
    e2e_times = []
    for _ in range(max(1, min(args.steps, 5))):
        barrier()
        t0 = time.perf_counter()
        e2e_step()
        e2e_times.append(time.perf_counter() - t0)
    tt = torch.tensor([statistics.median(e2e_times)], device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e = {"value": n_total / float(tt.item()), "unit": "samples/s",
           "h2d_bytes_per_step": int(pinned_feat.nbytes + pinned_tgt.nbytes + 4 * 5026),
           "d2h_bytes_per_step": int(4 * 5026 + 8),
           "path": "gbxcu_fit (whole log H2D)" if world == 1 else
                   "fit_sharded: 1/N of the log H2D per rank + NCCL all-gather on the device"}
    # its floor: the same bytes over the host link alone (pinned -> device, CUDA
    # events) plus the device-resident step; e2e is host-link bound when close
    df = torch.empty_like(pinned_feat_t, device="cuda")
    dtg = torch.empty_like(pinned_tgt_t, device="cuda")
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h2d = []
    for _ in range(3):
        h0.record()
        df.copy_(pinned_feat_t, non_blocking=True)
        dtg.copy_(pinned_tgt_t, non_blocking=True)
        h1.record()
        torch.cuda.synchronize()
        h2d.append(h0.elapsed_time(h1))
    h2d_ms = min(h2d)
    del df, dtg
    e2e.update({"ms_per_step": 1e3 * float(tt.item()), "h2d_ms": h2d_ms,
                "h2d_gbs": (pinned_feat.nbytes + pinned_tgt.nbytes) / (h2d_ms * 1e-3) / 1e9,
                "floor_ms": h2d_ms + ms_step,
                "note": "floor = the log's host-to-device copy alone + the device-resident step"})

    # ---- roofline of the dominant kernel (train_epoch_kernel)
    peaks = measured_peaks()
    dfma_peak, dmma_peak, fp32_peak = (None, None, None)
    secondary = {}
    if rank == 0:
        dfma_peak, dmma_peak, fp32_peak = pipe_peaks(local)
    # multi-CTA steps run on the FP64 tensor pipe (DMMA); the 1-CTA exact
    # kernel on DFMA. The roofline takes the higher of the two measured peaks.
    fp64_peak = max(dfma_peak, dmma_peak) if dfma_peak else None
    # dominant kernel: train_epoch_kernel, timed with CUDA events on its stream
    flop_per_record = 23936          # fwd 9,856 + bwd 14,080
    records_per_gpu = n_total / world
    k_ms = kernel_ms["train"] / args.steps if kernel_ms["train"] > 0 else ms_step
    train_tflops = records_per_gpu * flop_per_record / (k_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get("train_epoch_kernel")
            if tr and tr.get("records") == records_per_gpu and tr.get("batch") == batch:
                traffic = tr["dram_bytes"]
    except (OSError, ValueError):
        pass
    roofline = {
        "bound": "tensor" if batch > 32 else "fp64",  # FP64 tensor cores (DMMA) / DFMA chain
        "pipe": "fp64 DMMA m8n8k4" if batch > 32 else "fp64 DFMA",
        "achieved": train_tflops,
        "peak": fp64_peak,
        "unit": "TFLOP/s",
        "frac": (train_tflops / fp64_peak) if fp64_peak else None,
        "traffic": traffic,
        "kernel": "train_epoch_tc_kernel (fp64, DMMA)" if batch > 32 else "train_epoch_kernel (fp64 exact)",
        "kernel_ms_per_step": k_ms,
        "shuffle_ms_per_step": kernel_ms["shuffle"] / args.steps,
        "work_per_unit": "23,936 FLOP/record (fwd 9,856 + bwd 14,080), 196 B/record",
        "algorithmic_bytes": records_per_gpu * 196,
        "peak_source": "max of measured DMMA (FP64 tensor) and DFMA throughput, tools/peaks.cu "
                       "(MEASURED_PEAKS.json has no fp64)",
        "peaks_measured": {"dmma_tflops": dmma_peak, "dfma_tflops": dfma_peak},
        "hbm_view": {"achieved_gbs": records_per_gpu * 196 / (k_ms * 1e-3) / 1e9,
                     "peak_gbs": peaks.get("hbm_gbs", HBM_PEAK_FALLBACK)},
    }

    c5_sharded = None
    if world > 1 and not args.no_secondary:
        c5_sharded = run_c5_sharded(args, dev, torch, dist, rank, world)
    if world > 1:
        # the collective fits are done: every rank leaves its peer set /
        # communicator so rank 0's single-GPU secondaries (fits included) run
        # locally instead of waiting on ranks that have moved on
        dist.barrier()
        if args.dp == "fused":
            dev.peer_detach()
        else:
            dev.comm_destroy()
    if rank == 0 and not args.no_secondary:
        # inference / C5 use a policy of FIXED training (5 epochs of the headline
        # fit from the same init), so their numbers do not depend on --steps:
        # the guard's re-check share grows as a net fits the noise targets
        p_inf = torch.from_numpy(params0).cuda()
        dev.fit_dev(p_inf.data_ptr(), feat_d.data_ptr(), tgt_d.data_ptr(), n_total, args.lr, 5,
                    batch, 99, stream=dev.stream)
        torch.cuda.synchronize()
        secondary = run_secondary(args, dev, stream, p_inf, feat_d, torch, gbx, fp32_peak,
                                  dict(peaks, dfma_tflops=dfma_peak), local)

    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args, world),
        "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "clocks": clk.summary(),
    }
    if dp_note:
        line["dp_fallback"] = "fused peer exchange failed (" + dp_note + "); measured with nccl"

    for v in secondary.get("batch_sweep", {}).values():
        if v.get("tflops") and fp64_peak:
            v["roofline_frac"] = v["tflops"] / fp64_peak
    line.update(secondary)
    if c5_sharded:
        line["aggregation_sharded"] = c5_sharded
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
        line["cpu_baseline"]["host"] = host_info()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_secondary(args, dev, stream, params_d, feat_d, torch, gbx, fp32_peak, peaks, local):
    """Full-suite greedy inference over the 1M states + a C5-style aggregation sweep.
    params_d: the policy after 5 epochs of the headline fit (fixed training)."""
    out = {}
    # row f1: experience store — fold a synthetic C3-scale tuple log into a fresh
    # device Q-table (QTable::update x n) + snapshot_policy_dataset (device-resident)
    out["qtable"] = run_qtable(args, dev, stream, torch, gbx, peaks)
    torch.cuda.empty_cache()
    n = args.n
    act_d = torch.empty(n, dtype=torch.uint8, device="cuda")
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    for mode, name in ((gbx.FWD_FAST, "fast"), (gbx.FWD_EXACT, "exact")):
        for _ in range(3):
            dev.forward_dev(params_d.data_ptr(), feat_d.data_ptr(), n, None, act_d.data_ptr(),
                            mode, dev.stream)
        torch.cuda.synchronize()
        reps = 10
        ev0.record(stream)
        for _ in range(reps):
            dev.forward_dev(params_d.data_ptr(), feat_d.data_ptr(), n, None, act_d.data_ptr(),
                            mode, dev.stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / reps
        rate = n / (ms * 1e-3)
        out.setdefault("inference", {})[name] = {
            "value": rate, "unit": "decisions/s", "ms": ms, "states": n,
            "fp32_tflops": rate * 9856 / 1e12,
            "hbm_gbs": rate * 177 / 1e9}
        if mode == gbx.FWD_FAST:
            out["inference"][name]["recheck_fraction"] = dev.last_recheck_count() / n
        if fp32_peak:
            # FFMA-bound path (9,856 FLOP/state): fraction of the measured FFMA peak
            out["inference"][name]["roofline_frac_fp32"] = rate * 9856 / 1e12 / fp32_peak
    out["inference"]["fp32_peak_tflops_measured"] = fp32_peak
    out["inference"]["hbm_peak_gbs"] = peaks.get("hbm_gbs", HBM_PEAK_FALLBACK)
    if not args.no_cpu_baseline:
        import oracle
        if oracle.ref_available():
            m = 200_000
            f_s = feat_d[:m].cpu().numpy()
            p_s = params_d.cpu().numpy()
            t0 = time.perf_counter()
            oracle.Reference().select_greedy(p_s, f_s)
            dt = time.perf_counter() - t0
            out["inference"]["cpu_baseline"] = {
                "value": m / dt, "unit": "decisions/s", "cores": 1, "kind": "reference",
                "sample": f"select_greedy (PolicyNet::forward, fp64) over {m} states, {dt:.2f} s"}

    # train regimes beside the headline batch: the reference's default batch 32
    # (bit-exact 1-CTA kernel, a serial chain of n/32 dependent steps) and a
    # large batch (sync amortised); same 1M-record log, one epoch each
    out["batch_sweep"] = {}
    feat_n = feat_d.shape[0]
    tgt_n = torch.empty((feat_n, 2), dtype=torch.float64, device="cuda")
    tgt_n[:, 0] = 0.5
    tgt_n[:, 1] = 0.5
    for b in (32, 4096, 16384, 65536):
        p_b = params_d.clone()
        dev.fit_dev(p_b.data_ptr(), feat_d.data_ptr(), tgt_n.data_ptr(), feat_n, args.lr, 1, b, 99,
                    stream=dev.stream)
        torch.cuda.synchronize()
        ev0.record(stream)
        dev.fit_dev(p_b.data_ptr(), feat_d.data_ptr(), tgt_n.data_ptr(), feat_n, args.lr, 1, b, 99,
                    stream=dev.stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        _, k_ms = dev.last_fit_timing()
        row = {
            "value": feat_n / (ms * 1e-3), "unit": "samples/s", "ms_per_epoch": ms,
            "kernel": "train_epoch_cluster_kernel (fp64 exact, 4-CTA cluster)" if b <= 32 else "train_epoch_tc_kernel",
            "tflops": feat_n * 23936 / (k_ms * 1e-3) / 1e12 if k_ms > 0 else None}
        if b <= 32 and k_ms > 0:
            # latency regime: a serial chain of n/32 dependent steps
            # on ONE SM, so the roofline is per SM, not chip-wide: 11,968 MAC per
            # record x 32 records at the SM's fp64 FMA rate (measured DFMA peak / 148)
            steps = (feat_n + b - 1) // b
            us = k_ms * 1e3 / steps
            dfma = (peaks.get("dfma_tflops") or 34.1) * 1e12 / 2 / 148  # FMA/s per SM
            bound_us = 11968 * b / dfma * 1e6
            row.update({"us_per_step": us, "per_sm_bound_us": bound_us, "per_sm_frac": bound_us / us,
                        "bound_note": "one SM's throughput: 11,968 fp64 MAC/record at the measured DFMA "
                                      "rate / 148 SMs (the step now runs on a 4-CTA cluster, latency-bound: "
                                      "a ~270-deep dependent fp64 chain + 3 cluster barriers per step)"})
        out["batch_sweep"][str(b)] = row

    # north-star variants on the fused kernel (absent from the reference): TD
    # regression of Q(x, a) on the reward + Adam, same log and batch as the headline
    tgt_td = torch.empty((feat_n, 2), dtype=torch.float64, device="cuda")
    tgt_td[:, 0] = (feat_d[:, 8] > 3.5).to(torch.float64)   # action
    tgt_td[:, 1] = feat_d[:, 9].to(torch.float64) / 7.0     # reward
    out["variants"] = {}
    for loss, opt in (("td", "sgd"), ("kl", "adam"), ("td", "adam")):
        tg = tgt_td if loss == "td" else tgt_n
        p_v = params_d.clone()
        for rep in range(2):  # warm, then timed
            torch.cuda.synchronize()
            ev0.record(stream)
            dev.fit_dev(p_v.data_ptr(), feat_d.data_ptr(), tg.data_ptr(), feat_n, 1e-3, 1, args.batch,
                        99, stream=dev.stream, loss=loss, optimizer=opt)
            ev1.record(stream)
            torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        _, k_ms = dev.last_fit_timing()
        out["variants"][f"{loss}_{opt}"] = {
            "value": feat_n / (ms * 1e-3), "unit": "samples/s", "ms_per_epoch": ms,
            "batch": args.batch, "kernel": "train_epoch_tc_kernel (variant instantiation)",
            "tflops": feat_n * 23936 / (k_ms * 1e-3) / 1e12 if k_ms > 0 else None}
    del tgt_td

    # C5 sweep: inference + aggregation over n_apps x per_app shaders (generated
    # on the device; the default is the config's 1e8 shader feature vectors)
    s, feat = synthetic_suite_torch(torch, args.c5_apps, args.c5_shaders_per_app)
    ds = dev.suite_upload_dev(s, feat)
    n_slots_c5 = int(s["pipe_slot_off"][-1])
    del s
    torch.cuda.empty_cache()
    params = params_d.cpu().numpy()
    pd = torch.from_numpy(params).cuda()
    nsh = ds.n_shaders
    a_d = torch.empty(nsh, dtype=torch.uint8, device="cuda")
    rows_d = torch.empty((args.c5_apps, 5), dtype=torch.float64, device="cuda")
    for _ in range(3):
        ds.evaluate_dev(pd.data_ptr(), 10, 77, a_d.data_ptr(), rows_d.data_ptr(), dev.stream)
    torch.cuda.synchronize()
    reps = 5
    ev0.record(stream)
    for _ in range(reps):
        ds.evaluate_dev(pd.data_ptr(), 10, 77, a_d.data_ptr(), rows_d.data_ptr(), dev.stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    # split of the last evaluate into its inference (K2) and aggregation (K3)
    # launches, CUDA events recorded inside gbxcu_evaluate_dev on its stream
    ms_fwd, ms_agg = dev.last_eval_timing()
    del feat
    # K3 algorithmic bytes: per slot the shader index, fraction, latents (3 f64)
    # and action (37 B), per app its 5-double row (the 8-B fraction re-read of
    # each pipeline's A segment is not counted)
    agg_bytes = 37.0 * n_slots_c5 + 40.0 * args.c5_apps
    hbm_peak = measured_peaks().get("hbm_gbs", HBM_PEAK_FALLBACK)
    out["aggregation"] = {"value": nsh / (ms * 1e-3), "unit": "shader decisions/s (infer+agg)",
                          "ms": ms, "apps": args.c5_apps, "shaders": nsh,
                          "bytes_per_shader": 204, "hbm_gbs": nsh * 204 / (ms * 1e-3) / 1e9,
                          "inference_ms": ms_fwd, "aggregate_ms": ms_agg,
                          "aggregate_hbm_gbs": agg_bytes / (ms_agg * 1e-3) / 1e9,
                          "aggregate_roofline_frac": agg_bytes / (ms_agg * 1e-3) / 1e9 / hbm_peak,
                          "inference_fp32_tflops": nsh * 9856 / (ms_fwd * 1e-3) / 1e12,
                          "data": "synthetic suite generated on the device (C5: 1e8 shaders)"}
    ds.close()
    if not args.no_cpu_baseline:
        import oracle
        if oracle.ref_available():
            R = oracle.Reference()
            jobs = os.cpu_count() or 1
            h = R.suite_generate(benchmark_count=1000, seed=3)
            dims = np.empty(5, np.uint64)
            R.lib.gbxref_suite_dims(h, dims)
            n_slots = int(dims[3])
            t0 = time.perf_counter()
            R.evaluate(h, params_d.cpu().numpy(), 10, 77, jobs=jobs)
            dt = time.perf_counter() - t0
            R.suite_free(h)
            out["aggregation"]["cpu_baseline"] = {
                "value": n_slots / dt, "unit": "shader decisions/s (infer+agg)", "cores": jobs,
                "kind": "reference",
                "sample": f"evaluate() on a generated 1000-benchmark suite ({n_slots} slots), "
                          f"jobs={jobs}, {dt:.2f} s"}

    # Algorithm 1 on the device (row f3 wired to A5-A11, f1): iterations of
    # run_iteration on a generated 44-benchmark suite, reference
    # TrainConfig defaults (batch 32, 50 epochs), against the reference's run_training
    out["algorithm1"] = run_algorithm1(args, dev, gbx)

    # C4 (BASELINE configs[3]): wide MLP 44-512-512-2 on a synthetic 10M-tuple
    # log (G1-shaped, generated on the device), one fit epoch per precision on
    # tcgen05 (kind::f16 BF16, the default, and kind::tf32), B = 8192 per GPU
    # (C4's 8-GPU global batch is 65,536)
    H = 512
    n_w = args.wide_records
    g = torch.Generator(device="cuda").manual_seed(11)
    fw = torch.rand((n_w, 44), generator=g, device="cuda", dtype=torch.float32) * 7.0
    fw[:, :8] = 0.0
    fw[torch.arange(n_w, device="cuda"), torch.randint(0, 8, (n_w,), generator=g, device="cuda")] = 1.0
    pt = torch.rand(n_w, generator=g, device="cuda", dtype=torch.float64) * 0.96 + 0.02
    tw = torch.stack([pt, 1.0 - pt], 1).contiguous()
    del pt
    bf16_peak = peaks.get("bf16_tflops", 1590.0)
    wide = {}
    for prec, peak in (("bf16", bf16_peak), ("tf32", bf16_peak / 2)):
        pw = torch.from_numpy(dev.wide_init(H, 7)).cuda()
        torch.cuda.synchronize()
        dev.wide_fit_dev(H, pw.data_ptr(), fw.data_ptr(), tw.data_ptr(), n_w, 0.01, 1, args.batch, 1,
                         stream=dev.stream, precision=prec)
        torch.cuda.synchronize()
        ev0.record(stream)
        reps = 2
        for _ in range(reps):
            el_w = dev.wide_fit_dev(H, pw.data_ptr(), fw.data_ptr(), tw.data_ptr(), n_w, 0.01, 1,
                                    args.batch, 1, stream=dev.stream, precision=prec)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / reps
        tf = n_w * 1_669_120 / (ms * 1e-3) / 1e12
        wide[prec] = {"value": n_w / (ms * 1e-3), "unit": "samples/s", "ms_per_epoch": ms,
                      "us_per_step": ms * 1e3 / ((n_w + args.batch - 1) // args.batch),
                      "epoch_loss": float(el_w[0]), "tflops": tf, "peak_tflops": peak,
                      "roofline_frac": tf / peak}
    out["wide_mlp"] = dict(wide["bf16"], records=n_w, hidden=H, batch=args.batch, dtype="bf16",
                           flop_per_record=1_669_120, tf32=wide["tf32"],
                           data="synthetic G1-shaped 10M-tuple log generated on the device",
                           peak_note="dense BF16 = the measured bf16 cuBLAS peak "
                                     "(MEASURED_PEAKS.json); TF32 = half of it")
    del fw, tw
    torch.cuda.empty_cache()

    return out


def run_c5_sharded(args, dev, torch, dist, rank, world):
    """C5 sharded by app range over the ranks (BASELINE configs[4]
    "sharded 1/2/4/8 GPU"): every rank holds the same generated suite, infers
    and aggregates its app range (gbxcu_evaluate_shard), rank 0 gathers the
    rows; strong scaling — total shaders / max-over-ranks time."""
    s, feat = synthetic_suite_torch(torch, args.c5_apps, args.c5_shaders_per_app)
    ds = dev.suite_upload_dev(s, feat)
    del s, feat
    torch.cuda.empty_cache()
    params = dev.policy_init(7)
    per = (ds.n_apps + world - 1) // world
    lo, hi = min(ds.n_apps, rank * per), min(ds.n_apps, (rank + 1) * per)
    ds.evaluate_shard(params, 10, 77, lo, hi)  # warm
    times = []
    for _ in range(3):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rows = ds.evaluate_shard(params, 10, 77, lo, hi)
        times.append(time.perf_counter() - t0)
    # object collectives work on every backend (nccl in the bench, gloo in tests)
    gathered = [None] * world
    dist.all_gather_object(gathered, (statistics.median(times), rows))
    t_max = max(g[0] for g in gathered)
    nsh = ds.n_shaders
    ds.close()
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    n_rows = sum(len(g[1]) for g in gathered)
    return {"value": nsh / t_max, "unit": "shader decisions/s (infer+agg)",
            "ms": t_max * 1e3, "apps": args.c5_apps, "shaders": nsh, "ranks": world,
            "rows_gathered": n_rows, "scaling": "strong",
            "note": "app-range shards (gbxcu_evaluate_shard), rows gathered to rank 0; "
                    "host wall clock around each rank's shard, max over ranks"}


def run_algorithm1(args, dev, gbx):
    import oracle
    if not oracle.ref_available():
        return {"unavailable": "compiled reference (the environment) not built"}
    from paper_2111_12055_b200.tuner import DeviceTuner, TunerConfig
    R = oracle.Reference()
    iters, checkins = 3, 50
    h = R.suite_generate(benchmark_count=44, seed=7)
    res = {"iterations": iters, "benchmarks": 44}
    if not args.no_cpu_baseline:
        t0 = time.perf_counter()
        o = R.run_training(h, iters, checkins=checkins, seed=5)
        res["cpu_baseline"] = {"value": iters / (time.perf_counter() - t0), "unit": "iterations/s",
                               "cores": 1, "kind": "reference",
                               "sample": f"run_training, {iters} iterations (environment included)"}
    # untimed warm-up run of the same iterations on an identical suite: first
    # launches (lazy module loading) and every buffer size the timed run needs
    # (the table is then cleared and reused) stay out of the timing
    cfg_t = TunerConfig(num_iterations=iters, checkins_per_iteration=checkins, seed=5)
    warm = DeviceTuner(dev, cfg_t)
    hw = R.suite_generate(benchmark_count=44, seed=7)
    for i in range(iters):
        R.suite_advance(hw, checkins)
        sw = R.suite_export(hw)
        warm.run_iteration(i, sw, R.suite_keys(hw, len(sw["features"])), R.suite_checkin(hw))
    R.suite_free(hw)
    tuner = DeviceTuner(dev, cfg_t)
    tuner.table.close()
    tuner.table = warm.table
    tuner.table.clear()
    dt = 0.0
    for i in range(iters):
        R.suite_advance(h, checkins)
        s = R.suite_export(h)
        keys = R.suite_keys(h, len(s["features"]))
        now = R.suite_checkin(h)
        t0 = time.perf_counter()
        log = tuner.run_iteration(i, s, keys, now)
        dt += time.perf_counter() - t0
    R.suite_free(h)
    res.update({"value": iters / dt, "unit": "iterations/s",
                "slots": int(len(s["slot_shader"])), "table_size": log["table_size"],
                "note": "device run_iteration (collection, run_benchmark, fold, snapshot, fit, "
                        "agreement); the environment export per iteration is not timed"})
    if not args.no_cpu_baseline:
        t = tuner.table.export()
        hv = o["has"].astype(bool)
        res["matches_reference_table"] = bool(
            np.array_equal(t["keys"], o["keys"]) and np.array_equal(t["has"], o["has"]) and
            np.array_equal(t["q"][hv], o["q"][hv]))
    return res


def qtable_tuples_torch(torch, n, seed):
    """Synthetic experience tuples on the device: ~0.8 n distinct StateKeys
    (stage < 8, counters < 4096), actions 0/1, rewards ~ U[0.8, 1.2),
    non-decreasing check-ins."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    nd = max(1, int(0.8 * n))
    base = torch.randint(0, 4096, (nd, 30), generator=g, device="cuda", dtype=torch.int64)
    base[:, 0] %= 8
    idx = torch.randint(0, nd, (n,), generator=g, device="cuda")
    keys = base[idx].to(torch.int32).contiguous()
    act = torch.randint(0, 2, (n,), generator=g, device="cuda", dtype=torch.uint8)
    rew = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 0.4 + 0.8
    now = torch.sort(torch.randint(0, 1000, (n,), generator=g, device="cuda")).values.contiguous()
    return keys, act, rew, now


def run_qtable(args, dev, stream, torch, gbx, peaks):
    n = args.qt_tuples
    keys, act, rew, now = qtable_tuples_torch(torch, n, 5)
    torch.cuda.synchronize()
    feat = torch.empty((n, 44), dtype=torch.float32, device="cuda")
    tgt = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    qt = gbx.DeviceQTable(dev)

    def once():  # fresh (cleared) table each time; device buffers reused
        qt.clear()
        qt.update_batch_dev(keys.data_ptr(), act.data_ptr(), rew.data_ptr(), now.data_ptr(), n)
        rows = qt.snapshot_dev(0.1, feat.data_ptr(), tgt.data_ptr(), n)
        return rows, qt.m_states()

    once()
    torch.cuda.synchronize()
    times = []
    for _ in range(5):  # median of 5 (each rep: fresh fold of all n tuples + snapshot)
        ev0.record(stream)
        rows, states = once()
        ev1.record(stream)
        torch.cuda.synchronize()
        times.append(ev0.elapsed_time(ev1))
    qt.close()
    del feat, tgt
    ms = statistics.median(times)
    res = {"value": n / (ms * 1e-3), "unit": "tuples/s (fold + snapshot)", "ms": ms, "tuples": n,
           "states": states, "snapshot_rows": rows,
           "algorithmic_bytes_per_tuple": 137,
           "hbm_gbs": n * 137 / (ms * 1e-3) / 1e9,
           "hbm_peak_gbs": peaks.get("hbm_gbs", HBM_PEAK_FALLBACK)}
    if not args.no_cpu_baseline:
        import oracle
        if oracle.ref_available():
            m = min(n, 200_000)
            k = keys[:m].cpu().numpy().view(np.uint32)
            t0 = time.perf_counter()
            oracle.Reference().qtable_fold(k, act[:m].cpu().numpy(), rew[:m].cpu().numpy(),
                                           now[:m].cpu().numpy().astype(np.uint64))
            dt = time.perf_counter() - t0
            res["cpu_baseline"] = {"value": m / dt, "unit": "tuples/s (fold + snapshot)",
                                   "cores": 1, "kind": "reference",
                                   "sample": f"{m} tuples of the same log, QTable::update + "
                                             f"snapshot_policy_dataset, {dt:.1f} s on 1 host core"}
    del keys, act, rew, now
    return res


if __name__ == "__main__":
    main()
