"""gbx-b200: B200-native (sm_100a) implementation of the gbxtune hot path.

Python binding of the C ABI in ``include/gbxcu.h`` (ctypes). The compute
lives in ``libgbxcu.so`` (CUDA kernels for sm_100a, built in-tree by
``build()``); this module only marshals buffers and maps status codes to the
reference's exception types (proj/include/gbx/core.hpp:14-16,
policy.hpp:16-31, qtable.hpp:15-25). There is no CPU fallback: if the library
or a B200 is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgbxcu.so")
N_PARAMS = 5026
N_FEATURES = 44
DIMS = (44, 64, 32, 2)
WAVE32, WAVE64 = 0, 1
FWD_EXACT, FWD_FAST = 0, 1

OK, EINVAL, EDIVERGED, ECUDA, ENCCL, ENONFINITE, ETEMPERATURE, ECLOCK = range(8)
KEY_WORDS = 30


# ----------------------------------------------------------------- errors
class ValidationError(ValueError):
    """gbx::ValidationError (proj/include/gbx/core.hpp:14-16)."""


class TrainingDivergedError(RuntimeError):
    """gbx::TrainingDivergedError{epoch} (proj/include/gbx/policy.hpp:25-30)."""

    def __init__(self, epoch: int, what: str):
        super().__init__(what)
        self.epoch = epoch


class InvalidTemperatureError(ValueError):
    """gbx::InvalidTemperatureError (proj/include/gbx/qtable.hpp:23-25)."""


class ClockRegressionError(RuntimeError):
    """gbx::ClockRegressionError (proj/include/gbx/qtable.hpp:15-17)."""


class CudaError(RuntimeError):
    """CUDA / device failure (no reference analogue: the reference is CPU-only)."""


class NcclError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile libgbxcu.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc")], check=True)
    return LIB_PATH


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_sz = C.c_size_t
_u64 = C.c_uint64


class TrainCfg(C.Structure):
    _fields_ = [("learning_rate", C.c_double), ("epochs", C.c_int), ("batch_size", C.c_int),
                ("seed", C.c_uint64), ("max_ctas", C.c_int), ("virtual_ranks", C.c_int),
                ("loss_mode", C.c_int), ("optimizer", C.c_int), ("adam_beta1", C.c_double),
                ("adam_beta2", C.c_double), ("adam_eps", C.c_double)]


LOSSES = {"kl": 0, "td": 1}
OPTIMIZERS = {"sgd": 0, "adam": 1}


def _train_cfg(lr, epochs, batch, seed, max_ctas, virtual_ranks, loss, optimizer, betas, eps):
    if loss not in LOSSES or optimizer not in OPTIMIZERS:
        raise ValueError(f"loss in {sorted(LOSSES)}, optimizer in {sorted(OPTIMIZERS)}")
    return TrainCfg(lr, epochs, batch, seed, max_ctas, virtual_ranks, LOSSES[loss],
                    OPTIMIZERS[optimizer], betas[0], betas[1], eps)


class SuiteC(C.Structure):
    _fields_ = [("n_apps", _sz), ("n_pipes", _sz), ("n_slots", _sz), ("n_shaders", _sz),
                ("app_pipe_off", _vp), ("pipe_slot_off", _vp), ("slot_shader", _vp),
                ("slot_frac", _vp), ("pipe_wt", _vp), ("shader_lat", _vp), ("app_f64", _vp)]


WIDE_PRECISION = {"tf32": 0, "bf16": 1}  # GBXCU_WIDE_TF32 / GBXCU_WIDE_BF16

# Every symbol include/gbxcu.h declares (tests check the library exports them).
EXPORTS = (
    "gbxcu_abi_version", "gbxcu_last_error", "gbxcu_create", "gbxcu_destroy", "gbxcu_stream",
    "gbxcu_launch_count", "gbxcu_policy_init", "gbxcu_forward", "gbxcu_forward_dev",
    "gbxcu_collect", "gbxcu_collect_dev", "gbxcu_batch_kl_loss", "gbxcu_batch_kl_gradient",
    "gbxcu_fit", "gbxcu_fit_dev", "gbxcu_fit_order", "gbxcu_comm_unique_id", "gbxcu_comm_init",
    "gbxcu_comm_destroy", "gbxcu_aggregate", "gbxcu_histogram", "gbxcu_suite_upload",
    "gbxcu_suite_free", "gbxcu_suite_features", "gbxcu_evaluate", "gbxcu_evaluate_dev",
    "gbxcu_wide_param_count", "gbxcu_wide_init", "gbxcu_wide_forward", "gbxcu_wide_fit",
    "gbxcu_wide_fit_dev", "gbxcu_wide_fit_ex", "gbxcu_wide_fit_ex_dev", "gbxcu_tf32_gemm",
    "gbxcu_bf16_gemm", "gbxcu_last_fit_timing", "gbxcu_last_eval_timing", "gbxcu_last_recheck_count", "gbxcu_peer_export",
    "gbxcu_peer_attach", "gbxcu_peer_detach", "gbxcu_qtable_create", "gbxcu_qtable_free", "gbxcu_qtable_clear",
    "gbxcu_qtable_update_batch", "gbxcu_qtable_update_batch_dev", "gbxcu_qtable_size",
    "gbxcu_forward_batch", "gbxcu_sample_batch", "gbxcu_evaluate_shard",
    "gbxcu_qtable_import", "gbxcu_qtable_export", "gbxcu_qtable_save_columnar",
    "gbxcu_qtable_load_columnar",
    "gbxcu_qtable_snapshot", "gbxcu_qtable_snapshot_dev",
)
PEER_HANDLE_BYTES = 64

_LIB = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libgbxcu.so (raises if absent — there is no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise CudaError(f"{path} is missing: run paper_2111_12055_b200.build() (no CPU fallback)")
    L = C.CDLL(path)
    L.gbxcu_abi_version.restype = C.c_int
    L.gbxcu_last_error.restype = C.c_char_p
    L.gbxcu_create.argtypes = [C.c_int, C.POINTER(_vp)]
    L.gbxcu_destroy.argtypes = [_vp]
    L.gbxcu_destroy.restype = None
    L.gbxcu_stream.argtypes = [_vp]
    L.gbxcu_stream.restype = _vp
    L.gbxcu_launch_count.argtypes = [_vp]
    L.gbxcu_launch_count.restype = _u64
    L.gbxcu_policy_init.argtypes = [_vp, _u64, _f32p]
    L.gbxcu_forward.argtypes = [_vp, _f32p, _f32p, _sz, _vp, _vp, C.c_int]
    L.gbxcu_forward_dev.argtypes = [_vp, _vp, _vp, _sz, _vp, _vp, C.c_int, _vp]
    L.gbxcu_collect.argtypes = [_vp, _f32p, _f32p, _u64p, _sz, _u64p, C.c_double, _u8p]
    L.gbxcu_collect_dev.argtypes = [_vp, _vp, _vp, _vp, _sz, _vp, _sz, C.c_double, _vp, _vp]
    L.gbxcu_batch_kl_loss.argtypes = [_vp, _f32p, _f32p, _f64p, _sz, C.POINTER(C.c_double)]
    L.gbxcu_batch_kl_gradient.argtypes = [_vp, _f32p, _f32p, _f64p, _sz, _f64p]
    L.gbxcu_fit.argtypes = [_vp, _f32p, _f32p, _f64p, _sz, C.POINTER(TrainCfg), _vp,
                            C.POINTER(C.c_int)]
    L.gbxcu_fit_dev.argtypes = [_vp, _vp, _vp, _vp, _sz, C.POINTER(TrainCfg), _vp,
                                C.POINTER(C.c_int), _vp]
    L.gbxcu_fit_order.argtypes = [_vp, _sz, _u64, C.c_int, _u32p]
    L.gbxcu_comm_unique_id.argtypes = [C.c_char_p]
    L.gbxcu_comm_init.argtypes = [_vp, C.c_char_p, C.c_int, C.c_int]
    L.gbxcu_comm_destroy.argtypes = [_vp]
    L.gbxcu_peer_export.argtypes = [_vp, C.c_char_p]
    L.gbxcu_peer_attach.argtypes = [_vp, C.c_int, C.c_int, C.c_char_p]
    L.gbxcu_peer_detach.argtypes = [_vp]
    L.gbxcu_qtable_create.argtypes = [_vp, C.c_double, C.c_double, C.POINTER(_vp)]
    L.gbxcu_qtable_free.argtypes = [_vp]
    L.gbxcu_qtable_free.restype = None
    L.gbxcu_qtable_clear.argtypes = [_vp]
    L.gbxcu_qtable_update_batch.argtypes = [_vp, _vp, _vp, _vp, _vp, _sz, C.POINTER(_sz)]
    L.gbxcu_qtable_update_batch_dev.argtypes = [_vp, _vp, _vp, _vp, _vp, _sz, C.POINTER(_sz)]
    L.gbxcu_qtable_size.argtypes = [_vp, C.POINTER(_sz), C.POINTER(_sz)]
    L.gbxcu_qtable_export.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
    L.gbxcu_qtable_import.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _sz]
    L.gbxcu_forward_batch.argtypes = [_vp, _vp, _vp, _sz, _vp, _vp]
    L.gbxcu_evaluate_shard.argtypes = [_vp, _vp, _vp, C.c_int, _u64, _sz, _sz, _vp]
    L.gbxcu_sample_batch.argtypes = [_vp, _vp, _vp, _sz, _u64, _vp]
    L.gbxcu_qtable_save_columnar.argtypes = [_vp, C.c_char_p]
    L.gbxcu_qtable_load_columnar.argtypes = [_vp, C.c_char_p]
    L.gbxcu_qtable_snapshot.argtypes = [_vp, C.c_double, _vp, _vp, _sz, C.POINTER(_sz)]
    L.gbxcu_qtable_snapshot_dev.argtypes = [_vp, C.c_double, _vp, _vp, _sz, C.POINTER(_sz)]
    L.gbxcu_aggregate.argtypes = [_vp, C.POINTER(SuiteC), _u8p, _u64p, C.c_int, _f64p, _vp]
    L.gbxcu_histogram.argtypes = [_vp, _f64p, _sz, _f64p, _u64p, _sz, C.POINTER(_sz)]
    L.gbxcu_suite_upload.argtypes = [_vp, C.POINTER(SuiteC), _f32p, C.POINTER(_vp)]
    L.gbxcu_suite_free.argtypes = [_vp]
    L.gbxcu_suite_free.restype = None
    L.gbxcu_suite_features.argtypes = [_vp]
    L.gbxcu_suite_features.restype = _vp
    L.gbxcu_evaluate.argtypes = [_vp, _vp, _f32p, C.c_int, _u64, _f64p, _vp, _vp, _vp, _sz,
                                 C.POINTER(_sz)]
    L.gbxcu_evaluate_dev.argtypes = [_vp, _vp, _vp, C.c_int, _u64, _vp, _vp, _vp]
    L.gbxcu_wide_param_count.argtypes = [C.c_int]
    L.gbxcu_wide_param_count.restype = _sz
    L.gbxcu_wide_init.argtypes = [_vp, C.c_int, _u64, _f32p]
    L.gbxcu_wide_forward.argtypes = [_vp, C.c_int, _f32p, _f32p, _sz, _f64p]
    L.gbxcu_wide_fit.argtypes = [_vp, C.c_int, _f32p, _f32p, _f64p, _sz, C.POINTER(TrainCfg), _vp,
                                 C.POINTER(C.c_int)]
    L.gbxcu_wide_fit_dev.argtypes = [_vp, C.c_int, _vp, _vp, _vp, _sz, C.POINTER(TrainCfg), _vp,
                                     C.POINTER(C.c_int), _vp]
    L.gbxcu_tf32_gemm.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _f32p, _f32p, _f32p]
    L.gbxcu_bf16_gemm.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _f32p, _f32p, _f32p]
    L.gbxcu_wide_fit_ex.argtypes = [_vp, C.c_int, C.c_int, _f32p, _f32p, _f64p, _sz, C.POINTER(TrainCfg), _vp,
                                    C.POINTER(C.c_int)]
    L.gbxcu_wide_fit_ex_dev.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _sz, C.POINTER(TrainCfg), _vp,
                                        C.POINTER(C.c_int), _vp]
    L.gbxcu_last_fit_timing.argtypes = [_vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.gbxcu_last_eval_timing.argtypes = [_vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.gbxcu_last_recheck_count.argtypes = [_vp, C.POINTER(C.c_uint64)]
    _LIB = L
    return L


def _raise(L, rc: int, diverged_epoch: int = -1):
    msg = (L.gbxcu_last_error() or b"").decode()
    if rc == EINVAL:
        raise ValidationError(msg)
    if rc == ENONFINITE:
        raise ValidationError(msg)
    if rc == EDIVERGED:
        raise TrainingDivergedError(diverged_epoch, msg)
    if rc == ETEMPERATURE:
        raise InvalidTemperatureError(msg)
    if rc == ENCCL:
        raise NcclError(msg)
    if rc == ECLOCK:
        raise ClockRegressionError(msg)
    raise CudaError(msg)


def _after_torch(stream) -> None:
    """Device-pointer entry points with stream=None run on the context's
    non-blocking stream, which does not order itself after torch's current
    stream: wait for torch's pending work (the producer of the caller's
    tensors) first. An explicit stream means the caller orders it."""
    if stream is not None:
        return
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        torch.cuda.current_stream().synchronize()


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def suite_struct(s: dict) -> tuple[SuiteC, list]:
    """Build the C view of a CSR suite dict (keys as in oracle export); returns (struct, keepalive)."""
    keep = [np.ascontiguousarray(s["app_pipe_off"], np.uint64),
            np.ascontiguousarray(s["pipe_slot_off"], np.uint64),
            np.ascontiguousarray(s["slot_shader"], np.uint32),
            np.ascontiguousarray(s["slot_frac"], np.float64),
            np.ascontiguousarray(s["pipe_wt"], np.float64),
            np.ascontiguousarray(s["shader_lat"], np.float64),
            np.ascontiguousarray(s["app_f64"], np.float64)]
    st = SuiteC(len(keep[0]) - 1, len(keep[1]) - 1, len(keep[2]), keep[5].shape[0],
                *(k.ctypes.data for k in keep))
    return st, keep


class Device:
    """One gbxcu context (device buffers + stream) on one B200."""

    def __init__(self, device: int = 0):
        self.L = load_library()
        h = _vp()
        rc = self.L.gbxcu_create(device, C.byref(h))
        if rc:
            _raise(self.L, rc)
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.L.gbxcu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc, diverged_epoch=-1):
        if rc:
            _raise(self.L, rc, diverged_epoch)

    @property
    def stream(self) -> int:
        return int(self.L.gbxcu_stream(self.h) or 0)

    @property
    def launches(self) -> int:
        return int(self.L.gbxcu_launch_count(self.h))

    def last_fit_timing(self):
        """(shuffle_ms, train_kernel_ms) of the last single-GPU fit (CUDA events)."""
        a, b = C.c_double(), C.c_double()
        self._ck(self.L.gbxcu_last_fit_timing(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def last_eval_timing(self):
        """(inference_ms, aggregate_ms) of the last evaluate on this context (CUDA events)."""
        a, b = C.c_double(), C.c_double()
        self._ck(self.L.gbxcu_last_eval_timing(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def last_recheck_count(self) -> int:
        """States of the last FAST forward re-checked on the exact fp64 path."""
        v = C.c_uint64()
        self._ck(self.L.gbxcu_last_recheck_count(self.h, C.byref(v)))
        return v.value

    # ------------------------------------------------------------ policy
    def policy_init(self, seed: int) -> np.ndarray:
        p = np.empty(N_PARAMS, np.float32)
        self._ck(self.L.gbxcu_policy_init(self.h, seed, p))
        return p

    def forward(self, params, feat, mode=FWD_EXACT, want_probs=True, want_actions=True):
        feat = _f32(feat).reshape(-1, N_FEATURES)
        n = feat.shape[0]
        probs = np.empty((n, 2), np.float64) if want_probs else None
        act = np.empty(n, np.uint8) if want_actions else None
        self._ck(self.L.gbxcu_forward(self.h, _f32(params), feat, n,
                                      None if probs is None else probs.ctypes.data,
                                      None if act is None else act.ctypes.data, mode))
        return probs, act

    def select_greedy(self, params, feat, mode=FWD_FAST):
        return self.forward(params, feat, mode, want_probs=False)[1]

    def sample_batch(self, params, feat, rng_state: int) -> np.ndarray:
        """select_sample over a batch from one SplitMix64 stream (state rng_state):
        state j uses the stream's (j+1)-th draw; the caller's stream advances n."""
        feat = _f32(feat).reshape(-1, N_FEATURES)
        act = np.empty(feat.shape[0], np.uint8)
        self._ck(self.L.gbxcu_sample_batch(self.h, _f32(params).ctypes.data, feat.ctypes.data,
                                           feat.shape[0], rng_state & ((1 << 64) - 1),
                                           act.ctypes.data))
        return act

    def collect(self, params, feat, seg_off, seg_seed, eps):
        feat = _f32(feat).reshape(-1, N_FEATURES)
        seg_off = np.ascontiguousarray(seg_off, np.uint64)
        act = np.empty(feat.shape[0], np.uint8)
        self._ck(self.L.gbxcu_collect(self.h, _f32(params), feat, seg_off, len(seg_off) - 1,
                                      np.ascontiguousarray(seg_seed, np.uint64), eps, act))
        return act

    def batch_kl_loss(self, params, feat, tgt) -> float:
        out = C.c_double()
        feat = _f32(feat).reshape(-1, N_FEATURES)
        self._ck(self.L.gbxcu_batch_kl_loss(self.h, _f32(params), feat, _f64(tgt), feat.shape[0],
                                            C.byref(out)))
        return out.value

    def batch_kl_gradient(self, params, feat, tgt) -> np.ndarray:
        g = np.empty(N_PARAMS, np.float64)
        feat = _f32(feat).reshape(-1, N_FEATURES)
        self._ck(self.L.gbxcu_batch_kl_gradient(self.h, _f32(params), feat, _f64(tgt),
                                                feat.shape[0], g))
        return g

    def fit(self, params, feat, tgt, lr=0.01, epochs=50, batch=32, seed=0, max_ctas=0,
            raise_on_diverge=True, virtual_ranks=0, loss="kl", optimizer="sgd",
            betas=(0.9, 0.999), eps=1e-8):
        """fit(): returns (params, epoch_loss). Raises TrainingDivergedError like the reference
        (the partially trained params are attached as .params). virtual_ranks > 1 runs the
        multi-GPU peer-set kernel path with that many ranks inside one launch.
        loss="td" (tgt rows = (action, reward); L = mean (Q(x,a) - r)^2) and
        optimizer="adam" are the north star's variants, absent from the reference."""
        p = np.array(params, np.float32, copy=True)
        feat = _f32(feat).reshape(-1, N_FEATURES)
        el = np.full(max(epochs, 1), np.nan, np.float64)
        de = C.c_int(-1)
        cfg = _train_cfg(lr, epochs, batch, seed, max_ctas, virtual_ranks, loss, optimizer, betas,
                         eps)
        rc = self.L.gbxcu_fit(self.h, p, feat, _f64(tgt), feat.shape[0], C.byref(cfg),
                              el.ctypes.data, C.byref(de))
        if rc == EDIVERGED and not raise_on_diverge:
            return p, el, de.value
        if rc:
            try:
                _raise(self.L, rc, de.value)
            except TrainingDivergedError as e:
                e.params = p
                raise
        return (p, el, -1) if not raise_on_diverge else (p, el)

    def fit_sharded(self, params, feat_local, tgt_local, lr=0.01, epochs=1, batch=32, seed=0,
                    group=None):
        """Data-parallel fit with the log SHARDED over the ranks of a
        torch.distributed group (one process per GPU): rank r passes records
        [r * n_local, (r + 1) * n_local) of the global log (host arrays,
        pinned for full PCIe rate). Each rank uploads only its shard; the
        shards are all-gathered on the device (NCCL over NVLink), then every
        rank trains its slice of each global batch (peer set or communicator
        attached beforehand; `batch` is the GLOBAL batch). Returns
        (params, epoch_loss) — identical on every rank."""
        import torch
        import torch.distributed as dist

        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        fl = np.ascontiguousarray(feat_local, np.float32).reshape(-1, N_FEATURES)
        tl = np.ascontiguousarray(tgt_local, np.float64).reshape(-1, 2)
        nl = fl.shape[0]
        n = nl * world
        buf = getattr(self, "_shard_bufs", None)
        if buf is None or buf[0].shape[0] != n:
            buf = (torch.empty((n, N_FEATURES), dtype=torch.float32, device="cuda"),
                   torch.empty((n, 2), dtype=torch.float64, device="cuda"),
                   torch.empty(N_PARAMS, dtype=torch.float32, device="cuda"))
            self._shard_bufs = buf
        fa, ta, pd = buf
        lo, hi = rank * nl, (rank + 1) * nl
        fa[lo:hi].copy_(torch.from_numpy(fl), non_blocking=True)
        ta[lo:hi].copy_(torch.from_numpy(tl), non_blocking=True)
        pd.copy_(torch.from_numpy(np.ascontiguousarray(params, np.float32)), non_blocking=True)
        if world > 1 and dist.get_backend(group) == "nccl":
            # in place: each rank's input is its own slice of the output
            dist.all_gather_into_tensor(fa, fa[lo:hi], group=group)
            dist.all_gather_into_tensor(ta, ta[lo:hi], group=group)
        elif world > 1:  # gloo (CPU test mode): gather through host tensors
            for dst, src in ((fa, fl), (ta, tl)):
                parts = [torch.empty_like(torch.from_numpy(src)) for _ in range(world)]
                dist.all_gather(parts, torch.from_numpy(src), group=group)
                dst.copy_(torch.cat(parts).to("cuda"))
        el = self.fit_dev(pd.data_ptr(), fa.data_ptr(), ta.data_ptr(), n, lr, epochs, batch, seed)
        return pd.cpu().numpy(), el

    def fit_order(self, n: int, seed: int, epochs: int) -> np.ndarray:
        o = np.empty(n, np.uint32)
        self._ck(self.L.gbxcu_fit_order(self.h, n, seed, epochs, o))
        return o

    # ------------------------------------------------- device-resident forms
    def forward_dev(self, d_params: int, d_feat: int, n: int, d_probs: int | None,
                    d_actions: int | None, mode=FWD_FAST, stream: int | None = None):
        _after_torch(stream)
        self._ck(self.L.gbxcu_forward_dev(self.h, d_params, d_feat, n, d_probs, d_actions, mode,
                                          stream))

    def fit_dev(self, d_params: int, d_feat: int, d_tgt: int, n: int, lr=0.01, epochs=1,
                batch=32, seed=0, max_ctas=0, stream: int | None = None, virtual_ranks=0,
                loss="kl", optimizer="sgd", betas=(0.9, 0.999), eps=1e-8):
        el = np.full(max(epochs, 1), np.nan, np.float64)
        de = C.c_int(-1)
        cfg = _train_cfg(lr, epochs, batch, seed, max_ctas, virtual_ranks, loss, optimizer, betas,
                         eps)
        _after_torch(stream)
        rc = self.L.gbxcu_fit_dev(self.h, d_params, d_feat, d_tgt, n, C.byref(cfg),
                                  el.ctypes.data, C.byref(de), stream)
        self._ck(rc, de.value)
        return el

    # ------------------------------------------------------ wide MLP (C4)
    def wide_param_count(self, hidden: int) -> int:
        return int(self.L.gbxcu_wide_param_count(hidden))

    def wide_init(self, hidden: int, seed: int) -> np.ndarray:
        p = np.empty(self.wide_param_count(hidden), np.float32)
        self._ck(self.L.gbxcu_wide_init(self.h, hidden, seed, p))
        return p

    def wide_forward(self, hidden: int, params, feat) -> np.ndarray:
        feat = _f32(feat).reshape(-1, N_FEATURES)
        probs = np.empty((feat.shape[0], 2), np.float64)
        self._ck(self.L.gbxcu_wide_forward(self.h, hidden, _f32(params), feat, feat.shape[0], probs))
        return probs

    def wide_fit(self, hidden: int, params, feat, tgt, lr=0.01, epochs=1, batch=32, seed=0,
                 precision="tf32"):
        p = np.array(params, np.float32, copy=True)
        feat = _f32(feat).reshape(-1, N_FEATURES)
        el = np.full(max(epochs, 1), np.nan, np.float64)
        de = C.c_int(-1)
        cfg = TrainCfg(lr, epochs, batch, seed, 0, 0)
        rc = self.L.gbxcu_wide_fit_ex(self.h, hidden, WIDE_PRECISION[precision], p, feat, _f64(tgt),
                                      feat.shape[0], C.byref(cfg), el.ctypes.data, C.byref(de))
        self._ck(rc, de.value)
        return p, el

    def wide_fit_dev(self, hidden, d_params, d_feat, d_tgt, n, lr=0.01, epochs=1, batch=32, seed=0,
                     stream=None, precision="tf32"):
        el = np.full(max(epochs, 1), np.nan, np.float64)
        de = C.c_int(-1)
        cfg = TrainCfg(lr, epochs, batch, seed, 0, 0)
        _after_torch(stream)
        self._ck(self.L.gbxcu_wide_fit_ex_dev(self.h, hidden, WIDE_PRECISION[precision], d_params, d_feat,
                                              d_tgt, n, C.byref(cfg), el.ctypes.data, C.byref(de), stream),
                 de.value)
        return el

    def tf32_gemm(self, A, B) -> np.ndarray:
        A, B = _f32(A), _f32(B)
        M, K = A.shape
        N = B.shape[0]
        D = np.empty((M, N), np.float32)
        self._ck(self.L.gbxcu_tf32_gemm(self.h, M, N, K, A, B, D))
        return D

    def bf16_gemm(self, A, B) -> np.ndarray:
        A, B = _f32(A), _f32(B)
        M, K = A.shape
        N = B.shape[0]
        D = np.empty((M, N), np.float32)
        self._ck(self.L.gbxcu_bf16_gemm(self.h, M, N, K, A, B, D))
        return D

    # ----------------------------------------------------------- data parallel
    @staticmethod
    def comm_unique_id() -> bytes:
        L = load_library()
        buf = C.create_string_buffer(128)
        rc = L.gbxcu_comm_unique_id(buf)
        if rc:
            _raise(L, rc)
        return buf.raw

    def comm_init(self, uid: bytes, nranks: int, rank: int):
        self._ck(self.L.gbxcu_comm_init(self.h, uid, nranks, rank))

    def comm_destroy(self):
        self._ck(self.L.gbxcu_comm_destroy(self.h))

    # fused data-parallel path over NVLink peer memory (see include/gbxcu.h)
    def peer_export(self) -> bytes:
        buf = C.create_string_buffer(PEER_HANDLE_BYTES)
        self._ck(self.L.gbxcu_peer_export(self.h, buf))
        return buf.raw

    def peer_attach(self, handles: list, rank: int):
        blob = b"".join(bytes(h) for h in handles)
        assert len(blob) == PEER_HANDLE_BYTES * len(handles)
        self._ck(self.L.gbxcu_peer_attach(self.h, len(handles), rank, blob))

    def peer_detach(self):
        self._ck(self.L.gbxcu_peer_detach(self.h))

    # ------------------------------------------------------------ aggregation
    def aggregate(self, suite: dict, shader_actions, run_seed, n_samples, want_samples=False):
        st, keep = suite_struct(suite)
        rows = np.empty((st.n_apps, 5), np.float64)
        samples = np.empty((st.n_apps, n_samples), np.float64) if want_samples else None
        self._ck(self.L.gbxcu_aggregate(self.h, C.byref(st),
                                        np.ascontiguousarray(shader_actions, np.uint8),
                                        np.ascontiguousarray(run_seed, np.uint64), n_samples, rows,
                                        None if samples is None else samples.ctypes.data))
        return (rows, samples) if want_samples else rows

    def histogram(self, uplift):
        u = _f64(uplift)
        cap = 1 << 16
        lo = np.empty(cap, np.float64)
        cnt = np.empty(cap, np.uint64)
        nb = _sz()
        self._ck(self.L.gbxcu_histogram(self.h, u, len(u), lo, cnt, cap, C.byref(nb)))
        return lo[:nb.value].copy(), cnt[:nb.value].copy()

    def suite_upload(self, suite: dict, features) -> "DeviceSuite":
        return DeviceSuite(self, suite, features)

    def suite_upload_dev(self, suite: dict, features) -> "DeviceSuite":
        """Suite whose arrays are torch CUDA tensors (keys as suite_upload)."""
        return DeviceSuite(self, suite, features, device_arrays=True)


class DeviceSuite:
    """A suite resident in HBM (gbxcu_suite_upload)."""

    def __init__(self, dev: Device, suite: dict, features, device_arrays=False):
        self.dev = dev
        if device_arrays:
            names = ("app_pipe_off", "pipe_slot_off", "slot_shader", "slot_frac", "pipe_wt",
                     "shader_lat", "app_f64")
            t = [suite[k].contiguous() for k in names]
            st = SuiteC(t[0].numel() - 1, t[1].numel() - 1, t[2].numel(), t[5].shape[0],
                        *(x.data_ptr() for x in t))
            fptr = features.contiguous().data_ptr()
            _after_torch(None)  # the tensors may still be in flight on torch's stream
        else:
            st, keep = suite_struct(suite)
            fptr = _f32(features).ctypes.data
        self.n_apps, self.n_shaders = st.n_apps, st.n_shaders
        h = _vp()
        L = dev.L
        L.gbxcu_suite_upload.argtypes = [_vp, C.POINTER(SuiteC), _vp, C.POINTER(_vp)]
        dev._ck(L.gbxcu_suite_upload(dev.h, C.byref(st), fptr, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.dev.L.gbxcu_suite_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def features_ptr(self) -> int:
        return int(self.dev.L.gbxcu_suite_features(self.h))

    def evaluate(self, params, n_samples: int, seed: int, want_actions=False):
        """evaluate(): rows [n_apps][5], histogram (lower, count), optional shader actions."""
        rows = np.empty((self.n_apps, 5), np.float64)
        act = np.empty(self.n_shaders, np.uint8) if want_actions else None
        cap = 1 << 16
        lo = np.empty(cap, np.float64)
        cnt = np.empty(cap, np.uint64)
        nb = _sz()
        self.dev._ck(self.dev.L.gbxcu_evaluate(
            self.dev.h, self.h, _f32(params), n_samples, seed, rows,
            None if act is None else act.ctypes.data, lo.ctypes.data, cnt.ctypes.data, cap,
            C.byref(nb)))
        hist = (lo[:nb.value].copy(), cnt[:nb.value].copy())
        return (rows, hist, act) if want_actions else (rows, hist)

    def evaluate_shard(self, params, n_samples: int, seed: int, app_lo: int, app_hi: int):
        """Rows [app_hi - app_lo][5] of one app-range shard (gbxcu_evaluate_shard):
        concatenating the shards' rows gives evaluate()'s rows bit for bit."""
        rows = np.empty((max(0, app_hi - app_lo), 5), np.float64)
        self.dev._ck(self.dev.L.gbxcu_evaluate_shard(self.dev.h, self.h, _f32(params).ctypes.data,
                                                     n_samples, seed & ((1 << 64) - 1), app_lo,
                                                     app_hi, rows.ctypes.data))
        return rows

    def evaluate_distributed(self, params, n_samples: int, seed: int, rank: int, world: int,
                             group=None):
        """evaluate() sharded by app range over `world` ranks (torch.distributed,
        any backend): each rank evaluates its range, rank 0 gathers the rows in
        app order and builds the histogram. Returns (rows, hist) on rank 0,
        (own rows, None) elsewhere."""
        import torch.distributed as dist
        per = (self.n_apps + world - 1) // world
        lo, hi = min(self.n_apps, rank * per), min(self.n_apps, (rank + 1) * per)
        mine = self.evaluate_shard(params, n_samples, seed, lo, hi)
        parts = [None] * world if rank == 0 else None
        dist.gather_object(mine, parts, dst=0, group=group)
        if rank != 0:
            return mine, None
        rows = np.concatenate([p for p in parts if len(p)], axis=0)
        return rows, self.dev.histogram(rows[:, 3])

    def evaluate_dev(self, d_params: int, n_samples: int, seed: int, d_actions: int, d_rows: int,
                     stream: int | None = None):
        _after_torch(stream)
        self.dev._ck(self.dev.L.gbxcu_evaluate_dev(self.dev.h, self.h, d_params, n_samples, seed,
                                                   d_actions, d_rows, stream))


def _parse_u64(tok: str, what: str) -> int:
    if not tok.isdigit() or int(tok) >= 1 << 64:
        raise ValidationError(f"bad q-table field: {what}")
    return int(tok)


def _parse_f64(tok: str, what: str) -> float:
    try:
        return float(tok)
    except ValueError:
        raise ValidationError(f"bad q-table field: {what}") from None


class DeviceQTable:
    """QTable on the device (proj/include/gbx/qtable.hpp:53-100): batched
    QTable::update (Eq. 5) and snapshot_policy_dataset in key order."""

    def __init__(self, dev: "Device", alpha: float = 0.3, omega: float = 1.0):
        self.dev, self.L = dev, dev.L
        h = _vp()
        dev._ck(self.L.gbxcu_qtable_create(dev.h, alpha, omega, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.L.gbxcu_qtable_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def update_batch(self, keys, actions, rewards, now):
        keys = np.ascontiguousarray(keys, np.uint32).reshape(-1, KEY_WORDS)
        actions = np.ascontiguousarray(actions, np.uint8)
        rewards = np.ascontiguousarray(rewards, np.float64)
        now = np.ascontiguousarray(now, np.uint64)
        bad = _sz(0)
        rc = self.L.gbxcu_qtable_update_batch(self.h, keys.ctypes.data, actions.ctypes.data,
                                              rewards.ctypes.data, now.ctypes.data, len(actions),
                                              C.byref(bad))
        if rc == ECLOCK:
            try:
                _raise(self.L, rc)
            except ClockRegressionError as e:
                e.index = int(bad.value)
                raise
        self.dev._ck(rc)

    def clear(self):
        self.dev._ck(self.L.gbxcu_qtable_clear(self.h))

    def update_batch_dev(self, d_keys: int, d_actions: int, d_rewards: int, d_now: int, n: int):
        bad = _sz(0)
        _after_torch(None)
        rc = self.L.gbxcu_qtable_update_batch_dev(self.h, d_keys, d_actions, d_rewards, d_now, n,
                                                  C.byref(bad))
        if rc == ECLOCK:
            try:
                _raise(self.L, rc)
            except ClockRegressionError as e:
                e.index = int(bad.value)
                raise
        self.dev._ck(rc)

    def m_states(self) -> int:
        m = _sz(0)
        self.dev._ck(self.L.gbxcu_qtable_size(self.h, C.byref(m), None))
        return int(m.value)

    def size(self):
        m, e = _sz(0), _sz(0)
        self.dev._ck(self.L.gbxcu_qtable_size(self.h, C.byref(m), C.byref(e)))
        return int(m.value), int(e.value)

    def export(self) -> dict:
        m, _ = self.size()
        out = {"keys": np.empty((m, KEY_WORDS), np.uint32), "q": np.empty((m, 2)),
               "t": np.empty((m, 2), np.uint64), "cnt": np.empty((m, 2), np.uint64),
               "has": np.empty((m, 2), np.uint8)}
        if m:
            self.dev._ck(self.L.gbxcu_qtable_export(self.h, *(out[k].ctypes.data for k in
                                                              ("keys", "q", "t", "cnt", "has"))))
        return out

    def import_arrays(self, t: dict):
        m = len(t["keys"])
        arrs = [np.ascontiguousarray(t["keys"], np.uint32), np.ascontiguousarray(t["q"], np.float64),
                np.ascontiguousarray(t["t"], np.uint64), np.ascontiguousarray(t["cnt"], np.uint64),
                np.ascontiguousarray(t["has"], np.uint8)]
        self.dev._ck(self.L.gbxcu_qtable_import(self.h, *(a.ctypes.data for a in arrs), m))

    def save_columnar(self, path: str):
        """Binary columnar table file (include/gbxcu.h: gbxcu_qtable_save_columnar)."""
        self.dev._ck(self.L.gbxcu_qtable_save_columnar(self.h, os.fsencode(path)))

    @classmethod
    def load_columnar(cls, dev: "Device", path: str) -> "DeviceQTable":
        """The columnar file straight onto the device (table + alpha/omega)."""
        self = cls(dev)
        dev._ck(self.L.gbxcu_qtable_load_columnar(self.h, os.fsencode(path)))
        return self

    @classmethod
    def load(cls, dev: "Device", text: str) -> "DeviceQTable":
        """QTable::load (proj/src/qtable.cpp:188-231): the line-text table
        (header `gbx-qtable 1 alpha omega`, then `key[30] action q t count`
        records), parsed with the reference's validation, then placed on the
        device (ready for snapshot -> fit)."""
        lines = text.split("\n")
        head = lines[0].split() if lines and lines[0] else []
        if not head:
            raise ValidationError("empty q-table file")
        if len(head) != 4 or head[0] != "gbx-qtable":
            raise ValidationError("not a q-table file")
        if _parse_u64(head[1], "version") != 1:
            raise ValidationError("unsupported q-table format version")
        alpha, omega = _parse_f64(head[2], "alpha"), _parse_f64(head[3], "omega")
        self = cls(dev, alpha, omega)
        entries = {}
        for ln, line in enumerate(lines[1:], start=2):
            if not line:
                continue
            tok = line.split(" ")
            tok = [x for x in tok if x]
            if len(tok) != KEY_WORDS + 4:
                raise ValidationError(f"malformed q-table record at line {ln}")
            key = tuple(_parse_u64(x, "key") & 0xFFFFFFFF for x in tok[:KEY_WORDS])
            a = _parse_u64(tok[KEY_WORDS], "action")
            if a not in (0, 1):
                raise ValidationError(f"bad action index at line {ln}")
            q = _parse_f64(tok[KEY_WORDS + 1], "q")
            t = _parse_u64(tok[KEY_WORDS + 2], "last_update_t")
            n = _parse_u64(tok[KEY_WORDS + 3], "update_count")
            if n == 0:
                raise ValidationError("stored entry with zero update count")
            entries.setdefault(key, [None, None])[a] = (q, t, n)
        keys = sorted(entries)
        m = len(keys)
        arr = {"keys": np.array(keys, np.uint32).reshape(m, KEY_WORDS), "q": np.zeros((m, 2)),
               "t": np.zeros((m, 2), np.uint64), "cnt": np.zeros((m, 2), np.uint64),
               "has": np.zeros((m, 2), np.uint8)}
        for r, k in enumerate(keys):
            for a, e in enumerate(entries[k]):
                if e is not None:
                    arr["q"][r, a], arr["t"][r, a], arr["cnt"][r, a] = e
                    arr["has"][r, a] = 1
        self.import_arrays(arr)
        return self

    def snapshot(self, rho: float):
        r = _sz(0)
        self.dev._ck(self.L.gbxcu_qtable_snapshot(self.h, rho, None, None, 0, C.byref(r)))
        feat = np.empty((r.value, N_FEATURES), np.float32)
        tgt = np.empty((r.value, 2), np.float64)
        self.dev._ck(self.L.gbxcu_qtable_snapshot(self.h, rho, feat.ctypes.data, tgt.ctypes.data,
                                                  r.value, C.byref(r)))
        return feat, tgt

    def snapshot_dev(self, rho: float, d_feat: int, d_tgt: int, cap: int) -> int:
        r = _sz(0)
        _after_torch(None)
        self.dev._ck(self.L.gbxcu_qtable_snapshot_dev(self.h, rho, d_feat, d_tgt, cap, C.byref(r)))
        return int(r.value)
