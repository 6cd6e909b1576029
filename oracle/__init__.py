"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Python bindings (ctypes + numpy) for
  * ``liboracle.so``   — our C restatement of the reference hot path
                         (oracle/gbx_oracle.c, every function cites the
                         reference file:line it restates), and
  * ``_ref/libgbxref.so`` — the unmodified reference library compiled from
                         /root/reference/proj/src (oracle/Makefile) behind the
                         adapter oracle/ref_capi.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker.
The product package (paper_2111_12055_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
N_PARAMS = 5026
N_FEAT = 44
DIMS = (44, 64, 32, 2)

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_u64 = C.c_uint64


def build(ref: bool = True) -> None:
    """Compile the restatement (always) and the reference (.so) if its sources exist."""
    targets = ["restatement"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _opt(arr, dtype):
    return None if arr is None else np.ascontiguousarray(arr, dtype=dtype)


class _Lib:
    def __init__(self, path: str):
        self.path = path
        self.lib = C.CDLL(path)


# --------------------------------------------------------------------------
# Restatement
# --------------------------------------------------------------------------
class Restatement(_Lib):
    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        super().__init__(path)
        L = self.lib
        L.orc_mix64.restype = _u64
        L.orc_mix64.argtypes = [_u64]
        L.orc_derive_seed.restype = _u64
        L.orc_derive_seed.argtypes = [_u64p, C.c_int]
        L.orc_g1.argtypes = [_u64, _sz, _f32p, C.c_void_p]
        L.orc_policy_init.argtypes = [_u64, _f32p]
        L.orc_policy_init_dims.argtypes = [_u64, _i32p, C.c_int, _f32p]
        L.orc_param_count.restype = _sz
        L.orc_param_count.argtypes = [_i32p, C.c_int]
        L.orc_forward.restype = C.c_long
        L.orc_forward.argtypes = [_f32p, _f32p, _sz, C.c_void_p, C.c_void_p]
        L.orc_forward_dims.restype = C.c_long
        L.orc_forward_dims.argtypes = [_f32p, _i32p, C.c_int, _f32p, _sz, C.c_void_p, C.c_void_p]
        L.orc_logits.argtypes = [_f32p, _f32p, _sz, _f64p]
        L.orc_kl_loss.restype = C.c_double
        L.orc_kl_loss.argtypes = [C.c_double] * 4
        L.orc_batch_kl_loss.restype = C.c_double
        L.orc_batch_kl_loss.argtypes = [_f32p, _f32p, _f64p, _sz]
        L.orc_batch_kl_gradient.argtypes = [_f32p, _f32p, _f64p, _sz, _f64p]
        L.orc_batch_kl_gradient_dims.argtypes = [_f32p, _i32p, C.c_int, _f32p, _f64p, _sz, _f64p]
        L.orc_fit_order.argtypes = [_sz, _u64, C.c_int, _u64p]
        L.orc_fit.restype = C.c_int
        L.orc_fit.argtypes = [_f32p, _f32p, _f64p, _sz, C.c_double, C.c_int, C.c_int, _u64,
                              C.c_long, _f64p, C.POINTER(C.c_int)]
        L.orc_fit_dims.restype = C.c_int
        L.orc_fit_dims.argtypes = [_f32p, _i32p, C.c_int, _f32p, _f64p, _sz, C.c_double, C.c_int,
                                   C.c_int, _u64, C.c_long, _f64p, C.POINTER(C.c_int)]
        L.orc_collect.argtypes = [_f32p, _f32p, _u64p, _sz, _u64p, C.c_double, _u8p]
        L.orc_aggregate.argtypes = [_sz, _u64p, _u64p, _u32p, _f64p, _f64p, _f64p, _f64p, _u8p,
                                    _u64p, C.c_int, _f64p, C.c_void_p]
        L.orc_aggregate_ids.argtypes = [_sz, _u64p, _u64p, _u32p, _f64p, _f64p, _f64p, _f64p, _u8p,
                                        _u64p, C.c_void_p, C.c_int, _f64p, C.c_void_p]
        L.orc_histogram.restype = C.c_long
        L.orc_histogram.argtypes = [_f64p, _sz, _f64p, _u64p, _sz]
        L.orc_boltzmann_pair.argtypes = [C.c_double, C.c_double, C.c_double, _f64p]
        L.orc_partial_gradient.argtypes = [_f32p, _f32p, _f64p, _u64p, _sz, C.c_double, _f64p,
                                           C.POINTER(C.c_double)]
        L.orc_fit_variant.argtypes = [_f32p, _f32p, _f64p, _sz, C.c_double, C.c_int, C.c_int, _u64,
                                      C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _f64p,
                                      C.POINTER(C.c_int)]
        L.orc_log1pf_counts.restype = C.c_float
        L.orc_log1pf_counts.argtypes = [C.c_float]
        L.orc_fnv1a.restype = _u64
        L.orc_fnv1a.argtypes = [C.c_void_p, _sz]

    # rng ------------------------------------------------------------------
    def mix64(self, x: int) -> int:
        return int(self.lib.orc_mix64(x))

    def derive_seed(self, *parts: int) -> int:
        p = np.array(parts, dtype=np.uint64)
        return int(self.lib.orc_derive_seed(p, len(parts)))

    # inputs ---------------------------------------------------------------
    def g1(self, seed: int, n: int):
        feat = np.empty((n, N_FEAT), np.float32)
        tgt = np.empty((n, 2), np.float64)
        self.lib.orc_g1(seed, n, feat, tgt.ctypes.data)
        return feat, tgt

    # policy ---------------------------------------------------------------
    def policy_init(self, seed: int, dims=DIMS) -> np.ndarray:
        d = np.array(dims, np.int32)
        p = np.empty(self.lib.orc_param_count(d, len(dims) - 1), np.float32)
        self.lib.orc_policy_init_dims(seed, d, len(dims) - 1, p)
        return p

    def forward(self, params, feat, dims=DIMS):
        feat = np.ascontiguousarray(feat, np.float32)
        n = feat.shape[0]
        probs = np.empty((n, 2), np.float64)
        act = np.empty(n, np.uint8)
        d = np.array(dims, np.int32)
        bad = self.lib.orc_forward_dims(np.ascontiguousarray(params, np.float32), d, len(dims) - 1,
                                        feat, n, probs.ctypes.data, act.ctypes.data)
        if bad >= 0:
            raise ValueError(f"non-finite feature in shader state {bad}")
        return probs, act

    def logits(self, params, feat):
        feat = np.ascontiguousarray(feat, np.float32)
        out = np.empty((feat.shape[0], 2), np.float64)
        self.lib.orc_logits(np.ascontiguousarray(params, np.float32), feat, feat.shape[0], out)
        return out

    def kl_loss(self, p, t) -> float:
        return float(self.lib.orc_kl_loss(p[0], p[1], t[0], t[1]))

    def batch_kl_loss(self, params, feat, tgt) -> float:
        return float(self.lib.orc_batch_kl_loss(np.ascontiguousarray(params, np.float32),
                                                np.ascontiguousarray(feat, np.float32),
                                                np.ascontiguousarray(tgt, np.float64),
                                                feat.shape[0]))

    def batch_kl_gradient(self, params, feat, tgt, dims=DIMS):
        d = np.array(dims, np.int32)
        g = np.empty(self.lib.orc_param_count(d, len(dims) - 1), np.float64)
        self.lib.orc_batch_kl_gradient_dims(np.ascontiguousarray(params, np.float32), d,
                                            len(dims) - 1, np.ascontiguousarray(feat, np.float32),
                                            np.ascontiguousarray(tgt, np.float64), feat.shape[0], g)
        return g

    def fit_order(self, n: int, seed: int, epochs: int):
        o = np.empty(n, np.uint64)
        self.lib.orc_fit_order(n, seed, epochs, o)
        return o

    def partial_gradient(self, params, feat, tgt, idx, inv_batch):
        idx = np.ascontiguousarray(idx, np.uint64)
        g = np.empty(N_PARAMS, np.float64)
        ls = C.c_double()
        self.lib.orc_partial_gradient(np.ascontiguousarray(params, np.float32),
                                      np.ascontiguousarray(feat, np.float32),
                                      np.ascontiguousarray(tgt, np.float64), idx, len(idx),
                                      inv_batch, g, C.byref(ls))
        return g, ls.value

    def fit(self, params, feat, tgt, lr=0.01, epochs=1, batch=32, seed=0, max_steps=0,
            dims=DIMS):
        """Returns (rc, params_out, epoch_loss, diverged_epoch)."""
        p = np.array(params, np.float32, copy=True)
        el = np.full(max(epochs, 1), np.nan, np.float64)
        de = C.c_int(-1)
        d = np.array(dims, np.int32)
        rc = self.lib.orc_fit_dims(p, d, len(dims) - 1, np.ascontiguousarray(feat, np.float32),
                                   np.ascontiguousarray(tgt, np.float64), feat.shape[0], lr,
                                   epochs, batch, seed, max_steps, el, C.byref(de))
        return rc, p, el, de.value

    def fit_variant(self, params, feat, tgt, lr=0.01, epochs=1, batch=32, seed=0, loss="kl",
                    optimizer="sgd", beta1=0.9, beta2=0.999, eps=1e-8):
        """The TD-regression / Adam variants (parity unpinned by the reference).
        Returns (rc, params_out, epoch_loss, diverged_epoch)."""
        p = np.array(params, np.float32, copy=True)
        el = np.full(max(epochs, 1), np.nan, np.float64)
        de = C.c_int(-1)
        rc = self.lib.orc_fit_variant(p, np.ascontiguousarray(feat, np.float32),
                                      np.ascontiguousarray(tgt, np.float64), feat.shape[0], lr, epochs,
                                      batch, seed, 1 if loss == "td" else 0,
                                      1 if optimizer == "adam" else 0, beta1, beta2, eps, el,
                                      C.byref(de))
        return rc, p, el, de.value

    def collect(self, params, feat, seg_off, seg_seed, eps):
        feat = np.ascontiguousarray(feat, np.float32)
        act = np.empty(feat.shape[0], np.uint8)
        seg_off = np.ascontiguousarray(seg_off, np.uint64)
        self.lib.orc_collect(np.ascontiguousarray(params, np.float32), feat, seg_off,
                             len(seg_off) - 1, np.ascontiguousarray(seg_seed, np.uint64), eps, act)
        return act

    def aggregate(self, suite: dict, shader_action, run_seed, n_samples: int, want_samples=False,
                  app_ids=None):
        """app_ids: benchmark id per app (noise stream seed part), default the index."""
        napps = len(suite["app_pipe_off"]) - 1
        rows = np.empty((napps, 5), np.float64)
        samples = np.empty((napps, n_samples), np.float64) if want_samples else None
        ids = None if app_ids is None else np.ascontiguousarray(app_ids, np.uint64)
        self.lib.orc_aggregate_ids(
            napps, suite["app_pipe_off"], suite["pipe_slot_off"], suite["slot_shader"],
            suite["slot_frac"], suite["pipe_wt"], suite["shader_lat"], suite["app_f64"],
            np.ascontiguousarray(shader_action, np.uint8), np.ascontiguousarray(run_seed, np.uint64),
            None if ids is None else ids.ctypes.data, n_samples, rows,
            None if samples is None else samples.ctypes.data)
        return (rows, samples) if want_samples else rows

    def histogram(self, uplift):
        uplift = np.ascontiguousarray(uplift, np.float64)
        cap = 1 << 16
        lo = np.empty(cap, np.float64)
        cnt = np.empty(cap, np.uint64)
        nb = self.lib.orc_histogram(uplift, len(uplift), lo, cnt, cap)
        return lo[:nb].copy(), cnt[:nb].copy()

    def boltzmann_pair(self, q0, q1, rho):
        out = np.empty(2, np.float64)
        self.lib.orc_boltzmann_pair(q0, q1, rho, out)
        return out

    def fnv1a(self, arr) -> int:
        arr = np.ascontiguousarray(arr)
        return int(self.lib.orc_fnv1a(arr.ctypes.data, arr.nbytes))


# --------------------------------------------------------------------------
# Compiled reference
# --------------------------------------------------------------------------
REF_PATH = os.path.join(HERE, "_ref", "libgbxref.so")


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


class Reference(_Lib):
    def __init__(self, path: str = REF_PATH):
        super().__init__(path)
        L = self.lib
        L.gbxref_last_error.restype = C.c_char_p
        L.gbxref_g1.argtypes = [_u64, _sz, _f32p, C.c_void_p]
        L.gbxref_policy_init.argtypes = [_u64, _f32p]
        L.gbxref_forward.restype = C.c_int
        L.gbxref_forward.argtypes = [_f32p, _f32p, _sz, C.c_void_p, C.c_void_p]
        L.gbxref_kl_loss.restype = C.c_double
        L.gbxref_kl_loss.argtypes = [C.c_double] * 4
        L.gbxref_batch_kl_loss.restype = C.c_double
        L.gbxref_batch_kl_loss.argtypes = [_f32p, _f32p, _f64p, _sz]
        L.gbxref_batch_kl_gradient.argtypes = [_f32p, _f32p, _f64p, _sz, _f64p]
        L.gbxref_fit.restype = C.c_int
        L.gbxref_fit.argtypes = [_f32p, _f32p, _f64p, _sz, C.c_double, C.c_int, C.c_int, _u64,
                                 _f64p, C.POINTER(C.c_int)]
        L.gbxref_fit_order.argtypes = [_sz, _u64, C.c_int, _u64p]
        L.gbxref_derive_seed3.restype = _u64
        L.gbxref_derive_seed3.argtypes = [_u64, _u64, _u64]
        L.gbxref_reward_from_framerate.restype = C.c_int
        L.gbxref_reward_from_framerate.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.gbxref_attribute_reward.restype = C.c_int
        L.gbxref_attribute_reward.argtypes = [_f64p, _sz, C.c_double, C.POINTER(C.c_double)]
        L.gbxref_boltzmann_pair.argtypes = [C.c_double, C.c_double, C.c_double, _f64p]
        L.gbxref_qtable_snapshot.restype = C.c_long
        L.gbxref_qtable_snapshot.argtypes = [C.c_char_p, C.c_double, C.c_void_p, C.c_void_p]
        L.gbxref_qtable_fold.restype = C.c_long
        L.gbxref_qtable_fold.argtypes = [C.c_void_p] * 4 + [_sz, C.c_double, C.c_double, C.c_double,
                                                            C.c_void_p, C.c_void_p] + [C.c_void_p] * 7
        L.gbxref_suite_advance.argtypes = [C.c_void_p, _u64]
        L.gbxref_suite_checkin.restype = _u64
        L.gbxref_suite_checkin.argtypes = [C.c_void_p]
        L.gbxref_suite_keys.argtypes = [C.c_void_p, C.c_void_p]
        L.gbxref_run_training.restype = C.c_long
        L.gbxref_run_training.argtypes = ([C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                          C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                          C.c_double, C.c_double, C.c_double, _u64] + [C.c_void_p] * 7)
        L.gbxref_suite_generate.restype = C.c_void_p
        L.gbxref_suite_generate.argtypes = [C.c_int] * 5 + [C.c_double] * 3 + [_u64]
        L.gbxref_suite_free.argtypes = [C.c_void_p]
        L.gbxref_suite_dims.argtypes = [C.c_void_p, _u64p]
        L.gbxref_suite_export.argtypes = [C.c_void_p, _f64p, _f32p, _f64p, _u64p, _f64p, _u64p,
                                          _u32p, _f64p, _u64p, _u32p]
        L.gbxref_run_benchmark.restype = C.c_int
        L.gbxref_run_benchmark.argtypes = [C.c_void_p, C.c_uint32, _u8p, C.c_int, _u64, _f64p]
        L.gbxref_evaluate.restype = C.c_long
        L.gbxref_evaluate.argtypes = [C.c_void_p, _f32p, C.c_int, _u64, C.c_int, _f64p, _f64p,
                                      _u64p, _sz]

    def err(self) -> str:
        return self.lib.gbxref_last_error().decode()

    def g1(self, seed: int, n: int):
        feat = np.empty((n, N_FEAT), np.float32)
        tgt = np.empty((n, 2), np.float64)
        self.lib.gbxref_g1(seed, n, feat, tgt.ctypes.data)
        return feat, tgt

    def policy_init(self, seed: int):
        p = np.empty(N_PARAMS, np.float32)
        self.lib.gbxref_policy_init(seed, p)
        return p

    def forward(self, params, feat):
        feat = np.ascontiguousarray(feat, np.float32)
        n = feat.shape[0]
        probs = np.empty((n, 2), np.float64)
        act = np.empty(n, np.uint8)
        if self.lib.gbxref_forward(np.ascontiguousarray(params, np.float32), feat, n,
                                   probs.ctypes.data, act.ctypes.data):
            raise ValueError(self.err())
        return probs, act

    def select_greedy(self, params, feat):
        feat = np.ascontiguousarray(feat, np.float32)
        act = np.empty(feat.shape[0], np.uint8)
        if self.lib.gbxref_forward(np.ascontiguousarray(params, np.float32), feat,
                                   feat.shape[0], None, act.ctypes.data):
            raise ValueError(self.err())
        return act

    def kl_loss(self, p, t) -> float:
        return float(self.lib.gbxref_kl_loss(p[0], p[1], t[0], t[1]))

    def batch_kl_loss(self, params, feat, tgt) -> float:
        return float(self.lib.gbxref_batch_kl_loss(np.ascontiguousarray(params, np.float32),
                                                   np.ascontiguousarray(feat, np.float32),
                                                   np.ascontiguousarray(tgt, np.float64),
                                                   feat.shape[0]))

    def batch_kl_gradient(self, params, feat, tgt):
        g = np.empty(N_PARAMS, np.float64)
        self.lib.gbxref_batch_kl_gradient(np.ascontiguousarray(params, np.float32),
                                          np.ascontiguousarray(feat, np.float32),
                                          np.ascontiguousarray(tgt, np.float64), feat.shape[0], g)
        return g

    def fit(self, params, feat, tgt, lr=0.01, epochs=1, batch=32, seed=0):
        p = np.array(params, np.float32, copy=True)
        el = np.full(max(epochs, 1), np.nan, np.float64)
        de = C.c_int(-1)
        rc = self.lib.gbxref_fit(p, np.ascontiguousarray(feat, np.float32),
                                 np.ascontiguousarray(tgt, np.float64), feat.shape[0], lr, epochs,
                                 batch, seed, el, C.byref(de))
        return rc, p, el, de.value

    def fit_order(self, n, seed, epochs):
        o = np.empty(n, np.uint64)
        self.lib.gbxref_fit_order(n, seed, epochs, o)
        return o

    def derive_seed3(self, a, b, c) -> int:
        return int(self.lib.gbxref_derive_seed3(a, b, c))

    def reward_from_framerate(self, obs, base):
        out = C.c_double()
        if self.lib.gbxref_reward_from_framerate(obs, base, C.byref(out)):
            raise ValueError(self.err())
        return out.value

    def attribute_reward(self, samples, base):
        out = C.c_double()
        s = np.ascontiguousarray(samples, np.float64)
        if self.lib.gbxref_attribute_reward(s, len(s), base, C.byref(out)):
            raise ValueError(self.err())
        return out.value

    def boltzmann_pair(self, q0, q1, rho):
        out = np.empty(2, np.float64)
        self.lib.gbxref_boltzmann_pair(q0, q1, rho, out)
        return out

    def qtable_snapshot(self, text: str, rho: float):
        t = text.encode()
        n = self.lib.gbxref_qtable_snapshot(t, rho, None, None)
        if n < 0:
            raise ValueError(self.err())
        feat = np.empty((n, N_FEAT), np.float32)
        tgt = np.empty((n, 2), np.float64)
        self.lib.gbxref_qtable_snapshot(t, rho, feat.ctypes.data, tgt.ctypes.data)
        return feat, tgt

    def qtable_fold(self, keys, actions, rewards, now, alpha=0.3, omega=1.0, rho=0.1):
        """Fresh QTable, QTable::update over the tuples in order, then the table
        (key order) and snapshot_policy_dataset(rho). Returns a dict."""
        keys = np.ascontiguousarray(keys, np.uint32)
        actions = np.ascontiguousarray(actions, np.uint8)
        rewards = np.ascontiguousarray(rewards, np.float64)
        now = np.ascontiguousarray(now, np.uint64)
        n = len(actions)
        sizes = np.zeros(2, np.int64)
        bad = C.c_long(-1)
        args = [keys.ctypes.data, actions.ctypes.data, rewards.ctypes.data, now.ctypes.data, n,
                alpha, omega, rho, sizes.ctypes.data, C.byref(bad)]
        if self.lib.gbxref_qtable_fold(*args, *([None] * 7)) < 0:
            raise ValueError(self.err())
        m, r = int(sizes[0]), int(sizes[1])
        out = {"keys": np.empty((m, 30), np.uint32), "q": np.empty((m, 2)), "t": np.empty((m, 2), np.uint64),
               "cnt": np.empty((m, 2), np.uint64), "has": np.empty((m, 2), np.uint8),
               "feat": np.empty((r, N_FEAT), np.float32), "tgt": np.empty((r, 2))}
        self.lib.gbxref_qtable_fold(*args, *(out[k].ctypes.data for k in
                                             ("keys", "q", "t", "cnt", "has", "feat", "tgt")))
        out["bad"] = bad.value
        return out

    # suites -----------------------------------------------------------------
    def suite_generate(self, benchmark_count=16, shaders_min=184, shaders_max=276,
                       pipelines_min=2, pipelines_max=4, bandwidth_capacity=0.0,
                       noise_sigma=0.005, memory_bound_threshold=1.0, seed=1):
        h = self.lib.gbxref_suite_generate(benchmark_count, shaders_min, shaders_max,
                                           pipelines_min, pipelines_max, bandwidth_capacity,
                                           noise_sigma, memory_bound_threshold, seed)
        if not h:
            raise ValueError(self.err())
        return h

    def suite_advance(self, h, checkins: int):
        self.lib.gbxref_suite_advance(h, checkins)

    def suite_checkin(self, h) -> int:
        return int(self.lib.gbxref_suite_checkin(h))

    def suite_keys(self, h, n_shaders: int) -> np.ndarray:
        k = np.empty((n_shaders, 30), np.uint32)
        self.lib.gbxref_suite_keys(h, k.ctypes.data)
        return k

    def run_training(self, h, iterations, checkins=50, eps0=0.2, horizon=0, samples=10, alpha=0.3,
                     omega=1.0, lr=0.01, epochs=50, batch=32, rho0=0.1, rho_decay=0.95,
                     rho_min=0.01, seed=0) -> dict:
        """The reference's run_training on a copy of the suite (jobs = 1)."""
        a = [h, iterations, checkins, eps0, horizon, samples, alpha, omega, lr, epochs, batch, rho0,
             rho_decay, rho_min, seed]
        m = self.lib.gbxref_run_training(*a, *([None] * 7))
        if m < 0:
            raise ValueError(self.err())
        out = {"policy": np.empty(5026, np.float32), "logs": np.empty((iterations, 4)),
               "keys": np.empty((m, 30), np.uint32), "q": np.empty((m, 2)),
               "t": np.empty((m, 2), np.uint64), "cnt": np.empty((m, 2), np.uint64),
               "has": np.empty((m, 2), np.uint8)}
        self.lib.gbxref_run_training(*a, *(out[k].ctypes.data for k in
                                           ("policy", "logs", "keys", "q", "t", "cnt", "has")))
        return out

    def suite_free(self, h):
        self.lib.gbxref_suite_free(h)

    def suite_export(self, h) -> dict:
        dims = np.empty(5, np.uint64)
        self.lib.gbxref_suite_dims(h, dims)
        nsh, nb, npi, nsl, nm = (int(x) for x in dims)
        s = dict(
            shader_lat=np.empty((nsh, 3), np.float64),
            features=np.empty((nsh, N_FEAT), np.float32),
            app_f64=np.empty((nb, 4), np.float64),
            app_pipe_off=np.empty(nb + 1, np.uint64),
            pipe_wt=np.empty((npi, 2), np.float64),
            pipe_slot_off=np.empty(npi + 1, np.uint64),
            slot_shader=np.empty(nsl, np.uint32),
            slot_frac=np.empty(nsl, np.float64),
            app_member_off=np.empty(nb + 1, np.uint64),
            members=np.empty(nm, np.uint32),
        )
        self.lib.gbxref_suite_export(h, s["shader_lat"], s["features"], s["app_f64"],
                                     s["app_pipe_off"], s["pipe_wt"], s["pipe_slot_off"],
                                     s["slot_shader"], s["slot_frac"], s["app_member_off"],
                                     s["members"])
        return s

    def run_benchmark(self, h, bench_id, shader_actions, n_samples, seed):
        out = np.empty(n_samples, np.float64)
        if self.lib.gbxref_run_benchmark(h, bench_id, np.ascontiguousarray(shader_actions, np.uint8),
                                         n_samples, seed, out):
            raise ValueError(self.err())
        return out

    def evaluate(self, h, params, n_samples, seed, jobs=1, n_bench=None):
        if n_bench is None:
            dims = np.empty(5, np.uint64)
            self.lib.gbxref_suite_dims(h, dims)
            n_bench = int(dims[1])
        rows = np.empty((n_bench, 3), np.float64)
        cap = 1 << 16
        lo = np.empty(cap, np.float64)
        cnt = np.empty(cap, np.uint64)
        nb = self.lib.gbxref_evaluate(h, np.ascontiguousarray(params, np.float32), n_samples, seed,
                                      jobs, rows, lo, cnt, cap)
        if nb < 0:
            raise ValueError(self.err())
        return rows, lo[:nb].copy(), cnt[:nb].copy()
