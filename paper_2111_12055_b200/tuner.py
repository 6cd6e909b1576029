"""Algorithm 1 on the device — SURVEY §8 row f3 (experience production) wired
to rows A5-A11 and f1: one run_iteration (proj/src/tuner.cpp:172-239) whose
compute all runs in libgbxcu kernels:

  collection      gbxcu_collect       sampled, epsilon-mixed actions (A8)
  run_benchmark   gbxcu_aggregate     frame_time + noisy samples + reward (A9, A10)
  table fold      DeviceQTable        QTable::update over the run's tuples (f1)
  snapshot        DeviceQTable        snapshot_policy_dataset at rho_at(i) (A11)
  distillation    Device.fit          fit on the snapshot (A5)
  agreement       Device.forward      table_agreement's net decisions (A7)

Host code only does what the reference's loop does between those calls:
seeds (derive_seed), the epsilon / temperature schedules, the per-benchmark
bookkeeping (member lists, reward broadcast to observations) and the log.
The environment (SimSuite: drift, compile) stays outside, as in the
reference's tests: each iteration receives the suite at its check-in.
"""
from __future__ import annotations

import math

import numpy as np

from . import FWD_FAST, DeviceQTable, N_PARAMS

_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
K_ACTION, K_FPS, K_FIT, K_INIT = 0x414354, 0x465053, 0x464954, 0x494E49  # tuner.cpp:22-26


def _mix64(x: int) -> int:
    """SplitMix64 finaliser of x + gamma (proj/include/gbx/rng.hpp:11-16)."""
    x = (x + _GAMMA) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def derive_seed(*parts: int) -> int:
    """Order-sensitive seed derivation (proj/include/gbx/rng.hpp:20-26)."""
    h = 0x8557D1C3C2DB0F5B
    for p in parts:
        h = _mix64(h ^ (p & _M64))
    return h


class TunerConfig:
    """TunerConfig + TrainConfig + QHyperparams fields that run_iteration reads
    (proj/include/gbx/tuner.hpp:15-33, policy.hpp:77-89, qtable.hpp:33-38)."""

    def __init__(self, num_iterations=45, checkins_per_iteration=50, epsilon0=0.2,
                 epsilon_horizon=0, refresh_period=1, samples_per_benchmark=10, alpha=0.3,
                 omega=1.0, learning_rate=0.01, epochs=50, batch_size=32, rho0=0.1,
                 rho_decay=0.95, rho_min=0.01, seed=0):
        self.__dict__.update(locals())
        del self.__dict__["self"]

    def epsilon_at(self, i: int) -> float:  # tuner.cpp:52-57
        horizon = self.epsilon_horizon if self.epsilon_horizon > 0 else max(1, self.num_iterations // 2)
        return self.epsilon0 * max(0.0, 1.0 - i / horizon)

    def rho_at(self, i: int) -> float:  # policy.cpp:293-295
        return max(self.rho_min, self.rho0 * math.pow(self.rho_decay, i))


def member_suite(s: dict) -> dict:
    """The aggregation suite with one latent row per (benchmark, member shader):
    a shader shared by two benchmarks can get different sampled actions in each
    (per-benchmark RNG streams), so slots index their benchmark's member list."""
    moff = s["app_member_off"].astype(np.int64)
    members = s["members"]
    poff = s["app_pipe_off"].astype(np.int64)
    soff = s["pipe_slot_off"].astype(np.int64)
    slot_m = np.empty(len(s["slot_shader"]), np.uint32)
    for b in range(len(moff) - 1):
        lo, hi = soff[poff[b]], soff[poff[b + 1]]
        mem = members[moff[b]:moff[b + 1]]
        slot_m[lo:hi] = moff[b] + np.searchsorted(mem, s["slot_shader"][lo:hi])
    out = dict(s)
    out["slot_shader"] = slot_m
    out["shader_lat"] = np.ascontiguousarray(s["shader_lat"][members])
    return out


class DeviceTuner:
    """TunerState (decision / behavior nets, Q-table) with run_iteration on the device."""

    def __init__(self, dev, cfg: TunerConfig):
        self.dev, self.cfg = dev, cfg
        self.table = DeviceQTable(dev, cfg.alpha, cfg.omega)
        self.decision = dev.policy_init(derive_seed(cfg.seed, K_INIT))  # tuner.cpp:247
        self.behavior = self.decision.copy()

    def run_iteration(self, i: int, suite: dict, keys: np.ndarray, now: int) -> dict:
        """suite: CSR export at the iteration's check-in (features, latents,
        member lists); keys[n_shaders][30]: StateKeys at that check-in."""
        cfg, dev = self.cfg, self.dev
        moff = suite["app_member_off"].astype(np.uint64)
        members = suite["members"]
        n_bench = len(moff) - 1
        # collection: per benchmark SplitMix64(derive_seed(seed, ACT, i, b)), shader_ids order
        seg_seed = np.array([derive_seed(cfg.seed, K_ACTION, i, b) for b in range(n_bench)], np.uint64)
        act = dev.collect(self.behavior, suite["features"][members], moff, seg_seed, cfg.epsilon_at(i))
        # run_benchmark + attribute_rewards: reward of each run (row 4)
        run_seed = np.array([derive_seed(cfg.seed, K_FPS, i, b) for b in range(n_bench)], np.uint64)
        rows = dev.aggregate(member_suite(suite), act, run_seed, cfg.samples_per_benchmark)
        reward = rows[:, 4]
        # fold: benchmark order, observations in shader_ids order (tuner.cpp:207-213)
        counts = np.diff(moff).astype(np.int64)
        self.table.update_batch(keys[members], act, np.repeat(reward, counts),
                                np.full(len(members), now, np.uint64))
        feat, tgt = self.table.snapshot(cfg.rho_at(i))
        distill = 0.0
        if len(feat):
            p, el = dev.fit(self.decision, feat, tgt, cfg.learning_rate, cfg.epochs, cfg.batch_size,
                            derive_seed(cfg.seed, K_FIT, i))
            self.decision, distill = p, float(el[-1])
        if i % cfg.refresh_period == 0:
            self.behavior = self.decision.copy()
        reward_sum = 0.0
        for r in reward:  # left fold, benchmark order
            reward_sum += float(r)
        t = self.table.export()
        both = (t["has"][:, 0] == 1) & (t["has"][:, 1] == 1)
        agreement = 1.0
        if both.any():
            greedy = (t["q"][both, 1] >= t["q"][both, 0]).astype(np.uint8)
            _, net = dev.forward(self.decision, feat, FWD_FAST)
            agreement = float(np.count_nonzero(greedy == net)) / float(both.sum())
        return {"iteration": i, "checkin": now,
                "mean_reward": reward_sum / n_bench if n_bench else 1.0,
                "table_size": len(t["keys"]), "distill_loss": distill, "agreement_rate": agreement}


assert N_PARAMS == 5026
