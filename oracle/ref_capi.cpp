// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A flat C ABI over the *unmodified* reference library, compiled from
// /root/reference/proj/src/*.cpp with -Dgbx=gbxref (see oracle/Makefile).
// It exists so that Python tests, the golden-vector generator
// (oracle/make_golden.py) and bench.py's `cpu_baseline` / `--impl reference`
// leg can drive the reference's own code path:
//   * PolicyNet::init / forward / select_greedy  (proj/src/policy.cpp:128-148,339-342)
//   * batch_kl_loss / batch_kl_gradient / fit    (proj/src/policy.cpp:194-201,270-279,297-337)
//   * SimSuite::generate / run_benchmark         (proj/src/simenv.cpp:277-382,481-510)
//   * evaluate (uplift rows + 1% histogram)      (proj/src/tuner.cpp:266-315)
//   * attribute_rewards / reward_from_framerate  (proj/src/tuner.cpp:131-147, core.cpp:125-133)
//   * QTable::load + snapshot_policy_dataset     (proj/src/qtable.cpp:143-155,188-231)
// Inputs for the "G1" distribution follow the reference test helpers
// random_state / random_target (proj/tests/test_policy.cpp:15-28).
//
// Only the built shared object lives in oracle/_ref/ (git-ignored); this
// adapter is ours. No reference source is copied into the repository.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "gbx/core.hpp"
#include "gbx/policy.hpp"
#include "gbx/qtable.hpp"
#include "gbx/rng.hpp"
#include "gbx/simenv.hpp"
#include "gbx/tuner.hpp"

namespace {

constexpr int kF = gbx::kFeatureCount;

gbx::PolicyNet net_from_flat(const float* params) {
    gbx::PolicyNet net = gbx::PolicyNet::zeros();
    for (std::size_t i = 0; i < gbx::kPolicyParamCount; ++i) net.set_param(i, params[i]);
    return net;
}

void net_to_flat(const gbx::PolicyNet& net, float* params) {
    for (std::size_t i = 0; i < gbx::kPolicyParamCount; ++i) params[i] = net.param(i);
}

gbx::PolicyDataset dataset_from(const float* feat, const double* tgt, std::size_t n) {
    gbx::PolicyDataset d(n);
    for (std::size_t r = 0; r < n; ++r) {
        std::memcpy(d[r].first.features.data(), feat + r * kF, sizeof(float) * kF);
        d[r].second.prob = {tgt[2 * r], tgt[2 * r + 1]};
    }
    return d;
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* gbxref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- inputs
// G1 states/targets exactly as test_policy.cpp:15-28 draws them from one
// SplitMix64 stream: state i then target i, interleaved.
void gbxref_g1(std::uint64_t seed, std::size_t n, float* feat, double* tgt) {
    gbx::SplitMix64 rng(seed);
    for (std::size_t r = 0; r < n; ++r) {
        float* f = feat + r * kF;
        const auto stage = rng.next_below(8);
        for (int i = 0; i < 8; ++i) f[i] = i == static_cast<int>(stage) ? 1.0f : 0.0f;
        for (int i = 8; i < kF; ++i) f[i] = static_cast<float>(rng.next_range(0.0, 7.0));
        const double p = rng.next_range(0.02, 0.98);
        if (tgt) {
            tgt[2 * r] = p;
            tgt[2 * r + 1] = 1.0 - p;
        }
    }
}

// ---------------------------------------------------------------- policy
void gbxref_policy_init(std::uint64_t seed, float* params) {
    net_to_flat(gbx::PolicyNet::init(seed), params);
}

// probs: nullable [n][2]; actions: nullable [n] (0 = wave32, 1 = wave64).
int gbxref_forward(const float* params, const float* feat, std::size_t n, double* probs,
                   std::uint8_t* actions) {
    try {
        gbx::BehaviorPolicy beh{net_from_flat(params), 0, 0};
        gbx::ShaderState s;
        for (std::size_t r = 0; r < n; ++r) {
            std::memcpy(s.features.data(), feat + r * kF, sizeof(float) * kF);
            if (probs) {
                const auto p = beh.forward(s);
                probs[2 * r] = p[0];
                probs[2 * r + 1] = p[1];
            }
            if (actions) actions[r] = static_cast<std::uint8_t>(gbx::select_greedy(beh, s));
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

double gbxref_kl_loss(double p0, double p1, double t0, double t1) {
    return gbx::kl_loss({p0, p1}, gbx::EmpiricalPolicy{{t0, t1}});
}

double gbxref_batch_kl_loss(const float* params, const float* feat, const double* tgt,
                            std::size_t n) {
    const auto net = net_from_flat(params);
    const auto d = dataset_from(feat, tgt, n);
    return gbx::batch_kl_loss(net, d);
}

void gbxref_batch_kl_gradient(const float* params, const float* feat, const double* tgt,
                              std::size_t n, double* grad) {
    const auto net = net_from_flat(params);
    const auto d = dataset_from(feat, tgt, n);
    const auto g = gbx::batch_kl_gradient(net, d);
    std::memcpy(grad, g.data(), sizeof(double) * g.size());
}

// Returns 0 ok, 1 validation error, 2 diverged (epoch in *diverged_epoch).
int gbxref_fit(float* params, const float* feat, const double* tgt, std::size_t n, double lr,
               int epochs, int batch, std::uint64_t seed, double* epoch_loss,
               int* diverged_epoch) {
    auto net = net_from_flat(params);
    try {
        const auto d = dataset_from(feat, tgt, n);
        gbx::TrainConfig cfg;
        cfg.learning_rate = lr;
        cfg.epochs = epochs;
        cfg.batch_size = batch;
        cfg.seed = seed;
        const auto fr = gbx::fit(net, d, cfg);
        for (std::size_t e = 0; e < fr.epoch_loss.size(); ++e) epoch_loss[e] = fr.epoch_loss[e];
        net_to_flat(net, params);
        return 0;
    } catch (const gbx::TrainingDivergedError& e) {
        if (diverged_epoch) *diverged_epoch = e.epoch;
        net_to_flat(net, params);
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Per-epoch permutation `order` after `epochs` in-place Fisher-Yates passes
// (policy.cpp:303-314), reproduced through the reference's own SplitMix64.
void gbxref_fit_order(std::size_t n, std::uint64_t seed, int epochs, std::uint64_t* order) {
    for (std::size_t i = 0; i < n; ++i) order[i] = i;
    for (int e = 0; e < epochs; ++e) {
        gbx::SplitMix64 rng(gbx::derive_seed({seed, 0x5F17u, static_cast<std::uint64_t>(e)}));
        for (std::size_t i = n; i > 1; --i) {
            const std::size_t j = rng.next_below(i);
            std::swap(order[i - 1], order[j]);
        }
    }
}

std::uint64_t gbxref_derive_seed3(std::uint64_t a, std::uint64_t b, std::uint64_t c) {
    return gbx::derive_seed({a, b, c});
}

// ---------------------------------------------------------------- rewards
int gbxref_reward_from_framerate(double observed, double baseline, double* out) {
    try {
        *out = gbx::reward_from_framerate(observed, baseline);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int gbxref_attribute_reward(const double* samples, std::size_t n, double baseline, double* out) {
    try {
        gbx::RunRecord rec;
        rec.observations.resize(1);
        const auto r = gbx::attribute_rewards(rec, std::span<const double>(samples, n), baseline);
        *out = r.front().reward;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void gbxref_boltzmann_pair(double q0, double q1, double rho, double* out) {
    const auto p = gbx::boltzmann_pair(q0, q1, rho);
    out[0] = p.prob[0];
    out[1] = p.prob[1];
}

// ---------------------------------------------------------------- q-table
// Loads the line-text table and snapshots the key-ordered policy dataset.
// Call once with feat == nullptr to get the row count.
long gbxref_qtable_snapshot(const char* text, double rho, float* feat, double* tgt) {
    try {
        std::istringstream is(text);
        const auto t = gbx::QTable::load(is);
        const auto d = t.snapshot_policy_dataset(rho);
        if (feat) {
            for (std::size_t r = 0; r < d.size(); ++r) {
                std::memcpy(feat + r * kF, d[r].first.features.data(), sizeof(float) * kF);
                tgt[2 * r] = d[r].second.prob[0];
                tgt[2 * r + 1] = d[r].second.prob[1];
            }
        }
        return static_cast<long>(d.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Folds n tuples into a fresh QTable with QTable::update in order (the
// reference's Eq.-5 fold, proj/src/qtable.cpp:76-92); on ClockRegressionError
// the table keeps the updates before it (*bad = tuple index). Returns the
// table in key order and its snapshot. Call with out_keys == nullptr first to
// get sizes[0] = states, sizes[1] = snapshot rows.
long gbxref_qtable_fold(const std::uint32_t* keys, const std::uint8_t* actions, const double* rewards,
                        const std::uint64_t* now, std::size_t n, double alpha, double omega,
                        double rho, long* sizes, long* bad, std::uint32_t* out_keys, double* out_q,
                        std::uint64_t* out_t, std::uint64_t* out_cnt, std::uint8_t* out_has,
                        float* feat, double* tgt) {
    try {
        gbx::QTable t(gbx::QHyperparams{alpha, omega});
        *bad = -1;
        for (std::size_t i = 0; i < n; ++i) {
            gbx::StateKey k;
            std::memcpy(k.values.data(), keys + i * 30, sizeof(std::uint32_t) * 30);
            try {
                t.update(k, actions[i] ? gbx::Action::Wave64 : gbx::Action::Wave32, rewards[i], now[i]);
            } catch (const gbx::ClockRegressionError&) {
                *bad = (long)i;
                break;
            }
        }
        const auto d = t.snapshot_policy_dataset(rho);
        sizes[0] = (long)t.state_count();
        sizes[1] = (long)d.size();
        if (!out_keys) return 0;
        std::size_t r = 0;
        for (const auto& [key, pair] : t.entries()) {
            std::memcpy(out_keys + r * 30, key.values.data(), sizeof(std::uint32_t) * 30);
            for (int a = 0; a < 2; ++a) {
                const bool h = pair[a].has_value();
                out_has[2 * r + a] = h ? 1 : 0;
                out_q[2 * r + a] = h ? pair[a]->q : 0.0;
                out_t[2 * r + a] = h ? pair[a]->last_update_t : 0;
                out_cnt[2 * r + a] = h ? pair[a]->update_count : 0;
            }
            ++r;
        }
        for (std::size_t i = 0; i < d.size(); ++i) {
            std::memcpy(feat + i * kF, d[i].first.features.data(), sizeof(float) * kF);
            tgt[2 * i] = d[i].second.prob[0];
            tgt[2 * i + 1] = d[i].second.prob[1];
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// ---------------------------------------------------------------- suites
struct gbxref_suite {
    std::unique_ptr<gbx::SimSuite> s;
};

// spec: benchmark_count, shaders_min, shaders_max, pipelines_min, pipelines_max,
// bandwidth_capacity, noise_sigma, memory_bound_threshold (others default).
gbxref_suite* gbxref_suite_generate(int benchmark_count, int shaders_min, int shaders_max,
                                    int pipelines_min, int pipelines_max,
                                    double bandwidth_capacity, double noise_sigma,
                                    double memory_bound_threshold, std::uint64_t seed) {
    try {
        gbx::SuiteSpec spec;
        spec.benchmark_count = benchmark_count;
        spec.shaders_min = shaders_min;
        spec.shaders_max = shaders_max;
        spec.pipelines_min = pipelines_min;
        spec.pipelines_max = pipelines_max;
        spec.bandwidth_capacity = bandwidth_capacity;
        spec.noise_sigma = noise_sigma;
        spec.memory_bound_threshold = memory_bound_threshold;
        auto* h = new gbxref_suite;
        h->s = std::make_unique<gbx::SimSuite>(gbx::SimSuite::generate(spec, seed));
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void gbxref_suite_free(gbxref_suite* h) { delete h; }

// dims: n_shaders, n_bench, n_pipes, n_slots, n_members (sum of distinct ids)
void gbxref_suite_dims(const gbxref_suite* h, std::size_t* dims) {
    const auto& s = *h->s;
    std::size_t pipes = 0, slots = 0, members = 0;
    for (const auto& b : s.benchmarks()) {
        pipes += b.pipelines.size();
        for (const auto& p : b.pipelines) slots += p.slots.size();
        members += b.shader_ids.size();
    }
    dims[0] = s.shaders().size();
    dims[1] = s.benchmarks().size();
    dims[2] = pipes;
    dims[3] = slots;
    dims[4] = members;
}

// CSR export. shader_f64 [n_shaders][3] = divergence, bandwidth_demand,
// parallelism; features [n_shaders][44] from compile(); bench_f64 [n_bench][4]
// = baseline_fps, bandwidth_capacity, noise_sigma, memory_bound_threshold;
// bench_pipe_off [n_bench+1]; pipe_f64 [n_pipes][2] = weight, base_time;
// pipe_slot_off [n_pipes+1]; slot_shader [n_slots]; slot_frac [n_slots];
// bench_member_off [n_bench+1]; members [n_members].
void gbxref_suite_export(const gbxref_suite* h, double* shader_f64, float* features,
                         double* bench_f64, std::uint64_t* bench_pipe_off, double* pipe_f64,
                         std::uint64_t* pipe_slot_off, std::uint32_t* slot_shader,
                         double* slot_frac, std::uint64_t* bench_member_off,
                         std::uint32_t* members) {
    const auto& s = *h->s;
    for (std::size_t i = 0; i < s.shaders().size(); ++i) {
        const auto& sh = s.shaders()[i];
        shader_f64[3 * i] = sh.divergence;
        shader_f64[3 * i + 1] = sh.bandwidth_demand;
        shader_f64[3 * i + 2] = sh.parallelism;
        const auto st = s.compile(static_cast<std::uint32_t>(i), gbx::kDefaultAction).first;
        std::memcpy(features + i * kF, st.features.data(), sizeof(float) * kF);
    }
    std::size_t p = 0, sl = 0, m = 0;
    bench_pipe_off[0] = 0;
    pipe_slot_off[0] = 0;
    bench_member_off[0] = 0;
    for (std::size_t b = 0; b < s.benchmarks().size(); ++b) {
        const auto& bench = s.benchmarks()[b];
        bench_f64[4 * b] = bench.baseline_fps;
        bench_f64[4 * b + 1] = bench.bandwidth_capacity;
        bench_f64[4 * b + 2] = bench.noise_sigma;
        bench_f64[4 * b + 3] = bench.memory_bound_threshold;
        for (const auto& pipe : bench.pipelines) {
            pipe_f64[2 * p] = pipe.weight;
            pipe_f64[2 * p + 1] = pipe.base_time;
            for (const auto& slot : pipe.slots) {
                slot_shader[sl] = slot.shader_id;
                slot_frac[sl] = slot.exec_fraction;
                ++sl;
            }
            ++p;
            pipe_slot_off[p] = sl;
        }
        bench_pipe_off[b + 1] = p;
        for (auto id : bench.shader_ids) members[m++] = id;
        bench_member_off[b + 1] = m;
    }
}

// Per-benchmark noisy samples under a per-shader action vector (indexed by
// shader id), via the reference run_benchmark.
int gbxref_run_benchmark(const gbxref_suite* h, std::uint32_t bench_id,
                         const std::uint8_t* shader_actions, int n_samples, std::uint64_t seed,
                         double* samples) {
    try {
        const auto& bench = h->s->benchmark(bench_id);
        gbx::ActionAssignment a;
        for (auto id : bench.shader_ids) a[id] = static_cast<gbx::Action>(shader_actions[id]);
        const auto run = h->s->run_benchmark(bench_id, a, n_samples, seed);
        for (int k = 0; k < n_samples; ++k) samples[k] = run.samples[k];
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void gbxref_suite_advance(gbxref_suite* h, std::uint64_t checkins) { h->s->advance_checkins(checkins); }
std::uint64_t gbxref_suite_checkin(const gbxref_suite* h) { return h->s->checkin(); }

// StateKey of every shader at the current check-in (compile(), simenv.cpp:408-412).
void gbxref_suite_keys(const gbxref_suite* h, std::uint32_t* keys) {
    for (std::size_t i = 0; i < h->s->shaders().size(); ++i) {
        const auto key = h->s->compile(static_cast<std::uint32_t>(i), gbx::kDefaultAction).second;
        std::memcpy(keys + i * 30, key.values.data(), sizeof(std::uint32_t) * 30);
    }
}

// run_training (tuner.cpp:241-264) on a COPY of the suite: `iterations`
// Algorithm-1 iterations (checkins_per_iteration, epsilon0 / horizon, 10
// samples per benchmark, QHyperparams{alpha, omega}, TrainConfig{lr, epochs,
// batch, rho0, rho_decay, rho_min}, seed, jobs = 1). Outputs: the final behavior
// policy (flat params), logs[iterations][4] = {mean_reward, table_size,
// distill_loss, agreement_rate}, and the table in key order (two-call
// protocol: out_keys == nullptr returns the state count).
long gbxref_run_training(const gbxref_suite* h, int iterations, int checkins, double eps0,
                         int horizon, int samples, double alpha, double omega, double lr, int epochs,
                         int batch, double rho0, double rho_decay, double rho_min, std::uint64_t seed,
                         float* behavior_params, double* logs, std::uint32_t* out_keys,
                         double* out_q, std::uint64_t* out_t, std::uint64_t* out_cnt,
                         std::uint8_t* out_has) {
    try {
        gbx::TunerConfig cfg;
        cfg.num_iterations = iterations;
        cfg.checkins_per_iteration = checkins;
        cfg.epsilon0 = eps0;
        cfg.epsilon_horizon = horizon;
        cfg.samples_per_benchmark = samples;
        cfg.qtable = gbx::QHyperparams{alpha, omega};
        cfg.train.learning_rate = lr;
        cfg.train.epochs = epochs;
        cfg.train.batch_size = batch;
        cfg.train.rho0 = rho0;
        cfg.train.rho_decay = rho_decay;
        cfg.train.rho_min = rho_min;
        cfg.seed = seed;
        cfg.jobs = 1;
        const auto res = gbx::run_training(*h->s, cfg, std::nullopt);
        if (!out_keys) return (long)res.table.state_count();
        net_to_flat(res.policy.net, behavior_params);
        for (std::size_t i = 0; i < res.logs.size(); ++i) {
            logs[4 * i] = res.logs[i].mean_reward;
            logs[4 * i + 1] = (double)res.logs[i].table_size;
            logs[4 * i + 2] = res.logs[i].distill_loss;
            logs[4 * i + 3] = res.logs[i].agreement_rate;
        }
        std::size_t r = 0;
        for (const auto& [key, pair] : res.table.entries()) {
            std::memcpy(out_keys + r * 30, key.values.data(), sizeof(std::uint32_t) * 30);
            for (int a = 0; a < 2; ++a) {
                const bool hv = pair[a].has_value();
                out_has[2 * r + a] = hv ? 1 : 0;
                out_q[2 * r + a] = hv ? pair[a]->q : 0.0;
                out_t[2 * r + a] = hv ? pair[a]->last_update_t : 0;
                out_cnt[2 * r + a] = hv ? pair[a]->update_count : 0;
            }
            ++r;
        }
        return (long)r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Greedy evaluation through the reference evaluate(). rows [n_bench][3] =
// baseline_fps, tuned_fps, uplift_pct. Histogram written up to hist_cap bins;
// returns the bin count (or -1 on error).
long gbxref_evaluate(const gbxref_suite* h, const float* params, int n_samples,
                     std::uint64_t seed, int jobs, double* rows, double* hist_lower,
                     std::uint64_t* hist_count, std::size_t hist_cap) {
    try {
        gbx::BehaviorPolicy beh{net_from_flat(params), 0, 0};
        const auto rep = gbx::evaluate(*h->s, beh, n_samples, seed, jobs);
        for (std::size_t b = 0; b < rep.rows.size(); ++b) {
            rows[3 * b] = rep.rows[b].baseline_fps;
            rows[3 * b + 1] = rep.rows[b].tuned_fps;
            rows[3 * b + 2] = rep.rows[b].uplift_pct;
        }
        for (std::size_t k = 0; k < rep.histogram.size() && k < hist_cap; ++k) {
            hist_lower[k] = rep.histogram[k].lower_pct;
            hist_count[k] = rep.histogram[k].count;
        }
        return static_cast<long>(rep.histogram.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
