// test_dropin_alg1.cpp — the SimSuite-facing drop-in entry points
// (libgbx_b200_alg1.so: run_training / run_iteration / evaluate(const
// SimSuite&), compute on the B200) against the compiled reference
// (libgbxref.so through oracle/ref_capi.cpp) on the same generated suite.
// The SimSuite here is the reference's own environment code
// (oracle/_ref/libgbx_refenv.so = proj/src/simenv.cpp built against the
// drop-in headers), exactly what a caller of the drop-in keeps linking.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <cstring>
#include <sstream>

#include "gbx/tuner.hpp"

extern "C" {
void* gbxref_suite_generate(int, int, int, int, int, double, double, double, std::uint64_t);
void gbxref_suite_free(void*);
void gbxref_suite_advance(void*, std::uint64_t);
long gbxref_run_training(const void* h, int iterations, int checkins, double eps0, int horizon,
                         int samples, double alpha, double omega, double lr, int epochs, int batch,
                         double rho0, double rho_decay, double rho_min, std::uint64_t seed,
                         float* behavior_params, double* logs, std::uint32_t* out_keys, double* out_q,
                         std::uint64_t* out_t, std::uint64_t* out_cnt, std::uint8_t* out_has);
long gbxref_evaluate(const void*, const float*, int, std::uint64_t, int, double*, double*,
                     std::uint64_t*, std::size_t);
}

using namespace gbx;

namespace {

struct SuiteCase {
    int benchmarks, pipelines_max;
    double bw_capacity;
    std::uint64_t seed;
};

SimSuite generate(const SuiteCase& c) {
    SuiteSpec spec;
    spec.benchmark_count = c.benchmarks;
    spec.pipelines_max = c.pipelines_max;
    spec.bandwidth_capacity = c.bw_capacity;
    return SimSuite::generate(spec, c.seed);
}

void* generate_ref(const SuiteCase& c) {
    SuiteSpec d;  // the remaining fields at their defaults, as generate() above
    return gbxref_suite_generate(c.benchmarks, d.shaders_min, d.shaders_max, d.pipelines_min,
                                 c.pipelines_max, c.bw_capacity, d.noise_sigma, d.memory_bound_threshold,
                                 c.seed);
}

std::int64_t ulps(float a, float b) {
    std::int32_t x, y;
    std::memcpy(&x, &a, 4);
    std::memcpy(&y, &b, 4);
    return std::llabs((std::int64_t)x - (std::int64_t)y);
}

}  // namespace

TEST_CASE("run_training on the device equals the reference's run_training") {
    for (const SuiteCase sc : {SuiteCase{44, 4, 0.0, 7}, SuiteCase{12, 3, 1.0, 21}}) {
        TunerConfig cfg;
        cfg.num_iterations = 3;
        cfg.checkins_per_iteration = 50;
        cfg.seed = 5;
        const TrainResult res = run_training(generate(sc), cfg);

        void* h = generate_ref(sc);
        REQUIRE(h != nullptr);
        const long m = gbxref_run_training(h, cfg.num_iterations, cfg.checkins_per_iteration, cfg.epsilon0,
                                           cfg.epsilon_horizon, cfg.samples_per_benchmark,
                                           cfg.qtable.alpha, cfg.qtable.omega, cfg.train.learning_rate,
                                           cfg.train.epochs, cfg.train.batch_size, cfg.train.rho0,
                                           cfg.train.rho_decay, cfg.train.rho_min, cfg.seed, nullptr,
                                           nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
        REQUIRE(m > 0);
        std::vector<float> pol(5026);
        std::vector<double> logs(4 * cfg.num_iterations), q(2 * m);
        std::vector<std::uint32_t> keys(30 * m);
        std::vector<std::uint64_t> t(2 * m), cnt(2 * m);
        std::vector<std::uint8_t> has(2 * m);
        gbxref_run_training(h, cfg.num_iterations, cfg.checkins_per_iteration, cfg.epsilon0,
                            cfg.epsilon_horizon, cfg.samples_per_benchmark, cfg.qtable.alpha,
                            cfg.qtable.omega, cfg.train.learning_rate, cfg.train.epochs,
                            cfg.train.batch_size, cfg.train.rho0, cfg.train.rho_decay, cfg.train.rho_min,
                            cfg.seed, pol.data(), logs.data(), keys.data(), q.data(), t.data(), cnt.data(),
                            has.data());
        gbxref_suite_free(h);

        // the experience store: every key, value, timestamp and count identical
        REQUIRE(res.table.state_count() == (std::size_t)m);
        std::size_t r = 0, mism = 0;
        for (const auto& [key, pair] : res.table.entries()) {
            mism += std::memcmp(key.values.data(), keys.data() + 30 * r, 120) != 0;
            for (int a = 0; a < 2; ++a) {
                const bool hv = pair[a].has_value();
                mism += hv != (has[2 * r + a] != 0);
                if (hv)
                    mism += pair[a]->q != q[2 * r + a] || pair[a]->last_update_t != t[2 * r + a] ||
                            pair[a]->update_count != cnt[2 * r + a];
            }
            ++r;
        }
        CHECK(mism == 0);
        // the logs: rewards / sizes / agreement exact, distill loss rel 1e-12
        REQUIRE(res.logs.size() == (std::size_t)cfg.num_iterations);
        for (int i = 0; i < cfg.num_iterations; ++i) {
            CHECK(res.logs[i].mean_reward == logs[4 * i]);
            CHECK((double)res.logs[i].table_size == logs[4 * i + 1]);
            CHECK(std::fabs(res.logs[i].distill_loss - logs[4 * i + 2]) <= 1e-12 * std::fabs(logs[4 * i + 2]));
            CHECK(res.logs[i].agreement_rate == logs[4 * i + 3]);
        }
        // the behavior policy: <= 1 fp32 ulp per weight (batch-32 fits: 1-CTA kernel)
        const auto flat = res.policy.net.flat();
        std::int64_t worst = 0;
        for (std::size_t i = 0; i < pol.size(); ++i) worst = std::max(worst, ulps(flat[i], pol[i]));
        CHECK(worst <= 1);
    }
}

TEST_CASE("evaluate(const SimSuite&) equals the reference's evaluate bit for bit") {
    for (const SuiteCase sc : {SuiteCase{8, 4, 0.0, 3}, SuiteCase{6, 3, 1.0, 11}}) {
        SimSuite s = generate(sc);
        s.advance_checkins(120);
        void* h = generate_ref(sc);
        gbxref_suite_advance(h, 120);
        BehaviorPolicy beh{PolicyNet::init(17), 0, 0};
        const EvalReport rep = evaluate(s, beh, 10, 77);
        std::vector<double> rows(3 * sc.benchmarks), lo(4096);
        std::vector<std::uint64_t> cnt(4096);
        const auto flat = beh.net.flat();
        const long bins = gbxref_evaluate(h, flat.data(), 10, 77, 1, rows.data(), lo.data(), cnt.data(), 4096);
        gbxref_suite_free(h);
        REQUIRE(bins > 0);
        REQUIRE(rep.rows.size() == (std::size_t)sc.benchmarks);
        for (int b = 0; b < sc.benchmarks; ++b) {
            CHECK(rep.rows[b].baseline_fps == rows[3 * b]);
            CHECK(rep.rows[b].tuned_fps == rows[3 * b + 1]);
            CHECK(rep.rows[b].uplift_pct == rows[3 * b + 2]);
        }
        REQUIRE(rep.histogram.size() == (std::size_t)bins);
        for (long k = 0; k < bins; ++k) {
            CHECK(rep.histogram[k].lower_pct == lo[k]);
            CHECK(rep.histogram[k].count == cnt[k]);
        }
    }
}

TEST_CASE("QTable keeps one table across its host map and its device copy") {
    QTable t({0.3, 0.99});
    StateKey k1, k2;
    k1.values[0] = 1;
    k1.values[5] = 9;
    k2.values[0] = 2;
    t.update(k1, Action::Wave32, 1.0, 0);  // host
    std::vector<ExperienceTuple> batch{{k1, Action::Wave64, 1.2, 3}, {k2, Action::Wave32, 0.8, 3},
                                       {k1, Action::Wave32, 0.9, 4}};
    t.update_batch(batch);                 // device (after a host -> device sync)
    CHECK(t.state_count() == 2);
    REQUIRE(t.find(k1, Action::Wave32) != nullptr);  // device -> host sync
    CHECK(t.find(k1, Action::Wave32)->update_count == 2);
    CHECK(t.find(k1, Action::Wave32)->q == (1.0 - 0.3) * std::pow(0.99, 4.0) * 1.0 + 0.3 * 0.9);
    t.update(k2, Action::Wave64, 1.1, 5);  // host again: the device copy is stale now
    const auto ds = t.snapshot_policy_dataset(0.1);  // device, re-synced
    CHECK(ds.size() == 2);
    const QTable copy = t;  // copies never share the device table
    t.update_batch({{k2, Action::Wave64, 2.0, 6}});
    CHECK(copy.find(k2, Action::Wave64)->update_count == 1);
    CHECK(t.find(k2, Action::Wave64)->update_count == 2);
    std::ostringstream a, b;
    t.save(b);
    std::istringstream in(b.str());
    QTable::load(in).save(a);
    CHECK(a.str() == b.str());
    // a check-in older than the entry: the reference's error, prefix kept
    CHECK_THROWS_AS(t.update_batch({{k1, Action::Wave32, 1.0, 7}, {k1, Action::Wave32, 1.0, 2}}),
                    ClockRegressionError);
    CHECK(t.find(k1, Action::Wave32)->last_update_t == 7);
}
