// test_dropin_parity.cpp — the C++ drop-in (gbx:: API over libgbxcu, on the
// B200) against the compiled reference library (libgbxref.so, reached through
// its C adapter oracle/ref_capi.cpp) in one process, on the same inputs.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cstring>
#include <limits>
#include <sstream>

#include "gbx/device_qtable.hpp"
#include "gbx/policy.hpp"
#include "gbx/qtable.hpp"
#include "gbx/tuner.hpp"

extern "C" {
void gbxref_g1(std::uint64_t seed, std::size_t n, float* feat, double* tgt);
void gbxref_policy_init(std::uint64_t seed, float* params);
int gbxref_forward(const float* params, const float* feat, std::size_t n, double* probs,
                   std::uint8_t* actions);
void gbxref_batch_kl_gradient(const float* params, const float* feat, const double* tgt,
                              std::size_t n, double* grad);
int gbxref_fit(float* params, const float* feat, const double* tgt, std::size_t n, double lr,
               int epochs, int batch, std::uint64_t seed, double* epoch_loss, int* diverged_epoch);
long gbxref_qtable_snapshot(const char* text, double rho, float* feat, double* tgt);
long gbxref_qtable_fold(const std::uint32_t* keys, const std::uint8_t* actions, const double* rewards,
                        const std::uint64_t* now, std::size_t n, double alpha, double omega,
                        double rho, long* sizes, long* bad, std::uint32_t* out_keys, double* out_q,
                        std::uint64_t* out_t, std::uint64_t* out_cnt, std::uint8_t* out_has,
                        float* feat, double* tgt);
void* gbxref_suite_generate(int, int, int, int, int, double, double, double, std::uint64_t);
void gbxref_suite_free(void*);
void gbxref_suite_dims(const void*, std::size_t* dims);
void gbxref_suite_export(const void*, double*, float*, double*, std::uint64_t*, double*,
                         std::uint64_t*, std::uint32_t*, double*, std::uint64_t*, std::uint32_t*);
long gbxref_evaluate(const void*, const float*, int, std::uint64_t, int, double*, double*,
                     std::uint64_t*, std::size_t);
}

using namespace gbx;

namespace {

PolicyDataset g1(std::uint64_t seed, std::size_t n) {
    std::vector<float> f(n * kFeatureCount);
    std::vector<double> t(2 * n);
    gbxref_g1(seed, n, f.data(), t.data());
    PolicyDataset d(n);
    for (std::size_t r = 0; r < n; ++r) {
        std::memcpy(d[r].first.features.data(), f.data() + r * kFeatureCount, 4 * kFeatureCount);
        d[r].second.prob = {t[2 * r], t[2 * r + 1]};
    }
    return d;
}

void flat_data(const PolicyDataset& d, std::vector<float>& f, std::vector<double>& t) {
    f.resize(d.size() * kFeatureCount);
    t.resize(d.size() * 2);
    for (std::size_t r = 0; r < d.size(); ++r) {
        std::memcpy(f.data() + r * kFeatureCount, d[r].first.features.data(), 4 * kFeatureCount);
        t[2 * r] = d[r].second.prob[0];
        t[2 * r + 1] = d[r].second.prob[1];
    }
}

long ulp_gap(float a, float b) {
    std::int32_t x, y;
    std::memcpy(&x, &a, 4);
    std::memcpy(&y, &b, 4);
    return std::labs(static_cast<long>(x) - static_cast<long>(y));
}

}  // namespace

TEST_CASE("PolicyNet::init is bit-identical to the reference") {
    std::vector<float> ref(kPolicyParamCount);
    gbxref_policy_init(7, ref.data());
    CHECK(PolicyNet::init(7).flat() == ref);
}

TEST_CASE("fit (config C1) matches the reference to <= 1 fp32 ulp per weight") {
    const auto data = g1(42, 10000);
    PolicyNet net = PolicyNet::init(7);
    std::vector<float> ref = net.flat();
    TrainConfig cfg;
    cfg.epochs = 1;
    cfg.seed = 99;
    const FitResult fr = fit(net, data, cfg);
    std::vector<float> f;
    std::vector<double> t;
    flat_data(data, f, t);
    double ref_loss = 0;
    int div = -1;
    REQUIRE(gbxref_fit(ref.data(), f.data(), t.data(), data.size(), 0.01, 1, 32, 99, &ref_loss, &div) == 0);
    const auto got = net.flat();
    long worst = 0;
    for (std::size_t i = 0; i < got.size(); ++i) worst = std::max(worst, ulp_gap(got[i], ref[i]));
    CHECK(worst <= 1);
    CHECK(fr.epoch_loss[0] == doctest::Approx(ref_loss).epsilon(1e-12));
}

TEST_CASE("batch_kl_gradient matches the reference") {
    const auto data = g1(77, 32);
    const PolicyNet net = PolicyNet::init(7);
    const auto g = batch_kl_gradient(net, data);
    std::vector<float> f;
    std::vector<double> t;
    flat_data(data, f, t);
    std::vector<double> ref(kPolicyParamCount);
    gbxref_batch_kl_gradient(net.flat().data(), f.data(), t.data(), data.size(), ref.data());
    for (std::size_t i = 0; i < ref.size(); ++i)
        CHECK(g[i] == doctest::Approx(ref[i]).epsilon(1e-12));
}

TEST_CASE("greedy actions are bit-identical (per-state and batched)") {
    const auto data = g1(5, 20000);
    BehaviorPolicy beh{PolicyNet::init(9), 1, 0};
    std::vector<ShaderState> states;
    for (const auto& r : data) states.push_back(r.first);
    std::vector<float> f;
    std::vector<double> t;
    flat_data(data, f, t);
    std::vector<std::uint8_t> ref(states.size());
    std::vector<double> probs(2 * states.size());
    REQUIRE(gbxref_forward(beh.net.flat().data(), f.data(), states.size(), probs.data(), ref.data()) == 0);
    const auto got = select_greedy_batch(beh, states);
    std::size_t diff = 0;
    for (std::size_t i = 0; i < got.size(); ++i) diff += static_cast<int>(got[i]) != ref[i];
    CHECK(diff == 0);
    for (int i = 0; i < 50; ++i) {
        CHECK(static_cast<int>(select_greedy(beh, states[i])) == ref[i]);
        const auto p = beh.forward(states[i]);
        CHECK(p[0] == doctest::Approx(probs[2 * i]).epsilon(1e-15));
    }
}

TEST_CASE("batched select_sample equals select_sample in order; the stream advances alike") {
    const auto data = g1(8, 5000);
    BehaviorPolicy beh{PolicyNet::init(4), 1, 0};
    std::vector<ShaderState> states;
    for (const auto& r : data) states.push_back(r.first);
    SplitMix64 a(777), b(777);
    const auto got = select_sample_batch(beh, states, a);
    std::size_t diff = 0;
    for (std::size_t i = 0; i < states.size(); ++i)
        diff += got[i] != select_sample(beh, states[i], b);
    CHECK(diff == 0);
    CHECK(a.state() == b.state());
}

TEST_CASE("variants (extension): TD regression and Adam through the drop-in") {
    const auto data = g1(3, 4000);
    std::vector<ExperienceRecord> recs;
    SplitMix64 rng(5);
    for (const auto& r : data) {
        const Action a = rng.next_unit() < 0.5 ? Action::Wave32 : Action::Wave64;
        recs.push_back({r.first, a, 0.5 + 0.1 * r.first.features[8] * (a == Action::Wave64 ? 1 : -1)});
    }
    TrainConfig cfg;
    cfg.learning_rate = 1e-3;
    cfg.epochs = 4;
    cfg.batch_size = 64;
    cfg.seed = 3;
    OptimizerConfig adam;
    adam.kind = OptimizerKind::Adam;
    PolicyNet a = PolicyNet::init(1), b = PolicyNet::init(1);
    const auto ra = fit_td(a, recs, cfg, adam);
    const auto rb = fit_td(b, recs, cfg, adam);
    CHECK(ra.epoch_loss == rb.epoch_loss);            // deterministic
    CHECK(a.flat() == b.flat());
    CHECK(ra.epoch_loss.back() < 0.7 * ra.epoch_loss.front());  // it learns
    PolicyNet s = PolicyNet::init(2), m = PolicyNet::init(2);
    fit(s, data, cfg);
    fit(m, data, cfg, adam);
    CHECK(s.flat() != m.flat());
    recs[7].reward = std::numeric_limits<double>::infinity();
    PolicyNet d = PolicyNet::init(1);
    CHECK_THROWS_AS(fit_td(d, recs, cfg), TrainingDivergedError);
}

TEST_CASE("q-table load + snapshot equals the reference's dataset") {
    const char* text =
        "gbx-qtable 1 0.3 0.99\n"
        "0 5 40 20 5 5 5 30 10 10 5 25 15 10 2 8 5 20 10 10 3 10 6 2 3 90 40 0 0 0 0 1.05 10 1\n"
        "0 5 40 20 5 5 5 30 10 10 5 25 15 10 2 8 5 20 10 10 3 10 6 2 3 90 40 0 0 0 1 0.97 12 3\n"
        "7 9 120 80 30 12 9 70 40 33 19 60 48 30 7 21 14 55 34 30 11 31 20 6 9 200 77 0 0 0 1 1.5 100 9\n"
        "7 9 120 80 30 12 9 70 40 33 19 60 48 30 7 21 14 55 34 30 11 31 20 6 9 200 77 0 0 0 0 1.4 90 4\n";
    std::istringstream is(text);
    const auto ds = QTable::load(is).snapshot_policy_dataset(0.1);
    const long n = gbxref_qtable_snapshot(text, 0.1, nullptr, nullptr);
    REQUIRE(n == static_cast<long>(ds.size()));
    std::vector<float> f(n * kFeatureCount);
    std::vector<double> t(2 * n);
    gbxref_qtable_snapshot(text, 0.1, f.data(), t.data());
    for (long r = 0; r < n; ++r) {
        CHECK(std::memcmp(ds[r].first.features.data(), f.data() + r * kFeatureCount, 176) == 0);
        CHECK(ds[r].second.prob[0] == t[2 * r]);
        CHECK(ds[r].second.prob[1] == t[2 * r + 1]);
    }
}

TEST_CASE("evaluate over a reference-generated suite is bit-identical") {
    for (double cap : {0.0, 1.0}) {
        void* h = gbxref_suite_generate(10, 184, 276, 2, 4, cap, 0.005, 1.0, 21);
        REQUIRE(h != nullptr);
        std::size_t d[5];
        gbxref_suite_dims(h, d);
        SuiteArrays s;
        std::vector<float> feat(d[0] * kFeatureCount);
        s.shader_lat.resize(3 * d[0]);
        s.app_f64.resize(4 * d[1]);
        s.app_pipe_off.resize(d[1] + 1);
        s.pipe_wt.resize(2 * d[2]);
        s.pipe_slot_off.resize(d[2] + 1);
        s.slot_shader.resize(d[3]);
        s.slot_frac.resize(d[3]);
        std::vector<std::uint64_t> moff(d[1] + 1);
        std::vector<std::uint32_t> mem(d[4]);
        gbxref_suite_export(h, s.shader_lat.data(), feat.data(), s.app_f64.data(), s.app_pipe_off.data(),
                            s.pipe_wt.data(), s.pipe_slot_off.data(), s.slot_shader.data(),
                            s.slot_frac.data(), moff.data(), mem.data());
        s.shader_state.resize(d[0]);
        for (std::size_t i = 0; i < d[0]; ++i)
            std::memcpy(s.shader_state[i].features.data(), feat.data() + i * kFeatureCount, 176);
        BehaviorPolicy beh{PolicyNet::init(31), 0, 0};
        const EvalReport rep = evaluate(s, beh, 10, 77);
        std::vector<double> rows(3 * d[1]), lower(4096);
        std::vector<std::uint64_t> count(4096);
        const long bins = gbxref_evaluate(h, beh.net.flat().data(), 10, 77, 1, rows.data(),
                                          lower.data(), count.data(), 4096);
        gbxref_suite_free(h);
        REQUIRE(rep.rows.size() == d[1]);
        for (std::size_t b = 0; b < d[1]; ++b) {
            CHECK(rep.rows[b].tuned_fps == rows[3 * b + 1]);
            CHECK(rep.rows[b].uplift_pct == rows[3 * b + 2]);
        }
        REQUIRE(static_cast<long>(rep.histogram.size()) == bins);
        for (long k = 0; k < bins; ++k) {
            CHECK(rep.histogram[k].lower_pct == lower[k]);
            CHECK(rep.histogram[k].count == count[k]);
        }
    }
}

TEST_CASE("errors keep the reference's exception types") {
    PolicyNet net = PolicyNet::init(1);
    TrainConfig cfg;
    CHECK_THROWS_AS(fit(net, {}, cfg), ValidationError);
    cfg.learning_rate = 0.0;
    CHECK_THROWS_AS(fit(net, g1(1, 4), cfg), ValidationError);
    ShaderState bad;
    bad.features[3] = std::numeric_limits<float>::infinity();
    CHECK_THROWS_AS(net.forward(bad), ValidationError);
    CHECK_THROWS_AS(boltzmann_pair(1.0, 2.0, 0.0), InvalidTemperatureError);
}

TEST_CASE("DeviceQTable fold + snapshot equal the reference QTable; host round trip") {
    const std::size_t n = 30000;
    std::vector<std::uint32_t> keys(n * 30);
    std::vector<std::uint8_t> act(n);
    std::vector<double> rew(n);
    std::vector<std::uint64_t> now(n);
    std::uint64_t s = 12345;
    auto next = [&] { s = s * 6364136223846793005ull + 1442695040888963407ull; return s >> 33; };
    std::vector<ExperienceTuple> tup(n);
    for (std::size_t i = 0; i < n; ++i) {
        const std::uint64_t k = next() % 4000;  // ~4000 distinct keys
        for (int w = 0; w < 30; ++w) keys[i * 30 + w] = w == 0 ? k % 8 : (std::uint32_t)((k * (w + 7)) % 97);
        act[i] = next() & 1;
        rew[i] = 0.8 + (next() % 1000) / 2500.0;
        now[i] = i / 50;
        std::memcpy(tup[i].key.values.data(), keys.data() + i * 30, 120);
        tup[i].action = act[i] ? Action::Wave64 : Action::Wave32;
        tup[i].reward = rew[i];
        tup[i].now = now[i];
    }
    long sizes[2], bad = -1;
    gbxref_qtable_fold(keys.data(), act.data(), rew.data(), now.data(), n, 0.3, 1.0, 0.1, sizes, &bad,
                       nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    std::vector<std::uint32_t> rk(sizes[0] * 30);
    std::vector<double> rq(sizes[0] * 2), rt_f(sizes[1] * 2);
    std::vector<std::uint64_t> rt(sizes[0] * 2), rc(sizes[0] * 2);
    std::vector<std::uint8_t> rh(sizes[0] * 2);
    std::vector<float> rf(sizes[1] * kFeatureCount);
    gbxref_qtable_fold(keys.data(), act.data(), rew.data(), now.data(), n, 0.3, 1.0, 0.1, sizes, &bad,
                       rk.data(), rq.data(), rt.data(), rc.data(), rh.data(), rf.data(), rt_f.data());

    DeviceQTable dq(QHyperparams{0.3, 1.0});
    dq.update_batch(tup);
    CHECK(dq.state_count() == (std::size_t)sizes[0]);
    const auto snap = dq.snapshot_policy_dataset(0.1);
    REQUIRE(snap.size() == (std::size_t)sizes[1]);
    bool feat_ok = true, tgt_ok = true;
    for (std::size_t r = 0; r < snap.size(); ++r) {
        feat_ok &= std::memcmp(snap[r].first.features.data(), rf.data() + r * kFeatureCount,
                               4 * kFeatureCount) == 0;
        for (int a = 0; a < 2; ++a)
            tgt_ok &= std::abs(snap[r].second.prob[a] - rt_f[2 * r + a]) <= 1e-15 * rt_f[2 * r + a];
    }
    CHECK(feat_ok);
    CHECK(tgt_ok);
    // host round trip: to_host -> save -> load -> from_host -> same snapshot
    const QTable host = dq.to_host();
    std::ostringstream os;
    host.save(os);
    std::istringstream is(os.str());
    const auto back = DeviceQTable::from_host(QTable::load(is));
    const auto snap2 = back.snapshot_policy_dataset(0.1);
    REQUIRE(snap2.size() == snap.size());
    bool same = true;
    for (std::size_t r = 0; r < snap.size(); ++r)
        same &= snap[r].first == snap2[r].first && snap[r].second.prob == snap2[r].second.prob;
    CHECK(same);
    // ClockRegressionError: time going backwards for a repeated key
    std::vector<ExperienceTuple> bad_t(tup.begin(), tup.begin() + 3);
    bad_t[1] = bad_t[0];
    bad_t[0].now = 10;
    bad_t[1].now = 5;
    DeviceQTable dq2;
    CHECK_THROWS_AS(dq2.update_batch(bad_t), ClockRegressionError);
    CHECK(dq2.state_count() == 1);
}

