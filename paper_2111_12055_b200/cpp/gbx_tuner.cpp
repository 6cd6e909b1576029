// gbx_tuner.cpp — reward normalisation and the greedy evaluation sweep of the
// drop-in (proj/src/tuner.cpp:131-147, 266-315; proj/src/simenv.cpp:439-510),
// executed by libgbxcu's fused inference + segmented aggregation kernels.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <stdexcept>
#include <string>

#include "gbx/tuner.hpp"
#include "gbxcu.h"
#include "internal.hpp"

namespace gbx {

namespace {

gbxcu_ctx* device_ctx() { return detail::device_context(); }

void check(int rc) { detail::check_status(rc); }

gbxcu_suite view(const SuiteArrays& s) {
    gbxcu_suite v{};
    v.n_apps = s.n_apps();
    v.n_pipes = s.pipe_slot_off.empty() ? 0 : s.pipe_slot_off.size() - 1;
    v.n_slots = s.slot_shader.size();
    v.n_shaders = s.n_shaders();
    v.app_pipe_off = s.app_pipe_off.data();
    v.pipe_slot_off = s.pipe_slot_off.data();
    v.slot_shader = s.slot_shader.data();
    v.slot_frac = s.slot_frac.data();
    v.pipe_wt = s.pipe_wt.data();
    v.shader_lat = s.shader_lat.data();
    v.app_f64 = s.app_f64.data();
    return v;
}

}  // namespace

// TunerConfig checks and the epsilon schedule (tuner.cpp:36-57).
void TunerConfig::validate() const {
    if (num_iterations < 0) throw ValidationError("iteration count must be >= 0");
    if (checkins_per_iteration < 0) throw ValidationError("check-ins per iteration must be >= 0");
    if (!(epsilon0 >= 0.0 && epsilon0 <= 1.0)) throw ValidationError("epsilon0 must be in [0, 1]");
    if (epsilon_horizon < 0) throw ValidationError("epsilon horizon must be >= 0");
    if (refresh_period < 1) throw ValidationError("refresh period must be >= 1");
    if (samples_per_benchmark < 1) throw ValidationError("samples per benchmark must be >= 1");
    if (jobs < 1) throw ValidationError("jobs must be >= 1");
    qtable.validate();
    train.validate();
}

// epsilon decays linearly to 0 over the horizon (num_iterations / 2 by default)
double TunerConfig::epsilon_at(int iteration) const {
    const int horizon = epsilon_horizon > 0 ? epsilon_horizon : std::max(1, num_iterations / 2);
    return epsilon0 * std::max(0.0, 1.0 - static_cast<double>(iteration) / horizon);
}

std::vector<RewardAttribution> attribute_rewards(const RunRecord& record,
                                                 std::span<const double> samples,
                                                 double baseline_fps) {
    if (samples.empty()) throw ValidationError("reward attribution needs at least one sample");
    const double mean = std::accumulate(samples.begin(), samples.end(), 0.0) /
                        static_cast<double>(samples.size());
    const Reward r = reward_from_framerate(mean, baseline_fps);
    std::vector<RewardAttribution> out;
    out.reserve(record.observations.size());
    for (const auto& o : record.observations) out.push_back({o.key, o.action, r});
    return out;
}

EvalReport evaluate(const SuiteArrays& suite, const BehaviorPolicy& policy, int n_samples,
                    std::uint64_t seed, int /*jobs: the device sweep has no host threads*/) {
    if (n_samples < 1) throw ValidationError("sample count must be >= 1");
    const auto v = view(suite);
    if (suite.shader_state.size() != v.n_shaders)
        throw ValidationError("suite needs one compiled state per shader");
    std::vector<float> feat(v.n_shaders * kFeatureCount);
    for (std::size_t i = 0; i < v.n_shaders; ++i)
        std::copy(suite.shader_state[i].features.begin(), suite.shader_state[i].features.end(),
                  feat.begin() + i * kFeatureCount);
    gbxcu_ctx* c = device_ctx();
    gbxcu_dsuite* ds = nullptr;
    check(gbxcu_suite_upload(c, &v, feat.data(), &ds));
    const auto params = policy.net.flat();
    std::vector<double> rows(5 * v.n_apps);
    constexpr std::size_t kCap = 1 << 16;
    std::vector<double> lower(kCap);
    std::vector<std::uint64_t> count(kCap);
    std::size_t bins = 0;
    const int rc = gbxcu_evaluate(c, ds, params.data(), n_samples, seed, rows.data(), nullptr,
                                  lower.data(), count.data(), kCap, &bins);
    gbxcu_suite_free(ds);
    check(rc);
    EvalReport rep;
    rep.rows.resize(v.n_apps);
    for (std::size_t b = 0; b < v.n_apps; ++b)
        rep.rows[b] = {static_cast<std::uint32_t>(b), suite.app_f64[4 * b], rows[5 * b + 2], rows[5 * b + 3]};
    if (bins > kCap) throw std::runtime_error("uplift histogram exceeds 65536 bins");
    rep.histogram.resize(bins);
    for (std::size_t k = 0; k < bins; ++k)
        rep.histogram[k] = {lower[k], lower[k] + 1.0, static_cast<std::size_t>(count[k])};
    return rep;
}

std::vector<std::array<double, 5>> run_benchmarks(const SuiteArrays& suite,
                                                  std::span<const Action> shader_actions,
                                                  std::span<const std::uint64_t> run_seeds,
                                                  int n_samples) {
    const auto v = view(suite);
    if (shader_actions.size() != v.n_shaders || run_seeds.size() != v.n_apps)
        throw ValidationError("run_benchmarks: actions per shader and one seed per app required");
    std::vector<std::uint8_t> act(v.n_shaders);
    for (std::size_t i = 0; i < act.size(); ++i) act[i] = static_cast<std::uint8_t>(shader_actions[i]);
    std::vector<std::array<double, 5>> rows(v.n_apps);
    if (rows.empty()) return rows;
    check(gbxcu_aggregate(device_ctx(), &v, act.data(), run_seeds.data(), n_samples,
                          rows.empty() ? nullptr : rows.data()->data(), nullptr));
    return rows;
}

}  // namespace gbx
