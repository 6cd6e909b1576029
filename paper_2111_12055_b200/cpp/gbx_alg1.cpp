// gbx_alg1.cpp — the SimSuite-facing part of the drop-in (libgbx_b200_alg1.so):
// evaluate(const SimSuite&, ...) (proj/src/tuner.cpp:266-315), run_iteration
// (:172-239) and run_training (:241-264) with every data-parallel step on the
// B200 through the C ABI:
//
//   collection        gbxcu_collect     sampled, epsilon-mixed actions (A8)
//   run_benchmark     gbxcu_aggregate   frame_time, noisy samples, reward (A9, A10)
//   table fold        QTable::update_batch -> k_qtable.cu (f1)
//   snapshot          QTable::snapshot_policy_dataset -> k_qtable.cu (A11)
//   distillation      fit -> the fused train kernels (A5)
//   agreement         select_greedy_batch -> fwd kernels (A7)
//
// Host code does what the reference's loop does between those calls: seeds,
// schedules, the per-benchmark member lists, the reward fold and the log. The
// suite is read only through SimSuite's public accessors; its environment
// code (advance_checkins, compile) is the reference's own.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "gbx/rng.hpp"
#include "gbx/tuner.hpp"
#include "gbxcu.h"
#include "internal.hpp"

namespace gbx {

namespace {

// RNG stream tags of the tuner (proj/src/tuner.cpp:22-26)
constexpr std::uint64_t kActionTag = 0x414354;
constexpr std::uint64_t kFpsTag = 0x465053;
constexpr std::uint64_t kFitTag = 0x464954;
constexpr std::uint64_t kInitTag = 0x494E49;
constexpr std::uint64_t kEvalTag = 0x45564C;

using detail::check_status;
using detail::device_context;

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

// Pipelines and slots of every benchmark in order (the CSR skeleton shared by
// evaluate and the collection's member suite); slot_shader holds shader ids.
void csr_skeleton(const SimSuite& suite, SuiteArrays& a) {
    const auto& benches = suite.benchmarks();
    a.app_pipe_off.assign(1, 0);
    a.pipe_slot_off.assign(1, 0);
    a.slot_shader.clear();
    a.slot_frac.clear();
    a.pipe_wt.clear();
    a.app_f64.clear();
    for (const SimBenchmark& b : benches) {
        for (const SimPipeline& p : b.pipelines) {
            for (const PipelineSlot& sl : p.slots) {
                a.slot_shader.push_back(sl.shader_id);
                a.slot_frac.push_back(sl.exec_fraction);
            }
            a.pipe_wt.push_back(p.weight);
            a.pipe_wt.push_back(p.base_time);
            a.pipe_slot_off.push_back(a.slot_shader.size());
        }
        a.app_pipe_off.push_back(a.pipe_slot_off.size() - 1);
        a.app_f64.insert(a.app_f64.end(),
                         {b.baseline_fps, b.bandwidth_capacity, b.noise_sigma, b.memory_bound_threshold});
    }
}

void push_latents(const SimShader& sh, std::vector<double>& lat) {
    lat.insert(lat.end(), {sh.divergence, sh.bandwidth_demand, sh.parallelism});
}

}  // namespace

SuiteArrays SuiteArrays::from_suite(const SimSuite& suite) {
    SuiteArrays a;
    csr_skeleton(suite, a);
    const std::size_t n = suite.shaders().size();
    a.shader_lat.reserve(3 * n);
    a.shader_state.resize(n);
    for (std::size_t id = 0; id < n; ++id) {
        const SimShader& sh = suite.shader(static_cast<std::uint32_t>(id));
        push_latents(sh, a.shader_lat);
        a.shader_state[id] = suite.compile(static_cast<std::uint32_t>(id), kDefaultAction).first;
    }
    return a;
}

EvalReport evaluate(const SimSuite& suite, const BehaviorPolicy& policy, int n_samples,
                    std::uint64_t seed, int jobs) {
    if (n_samples < 1) throw ValidationError("sample count must be >= 1");
    const auto& benches = suite.benchmarks();
    bool dense_ids = true;  // gbxcu_evaluate seeds app b by its index
    for (std::size_t b = 0; b < benches.size(); ++b) dense_ids = dense_ids && benches[b].id == b;
    const SuiteArrays a = SuiteArrays::from_suite(suite);
    if (dense_ids) return evaluate(a, policy, n_samples, seed, jobs);
    // general ids: greedy actions, then run_benchmarks with each benchmark's
    // own derive_seed({seed, kEvalTag, bench.id}) (tuner.cpp:280-281)
    const std::vector<Action> act = select_greedy_batch(policy, a.shader_state);
    std::vector<std::uint64_t> seeds(benches.size());
    for (std::size_t b = 0; b < benches.size(); ++b) seeds[b] = derive_seed({seed, kEvalTag, benches[b].id});
    const auto rows = run_benchmarks(a, act, seeds, n_samples);
    std::vector<double> uplift(rows.size());
    for (std::size_t b = 0; b < rows.size(); ++b) uplift[b] = rows[b][3];
    EvalReport rep;
    rep.rows.resize(rows.size());
    for (std::size_t b = 0; b < rows.size(); ++b)
        rep.rows[b] = {benches[b].id, benches[b].baseline_fps, rows[b][2], rows[b][3]};
    constexpr std::size_t kCap = 1 << 16;
    std::vector<double> lower(kCap);
    std::vector<std::uint64_t> count(kCap);
    std::size_t bins = 0;
    if (!uplift.empty())
        check_status(gbxcu_histogram(device_context(), uplift.data(), uplift.size(), lower.data(),
                                     count.data(), kCap, &bins));
    if (bins > kCap) throw std::runtime_error("uplift histogram exceeds 65536 bins");
    rep.histogram.resize(bins);
    for (std::size_t k = 0; k < bins; ++k)
        rep.histogram[k] = {lower[k], lower[k] + 1.0, static_cast<std::size_t>(count[k])};
    return rep;
}

IterationLog run_iteration(TunerState& state, const TunerConfig& cfg, int iteration) {
    cfg.validate();
    state.suite.advance_checkins(static_cast<std::uint64_t>(cfg.checkins_per_iteration));
    const Checkin now = state.suite.checkin();
    const double eps = cfg.epsilon_at(iteration);
    const auto& benches = state.suite.benchmarks();
    const std::size_t nb = benches.size();
    const auto it64 = static_cast<std::uint64_t>(iteration);

    // Members: (benchmark, shader) pairs in benchmark order, shader_ids order
    // (a shared shader gets its own draw in each benchmark's stream). Each
    // distinct shader is compiled once at this check-in.
    const std::size_t n_sh = state.suite.shaders().size();
    std::vector<std::uint8_t> compiled(n_sh, 0);
    std::vector<float> sh_feat(n_sh * kFeatureCount);
    std::vector<StateKey> sh_key(n_sh);
    std::vector<std::uint64_t> moff(nb + 1, 0);
    std::vector<std::uint32_t> members;
    for (std::size_t b = 0; b < nb; ++b) {
        for (const std::uint32_t id : benches[b].shader_ids) {
            if (!compiled[id]) {
                const auto [st, key] = state.suite.compile(id, kDefaultAction);
                std::memcpy(sh_feat.data() + (std::size_t)id * kFeatureCount, st.features.data(),
                            sizeof(float) * kFeatureCount);
                sh_key[id] = key;
                compiled[id] = 1;
            }
            members.push_back(id);
        }
        moff[b + 1] = members.size();
    }
    const std::size_t nm = members.size();
    std::vector<float> m_feat(nm * kFeatureCount);
    for (std::size_t j = 0; j < nm; ++j)
        std::memcpy(m_feat.data() + j * kFeatureCount, sh_feat.data() + (std::size_t)members[j] * kFeatureCount,
                    sizeof(float) * kFeatureCount);

    // ---- collection: SplitMix64(derive_seed({seed, ACT, i, bench.id})), two
    //      draws per shader, epsilon-uniform or sampled from the behavior net
    std::vector<std::uint64_t> seg_seed(nb), run_seed(nb);
    for (std::size_t b = 0; b < nb; ++b) {
        seg_seed[b] = derive_seed({cfg.seed, kActionTag, it64, benches[b].id});
        run_seed[b] = derive_seed({cfg.seed, kFpsTag, it64, benches[b].id});
    }
    gbxcu_ctx* c = device_context();
    const std::vector<float> beh = state.behavior.net.flat();
    std::vector<std::uint8_t> act(nm);
    if (nm)
        check_status(gbxcu_collect(c, beh.data(), m_feat.data(), moff.data(), nb, seg_seed.data(), eps,
                                   act.data()));

    // ---- run_benchmark + attribute_rewards on the member suite: slots index
    //      their benchmark's member list, one latent row per member
    SuiteArrays ms;
    csr_skeleton(state.suite, ms);
    ms.shader_lat.reserve(3 * nm);
    for (std::size_t j = 0; j < nm; ++j) push_latents(state.suite.shader(members[j]), ms.shader_lat);
    for (std::size_t b = 0; b < nb; ++b) {
        const auto m_lo = members.begin() + (std::ptrdiff_t)moff[b];
        const auto m_hi = members.begin() + (std::ptrdiff_t)moff[b + 1];
        for (std::uint64_t p = ms.app_pipe_off[b]; p < ms.app_pipe_off[b + 1]; ++p)
            for (std::uint64_t s = ms.pipe_slot_off[p]; s < ms.pipe_slot_off[p + 1]; ++s)
                ms.slot_shader[s] = static_cast<std::uint32_t>(std::lower_bound(m_lo, m_hi, ms.slot_shader[s]) -
                                                               members.begin());
    }
    std::vector<double> rows(5 * nb);
    if (nb) {
        const gbxcu_suite v = view(ms);
        check_status(gbxcu_aggregate(c, &v, act.data(), run_seed.data(), cfg.samples_per_benchmark,
                                     rows.data(), nullptr));
    }

    // ---- fold (benchmark order, observations in shader-id order) on the device
    std::vector<ExperienceTuple> tuples(nm);
    double reward_sum = 0.0;
    for (std::size_t b = 0; b < nb; ++b) {
        const double r = rows[5 * b + 4];
        for (std::uint64_t j = moff[b]; j < moff[b + 1]; ++j)
            tuples[j] = {sh_key[members[j]], action_from_index(act[j]), r, now};
        reward_sum += moff[b + 1] > moff[b] ? r : 1.0;
    }
    state.table.update_batch(tuples);

    // ---- distillation on the snapshot at rho_i
    const PolicyDataset dataset = state.table.snapshot_policy_dataset(cfg.train.rho_at(iteration));
    double distill_loss = 0.0;
    if (!dataset.empty()) {
        TrainConfig tcfg = cfg.train;
        tcfg.seed = derive_seed({cfg.seed, kFitTag, it64});
        distill_loss = fit(state.decision, dataset, tcfg).epoch_loss.back();
    }
    if (iteration % cfg.refresh_period == 0)
        state.behavior = BehaviorPolicy{state.decision, static_cast<std::uint32_t>(iteration + 1), now};

    // ---- agreement: the table's greedy action vs the net's, over the states
    //      with both actions — exactly the snapshot's rows, in key order
    double agreement = 1.0;
    if (!dataset.empty()) {
        const std::vector<std::uint8_t> greedy = state.table.greedy_wave64_of_complete_states();
        std::vector<ShaderState> states(dataset.size());
        for (std::size_t r = 0; r < dataset.size(); ++r) states[r] = dataset[r].first;
        const std::vector<Action> net = select_greedy_batch(BehaviorPolicy{state.decision, 0, 0}, states);
        std::size_t agree = 0;
        for (std::size_t r = 0; r < net.size(); ++r)
            agree += (greedy[r] != 0) == (net[r] == Action::Wave64) ? 1 : 0;
        agreement = static_cast<double>(agree) / static_cast<double>(net.size());
    }

    IterationLog log;
    log.iteration = iteration;
    log.checkin = now;
    log.mean_reward = nb == 0 ? 1.0 : reward_sum / static_cast<double>(nb);
    log.table_size = state.table.state_count();
    log.distill_loss = distill_loss;
    log.agreement_rate = agreement;
    return log;
}

TrainResult run_training(SimSuite suite, const TunerConfig& cfg, const std::optional<WarmStart>& warm) {
    cfg.validate();
    TunerState state{std::move(suite), warm ? warm->table : QTable(cfg.qtable),
                     warm ? warm->policy : PolicyNet::init(derive_seed({cfg.seed, kInitTag})),
                     BehaviorPolicy{}};
    state.behavior = BehaviorPolicy{state.decision, 0, state.suite.checkin()};
    TrainResult result{state.behavior, state.table, {}};
    result.logs.reserve(static_cast<std::size_t>(cfg.num_iterations));
    for (int i = 0; i < cfg.num_iterations; ++i) {
        try {
            result.logs.push_back(run_iteration(state, cfg, i));
        } catch (const TrainingDivergedError& e) {
            throw TrainingDivergedError(i, "iteration " + std::to_string(i) + ": " + e.what());
        }
    }
    result.policy = state.behavior;
    result.table = std::move(state.table);
    return result;
}

}  // namespace gbx
