// gbx_policy.cpp — the policy API of the drop-in, executed on the B200.
//
// fit, batch_kl_loss, batch_kl_gradient, PolicyNet::init/forward and the
// select_* functions marshal into one flat fp32 parameter vector plus
// [n][44] fp32 features / [n][2] fp64 targets and call libgbxcu (C ABI,
// include/gbxcu.h). Status codes map back onto the reference's exception
// types (proj/include/gbx/policy.hpp:16-31). Only the GBXP byte format and the
// scalar kl_loss stay on the host (no batched work behind them).
#include <zlib.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <string>

#include "gbx/device_qtable.hpp"
#include "gbx/policy.hpp"
#include "gbxcu.h"
#include "internal.hpp"

namespace gbx {

namespace {

// ------------------------------------------------------------ device context
std::mutex g_mu;
gbxcu_ctx* g_ctx = nullptr;
int g_device = -1;

gbxcu_ctx* ctx() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_ctx) {
        int dev = g_device;
        if (dev < 0) {
            const char* env = std::getenv("GBX_DEVICE");
            dev = env ? std::atoi(env) : 0;
        }
        if (gbxcu_create(dev, &g_ctx) != GBXCU_OK) {
            g_ctx = nullptr;
            throw std::runtime_error(std::string("gbx: no usable B200 (no CPU fallback): ") +
                                     gbxcu_last_error());
        }
    }
    return g_ctx;
}

void check(int rc, int diverged_epoch = -1) {
    if (rc == GBXCU_OK) return;
    const std::string msg = gbxcu_last_error();
    switch (rc) {
        case GBXCU_EINVAL:
        case GBXCU_ENONFINITE: throw ValidationError(msg);
        case GBXCU_EDIVERGED: throw TrainingDivergedError(diverged_epoch, msg);
        case GBXCU_ETEMPERATURE: throw InvalidTemperatureError(msg);
        default: throw std::runtime_error("gbxcu: " + msg);
    }
}

constexpr double kProbClamp = 1e-7;

double clamp_prob(double p) { return std::min(std::max(p, kProbClamp), 1.0 - kProbClamp); }

void flatten_states(std::span<const ShaderState> s, std::vector<float>& out) {
    out.resize(s.size() * kFeatureCount);
    for (std::size_t r = 0; r < s.size(); ++r)
        std::memcpy(out.data() + r * kFeatureCount, s[r].features.data(), sizeof(float) * kFeatureCount);
}

void flatten_records(std::span<const std::pair<ShaderState, EmpiricalPolicy>> d,
                     std::vector<float>& feat, std::vector<double>& tgt) {
    feat.resize(d.size() * kFeatureCount);
    tgt.resize(d.size() * 2);
    for (std::size_t r = 0; r < d.size(); ++r) {
        std::memcpy(feat.data() + r * kFeatureCount, d[r].first.features.data(),
                    sizeof(float) * kFeatureCount);
        tgt[2 * r] = d[r].second.prob[0];
        tgt[2 * r + 1] = d[r].second.prob[1];
    }
}

}  // namespace

namespace detail {
gbxcu_ctx* device_context() { return ctx(); }
void check_status(int rc, int diverged_epoch) { check(rc, diverged_epoch); }
}  // namespace detail

void set_device(int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_ctx) {
        gbxcu_destroy(g_ctx);
        g_ctx = nullptr;
    }
    g_device = device;
}

// --------------------------------------------------------------- PolicyNet
PolicyNet PolicyNet::zeros() {
    PolicyNet net;
    for (int l = 0; l < kPolicyLayers; ++l) {
        net.weights[l].assign(static_cast<std::size_t>(kPolicyDims[l]) * kPolicyDims[l + 1], 0.0f);
        net.biases[l].assign(static_cast<std::size_t>(kPolicyDims[l + 1]), 0.0f);
    }
    return net;
}

std::vector<float> PolicyNet::flat() const {
    std::vector<float> p;
    p.reserve(kPolicyParamCount);
    for (int l = 0; l < kPolicyLayers; ++l) {
        p.insert(p.end(), weights[l].begin(), weights[l].end());
        p.insert(p.end(), biases[l].begin(), biases[l].end());
    }
    return p;
}

PolicyNet PolicyNet::from_flat(std::span<const float> p) {
    if (p.size() != kPolicyParamCount) throw ValidationError("flat parameter vector has wrong size");
    PolicyNet net = zeros();
    std::size_t o = 0;
    for (int l = 0; l < kPolicyLayers; ++l) {
        for (auto& w : net.weights[l]) w = p[o++];
        for (auto& b : net.biases[l]) b = p[o++];
    }
    return net;
}

PolicyNet PolicyNet::init(std::uint64_t seed) {
    std::vector<float> p(kPolicyParamCount);
    check(gbxcu_policy_init(ctx(), seed, p.data()));
    return from_flat(p);
}

std::array<double, 2> PolicyNet::forward(const ShaderState& s) const {
    for (float f : s.features)
        if (!std::isfinite(f)) throw ValidationError("non-finite feature in shader state");
    const auto p = flat();
    std::array<double, 2> probs{};
    check(gbxcu_forward(ctx(), p.data(), s.features.data(), 1, probs.data(), nullptr,
                        GBXCU_FWD_EXACT));
    return probs;
}

std::size_t PolicyNet::param_count() const {
    std::size_t n = 0;
    for (int l = 0; l < kPolicyLayers; ++l) n += weights[l].size() + biases[l].size();
    return n;
}

float PolicyNet::param(std::size_t i) const {
    for (int l = 0; l < kPolicyLayers; ++l) {
        if (i < weights[l].size()) return weights[l][i];
        i -= weights[l].size();
        if (i < biases[l].size()) return biases[l][i];
        i -= biases[l].size();
    }
    throw ValidationError("parameter index out of range");
}

void PolicyNet::set_param(std::size_t i, float v) {
    for (int l = 0; l < kPolicyLayers; ++l) {
        if (i < weights[l].size()) { weights[l][i] = v; return; }
        i -= weights[l].size();
        if (i < biases[l].size()) { biases[l][i] = v; return; }
        i -= biases[l].size();
    }
    throw ValidationError("parameter index out of range");
}

// -------------------------------------------------------------- loss / grad
double kl_loss(const std::array<double, 2>& predicted, const EmpiricalPolicy& target) {
    double loss = 0.0;
    for (int a = 0; a < 2; ++a) {
        const double p = clamp_prob(predicted[a]);
        loss += p * std::log(p / clamp_prob(target.prob[a]));
    }
    return loss;
}

double batch_kl_loss(const PolicyNet& net,
                     std::span<const std::pair<ShaderState, EmpiricalPolicy>> batch) {
    if (batch.empty()) return 0.0 / static_cast<double>(batch.size());  // reference: 0/0
    std::vector<float> feat;
    std::vector<double> tgt;
    flatten_records(batch, feat, tgt);
    const auto p = net.flat();
    double loss = 0.0;
    check(gbxcu_batch_kl_loss(ctx(), p.data(), feat.data(), tgt.data(), batch.size(), &loss));
    return loss;
}

std::vector<double> batch_kl_gradient(const PolicyNet& net,
                                      std::span<const std::pair<ShaderState, EmpiricalPolicy>> batch) {
    std::vector<double> g(net.param_count(), 0.0);
    if (batch.empty()) return g;
    std::vector<float> feat;
    std::vector<double> tgt;
    flatten_records(batch, feat, tgt);
    const auto p = net.flat();
    check(gbxcu_batch_kl_gradient(ctx(), p.data(), feat.data(), tgt.data(), batch.size(), g.data()));
    return g;
}

// ---------------------------------------------------------------------- fit
void TrainConfig::validate() const {
    if (!(learning_rate > 0.0)) throw ValidationError("learning rate must be positive");
    if (epochs < 1) throw ValidationError("epochs must be >= 1");
    if (batch_size < 1) throw ValidationError("batch size must be >= 1");
    if (!(rho_min > 0.0) || !(rho0 >= rho_min))
        throw ValidationError("temperature schedule requires rho0 >= rho_min > 0");
    if (!(rho_decay > 0.0 && rho_decay <= 1.0)) throw ValidationError("rho decay must be in (0, 1]");
}

double TrainConfig::rho_at(int iteration) const {
    return std::max(rho_min, rho0 * std::pow(rho_decay, iteration));
}

namespace {
FitResult fit_flat(PolicyNet& net, const std::vector<float>& feat, const std::vector<double>& tgt,
                   std::size_t n, const TrainConfig& cfg, int loss_mode, const OptimizerConfig& opt);
}  // namespace

FitResult fit(PolicyNet& net, const PolicyDataset& dataset, const TrainConfig& cfg) {
    return fit(net, dataset, cfg, OptimizerConfig{});
}

FitResult fit(PolicyNet& net, const PolicyDataset& dataset, const TrainConfig& cfg,
              const OptimizerConfig& opt) {
    cfg.validate();
    if (dataset.empty()) throw ValidationError("fit requires a non-empty dataset");
    std::vector<float> feat;
    std::vector<double> tgt;
    flatten_records(dataset, feat, tgt);
    return fit_flat(net, feat, tgt, dataset.size(), cfg, GBXCU_LOSS_KL, opt);
}

FitResult fit_td(PolicyNet& net, std::span<const ExperienceRecord> records, const TrainConfig& cfg,
                 const OptimizerConfig& opt) {
    cfg.validate();
    if (records.empty()) throw ValidationError("fit requires a non-empty dataset");
    std::vector<float> feat(records.size() * kFeatureCount);
    std::vector<double> tgt(records.size() * 2);
    for (std::size_t r = 0; r < records.size(); ++r) {
        for (int i = 0; i < kFeatureCount; ++i) feat[r * kFeatureCount + i] = records[r].state.features[i];
        tgt[2 * r] = records[r].action == Action::Wave64 ? 1.0 : 0.0;
        tgt[2 * r + 1] = records[r].reward;
    }
    return fit_flat(net, feat, tgt, records.size(), cfg, GBXCU_LOSS_TD, opt);
}

namespace {
FitResult fit_flat(PolicyNet& net, const std::vector<float>& feat, const std::vector<double>& tgt,
                   std::size_t n, const TrainConfig& cfg, int loss_mode, const OptimizerConfig& opt) {
    auto p = net.flat();
    gbxcu_train_cfg c{};  // zeros: the reference's KL loss + SGD, no CTA cap, no virtual ranks
    c.learning_rate = cfg.learning_rate;
    c.epochs = cfg.epochs;
    c.batch_size = cfg.batch_size;
    c.seed = cfg.seed;
    c.loss_mode = loss_mode;
    c.optimizer = opt.kind == OptimizerKind::Adam ? GBXCU_OPT_ADAM : GBXCU_OPT_SGD;
    c.adam_beta1 = opt.beta1;
    c.adam_beta2 = opt.beta2;
    c.adam_eps = opt.eps;
    const std::size_t dataset_size = n;
    FitResult res;
    res.epoch_loss.assign(cfg.epochs, 0.0);
    int diverged = -1;
    const int rc = gbxcu_fit(ctx(), p.data(), feat.data(), tgt.data(), dataset_size, &c,
                             res.epoch_loss.data(), &diverged);
    if (rc == GBXCU_OK || rc == GBXCU_EDIVERGED) net = PolicyNet::from_flat(p);
    if (rc == GBXCU_EDIVERGED)
        throw TrainingDivergedError(diverged, "training loss became non-finite at epoch " +
                                                  std::to_string(diverged));
    check(rc);
    return res;
}
}  // namespace

// ---------------------------------------------------------------- actions
Action select_greedy(const BehaviorPolicy& beh, const ShaderState& s) {
    const auto probs = beh.forward(s);
    return probs[1] >= probs[0] ? Action::Wave64 : Action::Wave32;
}

Action select_sample(const BehaviorPolicy& beh, const ShaderState& s, SplitMix64& rng) {
    const auto probs = beh.forward(s);
    return rng.next_unit() < probs[0] ? Action::Wave32 : Action::Wave64;
}

std::vector<std::array<double, 2>> forward_batch(const PolicyNet& net,
                                                 std::span<const ShaderState> states) {
    std::vector<std::array<double, 2>> out(states.size());
    if (states.empty()) return out;
    std::vector<float> feat;
    flatten_states(states, feat);
    const auto p = net.flat();
    check(gbxcu_forward(ctx(), p.data(), feat.data(), states.size(), out.data()->data(), nullptr,
                        GBXCU_FWD_EXACT));
    return out;
}

std::vector<Action> select_greedy_batch(const BehaviorPolicy& beh,
                                        std::span<const ShaderState> states) {
    std::vector<Action> out(states.size());
    if (states.empty()) return out;
    std::vector<float> feat;
    flatten_states(states, feat);
    std::vector<std::uint8_t> act(states.size());
    const auto p = beh.net.flat();
    check(gbxcu_forward(ctx(), p.data(), feat.data(), states.size(), nullptr, act.data(),
                        GBXCU_FWD_FAST));
    for (std::size_t i = 0; i < act.size(); ++i) out[i] = act[i] ? Action::Wave64 : Action::Wave32;
    return out;
}

std::vector<Action> select_sample_batch(const BehaviorPolicy& beh,
                                        std::span<const ShaderState> states, SplitMix64& rng) {
    std::vector<Action> out(states.size());
    if (states.empty()) return out;
    std::vector<float> feat;
    flatten_states(states, feat);
    std::vector<std::uint8_t> act(states.size());
    const auto p = beh.net.flat();
    check(gbxcu_sample_batch(ctx(), p.data(), feat.data(), states.size(), rng.state(), act.data()));
    rng.discard(states.size());
    for (std::size_t i = 0; i < act.size(); ++i) out[i] = act[i] ? Action::Wave64 : Action::Wave32;
    return out;
}

// ------------------------------------------------------------------- GBXP
namespace {

constexpr char kMagic[4] = {'G', 'B', 'X', 'P'};
constexpr std::uint16_t kFormat = 1;

template <typename T>
void put_le(std::vector<std::uint8_t>& o, T v) {
    for (std::size_t b = 0; b < sizeof(T); ++b) o.push_back(static_cast<std::uint8_t>(v >> (8 * b)));
}

struct ByteReader {
    std::span<const std::uint8_t> b;
    std::size_t pos = 0;
    std::span<const std::uint8_t> take(std::size_t n) {
        if (pos + n > b.size()) throw PolicyFormatError("truncated policy file");
        auto s = b.subspan(pos, n);
        pos += n;
        return s;
    }
    template <typename T>
    T le() {
        const auto s = take(sizeof(T));
        T v = 0;
        for (std::size_t i = 0; i < sizeof(T); ++i) v |= static_cast<T>(static_cast<T>(s[i]) << (8 * i));
        return v;
    }
};

}  // namespace

std::vector<std::uint8_t> serialize_policy(const BehaviorPolicy& beh) {
    std::vector<std::uint8_t> out(kMagic, kMagic + 4);
    put_le<std::uint16_t>(out, kFormat);
    out.push_back(static_cast<std::uint8_t>(kPolicyLayers));
    for (int l = 0; l < kPolicyLayers; ++l) {
        put_le<std::uint16_t>(out, static_cast<std::uint16_t>(kPolicyDims[l]));
        put_le<std::uint16_t>(out, static_cast<std::uint16_t>(kPolicyDims[l + 1]));
    }
    const std::size_t start = out.size();
    for (float v : beh.net.flat()) {
        std::uint32_t u;
        std::memcpy(&u, &v, 4);
        put_le<std::uint32_t>(out, u);
    }
    put_le<std::uint32_t>(out, static_cast<std::uint32_t>(
                                   crc32(0, out.data() + start, static_cast<uInt>(out.size() - start))));
    put_le<std::uint32_t>(out, beh.version_tag);
    put_le<std::uint64_t>(out, beh.source_checkin);
    return out;
}

BehaviorPolicy deserialize_policy(std::span<const std::uint8_t> bytes) {
    ByteReader r{bytes};
    if (std::memcmp(r.take(4).data(), kMagic, 4) != 0) throw PolicyFormatError("not a GBXP policy file");
    if (r.le<std::uint16_t>() != kFormat) throw PolicyFormatError("unsupported policy format version");
    const int layers = r.le<std::uint8_t>();
    if (layers != kPolicyLayers)
        throw PolicySchemaError("expected 3 layers, found " + std::to_string(layers));
    for (int l = 0; l < kPolicyLayers; ++l) {
        const int in = r.le<std::uint16_t>(), out = r.le<std::uint16_t>();
        if (in != kPolicyDims[l] || out != kPolicyDims[l + 1])
            throw PolicySchemaError("layer " + std::to_string(l) + " has shape " + std::to_string(in) +
                                    "x" + std::to_string(out));
    }
    const std::size_t start = r.pos;
    std::vector<float> p(kPolicyParamCount);
    for (auto& v : p) {
        const std::uint32_t u = r.le<std::uint32_t>();
        std::memcpy(&v, &u, 4);
    }
    const std::size_t end = r.pos;
    const std::uint32_t stored = r.le<std::uint32_t>();
    if (stored != static_cast<std::uint32_t>(crc32(0, bytes.data() + start, static_cast<uInt>(end - start))))
        throw PolicyFormatError("policy payload checksum mismatch");
    BehaviorPolicy beh;
    beh.net = PolicyNet::from_flat(p);
    beh.version_tag = r.le<std::uint32_t>();
    beh.source_checkin = r.le<std::uint64_t>();
    return beh;
}

void save_policy(const BehaviorPolicy& beh, const std::filesystem::path& path) {
    const auto bytes = serialize_policy(beh);
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) throw ValidationError("cannot open policy file for writing: " + path.string());
    os.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!os) throw ValidationError("failed writing policy file: " + path.string());
}

BehaviorPolicy load_policy(const std::filesystem::path& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw ValidationError("cannot open policy file: " + path.string());
    std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    return deserialize_policy(bytes);
}

// ------------------------------------------------------------ DeviceQTable
namespace {
void check_qt(int rc, std::size_t bad = 0) {
    if (rc == GBXCU_ECLOCK)
        throw ClockRegressionError("q_update check-in precedes entry timestamp (tuple " +
                                   std::to_string(bad) + ")");
    check(rc);
}
}  // namespace

DeviceQTable::DeviceQTable(QHyperparams hp) : hp_(hp) {
    hp_.validate();
    check(gbxcu_qtable_create(ctx(), hp.alpha, hp.omega, &h_));
}

DeviceQTable::~DeviceQTable() { gbxcu_qtable_free(h_); }

std::size_t DeviceQTable::state_count() const {
    std::size_t m = 0;
    check(gbxcu_qtable_size(h_, &m, nullptr));
    return m;
}

void DeviceQTable::update_batch(std::span<const ExperienceTuple> tuples) {
    const std::size_t n = tuples.size();
    std::vector<std::uint32_t> keys(n * kStateKeySize);
    std::vector<std::uint8_t> act(n);
    std::vector<double> rew(n);
    std::vector<std::uint64_t> now(n);
    for (std::size_t i = 0; i < n; ++i) {
        std::memcpy(keys.data() + i * kStateKeySize, tuples[i].key.values.data(),
                    sizeof(std::uint32_t) * kStateKeySize);
        act[i] = static_cast<std::uint8_t>(action_index(tuples[i].action));
        rew[i] = tuples[i].reward;
        now[i] = tuples[i].now;
    }
    std::size_t bad = 0;
    check_qt(gbxcu_qtable_update_batch(h_, keys.data(), act.data(), rew.data(), now.data(), n, &bad),
             bad);
}

std::vector<std::pair<ShaderState, EmpiricalPolicy>> DeviceQTable::snapshot_policy_dataset(
    double rho) const {
    std::size_t rows = 0;
    check(gbxcu_qtable_snapshot(h_, rho, nullptr, nullptr, 0, &rows));
    std::vector<float> f(rows * kFeatureCount);
    std::vector<double> t(rows * 2);
    check(gbxcu_qtable_snapshot(h_, rho, f.data(), t.data(), rows, &rows));
    std::vector<std::pair<ShaderState, EmpiricalPolicy>> out(rows);
    for (std::size_t r = 0; r < rows; ++r) {
        std::memcpy(out[r].first.features.data(), f.data() + r * kFeatureCount,
                    sizeof(float) * kFeatureCount);
        out[r].second.prob = {t[2 * r], t[2 * r + 1]};
    }
    return out;
}

QTable DeviceQTable::to_host() const {
    std::size_t m = 0;
    check(gbxcu_qtable_size(h_, &m, nullptr));
    std::vector<std::uint32_t> keys(m * kStateKeySize);
    std::vector<double> q(2 * m);
    std::vector<std::uint64_t> ts(2 * m), cnt(2 * m);
    std::vector<std::uint8_t> has(2 * m);
    check(gbxcu_qtable_export(h_, keys.data(), q.data(), ts.data(), cnt.data(), has.data()));
    QTable out(hp_);
    for (std::size_t r = 0; r < m; ++r) {
        StateKey k;
        std::memcpy(k.values.data(), keys.data() + r * kStateKeySize, sizeof(std::uint32_t) * kStateKeySize);
        auto& pair = out.entries_[k];
        for (int a = 0; a < 2; ++a)
            if (has[2 * r + a]) pair[a] = QEntry{q[2 * r + a], ts[2 * r + a], cnt[2 * r + a]};
    }
    return out;
}

DeviceQTable DeviceQTable::from_host(const QTable& table) {
    DeviceQTable d(table.hyperparams());
    d.assign(table);
    return d;
}

void DeviceQTable::assign(const QTable& table) {
    const std::size_t m = table.state_count();
    std::vector<std::uint32_t> keys(m * kStateKeySize);
    std::vector<double> q(2 * m, 0.0);
    std::vector<std::uint64_t> ts(2 * m, 0), cnt(2 * m, 0);
    std::vector<std::uint8_t> has(2 * m, 0);
    std::size_t r = 0;
    for (const auto& [key, pair] : table.entries()) {  // std::map: key order
        std::memcpy(keys.data() + r * kStateKeySize, key.values.data(), sizeof(std::uint32_t) * kStateKeySize);
        for (int a = 0; a < 2; ++a)
            if (pair[a]) {
                q[2 * r + a] = pair[a]->q;
                ts[2 * r + a] = pair[a]->last_update_t;
                cnt[2 * r + a] = pair[a]->update_count;
                has[2 * r + a] = 1;
            }
        ++r;
    }
    check(gbxcu_qtable_import(h_, keys.data(), q.data(), ts.data(), cnt.data(), has.data(), m));
}

std::vector<std::uint8_t> DeviceQTable::greedy_wave64_of_complete_states() const {
    std::size_t m = 0;
    check(gbxcu_qtable_size(h_, &m, nullptr));
    std::vector<double> q(2 * m);
    std::vector<std::uint8_t> has(2 * m), out;
    if (m) check(gbxcu_qtable_export(h_, nullptr, q.data(), nullptr, nullptr, has.data()));
    out.reserve(m);
    for (std::size_t r = 0; r < m; ++r)
        if (has[2 * r] && has[2 * r + 1]) out.push_back(q[2 * r + 1] >= q[2 * r] ? 1 : 0);
    return out;
}

// ------------------------------------------------- QTable's device copy
// (declared in gbx/qtable.hpp; the host-only members live in gbx_core.cpp)
QTable::QTable(const QTable& o) : hp_(o.hp_), entries_((o.sync_host(), o.entries_)) {}

QTable& QTable::operator=(const QTable& o) {
    if (this != &o) {
        o.sync_host();
        hp_ = o.hp_;
        entries_ = o.entries_;
        dev_.reset();  // never share a device copy between two tables
        dev_stale_ = true;
        host_stale_ = false;
    }
    return *this;
}

QTable::~QTable() = default;

std::size_t QTable::state_count() const {
    if (host_stale_) return dev_->state_count();
    return entries_.size();
}

void QTable::sync_host() const {
    if (!host_stale_) return;
    entries_ = std::move(dev_->to_host().entries_);
    host_stale_ = false;
    dev_stale_ = false;  // both copies hold the same table now
}

void QTable::sync_device() const {
    if (!dev_) dev_ = std::make_shared<DeviceQTable>(hp_);
    if (!dev_stale_) return;
    dev_->assign(*this);
    dev_stale_ = false;
}

void QTable::update_batch(const std::vector<ExperienceTuple>& tuples) {
    if (tuples.empty()) return;
    sync_device();
    host_stale_ = true;  // set first: on ClockRegressionError the device holds the prefix
    dev_->update_batch(tuples);
}

std::vector<std::pair<ShaderState, EmpiricalPolicy>> QTable::snapshot_policy_dataset(double rho) const {
    if (!(rho > 0.0)) throw InvalidTemperatureError("Boltzmann temperature must be > 0");
    if (state_count() == 0) return {};
    sync_device();
    return dev_->snapshot_policy_dataset(rho);
}

std::vector<std::uint8_t> QTable::greedy_wave64_of_complete_states() const {
    if (!host_stale_) {  // the map is current: no device round trip
        std::vector<std::uint8_t> out;
        for (const auto& kv : entries_)
            if (kv.second[0] && kv.second[1]) out.push_back(kv.second[1]->q >= kv.second[0]->q ? 1 : 0);
        return out;
    }
    return dev_->greedy_wave64_of_complete_states();
}

}  // namespace gbx
