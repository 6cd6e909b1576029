// gbx/device_qtable.hpp — the Q-table on the B200 (batched form added to the
// reference API, like forward_batch): QTable::update over a whole batch of
// tuples (proj/src/qtable.cpp:76-92) and snapshot_policy_dataset (:143-155)
// run as device kernels (csrc/k_qtable.cu); the records can stay on the
// device for fit. Conversions to/from the host QTable keep save/load
// (QTable::save / QTable::load) as the persistence path.
#pragma once

#include <cstdint>
#include <span>
#include <utility>
#include <vector>

#include "gbx/core.hpp"
#include "gbx/qtable.hpp"

struct gbxcu_qtable;

namespace gbx {

class DeviceQTable {
public:
    explicit DeviceQTable(QHyperparams hp = {});
    ~DeviceQTable();
    DeviceQTable(const DeviceQTable&) = delete;
    DeviceQTable& operator=(const DeviceQTable&) = delete;
    DeviceQTable(DeviceQTable&& o) noexcept : hp_(o.hp_), h_(o.h_) { o.h_ = nullptr; }
    DeviceQTable& operator=(DeviceQTable&& o) noexcept {
        std::swap(hp_, o.hp_);
        std::swap(h_, o.h_);
        return *this;
    }

    const QHyperparams& hyperparams() const { return hp_; }
    std::size_t state_count() const;

    // QTable::update for every tuple, in order. Throws ClockRegressionError at
    // the first tuple whose check-in precedes its entry's timestamp; the table
    // then holds exactly the updates before it (as the reference's does).
    void update_batch(std::span<const ExperienceTuple> tuples);

    // snapshot_policy_dataset(rho), key order (InvalidTemperatureError if rho <= 0).
    std::vector<std::pair<ShaderState, EmpiricalPolicy>> snapshot_policy_dataset(double rho) const;

    QTable to_host() const;
    static DeviceQTable from_host(const QTable& table);
    // replace this table's contents with the host table's map (same device handle)
    void assign(const QTable& table);
    // per state with both actions (key order): q64 >= q32
    std::vector<std::uint8_t> greedy_wave64_of_complete_states() const;

private:
    QHyperparams hp_;
    gbxcu_qtable* h_ = nullptr;
};

}  // namespace gbx
