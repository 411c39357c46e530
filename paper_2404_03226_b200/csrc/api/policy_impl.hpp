// policy_impl.hpp -- the built-in policy objects, shared by policies.cpp
// (host rules, make_policy) and engine.cpp (which runs them on the B200).
#pragma once

#include <array>
#include <string>

#include "tbsim/policies.hpp"

namespace tbsim::detail {

class BuiltinPolicy final : public Policy {
public:
    BuiltinPolicy(int id, std::string name, const TaskAttributes* attrs, const RegulatorConfig& cfg)
        : id_(id), name_(std::move(name)), attrs_(attrs), cfg_(cfg) {}
    const std::string& name() const override { return name_; }
    int select_worker(std::size_t task_pos, const EngineView& view) override;
    std::size_t select_entry(int worker, const std::vector<QueueEntry>& queue, const EngineView& view) override;
    void on_queue_event(double now_ms, std::int64_t nready) override;

    int id() const { return id_; }  // TBSIM_POLICY_* of include/tbsim_b200.h
    const TaskAttributes* attrs() const { return attrs_; }
    const RegulatorConfig& config() const { return cfg_; }
    RegulatorState& state() { return state_; }
    const RegulatorState& state() const { return state_; }
    std::array<std::int64_t, 3>& counts() { return counts_; }
    const std::array<std::int64_t, 3>& counts() const { return counts_; }

private:
    int id_;
    std::string name_;
    const TaskAttributes* attrs_;  // dmdap / inspirit keep a reference, like the reference; null otherwise
    RegulatorConfig cfg_;
    RegulatorState state_;
    std::array<std::int64_t, 3> counts_{};
};

}  // namespace tbsim::detail
