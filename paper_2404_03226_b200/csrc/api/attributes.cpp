// attributes.cpp -- attribute API of the drop-in boundary (reference:
// proj/src/attributes.cpp).  Every function is one tbsim_attributes() call:
// the B200 kernels compute ability, efficiency, calibration, rank and depth.
#include <ostream>
#include <stdexcept>

#include "device.hpp"
#include "tbsim/attributes.hpp"

namespace tbsim {

std::vector<std::int64_t> compute_inspiring_ability(const TaskGraph& g) {
    return device::attributes(g, CostTable{}, TBSIM_ATTR_ABILITY, TBSIM_PRIO_ZERO, 0.0).ability;
}

std::vector<std::int64_t> compute_inspiring_ability_serial(const TaskGraph& g) {
    return compute_inspiring_ability(g);
}

std::vector<std::int64_t> compute_inspiring_efficiency(const TaskGraph& g, const CostTable& costs,
                                                       double unit_time_ms) {
    if (!(unit_time_ms >= 0.0)) throw std::invalid_argument("unit time must be non-negative");
    if (g.tasks.empty()) return {};
    return device::attributes(g, costs, TBSIM_ATTR_EFFICIENCY, TBSIM_PRIO_ZERO, unit_time_ms).efficiency;
}

std::vector<std::int64_t> compute_inspiring_efficiency_serial(const TaskGraph& g, const CostTable& costs,
                                                              double unit_time_ms) {
    return compute_inspiring_efficiency(g, costs, unit_time_ms);
}

CalibrationResult calibrate_unit_time(const TaskGraph& g, const CostTable& costs) {
    const auto r = device::attributes(g, costs, TBSIM_ATTR_CALIBRATE, TBSIM_PRIO_ZERO, 0.0);
    CalibrationResult c;
    c.unit_time_ms = r.unit_time_ms;
    c.w0_ms = r.w0_ms;
    c.best_score = r.best_score;
    c.w0_score = r.w0_score;
    c.evaluations = r.evaluations;
    return c;
}

std::vector<std::int64_t> upward_rank_priority(const TaskGraph& g, const CostTable& costs) {
    return device::attributes(g, costs, TBSIM_ATTR_RANK, TBSIM_PRIO_UPWARD_RANK, 0.0).static_priority;
}

std::vector<std::int64_t> depth_priority(const TaskGraph& g) {
    return device::attributes(g, CostTable{}, TBSIM_ATTR_DEPTH, TBSIM_PRIO_ZERO, 0.0).depth;
}

TaskAttributes compute_attributes(const TaskGraph& g, const CostTable& costs, PriorityKind priority) {
    const int32_t pk = priority == PriorityKind::UpwardRank ? TBSIM_PRIO_UPWARD_RANK
                       : priority == PriorityKind::Depth    ? TBSIM_PRIO_DEPTH
                                                            : TBSIM_PRIO_ZERO;
    auto r = device::attributes(g, costs, TBSIM_ATTR_ALL, pk, 0.0);
    TaskAttributes a;
    a.ability = std::move(r.ability);
    a.efficiency = std::move(r.efficiency);
    a.static_priority = std::move(r.static_priority);
    a.unit_time_ms = r.unit_time_ms;
    return a;
}

void write_attributes_csv(std::ostream& out, const TaskGraph& g, const TaskAttributes& attrs) {
    const std::vector<int> layer = topological_layers(g);
    out << "task_id,type,layer,ability,efficiency,static_priority\n";
    for (size_t i = 0; i < g.tasks.size(); ++i)
        out << g.tasks[i].id << ',' << g.tasks[i].type << ',' << layer[i] << ',' << attrs.ability[i] << ','
            << attrs.efficiency[i] << ',' << attrs.static_priority[i] << '\n';
}

}  // namespace tbsim
