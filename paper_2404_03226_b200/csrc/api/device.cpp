// device.cpp -- C++ API -> C-ABI bridge (see device.hpp).
#include "device.hpp"

#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <unordered_map>

namespace tbsim::device {

void check(tbsim_status st) {
    if (st == TBSIM_OK) return;
    const std::string msg = tbsim_last_error();
    switch (st) {
        case TBSIM_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case TBSIM_E_LOGIC: throw std::logic_error(msg);
        case TBSIM_E_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

namespace {

struct CtxHolder {
    tbsim_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) tbsim_ctx_destroy(ctx);
    }
};

}  // namespace

tbsim_ctx* context() {
    thread_local CtxHolder holder;
    if (!holder.ctx) {
        const char* env = std::getenv("TBSIM_DEVICE");
        check(tbsim_ctx_create(env ? std::atoi(env) : 0, &holder.ctx));
    }
    return holder.ctx;
}

void Csr::add(const TaskGraph& g) {
    std::unordered_map<TaskId, int32_t> pos;
    std::unordered_map<HandleId, int32_t> hpos;
    pos.reserve(g.tasks.size());
    for (size_t i = 0; i < g.tasks.size(); ++i)
        if (!pos.emplace(g.tasks[i].id, static_cast<int32_t>(i)).second)
            throw std::invalid_argument("duplicate task id " + std::to_string(g.tasks[i].id));
    for (size_t i = 0; i < g.handles.size(); ++i)
        if (!hpos.emplace(g.handles[i].id, static_cast<int32_t>(i)).second)
            throw std::invalid_argument("duplicate handle id " + std::to_string(g.handles[i].id));
    std::unordered_map<std::string, int32_t> tid;
    for (size_t i = 0; i < type_names.size(); ++i) tid.emplace(type_names[i], static_cast<int32_t>(i));
    const int64_t e0 = dep.size(), i0 = in.size(), o0 = out.size();
    dep_off.push_back(0);
    in_off.push_back(0);
    out_off.push_back(0);
    for (const auto& t : g.tasks) {
        for (TaskId d : t.deps) {
            const auto it = pos.find(d);
            if (it == pos.end())
                throw std::invalid_argument("task " + std::to_string(t.id) + " depends on unknown task " +
                                            std::to_string(d));
            dep.push_back(it->second);
        }
        for (HandleId h : t.inputs) {
            const auto it = hpos.find(h);
            if (it == hpos.end()) unknown_handle = true;
            else in.push_back(it->second);
        }
        for (HandleId h : t.outputs) {
            const auto it = hpos.find(h);
            if (it == hpos.end()) unknown_handle = true;
            else out.push_back(it->second);
        }
        dep_off.push_back(static_cast<int32_t>(dep.size() - e0));
        in_off.push_back(static_cast<int32_t>(in.size() - i0));
        out_off.push_back(static_cast<int32_t>(out.size() - o0));
        auto it = tid.find(t.type);
        if (it == tid.end()) {
            it = tid.emplace(t.type, static_cast<int32_t>(type_names.size())).first;
            type_names.push_back(t.type);
        }
        type.push_back(it->second);
        task_id.push_back(t.id);
    }
    for (const auto& h : g.handles) handle_bytes.push_back(h.bytes);
    task_base.push_back(task_base.back() + static_cast<int64_t>(g.tasks.size()));
    edge_base.push_back(static_cast<int64_t>(dep.size()));
    handle_base.push_back(static_cast<int64_t>(handle_bytes.size()));
    in_base.push_back(static_cast<int64_t>(in.size()));
    out_base.push_back(static_cast<int64_t>(out.size()));
}

void Csr::require_known_handles() const {
    // the exception (type and text) the reference's engine gets from
    // handle_pos.at() -- raised by the same standard-library call
    if (unknown_handle) (void)std::unordered_map<HandleId, size_t>{}.at(HandleId{});
}

const tbsim_batch_desc& Csr::finish() {
    name_ptrs.clear();
    for (const auto& s : type_names) name_ptrs.push_back(s.c_str());
    desc.n_graphs = static_cast<int64_t>(task_base.size()) - 1;
    desc.task_base = task_base.data();
    desc.edge_base = edge_base.data();
    desc.handle_base = handle_base.data();
    desc.in_base = in_base.data();
    desc.out_base = out_base.data();
    desc.dep_off = dep_off.data();
    desc.dep = dep.data();
    desc.in_off = in_off.data();
    desc.in = in.data();
    desc.out_off = out_off.data();
    desc.out = out.data();
    desc.type = type.data();
    desc.handle_bytes = handle_bytes.data();
    desc.task_id = task_id.data();
    desc.n_type_names = static_cast<int32_t>(type_names.size());
    desc.type_names = name_ptrs.data();
    return desc;
}

Uploaded::Uploaded(Csr& csr) { check(tbsim_batch_upload(context(), &csr.finish(), &b_)); }
Uploaded::~Uploaded() {
    if (b_) tbsim_batch_free(context(), b_);
}

tbsim_costs CostArrays::view() const {
    tbsim_costs c;
    c.n_types = static_cast<int32_t>(cpu.size());
    c.cpu_ms = cpu.data();
    c.gpu_ms = gpu.data();
    return c;
}

CostArrays cost_arrays(const CostTable& t, const std::vector<std::string>& names) {
    CostArrays c;
    c.cpu.assign(names.size(), 0.0);
    c.gpu.assign(names.size(), 0.0);
    for (size_t i = 0; i < names.size(); ++i) {
        if (const auto v = t.find(names[i], DeviceKind::Cpu)) c.cpu[i] = *v;
        if (const auto v = t.find(names[i], DeviceKind::Gpu)) c.gpu[i] = *v;
    }
    return c;
}

PlatformArrays platform_arrays(const Platform& p, const std::vector<std::string>& names) {
    PlatformArrays a;
    for (const Worker& w : p.workers) {
        a.kind.push_back(w.kind == DeviceKind::Gpu ? 1 : 0);
        a.node.push_back(w.memory_node);
    }
    a.bw.assign(static_cast<size_t>(p.num_nodes) * p.num_nodes, 0.0);
    for (int x = 0; x < p.num_nodes; ++x)
        for (int y = 0; y < p.num_nodes && x < static_cast<int>(p.bandwidth.size()); ++y)
            if (y < static_cast<int>(p.bandwidth[x].size())) a.bw[x * p.num_nodes + y] = p.bandwidth[x][y];
    a.costs = cost_arrays(p.costs, names);
    a.desc.n_workers = static_cast<int32_t>(p.workers.size());
    a.desc.kind = a.kind.data();
    a.desc.memory_node = a.node.data();
    a.desc.n_nodes = p.num_nodes;
    a.desc.latency_ms = p.latency_ms;
    a.desc.bandwidth = a.bw.data();
    a.desc.costs = a.costs.view();
    return a;
}

std::vector<int> layers(const TaskGraph& g) {
    Csr csr;
    csr.add(g);
    Uploaded up(csr);
    std::vector<int32_t> layer(g.tasks.size());
    CostArrays none = cost_arrays(CostTable{}, csr.type_names);
    tbsim_costs c = none.view();
    tbsim_attr_out o{};
    o.layer = layer.data();
    check(tbsim_attributes(context(), up.get(), &c, TBSIM_ATTR_LAYERS, TBSIM_PRIO_ZERO, &o));
    return std::vector<int>(layer.begin(), layer.end());
}

AttrResult attributes(const TaskGraph& g, const CostTable& costs, int32_t request, int32_t prio_kind,
                      double unit_time_ms) {
    Csr csr;
    csr.add(g);
    Uploaded up(csr);
    const size_t n = g.tasks.size();
    AttrResult r;
    r.ability.assign(n, 0);
    r.efficiency.assign(n, 0);
    r.static_priority.assign(n, 0);
    r.depth.assign(n, 0);
    r.unit_time_ms = unit_time_ms;
    CostArrays ca = cost_arrays(costs, csr.type_names);
    tbsim_costs c = ca.view();
    tbsim_attr_out o{};
    o.ability = r.ability.data();
    o.efficiency = r.efficiency.data();
    o.static_priority = r.static_priority.data();
    o.depth = r.depth.data();
    o.unit_time_ms = &r.unit_time_ms;
    o.w0_ms = &r.w0_ms;
    o.best_score = &r.best_score;
    o.w0_score = &r.w0_score;
    o.evaluations = &r.evaluations;
    check(tbsim_attributes(context(), up.get(), &c, request, prio_kind, &o));
    return r;
}

}  // namespace tbsim::device
