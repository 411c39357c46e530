// bench.cpp -- sweep harness of the drop-in API (reference: proj/src/bench.cpp).
// Cells sharing a platform are scheduled as ONE device batch: attributes for
// every graph in one tbsim_attributes call, then one tbsim_simulate call per
// policy.  If a batch fails, its cells are re-run one by one so each failing
// cell becomes its own error row (the reference's per-cell semantics).
#include <algorithm>
#include <map>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <tuple>

#include "device.hpp"
#include "tbsim/bench.hpp"
#include "tbsim/engine.hpp"
#include "tbsim/policies.hpp"
#include "tbsim/text.hpp"

namespace tbsim {

namespace {

constexpr std::int64_t kCholeskyBytes = 960 * 960 * 4;
constexpr std::int64_t kLuBytes = 160 * 160 * 4;
constexpr std::int64_t kHeatBytes = 640 * 640 * 4;

TaskGraph app_graph(const BenchSpec& spec, std::int64_t size) {  // bench.cpp:23-40
    if (spec.app == "cholesky") return build_cholesky_dag(static_cast<int>(size), kCholeskyBytes);
    if (spec.app == "lu") return build_lu_dag(static_cast<int>(size), kLuBytes);
    if (spec.app == "heat") return build_stencil_dag(static_cast<int>(size), static_cast<int>(2 * size), kHeatBytes);
    if (spec.app == "autogen")
        return generate_layered_dag(static_cast<int>(size), spec.autogen_layers, spec.autogen_edge_prob, spec.seed);
    if (spec.app == "file") {
        if (size < 0 || size >= static_cast<std::int64_t>(spec.dag_files.size()))
            throw std::runtime_error("dag file index " + std::to_string(size) + " out of range");
        return load_dag_file(spec.dag_files[static_cast<size_t>(size)]);
    }
    throw std::runtime_error("unknown app '" + spec.app + "'");
}

std::string sanitize(std::string s) {
    for (char& c : s)
        if (c == ',' || c == '\n' || c == '\r') c = ';';
    return s;
}

RegulatorConfig overridden(RegulatorConfig cfg, const RegulatorOverride& ov) {
    if (ov.task_window) cfg.task_window = *ov.task_window;
    if (ov.s_inc) cfg.s_inc = *ov.s_inc;
    if (ov.k_inc) cfg.k_inc = *ov.k_inc;
    if (ov.s_dec) cfg.s_dec = *ov.s_dec;
    if (ov.c) cfg.c = *ov.c;
    if (ov.dec_step) cfg.dec_step = *ov.dec_step;
    if (ov.slope_samples) cfg.slope_samples = *ov.slope_samples;
    return cfg;
}

struct Cell {
    std::int64_t size;
    std::string platform_name;
    TaskGraph g;
    Platform platform;
    std::string error;       // setup/attribute failure: every policy row errors
    std::vector<BenchRow> rows;
};

BenchRow stub(const BenchSpec& spec, const Cell& c, const std::string& policy) {
    BenchRow r;
    r.app = spec.app;
    r.size = c.size;
    r.platform = c.platform_name;
    r.policy = policy;
    return r;
}

// One cell through the single-graph API (fallback and error attribution).
void run_cell(const BenchSpec& spec, Cell& c, const std::vector<std::string>& policies) {
    TaskAttributes attrs;
    try {
        attrs = compute_attributes(c.g, c.platform.costs, spec.priority);
    } catch (const std::exception& e) {
        for (const auto& p : policies) {
            BenchRow r = stub(spec, c, p);
            r.error = e.what();
            c.rows.push_back(r);
        }
        return;
    }
    const RegulatorConfig reg = overridden(default_regulator_config(c.platform, c.g), spec.regulator);
    SimOptions opts;
    opts.record_trace = false;
    for (const auto& name : policies) {
        BenchRow r = stub(spec, c, name);
        try {
            auto pol = make_policy(name, attrs, reg);
            r.makespan_ms = simulate(c.g, c.platform, *pol, opts).makespan_ms;
            r.ok = true;
        } catch (const std::exception& e) {
            r.error = e.what();
        }
        c.rows.push_back(r);
    }
}

// All cells of one platform as a device batch; false when any call failed.
bool run_group(const BenchSpec& spec, std::vector<Cell*>& cells, const std::vector<std::string>& policies) {
    try {
        device::Csr csr;
        for (Cell* c : cells) csr.add(c->g);
        csr.require_known_handles();
        device::Uploaded up(csr);
        const Platform& pl = cells.front()->platform;
        const int64_t T = csr.task_base.back(), G = static_cast<int64_t>(cells.size());
        device::PlatformArrays pa = device::platform_arrays(pl, csr.type_names);
        std::vector<int64_t> ab(T), ef(T), pr(T);
        std::vector<double> unit(G);
        tbsim_attr_out ao{};
        ao.ability = ab.data();
        ao.efficiency = ef.data();
        ao.static_priority = pr.data();
        ao.unit_time_ms = unit.data();
        const int32_t pk = spec.priority == PriorityKind::UpwardRank ? TBSIM_PRIO_UPWARD_RANK
                           : spec.priority == PriorityKind::Depth    ? TBSIM_PRIO_DEPTH
                                                                     : TBSIM_PRIO_ZERO;
        tbsim_costs cv = pa.costs.view();
        device::check(tbsim_attributes(device::context(), up.get(), &cv, TBSIM_ATTR_ALL, pk, &ao));
        std::vector<tbsim_regulator_cfg> reg(G);
        for (int64_t g = 0; g < G; ++g) {
            const RegulatorConfig r = overridden(default_regulator_config(pl, cells[g]->g), spec.regulator);
            reg[g] = {r.task_window, r.s_inc, r.k_inc, r.s_dec, r.c, r.dec_step, r.slope_samples, 0};
        }
        tbsim_attr_in ai{ab.data(), ef.data(), pr.data(), 0};
        std::vector<int32_t> worker(T);
        std::vector<double> st(T), en(T), ms(G);
        std::vector<int64_t> done(G);
        std::map<std::string, std::vector<double>> makespans;
        for (const auto& name : policies) {
            const auto names = policy_names();
            const int pid = static_cast<int>(std::find(names.begin(), names.end(), name) - names.begin());
            if (pid >= static_cast<int>(names.size())) return false;  // unknown policy: per-cell error rows
            tbsim_sim_out o{};
            o.worker = worker.data();
            o.start_ms = st.data();
            o.end_ms = en.data();
            o.makespan_ms = ms.data();
            o.completed = done.data();
            device::check(tbsim_simulate(device::context(), up.get(), &pa.desc, 1, nullptr, pid, reg.data(), &ai, &o));
            makespans[name] = ms;
        }
        for (int64_t g = 0; g < G; ++g)
            for (const auto& name : policies) {
                BenchRow r = stub(spec, *cells[g], name);
                r.makespan_ms = makespans[name][g];
                r.ok = true;
                cells[g]->rows.push_back(r);
            }
        return true;
    } catch (const std::exception&) {
        for (Cell* c : cells) c->rows.clear();
        return false;
    }
}

}  // namespace

BenchReport run_bench(const BenchSpec& spec) {  // bench.cpp:66-147
    std::vector<std::string> policies = spec.policies;
    if (policies.empty()) policies = policy_names();
    if (std::find(policies.begin(), policies.end(), spec.baseline) == policies.end()) policies.push_back(spec.baseline);
    std::vector<std::int64_t> sizes = spec.sizes;
    if (spec.app == "file" && sizes.empty())
        for (size_t i = 0; i < spec.dag_files.size(); ++i) sizes.push_back(static_cast<std::int64_t>(i));
    std::vector<std::unique_ptr<Cell>> cells;
    for (std::int64_t size : sizes)
        for (const auto& pname : spec.platforms) {
            auto c = std::make_unique<Cell>();
            c->size = size;
            c->platform_name = pname;
            try {
                c->g = app_graph(spec, size);
                c->platform = resolve_platform(pname);
            } catch (const std::exception& e) {
                c->error = e.what();
            }
            cells.push_back(std::move(c));
        }
    std::map<std::string, std::vector<Cell*>> groups;
    for (auto& c : cells) {
        if (!c->error.empty()) {
            for (const auto& p : policies) {
                BenchRow r = stub(spec, *c, p);
                r.error = c->error;
                c->rows.push_back(r);
            }
            continue;
        }
        groups[c->platform_name].push_back(c.get());
    }
    for (auto& [name, members] : groups)
        if (!run_group(spec, members, policies))
            for (Cell* c : members) run_cell(spec, *c, policies);
    BenchReport report;
    for (auto& c : cells) {
        double base = 0.0;
        for (const auto& r : c->rows)
            if (r.policy == spec.baseline && r.ok) base = r.makespan_ms;
        for (auto& r : c->rows) {
            if (r.ok && base > 0.0) r.speedup = r.policy == spec.baseline ? 1.0 : base / r.makespan_ms;
            report.rows.push_back(r);
        }
    }
    std::sort(report.rows.begin(), report.rows.end(), [](const BenchRow& a, const BenchRow& b) {
        return std::tie(a.app, a.size, a.platform, a.policy) < std::tie(b.app, b.size, b.platform, b.policy);
    });
    return report;
}

void write_bench_csv(std::ostream& out, const BenchReport& report) {
    out << "app,size,platform,policy,makespan_ms,speedup_vs_baseline,status\n";
    for (const auto& r : report.rows) {
        out << r.app << ',' << r.size << ',' << r.platform << ',' << r.policy << ',';
        if (r.ok) out << fmt_ms(r.makespan_ms) << ',' << fmt_ratio(r.speedup) << ",ok\n";
        else out << ",,error: " << sanitize(r.error) << '\n';
    }
}

}  // namespace tbsim
