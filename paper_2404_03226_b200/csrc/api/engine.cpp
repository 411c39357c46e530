// engine.cpp -- simulate() of the drop-in API (reference: proj/src/engine.cpp)
// runs the built-in policies on the B200 through tbsim_simulate (one warp per
// DAG); trace queries and CSV writers are host-side.
#include <algorithm>
#include <cmath>
#include <ostream>
#include <stdexcept>

#include "device.hpp"
#include "policy_impl.hpp"
#include "tbsim/engine.hpp"
#include "tbsim/text.hpp"

namespace tbsim {

namespace {

tbsim_regulator_state to_c(const RegulatorState& s) {
    tbsim_regulator_state c{};
    c.mode = static_cast<int32_t>(s.mode);
    c.phase = static_cast<int32_t>(s.state);
    c.peak = s.peak;
    c.prev_nready = s.prev_nready;
    c.last_trigger_nready = s.last_trigger_nready;
    c.s_dec_count = s.s_dec_count;
    c.cur_k = s.cur_k;
    if (s.samples.size() > TBSIM_MAX_SLOPE_SAMPLES)
        throw std::invalid_argument("regulator state holds more than 64 samples");
    c.n_samples = static_cast<int32_t>(s.samples.size());
    int i = 0;
    for (const auto& [t, v] : s.samples) {
        c.sample_time[i] = t;
        c.sample_nready[i] = v;
        ++i;
    }
    return c;
}

void from_c(const tbsim_regulator_state& c, RegulatorState& s) {
    s.mode = static_cast<PopMode>(c.mode);
    s.state = static_cast<RegulatorPhase>(c.phase);
    s.peak = c.peak;
    s.prev_nready = c.prev_nready;
    s.last_trigger_nready = c.last_trigger_nready;
    s.s_dec_count = c.s_dec_count;
    s.cur_k = c.cur_k;
    s.samples.clear();
    for (int i = 0; i < c.n_samples; ++i) s.samples.emplace_back(c.sample_time[i], c.sample_nready[i]);
}

std::vector<int64_t> attr_or_zero(const TaskAttributes* a, const std::vector<int64_t> TaskAttributes::*field,
                                  size_t n) {
    if (a && (a->*field).size() >= n) return std::vector<int64_t>((a->*field).begin(), (a->*field).begin() + n);
    return std::vector<int64_t>(n, 0);
}

}  // namespace

SimTrace simulate(const TaskGraph& g, const Platform& platform, Policy& policy, const SimOptions& opts) {
    auto* bp = dynamic_cast<detail::BuiltinPolicy*>(&policy);
    if (!bp)
        throw std::runtime_error("simulate: policy \"" + policy.name() +
                                 "\" is not a built-in; the B200 engine runs fifo, dm, dmda, dmdap and inspirit");
    device::Csr csr;
    csr.add(g);
    csr.require_known_handles();
    device::Uploaded up(csr);
    const size_t n = g.tasks.size();
    device::PlatformArrays pa = device::platform_arrays(platform, csr.type_names);
    const RegulatorConfig& rc = bp->config();
    tbsim_regulator_cfg cfg{};
    cfg.task_window = rc.task_window;
    cfg.s_inc = rc.s_inc;
    cfg.k_inc = rc.k_inc;
    cfg.s_dec = rc.s_dec;
    cfg.c = rc.c;
    cfg.dec_step = rc.dec_step;
    cfg.slope_samples = rc.slope_samples;
    const TaskAttributes* a = bp->attrs();
    std::vector<int64_t> ab = attr_or_zero(a, &TaskAttributes::ability, n);
    std::vector<int64_t> ef = attr_or_zero(a, &TaskAttributes::efficiency, n);
    std::vector<int64_t> pr = attr_or_zero(a, &TaskAttributes::static_priority, n);
    tbsim_attr_in ai{ab.data(), ef.data(), pr.data(), 0};
    std::vector<int32_t> worker(n);
    std::vector<double> start(n), end(n);
    double makespan = 0.0;
    int64_t completed = 0;
    int64_t pops[3] = {0, 0, 0};
    tbsim_regulator_state st = to_c(bp->state());
    std::vector<double> push_t(n), pop_t(n), samp_t(2 * n);
    std::vector<int32_t> push_k(n), pop_k(n), pop_w(n);
    std::vector<int64_t> samp_n(2 * n);
    tbsim_sim_out o{};
    o.worker = worker.data();
    o.start_ms = start.data();
    o.end_ms = end.data();
    o.makespan_ms = &makespan;
    o.completed = &completed;
    o.pop_mode_counts = pops;
    o.reg_state = &st;
    if (opts.record_trace) {
        o.push_time = push_t.data();
        o.push_task = push_k.data();
        o.pop_time = pop_t.data();
        o.pop_task = pop_k.data();
        o.pop_worker = pop_w.data();
        o.sample_time = samp_t.data();
        o.sample_nready = samp_n.data();
    }
    device::check(tbsim_simulate(device::context(), up.get(), &pa.desc, 1, nullptr, bp->id(), &cfg, &ai, &o));
    SimTrace tr;
    tr.makespan_ms = makespan;
    tr.per_task.resize(n);
    for (size_t i = 0; i < n; ++i) tr.per_task[i] = {worker[i], start[i], end[i]};
    if (opts.record_trace) {
        for (size_t k = 0; k < n; ++k) tr.pushes.push_back({push_t[k], g.tasks[push_k[k]].id});
        for (size_t k = 0; k < n; ++k) tr.pops.push_back({pop_t[k], g.tasks[pop_k[k]].id, pop_w[k]});
        for (size_t k = 0; k < 2 * n; ++k) tr.nready_samples.emplace_back(samp_t[k], samp_n[k]);
    }
    if (bp->id() == TBSIM_POLICY_INSPIRIT) {
        from_c(st, bp->state());
        for (int m = 0; m < 3; ++m) bp->counts()[m] += pops[m];
    }
    return tr;
}

std::int64_t nready_at(const SimTrace& trace, double t_ms) {  // engine.cpp:258-267
    if (t_ms < 0.0 || t_ms > trace.makespan_ms) throw std::out_of_range("time outside [0, makespan]");
    std::int64_t value = 0;
    for (const auto& [time, v] : trace.nready_samples) {
        if (time > t_ms) break;
        value = v;
    }
    return value;
}

std::vector<WindowRow> window_histogram(const SimTrace& trace, double window_ms) {  // engine.cpp:269-286
    if (!(window_ms > 0.0)) throw std::invalid_argument("window must be positive");
    if (trace.pushes.empty() && trace.pops.empty()) return {};
    double last = 0.0;
    for (const auto& p : trace.pushes) last = std::max(last, p.time_ms);
    for (const auto& p : trace.pops) last = std::max(last, p.time_ms);
    auto win = [window_ms](double t) { return static_cast<size_t>(std::floor(t / window_ms)); };
    std::vector<WindowRow> rows(win(last) + 1);
    for (size_t i = 0; i < rows.size(); ++i) rows[i] = {static_cast<double>(i) * window_ms, 0, 0};
    for (const auto& p : trace.pushes) rows[win(p.time_ms)].pushes += 1;
    for (const auto& p : trace.pops) rows[win(p.time_ms)].pops += 1;
    return rows;
}

void write_nready_csv(std::ostream& out, const SimTrace& trace) {
    out << "time_ms,nready\n";
    for (const auto& [t, v] : trace.nready_samples) out << fmt_ms(t) << ',' << v << '\n';
}

void write_push_pop_csv(std::ostream& out, const SimTrace& trace, double window_ms) {
    out << "window_start_ms,pushes,pops\n";
    for (const auto& r : window_histogram(trace, window_ms))
        out << fmt_ms(r.window_start_ms) << ',' << r.pushes << ',' << r.pops << '\n';
}

void write_gantt_csv(std::ostream& out, const TaskGraph& g, const SimTrace& trace) {
    out << "task_id,type,worker,start_ms,end_ms\n";
    for (size_t i = 0; i < g.tasks.size(); ++i) {
        const auto& t = trace.per_task[i];
        out << g.tasks[i].id << ',' << g.tasks[i].type << ',' << t.worker << ',' << fmt_ms(t.start_ms) << ','
            << fmt_ms(t.end_ms) << '\n';
    }
}

}  // namespace tbsim
