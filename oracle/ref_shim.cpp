// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (oracle/, see oracle/README.md).
//
// A thin extern "C" adapter over the *unmodified* reference library compiled
// from /root/reference/proj/src (recipe: oracle/Makefile -> oracle/_ref/).
// It lets tests/, bench.py's cpu_baseline leg and `bench.py --impl
// reference` drive the reference's own public API (include/tbsim/*.hpp) with
// the same CSR batch layout the B200 product consumes (include/tbsim_b200.h).
// Nothing here is linked into the product.

#include <omp.h>

#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracles.hpp"            // reference tests/oracles.hpp (random_dag, brute-force oracles)
#include "tbsim/attributes.hpp"
#include "tbsim/engine.hpp"
#include "tbsim/platform.hpp"
#include "tbsim/policies.hpp"
#include "tbsim/taskgraph.hpp"
#include "tbsim_b200.h"

using namespace tbsim;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::invalid_argument*>(&e)) return TBSIM_E_INVALID_ARGUMENT;
    if (dynamic_cast<const std::out_of_range*>(&e)) return TBSIM_E_OUT_OF_RANGE;
    if (dynamic_cast<const std::logic_error*>(&e)) return TBSIM_E_LOGIC;
    return TBSIM_E_RUNTIME;
}

CostTable make_costs(const tbsim_costs& c, const char* const* names) {
    CostTable t;
    for (int i = 0; i < c.n_types; ++i) {
        if (c.cpu_ms && c.cpu_ms[i] > 0.0) t.set(names[i], DeviceKind::Cpu, c.cpu_ms[i]);
        if (c.gpu_ms && c.gpu_ms[i] > 0.0) t.set(names[i], DeviceKind::Gpu, c.gpu_ms[i]);
    }
    return t;
}

Platform make_platform(const tbsim_platform_desc& p, const char* const* names) {
    Platform out;
    out.name = "shim";
    for (int w = 0; w < p.n_workers; ++w)
        out.workers.push_back({w, p.kind[w] ? DeviceKind::Gpu : DeviceKind::Cpu,
                               p.memory_node[w]});
    out.num_nodes = p.n_nodes;
    out.latency_ms = p.latency_ms;
    out.bandwidth.assign(p.n_nodes, std::vector<double>(p.n_nodes, 0.0));
    for (int a = 0; a < p.n_nodes; ++a)
        for (int b = 0; b < p.n_nodes; ++b) out.bandwidth[a][b] = p.bandwidth[a * p.n_nodes + b];
    out.costs = make_costs(p.costs, names);
    return out;
}

TaskGraph graph_of(const tbsim_batch_desc& d, int64_t g, const char* const* names) {
    TaskGraph out;
    out.name = "g" + std::to_string(g);
    const int64_t t0 = d.task_base[g], n = d.task_base[g + 1] - t0;
    const int64_t h0 = d.handle_base[g], nh = d.handle_base[g + 1] - h0;
    const int32_t* doff = d.dep_off + t0 + g;
    const int32_t* ioff = d.in_off + t0 + g;
    const int32_t* ooff = d.out_off + t0 + g;
    // External ids: task_id when given, else the position.  Handle ids are
    // positions (the batch carries handle positions only).
    auto tid = [&](int64_t local) { return d.task_id ? d.task_id[t0 + local] : local; };
    for (int64_t h = 0; h < nh; ++h) out.handles.push_back({h, d.handle_bytes[h0 + h]});
    out.tasks.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        TaskNode& t = out.tasks[i];
        t.id = tid(i);
        t.type = names[d.type[t0 + i]];
        for (int32_t k = doff[i]; k < doff[i + 1]; ++k) t.deps.push_back(tid(d.dep[d.edge_base[g] + k]));
        for (int32_t k = ioff[i]; k < ioff[i + 1]; ++k) t.inputs.push_back(d.in[d.in_base[g] + k]);
        for (int32_t k = ooff[i]; k < ooff[i + 1]; ++k) t.outputs.push_back(d.out[d.out_base[g] + k]);
    }
    return out;
}

// Exported graph (for generator parity): flat CSR of one TaskGraph.
struct Exported {
    std::vector<int32_t> dep_off{0}, dep, in_off{0}, in, out_off{0}, out, type;
    std::vector<int64_t> handle_bytes, task_id;
    std::vector<std::string> type_names;
};

Exported export_graph(const TaskGraph& g) {
    Exported e;
    GraphIndex idx = build_index(g);
    std::vector<std::string> names;
    for (const auto& t : g.tasks) {
        int tid = -1;
        for (size_t i = 0; i < e.type_names.size(); ++i)
            if (e.type_names[i] == t.type) tid = static_cast<int>(i);
        if (tid < 0) {
            tid = static_cast<int>(e.type_names.size());
            e.type_names.push_back(t.type);
        }
        e.type.push_back(tid);
        e.task_id.push_back(t.id);
        for (TaskId d : t.deps) e.dep.push_back(static_cast<int32_t>(idx.task_pos.at(d)));
        for (HandleId h : t.inputs) e.in.push_back(static_cast<int32_t>(idx.handle_pos.at(h)));
        for (HandleId h : t.outputs) e.out.push_back(static_cast<int32_t>(idx.handle_pos.at(h)));
        e.dep_off.push_back(static_cast<int32_t>(e.dep.size()));
        e.in_off.push_back(static_cast<int32_t>(e.in.size()));
        e.out_off.push_back(static_cast<int32_t>(e.out.size()));
    }
    for (const auto& h : g.handles) e.handle_bytes.push_back(h.bytes);
    return e;
}

const std::vector<std::string> kPolicyNames = {"fifo", "dm", "dmda", "dmdap", "inspirit"};

void copy_state_out(const RegulatorState& s, tbsim_regulator_state* o) {
    o->mode = static_cast<int32_t>(s.mode);
    o->phase = static_cast<int32_t>(s.state);
    o->peak = s.peak;
    o->prev_nready = s.prev_nready;
    o->last_trigger_nready = s.last_trigger_nready;
    o->s_dec_count = s.s_dec_count;
    o->cur_k = s.cur_k;
    o->n_samples = static_cast<int32_t>(s.samples.size());
    int i = 0;
    for (const auto& [t, v] : s.samples) {
        if (i >= TBSIM_MAX_SLOPE_SAMPLES) break;
        o->sample_time[i] = t;
        o->sample_nready[i] = v;
        ++i;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- generators (reference src/generators.cpp, tests/oracles.cpp) --------

void* ref_gen_layered(int n, int layers, double p, uint64_t seed) {
    try {
        return new Exported(export_graph(generate_layered_dag(n, layers, p, seed)));
    } catch (const std::exception& e) { fail(e); return nullptr; }
}
void* ref_gen_cholesky(int nb, int64_t bytes) {
    try { return new Exported(export_graph(build_cholesky_dag(nb, bytes))); }
    catch (const std::exception& e) { fail(e); return nullptr; }
}
void* ref_gen_lu(int nb, int64_t bytes) {
    try { return new Exported(export_graph(build_lu_dag(nb, bytes))); }
    catch (const std::exception& e) { fail(e); return nullptr; }
}
// oracle::random_dag from the reference tests (non-contiguous ids on purpose).
void* ref_gen_random(uint64_t seed, int n, double p, const char* const* types,
                     int n_types, int with_handles) {
    try {
        std::vector<std::string> ty(types, types + n_types);
        return new Exported(export_graph(oracle::random_dag(seed, n, p, ty, with_handles != 0)));
    } catch (const std::exception& e) { fail(e); return nullptr; }
}
void* ref_gen_file(const char* path) {
    try { return new Exported(export_graph(load_dag_file(path))); }
    catch (const std::exception& e) { fail(e); return nullptr; }
}
// sizes: n_tasks, n_deps, n_in, n_out, n_handles, n_types
void ref_exported_sizes(const void* h, int64_t* s) {
    const auto* e = static_cast<const Exported*>(h);
    s[0] = static_cast<int64_t>(e->type.size());
    s[1] = static_cast<int64_t>(e->dep.size());
    s[2] = static_cast<int64_t>(e->in.size());
    s[3] = static_cast<int64_t>(e->out.size());
    s[4] = static_cast<int64_t>(e->handle_bytes.size());
    s[5] = static_cast<int64_t>(e->type_names.size());
}
const char* ref_exported_type_name(const void* h, int i) {
    return static_cast<const Exported*>(h)->type_names[i].c_str();
}
void ref_exported_copy(const void* h, int32_t* dep_off, int32_t* dep, int32_t* in_off,
                       int32_t* in, int32_t* out_off, int32_t* out, int32_t* type,
                       int64_t* handle_bytes, int64_t* task_id) {
    const auto* e = static_cast<const Exported*>(h);
    auto cp = [](auto* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(dep_off, e->dep_off); cp(dep, e->dep); cp(in_off, e->in_off); cp(in, e->in);
    cp(out_off, e->out_off); cp(out, e->out); cp(type, e->type);
    cp(handle_bytes, e->handle_bytes); cp(task_id, e->task_id);
}
void ref_exported_free(void* h) { delete static_cast<Exported*>(h); }

// ---- attributes (reference src/attributes.cpp) ---------------------------

int ref_attributes(const tbsim_batch_desc* d, const char* const* names,
                   const tbsim_costs* costs, int request, int prio_kind,
                   tbsim_attr_out* o, int threads) {
    int status = 0;
    std::string err;
    const CostTable table = make_costs(*costs, names);
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : omp_get_max_threads())
    for (int64_t g = 0; g < d->n_graphs; ++g) {
        if (status) continue;
        try {
            TaskGraph tg = graph_of(*d, g, names);
            const int64_t t0 = d->task_base[g];
            auto put = [&](int64_t* dst, const std::vector<int64_t>& v) {
                if (dst) std::memcpy(dst + t0, v.data(), v.size() * sizeof(int64_t));
            };
            if (request & TBSIM_ATTR_ALL) {
                PriorityKind pk = prio_kind == 0 ? PriorityKind::UpwardRank
                                  : prio_kind == 1 ? PriorityKind::Depth : PriorityKind::Zero;
                TaskAttributes a = compute_attributes(tg, table, pk);
                put(o->ability, a.ability);
                put(o->efficiency, a.efficiency);
                put(o->static_priority, a.static_priority);
                if (o->unit_time_ms) o->unit_time_ms[g] = a.unit_time_ms;
            }
            if (request & TBSIM_ATTR_ABILITY) put(o->ability, compute_inspiring_ability_serial(tg));
            if (request & TBSIM_ATTR_CALIBRATE) {
                CalibrationResult r = calibrate_unit_time(tg, table);
                if (o->unit_time_ms) o->unit_time_ms[g] = r.unit_time_ms;
                if (o->w0_ms) o->w0_ms[g] = r.w0_ms;
                if (o->best_score) o->best_score[g] = r.best_score;
                if (o->w0_score) o->w0_score[g] = r.w0_score;
                if (o->evaluations) o->evaluations[g] = r.evaluations;
            }
            if (request & TBSIM_ATTR_EFFICIENCY)
                put(o->efficiency, compute_inspiring_efficiency_serial(tg, table, o->unit_time_ms[g]));
            if (request & TBSIM_ATTR_RANK) put(o->static_priority, upward_rank_priority(tg, table));
            if (request & TBSIM_ATTR_DEPTH) put(o->depth, depth_priority(tg));
            if (request & TBSIM_ATTR_LAYERS) {
                auto l = topological_layers(tg);
                if (o->layer) std::memcpy(o->layer + t0, l.data(), l.size() * sizeof(int));
            }
        } catch (const std::exception& e) {
#pragma omp critical
            {
                if (!status) { status = fail(e); err = g_err; }
            }
        }
    }
    if (status) g_err = err;
    return status;
}

// ---- simulate (reference src/engine.cpp + src/policies.cpp) --------------

int ref_simulate(const tbsim_batch_desc* d, const char* const* names,
                 const tbsim_platform_desc* platforms, const int32_t* platform_of,
                 int policy, const tbsim_regulator_cfg* reg, const tbsim_attr_in* ai,
                 tbsim_sim_out* o, int threads) {
    int status = 0;
    std::string err;
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : omp_get_max_threads())
    for (int64_t g = 0; g < d->n_graphs; ++g) {
        if (status) continue;
        try {
            TaskGraph tg = graph_of(*d, g, names);
            Platform p = make_platform(platforms[platform_of ? platform_of[g] : 0], names);
            const int64_t t0 = d->task_base[g], n = d->task_base[g + 1] - t0;
            TaskAttributes a;
            auto take = [&](const int64_t* src, std::vector<int64_t>& dst) {
                dst.assign(n, 0);
                if (ai && src) std::memcpy(dst.data(), src + t0, n * sizeof(int64_t));
            };
            take(ai ? ai->ability : nullptr, a.ability);
            take(ai ? ai->efficiency : nullptr, a.efficiency);
            take(ai ? ai->static_priority : nullptr, a.static_priority);
            RegulatorConfig cfg;
            if (reg) {
                const tbsim_regulator_cfg& r = reg[g];
                cfg.task_window = r.task_window; cfg.s_inc = r.s_inc; cfg.k_inc = r.k_inc;
                cfg.s_dec = r.s_dec; cfg.c = r.c; cfg.dec_step = r.dec_step;
                cfg.slope_samples = r.slope_samples;
            } else {
                cfg = default_regulator_config(p, tg);
            }
            auto pol = make_policy(kPolicyNames.at(policy), a, cfg);
            SimOptions opts;
            opts.record_trace = o->push_time != nullptr;
            SimTrace tr = simulate(tg, p, *pol, opts);
            for (int64_t i = 0; i < n; ++i) {
                if (o->worker) o->worker[t0 + i] = tr.per_task[i].worker;
                if (o->start_ms) o->start_ms[t0 + i] = tr.per_task[i].start_ms;
                if (o->end_ms) o->end_ms[t0 + i] = tr.per_task[i].end_ms;
            }
            if (o->makespan_ms) o->makespan_ms[g] = tr.makespan_ms;
            if (o->completed) o->completed[g] = n;
            if (opts.record_trace) {
                GraphIndex idx = build_index(tg);
                for (size_t k = 0; k < tr.pushes.size(); ++k) {
                    o->push_time[t0 + k] = tr.pushes[k].time_ms;
                    o->push_task[t0 + k] = static_cast<int32_t>(idx.task_pos.at(tr.pushes[k].task));
                }
                for (size_t k = 0; k < tr.pops.size(); ++k) {
                    o->pop_time[t0 + k] = tr.pops[k].time_ms;
                    o->pop_task[t0 + k] = static_cast<int32_t>(idx.task_pos.at(tr.pops[k].task));
                    o->pop_worker[t0 + k] = tr.pops[k].worker;
                }
                for (size_t k = 0; k < tr.nready_samples.size(); ++k) {
                    o->sample_time[2 * t0 + k] = tr.nready_samples[k].first;
                    o->sample_nready[2 * t0 + k] = tr.nready_samples[k].second;
                }
            }
            if (const auto* c = pop_mode_counts(*pol); c && o->pop_mode_counts)
                for (int m = 0; m < 3; ++m) o->pop_mode_counts[3 * g + m] = (*c)[m];
            if (const auto* s = regulator_state(*pol); s && o->reg_state)
                copy_state_out(*s, &o->reg_state[g]);
        } catch (const std::exception& e) {
#pragma omp critical
            {
                if (!status) { status = fail(e); err = g_err; }
            }
        }
    }
    if (status) g_err = err;
    return status;
}

// ---- CPU baseline: the bench-cell pipeline (src/bench.cpp:102-128) -------
//
// Graphs are generated by the reference's generate_layered_dag outside the
// timed region; the timed region is, per DAG, compute_attributes(UpwardRank)
// + default_regulator_config + make_policy + simulate (record_trace off),
// OpenMP over DAGs with the inner kernels serial (nested regions inactive,
// exactly as run_bench runs a cell).  Returns wall seconds of the timed part.

struct RefBenchSet {
    std::vector<TaskGraph> graphs;
    std::vector<Platform> platforms;  // per graph
};

void* ref_bench_prepare_layered(int64_t n_dags, int n, int layers, double p,
                                const uint64_t* seeds, const int32_t* n_cpus,
                                const int32_t* n_gpus, int threads) {
    try {
        auto* s = new RefBenchSet;
        s->graphs.resize(n_dags);
        s->platforms.resize(n_dags);
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : omp_get_max_threads())
        for (int64_t i = 0; i < n_dags; ++i) {
            s->graphs[i] = generate_layered_dag(n, layers, p, seeds[i]);
            Platform pl;
            pl.name = "mix";
            pl.costs = default_cost_table();
            int id = 0;
            for (int c = 0; c < n_cpus[i]; ++c) pl.workers.push_back({id++, DeviceKind::Cpu, 0});
            for (int gg = 0; gg < n_gpus[i]; ++gg) pl.workers.push_back({id++, DeviceKind::Gpu, 1 + gg});
            pl.num_nodes = 1 + n_gpus[i];
            pl.latency_ms = 0.01;
            pl.bandwidth.assign(pl.num_nodes, std::vector<double>(pl.num_nodes, 0.0));
            for (int a = 0; a < pl.num_nodes; ++a)
                for (int b = 0; b < pl.num_nodes; ++b)
                    if (a != b) pl.bandwidth[a][b] = (a > 0 && b > 0) ? 24e6 : 12e6;
            s->platforms[i] = std::move(pl);
        }
        return s;
    } catch (const std::exception& e) { fail(e); return nullptr; }
}

void ref_bench_free(void* h) { delete static_cast<RefBenchSet*>(h); }

int ref_bench_run(void* h, int policy, int threads, double* makespans, double* seconds) {
    auto* s = static_cast<RefBenchSet*>(h);
    const int64_t n = static_cast<int64_t>(s->graphs.size());
    int status = 0;
    auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : omp_get_max_threads())
    for (int64_t i = 0; i < n; ++i) {
        try {
            const TaskGraph& g = s->graphs[i];
            const Platform& p = s->platforms[i];
            TaskAttributes attrs = compute_attributes(g, p.costs, PriorityKind::UpwardRank);
            RegulatorConfig reg = default_regulator_config(p, g);
            SimOptions opts;
            opts.record_trace = false;
            auto pol = make_policy(kPolicyNames.at(policy), attrs, reg);
            SimTrace t = simulate(g, p, *pol, opts);
            if (makespans) makespans[i] = t.makespan_ms;
        } catch (const std::exception& e) {
#pragma omp critical
            { status = fail(e); }
        }
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return status;
}

// Brute-force pins from the reference's tests/oracles.cpp.
int ref_oracle_descendants(const tbsim_batch_desc* d, const char* const* names, int64_t* out) {
    try {
        for (int64_t g = 0; g < d->n_graphs; ++g) {
            auto v = oracle::descendant_counts(graph_of(*d, g, names));
            std::memcpy(out + d->task_base[g], v.data(), v.size() * sizeof(int64_t));
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}
int ref_oracle_best_unit_makespan(const tbsim_batch_desc* d, const char* const* names,
                                  int workers, int64_t* out) {
    try {
        for (int64_t g = 0; g < d->n_graphs; ++g)
            out[g] = oracle::best_unit_makespan(graph_of(*d, g, names), workers);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int ref_max_threads(void) { return omp_get_max_threads(); }

}  // extern "C"
