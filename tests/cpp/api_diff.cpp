// api_diff.cpp -- differential report of the drop-in C++ API.
//
// The same source is compiled twice: against this repo's headers and
// libtbsim_cpp.so (the B200 path), and -- by tests/golden/make_api_diff.sh,
// in a container that has the reference -- against the reference's own
// headers and its unmodified sources (oracle/_ref/libtbsim_ref.so).  Both
// print the report below; tests/test_api_diff.py requires them to be
// identical line for line.  Doubles print as hex floats (%a), so "identical"
// means bit-identical; long per-task vectors print as a 64-bit FNV-1a digest
// of their bytes plus a few entries.  Exceptions print as their type and
// what() text.  Inputs: the reference's generators, random DAGs of this
// file's own construction (non-contiguous and shuffled ids, multi-edges,
// inputs that are not dependencies, several handle sizes), degenerate shapes
// and invalid graphs.
#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <deque>
#include <fstream>
#include <functional>
#include <iostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tbsim/attributes.hpp"
#include "tbsim/bench.hpp"
#include "tbsim/engine.hpp"
#include "tbsim/platform.hpp"
#include "tbsim/policies.hpp"
#include "tbsim/taskgraph.hpp"
#include "tbsim/text.hpp"

using namespace tbsim;

namespace {

std::ostream& out = std::cout;

std::string hx(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%a", v);
    return b;
}

struct Digest {
    uint64_t h = 1469598103934665603ull;
    void bytes(const void* p, size_t n) {
        const auto* c = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
    }
    template <typename T>
    void val(const T& v) { bytes(&v, sizeof v); }
    void str(const std::string& s) {
        bytes(s.data(), s.size());
        val(s.size());
    }
};

template <typename T>
std::string show(const T& v) {
    if constexpr (std::is_floating_point_v<T>) return hx(v);
    else return std::to_string(v);
}

// short vectors in full, long ones as size + digest + the first/last entries
template <typename T>
void vec(const std::string& tag, const std::vector<T>& v) {
    out << tag << " n=" << v.size();
    if (v.size() <= 24) {
        for (const auto& x : v) out << ' ' << show(x);
    } else {
        Digest d;
        for (const auto& x : v) d.val(x);
        out << " fnv=" << std::hex << d.h << std::dec << " head=" << show(v.front()) << ',' << show(v[1])
            << " tail=" << show(v.back());
    }
    out << '\n';
}

void text(const std::string& tag, const std::string& s) {
    if (s.size() <= 400) {
        out << tag << " [" << s << "]\n";
    } else {
        Digest d;
        d.str(s);
        out << tag << " bytes=" << s.size() << " fnv=" << std::hex << d.h << std::dec << '\n';
    }
}

// An exception's text; a JSON syntax error keeps the loader's own prefix
// ("<where>: bad JSON:") -- the detail after it is the JSON parser's wording
// (nlohmann::json in the reference, a third-party library), not the API's.
std::string what_of(const std::exception& e) {
    std::string m = e.what();
    const auto k = m.find("bad JSON:");
    if (k != std::string::npos) m = m.substr(0, k + 9) + " ...";
    return m;
}

// runs f; an exception prints as its type and text
void guard(const std::string& tag, const std::function<void()>& f) {
    try {
        f();
    } catch (const std::invalid_argument& e) {
        out << tag << " THROW invalid_argument: " << what_of(e) << '\n';
    } catch (const std::out_of_range& e) {
        out << tag << " THROW out_of_range: " << what_of(e) << '\n';
    } catch (const std::logic_error& e) {
        out << tag << " THROW logic_error: " << what_of(e) << '\n';
    } catch (const std::runtime_error& e) {
        out << tag << " THROW runtime_error: " << what_of(e) << '\n';
    }
}

const std::vector<std::string> kMixed = {"LAYERK0", "LAYERK1", "LAYERK2", "LAYERK3", "UNIT", "GEMM", "TRSM"};

// a random DAG of this file's own construction
TaskGraph random_dag(uint64_t seed, int n, double p, bool handles) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> coin(0.0, 1.0);
    TaskGraph g;
    g.name = "rnd" + std::to_string(seed);
    std::vector<TaskId> ids(n);
    for (int i = 0; i < n; ++i) ids[i] = 5000 + 13 * i;
    std::shuffle(ids.begin(), ids.end(), rng);
    if (handles)
        for (int h = 0; h < n; ++h) g.handles.push_back({900 + 3 * h, static_cast<int64_t>(1 + rng() % 4) * 409600});
    for (int i = 0; i < n; ++i) {
        TaskNode t;
        t.id = ids[i];
        t.type = kMixed[rng() % kMixed.size()];
        for (int j = 0; j < i; ++j)
            if (coin(rng) < p) t.deps.push_back(ids[j]);
        if (!t.deps.empty() && coin(rng) < 0.15) t.deps.push_back(t.deps.front());  // multi-edge
        if (handles) {
            const int nin = static_cast<int>(rng() % 4);
            for (int k = 0; k < nin; ++k) t.inputs.push_back(900 + 3 * static_cast<int64_t>(rng() % n));
            t.outputs.push_back(900 + 3 * static_cast<int64_t>(i));
        }
        g.tasks.push_back(t);
    }
    return g;
}

CostTable mixed_costs() {
    CostTable c = default_cost_table();
    c.set("GEMM", DeviceKind::Gpu, 0.75);
    c.set("TRSM", DeviceKind::Cpu, 3.5);
    return c;
}

Platform mixed_platform(const char* name, int cpus, int gpus, double lat) {
    Platform p = make_preset("26cpu_2gpu");
    p.name = name;
    p.costs = mixed_costs();
    p.workers.clear();
    int id = 0;
    for (int i = 0; i < cpus; ++i) p.workers.push_back({id++, DeviceKind::Cpu, 0});
    for (int i = 0; i < gpus; ++i) p.workers.push_back({id++, DeviceKind::Gpu, 1 + i});
    p.num_nodes = 1 + gpus;
    p.latency_ms = lat;
    p.bandwidth.assign(p.num_nodes, std::vector<double>(p.num_nodes, 0.0));
    for (int a = 0; a < p.num_nodes; ++a)
        for (int b = 0; b < p.num_nodes; ++b)
            if (a != b) p.bandwidth[a][b] = (a && b) ? 3e7 + 1e6 * (a + b) : 1.1e7;
    return p;
}

void structure(const TaskGraph& g) {
    out << "edges " << edge_count(g) << '\n';
    guard("layers", [&] { vec("layers", topological_layers(g)); });
    guard("order", [&] { vec("order", topological_order(g)); });
    guard("validate", [&] {
        for (const auto& v : validate(g)) out << "violation " << v.message << '\n';
    });
    guard("writers", [&] {
        for (const auto& v : check_writer_chains(g)) out << "writer " << v.message << '\n';
    });
}

void attributes(const TaskGraph& g, const CostTable& costs) {
    guard("ability", [&] { vec("ability", compute_inspiring_ability(g)); });
    guard("ability_serial", [&] { vec("ability_serial", compute_inspiring_ability_serial(g)); });
    for (double w : {0.0, 0.5, 1.0, 2.5, 16.0})
        guard("eff" + hx(w), [&] { vec("eff " + hx(w), compute_inspiring_efficiency(g, costs, w)); });
    guard("eff_serial", [&] { vec("eff_serial", compute_inspiring_efficiency_serial(g, costs, 1.0)); });
    guard("calib", [&] {
        const CalibrationResult c = calibrate_unit_time(g, costs);
        out << "calib " << hx(c.unit_time_ms) << ' ' << hx(c.w0_ms) << ' ' << c.best_score << ' ' << c.w0_score
            << ' ' << c.evaluations << '\n';
    });
    guard("rank", [&] { vec("rank", upward_rank_priority(g, costs)); });
    guard("depth", [&] { vec("depth", depth_priority(g)); });
    guard("median", [&] { out << "median " << hx(median_gpu_time_ms(g, costs)) << '\n'; });
    for (PriorityKind k : {PriorityKind::UpwardRank, PriorityKind::Depth, PriorityKind::Zero})
        guard("attrs", [&] {
            const TaskAttributes a = compute_attributes(g, costs, k);
            out << "attrs kind=" << static_cast<int>(k) << " unit=" << hx(a.unit_time_ms) << '\n';
            vec("attrs.ability", a.ability);
            vec("attrs.efficiency", a.efficiency);
            vec("attrs.prio", a.static_priority);
            std::ostringstream s;
            write_attributes_csv(s, g, a);
            text("attrs.csv", s.str());
        });
}

void schedules(const TaskGraph& g, const Platform& p) {
    out << "platform " << p.name << '\n';
    guard("regcfg", [&] {
        const RegulatorConfig c = default_regulator_config(p, g);
        out << "regcfg " << c.task_window << ' ' << c.s_inc << ' ' << hx(c.k_inc) << ' ' << c.s_dec << ' ' << c.c
            << ' ' << c.dec_step << ' ' << c.slope_samples << '\n';
    });
    TaskAttributes a;
    bool have = true;
    guard("sched.attrs", [&] {
        have = false;
        a = compute_attributes(g, p.costs, PriorityKind::UpwardRank);
        have = true;
    });
    if (!have) a = TaskAttributes{};
    // the policies need a regulator config; without one (no median) the
    // graph is not simulated
    RegulatorConfig rc{};
    bool have_rc = false;
    guard("sim.regcfg", [&] {
        rc = default_regulator_config(p, g);
        have_rc = true;
    });
    if (!have_rc) return;
    for (const std::string& pol : policy_names()) {
        guard("sim " + pol, [&] {
            auto policy = make_policy(pol, a, rc);
            const SimTrace t = simulate(g, p, *policy);
            out << "sim " << pol << " makespan=" << hx(t.makespan_ms) << '\n';
            std::vector<int> wk;
            std::vector<double> st, en;
            for (const auto& e : t.per_task) {
                wk.push_back(e.worker);
                st.push_back(e.start_ms);
                en.push_back(e.end_ms);
            }
            vec("sim.worker", wk);
            vec("sim.start", st);
            vec("sim.end", en);
            std::vector<double> pt, ot, nt;
            std::vector<int64_t> pk, ok, nn;
            std::vector<int> ow;
            for (const auto& r : t.pushes) { pt.push_back(r.time_ms); pk.push_back(r.task); }
            for (const auto& r : t.pops) { ot.push_back(r.time_ms); ok.push_back(r.task); ow.push_back(r.worker); }
            for (const auto& r : t.nready_samples) { nt.push_back(r.first); nn.push_back(r.second); }
            vec("sim.push_t", pt);
            vec("sim.push_task", pk);
            vec("sim.pop_t", ot);
            vec("sim.pop_task", ok);
            vec("sim.pop_worker", ow);
            vec("sim.nready_t", nt);
            vec("sim.nready", nn);
            if (const auto* c = pop_mode_counts(*policy)) out << "popmodes " << (*c)[0] << ' ' << (*c)[1] << ' ' << (*c)[2] << '\n';
            if (const auto* s = regulator_state(*policy))
                out << "regstate " << static_cast<int>(s->mode) << ' ' << static_cast<int>(s->state) << ' ' << s->peak
                    << ' ' << s->prev_nready << ' ' << s->last_trigger_nready << ' ' << s->s_dec_count << ' '
                    << hx(s->cur_k) << ' ' << s->samples.size() << '\n';
            for (double q : {0.0, t.makespan_ms / 3, t.makespan_ms / 2, t.makespan_ms})
                guard("nready_at", [&] { out << "nready_at " << hx(q) << ' ' << nready_at(t, q) << '\n'; });
            guard("window", [&] {
                for (const auto& w : window_histogram(t, 5.0))
                    out << "window " << hx(w.window_start_ms) << ' ' << w.pushes << ' ' << w.pops << '\n';
            });
            std::ostringstream gc, nc, pc;
            write_gantt_csv(gc, g, t);
            write_nready_csv(nc, t);
            write_push_pop_csv(pc, t, 2.5);
            text("gantt.csv", gc.str());
            text("nready.csv", nc.str());
            text("pushpop.csv", pc.str());
            SimOptions quiet;
            quiet.record_trace = false;
            auto again = make_policy(pol, a, rc);
            const SimTrace q = simulate(g, p, *again, quiet);
            out << "quiet makespan=" << hx(q.makespan_ms) << " pushes=" << q.pushes.size() << " pops=" << q.pops.size()
                << " samples=" << q.nready_samples.size() << '\n';
        });
    }
}

// structure_only: the reference's attribute functions have no cycle check
// (a cyclic graph is undefined behaviour there), so a cycle is only fed to
// the functions that define an error for it
void graph_section(const std::string& name, const TaskGraph& g, const std::vector<Platform>& pls,
                   const CostTable& costs, bool structure_only = false) {
    out << "== " << name << " tasks=" << g.tasks.size() << " handles=" << g.handles.size() << '\n';
    structure(g);
    if (structure_only) return;
    attributes(g, costs);
    for (const Platform& p : pls) schedules(g, p);
    std::ostringstream s;
    guard("save", [&] {
        save_dag(g, s);
        text("dag", s.str());
        std::istringstream in(s.str());
        const TaskGraph back = load_dag(in);
        out << "roundtrip " << (back == g ? "equal" : "differs") << '\n';
    });
}

// An EngineView of arbitrary state, for the push/pop free functions
struct FakeView final : EngineView {
    const TaskGraph* g = nullptr;
    const Platform* p = nullptr;
    double now_ms = 0.0;
    std::vector<size_t> qlen;
    std::vector<char> busy;
    std::vector<double> free_at;
    std::vector<std::vector<double>> transfer, fraction;
    double now() const override { return now_ms; }
    const TaskGraph& graph() const override { return *g; }
    const Platform& platform() const override { return *p; }
    size_t queue_length(int w) const override { return qlen[w]; }
    bool worker_busy(int w) const override { return busy[w] != 0; }
    double worker_free_at(int w) const override { return free_at[w]; }
    double estimated_transfer_ms(size_t t, int w) const override { return transfer[t][w]; }
    double resident_fraction(size_t t, int n) const override { return fraction[t][n]; }
};

// push_* / pop_* over random views and queues: ties are frequent (values
// on a coarse grid), so the tie-breaks are exercised
void rules_section(uint64_t seed, const Platform& p) {
    out << "== rules " << seed << ' ' << p.name << '\n';
    std::mt19937_64 rng(seed);
    const TaskGraph g = random_dag(seed, 40, 0.1, true);
    FakeView v;
    v.g = &g;
    v.p = &p;
    const size_t W = p.workers.size();
    auto grid = [&](int k) { return 0.25 * static_cast<double>(rng() % k); };
    for (int round = 0; round < 6; ++round) {
        v.now_ms = grid(40);
        v.qlen.assign(W, 0);
        v.busy.assign(W, 0);
        v.free_at.assign(W, 0.0);
        for (size_t w = 0; w < W; ++w) {
            v.qlen[w] = rng() % 4;
            v.busy[w] = static_cast<char>(rng() % 2);
            v.free_at[w] = grid(60);
        }
        v.transfer.assign(g.tasks.size(), std::vector<double>(W, 0.0));
        v.fraction.assign(g.tasks.size(), std::vector<double>(p.num_nodes, 1.0));
        for (auto& r : v.transfer)
            for (auto& x : r) x = grid(8);
        for (auto& r : v.fraction)
            for (auto& x : r) x = 0.125 * static_cast<double>(rng() % 9);
        std::vector<int> pf, pd, pa;
        for (size_t t = 0; t < g.tasks.size(); ++t) {
            guard("push_fifo", [&] { pf.push_back(push_fifo(t, v)); });
            guard("push_dm", [&] { pd.push_back(push_dm(t, v)); });
            guard("push_dmda", [&] { pa.push_back(push_dmda(t, v)); });
        }
        vec("push_fifo", pf);
        vec("push_dm", pd);
        vec("push_dmda", pa);
        TaskAttributes a;
        for (size_t t = 0; t < g.tasks.size(); ++t) {
            a.ability.push_back(static_cast<int64_t>(rng() % 4));
            a.efficiency.push_back(static_cast<int64_t>(rng() % 3));
            a.static_priority.push_back(static_cast<int64_t>(rng() % 3) * 1000);
        }
        std::vector<QueueEntry> q;
        for (int k = 0; k < 12; ++k) q.push_back({static_cast<size_t>(rng() % g.tasks.size()), rng() % 50});
        out << "pop_fifo " << pop_fifo(q) << " pop_priority " << pop_priority(q, a);
        for (PopMode m : {PopMode::HighAbility, PopMode::HighEfficiency, PopMode::HighEfficiencyLocality})
            out << ' ' << to_string(m) << '=' << pop_adaptive(m, static_cast<int>(rng() % W), q, a, v);
        out << '\n';
    }
}

}  // namespace

int main() {
    std::cout << std::unitbuf;
    const CostTable dc = default_cost_table();
    const std::vector<Platform> presets = {make_preset("26cpu_2gpu"), make_preset("homog2"), make_preset("2gpu"),
                                           make_preset("26cpu_1gpu")};
    const std::vector<Platform> mixed = {mixed_platform("m4c1g", 4, 1, 0.01), mixed_platform("m8c3g", 8, 3, 0.125),
                                         mixed_platform("m30c6g", 30, 6, 0.0)};
    const CostTable mc = mixed_costs();
    // the reference's generators
    for (int nb : {1, 3, 6}) graph_section("cholesky" + std::to_string(nb), build_cholesky_dag(nb, 960 * 960 * 4), presets, dc);
    for (int nb : {2, 5}) graph_section("lu" + std::to_string(nb), build_lu_dag(nb, 320 * 320 * 4), presets, dc);
    graph_section("stencil", build_stencil_dag(4, 3, 160 * 160 * 4), presets, dc);
    graph_section("layered60", generate_layered_dag(60, 5, 0.1, 1), presets, dc);
    graph_section("layered300", generate_layered_dag(300, 8, 0.05, 2), {presets[0], presets[1]}, dc);
    graph_section("layered1000", generate_layered_dag(1000, 10, 0.05, 3), {presets[0]}, dc);
    // random DAGs of this file's own construction on mixed platforms
    for (uint64_t s = 1; s <= 8; ++s)
        graph_section("random" + std::to_string(s), random_dag(s, 10 + 17 * static_cast<int>(s), 0.08, s % 3 != 0),
                      mixed, mc);
    // degenerate shapes
    {
        TaskGraph e;
        e.name = "empty";
        graph_section("empty", e, presets, dc);
        TaskGraph one;
        one.tasks = {{7, "UNIT", {}, {}, {}}};
        graph_section("one", one, presets, dc);
        TaskGraph flat;
        for (int i = 0; i < 40; ++i) flat.tasks.push_back({i, "LAYERK1", {}, {}, {}});
        graph_section("flat", flat, presets, dc);
        TaskGraph chain;
        for (int i = 0; i < 50; ++i) chain.tasks.push_back({i, "LAYERK2", i ? std::vector<TaskId>{i - 1} : std::vector<TaskId>{}, {}, {}});
        graph_section("chain", chain, presets, dc);
        TaskGraph star;
        star.tasks.push_back({0, "LAYERK3", {}, {}, {}});
        for (int i = 1; i < 40; ++i) star.tasks.push_back({i, "LAYERK0", {0}, {}, {}});
        graph_section("star", star, presets, dc);
    }
    // invalid graphs and inputs
    {
        TaskGraph dup;
        dup.tasks = {{1, "UNIT", {}, {}, {}}, {1, "UNIT", {}, {}, {}}};
        graph_section("dup_ids", dup, {presets[1]}, dc);
        TaskGraph dang;
        dang.tasks = {{1, "UNIT", {42}, {}, {}}};
        graph_section("dangling", dang, {presets[1]}, dc);
        TaskGraph cyc;
        cyc.tasks = {{0, "UNIT", {1}, {}, {}}, {1, "UNIT", {0}, {}, {}}};
        graph_section("cycle", cyc, {presets[1]}, dc, true);
        TaskGraph nocost;
        nocost.tasks = {{0, "NO_SUCH_TYPE", {}, {}, {}}};
        graph_section("nocost", nocost, {presets[1]}, dc);
        TaskGraph gonly;
        gonly.tasks = {{0, "GONLY", {}, {}, {}}};
        Platform hp = make_preset("homog2");
        hp.costs.set("GONLY", DeviceKind::Gpu, 1.0);
        graph_section("gpu_only_type", gonly, {hp}, hp.costs);
        guard("negative W", [&] { vec("effneg", compute_inspiring_efficiency(build_cholesky_dag(2, 64), dc, -1.0)); });
        guard("unknown policy", [&] { make_policy("nope", TaskAttributes{}); });
        guard("unknown preset", [&] { make_preset("nope"); });
        guard("cost set", [&] { CostTable c; c.set("X", DeviceKind::Cpu, 0.0); });
        guard("cost get", [&] { dc.get("NOPE", DeviceKind::Gpu); });
        guard("exec", [&] { presets[1].exec_time_ms("NOPE", presets[1].workers[0]); });
        guard("transfer", [&] { out << "xfer " << hx(presets[0].transfer_time_ms(1 << 20, 0, 2)) << '\n'; });
        guard("transfer bad", [&] { presets[0].transfer_time_ms(1, 0, 9); });
        guard("pop empty", [&] { pop_fifo({}); });
        guard("layered bad", [&] { generate_layered_dag(10, 0, 0.1, 1); });
        guard("cholesky bad", [&] { build_cholesky_dag(0, 1); });
        std::istringstream bad("{\"name\": \"x\", \"tasks\": [\n{\"id\": 1, \"type\": \"UNIT\", \"deps\": [}\n");
        guard("load bad", [&] { load_dag(bad); });
    }
    // a task reading an undeclared handle (the engine's handle_pos.at())
    {
        TaskGraph stray;
        stray.handles = {{7, 4096}};
        stray.tasks = {{0, "UNIT", {}, {7}, {7}}, {1, "UNIT", {0}, {99}, {}}};
        graph_section("stray_handle", stray, {presets[0]}, dc);
    }
    // larger shapes: C5's DAG shape on a 36-worker mix, an LU factorization
    graph_section("layered4096", generate_layered_dag(4096, 10, 0.05, 7), {mixed_platform("m32c4g", 32, 4, 0.01)}, mc);
    graph_section("lu12", build_lu_dag(12, 320 * 320 * 4), {presets[0]}, dc);
    // DAG files: every error the NDJSON loader names
    {
        const std::string meta = "{\"kind\":\"meta\",\"name\":\"x\",\"version\":1}\n";
        const std::vector<std::string> docs = {
            "",
            meta + "\n",
            meta + "[1,2]\n",
            meta + "{\"id\":1}\n",
            meta + "{\"kind\":\"edge\"}\n",
            meta + meta,
            "{\"kind\":\"task\",\"id\":0,\"type\":\"UNIT\",\"deps\":[],\"inputs\":[],\"outputs\":[]}\n" + meta,
            "{\"kind\":\"meta\",\"name\":\"x\",\"version\":2}\n",
            "{\"kind\":\"meta\",\"version\":1}\n",
            meta + "{\"kind\":\"task\",\"type\":\"UNIT\",\"deps\":[],\"inputs\":[],\"outputs\":[]}\n",
            meta + "{\"kind\":\"task\",\"id\":\"a\",\"type\":\"UNIT\",\"deps\":[],\"inputs\":[],\"outputs\":[]}\n",
            meta + "{\"kind\":\"task\",\"id\":0,\"type\":5,\"deps\":[],\"inputs\":[],\"outputs\":[]}\n",
            meta + "{\"kind\":\"task\",\"id\":0,\"type\":\"UNIT\",\"deps\":3,\"inputs\":[],\"outputs\":[]}\n",
            meta + "{\"kind\":\"task\",\"id\":0,\"type\":\"UNIT\",\"deps\":[1.5],\"inputs\":[],\"outputs\":[]}\n",
            meta + "{\"kind\":\"handle\",\"id\":3}\n",
            meta + "{\"kind\":\"task\",\"id\":0,\"type\":\"UNIT\",\"deps\":[4],\"inputs\":[],\"outputs\":[9]}\n",
            meta + "{\"kind\":\"handle\",\"id\":1,\"bytes\":8}\n{\"kind\":\"task\",\"id\":0,\"type\":\"UNIT\",\"deps\":[],\"inputs\":[1],\"outputs\":[1]}\n",
        };
        for (size_t i = 0; i < docs.size(); ++i)
            guard("dagdoc" + std::to_string(i), [&] {
                std::istringstream in(docs[i]);
                const TaskGraph g = load_dag(in);
                out << "dagdoc" << i << " tasks=" << g.tasks.size() << " handles=" << g.handles.size() << " name=" << g.name
                    << '\n';
            });
        guard("dagfile missing", [&] { load_dag_file("/nonexistent/api_diff.dag"); });
    }
    // platform files: a valid one scheduling a random DAG, and the loader's
    // named errors (fields the reference reads with json::at() are left in
    // place: a missing one throws nlohmann's own exception type there)
    {
        const std::string w = "\"workers\":[{\"id\":0,\"kind\":\"cpu\",\"memory_node\":0},"
                              "{\"id\":1,\"kind\":\"cpu\",\"memory_node\":0},{\"id\":2,\"kind\":\"gpu\",\"memory_node\":1},"
                              "{\"id\":3,\"kind\":\"gpu\",\"memory_node\":2}]";
        const std::string c = "\"costs\":{\"LAYERK0\":{\"cpu\":2.5,\"gpu\":0.5},\"LAYERK1\":{\"cpu\":8,\"gpu\":1},"
                              "\"LAYERK2\":{\"cpu\":6,\"gpu\":2},\"LAYERK3\":{\"cpu\":24,\"gpu\":4},\"UNIT\":{\"cpu\":1,\"gpu\":1},"
                              "\"GEMM\":{\"gpu\":0.375},\"TRSM\":{\"cpu\":3,\"gpu\":1.5}}";
        const std::string bw = "\"bandwidth\":[[0,1.2e7,1.2e7],[1.2e7,0,2.5e7],[1.2e7,2.5e7,0]]";
        const std::vector<std::string> files = {
            "{" + w + "," + c + "," + bw + ",\"latency_ms\":0.02}",
            "{" + w + "," + c + "," + bw + "}",
            "{" + c + "," + bw + "}",
            "{" + w + "," + bw + "}",
            "{" + w + "," + c + "}",
            "{\"workers\":[{\"id\":1,\"kind\":\"cpu\",\"memory_node\":0}]," + c + ",\"bandwidth\":[[0]]}",
            "{\"workers\":[{\"id\":0,\"kind\":\"cpu\",\"memory_node\":1}]," + c + "," + bw + "}",
            "{\"workers\":[{\"id\":0,\"kind\":\"gpu\",\"memory_node\":5}]," + c + "," + bw + "}",
            "{" + w + "," + c + ",\"bandwidth\":[[0,1.2e7,1.2e7],[1.3e7,0,2.5e7],[1.2e7,2.5e7,0]]}",
            "{" + w + "," + c + ",\"bandwidth\":[[0,0,1.2e7],[0,0,2.5e7],[1.2e7,2.5e7,0]]}",
            "{" + w + "," + c + "," + bw + ",\"latency_ms\":-1}",
            "{\"workers\":[]," + c + "," + bw + "}",
        };
        for (size_t i = 0; i < files.size(); ++i) {
            const std::string path = "/tmp/tbsim_api_diff_platform_" + std::to_string(i) + ".json";
            {
                std::ofstream f(path);
                f << files[i];
            }
            guard("platfile" + std::to_string(i), [&] {
                const Platform p = load_platform_file(path);
                out << "platfile" << i << " workers=" << p.workers.size() << " nodes=" << p.num_nodes
                    << " lat=" << hx(p.latency_ms) << '\n';
                if (i == 0) {
                    const TaskGraph g = random_dag(77, 90, 0.06, true);
                    attributes(g, p.costs);
                    schedules(g, p);
                }
            });
            std::remove(path.c_str());
        }
        guard("platfile missing", [&] { load_platform_file("/nonexistent/api_diff.json"); });
        guard("resolve", [&] { out << "resolve " << resolve_platform("2gpu").workers.size() << '\n'; });
        for (const auto& n : preset_names()) out << "preset " << n << '\n';
    }
    // the push/pop free functions on views of arbitrary state
    for (uint64_t r = 1; r <= 3; ++r) rules_section(r, mixed[r % mixed.size()]);
    // stress shapes for the device paths: many inputs per task over many
    // memory nodes, more than 32 workers, deep and dense graphs, >= 32768 tasks
    {
        TaskGraph wide = random_dag(101, 120, 0.05, true);
        std::mt19937_64 rng(5);
        for (auto& t : wide.tasks)
            for (int k = 0; k < 40 + static_cast<int>(rng() % 30); ++k)
                t.inputs.push_back(900 + 3 * static_cast<int64_t>(rng() % wide.handles.size()));
        graph_section("wide_inputs", wide, {mixed_platform("m2c9g", 2, 9, 0.005), mixed_platform("m6c3g", 6, 3, 0.05)}, mc);
        graph_section("many_workers", random_dag(102, 400, 0.02, true),
                      {mixed_platform("m40c8g", 40, 8, 0.01), mixed_platform("m33c1g", 33, 1, 0.0)}, mc);
        graph_section("deep", generate_layered_dag(3000, 300, 0.01, 11), {presets[0], mixed[1]}, dc);
        graph_section("dense", random_dag(103, 150, 0.5, true), {mixed[0], mixed[2]}, mc);
        graph_section("big", generate_layered_dag(40000, 100, 0.0005, 13), {presets[0]}, dc);
        // asymmetric links, GPUs sharing a memory node, a GPU on the host
        // node (Platform objects built in code skip check_platform)
        Platform odd = mixed_platform("m_odd", 3, 3, 0.03);
        odd.workers[3].memory_node = 1;
        odd.workers[4].memory_node = 1;
        odd.workers[5].memory_node = 0;
        odd.num_nodes = 3;
        odd.bandwidth = {{0.0, 9e6, 1.7e7}, {2.1e7, 0.0, 4e7}, {6e6, 3.3e7, 0.0}};
        graph_section("odd_platform", random_dag(104, 160, 0.06, true), {odd}, mc);
    }
    // formatting and the regulator's host functions
    for (double v : {0.0, 1.0, 1.5, 2.125, 1234.5678901, 1e-7, 3.0000001})
        out << "fmt " << hx(v) << ' ' << fmt_ms(v) << ' ' << fmt_ratio(v) << '\n';
    {
        std::deque<std::pair<double, std::int64_t>> s;
        for (int i = 0; i < 8; ++i) s.push_back({0.5 * i + 0.1 * (i % 3), 3 * i - (i % 2)});
        out << "calculate_k " << hx(calculate_k(s)) << '\n';
        RegulatorConfig cfg = default_regulator_config(presets[0], build_cholesky_dag(8, 64));
        RegulatorState st;
        for (int i = 0; i < 60; ++i) {
            const int64_t cur = (i < 30) ? 2 * i + (i % 4) : 90 - 2 * i + (i % 3);
            regulator_step(st, cfg, cur, 0.75 * i);
            out << "reg " << i << ' ' << static_cast<int>(st.mode) << ' ' << static_cast<int>(st.state) << ' ' << st.peak
                << ' ' << st.s_dec_count << ' ' << hx(st.cur_k) << '\n';
        }
    }
    // run_bench
    {
        BenchSpec spec;
        spec.app = "cholesky";
        spec.sizes = {4, 6};
        spec.platforms = {"26cpu_2gpu", "homog2"};
        spec.policies = policy_names();
        std::ostringstream s;
        guard("bench", [&] {
            write_bench_csv(s, run_bench(spec));
            text("bench.csv", s.str());
        });
        BenchSpec lay;
        lay.app = "autogen";
        lay.sizes = {200, 500};
        lay.platforms = {"26cpu_1gpu"};
        lay.policies = {"dmda", "inspirit"};
        lay.seed = 5;
        lay.regulator.task_window = 3;
        lay.regulator.k_inc = 0.25;
        std::ostringstream s2;
        guard("bench2", [&] {
            write_bench_csv(s2, run_bench(lay));
            text("bench2.csv", s2.str());
        });
        BenchSpec heat;
        heat.app = "heat";
        heat.sizes = {3, 4};
        heat.platforms = {"2gpu", "26cpu_2gpu"};
        heat.policies = {"fifo", "dmdap", "inspirit"};
        heat.baseline = "fifo";
        heat.priority = PriorityKind::Depth;
        std::ostringstream s3;
        guard("bench3", [&] {
            write_bench_csv(s3, run_bench(heat));
            text("bench3.csv", s3.str());
        });
        BenchSpec bad;
        bad.app = "nope";
        bad.sizes = {1};
        bad.platforms = {"homog2", "nope"};
        bad.policies = {"dmda", "nope"};
        std::ostringstream s4;
        guard("bench4", [&] {
            write_bench_csv(s4, run_bench(bad));
            text("bench4.csv", s4.str());
        });
    }
    out << "end\n";
    return 0;
}
