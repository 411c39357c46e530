// test_api.cpp -- behaviour of the drop-in C++ API (include/tbsim/*.hpp) as
// the reference's own suites pin it (proj/tests/test_*.cpp, README goldens).
// GPU_CASEs need a B200 (attributes and simulate run on the device);
// TEST_CASEs are host-side and also run with --cpu-only.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <random>
#include <set>
#include <sstream>

#include "mini_test.hpp"
#include "tbsim/attributes.hpp"
#include "tbsim/bench.hpp"
#include "tbsim/csr_cache.hpp"
#include "tbsim/engine.hpp"
#include "tbsim/platform.hpp"
#include "tbsim/policies.hpp"
#include "tbsim/taskgraph.hpp"
#include "tbsim/text.hpp"
#include "tbsim_b200.h"

using namespace tbsim;

namespace {

const std::vector<std::string> kMixed = {"LAYERK0", "LAYERK1", "LAYERK2", "LAYERK3", "UNIT"};

TaskGraph chain3() {
    TaskGraph g;
    g.tasks = {{0, "UNIT", {}, {}, {}}, {1, "UNIT", {0}, {}, {}}, {2, "UNIT", {1}, {}, {}}};
    return g;
}

TaskGraph diamond() {
    TaskGraph g;
    g.tasks = {{0, "A", {}, {}, {}}, {1, "B", {0}, {}, {}}, {2, "C", {0}, {}, {}}, {3, "D", {1, 2}, {}, {}}};
    return g;
}

// Five independent roots feeding a 2-chain (the reference's chain_wave fixture).
TaskGraph chain_wave() {
    TaskGraph g;
    g.name = "chain_wave";
    for (int i = 0; i < 5; ++i) g.tasks.push_back({i, "UNIT", {}, {}, {}});
    g.tasks.push_back({5, "UNIT", {4}, {}, {}});
    g.tasks.push_back({6, "UNIT", {5}, {}, {}});
    return g;
}

// Random DAG with non-contiguous ids (a construction of its own).
TaskGraph random_dag(uint64_t seed, int n, double p, const std::vector<std::string>& types, bool handles) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> coin(0.0, 1.0);
    TaskGraph g;
    g.name = "rnd";
    auto tid = [](int i) { return TaskId{2000} + 11 * i; };
    auto hid = [](int i) { return HandleId{9000} + 5 * i; };
    for (int i = 0; i < n; ++i) {
        TaskNode t;
        t.id = tid(i);
        t.type = types[i % types.size()];
        for (int j = 0; j < i; ++j)
            if (coin(rng) < p) t.deps.push_back(tid(j));
        if (handles) {
            g.handles.push_back({hid(i), 1000 * (1 + i % 5)});
            t.outputs.push_back(hid(i));
            for (TaskId d : t.deps) t.inputs.push_back(hid(static_cast<int>((d - 2000) / 11)));
        }
        g.tasks.push_back(std::move(t));
    }
    return g;
}

std::vector<int64_t> descendants_bruteforce(const TaskGraph& g) {
    GraphIndex idx = build_index(g);
    std::vector<int64_t> out(g.tasks.size());
    for (size_t s = 0; s < g.tasks.size(); ++s) {
        std::set<size_t> seen;
        std::vector<size_t> stack{s};
        while (!stack.empty()) {
            size_t u = stack.back();
            stack.pop_back();
            for (size_t v : idx.succ[u])
                if (seen.insert(v).second) stack.push_back(v);
        }
        out[s] = static_cast<int64_t>(seen.size());
    }
    return out;
}

struct FakeView final : EngineView {
    const TaskGraph* g = nullptr;
    const Platform* p = nullptr;
    double now_ms = 0.0;
    std::vector<size_t> qlen;
    std::vector<char> busy;
    std::vector<double> free_at;
    std::vector<std::vector<double>> transfer;
    std::vector<std::vector<double>> fraction;
    double now() const override { return now_ms; }
    const TaskGraph& graph() const override { return *g; }
    const Platform& platform() const override { return *p; }
    size_t queue_length(int w) const override { return qlen[w]; }
    bool worker_busy(int w) const override { return busy[w] != 0; }
    double worker_free_at(int w) const override { return free_at[w]; }
    double estimated_transfer_ms(size_t t, int w) const override { return transfer.empty() ? 0.0 : transfer[t][w]; }
    double resident_fraction(size_t t, int n) const override { return fraction.empty() ? 1.0 : fraction[t][n]; }
};

Platform mixed() {
    Platform p;
    p.name = "mixed";
    p.workers = {{0, DeviceKind::Cpu, 0}, {1, DeviceKind::Gpu, 1}};
    p.num_nodes = 2;
    p.bandwidth = {{0.0, 1e6}, {1e6, 0.0}};
    p.costs.set("BOTH", DeviceKind::Cpu, 10.0);
    p.costs.set("BOTH", DeviceKind::Gpu, 2.0);
    p.costs.set("CONLY", DeviceKind::Cpu, 1.0);
    p.costs.set("GONLY", DeviceKind::Gpu, 1.0);
    return p;
}

FakeView idle(const TaskGraph& g, const Platform& p) {
    FakeView v;
    v.g = &g;
    v.p = &p;
    v.qlen.assign(p.workers.size(), 0);
    v.busy.assign(p.workers.size(), 0);
    v.free_at.assign(p.workers.size(), 0.0);
    return v;
}

TaskGraph three(const char* type) {
    TaskGraph g;
    g.tasks = {{0, type, {}, {}, {}}, {1, type, {}, {}, {}}, {2, type, {}, {}, {}}};
    return g;
}

SimTrace run(const TaskGraph& g, const Platform& p, const std::string& pol, const TaskAttributes& a,
             SimOptions o = {}) {
    auto policy = make_policy(pol, a, default_regulator_config(p, g));
    return simulate(g, p, *policy, o);
}

std::string gantt(const TaskGraph& g, const SimTrace& t) {
    std::ostringstream out;
    write_gantt_csv(out, g, t);
    return out.str();
}

// Precedence, one worker at a time, capability (trace_checks.hpp semantics).
std::vector<std::string> audit(const TaskGraph& g, const Platform& p, const SimTrace& t) {
    std::vector<std::string> bad;
    GraphIndex idx = build_index(g);
    for (size_t i = 0; i < g.tasks.size(); ++i) {
        const auto& e = t.per_task[i];
        if (e.worker < 0 || e.worker >= static_cast<int>(p.workers.size())) { bad.push_back("unscheduled"); continue; }
        if (!p.can_run(g.tasks[i].type, p.workers[e.worker])) bad.push_back("incapable");
        if (e.end_ms > t.makespan_ms) bad.push_back("after makespan");
        for (size_t q : idx.pred[i])
            if (e.start_ms < t.per_task[q].end_ms) bad.push_back("precedence");
    }
    if (!t.pops.empty()) {
        std::map<TaskId, double> pop_at;
        for (const auto& r : t.pops) pop_at[r.task] = r.time_ms;
        std::map<int, std::vector<std::pair<double, double>>> busy;
        for (size_t i = 0; i < g.tasks.size(); ++i)
            busy[t.per_task[i].worker].push_back({pop_at[g.tasks[i].id], t.per_task[i].end_ms});
        for (auto& [w, s] : busy) {
            std::sort(s.begin(), s.end());
            for (size_t i = 1; i < s.size(); ++i)
                if (s[i].first < s[i - 1].second) bad.push_back("overlap");
        }
        if (t.nready_samples.size() != t.pushes.size() + t.pops.size()) bad.push_back("nready ledger");
        if (!t.nready_samples.empty() && t.nready_samples.back().second != 0) bad.push_back("nready end");
    }
    return bad;
}

}  // namespace

// ------------------------------------------------------------- task graphs

TEST_CASE("build_index sorts adjacency and rejects bad ids") {
    TaskGraph g;
    g.tasks = {{10, "UNIT", {}, {}, {}}, {20, "UNIT", {30, 10}, {}, {}}, {30, "UNIT", {10}, {}, {}}};
    GraphIndex idx = build_index(g);
    CHECK(idx.task_pos.at(30) == 2);
    CHECK((idx.pred[1] == std::vector<size_t>{0, 2}));
    CHECK((idx.succ[0] == std::vector<size_t>{1, 2}));
    TaskGraph dup;
    dup.tasks = {{1, "UNIT", {}, {}, {}}, {1, "UNIT", {}, {}, {}}};
    CHECK_THROWS_WITH_AS(build_index(dup), "duplicate task id 1", std::invalid_argument);
    TaskGraph dangling;
    dangling.tasks = {{1, "UNIT", {7}, {}, {}}};
    CHECK_THROWS_WITH_AS(build_index(dangling), "task 1 depends on unknown task 7", std::invalid_argument);
}

TEST_CASE("validate names structural problems and a cycle") {
    CHECK(validate(build_cholesky_dag(4, 64)).empty());
    TaskGraph g;
    g.handles = {{1, 0}};
    g.tasks = {{0, "UNIT", {0}, {5}, {}}, {1, "UNIT", {9}, {}, {6}}};
    auto v = validate(g);
    std::string all;
    for (const auto& x : v) all += x.message + "|";
    CHECK(all.find("handle 1 has non-positive bytes") != std::string::npos);
    CHECK(all.find("task 0 depends on itself") != std::string::npos);
    CHECK(all.find("task 1 depends on unknown task 9") != std::string::npos);
    CHECK(all.find("task 0 reads unknown handle 5") != std::string::npos);
    CHECK(all.find("task 1 writes unknown handle 6") != std::string::npos);
    TaskGraph cyc;
    cyc.tasks = {{1, "UNIT", {3}, {}, {}}, {2, "UNIT", {1}, {}, {}}, {3, "UNIT", {2}, {}, {}}};
    auto c = validate(cyc);
    REQUIRE(c.size() == 1);
    CHECK(c[0].message.find("dependency cycle:") == 0);
}

TEST_CASE("generated factorizations serialize their writers") {
    for (int n = 1; n <= 6; ++n) {
        CHECK(check_writer_chains(build_cholesky_dag(n, 64)).empty());
        CHECK(check_writer_chains(build_lu_dag(n, 64)).empty());
    }
}

TEST_CASE("generators produce the closed-form task mixes") {
    for (int n = 1; n <= 8; ++n) {
        std::map<std::string, int64_t> c, want;
        for (const auto& t : build_cholesky_dag(n, 4096).tasks) c[t.type]++;
        for (int k = 0; k < n; ++k) {
            want["POTRF"]++;
            want["TRSM"] += n - k - 1;
            want["SYRK"] += n - k - 1;
            want["GEMM"] += (n - k - 1) * (n - k - 2) / 2;
        }
        for (auto it = want.begin(); it != want.end();) it = it->second == 0 ? want.erase(it) : std::next(it);
        CHECK(c == want);
        CHECK(build_cholesky_dag(n, 4096).handles.size() == static_cast<size_t>(n * (n + 1) / 2));
        CHECK(build_lu_dag(n, 4096).handles.size() == static_cast<size_t>(n * n));
    }
    CHECK(build_cholesky_dag(8, 64).name == "cholesky_n8");
    CHECK_THROWS_AS(build_lu_dag(0, 64), std::invalid_argument);
    auto heat = build_stencil_dag(3, 2, 64);
    CHECK(heat.tasks.size() == 18);
    CHECK(heat.tasks[9].deps.size() == 3);   // corner at t=2: itself + 2 neighbours
    CHECK(heat.tasks[13].deps.size() == 5);  // centre
}

TEST_CASE("layered generator is reproducible and layer-structured") {
    auto a = generate_layered_dag(200, 7, 0.1, 42), b = generate_layered_dag(200, 7, 0.1, 42);
    CHECK(a == b);
    CHECK(a.name == "autogen_n200_l7_p0.1_s42");
    CHECK(!(a == generate_layered_dag(200, 7, 0.1, 43)));
    for (const auto& t : a.tasks) {
        if (t.id % 7 == 0) CHECK(t.deps.empty());
        for (TaskId d : t.deps) CHECK(d % 7 == t.id % 7 - 1);
        if (t.id % 7) CHECK(!t.deps.empty());
    }
    CHECK_THROWS_AS(generate_layered_dag(3, 5, 0.1, 0), std::invalid_argument);
}

TEST_CASE("topological_order respects dependencies") {
    auto g = random_dag(5, 60, 0.1, kMixed, false);
    auto order = topological_order(g);
    REQUIRE(order.size() == g.tasks.size());
    std::vector<size_t> at(order.size());
    for (size_t i = 0; i < order.size(); ++i) at[order[i]] = i;
    GraphIndex idx = build_index(g);
    for (size_t v = 0; v < g.tasks.size(); ++v)
        for (size_t p : idx.pred[v]) CHECK(at[p] < at[v]);
    CHECK(edge_count(chain_wave()) == 2);
}

TEST_CASE("dag files round-trip and the loader names the offending line") {
    auto g = build_cholesky_dag(3, 128);
    std::ostringstream first;
    save_dag(g, first);
    std::istringstream in(first.str());
    TaskGraph back = load_dag(in);
    CHECK(back == g);
    std::ostringstream second;
    save_dag(back, second);
    CHECK(second.str() == first.str());
    std::ostringstream cw;
    save_dag(chain_wave(), cw);
    CHECK(cw.str() ==
          "{\"kind\":\"meta\",\"name\":\"chain_wave\",\"version\":1}\n"
          "{\"kind\":\"task\",\"id\":0,\"type\":\"UNIT\",\"deps\":[],\"inputs\":[],\"outputs\":[]}\n"
          "{\"kind\":\"task\",\"id\":1,\"type\":\"UNIT\",\"deps\":[],\"inputs\":[],\"outputs\":[]}\n"
          "{\"kind\":\"task\",\"id\":2,\"type\":\"UNIT\",\"deps\":[],\"inputs\":[],\"outputs\":[]}\n"
          "{\"kind\":\"task\",\"id\":3,\"type\":\"UNIT\",\"deps\":[],\"inputs\":[],\"outputs\":[]}\n"
          "{\"kind\":\"task\",\"id\":4,\"type\":\"UNIT\",\"deps\":[],\"inputs\":[],\"outputs\":[]}\n"
          "{\"kind\":\"task\",\"id\":5,\"type\":\"UNIT\",\"deps\":[4],\"inputs\":[],\"outputs\":[]}\n"
          "{\"kind\":\"task\",\"id\":6,\"type\":\"UNIT\",\"deps\":[5],\"inputs\":[],\"outputs\":[]}\n");
    auto load = [](const std::string& text) {
        std::istringstream s(text);
        return load_dag(s);
    };
    const std::string meta = R"({"kind":"meta","name":"x","version":1})";
    CHECK_THROWS_WITH_AS(load("not json\n"), "line 1", std::runtime_error);
    CHECK_THROWS_WITH_AS(load(R"({"kind":"task","id":0,"type":"UNIT","deps":[],"inputs":[],"outputs":[]})" "\n"),
                         "record before meta", std::runtime_error);
    CHECK_THROWS_WITH_AS(load(meta + "\n" + meta + "\n"), "duplicate meta", std::runtime_error);
    CHECK_THROWS_WITH_AS(load(R"({"kind":"meta","name":"x","version":2})" "\n"), "unsupported version",
                         std::runtime_error);
    CHECK_THROWS_WITH_AS(load(meta + "\n" + R"({"kind":"widget"})" "\n"), "unknown record kind", std::runtime_error);
    CHECK_THROWS_WITH_AS(load(meta + "\n" + R"({"kind":"task","id":0})" "\n"), "missing field", std::runtime_error);
    CHECK_THROWS_WITH_AS(load(meta + "\n\n"), "empty line", std::runtime_error);
    CHECK_THROWS_WITH_AS(load(""), "missing meta", std::runtime_error);
    CHECK_THROWS_WITH_AS(load(meta + "\n" + R"({"kind":"task","id":0,"type":"UNIT","deps":[9],"inputs":[],"outputs":[]})" "\n"),
                         "depends on unknown task 9", std::runtime_error);
    auto dir = std::filesystem::temp_directory_path() / "tbsim_cpp_test";
    std::filesystem::create_directories(dir);
    auto layered = generate_layered_dag(40, 5, 0.2, 3);
    save_dag_file(layered, (dir / "g.dag").string());
    CHECK(load_dag_file((dir / "g.dag").string()) == layered);
    CHECK_THROWS_WITH_AS(load_dag_file((dir / "absent.dag").string()), "cannot open", std::runtime_error);
}

TEST_CASE("dag files compile into a binary CSR cache") {
    auto dir = std::filesystem::temp_directory_path() / "tbsim_cpp_test";
    std::filesystem::create_directories(dir);
    auto a = build_lu_dag(4, 640), b = generate_layered_dag(60, 6, 0.1, 9);
    save_dag_file(a, (dir / "a.dag").string());
    save_dag_file(b, (dir / "b.dag").string());
    const std::string cache = (dir / "ab.csr").string();
    compile_dag_cache({(dir / "a.dag").string(), (dir / "b.dag").string()}, cache);
    tbsim_hostbatch* hb = nullptr;
    CHECK(tbsim_hostbatch_load(cache.c_str(), &hb) == TBSIM_OK);
    tbsim_batch_desc d{};
    CHECK(tbsim_hostbatch_desc(hb, &d) == TBSIM_OK);
    CHECK(d.n_graphs == 2);
    CHECK(d.task_base[1] == static_cast<int64_t>(a.tasks.size()));
    CHECK(d.task_base[2] == static_cast<int64_t>(a.tasks.size() + b.tasks.size()));
    CHECK(d.edge_base[2] == static_cast<int64_t>(edge_count(a) + edge_count(b)));
    // the second graph's first task with deps: positions of its ids
    int64_t deps = 0;
    for (int64_t t = d.task_base[1]; t < d.task_base[2]; ++t) deps += d.dep_off[t + 2] - d.dep_off[t + 1];
    CHECK(deps == static_cast<int64_t>(edge_count(b)));
    CHECK(std::string(d.type_names[d.type[0]]) == a.tasks[0].type);
    tbsim_hostbatch_free(hb);
    CHECK_THROWS_WITH_AS(compile_dag_cache({(dir / "absent.dag").string()}, cache), "cannot open",
                         std::runtime_error);
}

// ---------------------------------------------------------------- platform

TEST_CASE("cost table, presets, transfer and exec times") {
    CostTable t;
    t.set("X", DeviceKind::Gpu, 2.0);
    CHECK(t.gpu_ms("X") == 2.0);
    CHECK(t.mean_ms("X") == 2.0);
    t.set("X", DeviceKind::Cpu, 6.0);
    CHECK(t.mean_ms("X") == 4.0);
    CHECK_THROWS_WITH_AS(t.get("Y", DeviceKind::Cpu), "no cpu cost entry for task type Y", std::runtime_error);
    CHECK_THROWS_AS(t.set("Z", DeviceKind::Cpu, 0.0), std::invalid_argument);
    CostTable d = default_cost_table();
    CHECK(d.get("GEMM", DeviceKind::Cpu) / d.get("GEMM", DeviceKind::Gpu) == 10.0);
    CHECK(d.get("POTRF", DeviceKind::Cpu) == 6.0);
    Platform p = make_preset("26cpu_2gpu");
    CHECK(p.workers.size() == 28);
    CHECK(p.num_nodes == 3);
    CHECK(p.workers[26].kind == DeviceKind::Gpu && p.workers[26].memory_node == 1);
    CHECK(p.transfer_time_ms(12'000'000, 0, 1) == 0.01 + 1.0);
    CHECK(p.transfer_time_ms(24'000'000, 1, 2) == 0.01 + 1.0);
    CHECK(p.transfer_time_ms(5, 1, 1) == 0.0);
    CHECK(make_preset("homog2").num_nodes == 1);
    CHECK_THROWS_WITH_AS(make_preset("nope"), "unknown platform preset", std::runtime_error);
    Platform m = mixed();
    CHECK_THROWS_WITH_AS(m.exec_time_ms("GONLY", m.workers[0]), "cannot run on cpu worker 0", std::runtime_error);
    CHECK_THROWS_WITH_AS(m.exec_time_ms("NOPE", m.workers[0]), "no cost entry for task type NOPE", std::runtime_error);
}

TEST_CASE("platform files load and are checked") {
    auto dir = std::filesystem::temp_directory_path() / "tbsim_cpp_test";
    std::filesystem::create_directories(dir);
    auto write = [&](const std::string& name, const std::string& text) {
        std::ofstream(dir / name) << text;
        return (dir / name).string();
    };
    Platform p = load_platform_file(write("ok.json", R"({
      "workers": [{"id": 0, "kind": "cpu", "memory_node": 0}, {"id": 1, "kind": "gpu", "memory_node": 1}],
      "costs": {"UNIT": {"cpu": 2.0, "gpu": 1.0}, "GONLY": {"gpu": 3}},
      "bandwidth": [[0, 1000], [1000, 0]], "latency_ms": 1.0})"));
    CHECK(p.workers.size() == 2 && p.num_nodes == 2);
    CHECK(!p.costs.covers("GONLY", DeviceKind::Cpu));
    CHECK(p.transfer_time_ms(1'000'000, 0, 1) == 1001.0);
    CHECK_THROWS_WITH_AS(load_platform_file(write("b1.json", "{]")), "bad JSON", std::runtime_error);
    CHECK_THROWS_WITH_AS(load_platform_file(write("b2.json", R"({"costs":{},"bandwidth":[[0]]})")),
                         "missing \"workers\"", std::runtime_error);
    CHECK_THROWS_WITH_AS(load_platform_file(write("b3.json",
        R"({"workers":[{"id":0,"kind":"tpu","memory_node":0}],"costs":{},"bandwidth":[[0]]})")),
                         "unknown device kind", std::runtime_error);
    CHECK_THROWS_WITH_AS(load_platform_file(write("b4.json",
        R"({"workers":[{"id":1,"kind":"cpu","memory_node":0}],"costs":{},"bandwidth":[[0]]})")),
                         "dense", std::runtime_error);
    CHECK_THROWS_WITH_AS(load_platform_file(write("b5.json",
        R"({"workers":[{"id":0,"kind":"cpu","memory_node":0},{"id":1,"kind":"gpu","memory_node":1}],"costs":{},"bandwidth":[[0,10],[20,0]]})")),
                         "symmetric", std::runtime_error);
    CHECK(resolve_platform("homog2").workers.size() == 2);
    CHECK_THROWS_WITH_AS(resolve_platform("no_such_thing"), "cannot open", std::runtime_error);
    CostTable t;
    t.set("A", DeviceKind::Gpu, 1.0);
    t.set("B", DeviceKind::Gpu, 2.0);
    t.set("C", DeviceKind::Gpu, 8.0);
    TaskGraph g;
    g.tasks = {{0, "A", {}, {}, {}}, {1, "B", {}, {}, {}}};
    CHECK(median_gpu_time_ms(g, t) == 1.0);
    g.tasks.push_back({2, "C", {}, {}, {}});
    CHECK(median_gpu_time_ms(g, t) == 2.0);
    CHECK_THROWS_AS(median_gpu_time_ms(TaskGraph{}, t), std::runtime_error);
}

// ----------------------------------------------------- push / pop / regulator

TEST_CASE("push rules over an EngineView") {
    Platform h = make_preset("homog2");
    TaskGraph u = three("UNIT");
    FakeView v = idle(u, h);
    CHECK(push_fifo(0, v) == 0);
    v.qlen = {2, 0};
    CHECK(push_fifo(0, v) == 1);
    v.qlen = {1, 1};
    v.busy = {0, 1};
    CHECK(push_fifo(0, v) == 0);
    Platform m = mixed();
    TaskGraph b = three("BOTH");
    FakeView w = idle(b, m);
    w.free_at = {0.0, 5.0};
    CHECK(push_dm(0, w) == 1);
    w.free_at = {0.0, 8.0};
    CHECK(push_dm(0, w) == 0);  // exact tie: lowest id
    w.now_ms = 20.0;
    w.free_at = {0.0, 19.0};
    CHECK(push_dm(0, w) == 1);
    w.now_ms = 0.0;
    w.free_at = {0.0, 0.0};
    w.transfer = {{0.0, 30.0}, {0.0, 1.0}, {0.0, 8.0}};
    CHECK(push_dmda(0, w) == 0);
    CHECK(push_dmda(1, w) == 1);
    CHECK(push_dmda(2, w) == 0);
    TaskGraph nowhere;
    nowhere.tasks = {{0, "NOWHERE", {}, {}, {}}};
    FakeView x = idle(nowhere, m);
    CHECK_THROWS_WITH_AS(push_fifo(0, x), "no worker can run task type NOWHERE", std::runtime_error);
}

TEST_CASE("pop rules and adaptive modes") {
    std::vector<QueueEntry> q = {{0, 5}, {1, 2}, {2, 9}};
    CHECK(pop_fifo(q) == 1);
    CHECK_THROWS_AS(pop_fifo({}), std::logic_error);
    TaskAttributes a;
    a.static_priority = {3, 7, 7};
    std::vector<QueueEntry> q2 = {{0, 1}, {1, 2}, {2, 3}};
    CHECK(pop_priority(q2, a) == 1);
    Platform m = mixed();
    TaskGraph b = three("BOTH");
    FakeView v = idle(b, m);
    a.ability = {5, 9, 9};
    a.efficiency = {4, 4, 1};
    a.static_priority = {2, 8, 100};
    std::vector<QueueEntry> q3 = {{0, 1}, {1, 2}};
    CHECK(pop_adaptive(PopMode::HighAbility, 0, q3, a, v) == 1);
    CHECK(pop_adaptive(PopMode::HighEfficiency, 0, q3, a, v) == 1);
    std::vector<QueueEntry> q4 = {{1, 2}, {2, 3}};
    CHECK(pop_adaptive(PopMode::HighAbility, 0, q4, a, v) == 1);
    a.efficiency = {1, 99, 50};
    a.static_priority = {0, 0, 0};
    v.fraction = {{0.0, 1.0}, {0.0, 0.5}, {0.0, 1.0}};
    CHECK(pop_adaptive(PopMode::HighEfficiencyLocality, 1, q3, a, v) == 0);
    CHECK(pop_adaptive(PopMode::HighEfficiencyLocality, 0, q3, a, v) == 1);
    CHECK(std::string(to_string(PopMode::HighEfficiencyLocality)) == "high_efficiency_locality");
}

TEST_CASE("policy objects and the inspirit regulator") {
    TaskAttributes a;
    a.ability = {9, 1, 1};
    a.efficiency = {1, 9, 1};
    a.static_priority = {0, 0, 0};
    CHECK((policy_names() == std::vector<std::string>{"fifo", "dm", "dmda", "dmdap", "inspirit"}));
    for (const auto& n : policy_names()) CHECK(make_policy(n, a)->name() == n);
    CHECK_THROWS_WITH_AS(make_policy("bogus", a), "unknown policy \"bogus\"", std::runtime_error);
    RegulatorConfig cfg;
    cfg.task_window = 1;
    cfg.s_inc = 1;
    cfg.k_inc = 0.5;
    cfg.dec_step = 1000;
    auto pol = make_policy("inspirit", a, cfg);
    const RegulatorState* st = regulator_state(*pol);
    const auto* counts = pop_mode_counts(*pol);
    REQUIRE(st && counts);
    Platform m = mixed();
    TaskGraph b = three("BOTH");
    FakeView v = idle(b, m);
    std::vector<QueueEntry> q = {{0, 1}, {1, 2}};
    CHECK(pol->select_entry(0, q, v) == 1);
    pol->on_queue_event(0.0, 4);
    pol->on_queue_event(1.0, 8);
    CHECK(st->mode == PopMode::HighAbility);
    CHECK(pol->select_entry(0, q, v) == 0);
    CHECK((*counts)[0] == 1 && (*counts)[1] == 1);
    auto dmda = make_policy("dmda", a);
    CHECK(regulator_state(*dmda) == nullptr);
}

TEST_CASE("regulator slope fit and drain bands") {
    using S = std::deque<std::pair<double, std::int64_t>>;
    CHECK(calculate_k(S{}) == 0.0);
    CHECK_NEAR(calculate_k(S{{0.0, 0}, {1.0, 2}, {2.0, 4}}), 2.0, 1e-12);
    CHECK(calculate_k(S{{5.0, 1}, {5.0, 9}}) == 0.0);
    RegulatorConfig cfg;
    cfg.task_window = 1;
    cfg.s_inc = 1000;
    cfg.dec_step = 2;
    cfg.s_dec = 5;
    cfg.c = 1;
    RegulatorState st;
    st.peak = st.prev_nready = st.last_trigger_nready = 20;
    const std::vector<std::tuple<int64_t, PopMode, int64_t>> steps = {
        {18, PopMode::HighEfficiency, 1}, {17, PopMode::HighAbility, 1}, {13, PopMode::HighAbility, 1},
        {11, PopMode::HighEfficiencyLocality, 1}, {10, PopMode::HighEfficiencyLocality, 2},
        {12, PopMode::HighAbility, 2}, {5, PopMode::HighEfficiencyLocality, 3}};
    double t = 1.0;
    for (const auto& [cur, mode, count] : steps) {
        regulator_step(st, cfg, cur, t);
        t += 1.0;
        CHECK(st.mode == mode);
        CHECK(st.s_dec_count == count);
    }
    auto g = build_cholesky_dag(8, 64);
    RegulatorConfig d = default_regulator_config(make_preset("26cpu_2gpu"), g);
    CHECK(d.task_window == 7 && d.s_inc == 28 && d.k_inc == 28.0 && d.s_dec == 7 && d.c == 4 && d.dec_step == 7);
}

TEST_CASE("trace queries and number formatting") {
    SimTrace t;
    t.makespan_ms = 10.0;
    t.nready_samples = {{0.0, 1}, {2.0, 3}, {5.0, 0}};
    CHECK(nready_at(t, 1.999) == 1);
    CHECK(nready_at(t, 2.0) == 3);
    CHECK(nready_at(t, 10.0) == 0);
    CHECK_THROWS_AS(nready_at(t, 10.001), std::out_of_range);
    SimTrace h;
    h.pushes = {{0.0, 0}, {1.5, 1}, {7.2, 2}, {2.0, 3}};
    h.pops = {{1.6, 0, 0}, {7.9, 1, 0}};
    auto rows = window_histogram(h, 2.0);
    REQUIRE(rows.size() == 4);
    CHECK(rows[0].pushes == 2 && rows[0].pops == 1 && rows[1].pushes == 1 && rows[3].pops == 1);
    CHECK_THROWS_AS(window_histogram(h, 0.0), std::invalid_argument);
    CHECK(fmt_ms(3.0) == "3");
    CHECK(fmt_ms(1001.01) == "1001.01");
    CHECK(fmt_ms(-0.0) == "0");
    CHECK(fmt_ratio(1.0) == "1.000");
}

// ------------------------------------------------------- device: attributes

GPU_CASE("ability on hand graphs and against brute force") {
    CHECK((compute_inspiring_ability(chain3()) == std::vector<int64_t>{2, 1, 0}));
    CHECK((compute_inspiring_ability(diamond()) == std::vector<int64_t>{3, 1, 1, 0}));
    CHECK(compute_inspiring_ability(TaskGraph{}).empty());
    for (uint64_t s = 1; s <= 20; ++s) {
        auto g = random_dag(s, 20 + 9 * static_cast<int>(s), 0.06, kMixed, false);
        CHECK(compute_inspiring_ability(g) == descendants_bruteforce(g));
        CHECK(compute_inspiring_ability_serial(g) == compute_inspiring_ability(g));
    }
}

GPU_CASE("efficiency windows, worst paths and identities") {
    CostTable unit;
    unit.set("UNIT", DeviceKind::Gpu, 1.0);
    CHECK((compute_inspiring_efficiency(chain3(), unit, 0.5) == std::vector<int64_t>{0, 0, 0}));
    CHECK((compute_inspiring_efficiency(chain3(), unit, 1.0) == std::vector<int64_t>{1, 1, 0}));
    CHECK((compute_inspiring_efficiency(chain3(), unit, 2.0) == std::vector<int64_t>{2, 1, 0}));
    CHECK_THROWS_AS(compute_inspiring_efficiency(chain3(), unit, -1.0), std::invalid_argument);
    CostTable t;
    t.set("A", DeviceKind::Gpu, 1.0);
    t.set("B", DeviceKind::Gpu, 2.0);
    t.set("C", DeviceKind::Gpu, 3.0);
    t.set("D", DeviceKind::Gpu, 1.0);
    CHECK((compute_inspiring_efficiency(diamond(), t, 3.0) == std::vector<int64_t>{2, 1, 1, 0}));
    CHECK((compute_inspiring_efficiency(diamond(), t, 4.0) == std::vector<int64_t>{3, 1, 1, 0}));
    CostTable costs = default_cost_table();
    for (uint64_t s = 30; s < 36; ++s) {
        auto g = random_dag(s, 50, 0.08, kMixed, false);
        auto ab = compute_inspiring_ability(g);
        double total = 0.0, mn = 1e300;
        for (const auto& task : g.tasks) {
            total += costs.gpu_ms(task.type);
            mn = std::min(mn, costs.gpu_ms(task.type));
        }
        auto mid = compute_inspiring_efficiency(g, costs, total / 8.0);
        for (size_t i = 0; i < g.tasks.size(); ++i) CHECK(mid[i] <= ab[i]);
        CHECK(compute_inspiring_efficiency(g, costs, total) == ab);
        CHECK(compute_inspiring_efficiency(g, costs, mn * 0.5) == std::vector<int64_t>(g.tasks.size(), 0));
    }
}

GPU_CASE("calibration, priorities and assembly") {
    CostTable costs = default_cost_table();
    auto r = calibrate_unit_time(build_cholesky_dag(6, 64), costs);
    CHECK(r.evaluations == 11);
    CHECK(r.w0_ms == 2.0 * median_gpu_time_ms(build_cholesky_dag(6, 64), costs));
    CHECK(r.best_score >= r.w0_score && r.best_score >= 1);
    TaskGraph single;
    single.tasks = {{0, "UNIT", {}, {}, {}}};
    auto s = calibrate_unit_time(single, costs);
    CHECK(s.w0_ms == 2.0 && s.best_score == 1 && s.unit_time_ms == 2.0 / 16.0);
    auto cw = calibrate_unit_time(chain_wave(), costs);
    CHECK(cw.unit_time_ms == 1.0 && cw.best_score == 3);
    CHECK((upward_rank_priority(chain3(), costs) == std::vector<int64_t>{3000, 2000, 1000}));
    CHECK((depth_priority(diamond()) == std::vector<int64_t>{2, 1, 1, 0}));
    auto g = build_cholesky_dag(4, 64);
    auto a = compute_attributes(g, costs, PriorityKind::UpwardRank);
    CHECK(a.ability == compute_inspiring_ability(g));
    CHECK(a.efficiency == compute_inspiring_efficiency(g, costs, a.unit_time_ms));
    CHECK(a.static_priority == upward_rank_priority(g, costs));
    CHECK(compute_attributes(g, costs, PriorityKind::Depth).static_priority == depth_priority(g));
    CHECK(compute_attributes(g, costs, PriorityKind::Zero).static_priority == std::vector<int64_t>(g.tasks.size(), 0));
    std::ostringstream csv;
    write_attributes_csv(csv, chain3(), compute_attributes(chain3(), costs, PriorityKind::UpwardRank));
    CHECK(csv.str() == "task_id,type,layer,ability,efficiency,static_priority\n0,UNIT,0,2,2,3000\n"
                       "1,UNIT,1,1,1,2000\n2,UNIT,2,0,0,1000\n");
    CHECK((topological_layers(diamond()) == std::vector<int>{0, 1, 1, 2}));
    TaskGraph cyc;
    cyc.tasks = {{0, "UNIT", {1}, {}, {}}, {1, "UNIT", {0}, {}, {}}};
    CHECK_THROWS_WITH_AS(topological_layers(cyc), "graph has a dependency cycle", std::runtime_error);
}

// ----------------------------------------------------------- device: engine

GPU_CASE("single task, chain and the chain_wave optimum") {
    Platform one;
    one.name = "one_cpu";
    one.workers = {{0, DeviceKind::Cpu, 0}};
    one.costs.set("UNIT", DeviceKind::Cpu, 5.0);
    one.costs.set("UNIT", DeviceKind::Gpu, 5.0);
    TaskGraph g;
    g.tasks = {{0, "UNIT", {}, {}, {}}};
    TaskAttributes none;
    SimTrace t = run(g, one, "fifo", none);
    CHECK(t.makespan_ms == 5.0 && t.per_task[0].end_ms == 5.0 && t.pushes.size() == 1 && t.pops.size() == 1);
    std::ostringstream nr;
    write_nready_csv(nr, run(g, make_preset("homog2"), "fifo", none));
    CHECK(nr.str() == "time_ms,nready\n0,1\n0,0\n");
    for (const char* p : {"fifo", "dm", "dmda"}) {
        SimTrace c = run(chain3(), make_preset("homog2"), p, none);
        CHECK(c.makespan_ms == 3.0);
        CHECK(c.per_task[2].start_ms == c.per_task[1].end_ms);
    }
    Platform h = make_preset("homog2");
    TaskGraph cw = chain_wave();
    CHECK(run(cw, h, "fifo", none).makespan_ms == 5.0);
    TaskAttributes depth = compute_attributes(cw, h.costs, PriorityKind::Depth);
    CHECK(run(cw, h, "dmdap", depth).makespan_ms == 4.0);
    TaskAttributes full = compute_attributes(cw, h.costs, PriorityKind::UpwardRank);
    CHECK(run(cw, h, "inspirit", full).makespan_ms == 4.0);
}

GPU_CASE("every policy yields an audited schedule") {
    for (const char* preset : {"homog2", "26cpu_2gpu", "2gpu"}) {
        Platform p = make_preset(preset);
        for (uint64_t s = 1; s <= 4; ++s) {
            auto g = random_dag(s * 101, 60, 0.08, kMixed, true);
            TaskAttributes a = compute_attributes(g, p.costs, PriorityKind::UpwardRank);
            for (const auto& pol : policy_names()) {
                SimTrace t = run(g, p, pol, a);
                auto bad = audit(g, p, t);
                CHECK(bad.empty());
                CHECK(t.makespan_ms > 0.0);
            }
        }
    }
}

GPU_CASE("dm equals dmda without transfers; dmdap(zero) equals dmda") {
    Platform p = make_preset("26cpu_2gpu");
    TaskAttributes none;
    for (uint64_t s = 60; s < 66; ++s) {
        auto g = random_dag(s, 50, 0.08, kMixed, false);
        CHECK(gantt(g, run(g, p, "dm", none)) == gantt(g, run(g, p, "dmda", none)));
        auto gh = random_dag(s, 50, 0.08, kMixed, true);
        TaskAttributes zero = compute_attributes(gh, p.costs, PriorityKind::Zero);
        CHECK(gantt(gh, run(gh, p, "dmda", zero)) == gantt(gh, run(gh, p, "dmdap", zero)));
    }
}

GPU_CASE("transfers fetch from the fastest copy") {
    Platform p;
    p.name = "fast_link";
    p.workers = {{0, DeviceKind::Cpu, 0}, {1, DeviceKind::Gpu, 1}, {2, DeviceKind::Gpu, 2}};
    p.num_nodes = 3;
    p.bandwidth = {{0.0, 10.0, 10.0}, {10.0, 0.0, 1000.0}, {10.0, 1000.0, 0.0}};
    p.costs.set("ZLONG", DeviceKind::Gpu, 10.0);
    p.costs.set("AQUICK", DeviceKind::Gpu, 1.0);
    p.costs.set("WBLOCK", DeviceKind::Gpu, 100.0);
    p.costs.set("BREAD", DeviceKind::Gpu, 1.0);
    TaskGraph g;
    g.handles = {{0, 1000}};
    g.tasks = {{0, "ZLONG", {}, {}, {}}, {1, "AQUICK", {}, {}, {0}}, {2, "WBLOCK", {1}, {}, {}},
               {3, "BREAD", {0, 1}, {0}, {}}};
    TaskAttributes none;
    auto pol = make_policy("dmda", none);
    SimTrace t = simulate(g, p, *pol);
    CHECK(t.per_task[0].worker == 1 && t.per_task[1].worker == 2 && t.per_task[2].worker == 2);
    CHECK(t.per_task[3].worker == 1);
    CHECK(t.per_task[3].start_ms == 11.0 && t.per_task[3].end_ms == 12.0);
}

GPU_CASE("determinism, trace switch, policy ordering and failures") {
    Platform p = make_preset("26cpu_2gpu");
    auto g = build_cholesky_dag(6, 960 * 960 * 4);
    TaskAttributes a = compute_attributes(g, p.costs, PriorityKind::UpwardRank);
    SimTrace x = run(g, p, "inspirit", a), y = run(g, p, "inspirit", a);
    CHECK(gantt(g, x) == gantt(g, y));
    auto c8 = build_cholesky_dag(8, 960 * 960 * 4);
    TaskAttributes a8 = compute_attributes(c8, p.costs, PriorityKind::UpwardRank);
    CHECK(run(c8, p, "fifo", a8).makespan_ms > run(c8, p, "dmda", a8).makespan_ms);
    auto lu = build_lu_dag(4, 160 * 160 * 4);
    TaskAttributes none;
    SimOptions quiet;
    quiet.record_trace = false;
    SimTrace full = run(lu, p, "dmda", none), bare = run(lu, p, "dmda", none, quiet);
    CHECK(bare.pushes.empty() && bare.nready_samples.empty());
    CHECK(gantt(lu, bare) == gantt(lu, full));
    TaskGraph dead;
    dead.tasks = {{0, "UNIT", {1}, {}, {}}, {1, "UNIT", {0}, {}, {}}};
    auto fifo = make_policy("fifo", none);
    CHECK_THROWS_WITH_AS(simulate(dead, make_preset("homog2"), *fifo), "simulation stuck with 2 tasks unfinished: 0 1",
                         std::runtime_error);
    TaskGraph gonly;
    gonly.tasks = {{0, "GONLY_TYPE", {}, {}, {}}};
    auto dmda = make_policy("dmda", none);
    CHECK_THROWS_WITH_AS(simulate(gonly, make_preset("homog2"), *dmda), "no worker can run task type GONLY_TYPE",
                         std::runtime_error);
    struct Custom final : Policy {
        std::string n = "custom";
        const std::string& name() const override { return n; }
        int select_worker(size_t, const EngineView&) override { return 0; }
        size_t select_entry(int, const std::vector<QueueEntry>&, const EngineView&) override { return 0; }
    } custom;
    CHECK_THROWS_AS(simulate(chain3(), make_preset("homog2"), custom), std::runtime_error);
    // a task reading an undeclared handle: the attribute functions never
    // look at handles; the engine fails on it (handle_pos.at(),
    // src/engine.cpp:68,108) with std::out_of_range
    TaskGraph stray;
    stray.handles = {{7, 4096}};
    stray.tasks = {{0, "UNIT", {}, {7}, {7}}, {1, "UNIT", {0}, {99}, {}}};
    TaskAttributes sa = compute_attributes(stray, make_preset("homog2").costs, PriorityKind::UpwardRank);
    CHECK(sa.ability.size() == 2 && sa.ability[0] == 1);
    CHECK_THROWS_AS(simulate(stray, make_preset("homog2"), *dmda), std::out_of_range);
}

GPU_CASE("README goldens through run_bench") {
    BenchSpec spec;
    spec.app = "cholesky";
    spec.sizes = {8, 12};
    spec.platforms = {"26cpu_2gpu"};
    spec.policies = {"dmda", "inspirit"};
    BenchReport r = run_bench(spec);
    std::ostringstream out;
    write_bench_csv(out, r);
    CHECK(out.str() ==
          "app,size,platform,policy,makespan_ms,speedup_vs_baseline,status\n"
          "cholesky,8,26cpu_2gpu,dmda,58.2484,1.000,ok\n"
          "cholesky,8,26cpu_2gpu,inspirit,54.22,1.074,ok\n"
          "cholesky,12,26cpu_2gpu,dmda,115.162,1.000,ok\n"
          "cholesky,12,26cpu_2gpu,inspirit,112.9496,1.020,ok\n");
    Platform p = make_preset("26cpu_2gpu");
    auto g = build_cholesky_dag(8, 960 * 960 * 4);
    auto a = compute_attributes(g, p.costs, PriorityKind::UpwardRank);
    auto pol = make_policy("inspirit", a, default_regulator_config(p, g));
    simulate(g, p, *pol);
    CHECK((*pop_mode_counts(*pol))[1] == 120);
}

GPU_CASE("run_bench rows, baseline, error rows and overrides") {
    BenchSpec spec;
    spec.app = "autogen";
    spec.sizes = {120, 60};
    spec.platforms = {"26cpu_2gpu", "2gpu", "bogus_platform"};
    spec.policies = {"inspirit", "fifo"};
    BenchReport r = run_bench(spec);
    CHECK(r.rows.size() == 2 * 3 * 3);
    for (size_t i = 1; i < r.rows.size(); ++i)
        CHECK(std::tie(r.rows[i - 1].size, r.rows[i - 1].platform, r.rows[i - 1].policy) <
              std::tie(r.rows[i].size, r.rows[i].platform, r.rows[i].policy));
    for (const auto& row : r.rows) {
        if (row.platform == "bogus_platform") CHECK(!row.ok && row.error.find("cannot open") != std::string::npos);
        else CHECK(row.ok && row.makespan_ms > 0.0);
        if (row.ok && row.policy == "dmda") CHECK(row.speedup == 1.0);
    }
    // a bench cell equals a direct simulation
    auto g = generate_layered_dag(120, 10, 0.05, 0);
    Platform p = make_preset("26cpu_2gpu");
    auto a = compute_attributes(g, p.costs, PriorityKind::UpwardRank);
    const double direct = run(g, p, "inspirit", a).makespan_ms;
    for (const auto& row : r.rows)
        if (row.size == 120 && row.platform == "26cpu_2gpu" && row.policy == "inspirit") CHECK(row.makespan_ms == direct);
    BenchSpec o = spec;
    o.platforms = {"26cpu_2gpu"};
    o.regulator.task_window = 1;
    o.regulator.k_inc = 1e9;
    BenchReport ro = run_bench(o);
    CHECK(ro.rows.size() == 2 * 3);
}

// ----------------------------------------- acceptance gate (tests/acceptance.cpp)

GPU_CASE("acceptance c7: INSPIRIT vs DMDA grid equals the reference's CSV") {
    std::string csv;
    for (const char* app : {"autogen", "cholesky", "lu"}) {
        BenchSpec spec;
        spec.app = app;
        spec.sizes = std::string(app) == "autogen" ? std::vector<int64_t>{1000, 5000}
                     : std::string(app) == "cholesky" ? std::vector<int64_t>{8, 12, 16, 20, 24}
                                                      : std::vector<int64_t>{8, 12, 16};
        spec.platforms = {"26cpu_2gpu"};
        spec.policies = {"dmda", "inspirit"};
        spec.seed = 7;
        BenchReport r = run_bench(spec);
        std::ostringstream out;
        write_bench_csv(out, r);
        std::string body = out.str();
        csv += csv.empty() ? body : body.substr(body.find('\n') + 1);
        double log_sum = 0.0, mn = 1e300;
        for (const auto& row : r.rows) {
            REQUIRE(row.ok);
            if (row.policy == "inspirit") {
                log_sum += std::log(row.speedup);
                mn = std::min(mn, row.speedup);
            }
        }
        CHECK(mn >= 0.95);
        CHECK(log_sum >= 0.0);
    }
    std::ifstream golden(std::string(GOLDEN_DIR) + "/grid_bench.csv");
    std::stringstream want;
    want << golden.rdbuf();
    CHECK(csv == want.str());
}

GPU_CASE("acceptance c8: reruns are identical") {
    Platform p = make_preset("26cpu_2gpu");
    auto g = build_cholesky_dag(12, 960 * 960 * 4);
    TaskAttributes a = compute_attributes(g, p.costs, PriorityKind::UpwardRank);
    SimTrace x = run(g, p, "inspirit", a), y = run(g, p, "inspirit", a);
    CHECK(gantt(g, x) == gantt(g, y));
    CHECK(x.nready_samples == y.nready_samples);
    BenchSpec spec;
    spec.app = "cholesky";
    spec.sizes = {12};
    spec.platforms = {"26cpu_2gpu", "homog2"};
    spec.seed = 3;
    auto csv = [&spec]() {
        std::ostringstream out;
        write_bench_csv(out, run_bench(spec));
        return out.str();
    };
    const std::string first = csv();
    CHECK(first == csv());
    spec.jobs = 4;
    CHECK(first == csv());
}

GPU_CASE("acceptance c9: calibration stays within eleven evaluations") {
    CostTable costs = make_preset("26cpu_2gpu").costs;
    std::vector<TaskGraph> graphs;
    for (int n : {8, 12, 16, 20, 24}) graphs.push_back(build_cholesky_dag(n, 4096));
    for (int n : {8, 12, 16}) graphs.push_back(build_lu_dag(n, 4096));
    for (int n : {1000, 5000}) graphs.push_back(generate_layered_dag(n, 10, 0.05, 7));
    for (const auto& g : graphs) {
        CalibrationResult c = calibrate_unit_time(g, costs);
        CHECK(c.evaluations <= 11);
        CHECK(c.best_score >= c.w0_score);
        CHECK(c.unit_time_ms > 0.0);
    }
}

int main(int argc, char** argv) { return mt::run_all(argc, argv); }
