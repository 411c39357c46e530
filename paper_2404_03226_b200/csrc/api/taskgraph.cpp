// taskgraph.cpp -- host utilities of the drop-in task-graph API
// (reference: proj/src/taskgraph.cpp, generators.cpp, dagio.cpp).
// topological_layers() runs on the B200 (device.cpp); the rest is host-side
// graph bookkeeping that returns host data structures.
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <queue>
#include <set>
#include <sstream>
#include <stdexcept>
#include <unordered_set>

#include "../hostbatch.hpp"
#include "device.hpp"
#include "json_lite.hpp"
#include "tbsim/taskgraph.hpp"

namespace tbsim {

GraphIndex build_index(const TaskGraph& g) {  // taskgraph.cpp:11-43
    GraphIndex idx;
    const size_t n = g.tasks.size();
    idx.task_pos.reserve(n);
    for (size_t i = 0; i < n; ++i)
        if (!idx.task_pos.emplace(g.tasks[i].id, i).second)
            throw std::invalid_argument("duplicate task id " + std::to_string(g.tasks[i].id));
    idx.handle_pos.reserve(g.handles.size());
    for (size_t i = 0; i < g.handles.size(); ++i)
        if (!idx.handle_pos.emplace(g.handles[i].id, i).second)
            throw std::invalid_argument("duplicate handle id " + std::to_string(g.handles[i].id));
    idx.succ.assign(n, {});
    idx.pred.assign(n, {});
    for (size_t i = 0; i < n; ++i)
        for (TaskId d : g.tasks[i].deps) {
            const auto it = idx.task_pos.find(d);
            if (it == idx.task_pos.end())
                throw std::invalid_argument("task " + std::to_string(g.tasks[i].id) + " depends on unknown task " +
                                            std::to_string(d));
            idx.pred[i].push_back(it->second);
            idx.succ[it->second].push_back(i);  // dependents visited in position order: sorted
        }
    for (auto& p : idx.pred) std::sort(p.begin(), p.end());
    return idx;
}

namespace {

void id_checks(const TaskGraph& g, std::vector<Violation>& out) {
    std::unordered_set<TaskId> tids;
    for (const auto& t : g.tasks)
        if (!tids.insert(t.id).second) out.push_back({"duplicate task id " + std::to_string(t.id)});
    std::unordered_set<HandleId> hids;
    for (const auto& h : g.handles) {
        if (!hids.insert(h.id).second) out.push_back({"duplicate handle id " + std::to_string(h.id)});
        if (h.bytes <= 0) out.push_back({"handle " + std::to_string(h.id) + " has non-positive bytes"});
    }
    for (const auto& t : g.tasks) {
        const std::string who = "task " + std::to_string(t.id);
        for (TaskId d : t.deps) {
            if (d == t.id) out.push_back({who + " depends on itself"});
            else if (!tids.count(d)) out.push_back({who + " depends on unknown task " + std::to_string(d)});
        }
        for (HandleId h : t.inputs)
            if (!hids.count(h)) out.push_back({who + " reads unknown handle " + std::to_string(h)});
        for (HandleId h : t.outputs)
            if (!hids.count(h)) out.push_back({who + " writes unknown handle " + std::to_string(h)});
    }
}

// Kahn over the walkable part of the graph; on leftovers, follow stuck
// predecessors until a task repeats and report that loop (taskgraph.cpp:78-135).
void cycle_check(const TaskGraph& g, std::vector<Violation>& out) {
    const size_t n = g.tasks.size();
    std::unordered_map<TaskId, size_t> pos;
    for (size_t i = 0; i < n; ++i) pos.emplace(g.tasks[i].id, i);
    std::vector<std::vector<size_t>> succ(n);
    std::vector<int> unmet(n, 0);
    for (size_t i = 0; i < n; ++i)
        for (TaskId d : g.tasks[i].deps) {
            const auto it = pos.find(d);
            if (it == pos.end() || it->second == i) continue;
            succ[it->second].push_back(i);
            ++unmet[i];
        }
    std::queue<size_t> q;
    for (size_t i = 0; i < n; ++i)
        if (!unmet[i]) q.push(i);
    size_t done = 0;
    while (!q.empty()) {
        const size_t u = q.front();
        q.pop();
        ++done;
        for (size_t v : succ[u])
            if (--unmet[v] == 0) q.push(v);
    }
    if (done == n) return;
    std::vector<char> stuck(n, 0);
    size_t start = n;
    for (size_t i = 0; i < n; ++i)
        if (unmet[i] > 0) {
            stuck[i] = 1;
            if (start == n) start = i;
        }
    std::vector<size_t> path;
    std::vector<char> seen(n, 0);
    size_t cur = start;
    while (!seen[cur]) {
        seen[cur] = 1;
        path.push_back(cur);
        for (TaskId d : g.tasks[cur].deps) {
            const auto it = pos.find(d);
            if (it != pos.end() && stuck[it->second]) {
                cur = it->second;
                break;
            }
        }
    }
    std::ostringstream msg;
    msg << "dependency cycle:";
    for (auto it = std::find(path.begin(), path.end(), cur); it != path.end(); ++it) msg << ' ' << g.tasks[*it].id;
    out.push_back({msg.str()});
}

}  // namespace

std::vector<Violation> validate(const TaskGraph& g) {
    std::vector<Violation> out;
    id_checks(g, out);
    cycle_check(g, out);
    return out;
}

std::vector<Violation> check_writer_chains(const TaskGraph& g) {  // taskgraph.cpp:147-195
    std::vector<Violation> out;
    std::unordered_map<HandleId, std::vector<size_t>> writers;
    for (size_t i = 0; i < g.tasks.size(); ++i)
        for (HandleId h : g.tasks[i].outputs) writers[h].push_back(i);
    std::unordered_map<TaskId, size_t> pos;
    for (size_t i = 0; i < g.tasks.size(); ++i) pos.emplace(g.tasks[i].id, i);
    for (const auto& h : g.handles) {
        const auto wit = writers.find(h.id);
        if (wit == writers.end() || wit->second.size() < 2) continue;
        const auto& w = wit->second;
        const std::unordered_set<size_t> wset(w.begin(), w.end());
        std::unordered_map<size_t, size_t> next;
        std::unordered_set<size_t> has_pred;
        bool broken = false;
        for (size_t wi : w)
            for (TaskId d : g.tasks[wi].deps) {
                const auto p = pos.find(d);
                if (p == pos.end() || !wset.count(p->second)) continue;
                if (!next.emplace(p->second, wi).second) broken = true;
                if (!has_pred.insert(wi).second) broken = true;
            }
        size_t head = g.tasks.size();
        for (size_t wi : w)
            if (!has_pred.count(wi)) {
                if (head != g.tasks.size()) broken = true;
                head = wi;
            }
        if (!broken && head != g.tasks.size()) {
            size_t len = 1, cur = head;
            while (next.count(cur)) {
                cur = next[cur];
                ++len;
            }
            if (len != w.size()) broken = true;
        } else {
            broken = true;
        }
        if (broken) out.push_back({"handle " + std::to_string(h.id) + " writers are not serialized by direct dependencies"});
    }
    return out;
}

std::vector<int> topological_layers(const TaskGraph& g) {
    return device::layers(g);  // K1 on the B200
}

std::vector<size_t> topological_order(const TaskGraph& g) {  // taskgraph.cpp:221-241
    const GraphIndex idx = build_index(g);
    const size_t n = g.tasks.size();
    std::vector<int> unmet(n);
    std::priority_queue<size_t, std::vector<size_t>, std::greater<>> ready;
    for (size_t i = 0; i < n; ++i) {
        unmet[i] = static_cast<int>(idx.pred[i].size());
        if (!unmet[i]) ready.push(i);
    }
    std::vector<size_t> order;
    order.reserve(n);
    while (!ready.empty()) {
        const size_t u = ready.top();
        ready.pop();
        order.push_back(u);
        for (size_t v : idx.succ[u])
            if (--unmet[v] == 0) ready.push(v);
    }
    if (order.size() != n) throw std::runtime_error("graph has a dependency cycle");
    return order;
}

size_t edge_count(const TaskGraph& g) {
    size_t e = 0;
    for (const auto& t : g.tasks) e += t.deps.size();
    return e;
}

// ------------------------------------------------------------- generators

namespace {

TaskGraph from_csr(const tbsim_host::GraphCSR& c, std::string name) {
    TaskGraph g;
    g.name = std::move(name);
    g.handles.resize(c.handle_bytes.size());
    for (size_t h = 0; h < c.handle_bytes.size(); ++h) g.handles[h] = {static_cast<HandleId>(h), c.handle_bytes[h]};
    const int32_t n = c.n();
    g.tasks.resize(n);
    for (int32_t i = 0; i < n; ++i) {
        TaskNode& t = g.tasks[i];
        t.id = i;
        t.type = tbsim_host::kTypeNames[c.type[i]];
        t.deps.assign(c.dep.begin() + c.dep_off[i], c.dep.begin() + c.dep_off[i + 1]);
        t.inputs.assign(c.in.begin() + c.in_off[i], c.in.begin() + c.in_off[i + 1]);
        t.outputs.assign(c.out.begin() + c.out_off[i], c.out.begin() + c.out_off[i + 1]);
    }
    return g;
}

}  // namespace

TaskGraph build_cholesky_dag(int nblocks, std::int64_t block_bytes) {
    return from_csr(tbsim_host::gen_cholesky(nblocks, block_bytes), "cholesky_n" + std::to_string(nblocks));
}

TaskGraph build_lu_dag(int nblocks, std::int64_t block_bytes) {
    return from_csr(tbsim_host::gen_lu(nblocks, block_bytes), "lu_n" + std::to_string(nblocks));
}

TaskGraph build_stencil_dag(int nblocks, int timesteps, std::int64_t block_bytes) {  // generators.cpp:144-182
    if (nblocks < 1) throw std::invalid_argument("heat: nblocks must be >= 1");
    if (timesteps < 1) throw std::invalid_argument("heat: timesteps must be >= 1");
    if (block_bytes <= 0) throw std::invalid_argument("heat: block_bytes must be > 0");
    const int n = nblocks;
    TaskGraph g;
    g.name = "heat_n" + std::to_string(n) + "_t" + std::to_string(timesteps);
    for (int c = 0; c < n * n; ++c) g.handles.push_back({c, block_bytes});
    auto tid = [n](int t, int i, int j) { return static_cast<TaskId>(t - 1) * n * n + i * n + j; };
    static const int di[5] = {0, -1, 1, 0, 0}, dj[5] = {0, 0, 0, -1, 1};
    g.tasks.reserve(static_cast<size_t>(timesteps) * n * n);
    for (int t = 1; t <= timesteps; ++t)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                TaskNode task;
                task.id = tid(t, i, j);
                task.type = "STENCIL";
                for (int k = 0; k < 5; ++k) {
                    const int a = i + di[k], b = j + dj[k];
                    if (a < 0 || a >= n || b < 0 || b >= n) continue;
                    if (t > 1) task.deps.push_back(tid(t - 1, a, b));
                    task.inputs.push_back(a * n + b);
                }
                task.outputs.push_back(i * n + j);
                g.tasks.push_back(std::move(task));
            }
    return g;
}

TaskGraph generate_layered_dag(int n_tasks, int n_layers, double edge_prob, std::uint64_t seed) {
    tbsim_host::GraphCSR c = tbsim_host::gen_layered(n_tasks, n_layers, edge_prob, seed);
    char p[32];
    std::snprintf(p, sizeof p, "%g", edge_prob);
    return from_csr(c, "autogen_n" + std::to_string(n_tasks) + "_l" + std::to_string(n_layers) + "_p" + p + "_s" +
                           std::to_string(seed));
}

// ---------------------------------------------------------------- NDJSON

namespace {

void put_ints(std::string& out, const std::vector<std::int64_t>& v) {
    out += '[';
    for (size_t i = 0; i < v.size(); ++i) {
        if (i) out += ',';
        out += std::to_string(v[i]);
    }
    out += ']';
}

[[noreturn]] void line_fail(int line, const std::string& what) {
    throw std::runtime_error("line " + std::to_string(line) + ": " + what);
}

const tbsim_json::Value& field(const tbsim_json::Value& rec, const char* name, int line) {
    const tbsim_json::Value* v = rec.find(name);
    if (!v) line_fail(line, std::string("missing field \"") + name + "\"");
    return *v;
}

std::int64_t int_field(const tbsim_json::Value& rec, const char* name, int line) {
    const auto& v = field(rec, name, line);
    if (!v.is_integer()) line_fail(line, std::string("field \"") + name + "\" must be an integer");
    return v.i;
}

std::string str_field(const tbsim_json::Value& rec, const char* name, int line) {
    const auto& v = field(rec, name, line);
    if (v.type != tbsim_json::Value::String) line_fail(line, std::string("field \"") + name + "\" must be a string");
    return v.s;
}

std::vector<std::int64_t> ints_field(const tbsim_json::Value& rec, const char* name, int line) {
    const auto& v = field(rec, name, line);
    if (v.type != tbsim_json::Value::Array) line_fail(line, std::string("field \"") + name + "\" must be an array");
    std::vector<std::int64_t> out;
    out.reserve(v.arr.size());
    for (const auto& x : v.arr) {
        if (!x.is_integer()) line_fail(line, std::string("field \"") + name + "\" must hold integers");
        out.push_back(x.i);
    }
    return out;
}

}  // namespace

void save_dag(const TaskGraph& g, std::ostream& out) {  // dagio.cpp:15-38, record layout byte-identical
    std::string line;
    line = "{\"kind\":\"meta\",\"name\":";
    tbsim_json::dump_string(line, g.name);
    line += ",\"version\":1}\n";
    out << line;
    for (const auto& h : g.handles)
        out << "{\"kind\":\"handle\",\"id\":" << h.id << ",\"bytes\":" << h.bytes << "}\n";
    for (const auto& t : g.tasks) {
        line = "{\"kind\":\"task\",\"id\":" + std::to_string(t.id) + ",\"type\":";
        tbsim_json::dump_string(line, t.type);
        line += ",\"deps\":";
        put_ints(line, t.deps);
        line += ",\"inputs\":";
        put_ints(line, t.inputs);
        line += ",\"outputs\":";
        put_ints(line, t.outputs);
        line += "}\n";
        out << line;
    }
}

void save_dag_file(const TaskGraph& g, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open " + path + " for writing");
    save_dag(g, out);
    if (!out) throw std::runtime_error("write failed: " + path);
}

TaskGraph load_dag(std::istream& in) {  // dagio.cpp:86-132
    TaskGraph g;
    std::string text;
    int line = 0;
    bool meta = false;
    while (std::getline(in, text)) {
        ++line;
        if (text.empty()) line_fail(line, "empty line");
        tbsim_json::Value rec;
        try {
            rec = tbsim_json::parse(text);
        } catch (const tbsim_json::ParseError& e) {
            line_fail(line, std::string("bad JSON: ") + e.what());
        }
        if (rec.type != tbsim_json::Value::Object) line_fail(line, "record is not an object");
        const std::string kind = str_field(rec, "kind", line);
        if (kind == "meta") {
            if (meta) line_fail(line, "duplicate meta record");
            if (line != 1) line_fail(line, "meta record must come first");
            meta = true;
            g.name = str_field(rec, "name", line);
            if (int_field(rec, "version", line) != 1) line_fail(line, "unsupported version");
        } else if (kind == "handle") {
            if (!meta) line_fail(line, "record before meta");
            DataHandle h;
            h.id = int_field(rec, "id", line);
            h.bytes = int_field(rec, "bytes", line);
            g.handles.push_back(h);
        } else if (kind == "task") {
            if (!meta) line_fail(line, "record before meta");
            TaskNode t;
            t.id = int_field(rec, "id", line);
            t.type = str_field(rec, "type", line);
            t.deps = ints_field(rec, "deps", line);
            t.inputs = ints_field(rec, "inputs", line);
            t.outputs = ints_field(rec, "outputs", line);
            g.tasks.push_back(std::move(t));
        } else {
            line_fail(line, "unknown record kind \"" + kind + "\"");
        }
    }
    if (!meta) throw std::runtime_error("missing meta record");
    const auto bad = validate(g);
    if (!bad.empty()) {
        std::string msg = "invalid graph:";
        for (const auto& v : bad) msg += "\n  " + v.message;
        throw std::runtime_error(msg);
    }
    return g;
}

TaskGraph load_dag_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    return load_dag(in);
}

}  // namespace tbsim
