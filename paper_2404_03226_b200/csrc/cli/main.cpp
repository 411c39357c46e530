// tbsim -- the command-line front end over the drop-in C++ API
// (include/tbsim/*.hpp, libtbsim_cpp.so): generate task graphs, compute
// scheduling attributes, run one simulation, sweep a benchmark grid.  The
// same subcommands, flags, outputs and exit codes as the reference's CLI
// (proj/tools/main.cpp:139-345): 0 success, 1 usage error, 2 runtime failure.
// Attributes and simulations run on the B200 through the C-ABI; the argument
// parser is a small hand-written one (the reference uses CLI11).

#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
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

namespace fs = std::filesystem;
using namespace tbsim;

namespace {

// Default tile sizes of the generators (tools/main.cpp:29-31).
constexpr std::int64_t kCholeskyBytes = 960 * 960 * 4;
constexpr std::int64_t kLuBytes = 160 * 160 * 4;
constexpr std::int64_t kHeatBytes = 640 * 640 * 4;

// A usage error: printed to stderr, exit code 1.
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

const char* kHelp =
    "task-based runtime scheduling simulator (B200)\n"
    "Usage: tbsim [OPTIONS] SUBCOMMAND\n\n"
    "Options:\n"
    "  -h,--help          print this help and exit\n"
    "  --platform TEXT    platform preset name or JSON file (repeatable for bench) [26cpu_2gpu]\n"
    "  --seed UINT        base RNG seed [0]\n"
    "  --out-dir TEXT     directory for generated files [.]\n"
    "  --jobs INT         parallel bench cells (<=0 means all host CPUs)\n\n"
    "Subcommands:\n"
    "  gen                generate a task graph file (cholesky | lu | heat | autogen)\n"
    "  attrs              compute per-task attributes\n"
    "  sim                simulate one DAG under one policy\n"
    "  bench              sweep app x size x platform x policy\n";

// Tokens after the program name; options may appear before or after the
// subcommand names (CLI11 fallthrough).
class Args {
  public:
    explicit Args(std::vector<std::string> t) : tok_(std::move(t)), used_(tok_.size(), false) {}

    bool flag(const std::string& name) {
        bool seen = false;
        for (size_t i = 0; i < tok_.size(); ++i)
            if (!used_[i] && tok_[i] == name) { used_[i] = true; seen = true; }
        return seen;
    }
    // every value of a repeatable single-value option
    std::vector<std::string> values(const std::string& name) {
        std::vector<std::string> out;
        for (size_t i = 0; i < tok_.size(); ++i) {
            if (used_[i] || tok_[i] != name) continue;
            if (i + 1 >= tok_.size() || used_[i + 1]) throw UsageError(name + ": 1 required TEXT missing");
            used_[i] = used_[i + 1] = true;
            out.push_back(tok_[i + 1]);
            ++i;
        }
        return out;
    }
    std::optional<std::string> value(const std::string& name) {
        auto v = values(name);
        if (v.empty()) return std::nullopt;
        return v.back();
    }
    // a list option: every following token that is not an option
    std::vector<std::string> list(const std::string& name) {
        std::vector<std::string> out;
        for (size_t i = 0; i < tok_.size(); ++i) {
            if (used_[i] || tok_[i] != name) continue;
            used_[i] = true;
            size_t j = i + 1;
            for (; j < tok_.size() && !used_[j] && !is_option(tok_[j]) && !is_word(tok_[j]); ++j) {
                used_[j] = true;
                out.push_back(tok_[j]);
            }
            if (j == i + 1) throw UsageError(name + ": at least 1 value required");
            i = j - 1;
        }
        return out;
    }
    // the next unused positional token (a subcommand name)
    std::optional<std::string> word() {
        for (size_t i = 0; i < tok_.size(); ++i)
            if (!used_[i] && !is_option(tok_[i])) {
                used_[i] = true;
                return tok_[i];
            }
        return std::nullopt;
    }
    void finish() const {
        for (size_t i = 0; i < tok_.size(); ++i)
            if (!used_[i]) throw UsageError("The following arguments were not expected: " + tok_[i]);
    }
    void set_words(std::set<std::string> w) { words_ = std::move(w); }

  private:
    static bool is_option(const std::string& s) {
        if (s.size() < 2 || s[0] != '-') return false;
        // negative numbers are values
        return !(std::isdigit(static_cast<unsigned char>(s[1])) || s[1] == '.');
    }
    bool is_word(const std::string& s) const { return words_.count(s) > 0; }
    std::vector<std::string> tok_;
    std::vector<bool> used_;
    std::set<std::string> words_;
};

std::int64_t to_int(const std::string& opt, const std::string& s) {
    try {
        size_t pos = 0;
        const long long v = std::stoll(s, &pos);
        if (pos != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        throw UsageError(opt + ": value " + s + " not an integer");
    }
}

double to_double(const std::string& opt, const std::string& s) {
    try {
        size_t pos = 0;
        const double v = std::stod(s, &pos);
        if (pos != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        throw UsageError(opt + ": value " + s + " not a number");
    }
}

std::int64_t positive(const std::string& opt, std::int64_t v) {
    if (v <= 0) throw UsageError(opt + ": Value " + std::to_string(v) + " not in range [0 - max]");
    return v;
}

PriorityKind priority_of(Args& a) {
    static const std::map<std::string, PriorityKind> names{
        {"rank", PriorityKind::UpwardRank}, {"depth", PriorityKind::Depth}, {"zero", PriorityKind::Zero}};
    auto v = a.value("--priority");
    if (!v) return PriorityKind::UpwardRank;
    auto it = names.find(*v);
    if (it == names.end()) throw UsageError("--priority: Check " + *v + " value in {rank,depth,zero} FAILED");
    return it->second;
}

std::string member(const std::string& opt, const std::string& v, const std::vector<std::string>& allowed) {
    for (const auto& s : allowed)
        if (s == v) return v;
    throw UsageError(opt + ": " + v + " not in {...}");
}

struct Globals {
    std::vector<std::string> platforms{"26cpu_2gpu"};
    std::uint64_t seed = 0;
    std::string out_dir = ".";
    int jobs = 0;
};

// Regulator flags shared by sim and bench: only the flags given override
// the per-graph defaults (tools/main.cpp:42-91).
RegulatorOverride reg_flags(Args& a) {
    RegulatorOverride ov;
    if (auto v = a.value("--task-window")) ov.task_window = to_int("--task-window", *v);
    if (auto v = a.value("--s-inc")) ov.s_inc = to_int("--s-inc", *v);
    if (auto v = a.value("--k-inc")) ov.k_inc = to_double("--k-inc", *v);
    if (auto v = a.value("--s-dec")) ov.s_dec = to_int("--s-dec", *v);
    if (auto v = a.value("--c")) ov.c = to_int("--c", *v);
    if (auto v = a.value("--dec-step")) ov.dec_step = to_int("--dec-step", *v);
    if (auto v = a.value("--slope-samples")) ov.slope_samples = static_cast<int>(to_int("--slope-samples", *v));
    return ov;
}

RegulatorConfig apply(RegulatorConfig cfg, const RegulatorOverride& ov) {
    if (ov.task_window) cfg.task_window = *ov.task_window;
    if (ov.s_inc) cfg.s_inc = *ov.s_inc;
    if (ov.k_inc) cfg.k_inc = *ov.k_inc;
    if (ov.s_dec) cfg.s_dec = *ov.s_dec;
    if (ov.c) cfg.c = *ov.c;
    if (ov.dec_step) cfg.dec_step = *ov.dec_step;
    if (ov.slope_samples) cfg.slope_samples = *ov.slope_samples;
    return cfg;
}

std::string single_platform(const Globals& g) {
    if (g.platforms.size() != 1) throw UsageError("--platform: exactly one platform expected here");
    return g.platforms.front();
}

fs::path resolve_out(const Globals& g, const std::string& explicit_path, const std::string& default_name) {
    fs::path p = explicit_path.empty() ? fs::path(g.out_dir) / default_name : fs::path(explicit_path);
    if (p.has_parent_path()) fs::create_directories(p.parent_path());
    return p;
}

std::ofstream open_out(const fs::path& p) {
    std::ofstream out(p, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write " + p.string());
    return out;
}

void write_graph(const Globals& g, const TaskGraph& graph, const std::string& explicit_path) {
    const fs::path p = resolve_out(g, explicit_path, graph.name + ".dag");
    save_dag_file(graph, p.string());
    std::cout << "wrote " << p.string() << ": " << graph.tasks.size() << " tasks, " << edge_count(graph)
              << " edges\n";
}

void cmd_gen(const Globals& g, Args& a) {
    const std::string out = a.value("--out").value_or("");
    const auto kind = a.word();
    if (!kind) throw UsageError("gen: a subcommand is required (cholesky | lu | heat | autogen)");
    if (*kind == "autogen") {
        auto t = a.value("--tasks");
        if (!t) throw UsageError("--tasks is required");
        const std::int64_t tasks = positive("--tasks", to_int("--tasks", *t));
        const int layers = static_cast<int>(positive("--layers", to_int("--layers", a.value("--layers").value_or("10"))));
        const double p = to_double("--edge-prob", a.value("--edge-prob").value_or("0.05"));
        if (!(p >= 0.0 && p <= 1.0)) throw UsageError("--edge-prob: Value not in range [0 - 1]");
        a.finish();
        write_graph(g, generate_layered_dag(static_cast<int>(tasks), layers, p, g.seed), out);
        return;
    }
    if (*kind != "cholesky" && *kind != "lu" && *kind != "heat")
        throw UsageError("gen: unknown subcommand " + *kind);
    auto nb = a.value("--nblocks");
    if (!nb) throw UsageError("--nblocks is required");
    const int nblocks = static_cast<int>(positive("--nblocks", to_int("--nblocks", *nb)));
    std::int64_t bytes = 0;
    if (auto v = a.value("--block-bytes")) bytes = positive("--block-bytes", to_int("--block-bytes", *v));
    int steps = 0;
    if (*kind == "heat")
        if (auto v = a.value("--timesteps")) steps = static_cast<int>(positive("--timesteps", to_int("--timesteps", *v)));
    a.finish();
    if (*kind == "cholesky") write_graph(g, build_cholesky_dag(nblocks, bytes > 0 ? bytes : kCholeskyBytes), out);
    else if (*kind == "lu") write_graph(g, build_lu_dag(nblocks, bytes > 0 ? bytes : kLuBytes), out);
    else write_graph(g, build_stencil_dag(nblocks, steps > 0 ? steps : 2 * nblocks, bytes > 0 ? bytes : kHeatBytes), out);
}

void cmd_attrs(const Globals& g, Args& a) {
    auto dag = a.value("--dag");
    if (!dag) throw UsageError("--dag is required");
    const std::string out = a.value("--out").value_or("");
    const PriorityKind prio = priority_of(a);
    a.finish();
    TaskGraph graph = load_dag_file(*dag);
    Platform platform = resolve_platform(single_platform(g));
    CalibrationResult cal = calibrate_unit_time(graph, platform.costs);
    TaskAttributes attrs = compute_attributes(graph, platform.costs, prio);
    const fs::path p = resolve_out(g, out, "attributes.csv");
    auto f = open_out(p);
    write_attributes_csv(f, graph, attrs);
    std::cout << "wrote " << p.string() << ": " << graph.tasks.size() << " rows\n";
    std::cerr << "unit_time_ms: " << fmt_ms(cal.unit_time_ms) << " (start " << fmt_ms(cal.w0_ms) << ", score "
              << cal.w0_score << " -> " << cal.best_score << ", " << cal.evaluations << " evaluations)\n";
}

void cmd_sim(const Globals& g, Args& a) {
    auto dag = a.value("--dag");
    if (!dag) throw UsageError("--dag is required");
    const std::string policy_name = member("--policy", a.value("--policy").value_or("dmda"), policy_names());
    const PriorityKind prio = priority_of(a);
    const bool trace = a.flag("--trace");
    double window_ms = 0.0;
    if (auto v = a.value("--window")) {
        window_ms = to_double("--window", *v);
        if (!(window_ms > 0.0)) throw UsageError("--window: Value not in range [0 - max]");
    }
    const RegulatorOverride ov = reg_flags(a);
    a.finish();
    TaskGraph graph = load_dag_file(*dag);
    Platform platform = resolve_platform(single_platform(g));
    TaskAttributes attrs = compute_attributes(graph, platform.costs, prio);
    RegulatorConfig cfg = apply(default_regulator_config(platform, graph), ov);
    auto policy = make_policy(policy_name, attrs, cfg);
    SimOptions opts;
    opts.record_trace = trace;
    SimTrace result = simulate(graph, platform, *policy, opts);
    std::cout << "dag: " << graph.name << " (" << graph.tasks.size() << " tasks)\n";
    std::cout << "platform: " << platform.name << "\n";
    std::cout << "policy: " << policy_name << "\n";
    if (policy_name == "inspirit") {
        std::cout << "regulator: task_window=" << cfg.task_window << " s_inc=" << cfg.s_inc
                  << " k_inc=" << fmt_ms(cfg.k_inc) << " s_dec=" << cfg.s_dec << " c=" << cfg.c
                  << " dec_step=" << cfg.dec_step << " slope_samples=" << cfg.slope_samples << "\n";
        if (const auto* counts = pop_mode_counts(*policy))
            std::cout << "pops_by_mode: ability=" << (*counts)[0] << " efficiency=" << (*counts)[1]
                      << " efficiency_locality=" << (*counts)[2] << "\n";
    }
    std::cout << "makespan_ms: " << fmt_ms(result.makespan_ms) << "\n";
    if (trace) {
        const double window = window_ms > 0.0 ? window_ms : 10.0 * median_gpu_time_ms(graph, platform.costs);
        fs::create_directories(g.out_dir);
        {
            auto f = open_out(fs::path(g.out_dir) / "nready_time.csv");
            write_nready_csv(f, result);
        }
        {
            auto f = open_out(fs::path(g.out_dir) / "push_pop.csv");
            write_push_pop_csv(f, result, window);
        }
        {
            auto f = open_out(fs::path(g.out_dir) / "gantt.csv");
            write_gantt_csv(f, graph, result);
        }
        std::cout << "trace: " << g.out_dir << " (nready_time.csv push_pop.csv gantt.csv, window " << fmt_ms(window)
                  << " ms)\n";
    }
}

void cmd_bench(const Globals& g, Args& a) {
    BenchSpec spec;
    auto app = a.value("--app");
    if (!app) throw UsageError("--app is required");
    spec.app = member("--app", *app, {"cholesky", "lu", "heat", "autogen", "file"});
    for (const auto& s : a.list("--sizes")) spec.sizes.push_back(to_int("--sizes", s));
    const auto pols = policy_names();
    for (const auto& s : a.list("--policies")) spec.policies.push_back(member("--policies", s, pols));
    if (auto v = a.value("--baseline")) spec.baseline = member("--baseline", *v, pols);
    if (auto v = a.value("--layers")) spec.autogen_layers = static_cast<int>(positive("--layers", to_int("--layers", *v)));
    if (auto v = a.value("--edge-prob")) {
        spec.autogen_edge_prob = to_double("--edge-prob", *v);
        if (!(spec.autogen_edge_prob >= 0.0 && spec.autogen_edge_prob <= 1.0))
            throw UsageError("--edge-prob: Value not in range [0 - 1]");
    }
    spec.dag_files = a.list("--dag");
    spec.priority = priority_of(a);
    const std::string out = a.value("--out").value_or("");
    spec.regulator = reg_flags(a);
    a.finish();
    spec.platforms = g.platforms;
    spec.seed = g.seed;
    spec.jobs = g.jobs;
    BenchReport report = run_bench(spec);
    size_t failed = 0;
    for (const BenchRow& r : report.rows)
        if (!r.ok) failed += 1;
    const fs::path p = resolve_out(g, out, "bench.csv");
    auto f = open_out(p);
    write_bench_csv(f, report);
    std::cout << "wrote " << p.string() << ": " << report.rows.size() << " rows\n";
    if (failed > 0) std::cerr << failed << " cells failed; see status column\n";
}

}  // namespace

int main(int argc, char** argv) {
    Args a(std::vector<std::string>(argv + 1, argv + argc));
    a.set_words({"gen", "attrs", "sim", "bench", "cholesky", "lu", "heat", "autogen"});
    try {
        if (a.flag("--help") || a.flag("-h")) {
            std::cout << kHelp;
            return 0;
        }
        Globals g;
        auto plats = a.values("--platform");
        if (!plats.empty()) g.platforms = plats;
        if (auto v = a.value("--seed")) g.seed = static_cast<std::uint64_t>(to_int("--seed", *v));
        if (auto v = a.value("--out-dir")) g.out_dir = *v;
        if (auto v = a.value("--jobs")) g.jobs = static_cast<int>(to_int("--jobs", *v));
        const auto cmd = a.word();
        if (!cmd) throw UsageError("A subcommand is required");
        try {
            if (*cmd == "gen") cmd_gen(g, a);
            else if (*cmd == "attrs") cmd_attrs(g, a);
            else if (*cmd == "sim") cmd_sim(g, a);
            else if (*cmd == "bench") cmd_bench(g, a);
            else throw UsageError("The following arguments were not expected: " + *cmd);
        } catch (const UsageError&) {
            throw;
        } catch (const std::exception& e) {
            std::cerr << "error: " << e.what() << "\n";
            return 2;
        }
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return 1;
    }
    return 0;
}
