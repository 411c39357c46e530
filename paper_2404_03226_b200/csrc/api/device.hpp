// device.hpp -- bridge from the drop-in C++ API (tbsim::) to the C-ABI
// (include/tbsim_b200.h): TaskGraph -> CSR batch, per-thread device context,
// status -> exception mapping.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "tbsim/attributes.hpp"
#include "tbsim/engine.hpp"
#include "tbsim/platform.hpp"
#include "tbsim/policies.hpp"
#include "tbsim/taskgraph.hpp"
#include "tbsim_b200.h"

namespace tbsim::device {

// Throws the reference exception type for a failing C-ABI status.
void check(tbsim_status st);

// Context of the calling thread (created on first use; device from the
// TBSIM_DEVICE environment variable, default 0).
tbsim_ctx* context();

// A batch of TaskGraphs converted to the C-ABI CSR layout.
struct Csr {
    std::vector<int64_t> task_base{0}, edge_base{0}, handle_base{0}, in_base{0}, out_base{0};
    std::vector<int32_t> dep_off, dep, in_off, in, out_off, out, type;
    std::vector<int64_t> handle_bytes, task_id;
    std::vector<std::string> type_names;
    std::vector<const char*> name_ptrs;
    tbsim_batch_desc desc{};
    // a task names a handle the graph does not declare: the reference's
    // engine fails on it (std::out_of_range from handle_pos.at(),
    // src/engine.cpp:68,108,171) while its attribute functions never look;
    // such entries are left out here and simulate() throws
    bool unknown_handle = false;
    void add(const TaskGraph& g);  // throws build_index's errors
    void require_known_handles() const;
    const tbsim_batch_desc& finish();
};

// Device-resident batch, freed on destruction.
class Uploaded {
public:
    explicit Uploaded(Csr& csr);
    ~Uploaded();
    Uploaded(const Uploaded&) = delete;
    Uploaded& operator=(const Uploaded&) = delete;
    tbsim_batch* get() const { return b_; }

private:
    tbsim_batch* b_ = nullptr;
};

// Cost arrays aligned with a type-name table.
struct CostArrays {
    std::vector<double> cpu, gpu;
    tbsim_costs view() const;
};
CostArrays cost_arrays(const CostTable& t, const std::vector<std::string>& names);

// Platform descriptor (+ owned arrays) aligned with a type-name table.
struct PlatformArrays {
    std::vector<int32_t> kind, node;
    std::vector<double> bw;
    CostArrays costs;
    tbsim_platform_desc desc{};
};
PlatformArrays platform_arrays(const Platform& p, const std::vector<std::string>& names);

std::vector<int> layers(const TaskGraph& g);

struct AttrResult {
    std::vector<int64_t> ability, efficiency, static_priority, depth;
    double unit_time_ms = 0.0, w0_ms = 0.0;
    int64_t best_score = 0, w0_score = 0;
    int32_t evaluations = 0;
};
AttrResult attributes(const TaskGraph& g, const CostTable& costs, int32_t request, int32_t prio_kind,
                      double unit_time_ms);

}  // namespace tbsim::device
