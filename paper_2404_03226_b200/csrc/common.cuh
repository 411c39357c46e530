// common.cuh -- device-side data layout shared by every kernel.
//
// HBM layout of a batch (one packed H2D copy, see abi.cpp upload):
//   per graph  : task/edge/handle/in/out bases (int64, [G+1] each)
//   per task   : dep_off/in_off/out_off (int32 local offsets, n_g+1 per graph),
//                type (int32)
//   per entry  : dep/in/out (int32 local positions), handle_bytes (int64)
//   derived    : succ_off/succ (int32, sorted ascending per list, multi-edges
//                kept; built by k_ingest exactly like build_index,
//                src/taskgraph.cpp:11-43)
#pragma once

#include <cstdint>

#include "tbsim_b200.h"

namespace tbsim_dev {

constexpr int kMaxWorkers = 64;   // device simulator limit (2 workers per lane)
constexpr int kMaxNodes = 16;     // memory nodes per platform
constexpr int kMaxTypes = 64;     // task types per batch
constexpr int kWindows = 11;      // calibration candidates k = -4..6 (attributes.cpp:221)
constexpr int kBins = 12;         // 11 windows + "reachable beyond every window"

// Per-graph status codes written by kernels (0 = ok).  The host turns them
// into the reference's exception type + text.
enum GraphStatus : int32_t {
    GS_OK = 0,
    GS_CYCLE = 1,            // "graph has a dependency cycle"
    GS_NO_GPU_COST = 2,      // "no gpu cost entry for task type X"   (aux = task pos)
    GS_NO_COST = 3,          // "no cost entry for task type X"       (aux = task pos)
    GS_EMPTY_MEDIAN = 4,     // "empty graph has no median time"
    GS_NO_WORKER = 5,        // "no worker can run task type X"       (aux = task pos)
    GS_STUCK = 6,            // "simulation stuck with K tasks unfinished: ..."
    GS_QUEUE_OVERFLOW = 7,   // internal: smem queue capacity exceeded -> rerun in HBM
    GS_DEGENERATE_TIME = 8,  // event created at `now` (exec/transfer below ulp)
    GS_NEG_WINDOW = 9,       // "unit time must be non-negative"
    GS_TOO_LARGE = 10,       // graph exceeds a device limit
};

struct DevBatch {
    int64_t G;
    int64_t T, E, H, I, O;
    const int64_t* task_base;
    const int64_t* edge_base;
    const int64_t* handle_base;
    const int64_t* in_base;
    const int64_t* out_base;
    const int32_t* dep_off;
    const int32_t* dep;
    const int32_t* in_off;
    const int32_t* in;
    const int32_t* out_off;
    const int32_t* out;
    const int32_t* type;
    const int64_t* handle_bytes;
    int32_t* succ_off;  // derived [T+G]
    int32_t* succ;      // derived [E]
    int32_t max_n;
    int32_t max_e;
    int32_t max_h;
    int32_t n_types;
};

// Cost table on the device: present iff > 0 (CostTable, platform.hpp:23-47).
struct DevCosts {
    int32_t n_types;
    double cpu[kMaxTypes];
    double gpu[kMaxTypes];
};

struct DevPlatform {
    int32_t n_workers;
    int32_t n_nodes;
    double latency_ms;
    int32_t kind[kMaxWorkers];
    int32_t node[kMaxWorkers];
    double bw[kMaxNodes * kMaxNodes];
    DevCosts costs;
};

__host__ __device__ inline double cost_of(const DevCosts& c, int32_t ty, int32_t kind) {
    if (ty < 0 || ty >= c.n_types) return 0.0;
    return kind ? c.gpu[ty] : c.cpu[ty];
}

// Non-negative doubles order like their bit patterns (as uint64).
__device__ __forceinline__ uint64_t dbits(double x) {
    return static_cast<uint64_t>(__double_as_longlong(x));
}

// Warp-wide lexicographic min/max of 64-bit keys with REDUX on 32-bit halves.
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v, unsigned mask = 0xffffffffu) {
    uint32_t hi = static_cast<uint32_t>(v >> 32), lo = static_cast<uint32_t>(v);
    uint32_t mhi = __reduce_min_sync(mask, hi);
    unsigned m2 = __ballot_sync(mask, hi == mhi);
    uint32_t mlo = __reduce_min_sync(mask, hi == mhi ? lo : 0xffffffffu);
    (void)m2;
    return (static_cast<uint64_t>(mhi) << 32) | mlo;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v, unsigned mask = 0xffffffffu) {
    uint32_t hi = static_cast<uint32_t>(v >> 32), lo = static_cast<uint32_t>(v);
    uint32_t mhi = __reduce_max_sync(mask, hi);
    uint32_t mlo = __reduce_max_sync(mask, hi == mhi ? lo : 0u);
    return (static_cast<uint64_t>(mhi) << 32) | mlo;
}

}  // namespace tbsim_dev
