// simulate.cuh -- launch interface of the batched event simulator.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace tbsim_dev {

// Per-warp state layout (bytes, 16-aligned sections).  Compact state
// (n < 32768, <= 8 memory nodes) stores unmet counts and the ready list as
// int16 and residency masks as uint8.
struct SimLayout {
    int64_t unmet, resid, ready, queue, qab, qef, qprio, ring, costs, bw, total;
};

// Pop keys cached per queue entry: inspirit (policy 4) ability + efficiency
// (int32) + static priority (int64); dmdap (3) the priority only.
__host__ __device__ inline int key_bytes(int32_t policy) { return policy == 4 ? 16 : policy == 3 ? 8 : 0; }

__host__ __device__ inline SimLayout sim_layout(int64_t max_n, int64_t max_h, int64_t max_workers, int64_t qcap,
                                                int64_t ring, int64_t n_types, int64_t max_nodes, bool compact,
                                                int32_t policy) {
    auto al = [](int64_t x) { return (x + 15) & ~int64_t(15); };
    SimLayout L;
    int64_t off = 0;
    L.unmet = off; off += al((compact ? 2 : 4) * max_n);
    L.resid = off; off += al((compact ? 1 : 4) * max_h);
    L.ready = off; off += al((compact ? 2 : 4) * max_n);
    L.queue = off; off += al(4 * max_workers * qcap);
    const bool ins = policy == 4, pri = policy >= 3;
    L.qab = off; off += ins ? al(4 * max_workers * qcap) : 0;
    L.qef = off; off += ins ? al(4 * max_workers * qcap) : 0;
    L.qprio = off; off += pri ? al(8 * max_workers * qcap) : 0;
    L.ring = off; off += al(16 * ring);
    L.costs = off; off += al(16 * n_types);
    L.bw = off; off += al(8 * max_nodes * max_nodes);
    L.total = off;
    return L;
}

struct SimParams {
    DevBatch b;
    const DevPlatform* platforms;
    const int32_t* platform_of;       // [G] or null
    int32_t policy;
    const tbsim_regulator_cfg* reg;   // [G] or null -> default from median
    const double* median;             // [G] lower-median GPU time (default cfg)
    int32_t median_stride;            // elements between consecutive graphs' medians
    const int64_t* ability;           // [T] or null
    const int64_t* efficiency;        // [T] or null
    const int64_t* prio;              // [T] or null
    // outputs
    int32_t* worker;
    double* start_ms;
    double* end_ms;
    double* makespan;                 // [G]
    int64_t* completed;               // [G]
    int64_t* pop_counts;              // [3G] or null
    tbsim_regulator_state* reg_state; // [G] in/out or null
    double* push_time;  int32_t* push_task;
    double* pop_time;   int32_t* pop_task;  int32_t* pop_worker;
    double* sample_time; int64_t* sample_nready;
    int32_t* status;                  // [G]
    int32_t* status_aux;              // [G]
    // per-warp state
    char* gstate;                     // global fallback region base
    int64_t state_bytes;              // bytes per warp state
    int32_t qcap;                     // queue capacity per worker
    int32_t use_smem;
    int32_t max_workers;
    int32_t max_nodes;                // platform copy: nodes x nodes bandwidth
    int32_t n_types;                  // platform copy: cost rows
    int32_t ring;                     // regulator sample ring capacity (power of 2)
    SimLayout layout;                 // per-warp state sections (set by launch_sim)
    const int32_t* graph_list;        // subset of graphs (rerun) or null
    int64_t n_items;                  // graphs to process (list length or G)
    unsigned long long* work_counter;
};

__global__ void k_simulate_w1c(const __grid_constant__ SimParams p);  // <= 32 workers, compact state
__global__ void k_simulate_w2c(const __grid_constant__ SimParams p);  // <= 64 workers, compact state
__global__ void k_simulate_w1(const __grid_constant__ SimParams p);   // <= 32 workers, wide state
__global__ void k_simulate_w2(const __grid_constant__ SimParams p);   // <= 64 workers, wide state

}  // namespace tbsim_dev
