// simulate.cuh -- launch interface of the batched event simulator.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace tbsim_dev {

// Rarely touched per-warp scalars (regulator, counters, graph ids) live in
// the warp's state memory instead of registers: the event loop keeps only
// the hot state in registers, which lets more warps share an SM.
struct SimCold {
    tbsim_regulator_cfg cfg;
    int64_t peak, prev_nready, last_trigger, s_dec_count;
    double cur_k;
    double lat;          // platform transfer latency (ms)
    int64_t n_push, n_samp, pop0, pop1, pop2;
    int64_t g, t0;
    int32_t phase, r_head, r_count, aux;
    int32_t nn;          // platform memory nodes
    const double* xt;    // this platform's transfer table (SimParams::xtab)
    int64_t hb;          // the graph's handle base (escaped handle sizes)
    int32_t n_pop;       // dispatches so far (log slot)
    int32_t rtail;       // last task of the ready list
};

// Per-warp state layout (bytes, 16-aligned sections).  Compact state
// (n < 32768, <= 8 memory nodes) stores unmet counts as int16, residency
// masks as uint8, and queue keys narrowed: ability/efficiency int16, static
// priority read from the task record.
// The ready list has no section: it is a linked list threaded through the
// unmet counters of ready tasks (a ready task's counter is never read again).
struct SimLayout {
    int64_t cold, unmet, resid, queue, qab, qef, qprio, ring, costs, bw, total;
};

// Pop keys cached per queue entry: inspirit (policy 4) ability + efficiency
// + static priority; dmdap (3) the priority only.
// Compact state reads the static priority from the task record instead
// (smaller queues leave L1 room for the simulator's spills).
__host__ __device__ inline int key_bytes(int32_t policy, bool compact) {
    return policy == 4 ? (compact ? 4 : 16) : policy == 3 ? (compact ? 0 : 8) : 0;
}

__host__ __device__ inline SimLayout sim_layout(int64_t max_n, int64_t max_h, int64_t max_workers, int64_t qcap,
                                                int64_t ring, int64_t n_types, int64_t max_nodes, bool compact,
                                                int32_t policy) {
    auto al = [](int64_t x) { return (x + 15) & ~int64_t(15); };
    SimLayout L;
    int64_t off = 0;
    L.cold = off; off += al(static_cast<int64_t>(sizeof(SimCold)));
    L.unmet = off; off += al((compact ? 2 : 4) * max_n);
    L.resid = off; off += al((compact ? 1 : 4) * max_h);
    L.queue = off; off += al(4 * max_workers * qcap);
    const bool ins = policy == 4, pri = policy >= 3;
    const int kb = compact ? 2 : 4;
    L.qab = off; off += ins ? al(kb * max_workers * qcap) : 0;
    L.qef = off; off += ins ? al(kb * max_workers * qcap) : 0;
    L.qprio = off; off += pri && !compact ? al(2 * kb * max_workers * qcap) : 0;
    L.ring = off; off += al(16 * ring);
    L.costs = off; off += al(16 * n_types);
    L.bw = off; off += al(8 * max_nodes * max_nodes);
    L.total = off;
    return L;
}

// Handle byte classes.  The batch's distinct handle sizes (up to 15, one
// dictionary per batch, k_bytes_dict) are numbered; an input list entry is
// handle | class << 28 (class 15: the size is not in the dictionary, read
// handle_bytes).  The transfer estimate lat + bytes / bw(src, dst) of a class
// is then one lookup in a per-call table (k_xfer_table, the same FP64
// operations the reference performs, computed once) instead of an 8-byte
// load and an FP64 divide per input.
constexpr int kHandleBits = 28;
constexpr int32_t kHandleMask = (1 << kHandleBits) - 1;
constexpr int kByteClasses = 16;      // table rows; class 15 is the escape
constexpr int kEscapeClass = kByteClasses - 1;
constexpr int64_t kDictEmpty = INT64_MIN;

// Per-task record of the packed simulation graph (k_sim_pack): everything a
// push, dispatch or completion reads about one task in one 32-byte sector,
// plus an offset (in 4-byte units) to the task's contiguous lists
//   [inputs: int32 handle | class << 28 x nin][outputs: int32 x nout][successors: int32 x nsucc]
// The CSR sections of the batch are scattered over ten arrays; packed, a task
// touches ~2 consecutive sectors instead of ~25 scattered ones.
struct alignas(16) SimTaskHdr {
    uint32_t adj4;      // list offset / 4 from the adjacency base
    uint32_t nin;
    uint32_t nout;
    uint32_t nsucc_ty;  // successors (24 bits) | type << 24
    int32_t ab, ef;     // inspirit pop keys (int32 queue keys; ab < 0: does not fit)
    int64_t prio;       // static priority
};
static_assert(sizeof(SimTaskHdr) == 32, "one sector per task");

// Dispatch log entry: the simulator appends one per dispatch in dispatch
// order (sequential stores); k_sim_scatter moves them to the per-task output
// arrays afterwards.
struct SimLog {
    int32_t task, worker;
    double start, end;
};

// Byte size of the adjacency region for a batch (closed-form per-task
// offsets: every list entry is 4 bytes).
__host__ __device__ inline int64_t sim_adj_bytes(int64_t T, int64_t I, int64_t O, int64_t E) {
    (void)T;
    return 4 * I + 4 * O + 4 * E + 16;
}

struct SimParams {
    DevBatch b;
    const DevPlatform* platforms;
    const int32_t* platform_of;       // [G] or null
    int32_t policy;
    const tbsim_regulator_cfg* reg;   // [G] or null -> default from median
    const double* median;             // [G] lower-median GPU time (default cfg)
    int32_t median_stride;            // elements between consecutive graphs' medians
    const SimTaskHdr* hdr;            // [T] packed task records (k_sim_pack)
    const int32_t* adj;               // packed per-task lists
    const int64_t* class_bytes;       // [kByteClasses] the batch's handle-size dictionary
    const double* xtab;               // [platform][class][max_nodes][max_nodes] transfer times
    SimLog* log;                      // [T] dispatch log
    int32_t* n_disp;                  // [G] log length, -1: outputs written directly
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
    const int64_t* n_items_dev;       // or read on the device (rerun lists), when set
    unsigned long long* work_counter;
};

// Builds the packed records' structural words and lists (once per batch);
// k_sim_keys fills the pop keys of one call.  One thread per task.
template <int TL>  // lanes per task (8 instantiated)
__global__ void k_sim_pack(DevBatch b, const uint8_t* hcls, SimTaskHdr* hdr, int32_t* adj);
__global__ void k_bytes_class(DevBatch b, const int64_t* dict, uint8_t* hcls);
// k_ingest and k_sim_pack of an uploaded batch in one pass per graph
__global__ void k_ingest_pack(DevBatch b, int32_t* cursor_scratch, int32_t smem_ints, const uint8_t* hcls,
                              SimTaskHdr* hdr, int32_t* adj);
// The batch's distinct handle sizes (first come, first numbered; at most
// kEscapeClass of them, the rest read handle_bytes).  dict: kByteClasses
// entries preset to kDictEmpty.
__global__ void k_bytes_dict(DevBatch b, unsigned long long* dict);
// Transfer time of every (platform, class, source node, destination node):
// Platform::transfer_time_ms (platform.cpp:56-63), 0 on the same node.
__global__ void k_xfer_table(const DevPlatform* pf, int32_t n_platforms, const int64_t* dict, int32_t mn,
                             double* xtab);
__global__ void k_sim_keys(DevBatch b, const int64_t* ability, const int64_t* efficiency, const int64_t* prio,
                           int32_t policy, SimTaskHdr* hdr);
// Moves the dispatch logs into worker/start/end; one thread per log slot.
__global__ void k_sim_collect_reruns(int64_t G, const int32_t* status, int32_t* list, int64_t* n);
__global__ void k_sim_scatter(DevBatch b, const SimLog* log, const int32_t* n_disp, int32_t* worker, double* start_ms,
                              double* end_ms);

__global__ void k_simulate_w1c(const __grid_constant__ SimParams p);  // <= 32 workers, compact state (128-thread CTAs)
__global__ void k_simulate_w1c_ins(const __grid_constant__ SimParams p);  // the same, inspirit only
__global__ void k_simulate_w1c_mi_ins(const __grid_constant__ SimParams p);
__global__ void k_simulate_w2c_ins(const __grid_constant__ SimParams p);
__global__ void k_simulate_w2c_mi_ins(const __grid_constant__ SimParams p);
__global__ void k_simulate_w1c_mi(const __grid_constant__ SimParams p);   // the same, many inputs per task
__global__ void k_simulate_w2c(const __grid_constant__ SimParams p);  // <= 64 workers, compact state
__global__ void k_simulate_w2c_mi(const __grid_constant__ SimParams p);  // the same, many inputs per task
__global__ void k_simulate_w1(const __grid_constant__ SimParams p);   // <= 32 workers, wide state
__global__ void k_simulate_w2(const __grid_constant__ SimParams p);   // <= 64 workers, wide state

}  // namespace tbsim_dev
