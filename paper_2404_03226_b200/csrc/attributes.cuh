// attributes.cuh -- scratch layout and launch interface of the attribute kernels.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace tbsim_dev {

constexpr int kMaxTile = 256;                 // widest sweep tile (FP32 windows)
constexpr int32_t kTileWidthMask = 0xffff;    // tile_s: sources per tile ...
constexpr int32_t kTileF32 = 1 << 16;         // ... | FP32-exact window

enum SweepMode : int32_t {
    SWEEP_CALIBRATE = 0,  // 11-window calibration grid (also final efficiency + ability)
    SWEEP_SINGLE = 1,     // efficiency at a caller-given window (unit_time_ms[g])
    SWEEP_ABILITY = 2,    // reachable counts only
};

struct GraphInfo {
    int32_t n_levels;    // topological layers (0 for an empty graph)
    int32_t processed;   // tasks released by Kahn (< n means a cycle)
    int32_t peak_slots;  // distance-column slots the sweep needs
    int32_t n_classes;   // distinct (layer, type) calibration classes
    int32_t peak_rslots; // bitset slots of the reverse closure (large-graph path)
    int32_t max_span;    // max level(v) - level(u) over edges (large-graph path)
    int32_t miss_gpu;    // first task position without a GPU cost, -1 if none
    int32_t miss_any;    // first task position without any cost, -1 if none
    int32_t order_det;   // level order sorted by position inside each level (large-graph path)
    int32_t miss_types;  // type ids of the miss_gpu / miss_any tasks (bits 0-15 / 16-31), for error texts
    uint64_t gpu_types;  // task types present (with a GPU time): bit t
    double median;       // lower-median GPU time (valid when miss_gpu < 0 and n > 0)
};

// Device scratch of one attribute pass over a batch (T tasks, E edges,
// G graphs, NT types).
struct AttrScratch {
    int32_t* tmp;        // [T+G]
    int32_t* tmp2;       // [T+G]
    int32_t* order;      // [T]  level order (local positions)
    int32_t* level;      // [T]
    int32_t* lstart;     // [T+G] per graph n_levels+1 offsets into order
    int32_t* height;     // [T]
    int32_t* lastuse;    // [T]
    int32_t* slot;       // [T]
    int32_t* rel_order;  // [T]
    int32_t* fstack;     // [T]
    int32_t* cls;        // [T]
    int32_t* cls_mark;   // [T*NT]
    int32_t* opos;       // [T] order position of each node (large-graph path)
    int32_t* firstuse;   // [T] lowest level of a predecessor (large-graph path)
    int32_t* rslot;      // [T] reverse-closure slot (large-graph path)
    int32_t* om_slot;    // [T]   order-major: slot of the node at level-order position i
    double* om_gpu;      // [T]   order-major: GPU time of that node
    int32_t* om_poff;    // [T+G] order-major CSR offsets of predecessor slots
    int32_t* om_pslot;   // [E]   order-major predecessor slots
    double* rank;        // [T]
    uint32_t* hist;      // [12T] window-bin counts per source (kBins x uint32, 16-B aligned rows)
    GraphInfo* info;     // [G]
    double* median;      // [G] lower-median GPU time (regulator defaults)
    int64_t* tile_base;  // [G+1]
    int32_t* tile_s;     // [G]
    int32_t* tile_graph; // [tiles] graph of each sweep tile (<= T/8 + G)
    int32_t* plan_fp32;  // [2] every tile is an FP32-exact shape k_sweep_fp32 runs; max P of global-window graphs
};

// Grid-wide counters of k_structure_large (zeroed before the launch),
// followed by gridDim.x ints of scan partials.
struct LargeCtl {
    int32_t ctr[4];      // rotating per-level append counters
    int32_t miss_gpu;    // max (n - v) over tasks without a GPU cost (0: none)
    int32_t miss_any;    // same, tasks without any cost
    int32_t span;        // max level(v) - level(u) over edges
    int32_t ring;        // widest window of span+1 consecutive levels
    int32_t wide2;       // widest window of two consecutive levels
    int32_t unsorted;    // a level too wide for the deterministic in-level sort
    int32_t pad[6];
    int32_t tcount[kMaxTypes];
    int32_t part[1];     // [gridDim.x]
};

struct AttrOutDev {
    int64_t* ability;
    int64_t* efficiency;
    int64_t* static_priority;
    int64_t* depth;
    int32_t* layer;
    double* unit_time_ms;
    double* w0_ms;
    int64_t* best_score;
    int64_t* w0_score;
    int32_t* evaluations;
};

__global__ void k_ingest(DevBatch b, int32_t* cursor_scratch, int32_t smem_ints);
// smem_ints: dynamic shared ints, two halves (in-degrees / allocator counts,
// allocator cursors), used when n+1 fit in a half
__global__ void k_structure(DevBatch b, const DevCosts* costs, const int32_t* cost_idx, AttrScratch s,
                            int32_t want_rank, int32_t want_large, int32_t smem_ints);
__global__ void k_structure_large(DevBatch b, const DevCosts* costs, const int32_t* cost_idx, AttrScratch s,
                                  int32_t want_rank, LargeCtl* ctl, int32_t sort_levels);
__global__ void k_tile_plan(DevBatch b, AttrScratch s, int64_t smem_bytes, int32_t force_s, const DevCosts* costs,
                            const int32_t* cost_idx, int32_t sweep_mode);
__global__ void k_sweep(DevBatch b, const DevCosts* costs, const int32_t* cost_idx, AttrScratch s,
                        int32_t sweep_mode,
                        const double* unit_time, int64_t total_tiles, unsigned long long* work_counter,
                        int64_t smem_bytes, double* gwin, int64_t gwin_stride, int32_t prune,
                        unsigned long long* relax_ctr);
__global__ void k_sweep_fp32(DevBatch b, AttrScratch s, int32_t sweep_mode, const double* unit_time,
                             unsigned long long* work_counter, int32_t prune, unsigned long long* relax_ctr);
__global__ void k_finalize(DevBatch b, AttrScratch s, int32_t sweep_mode, const double* unit_time_in,
                           AttrOutDev o, int64_t* cls_scratch, int64_t cls_stride, int32_t write_ability);
enum FinPhase : int32_t { FIN_ALL = 0, FIN_PARTIAL = 1, FIN_FINISH = 2 };
__global__ void k_finalize_large(DevBatch b, AttrScratch s, int32_t sweep_mode, AttrOutDev o, int64_t* scratch,
                                 int32_t* tab, int64_t tab_cap, int32_t* score, int32_t write_ability, int32_t phase,
                                 int32_t pos_lo, int32_t pos_hi, const int64_t* sums_in);
template <int kStages, int CH, int kWarps>  // stages of CH x 256 B per warp (TMA bulk copies)
__global__ void k_closure_tma(DevBatch b, AttrScratch s, int64_t g, uint64_t* sets, int64_t wlo, int64_t whi,
                              unsigned long long* ability);
template <int CH>  // words per lane
__global__ void k_closure(DevBatch b, AttrScratch s, int64_t g, uint64_t* sets, int64_t wlo, int64_t whi,
                          unsigned long long* ability);
__global__ void k_structure_out(DevBatch b, AttrScratch s, AttrOutDev o, int32_t prio_kind,
                                int32_t want_prio);
// probe.cu: the sweep's inner loop alone (its roofline denominator)
__global__ void k_probe_relax(int32_t rows_mask, int32_t iters, double* out);
__global__ void k_probe_relax_f32(int32_t rows_mask, int32_t iters, double* out);

}  // namespace tbsim_dev
