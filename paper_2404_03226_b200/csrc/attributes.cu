// attributes.cu -- CSR ingestion and the attribute kernels of the INSPIRIT
// hot path (reference: src/taskgraph.cpp, src/attributes.cpp).
//
//   k_ingest     successor CSR from the dependency CSR (build_index,
//                taskgraph.cpp:11-43): counting sort + per-list sort, so every
//                succ list is ascending with multi-edges kept.
//   k_structure  one CTA per graph: level-synchronous Kahn frontiers
//                (topological_layers, taskgraph.cpp:197-219) producing a
//                level order; reverse level sweep for height (= depth_priority,
//                attributes.cpp:255-265) and HEFT upward rank
//                (attributes.cpp:234-253); lower-median GPU time
//                (platform.cpp:233-240); (layer,type) calibration classes
//                (attributes.cpp:193-201); and a live-range slot assignment
//                for the source sweep.
//   k_sweep      the efficiency kernel.  One CTA per (graph, tile of S
//                sources): a forward max-plus sweep over the level order with
//                the sources' distance columns resident in shared memory.
//                dist(s,v) = gpu[v] + max_{u in pred(v)} dist(s,u) reproduces
//                efficiency_of (attributes.cpp:110-137) bit-for-bit because FP64
//                rounding is monotone, so max(a+g, b+g) == max(a,b)+g.  One pass
//                bins every reachable descendant by the first calibration window
//                it fits (k = -4..6, attributes.cpp:221-230), which yields all
//                11 calibration evaluations, the final efficiency and the
//                inspiring ability (reachable count, attributes.cpp:57-92) at once.
//   k_finalize   per graph: per-class sums for each window, distinct reduced
//                fractions (attributes.cpp:205-217), the strict-> winner, and the
//                per-task efficiency / ability.
#include <cooperative_groups.h>
#include <math_constants.h>

#include <cfloat>
#include <cstdint>

#include "attributes.cuh"
#include "blockscan.cuh"
#include "common.cuh"
#include "ingest.cuh"
#include "rules.cuh"

namespace tbsim_dev {

// ------------------------------------------------------------------ ingest

// Successor CSR of each graph (one CTA per graph, ingest.cuh).
__global__ void __launch_bounds__(256) k_ingest(DevBatch b, int32_t* cursor_scratch, int32_t smem_ints) {
    __shared__ int32_t warp_tot[32];
    extern __shared__ int32_t s_ctr[];
    for (int64_t g = blockIdx.x; g < b.G; g += gridDim.x) ingest_graph(b, g, cursor_scratch, smem_ints, s_ctr, warp_tot);
}

// --------------------------------------------------------------- structure

// Live-range slot assignment over the level order.  Nodes of a level take
// free slots (stack) or fresh ones; a node's slot is released after level
// key[v] has been processed.  reverse = walk levels from the last to the
// first.  Returns the number of slots used (peak live set).
// order/lstart/key are read through L2 (__ldcg): in the cooperative
// large-graph kernel they were written by other CTAs earlier in the launch.
__device__ int32_t assign_slots(const int32_t* order, const int32_t* lstart, int32_t L, int32_t processed,
                                const int32_t* key, bool reverse, int32_t* slot, int32_t* cnt, int32_t* cur,
                                int32_t* rel_order, int32_t* fstack, int32_t* warp_tot) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    for (int32_t i = tid; i <= L; i += nthr) cnt[i] = 0;
    __syncthreads();
    for (int32_t i = tid; i < processed; i += nthr) atomicAdd(&cnt[__ldcg(&key[__ldcg(&order[i])])], 1);
    __syncthreads();
    block_exclusive_scan_inplace(cnt, L + 1, warp_tot);
    for (int32_t i = tid; i <= L; i += nthr) cur[i] = cnt[i];
    __syncthreads();
    for (int32_t i = tid; i < processed; i += nthr) {
        const int32_t v = __ldcg(&order[i]);
        rel_order[atomicAdd(&cur[__ldcg(&key[v])], 1)] = v;
    }
    __syncthreads();
    int32_t fs = 0, P = 0;
    for (int32_t step = 0; step < L; ++step) {
        const int32_t lv = reverse ? L - 1 - step : step;
        const int32_t a0 = __ldcg(&lstart[lv]), a = __ldcg(&lstart[lv + 1]) - a0;
        for (int32_t i = tid; i < a; i += nthr) slot[__ldcg(&order[a0 + i])] = i < fs ? fstack[fs - 1 - i] : P + (i - fs);
        __syncthreads();
        const int32_t nfs = max(fs - a, 0);
        P += max(a - fs, 0);
        const int32_t r0 = cnt[lv], r = cnt[lv + 1] - r0;
        for (int32_t j = tid; j < r; j += nthr) fstack[nfs + j] = slot[rel_order[r0 + j]];
        __syncthreads();
        fs = nfs + r;
    }
    return P;
}

// median_gpu_time_ms (platform.cpp:233-240): the lower median of the tasks'
// GPU times, from the per-type task counts -- present types sorted by GPU
// time, counts walked to rank (n-1)/2.
__device__ double lower_median_gpu(const DevCosts& sc, const int32_t* tcount, int32_t NT, int32_t n) {
    int32_t ids[kMaxTypes];
    int32_t m = 0;
    for (int32_t t = 0; t < NT && t < kMaxTypes; ++t)
        if (tcount[t] > 0) {
            int32_t j = m++;
            while (j > 0 && sc.gpu[ids[j - 1]] > sc.gpu[t]) { ids[j] = ids[j - 1]; --j; }
            ids[j] = t;
        }
    const int32_t want = (n - 1) / 2;
    int32_t acc = 0;
    for (int32_t j = 0; j < m; ++j) {
        acc += tcount[ids[j]];
        if (acc > want) return sc.gpu[ids[j]];
    }
    return 0.0;
}

// Cost table of graph g into shared memory, plus mean_ms per type
// (platform.cpp:39-50: ((0 + cpu) + gpu) / count).
__device__ void load_costs(const DevCosts* costs_g, int32_t ci, DevCosts& sc, double* s_mean) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    __syncthreads();
    for (int i = tid; i < static_cast<int>(sizeof(DevCosts) / 8); i += nthr)
        reinterpret_cast<double*>(&sc)[i] = reinterpret_cast<const double*>(costs_g + ci)[i];
    __syncthreads();
    if (tid < kMaxTypes) {
        const bool in = tid < sc.n_types;
        s_mean[tid] = tbsim_rules::mean_cost_ms(in && sc.cpu[tid] > 0.0, sc.cpu[tid], in && sc.gpu[tid] > 0.0,
                                                sc.gpu[tid]);
    }
    __syncthreads();
}

// Warp-aggregated append of the lanes with `pred` to list[base + *ctr ...]
// (any active-lane mask).  Returns the slot of this lane (or -1).
__device__ __forceinline__ int32_t warp_append(bool pred, int32_t* ctr) {
    const unsigned am = __activemask();
    const unsigned bal = __ballot_sync(am, pred);
    if (!bal) return -1;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(am) - 1;
    int32_t base = 0;
    if (lane == leader) base = atomicAdd(ctr, __popc(bal));
    base = __shfl_sync(am, base, leader);
    return pred ? base + __popc(bal & ((1u << lane) - 1u)) : -1;
}

__global__ void __launch_bounds__(512) k_structure(DevBatch b, const DevCosts* costs_g,
                                                  const int32_t* cost_idx, AttrScratch s,
                                                  int32_t want_rank, int32_t want_large, int32_t smem_ints) {
    // [smem_ints]: Kahn's in-degrees (later the slot allocator's counts) in
    // the first half, the allocator's cursors in the second, when n + 1 fit
    extern __shared__ int32_t s_indeg[];
    __shared__ DevCosts sc;
    __shared__ double s_mean[kMaxTypes];
    __shared__ int32_t s_tcount[kMaxTypes];
    __shared__ int32_t warp_tot[32];
    __shared__ int32_t s_tail, s_end, s_miss_gpu, s_miss_any, s_span;
    constexpr int32_t kDegSortMin = 192, kDegSortMax = 1024;
    __shared__ int32_t s_key[kDegSortMax];
    const int tid = threadIdx.x, nthr = blockDim.x;
    int32_t loaded = -1;
    for (int64_t g = blockIdx.x; g < b.G; g += gridDim.x) {
        const int64_t t0 = b.task_base[g];
        const int32_t n = static_cast<int32_t>(b.task_base[g + 1] - t0);
        const int32_t* doff = b.dep_off + t0 + g;
        const int32_t* dep = b.dep + b.edge_base[g];
        const int32_t* soff = b.succ_off + t0 + g;
        const int32_t* succ = b.succ + b.edge_base[g];
        const int32_t* type = b.type + t0;
        const bool in_smem = n + 1 <= smem_ints / 2;
        int32_t* indeg = in_smem ? s_indeg : s.tmp + t0 + g;
        int32_t* cursors = in_smem ? s_indeg + smem_ints / 2 : s.tmp2 + t0 + g;
        int32_t* order = s.order + t0;
        int32_t* level = s.level + t0;
        int32_t* lstart = s.lstart + t0 + g;
        int32_t* height = s.height + t0;
        int32_t* lastuse = s.lastuse + t0;
        int32_t* slot = s.slot + t0;
        double* rank = s.rank + t0;

        // cost table of this graph (per-platform tables in a schedule batch)
        const int32_t ci = cost_idx ? cost_idx[g] : 0;
        if (ci != loaded) {
            load_costs(costs_g, ci, sc, s_mean);
            loaded = ci;
        }
        const int32_t NT = b.n_types;
        if (tid == 0) { s_tail = 0; s_miss_gpu = INT32_MAX; s_miss_any = INT32_MAX; }
        if (tid < kMaxTypes) s_tcount[tid] = 0;
        __syncthreads();
        // ---- entries, cost diagnostics, type histogram
        for (int32_t v = tid; v < n; v += nthr) {
            indeg[v] = doff[v + 1] - doff[v];
            level[v] = 0;
            const int32_t ty = type[v];
            const bool has_gpu = ty < NT && sc.gpu[ty] > 0.0;
            const bool has_cpu = ty < NT && sc.cpu[ty] > 0.0;
            if (!has_gpu) atomicMin(&s_miss_gpu, v);
            if (!has_gpu && !has_cpu) atomicMin(&s_miss_any, v);
            if (has_gpu) atomicAdd(&s_tcount[ty], 1);
            const int32_t at = warp_append(indeg[v] == 0, &s_tail);  // frontier: ballot + popc, one atomic per warp
            if (at >= 0) order[at] = v;
        }
        // ---- level-synchronous Kahn (topological_layers)
        int32_t head = 0, L = 0;
        if (tid == 0) lstart[0] = 0;
        for (;;) {
            __syncthreads();
            if (tid == 0) s_end = s_tail;
            __syncthreads();
            const int32_t end = s_end;
            if (end == head) break;
            if (tid == 0) lstart[L + 1] = end;
            for (int32_t i = head + tid; i < end; i += nthr) {
                const int32_t u = order[i];
                const int32_t k1 = soff[u + 1];
                for (int32_t k = soff[u]; k < k1; k += 4) {  // successor ids loaded four at a time
                    int32_t vv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) vv[q] = k + q < k1 ? succ[k + q] : -1;
                    // per-thread shared-memory appends: a warp-aggregated
                    // append (ballot + popc, one atomic per warp) per
                    // successor measured slower here (C2 0.57 -> 0.60 ms);
                    // the whole-GPU k_structure_large uses it
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int32_t v = vv[q];
                        if (v >= 0 && atomicSub(&indeg[v], 1) == 1) {
                            level[v] = L + 1;
                            order[atomicAdd(&s_tail, 1)] = v;
                        }
                    }
                }
            }
            head = end;
            ++L;
        }
        const int32_t processed = head;
        // ---- wide levels sorted by in-degree (bitonic, shared memory): the
        // sweep's row tiles (8 or 4 lanes per node, chosen for graphs whose
        // live window is wide) give a warp consecutive nodes, which then have
        // equal predecessor counts; one-node-per-warp tiles of narrow graphs
        // do not need it (as k_structure_large).  Descending: C5 sweep 280 ->
        // 270 ms against ascending; C2's 100-node levels sorted either way
        // measured slower (4.32 -> 4.63 ms), hence the 192-node floor.
        for (int32_t lv = 0; lv < L; ++lv) {
            const int32_t a0 = lstart[lv], m = lstart[lv + 1] - a0;
            if (m < kDegSortMin || m > kDegSortMax) continue;  // uniform
            int32_t N = 1;
            while (N < m) N <<= 1;
            for (int32_t i = tid; i < N; i += nthr) {
                int32_t key = INT32_MAX;
                if (i < m) {
                    const int32_t v = order[a0 + i];
                    key = ((127 - min(doff[v + 1] - doff[v], 127)) << 24) | v;  // n < 2^24, deg descending
                }
                s_key[i] = key;
            }
            __syncthreads();
            for (int32_t k = 2; k <= N; k <<= 1) {
                for (int32_t j = k >> 1; j > 0; j >>= 1) {
                    for (int32_t i = tid; i < N; i += nthr) {
                        const int32_t ixj = i ^ j;
                        if (ixj > i) {
                            const int32_t x = s_key[i], y = s_key[ixj];
                            if ((x > y) == ((i & k) == 0)) { s_key[i] = y; s_key[ixj] = x; }
                        }
                    }
                    __syncthreads();
                }
            }
            for (int32_t i = tid; i < m; i += nthr) order[a0 + i] = s_key[i] & 0xffffff;
            __syncthreads();
        }
        // ---- reverse level sweep: height (depth), upward rank, last use
        for (int32_t lv = L - 1; lv >= 0; --lv) {
            for (int32_t i = lstart[lv] + tid; i < lstart[lv + 1]; i += nthr) {
                const int32_t u = order[i];
                int32_t h = 0, lu = lv;
                double best = 0.0;
                const int32_t k1 = soff[u + 1];
                for (int32_t k = soff[u]; k < k1; k += 4) {  // four successors' records in flight
                    int32_t vv[4], hv[4], lvv[4];
                    double rv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) vv[q] = k + q < k1 ? succ[k + q] : -1;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        hv[q] = vv[q] >= 0 ? height[vv[q]] : -1;
                        rv[q] = vv[q] >= 0 ? rank[vv[q]] : 0.0;
                        lvv[q] = vv[q] >= 0 ? level[vv[q]] : lv;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        h = max(h, hv[q] + 1);
                        best = fmax(best, rv[q]);
                        lu = max(lu, lvv[q]);
                    }
                }
                height[u] = h;
                lastuse[u] = lu;
                if (want_rank) rank[u] = s_mean[type[u] < kMaxTypes ? type[u] : 0] + best;
            }
            __syncthreads();
        }
        // ---- live-range slots for the forward sweep (released after the
        //      node's last consumer level)
        const int32_t P = assign_slots(order, lstart, L, processed, lastuse, false, slot, indeg, cursors,
                                       s.rel_order + t0, s.fstack + t0, warp_tot);
        // ---- large graphs: inverse order, edge level span, reverse slots for
        //      the bitset closure (released after the node's first consumer)
        int32_t Pr = 0;
        if (want_large) {
            int32_t* opos = s.opos + t0;
            int32_t* firstuse = s.firstuse + t0;
            if (tid == 0) s_span = 1;
            __syncthreads();
            for (int32_t i = tid; i < processed; i += nthr) opos[order[i]] = i;
            for (int32_t v = tid; v < n; v += nthr) {
                int32_t fu = level[v];
                for (int32_t k = doff[v]; k < doff[v + 1]; ++k) {
                    const int32_t lu = level[dep[k]];
                    fu = min(fu, lu);
                    if (level[v] - lu > 1) atomicMax(&s_span, level[v] - lu);
                }
                firstuse[v] = fu;
            }
            __syncthreads();
            Pr = assign_slots(order, lstart, L, processed, firstuse, true, s.rslot + t0, indeg, cursors,
                              s.rel_order + t0, s.fstack + t0, warp_tot);
        }
        // ---- order-major node records for the sweep: slot, GPU time and
        //      the predecessors' slots, contiguous in level order
        int32_t* om_slot = s.om_slot + t0;
        double* om_gpu = s.om_gpu + t0;
        int32_t* om_poff = s.om_poff + t0 + g;
        int32_t* om_ps = s.om_pslot + b.edge_base[g];
        for (int32_t i = tid; i < processed; i += nthr) {
            const int32_t v = order[i];
            om_slot[i] = slot[v];
            const int32_t ty = type[v];
            om_gpu[i] = ty < NT ? sc.gpu[ty] : 0.0;
            om_poff[i] = doff[v + 1] - doff[v];
        }
        if (tid == 0) om_poff[processed] = 0;
        __syncthreads();
        block_exclusive_scan_inplace(om_poff, processed + 1, warp_tot);
        for (int32_t i = tid; i < processed; i += nthr) {
            const int32_t v = order[i];
            const int32_t o = om_poff[i] - doff[v];
            const int32_t k1 = doff[v + 1];
            // four predecessors at a time: loads issued before the stores
            for (int32_t k = doff[v]; k < k1; k += 4) {
                int32_t d[4], sl[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) d[u] = k + u < k1 ? dep[k + u] : 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) sl[u] = k + u < k1 ? slot[d[u]] : 0;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (k + u < k1) om_ps[o + k + u] = sl[u];
            }
        }
        // ---- calibration classes: dense ids of present (layer, type) pairs
        int32_t* mark = s.cls_mark + t0 * NT;   // [L * NT] <= n * NT
        const int64_t nkeys = static_cast<int64_t>(L) * NT;
        for (int64_t i = tid; i < nkeys; i += nthr) mark[i] = 0;
        __syncthreads();
        for (int32_t v = tid; v < n; v += nthr) {
            const int32_t ty = type[v];
            if (ty < NT) mark[static_cast<int64_t>(level[v]) * NT + ty] = 1;
        }
        __syncthreads();
        int32_t n_cls = 0;
        {
            // exclusive scan over nkeys (int64 length, int32 values)
            int32_t carry = 0;
            for (int64_t base = 0; base < nkeys; base += nthr) {
                const int64_t i = base + tid;
                int32_t x = i < nkeys ? mark[i] : 0;
                int32_t tot;
                int32_t inc = block_inclusive_scan(x, warp_tot, &tot);
                if (i < nkeys) mark[i] = carry + inc - x;
                carry += tot;
            }
            n_cls = carry;
        }
        __syncthreads();
        for (int32_t v = tid; v < n; v += nthr) {
            const int32_t ty = type[v];
            s.cls[t0 + v] = ty < NT ? mark[static_cast<int64_t>(level[v]) * NT + ty] : 0;
        }
        // ---- per-graph scalars: lower median of GPU times
        if (tid == 0) {
            GraphInfo gi;
            gi.n_levels = L;
            gi.processed = processed;
            gi.peak_slots = P;
            gi.peak_rslots = Pr;
            gi.max_span = want_large ? s_span : 0;
            gi.n_classes = n_cls;
            gi.miss_gpu = s_miss_gpu == INT32_MAX ? -1 : s_miss_gpu;
            gi.miss_any = s_miss_any == INT32_MAX ? -1 : s_miss_any;
            gi.order_det = 0;
            gi.miss_types = (gi.miss_gpu >= 0 ? type[gi.miss_gpu] : 0) | ((gi.miss_any >= 0 ? type[gi.miss_any] : 0) << 16);
            gi.gpu_types = 0;
            for (int t = 0; t < kMaxTypes; ++t)
                if (s_tcount[t] > 0) gi.gpu_types |= 1ull << t;
            gi.median = (n > 0 && gi.miss_gpu < 0) ? lower_median_gpu(sc, s_tcount, NT, n) : 0.0;
            s.info[g] = gi;
            s.median[g] = gi.median;
        }
        __syncthreads();
    }
}

// ------------------------------------------------- structure, one large graph

namespace cg = cooperative_groups;

// Exclusive scan of a[0..len) in place across a cooperative grid: each CTA
// owns one contiguous chunk; chunk totals go through part[gridDim.x].
// Returns the grand total.  All threads of the grid must call it.
__device__ int32_t grid_exclusive_scan(cg::grid_group& grid, int32_t* a, int64_t len, int32_t* part,
                                       int32_t* warp_tot) {
    const int64_t nb = gridDim.x;
    const int64_t chunk = (len + nb - 1) / nb;
    const int64_t lo = min(len, static_cast<int64_t>(blockIdx.x) * chunk), hi = min(len, lo + chunk);
    int32_t sum = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) sum += __ldcg(&a[i]);
    int32_t tot;
    block_inclusive_scan(sum, warp_tot, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
    grid.sync();
    int32_t before = 0, all = 0;
    for (int64_t j = threadIdx.x; j < nb; j += blockDim.x) {
        const int32_t x = __ldcg(&part[j]);
        all += x;
        if (j < blockIdx.x) before += x;
    }
    int32_t carry, total;
    block_inclusive_scan(before, warp_tot, &carry);  // CTA sums: chunks before this one
    block_inclusive_scan(all, warp_tot, &total);
    for (int64_t base = lo; base < hi; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int32_t x = i < hi ? __ldcg(&a[i]) : 0;
        int32_t t;
        const int32_t inc = block_inclusive_scan(x, warp_tot, &t);
        if (i < hi) a[i] = carry + inc - x;
        carry += t;
    }
    grid.sync();
    return total;
}

__device__ __forceinline__ double warp_max_f64(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// k_structure for ONE graph with the whole GPU (cooperative launch): the
// same outputs as k_structure (levels, level order, height/depth, upward
// rank, live-range slots, order-major records, calibration classes, lower
// median), level-synchronous across the grid with one grid barrier per level
// instead of one CTA walking a million-task graph.  A warp owns a frontier
// node, its lanes the node's successors (warp-aggregated appends to the next
// level).  Level order inside a level is arbitrary; every consumer is
// order-free (max-plus, max, set union).  Live-range slots: when every live
// set fits in a ring over level-order positions (R = widest window of
// span+1 consecutive levels, at most twice the widest two-level window),
// slot = position mod R -- a node is live only while positions within R of
// it are being processed; otherwise CTA 0 runs the stack allocator.
// Everything written by other CTAs inside this launch is read through L2.
__global__ void __launch_bounds__(512) k_structure_large(DevBatch b, const DevCosts* costs_g, const int32_t* cost_idx,
                                                        AttrScratch s, int32_t want_rank, LargeCtl* ctl,
                                                        int32_t sort_levels) {
    cg::grid_group grid = cg::this_grid();
    constexpr int32_t kSortLevel = 4096;  // widest level sorted in shared memory
    __shared__ int32_t s_sort[kSortLevel];
    __shared__ DevCosts sc;
    __shared__ double s_mean[kMaxTypes];
    __shared__ int32_t s_tc[kMaxTypes];
    __shared__ int32_t warp_tot[32];
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * nthr + tid;
    const int64_t gthreads = static_cast<int64_t>(gridDim.x) * nthr;
    const int64_t gwarp = gtid >> 5, gwarps = gthreads >> 5;
    constexpr int64_t g = 0;
    const int64_t t0 = b.task_base[g];
    const int32_t n = static_cast<int32_t>(b.task_base[g + 1] - t0);
    const int32_t* doff = b.dep_off + t0 + g;
    const int32_t* dep = b.dep + b.edge_base[g];
    const int32_t* soff = b.succ_off + t0 + g;
    const int32_t* succ = b.succ + b.edge_base[g];
    const int32_t* type = b.type + t0;
    int32_t* indeg = s.tmp + t0 + g;
    int32_t* order = s.order + t0;
    int32_t* level = s.level + t0;
    int32_t* lstart = s.lstart + t0 + g;
    int32_t* height = s.height + t0;
    int32_t* lastuse = s.lastuse + t0;
    int32_t* slot = s.slot + t0;
    int32_t* opos = s.opos + t0;
    int32_t* firstuse = s.firstuse + t0;
    int32_t* rslot = s.rslot + t0;
    double* rank = s.rank + t0;
    const int32_t NT = b.n_types;

    load_costs(costs_g, cost_idx ? cost_idx[g] : 0, sc, s_mean);
    if (tid < kMaxTypes) s_tc[tid] = 0;
    __syncthreads();
    // ---- entries, cost diagnostics, type histogram, roots
    for (int64_t v = gtid; v < n; v += gthreads) {
        const int32_t deg = doff[v + 1] - doff[v];
        indeg[v] = deg;
        level[v] = 0;
        const int32_t ty = type[v];
        const bool has_gpu = ty < NT && sc.gpu[ty] > 0.0;
        const bool has_cpu = ty < NT && sc.cpu[ty] > 0.0;
        if (!has_gpu) atomicMax(&ctl->miss_gpu, n - static_cast<int32_t>(v));
        if (!has_gpu && !has_cpu) atomicMax(&ctl->miss_any, n - static_cast<int32_t>(v));
        if (has_gpu) atomicAdd(&s_tc[ty], 1);
        const int32_t at = warp_append(deg == 0, &ctl->ctr[0]);
        if (at >= 0) order[at] = static_cast<int32_t>(v);
    }
    __syncthreads();
    if (tid < kMaxTypes && s_tc[tid]) atomicAdd(&ctl->tcount[tid], s_tc[tid]);
    grid.sync();
    // ---- level-synchronous Kahn (topological_layers, taskgraph.cpp:197-219).
    // Three rotating counters: level L appends to ctr[(L+1)%3] while
    // ctr[(L+2)%3] (read two levels ago) is reset.
    int32_t begin = 0, L = 0;
    int32_t cnt = __ldcg(&ctl->ctr[0]);
    if (gtid == 0) lstart[0] = 0;
    while (cnt > 0) {
        const int32_t end = begin + cnt;
        if (gtid == 0) {
            lstart[L + 1] = end;
            ctl->ctr[(L + 2) % 3] = 0;
        }
        int32_t* nxt = &ctl->ctr[(L + 1) % 3];
        for (int64_t i = begin + gwarp; i < end; i += gwarps) {
            const int32_t u = __ldcg(&order[i]);
            const int32_t k1 = soff[u + 1];
            for (int32_t k = soff[u] + lane; k - lane < k1; k += 32) {
                bool rdy = false;
                int32_t v = 0;
                if (k < k1) {
                    v = succ[k];
                    rdy = atomicSub(&indeg[v], 1) == 1;
                }
                const int32_t at = warp_append(rdy, nxt);
                if (at >= 0) {
                    level[v] = L + 1;
                    order[end + at] = v;
                }
            }
        }
        grid.sync();
        begin = end;
        ++L;
        cnt = __ldcg(&ctl->ctr[L % 3]);
    }
    const int32_t processed = begin;
    // ---- level order: each level's nodes sorted in shared memory (bitonic,
    // a CTA per level).  The atomic appends above leave an arbitrary order
    // inside a level and every single-GPU consumer is order-free, so one GPU
    // sorts by in-degree: the sweep's lane groups take consecutive nodes, so
    // a warp's nodes then have equal predecessor counts and its relaxation
    // loop runs without idle lanes.  Ranks sharing one graph's bit space
    // (sharded closure) must agree on every node's bit index: they sort by
    // position.
    for (int32_t lv = blockIdx.x; lv < L; lv += gridDim.x) {
        const int32_t a0 = __ldcg(&lstart[lv]), m = __ldcg(&lstart[lv + 1]) - a0;
        if (m > kSortLevel) {
            if (sort_levels && tid == 0) atomicMax(&ctl->unsorted, 1);
            continue;  // uniform per CTA
        }
        if (m <= 1) continue;
        int32_t N = 1;
        while (N < m) N <<= 1;
        // key: position (n < 2^24), or in-degree (clipped at 127) above it
        for (int32_t i = tid; i < N; i += nthr) {
            int32_t key = INT32_MAX;
            if (i < m) {
                const int32_t v = __ldcg(&order[a0 + i]);
                key = sort_levels ? v : ((127 - min(doff[v + 1] - doff[v], 127)) << 24) | v;
            }
            s_sort[i] = key;
        }
        __syncthreads();
        for (int32_t k = 2; k <= N; k <<= 1) {
            for (int32_t j = k >> 1; j > 0; j >>= 1) {
                for (int32_t i = tid; i < N; i += nthr) {
                    const int32_t ixj = i ^ j;
                    if (ixj > i) {
                        const int32_t x = s_sort[i], y = s_sort[ixj];
                        if ((x > y) == ((i & k) == 0)) { s_sort[i] = y; s_sort[ixj] = x; }
                    }
                }
                __syncthreads();
            }
        }
        for (int32_t i = tid; i < m; i += nthr) order[a0 + i] = s_sort[i] & 0xffffff;
        __syncthreads();
    }
    grid.sync();
    // ---- reverse level sweep: height (depth), upward rank, last use
    for (int32_t lv = L - 1; lv >= 0; --lv) {
        const int32_t a0 = __ldcg(&lstart[lv]), a1 = __ldcg(&lstart[lv + 1]);
        for (int64_t i = a0 + gwarp; i < a1; i += gwarps) {
            const int32_t u = __ldcg(&order[i]);
            int32_t h = 0, lu = lv;
            double best = 0.0;
            for (int32_t k = soff[u] + lane; k < soff[u + 1]; k += 32) {
                const int32_t v = succ[k];
                h = max(h, __ldcg(&height[v]) + 1);
                best = fmax(best, __ldcg(&rank[v]));
                lu = max(lu, __ldcg(&level[v]));
            }
            h = __reduce_max_sync(0xffffffffu, h);
            lu = __reduce_max_sync(0xffffffffu, lu);
            if (want_rank) best = warp_max_f64(best);
            if (lane == 0) {
                height[u] = h;
                lastuse[u] = lu;
                if (want_rank) rank[u] = s_mean[type[u] < kMaxTypes ? type[u] : 0] + best;
            }
        }
        grid.sync();
    }
    // ---- inverse order, first use, edge level span
    for (int64_t i = gtid; i < processed; i += gthreads) opos[__ldcg(&order[i])] = static_cast<int32_t>(i);
    for (int64_t v = gtid; v < n; v += gthreads) {
        const int32_t lvv = __ldcg(&level[v]);
        int32_t fu = lvv, sp = 1;
        for (int32_t k = doff[v]; k < doff[v + 1]; ++k) {
            const int32_t lu = __ldcg(&level[dep[k]]);
            fu = min(fu, lu);
            sp = max(sp, lvv - lu);
        }
        firstuse[v] = fu;
        const unsigned am = __activemask();
        sp = __reduce_max_sync(am, sp);
        if (lane == __ffs(am) - 1) atomicMax(&ctl->span, sp);
    }
    grid.sync();
    const int32_t span = max(__ldcg(&ctl->span), 1);
    // widest window of span+1 consecutive levels (ring size), and of two
    for (int64_t lv = gtid; lv < L; lv += gthreads) {
        const int32_t hi = __ldcg(&lstart[lv + 1]);
        const int32_t r = hi - __ldcg(&lstart[lv > span ? lv - span : 0]);
        const int32_t w2 = __ldcg(&lstart[lv + 2 < L ? lv + 2 : L]) - __ldcg(&lstart[lv]);
        atomicMax(&ctl->ring, r);
        atomicMax(&ctl->wide2, w2);
    }
    grid.sync();
    const int32_t R = max(__ldcg(&ctl->ring), 1);
    const bool ring = static_cast<int64_t>(R) <= 2 * static_cast<int64_t>(max(__ldcg(&ctl->wide2), 1));
    int32_t P = R, Pr = R;
    if (ring) {
        for (int64_t i = gtid; i < processed; i += gthreads) {
            const int32_t v = __ldcg(&order[i]);
            slot[v] = static_cast<int32_t>(i % R);
            rslot[v] = static_cast<int32_t>(i % R);
        }
    } else if (blockIdx.x == 0) {
        P = assign_slots(order, lstart, L, processed, lastuse, false, slot, indeg, s.tmp2 + t0 + g,
                         s.rel_order + t0, s.fstack + t0, warp_tot);
        Pr = assign_slots(order, lstart, L, processed, firstuse, true, rslot, indeg, s.tmp2 + t0 + g,
                          s.rel_order + t0, s.fstack + t0, warp_tot);
    }
    grid.sync();
    // ---- order-major node records for the sweep
    int32_t* om_slot = s.om_slot + t0;
    double* om_gpu = s.om_gpu + t0;
    int32_t* om_poff = s.om_poff + t0 + g;
    int32_t* om_ps = s.om_pslot + b.edge_base[g];
    for (int64_t i = gtid; i < processed; i += gthreads) {
        const int32_t v = __ldcg(&order[i]);
        om_slot[i] = __ldcg(&slot[v]);
        const int32_t ty = type[v];
        om_gpu[i] = ty < NT ? sc.gpu[ty] : 0.0;
        om_poff[i] = doff[v + 1] - doff[v];
    }
    if (gtid == 0) om_poff[processed] = 0;
    grid.sync();
    grid_exclusive_scan(grid, om_poff, processed + 1, ctl->part, warp_tot);
    for (int64_t i = gtid; i < processed; i += gthreads) {
        const int32_t v = __ldcg(&order[i]);
        const int32_t o = __ldcg(&om_poff[i]) - doff[v];
        for (int32_t k = doff[v]; k < doff[v + 1]; ++k) om_ps[o + k] = __ldcg(&slot[dep[k]]);
    }
    // ---- calibration classes: dense ids of present (layer, type) pairs
    int32_t* mark = s.cls_mark + t0 * NT;
    const int64_t nkeys = static_cast<int64_t>(L) * NT;
    for (int64_t i = gtid; i < nkeys; i += gthreads) mark[i] = 0;
    grid.sync();
    for (int64_t v = gtid; v < n; v += gthreads) {
        const int32_t ty = type[v];
        if (ty < NT) mark[static_cast<int64_t>(__ldcg(&level[v])) * NT + ty] = 1;
    }
    grid.sync();
    const int32_t n_cls = grid_exclusive_scan(grid, mark, nkeys, ctl->part, warp_tot);
    for (int64_t v = gtid; v < n; v += gthreads) {
        const int32_t ty = type[v];
        s.cls[t0 + v] = ty < NT ? __ldcg(&mark[static_cast<int64_t>(__ldcg(&level[v])) * NT + ty]) : 0;
    }
    // ---- per-graph scalars
    if (blockIdx.x == 0 && tid == 0) {
        int32_t tc[kMaxTypes];
        for (int t = 0; t < kMaxTypes; ++t) tc[t] = __ldcg(&ctl->tcount[t]);
        const int32_t mg = __ldcg(&ctl->miss_gpu), ma = __ldcg(&ctl->miss_any);
        GraphInfo gi;
        gi.n_levels = L;
        gi.processed = processed;
        gi.peak_slots = P;
        gi.peak_rslots = Pr;
        gi.max_span = span;
        gi.n_classes = n_cls;
        gi.miss_gpu = mg > 0 ? n - mg : -1;
        gi.miss_any = ma > 0 ? n - ma : -1;
        gi.miss_types = (gi.miss_gpu >= 0 ? type[gi.miss_gpu] : 0) | ((gi.miss_any >= 0 ? type[gi.miss_any] : 0) << 16);
        gi.order_det = sort_levels && !__ldcg(&ctl->unsorted) ? 1 : 0;
        gi.gpu_types = 0;
        for (int t = 0; t < kMaxTypes; ++t)
            if (tc[t] > 0) gi.gpu_types |= 1ull << t;
        gi.median = (n > 0 && gi.miss_gpu < 0) ? lower_median_gpu(sc, tc, NT, n) : 0.0;
        s.info[g] = gi;
        s.median[g] = gi.median;
    }
}

// ------------------------------------------------------------------- sweep

// Window bin of a reachable distance d (attributes.cpp:124): the first k with
// d <= W_k, kBins-1 when beyond every window.  Fast path compares exponent
// and mantissa bits at once: W_k = W_0 * 2^k exactly (ldexp), so for normal
// thresholds bits(W_k) = bits(W_0) + k<<52 and non-negative doubles order
// like their bit patterns.
struct Thresholds {
    int32_t mode;       // 0: calibration grid fast path, 1: ladder, 2: ability only
    int32_t w0bits32;   // bits((float)W_0) -- FP32 windows (exact there, see k_tile_plan)
    int64_t w0bits;     // bits(W_0)
    double w[kWindows];
};

// 16 bytes of distance columns: 2 doubles or 4 floats (one LDS/STS.128).
template <typename T>
struct __align__(16) Chunk {
    static constexpr int N = 16 / static_cast<int>(sizeof(T));
    T v[N];
};

// max of two distances (-inf or non-negative, never NaN): FMNMX for FP32,
// compare-select for FP64 (no FP64 min/max instruction)
__device__ __forceinline__ float dmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

__device__ __forceinline__ int bin_of(double d, const Thresholds& th) {
    if (th.mode == 0) {
        const int64_t delta = __double_as_longlong(d) - th.w0bits;
        if (delta <= 0) return 0;
        const int64_t k = ((delta - 1) >> 52) + 1;
        return k > kWindows ? kWindows : static_cast<int>(k);
    }
    if (th.mode == 2) return kWindows;
    int k = 0;
#pragma unroll
    for (int j = 0; j < kWindows; ++j) k += d > th.w[j];
    return k;
}

__device__ Thresholds make_thresholds(int32_t mode_req, double w0_or_unit) {
    Thresholds th;
    th.w0bits32 = 0;
    if (mode_req == SWEEP_ABILITY) {
        th.mode = 2;
        th.w0bits = 0;
        for (int j = 0; j < kWindows; ++j) th.w[j] = 0.0;
        return th;
    }
    if (mode_req == SWEEP_SINGLE) {
        th.mode = 1;
        th.w0bits = 0;
        for (int j = 0; j < kWindows; ++j) th.w[j] = w0_or_unit;
        return th;
    }
    for (int j = 0; j < kWindows; ++j) th.w[j] = ldexp(w0_or_unit, j - 4);
    th.w0bits = __double_as_longlong(th.w[0]);
    th.w0bits32 = __float_as_int(static_cast<float>(th.w[0]));
    const bool normal = th.w[0] >= DBL_MIN && th.w[kWindows - 1] <= DBL_MAX;
    th.mode = normal ? 0 : 1;
    return th;
}

// Group of GL lanes handles one node for S sources (S/GL per lane).  Node
// records are read in level order (order-major arrays), the sources' distance
// columns live in shared memory: win[slot][S].
// Window bin with the threshold mode known at compile time.
// FP32 distances (exact, see k_tile_plan): W_k = W_0 * 2^k are exact floats,
// bits(W_k) = bits(W_0) + k << 23.
template <int TMODE>
__device__ __forceinline__ int bin_t(float d, const Thresholds& th) {
    if constexpr (TMODE == 0) {
        const int32_t delta = __float_as_int(d) - th.w0bits32;
        const int k = (delta + ((1 << 23) - 1)) >> 23;
        return min(max(k, 0), kWindows);
    } else if constexpr (TMODE == 2) {
        return kWindows;
    } else {
        int k = 0;
        const double dd = d;
#pragma unroll
        for (int j = 0; j < kWindows; ++j) k += dd > th.w[j];
        return k;
    }
}

template <int TMODE>
__device__ __forceinline__ int bin_t(double d, const Thresholds& th) {
    if constexpr (TMODE == 0) {
        // first k with d <= W_k: ceil(delta / 2^52) clamped to [0, 11]
        // (arithmetic shift; no overflow for any double incl. -inf, +inf)
        const int64_t delta = __double_as_longlong(d) - th.w0bits;
        const int k = static_cast<int>((delta + ((int64_t(1) << 52) - 1)) >> 52);
        return min(max(k, 0), kWindows);
    } else if constexpr (TMODE == 2) {
        return kWindows;
    } else {
        int k = 0;
#pragma unroll
        for (int j = 0; j < kWindows; ++j) k += d > th.w[j];
        return k;
    }
}

// Per-lane window-bin counters: 12 fields of 5 bits in one u64 per source.
// A pair that is not counted shifts by 64, which PTX defines as 0 (no
// select on the increment).  Flushed into per-bin u32 shared counters
// (native ATOMS.ADD; the 64-bit shared atomic is a CAS loop) every 31 visits.
constexpr int kFieldBits = 5;
constexpr int kFlushEvery = (1 << kFieldBits) - 1;

__device__ __forceinline__ uint64_t shl64(uint64_t x, uint32_t sh) {
    uint64_t r;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(sh));
    return r;
}

// a tile's per-source window-bin counts (s_hist[src * kBins + bin]) to the
// task-indexed scratch read by k_finalize: 12 x uint32 per task, three
// 16-byte stores per source (counts up to n - 1 < 2^24: no packing limit)
__device__ __forceinline__ void store_bins(const AttrScratch& s, int64_t t0, const int32_t* order, int32_t nsrc,
                                           const uint32_t* s_hist, int tid, int nthr) {
    for (int i = tid; i < nsrc * (kBins / 4); i += nthr) {
        const int32_t q = i / (kBins / 4), k = i - q * (kBins / 4);
        reinterpret_cast<uint4*>(s.hist + (t0 + order[q]) * kBins)[k] =
            reinterpret_cast<const uint4*>(s_hist + q * kBins)[k];
    }
}

// Final flush of a tile's packed counters without shared atomics.  The
// distance rows are dead after the last level, so each group has dumped its
// counter words there: dump[group * S + source].  One thread per (source,
// part) sums a third of the fields over all groups in registers: fields
// p, p+3, p+6, p+9 spread to 15-bit lanes (groups x 31 < 32768).
template <int S>
__device__ __forceinline__ void dump_reduce(const uint64_t* dump, int32_t ngroups, int32_t nsrc, uint32_t* s_hist) {
    static_assert(kBins == 12 && kFieldBits == 5, "three 4-field parts per counter word");
    constexpr uint64_t kPart = 0x1Full | (0x1Full << 15) | (0x1Full << 30) | (0x1Full << 45);
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * nsrc; i += blockDim.x) {
        const int sc = i / 3, p = i - 3 * sc;
        uint64_t acc = 0;
        for (int gi = 0; gi < ngroups; ++gi) acc += (dump[gi * S + sc] >> (kFieldBits * p)) & kPart;
#pragma unroll
        for (int k = 0; k < 4; ++k) s_hist[sc * kBins + p + 3 * k] += static_cast<uint32_t>(acc >> (15 * k)) & 0x7fffu;
    }
}

__device__ __forceinline__ void flush5(uint64_t& h, uint32_t* dst) {
#pragma unroll
    for (int bn = 0; bn < kBins; ++bn) {
        const uint32_t c = static_cast<uint32_t>(h >> (kFieldBits * bn)) & kFlushEvery;
        if (c) atomicAdd(&dst[bn], c);
    }
    h = 0;
}

// Group of GL lanes handles one node for S sources (S/GL per lane).  Node
// records are read in level order (order-major arrays); the sources' distance
// columns live in shared memory, win[slot][S], with each lane's pairs of
// sources interleaved across the group so every double2 access is contiguous
// over the lanes (conflict-free 128-bit LDS/STS).
// T = float: the FP32-exact window (k_tile_plan) -- half the bytes per
// column (twice the sources per tile) and FMNMX instead of compare-select.
template <int S, bool SMEM, int TMODE, typename T = double>
__device__ __forceinline__ void sweep_tile(const DevBatch& b, const AttrScratch& s, int64_t g, int32_t tile,
                                           double* gwin, int32_t P, const Thresholds& th,
                                           uint32_t* s_hist, int32_t prune_span, unsigned long long* relax_ctr) {
    extern __shared__ double win_smem[];
    T* win = SMEM ? reinterpret_cast<T*>(win_smem) : reinterpret_cast<T*>(gwin);
    uint64_t nrel = 0;  // predecessor rows relaxed (x S columns), thread 0
    constexpr int GL = S < 32 ? S : 32;   // lanes per node group
    constexpr int SPL = S / GL;           // sources per lane
    constexpr int VEC = Chunk<T>::N;      // columns per 16-byte access
    constexpr bool VECTOR = SPL >= VEC;
    constexpr int GPW = 32 / GL;          // groups per warp
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int gl = lane % GL, grp = lane / GL;
    const unsigned gmask = GL == 32 ? 0xffffffffu : (((1u << GL) - 1u) << (grp * GL));

    const int64_t t0 = b.task_base[g];
    const int32_t* lstart = s.lstart + t0 + g;
    const int32_t* om_slot = s.om_slot + t0;
    const double* om_gpu = s.om_gpu + t0;
    const int32_t* om_poff = s.om_poff + t0 + g;
    const int32_t* om_ps = s.om_pslot + b.edge_base[g];
    const GraphInfo gi = s.info[g];
    const int32_t first = tile * S;
    const int32_t nsrc = min(S, gi.processed - first);

    const T ninf = static_cast<T>(-CUDART_INF);
    {
        Chunk<T>* w2 = reinterpret_cast<Chunk<T>*>(win);
        Chunk<T> neg;
#pragma unroll
        for (int e = 0; e < VEC; ++e) neg.v[e] = ninf;  // unreachable
        for (int64_t i = threadIdx.x; i < static_cast<int64_t>(P) * (S / VEC); i += blockDim.x) w2[i] = neg;
    }
    for (int i = threadIdx.x; i < S * kBins; i += blockDim.x) s_hist[i] = 0u;
    uint64_t hist[SPL];
#pragma unroll
    for (int q = 0; q < SPL; ++q) hist[q] = 0;
    int32_t visits = 0;  // node visits since the last flush (uniform per group)
    const int32_t La = s.level[t0 + s.order[t0 + first]];
    // column of this lane's q-th source: 16-byte chunks interleaved over the
    // group's lanes (conflict-free LDS.128 / STS.128)
    auto src = [&](int q) { return VECTOR ? (q / VEC) * VEC * GL + VEC * gl + (q % VEC) : gl * SPL + q; };
    // Pruning (large graphs, ability computed elsewhere): distances only grow
    // along paths, so once no distance within the largest window was written
    // in the last `prune_span` levels (the longest edge span), no later node
    // can fall inside any window and the tile is done.
    const T wmax = static_cast<T>(th.w[kWindows - 1]);
    const uint64_t span_mask = prune_span >= 64 ? ~0ull : ((1ull << prune_span) - 1ull);
    uint64_t recent = 0;
    __syncthreads();
    // Level La holds the tile's first sources and nothing reachable from any
    // source of the tile (an edge always ends at a higher level; the tile's
    // other sources come later): its rows stay -inf except each source's own
    // distance-0 cell, so that level is written, not swept.
    {
        const int32_t e = min(first + nsrc, lstart[La + 1]);
        for (int32_t i = first + static_cast<int32_t>(threadIdx.x); i < e; i += blockDim.x)
            win[static_cast<int64_t>(__ldg(&om_slot[i])) * S + (i - first)] = static_cast<T>(0);
    }
    recent = 1;  // level La wrote distances <= wmax (the sources' zeros)
    __syncthreads();

    for (int32_t lv = La + 1; lv < gi.n_levels; ++lv) {
        int small = 0;
        const int32_t a1 = lstart[lv + 1];
        if (relax_ctr && threadIdx.x == 0) nrel += static_cast<uint64_t>(__ldg(&om_poff[a1]) - __ldg(&om_poff[lstart[lv]]));
        // groups are independent: every lane of a group sees the same node
        for (int32_t i = lstart[lv] + warp * GPW + grp; i < a1; i += nwarps * GPW) {
            const int32_t p0 = __ldg(&om_poff[i]);
            const int32_t deg = __ldg(&om_poff[i + 1]) - p0;
            const T gv = TMODE == 2 ? static_cast<T>(1) : static_cast<T>(__ldg(&om_gpu[i]));
            const int32_t sl = __ldg(&om_slot[i]);
            T m[SPL];
#pragma unroll
            for (int q = 0; q < SPL; ++q) m[q] = ninf;
            auto relax = [&](int32_t ps) {
                const T* row = win + ps * S;
                if constexpr (VECTOR) {
#pragma unroll
                    for (int q = 0; q < SPL; q += VEC) {
                        const Chunk<T> x = *reinterpret_cast<const Chunk<T>*>(row + src(q));
#pragma unroll
                        for (int e = 0; e < VEC; ++e) m[q + e] = dmax(x.v[e], m[q + e]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < SPL; ++q) m[q] = dmax(row[src(q)], m[q]);
                }
            };
            auto relax_chunk = [&](int32_t myps, int32_t lim) {
                int32_t j = 0;
                for (; j + 2 <= lim; j += 2) {  // two predecessors in flight
                    const int32_t ps0 = __shfl_sync(gmask, myps, grp * GL + j);
                    const int32_t ps1 = __shfl_sync(gmask, myps, grp * GL + j + 1);
                    relax(ps0);
                    relax(ps1);
                }
                if (j < lim) relax(__shfl_sync(gmask, myps, grp * GL + j));
            };
            if (deg <= GL) {  // the common case: one chunk of predecessors
                relax_chunk(gl < deg ? __ldg(&om_ps[p0 + gl]) : 0, deg);
            } else {
                for (int32_t c = 0; c < deg; c += GL)
                    relax_chunk((c + gl < deg) ? __ldg(&om_ps[p0 + c + gl]) : 0, min(GL, deg - c));
            }
            // unreachable stays -inf (-inf + gv); reachable distances are >= 0
            T d[SPL];
            const bool node_is_src = static_cast<uint32_t>(i - first) < static_cast<uint32_t>(S);
#pragma unroll
            for (int q = 0; q < SPL; ++q) {
                d[q] = m[q] + gv;
                const bool counted = d[q] >= static_cast<T>(0);
                const int bn = bin_t<TMODE>(d[q], th);
                hist[q] += shl64(1ull, counted ? static_cast<uint32_t>(kFieldBits * bn) : 64u);
            }
            if (node_is_src) {  // the source itself: distance 0, not its own descendant
#pragma unroll
                for (int q = 0; q < SPL; ++q)
                    if (i == first + src(q)) {
                        if (d[q] >= static_cast<T>(0))
                            hist[q] -= shl64(1ull, static_cast<uint32_t>(kFieldBits * bin_t<TMODE>(d[q], th)));
                        d[q] = static_cast<T>(0);
                    }
            }
            if (prune_span > 0) {
#pragma unroll
                for (int q = 0; q < SPL; ++q) small |= d[q] >= static_cast<T>(0) && d[q] <= wmax;
            }
            T* outp = win + sl * S;
            if constexpr (VECTOR) {
#pragma unroll
                for (int q = 0; q < SPL; q += VEC) {
                    Chunk<T> x;
#pragma unroll
                    for (int e = 0; e < VEC; ++e) x.v[e] = d[q + e];
                    *reinterpret_cast<Chunk<T>*>(outp + src(q)) = x;
                }
            } else {
#pragma unroll
                for (int q = 0; q < SPL; ++q) outp[src(q)] = d[q];
            }
            if (++visits == kFlushEvery) {
#pragma unroll
                for (int q = 0; q < SPL; ++q)
                    if (src(q) < nsrc) flush5(hist[q], s_hist + src(q) * kBins);
                visits = 0;
            }
        }
        if (prune_span > 0) {
            recent = (recent << 1) | static_cast<uint64_t>(__syncthreads_or(small) != 0);
            if (lv - La + 1 >= prune_span && (recent & span_mask) == 0) break;
        } else {
            __syncthreads();
        }
    }
    // Final flush: through the dead rows when they hold every warp's
    // counters (dump_reduce), else atomics per bin.
    if (SMEM && GPW == 1 && static_cast<int64_t>(P) * sizeof(T) >= static_cast<int64_t>(nwarps) * 8) {
        uint64_t* dump = reinterpret_cast<uint64_t*>(win);
#pragma unroll
        for (int q = 0; q < SPL; ++q) dump[warp * S + src(q)] = hist[q];
        dump_reduce<S>(dump, nwarps, nsrc, s_hist);
    } else {
#pragma unroll
        for (int q = 0; q < SPL; ++q)
            if (src(q) < nsrc) flush5(hist[q], s_hist + src(q) * kBins);
    }
    __syncthreads();
    if (relax_ctr && threadIdx.x == 0)  // [0]: FP64 windows, [1]: FP32
        atomicAdd(relax_ctr + (sizeof(T) == 4 ? 1 : 0), static_cast<unsigned long long>(nrel * S));
    store_bins(s, t0, s.order + t0 + first, nsrc, s_hist, threadIdx.x, blockDim.x);
}

// FP32 windows run only in modes 0 and 2 (k_tile_plan never picks them for
// the ladder of a caller-given window)
template <int S, bool SMEM, typename T = double>
__device__ __forceinline__ void sweep_tile_mode(const DevBatch& b, const AttrScratch& s, int64_t g, int32_t tile,
                                                double* gwin, int32_t P, const Thresholds& th,
                                                uint32_t* s_hist, int32_t prune_span, unsigned long long* rc) {
    if (th.mode == 0) sweep_tile<S, SMEM, 0, T>(b, s, g, tile, gwin, P, th, s_hist, prune_span, rc);
    else if (th.mode == 2) sweep_tile<S, SMEM, 2, T>(b, s, g, tile, gwin, P, th, s_hist, 0, rc);
    else if constexpr (sizeof(T) == 8) sweep_tile<S, SMEM, 1, T>(b, s, g, tile, gwin, P, th, s_hist, prune_span, rc);
}

// Row-per-group sweep: a group of GL lanes (GL = 1, 2, 4, 8) owns one node
// and relaxes all S distance columns of it from each predecessor's row; each
// lane holds SPL = S / GL columns in registers.  The per-node work --
// record loads, binning, the row store -- is paid once per node and lane
// for SPL sources, and predecessor slots need no shuffles (the group's lanes
// load the same address).  A lane reads its columns as NCL = SPL / 2 16-byte
// chunks, chunk ((j + rot) mod NCL) * GL + gl at step j, where rot is the
// group index: the groups of a warp start at different chunks, which spreads
// a warp's LDS.128 / STS.128 over the banks.  The accumulators stay in that
// rotated order (m[j]), so no register is indexed dynamically.  The next
// level's first node record of each group is loaded while the current level
// runs.
template <int S, int GL, int TMODE, typename T = double>
__device__ __forceinline__ void sweep_tile_rows(const DevBatch& b, const AttrScratch& s, int64_t g, int32_t tile,
                                                int32_t P, const Thresholds& th, uint32_t* s_hist,
                                                int32_t prune_span, unsigned long long* relax_ctr) {
    extern __shared__ double win_smem[];
    uint64_t nrel = 0;  // predecessor rows relaxed (x S columns), thread 0
    constexpr int VEC = Chunk<T>::N;  // columns per 16-byte chunk
    constexpr int SPL = S / GL;       // columns per lane
    constexpr int NCL = SPL / VEC;    // chunks per lane
    constexpr int NC = S / VEC;       // chunks per row
    static_assert(NCL >= 1 && (NCL & (NCL - 1)) == 0, "power-of-two chunks per lane");
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int gl = tid % GL, gidx = tid / GL, ngroups = nthr / GL;
    const int rot = gidx & (NCL - 1);
    const int64_t t0 = b.task_base[g];
    const int32_t* lstart = s.lstart + t0 + g;
    const int32_t* om_slot = s.om_slot + t0;
    const double* om_gpu = s.om_gpu + t0;
    const int32_t* om_poff = s.om_poff + t0 + g;
    const int32_t* om_ps = s.om_pslot + b.edge_base[g];
    const GraphInfo gi = s.info[g];
    const int32_t first = tile * S;
    const int32_t nsrc = min(S, gi.processed - first);
    const T ninf = static_cast<T>(-CUDART_INF);
    Chunk<T>* w2 = reinterpret_cast<Chunk<T>*>(win_smem);
    {
        Chunk<T> neg;
#pragma unroll
        for (int e = 0; e < VEC; ++e) neg.v[e] = ninf;  // unreachable
        for (int64_t i = tid; i < static_cast<int64_t>(P) * NC; i += nthr) w2[i] = neg;
    }
    for (int i = tid; i < S * kBins; i += nthr) s_hist[i] = 0u;
    uint64_t hist[SPL];  // hist[VEC*j+e]: source VEC*chunk(j)+e
#pragma unroll
    for (int q = 0; q < SPL; ++q) hist[q] = 0;
    auto chunk = [&](int j) { return ((j + rot) & (NCL - 1)) * GL + gl; };
    int32_t visits = 0;
    const int32_t La = s.level[t0 + s.order[t0 + first]];
    const T wmax = static_cast<T>(th.w[kWindows - 1]);
    const uint64_t span_mask = prune_span >= 64 ? ~0ull : ((1ull << prune_span) - 1ull);
    uint64_t recent = 0;
    struct Rec {
        int32_t p0, p1, sl;
        T gv;
    };
    auto load_rec = [&](int32_t i) {
        Rec r;
        r.p0 = __ldg(&om_poff[i]);
        r.p1 = __ldg(&om_poff[i + 1]);
        r.sl = __ldg(&om_slot[i]);
        r.gv = TMODE == 2 ? static_cast<T>(1) : static_cast<T>(__ldg(&om_gpu[i]));
        return r;
    };
    Rec nx{0, 0, 0, static_cast<T>(0)};
    if (La + 1 < gi.n_levels && lstart[La + 1] + gidx < lstart[La + 2]) nx = load_rec(lstart[La + 1] + gidx);
    __syncthreads();
    // Level La holds the tile's first sources and nothing reachable from any
    // source of the tile (an edge always ends at a higher level; the tile's
    // other sources come later): its rows stay -inf except each source's own
    // distance-0 cell, so that level is written, not swept.
    {
        const int32_t e = min(first + nsrc, lstart[La + 1]);
        for (int32_t i = first + static_cast<int32_t>(tid); i < e; i += nthr)
            reinterpret_cast<T*>(w2)[static_cast<int64_t>(__ldg(&om_slot[i])) * S + (i - first)] = static_cast<T>(0);
    }
    recent = 1;  // level La wrote distances <= wmax (the sources' zeros)
    __syncthreads();

    for (int32_t lv = La + 1; lv < gi.n_levels; ++lv) {
        int small = 0;
        const int32_t a0 = lstart[lv], a1 = lstart[lv + 1];
        const int32_t a2 = lv + 1 < gi.n_levels ? lstart[lv + 2] : a1;
        const Rec cur = nx;
        if (a1 + gidx < a2) nx = load_rec(a1 + gidx);  // next level's first node of this group
        if (relax_ctr && tid == 0) nrel += static_cast<uint64_t>(__ldg(&om_poff[a1]) - __ldg(&om_poff[a0]));
        for (int32_t i = a0 + gidx; i < a1; i += ngroups) {
            const Rec r = i == a0 + gidx ? cur : load_rec(i);
            T m[NCL][VEC];
#pragma unroll
            for (int j = 0; j < NCL; ++j)
#pragma unroll
                for (int e = 0; e < VEC; ++e) m[j][e] = ninf;
            auto relax = [&](int32_t ps) {
                const Chunk<T>* row = w2 + static_cast<int64_t>(ps) * NC;
#pragma unroll
                for (int j = 0; j < NCL; ++j) {
                    const Chunk<T> x = row[chunk(j)];
#pragma unroll
                    for (int e = 0; e < VEC; ++e) m[j][e] = dmax(x.v[e], m[j][e]);
                }
            };
            int32_t k = r.p0;
            for (; k + 2 <= r.p1; k += 2) {  // two predecessors in flight
                const int32_t ps0 = __ldg(&om_ps[k]), ps1 = __ldg(&om_ps[k + 1]);
                relax(ps0);
                relax(ps1);
            }
            if (k < r.p1) relax(__ldg(&om_ps[k]));
            const int32_t si = i - first;  // this node's own source column, if it is one
            Chunk<T>* outp = w2 + static_cast<int64_t>(r.sl) * NC;
#pragma unroll
            for (int j = 0; j < NCL; ++j) {
                Chunk<T> out;
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    T d = m[j][e] + r.gv;
                    const bool c = d >= static_cast<T>(0);
                    uint64_t& h = hist[VEC * j + e];
                    h += shl64(1ull, c ? static_cast<uint32_t>(kFieldBits * bin_t<TMODE>(d, th)) : 64u);
                    if (static_cast<uint32_t>(si) < static_cast<uint32_t>(S) && VEC * chunk(j) + e == si) {
                        // the source itself: distance 0, not its own descendant
                        if (c) h -= shl64(1ull, static_cast<uint32_t>(kFieldBits * bin_t<TMODE>(d, th)));
                        d = static_cast<T>(0);
                    }
                    if (prune_span > 0) small |= d >= static_cast<T>(0) && d <= wmax;
                    out.v[e] = d;
                }
                outp[chunk(j)] = out;
            }
            if (++visits == kFlushEvery) {
#pragma unroll
                for (int j = 0; j < NCL; ++j)
#pragma unroll
                    for (int e = 0; e < VEC; ++e)
                        if (VEC * chunk(j) + e < nsrc) flush5(hist[VEC * j + e], s_hist + (VEC * chunk(j) + e) * kBins);
                visits = 0;
            }
        }
        if (prune_span > 0) {
            recent = (recent << 1) | static_cast<uint64_t>(__syncthreads_or(small) != 0);
            if (lv - La + 1 >= prune_span && (recent & span_mask) == 0) break;
        } else {
            __syncthreads();
        }
    }
    // (narrow tiles keep the atomics: 3 x S threads would each sum over
    // hundreds of groups)
    if (S >= 32 && static_cast<int64_t>(P) * sizeof(T) >= static_cast<int64_t>(ngroups) * 8 &&
        ngroups * kFlushEvery < 32768) {
        uint64_t* dump = reinterpret_cast<uint64_t*>(w2);  // the rows are dead: dump_reduce
#pragma unroll
        for (int j = 0; j < NCL; ++j)
#pragma unroll
            for (int e = 0; e < VEC; ++e) dump[gidx * S + VEC * chunk(j) + e] = hist[VEC * j + e];
        dump_reduce<S>(dump, ngroups, nsrc, s_hist);
    } else {
#pragma unroll
        for (int j = 0; j < NCL; ++j)
#pragma unroll
            for (int e = 0; e < VEC; ++e)
                if (VEC * chunk(j) + e < nsrc) flush5(hist[VEC * j + e], s_hist + (VEC * chunk(j) + e) * kBins);
    }
    __syncthreads();
    if (relax_ctr && tid == 0)  // [0]: FP64 windows, [1]: FP32
        atomicAdd(relax_ctr + (sizeof(T) == 4 ? 1 : 0), static_cast<unsigned long long>(nrel * S));
    store_bins(s, t0, s.order + t0 + first, nsrc, s_hist, tid, nthr);
}

template <int S, int GL, typename T = double>
__device__ __forceinline__ void sweep_tile_rows_mode(const DevBatch& b, const AttrScratch& s, int64_t g, int32_t tile,
                                                     int32_t P, const Thresholds& th, uint32_t* s_hist,
                                                     int32_t prune_span, unsigned long long* rc) {
    if (th.mode == 0) sweep_tile_rows<S, GL, 0, T>(b, s, g, tile, P, th, s_hist, prune_span, rc);
    else if (th.mode == 2) sweep_tile_rows<S, GL, 2, T>(b, s, g, tile, P, th, s_hist, 0, rc);
    else if constexpr (sizeof(T) == 8) sweep_tile_rows<S, GL, 1, T>(b, s, g, tile, P, th, s_hist, prune_span, rc);
}

// Batches whose every tile is an FP32-exact shape of >= 32 sources (C2, C5)
// run here instead: the same tile code at 1024 threads per CTA (64 registers)
// -- twice the warps per SM to hide the record loads and level barriers.
// k_sweep and k_sweep_fp32 are both launched; the one the plan does not
// select returns at once (no host round trip between plan and sweep).
__global__ void __launch_bounds__(1024, 1) k_sweep_fp32(DevBatch b, AttrScratch s, int32_t sweep_mode,
                                                       const double* unit_time, unsigned long long* work_counter,
                                                       int32_t prune, unsigned long long* relax_ctr) {
    __shared__ int64_t s_item[2];
    __shared__ __align__(16) uint32_t s_hist[kMaxTile * kBins];
    if (!*s.plan_fp32) return;
    const int64_t total_tiles = s.tile_base[b.G];
    if (threadIdx.x == 0) s_item[0] = atomicAdd(work_counter, 1ull);
    __syncthreads();
    for (int k = 0;; k ^= 1) {
        const int64_t item = s_item[k];
        if (item >= total_tiles) break;
        if (threadIdx.x == 0) s_item[k ^ 1] = atomicAdd(work_counter, 1ull);
        const int64_t g = s.tile_graph[item];
        const int32_t tile = static_cast<int32_t>(item - s.tile_base[g]);
        const GraphInfo gi = s.info[g];
        if (gi.processed == static_cast<int32_t>(b.task_base[g + 1] - b.task_base[g])) {  // else cyclic
            const int32_t P = max(gi.peak_slots, 1);
            const Thresholds th = make_thresholds(sweep_mode, 2.0 * gi.median);
            const int32_t prune_span = (prune && gi.max_span > 0 && gi.max_span < 64) ? gi.max_span : 0;
            switch (s.tile_s[g] & kTileWidthMask) {
                case 256: sweep_tile_mode<256, true, float>(b, s, g, tile, nullptr, P, th, s_hist, prune_span, relax_ctr); break;
                case 128: sweep_tile_mode<128, true, float>(b, s, g, tile, nullptr, P, th, s_hist, prune_span, relax_ctr); break;
                case 64: sweep_tile_rows_mode<64, 8, float>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                case 32: sweep_tile_rows_mode<32, 4, float>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                default: sweep_tile_rows_mode<16, 2, float>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
            }
        }
        __syncthreads();
    }
    (void)unit_time;
}

__global__ void __launch_bounds__(512) k_sweep(DevBatch b, const DevCosts* costs_g,
                                              const int32_t* cost_idx, AttrScratch s,
                                              int32_t sweep_mode, const double* unit_time,
                                              int64_t total_tiles, unsigned long long* work_counter,
                                              int64_t smem_bytes, double* gwin, int64_t gwin_stride,
                                              int32_t prune, unsigned long long* relax_ctr) {
    __shared__ int64_t s_item[2];
    __shared__ __align__(16) uint32_t s_hist[kMaxTile * kBins];
    (void)costs_g;
    (void)cost_idx;
    if (total_tiles < 0) {  // whole-batch launch: k_sweep_fp32 takes all-FP32 plans
        if (*s.plan_fp32) return;
        total_tiles = s.tile_base[b.G];
    }
    if (threadIdx.x == 0) s_item[0] = atomicAdd(work_counter, 1ull);
    __syncthreads();
    for (int k = 0;; k ^= 1) {
        const int64_t item = s_item[k];
        if (item >= total_tiles) break;
        // the next item is claimed while this tile runs
        if (threadIdx.x == 0) s_item[k ^ 1] = atomicAdd(work_counter, 1ull);
        const int64_t g = s.tile_graph[item];
        const int32_t tile = static_cast<int32_t>(item - s.tile_base[g]);
        const GraphInfo gi = s.info[g];
        if (gi.processed == static_cast<int32_t>(b.task_base[g + 1] - b.task_base[g])) {  // else cyclic
            const int32_t P = max(gi.peak_slots, 1);
            Thresholds th;
            if (sweep_mode == SWEEP_SINGLE) th = make_thresholds(SWEEP_SINGLE, unit_time[g]);
            else th = make_thresholds(sweep_mode, 2.0 * gi.median);
            const int32_t S = s.tile_s[g] & kTileWidthMask;
            const bool f32 = s.tile_s[g] & kTileF32;
            double* gw = gwin + blockIdx.x * gwin_stride;
            // prune only when the edge span fits the 64-level history
            const int32_t prune_span = (prune && gi.max_span > 0 && gi.max_span < 64) ? gi.max_span : 0;
            if (static_cast<int64_t>(P) * S * (f32 ? 4 : 8) > smem_bytes) {
                sweep_tile_mode<32, false>(b, s, g, tile, gw, P, th, s_hist, prune_span, relax_ctr);
            } else if (f32) {
                // FP32-exact windows: the same kernel shapes at twice the width
                switch (S) {
                    case 256: sweep_tile_mode<256, true, float>(b, s, g, tile, gw, P, th, s_hist, prune_span, relax_ctr); break;
                    case 128: sweep_tile_mode<128, true, float>(b, s, g, tile, gw, P, th, s_hist, prune_span, relax_ctr); break;
                    case 64: sweep_tile_rows_mode<64, 8, float>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                    case 32: sweep_tile_rows_mode<32, 4, float>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                    case 16: sweep_tile_rows_mode<16, 1, float>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                    default: sweep_tile_rows_mode<8, 1, float>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                }
            } else {
                switch (S) {
                    // measured on B200 (C2 graphs forced to each width; C5):
                    // 128 sources -- one node per warp, 4 columns per lane
                    // (9.0 ms vs 10.0 for 16-lane rows); 64 and 32 -- rows of
                    // 8 / 4 lanes (C2: 12.3 vs 13.9 ms, 16.1 vs 23.7 ms; C5
                    // k_sweep 1012 -> 743 ms); 16 and 8 -- one lane per node
                    case 128: sweep_tile_mode<128, true>(b, s, g, tile, gw, P, th, s_hist, prune_span, relax_ctr); break;
                    case 64: sweep_tile_rows_mode<64, 8>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                    case 32: sweep_tile_rows_mode<32, 4>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                    case 16: sweep_tile_rows_mode<16, 1>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                    default: sweep_tile_rows_mode<8, 1>(b, s, g, tile, P, th, s_hist, prune_span, relax_ctr); break;
                }
            }
        }
        __syncthreads();
    }
}

// FP32-exact windows: the graph's GPU times (types present) as odd integer
// m * 2^scale; with the common (smallest) scale e, every time is M * 2^e with
// M <= the returned maximum (0: a time is not such a dyadic number).
__device__ double f32_mmax_of(const DevCosts& c, uint64_t types) {
    int e = INT_MAX;
    for (uint64_t t = types; t; t &= t - 1) {
        const double v = c.gpu[__ffsll(static_cast<long long>(t)) - 1];
        if (!(v >= 1e-30 && v <= 1e30)) return 0.0;
        int x = 0;
        const double f = frexp(v, &x);
        const long long m = static_cast<long long>(ldexp(f, 53));
        e = min(e, x - 53 + (__ffsll(m) - 1));
    }
    double mmax = 0.0;
    for (uint64_t t = types; t; t &= t - 1) {
        const double v = c.gpu[__ffsll(static_cast<long long>(t)) - 1];
        mmax = fmax(mmax, ldexp(v, -e));  // exact: v / 2^e is an integer
    }
    return mmax;
}

// Tiles per graph, their prefix and the tile -> graph map (single CTA; G can
// be large).  FP32 windows when they are exact: every
// distance of a graph with L levels is M * 2^e with M <= L * f32_mmax < 2^24,
// and the calibration windows W_0 * 2^k are normal floats -- FP32 max/add
// then reproduce the FP64 values bit for bit (f32_mmax_of).  Never for a
// caller-given window (its ladder compares in FP64).
__global__ void k_tile_plan(DevBatch b, AttrScratch s, int64_t smem_bytes, int32_t force_s,
                            const DevCosts* costs_g, const int32_t* cost_idx, int32_t sweep_mode) {
    __shared__ int32_t warp_tot[32];
    __shared__ int64_t carry;
    __shared__ int32_t all_fp32;
    __shared__ int32_t n_wide;
    __shared__ int64_t wide[1024];  // graphs of this chunk with > 64 tiles (written by warps)
    if (threadIdx.x == 0) {
        carry = 0;
        all_fp32 = 1;
        n_wide = 0;
        s.plan_fp32[1] = 0;
    }
    __syncthreads();
    for (int64_t base = 0; base < b.G; base += blockDim.x) {
        const int64_t g = base + threadIdx.x;
        int32_t tiles = 0;
        if (g < b.G) {
            const GraphInfo gi = s.info[g];
            const int32_t P = max(gi.peak_slots, 1);
            bool f32 = false;
            if (sweep_mode == SWEEP_ABILITY) {
                f32 = gi.n_levels < (1 << 24);
            } else if (sweep_mode == SWEEP_CALIBRATE && costs_g) {
                const double mmax = f32_mmax_of(costs_g[cost_idx ? cost_idx[g] : 0], gi.gpu_types);
                const double w0 = 2.0 * gi.median;
                f32 = mmax > 0.0 && static_cast<double>(gi.n_levels) * mmax < 16777216.0 &&
                      w0 >= 1e-30 && w0 * 64.0 <= 1e30;
            }
            const int64_t eb = f32 ? 4 : 8;
            int32_t S = 8;
            if (force_s) S = force_s;
            else if (f32 && static_cast<int64_t>(P) * 256 * eb <= smem_bytes) S = 256;
            else if (static_cast<int64_t>(P) * 128 * eb <= smem_bytes) S = 128;
            else if (static_cast<int64_t>(P) * 64 * eb <= smem_bytes) S = 64;
            else if (static_cast<int64_t>(P) * 32 * eb <= smem_bytes) S = 32;
            else if (static_cast<int64_t>(P) * 16 * eb <= smem_bytes) S = 16;
            else if (static_cast<int64_t>(P) * 8 * eb <= smem_bytes) S = 8;
            else { S = 32; f32 = false; }  // global-memory window (FP64)
            if (S == 256 && !f32) S = 128;  // 256 columns only as FP32
            if (static_cast<int64_t>(P) * S * (f32 ? 4 : 8) > smem_bytes) { S = 32; f32 = false; }  // forced, too wide
            // global-window graphs: the host sizes the per-CTA window (P x 32)
            if (static_cast<int64_t>(P) * S * (f32 ? 4 : 8) > smem_bytes) atomicMax(s.plan_fp32 + 1, P);
            s.tile_s[g] = S | (f32 ? kTileF32 : 0);
            if (!f32 || S < 16) atomicAnd(&all_fp32, 0);
            tiles = (gi.processed + S - 1) / S;
        }
        int32_t tot;
        const int32_t inc = block_inclusive_scan(tiles, warp_tot, &tot);
        const int64_t tb = carry + inc - tiles;
        if (g < b.G) s.tile_base[g] = tb;
        // tile -> graph: a graph of <= 64 tiles by its own thread, wider
        // ones by a warp each (listed here)
        if (g < b.G) {
            if (tiles <= 64) {
                for (int32_t t = 0; t < tiles; ++t) s.tile_graph[tb + t] = static_cast<int32_t>(g);
            } else {
                wide[atomicAdd(&n_wide, 1)] = g;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        const int lane = threadIdx.x & 31;
        for (int32_t w = threadIdx.x >> 5; w < n_wide; w += blockDim.x >> 5) {
            const int64_t gg = wide[w];
            const int64_t t_begin = s.tile_base[gg];
            const int32_t sw = s.tile_s[gg] & kTileWidthMask;
            const int32_t nt = (s.info[gg].processed + sw - 1) / sw;
            for (int32_t t = lane; t < nt; t += 32) s.tile_graph[t_begin + t] = static_cast<int32_t>(gg);
        }
        __syncthreads();
        if (threadIdx.x == 0) n_wide = 0;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        s.tile_base[b.G] = carry;
        *s.plan_fp32 = b.G > 0 ? all_fp32 : 0;
    }
}

// ---------------------------------------------------------------- finalize

// a source's 12 window-bin counts (kBins uint32, 48 B, 16-B aligned)
__device__ __forceinline__ void load_bins(const uint32_t* h, uint32_t (&c)[kBins]) {
    const uint4* h4 = reinterpret_cast<const uint4*>(h);
#pragma unroll
    for (int q = 0; q < kBins / 4; ++q) {
        const uint4 w = h4[q];
        c[4 * q] = w.x; c[4 * q + 1] = w.y; c[4 * q + 2] = w.z; c[4 * q + 3] = w.w;
    }
}

__device__ int64_t gcd64(int64_t a, int64_t b) {
    a = a < 0 ? -a : a;
    b = b < 0 ? -b : b;
    while (b) { const int64_t t = a % b; a = b; b = t; }
    return a;
}

__global__ void __launch_bounds__(256) k_finalize(DevBatch b, AttrScratch s, int32_t sweep_mode,
                                                 const double* unit_time_in, AttrOutDev o,
                                                 int64_t* cls_scratch, int64_t cls_stride, int32_t write_ability) {
    __shared__ int32_t s_score[kWindows];
    // class sums, counts and reduced fractions: in shared memory for graphs
    // of <= kSmemClasses calibration classes, else in the CTA's HBM scratch
    constexpr int kSmemClasses = 64;
    __shared__ int64_t s_cls[kSmemClasses * (3 * kWindows + 1)];
    int64_t* const g_sums = cls_scratch + blockIdx.x * cls_stride;  // [C][kWindows] then cnt[C]
    for (int64_t g = blockIdx.x; g < b.G; g += gridDim.x) {
        const int64_t t0 = b.task_base[g];
        const int32_t n = static_cast<int32_t>(b.task_base[g + 1] - t0);
        const GraphInfo gi = s.info[g];
        if (gi.processed != n) continue;
        const uint32_t* hist = s.hist + t0 * kBins;
        int best = 0;
        if (sweep_mode == SWEEP_CALIBRATE) {
            const int32_t C = gi.n_classes;
            int64_t* sums = C <= kSmemClasses ? s_cls : g_sums;
            int64_t* cnt = sums + static_cast<int64_t>(C) * kWindows;
            for (int64_t i = threadIdx.x; i < static_cast<int64_t>(C) * (kWindows + 1); i += blockDim.x) sums[i] = 0;
            if (threadIdx.x < kWindows) s_score[threadIdx.x] = 0;
            __syncthreads();
            for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
                const int32_t c = s.cls[t0 + v];
                uint32_t f[kBins];
                load_bins(hist + static_cast<int64_t>(v) * kBins, f);
                int64_t acc = 0;
#pragma unroll
                for (int k = 0; k < kWindows; ++k) {
                    acc += f[k];
                    if (acc) atomicAdd(reinterpret_cast<unsigned long long*>(&sums[static_cast<int64_t>(c) * kWindows + k]),
                                       static_cast<unsigned long long>(acc));
                }
                atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[c]), 1ull);
            }
            __syncthreads();
            // distinct reduced fractions per window (attributes.cpp:205-217):
            // reduce every (class, window) once, then count first occurrences
            int64_t* fa = cnt + C;
            int64_t* fq = fa + static_cast<int64_t>(C) * kWindows;
            for (int64_t item = threadIdx.x; item < static_cast<int64_t>(C) * kWindows; item += blockDim.x) {
                const int32_t c = static_cast<int32_t>(item / kWindows);
                const int64_t sc_ = sums[item], cc = cnt[c];
                const int64_t d = gcd64(sc_ == 0 ? cc : sc_, cc);
                fa[item] = sc_ / d;
                fq[item] = cc / d;
            }
            __syncthreads();
            for (int64_t item = threadIdx.x; item < static_cast<int64_t>(C) * kWindows; item += blockDim.x) {
                const int32_t c = static_cast<int32_t>(item / kWindows);
                const int k = static_cast<int>(item % kWindows);
                const int64_t a = fa[item], q = fq[item];
                bool first = true;
                for (int32_t c2 = 0; c2 < c && first; ++c2)
                    if (fa[static_cast<int64_t>(c2) * kWindows + k] == a && fq[static_cast<int64_t>(c2) * kWindows + k] == q)
                        first = false;
                if (first) atomicAdd(&s_score[k], 1);
            }
            __syncthreads();
            int64_t best_score = -1;
            for (int k = 0; k < kWindows; ++k)
                if (s_score[k] > best_score) { best_score = s_score[k]; best = k; }
            if (threadIdx.x == 0) {
                const double w0 = 2.0 * gi.median;
                if (o.unit_time_ms) o.unit_time_ms[g] = ldexp(w0, best - 4);
                if (o.w0_ms) o.w0_ms[g] = w0;
                if (o.best_score) o.best_score[g] = best_score;
                if (o.w0_score) o.w0_score[g] = s_score[4];
                if (o.evaluations) o.evaluations[g] = kWindows;
            }
        }
        for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
            uint32_t f[kBins];
            load_bins(hist + static_cast<int64_t>(v) * kBins, f);
            int64_t eff = 0, abil = 0;
#pragma unroll
            for (int k = 0; k < kBins; ++k) {
                if (k <= best) eff += f[k];
                abil += f[k];
            }
            if (o.efficiency && sweep_mode != SWEEP_ABILITY) o.efficiency[t0 + v] = eff;
            if (o.ability && write_ability) o.ability[t0 + v] = abil;
        }
        __syncthreads();
    }
}

// k_finalize for ONE large graph with the whole GPU (cooperative launch).
// Same results as k_finalize; the phases are grid-wide: per-class window
// sums (L2 atomics), reduced fractions per (class, window), distinct
// fractions per window by insertion into an open-addressing table (a slot,
// once claimed by a class, never changes, so equal fractions meet on the
// same probe sequence), then per-task efficiency / ability.
// scratch: [C*11] sums, [C] counts, [C*11] numerators, [C*11] denominators;
// tab: 11 tables of `tab_size` int32 (power of two >= 2C), score[11].
// Sharded (multi-GPU): sources are the level-order positions [pos_lo,
// pos_hi); phase FIN_PARTIAL stops after this shard's class sums (the
// caller all-reduces them), FIN_FINISH starts from the reduced sums.
__global__ void __launch_bounds__(512) k_finalize_large(DevBatch b, AttrScratch s, int32_t sweep_mode, AttrOutDev o,
                                                       int64_t* scratch, int32_t* tab, int64_t tab_cap,
                                                       int32_t* score, int32_t write_ability, int32_t phase,
                                                       int32_t pos_lo, int32_t pos_hi, const int64_t* sums_in) {
    cg::grid_group grid = cg::this_grid();
    constexpr int64_t g = 0;
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = b.task_base[g];
    const int32_t n = static_cast<int32_t>(b.task_base[g + 1] - t0);
    const GraphInfo gi = s.info[g];
    if (gi.processed != n) return;  // uniform: cyclic graphs are reported by the host
    const uint32_t* hist = s.hist + t0 * kBins;
    int best = 0;
    if (sweep_mode == SWEEP_CALIBRATE) {
        const int64_t C = gi.n_classes;
        int64_t* sums = scratch;
        int64_t* cnt = sums + C * kWindows;
        int64_t* fa = cnt + C;
        int64_t* fq = fa + C * kWindows;
        int64_t ts = 1;
        while (ts < 2 * C) ts <<= 1;
        ts = min(ts, tab_cap);
        for (int64_t i = gtid; i < C * (kWindows + 1); i += gthreads) sums[i] = sums_in ? sums_in[i] : 0;
        for (int64_t i = gtid; i < ts * kWindows; i += gthreads) tab[i] = 0;
        if (gtid < kWindows) score[gtid] = 0;
        grid.sync();
        if (phase != FIN_FINISH) {
            for (int64_t i = pos_lo + gtid; i < pos_hi; i += gthreads) {
                const int64_t v = s.order[t0 + i];
                const int32_t c = s.cls[t0 + v];
                uint32_t f[kBins];
                load_bins(hist + v * kBins, f);
                int64_t acc = 0;
#pragma unroll
                for (int k = 0; k < kWindows; ++k) {
                    acc += f[k];
                    if (acc)
                        atomicAdd(reinterpret_cast<unsigned long long*>(&sums[static_cast<int64_t>(c) * kWindows + k]),
                                  static_cast<unsigned long long>(acc));
                }
                atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[c]), 1ull);
            }
            if (phase == FIN_PARTIAL) return;  // uniform: the caller reduces scratch[0 .. 12C)
            grid.sync();
        }
        for (int64_t item = gtid; item < C * kWindows; item += gthreads) {
            const int64_t c = item / kWindows;
            const int64_t sc_ = __ldcg(&sums[item]), cc = __ldcg(&cnt[c]);
            const int64_t d = gcd64(sc_ == 0 ? cc : sc_, cc);
            fa[item] = sc_ / d;
            fq[item] = cc / d;
        }
        grid.sync();
        for (int64_t item = gtid; item < C * kWindows; item += gthreads) {
            const int64_t c = item / kWindows;
            const int k = static_cast<int>(item - c * kWindows);
            const int64_t a = __ldcg(&fa[item]), q = __ldcg(&fq[item]);
            int32_t* t = tab + static_cast<int64_t>(k) * ts;
            uint64_t hsh = static_cast<uint64_t>(a) * 0x9E3779B97F4A7C15ull ^ (static_cast<uint64_t>(q) * 0xC2B2AE3D27D4EB4Full);
            hsh ^= hsh >> 29;
            int64_t pos = static_cast<int64_t>(hsh & static_cast<uint64_t>(ts - 1));
            for (;;) {
                const int32_t cur = atomicCAS(&t[pos], 0, static_cast<int32_t>(c) + 1);
                if (cur == 0) { atomicAdd(&score[k], 1); break; }
                const int64_t oi = static_cast<int64_t>(cur - 1) * kWindows + k;
                if (__ldcg(&fa[oi]) == a && __ldcg(&fq[oi]) == q) break;
                pos = (pos + 1) & (ts - 1);
            }
        }
        grid.sync();
        int64_t best_score = -1;
        int32_t sk[kWindows];
        for (int k = 0; k < kWindows; ++k) {
            sk[k] = __ldcg(&score[k]);
            if (sk[k] > best_score) { best_score = sk[k]; best = k; }  // strict >: ties keep the smaller W
        }
        if (gtid == 0) {
            const double w0 = 2.0 * gi.median;
            if (o.unit_time_ms) o.unit_time_ms[g] = ldexp(w0, best - 4);
            if (o.w0_ms) o.w0_ms[g] = w0;
            if (o.best_score) o.best_score[g] = best_score;
            if (o.w0_score) o.w0_score[g] = sk[4];
            if (o.evaluations) o.evaluations[g] = kWindows;
        }
    }
    for (int64_t i = pos_lo + gtid; i < pos_hi; i += gthreads) {
        const int64_t v = s.order[t0 + i];
        uint32_t f[kBins];
        load_bins(hist + v * kBins, f);
        int64_t eff = 0, abil = 0;
#pragma unroll
        for (int k = 0; k < kBins; ++k) {
            if (k <= best) eff += f[k];
            abil += f[k];
        }
        if (o.efficiency && sweep_mode != SWEEP_ABILITY) o.efficiency[t0 + v] = eff;
        if (o.ability && write_ability) o.ability[t0 + v] = abil;
    }
}

// ---------------------------------------------------------------- closure

// Inspiring ability of one large graph as a descendant-bitset closure
// (ability_impl, attributes.cpp:57-92) streaming through HBM.  Bits index the
// level order, so the descendants of a node at level L occupy only words
// >= lstart[L+1]/64: each set is written from that word on and read from its
// own lower bound (lower words are zero by construction).  Levels are
// processed from the last to the first with a grid-wide barrier in between;
// sets live in reverse live-range slots (firstuse) so only the level cut is
// resident.  A warp owns (node, 32*CH-word chunk): coalesced loads of every
// successor's chunk, OR, store, popcount.
// Sharded (multi-GPU): this launch owns words [wlo, whi) of
// every set -- the OR is word-wise independent, so ranks need no exchange
// during the closure and ability = the sum over ranks of the partial
// popcounts.  `sets` holds only the owned words (stride whi - wlo).
template <int CH>
__global__ void __launch_bounds__(256) k_closure(DevBatch b, AttrScratch s, int64_t g, uint64_t* sets, int64_t wlo,
                                               int64_t whi, unsigned long long* ability) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int64_t t0 = b.task_base[g];
    const GraphInfo gi = s.info[g];
    const int32_t* lstart = s.lstart + t0 + g;
    const int32_t* order = s.order + t0;
    const int32_t* opos = s.opos + t0;
    const int32_t* rslot = s.rslot + t0;
    const int32_t* level = s.level + t0;
    const int32_t* soff = b.succ_off + t0 + g;
    const int32_t* succ = b.succ + b.edge_base[g];
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    constexpr int64_t kChunk = 32 * CH;
    const int64_t nwr = whi - wlo;
    for (int32_t lv = gi.n_levels - 1; lv >= 0; --lv) {
        const int32_t a0 = lstart[lv], cnt = lstart[lv + 1] - a0;
        const int64_t lo = max(static_cast<int64_t>(lstart[lv + 1] >> 6), wlo);
        const int64_t chunks = whi > lo ? (whi - lo + kChunk - 1) / kChunk : 0;
        const int64_t items = static_cast<int64_t>(cnt) * chunks;
        for (int64_t item = gwarp; item < items; item += nwarps) {
            const int32_t i = a0 + static_cast<int32_t>(item / chunks);
            const int64_t w0 = lo + (item % chunks) * kChunk;
            const int32_t u = order[i];
            uint64_t acc[CH];
#pragma unroll
            for (int j = 0; j < CH; ++j) acc[j] = 0;
            // successor metadata for 32 successors at once (a lane each),
            // then a broadcast per successor: no dependent load chain
            // between one successor's set reads and the next's
            const int32_t k0 = __ldg(&soff[u]), k1 = __ldg(&soff[u + 1]);
            for (int32_t kb = k0; kb < k1; kb += 32) {
                int32_t m_ov = 0, m_slot = 0, m_lov = 0;
                if (kb + lane < k1) {
                    const int32_t v = __ldg(&succ[kb + lane]);
                    m_ov = opos[v];
                    m_lov = lstart[level[v] + 1] >> 6;
                    m_slot = rslot[v];
                }
                const int32_t cnt = min(32, k1 - kb);
                // two successors per round: 2 x CH loads per lane in flight
                // (C4: 70.5 -> 64.9 ms; a generic U-successor loop nest
                // compiled to the same registers but measured 73.4 ms)
                for (int32_t t = 0; t < cnt; t += 2) {
                    const int32_t t1 = t + 1 < cnt ? t + 1 : t;
                    const int32_t ov = __shfl_sync(0xffffffffu, m_ov, t);
                    const int64_t lov = __shfl_sync(0xffffffffu, m_lov, t);
                    const int32_t slot = __shfl_sync(0xffffffffu, m_slot, t);
                    const int32_t ov1 = __shfl_sync(0xffffffffu, m_ov, t1);
                    const int64_t lov1 = __shfl_sync(0xffffffffu, m_lov, t1);
                    const int32_t slot1 = __shfl_sync(0xffffffffu, m_slot, t1);
                    const uint64_t* sv = sets + static_cast<int64_t>(slot) * nwr - wlo;
                    const uint64_t* sv1 = sets + static_cast<int64_t>(slot1) * nwr - wlo;
                    uint64_t x[CH], y[CH];
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        const int64_t w = w0 + lane + 32 * j;
                        x[j] = (w >= lov && w < whi) ? __ldcg(&sv[w]) : 0ull;
                        y[j] = (w >= lov1 && w < whi) ? __ldcg(&sv1[w]) : 0ull;
                    }
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        const int64_t w = w0 + lane + 32 * j;
                        acc[j] |= x[j] | y[j];  // t1 == t repeats a successor: OR is idempotent
                        if (w == (ov >> 6)) acc[j] |= 1ull << (ov & 63);
                        if (w == (ov1 >> 6)) acc[j] |= 1ull << (ov1 & 63);
                    }
                }
            }
            uint64_t* su = sets + static_cast<int64_t>(rslot[u]) * nwr - wlo;
            int pc = 0;
#pragma unroll
            for (int j = 0; j < CH; ++j) {
                const int64_t w = w0 + lane + 32 * j;
                if (w < whi) {
                    __stcg(&su[w], acc[j]);
                    pc += __popcll(acc[j]);
                }
            }
            pc = __reduce_add_sync(0xffffffffu, pc);
            if (lane == 0 && pc) atomicAdd(&ability[t0 + u], static_cast<unsigned long long>(pc));
        }
        grid.sync();
    }
}

template __global__ void k_closure<4>(DevBatch, AttrScratch, int64_t, uint64_t*, int64_t, int64_t, unsigned long long*);

// ---- the same closure with the successor chunks moved by TMA bulk copies
//
// Each warp keeps a ring of kStages 1-KB shared-memory stages with one
// mbarrier each: lane 0 issues `cp.async.bulk` global->shared copies for up
// to kStages successors' chunks of the current item (the asynchronous proxy
// moves them; no registers hold in-flight data), the warp ORs each stage as
// its barrier completes.  A successor's chunk is copied from its lower word
// bound rounded down to 16 bytes; words below the bound (stale memory of a
// reused slot) and beyond whi are masked at the OR, as in k_closure.
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace

template <int kStages, int CH, int kWarps>
__global__ void __launch_bounds__(32 * kWarps) k_closure_tma(DevBatch b, AttrScratch s, int64_t g, uint64_t* sets,
                                                             int64_t wlo, int64_t whi, unsigned long long* ability) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    constexpr int64_t kChunk = 32 * CH;  // words per item (CH x 256 B)
    // stage rows of kChunk + 2 words: a chunk starting at an odd word lands
    // one word in (16-byte alignment of both ends of the copy)
    __shared__ __align__(128) uint64_t s_stage[kWarps][kStages][kChunk + 2];
    __shared__ __align__(8) uint64_t s_bar[kWarps][kStages];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint64_t* bars = s_bar[wib];
    if (lane < kStages) mbar_init(&bars[lane], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t issued = 0, consumed = 0;  // copies through this warp's ring (stage = n % kStages)

    const int64_t t0 = b.task_base[g];
    const GraphInfo gi = s.info[g];
    const int32_t* lstart = s.lstart + t0 + g;
    const int32_t* order = s.order + t0;
    const int32_t* opos = s.opos + t0;
    const int32_t* rslot = s.rslot + t0;
    const int32_t* level = s.level + t0;
    const int32_t* soff = b.succ_off + t0 + g;
    const int32_t* succ = b.succ + b.edge_base[g];
    const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t nwr = whi - wlo;
    for (int32_t lv = gi.n_levels - 1; lv >= 0; --lv) {
        // the previous level's sets (generic-proxy stores, grid barrier)
        // are read by the asynchronous proxy from here on
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const int32_t a0 = lstart[lv], cnt = lstart[lv + 1] - a0;
        const int64_t lo = max(static_cast<int64_t>(lstart[lv + 1] >> 6), wlo);
        const int64_t chunks = whi > lo ? (whi - lo + kChunk - 1) / kChunk : 0;
        const int64_t items = static_cast<int64_t>(cnt) * chunks;
        for (int64_t item = gwarp; item < items; item += nwarps) {
            const int32_t i = a0 + static_cast<int32_t>(item / chunks);
            const int64_t w0 = lo + (item % chunks) * kChunk;
            const int32_t u = order[i];
            const int32_t shift = static_cast<int32_t>(w0 & 1);  // word w at stage index w - w0 + shift
            uint64_t acc[CH];
#pragma unroll
            for (int j = 0; j < CH; ++j) acc[j] = 0;
            const int32_t k0 = __ldg(&soff[u]), k1 = __ldg(&soff[u + 1]);
            for (int32_t kb = k0; kb < k1; kb += 32) {
                int32_t m_ov = 0, m_slot = 0, m_lov = 0;
                if (kb + lane < k1) {
                    const int32_t v = __ldg(&succ[kb + lane]);
                    m_ov = opos[v];
                    m_lov = lstart[level[v] + 1] >> 6;
                    m_slot = rslot[v];
                }
                const int32_t cnt_s = min(32, k1 - kb);
                // copy of successor t into stage `issued % kStages`
                auto issue = [&](int32_t t) {
                    const int64_t lov = __shfl_sync(0xffffffffu, m_lov, t);
                    const int32_t slot = __shfl_sync(0xffffffffu, m_slot, t);
                    if (lane == 0) {
                        const uint32_t st = issued % kStages;
                        const int64_t a = max(lov, w0) & ~int64_t(1);  // 16-byte aligned start
                        int64_t e = min(w0 + kChunk, whi);
                        e = (e + 1) & ~int64_t(1);
                        if (e > a) {
                            const uint64_t* src = sets + static_cast<int64_t>(slot) * nwr + (a - wlo);
                            const uint32_t bytes = static_cast<uint32_t>((e - a) * 8);
                            mbar_expect_tx(&bars[st], bytes);
                            bulk_g2s(&s_stage[wib][st][a - w0 + shift], src, bytes, &bars[st]);
                        } else {
                            mbar_arrive(&bars[st]);
                        }
                    }
                    ++issued;
                };
                int32_t next = 0;
                for (; next < cnt_s && next < kStages; ++next) issue(next);
                for (int32_t t = 0; t < cnt_s; ++t) {
                    const uint32_t st = consumed % kStages;
                    mbar_wait(&bars[st], (consumed / kStages) & 1u);
                    const int32_t ov = __shfl_sync(0xffffffffu, m_ov, t);
                    const int64_t lov = __shfl_sync(0xffffffffu, m_lov, t);
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        const int64_t w = w0 + lane + 32 * j;
                        if (w >= lov && w < whi) acc[j] |= s_stage[wib][st][lane + 32 * j + shift];
                        if (w == (ov >> 6)) acc[j] |= 1ull << (ov & 63);
                    }
                    ++consumed;
                    __syncwarp();  // every lane is done with the stage before it is refilled
                    if (next < cnt_s) {
                        if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        issue(next++);
                    }
                }
            }
            uint64_t* su = sets + static_cast<int64_t>(rslot[u]) * nwr - wlo;
            int pc = 0;
#pragma unroll
            for (int j = 0; j < CH; ++j) {
                const int64_t w = w0 + lane + 32 * j;
                if (w < whi) {
                    __stcg(&su[w], acc[j]);
                    pc += __popcll(acc[j]);
                }
            }
            pc = __reduce_add_sync(0xffffffffu, pc);
            if (lane == 0 && pc) atomicAdd(&ability[t0 + u], static_cast<unsigned long long>(pc));
        }
        grid.sync();
    }
}

// measured on C4 (stages, words per lane, warps per CTA): <4,4,8> 85.5 ms,
// <4,8,4> 64.4, <4,16,2> 63.0, <2,16,2> 59.6, <3,16,2> 59.1, <1,16,2> 65.8,
// <4,32,1> 88.0; the register-staged k_closure<4> 64.9
template __global__ void k_closure_tma<3, 16, 2>(DevBatch, AttrScratch, int64_t, uint64_t*, int64_t, int64_t,
                                                 unsigned long long*);

// Per-task outputs of the structure pass (layers, depth, static priority).
__global__ void k_structure_out(DevBatch b, AttrScratch s, AttrOutDev o, int32_t prio_kind, int32_t want_prio) {
    const int64_t T = b.T;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (o.layer) o.layer[i] = s.level[i];
        if (o.depth) o.depth[i] = s.height[i];
        if (want_prio && o.static_priority) {
            int64_t p = 0;
            if (prio_kind == TBSIM_PRIO_UPWARD_RANK) p = tbsim_rules::rank_priority(s.rank[i]);
            else if (prio_kind == TBSIM_PRIO_DEPTH) p = s.height[i];
            o.static_priority[i] = p;
        }
    }
}

}  // namespace tbsim_dev
