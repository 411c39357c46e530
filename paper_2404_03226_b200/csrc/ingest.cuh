// ingest.cuh -- successor CSR of one graph from its dependency CSR
// (build_index, taskgraph.cpp:11-43), shared by k_ingest (attributes.cu) and
// the fused ingest + simulator pack of uploaded batches (simulate.cu).
#pragma once

#include <cstdint>

#include "blockscan.cuh"
#include "common.cuh"

namespace tbsim_dev {

__device__ __forceinline__ void sort_small(int32_t* a, int32_t len) {
    if (len <= 32) {  // in a thread-local copy (L1-resident) instead of in place in HBM
        int32_t loc[32];
        for (int32_t i = 0; i < len; ++i) {
            const int32_t x = a[i];
            int32_t j = i - 1;
            while (j >= 0 && loc[j] > x) { loc[j + 1] = loc[j]; --j; }
            loc[j + 1] = x;
        }
        for (int32_t i = 0; i < len; ++i) a[i] = loc[i];
        return;
    }
    if (len <= 48) {
        for (int32_t i = 1; i < len; ++i) {
            int32_t x = a[i], j = i - 1;
            while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
            a[j + 1] = x;
        }
        return;
    }
    // heapsort for long lists
    auto sift = [&](int32_t root, int32_t end) {
        while (2 * root + 1 < end) {
            int32_t c = 2 * root + 1;
            if (c + 1 < end && a[c] < a[c + 1]) ++c;
            if (a[root] >= a[c]) return;
            int32_t t = a[root]; a[root] = a[c]; a[c] = t;
            root = c;
        }
    };
    for (int32_t i = len / 2 - 1; i >= 0; --i) sift(i, len);
    for (int32_t end = len - 1; end > 0; --end) {
        int32_t t = a[0]; a[0] = a[end]; a[end] = t;
        sift(0, end);
    }
}

// Successor CSR of graph g by one CTA: count, scan, scatter, sort each
// list, so every list is ascending with multi-edges kept.  Counts and
// cursors live in shared memory (s_ctr) when the graph fits
// (smem_ints >= n + 1), else in global memory (cursor_scratch).  Ends with
// the CTA synchronised; succ_off/succ are then readable (plain loads) by the
// whole CTA.
__device__ __forceinline__ void ingest_graph(const DevBatch& b, int64_t g, int32_t* cursor_scratch, int32_t smem_ints,
                                             int32_t* s_ctr, int32_t* warp_tot) {
    const int64_t t0 = b.task_base[g];
    const int32_t n = static_cast<int32_t>(b.task_base[g + 1] - t0);
    const int32_t* doff = b.dep_off + t0 + g;
    const int32_t* dep = b.dep + b.edge_base[g];
    int32_t* soff = b.succ_off + t0 + g;
    int32_t* succ = b.succ + b.edge_base[g];
    if (n + 1 <= smem_ints) {
        for (int32_t i = threadIdx.x; i <= n; i += blockDim.x) s_ctr[i] = 0;
        __syncthreads();
        for (int32_t v = threadIdx.x; v < n; v += blockDim.x)
            for (int32_t k = __ldg(&doff[v]); k < __ldg(&doff[v + 1]); ++k) atomicAdd(&s_ctr[__ldg(&dep[k])], 1);
        __syncthreads();
        block_exclusive_scan_inplace(s_ctr, n + 1, warp_tot);
        for (int32_t i = threadIdx.x; i <= n; i += blockDim.x) soff[i] = s_ctr[i];
        __syncthreads();
        for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
            const int32_t k1 = __ldg(&doff[v + 1]);
            for (int32_t k = __ldg(&doff[v]); k < k1; k += 4) {  // four dep ids ahead of the stores
                int32_t d[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) d[q] = k + q < k1 ? __ldg(&dep[k + q]) : -1;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (d[q] >= 0) succ[atomicAdd(&s_ctr[d[q]], 1)] = v;
            }
        }
        __syncthreads();
        // s_ctr[u] is now the end of u's list
        for (int32_t u = threadIdx.x; u < n; u += blockDim.x) {
            const int32_t e = s_ctr[u], s = u == 0 ? 0 : s_ctr[u - 1];
            sort_small(succ + s, e - s);
        }
        __syncthreads();
        return;
    }
    int32_t* cur = cursor_scratch + t0 + g;
    for (int32_t i = threadIdx.x; i <= n; i += blockDim.x) soff[i] = 0;
    __syncthreads();
    for (int32_t v = threadIdx.x; v < n; v += blockDim.x)
        for (int32_t k = doff[v]; k < doff[v + 1]; ++k) atomicAdd(&soff[dep[k]], 1);
    __syncthreads();
    block_exclusive_scan_inplace(soff, n + 1, warp_tot);
    for (int32_t i = threadIdx.x; i <= n; i += blockDim.x) cur[i] = soff[i];
    __syncthreads();
    for (int32_t v = threadIdx.x; v < n; v += blockDim.x)
        for (int32_t k = doff[v]; k < doff[v + 1]; ++k) succ[atomicAdd(&cur[dep[k]], 1)] = v;
    __syncthreads();
    for (int32_t u = threadIdx.x; u < n; u += blockDim.x) sort_small(succ + soff[u], soff[u + 1] - soff[u]);
    __syncthreads();
}

}  // namespace tbsim_dev
