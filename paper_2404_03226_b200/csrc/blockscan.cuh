// blockscan.cuh -- small CTA-wide scan helpers used by the ingest/structure
// kernels (in-place exclusive scans over global or shared int32 arrays).
#pragma once

#include <cstdint>

namespace tbsim_dev {

// Inclusive scan of one value per thread across the CTA.  `warp_tot` must
// hold blockDim.x/32 ints of shared scratch.  Returns the inclusive prefix;
// *total receives the CTA total.
__device__ inline int32_t block_inclusive_scan(int32_t x, int32_t* warp_tot, int32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int32_t w = lane < nwarps ? warp_tot[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, w, d);
            if (lane >= d) w += y;
        }
        if (lane < nwarps) warp_tot[lane] = w;
    }
    __syncthreads();
    if (warp > 0) x += warp_tot[warp - 1];
    *total = warp_tot[nwarps - 1];
    __syncthreads();
    return x;
}

// In-place exclusive scan of a[0..len) (any memory space), CTA-cooperative.
// Returns the grand total.
__device__ inline int32_t block_exclusive_scan_inplace(int32_t* a, int64_t len, int32_t* warp_tot) {
    int32_t carry = 0;
    for (int64_t base = 0; base < len; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        int32_t x = i < len ? a[i] : 0;
        int32_t tot;
        int32_t inc = block_inclusive_scan(x, warp_tot, &tot);
        if (i < len) a[i] = carry + inc - x;
        carry += tot;
    }
    __syncthreads();
    return carry;
}

}  // namespace tbsim_dev
