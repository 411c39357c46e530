// probe.cu -- the efficiency sweep's own inner-loop peak on this GPU.
//
// The sweep (attributes.cu, k_sweep) is not HBM-bound: its work is the
// max-plus relaxation -- a predecessor's distance row read from shared
// memory (LDS.128) folded into register accumulators with FP64
// compare-select (DSETP + 2 FSEL).  k_probe_relax runs exactly that loop
// (128-column rows, two predecessors in flight, one CTA of 512 threads per
// SM like k_sweep) with no graph around it; bench.py divides the sweep's
// executed relaxations per second by this rate to report its roofline
// fraction.  Measured live, so the denominator is this GPU at its clocks.
#include <math_constants.h>

#include <cstdint>

namespace tbsim_dev {

// FP32-exact windows (k_tile_plan): the same loop on 128-column float rows
// (one LDS.128 per predecessor and lane, FMNMX)
__global__ void __launch_bounds__(512, 1) k_probe_relax_f32(int32_t rows_mask, int32_t iters, double* out) {
    extern __shared__ float4 pwin4[];  // (rows_mask + 1) rows x 32 float4 = 128 columns
    const int32_t rows = rows_mask + 1;
    for (int32_t i = threadIdx.x; i < rows * 32; i += blockDim.x) pwin4[i] = make_float4(0.5f * i, 0.25f * i, i, 2.f * i);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, m2 = -CUDART_INF_F, m3 = -CUDART_INF_F;
    uint32_t r = 2654435761u * (warp + 1) + blockIdx.x;
#pragma unroll 1
    for (int32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int p = 0; p < 4; p += 2) {
            r = r * 1664525u + 1013904223u;
            const float4 a = pwin4[((r >> 9) & rows_mask) * 32 + lane];
            r = r * 1664525u + 1013904223u;
            const float4 b = pwin4[((r >> 9) & rows_mask) * 32 + lane];
            m0 = fmaxf(m0, a.x); m1 = fmaxf(m1, a.y); m2 = fmaxf(m2, a.z); m3 = fmaxf(m3, a.w);
            m0 = fmaxf(m0, b.x); m1 = fmaxf(m1, b.y); m2 = fmaxf(m2, b.z); m3 = fmaxf(m3, b.w);
        }
    }
    const float v = (m0 + m1) + (m2 + m3);
    if (v == 12345.678f) out[blockIdx.x] = v;  // never true; keeps the loop alive
}

__global__ void __launch_bounds__(512, 1) k_probe_relax(int32_t rows_mask, int32_t iters, double* out) {
    extern __shared__ double2 pwin[];  // (rows_mask + 1) rows x 64 double2 = 128 columns
    const int32_t rows = rows_mask + 1;
    for (int32_t i = threadIdx.x; i < rows * 64; i += blockDim.x) pwin[i] = make_double2(0.5 * i, 0.25 * i);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double m0 = -CUDART_INF, m1 = -CUDART_INF, m2 = -CUDART_INF, m3 = -CUDART_INF;
    uint32_t r = 2654435761u * (warp + 1) + blockIdx.x;
#pragma unroll 1
    for (int32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int p = 0; p < 4; p += 2) {  // two predecessor rows in flight
            r = r * 1664525u + 1013904223u;
            const double2* ra = pwin + ((r >> 9) & rows_mask) * 64;
            r = r * 1664525u + 1013904223u;
            const double2* rb = pwin + ((r >> 9) & rows_mask) * 64;
            const double2 a0 = ra[lane], a1 = ra[32 + lane], b0 = rb[lane], b1 = rb[32 + lane];
            m0 = a0.x > m0 ? a0.x : m0;
            m1 = a0.y > m1 ? a0.y : m1;
            m2 = a1.x > m2 ? a1.x : m2;
            m3 = a1.y > m3 ? a1.y : m3;
            m0 = b0.x > m0 ? b0.x : m0;
            m1 = b0.y > m1 ? b0.y : m1;
            m2 = b1.x > m2 ? b1.x : m2;
            m3 = b1.y > m3 ? b1.y : m3;
        }
    }
    const double v = (m0 + m1) + (m2 + m3);
    if (v == 12345.678) out[blockIdx.x] = v;  // never true; keeps the loop alive
}

}  // namespace tbsim_dev
