// generate.cuh -- device-side synthetic DAG generation (layered generator).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace tbsim_dev {

struct GenParams {
    int64_t G;
    int32_t n, L;
    double p;
    const uint64_t* seeds;    // [G]
    int32_t* ndep;            // [G*n] scratch: dependency count per task
    int32_t* degree;          // [G*n] scratch: total degree per task
    int32_t* hist;            // [G*(max_degree+1)] scratch
    int32_t max_degree;
    int64_t* edges;           // [G] dependency entries per DAG
    int32_t* type;            // [G*n] output (batch section)
    int64_t* handle_bytes;    // [G*n] output (batch section)
    int32_t type_base;        // id of LAYERK0 in the type table
    // the dependency draws' outcome, recorded by pass 1 so pass 2 needs no
    // second replay of the generator: one bit per member of the previous
    // layer (words(task) = ceil(members / 32), periodic in the layer) and
    // the forced pick of a task that took none (-1 otherwise)
    uint32_t* mask;           // [G * mask_per_dag], zeroed
    int32_t* forced;          // [G*n]
    const int32_t* wl_prefix; // [L+1] mask words of layers 0..l-1 (one period)
    int64_t mask_per_dag;     // mask words per DAG
};

__global__ void k_gen_layered_count(GenParams q);
// tiled factorizations (generate_tiled.cu): kind = TBSIM_TILED_*
int64_t tiled_task_count(int kind, int32_t nb);
__global__ void k_gen_tiled_count(int kind, int32_t nb, int32_t n, int32_t* off);
__global__ void k_gen_tiled_scan(int32_t n, int32_t* off, int64_t* tot);
__global__ void k_gen_tiled_fill(int kind, int32_t nb, int32_t n, int32_t n_handles, int64_t block_bytes,
                                 const int32_t* off, DevBatch b);
__global__ void k_gen_layered_expand(GenParams q, DevBatch b);

}  // namespace tbsim_dev
