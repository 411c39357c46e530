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
};

__global__ void k_gen_layered_count(GenParams q);
// tiled factorizations (generate_tiled.cu): kind = TBSIM_TILED_*
int64_t tiled_task_count(int kind, int32_t nb);
__global__ void k_gen_tiled_count(int kind, int32_t nb, int32_t n, int32_t* off);
__global__ void k_gen_tiled_scan(int32_t n, int32_t* off, int64_t* tot);
__global__ void k_gen_tiled_fill(int kind, int32_t nb, int32_t n, int32_t n_handles, int64_t block_bytes,
                                 const int32_t* off, DevBatch b);
__global__ void k_gen_layered_fill(GenParams q, DevBatch b);

}  // namespace tbsim_dev
