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
__global__ void k_gen_layered_fill(GenParams q, DevBatch b);

}  // namespace tbsim_dev
