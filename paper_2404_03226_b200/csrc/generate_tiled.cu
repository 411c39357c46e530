// generate_tiled.cu -- the tiled factorization DAGs built on the device,
// bit-identical to the host builders (csrc/hostbatch.cpp, which replay the
// reference's build_cholesky_dag / build_lu_dag, src/generators.cpp:30-142;
// tiled QR is this repo's own).
//
// The host builders are loop nests that track the last writer of every tile.
// Here every task is decoded independently from its position: step k holds
// a fixed sequence of roles whose counts depend only on m = nb - k - 1, and
// every "last writer" is a closed-form task of step k or k - 1, so a thread
// per task writes its own dependencies, inputs and outputs.  Three kernels:
// per-task list lengths of ONE graph (all copies are identical), an exclusive
// scan of those lengths (the per-graph local offsets the batch layout uses),
// then every copy's entries.
#include <cstdint>

#include "blockscan.cuh"
#include "common.cuh"
#include "generate.cuh"
#include "hostbatch.hpp"

namespace tbsim_dev {

namespace {

using tbsim_host::T_GEMM;
using tbsim_host::T_GEQRT;
using tbsim_host::T_GETRF;
using tbsim_host::T_POTRF;
using tbsim_host::T_SYRK;
using tbsim_host::T_TRSM;
using tbsim_host::T_TSMQR;
using tbsim_host::T_TSQRT;
using tbsim_host::T_UNMQR;

// tasks of step k (m = nb - k - 1)
__host__ __device__ inline int64_t step_count(int kind, int64_t m) {
    if (kind == TBSIM_TILED_CHOLESKY) return 1 + 2 * m + m * (m - 1) / 2;  // POTRF, m TRSM, m SYRK, m(m-1)/2 GEMM
    return 1 + 2 * m + m * m;  // LU: GETRF, m+m TRSM, m^2 GEMM; QR: GEQRT, m UNMQR, m TSQRT, m^2 TSMQR
}

struct Task {
    int32_t type = 0, nd = 0, ni = 0, no = 0;
    int32_t dep[3], in[3], out[2];
    __device__ void d(int32_t x) {
        if (x < 0) return;
        for (int q = 0; q < nd; ++q)
            if (dep[q] == x) return;  // unique, first occurrence kept (gen_qr's dedup)
        dep[nd++] = x;
    }
};

struct Tiled {
    int kind;
    int32_t nb;
    __device__ int64_t base(int32_t k) const {  // first task of step k
        int64_t b = 0;
        for (int32_t s = 0; s < k; ++s) b += step_count(kind, nb - s - 1);
        return b;
    }
    // ---- Cholesky (tile(i,j) = i(i+1)/2 + j, generators.cpp:30-87)
    __device__ int32_t c_potrf(int32_t k) const { return static_cast<int32_t>(base(k)); }
    __device__ int32_t c_trsm(int32_t k, int32_t i) const { return static_cast<int32_t>(base(k) + 1 + (i - k - 1)); }
    __device__ int32_t c_syrk(int32_t k, int32_t i) const {
        const int64_t m = nb - k - 1, r = i - k - 1;
        return static_cast<int32_t>(base(k) + 1 + m + r + r * (r - 1) / 2);
    }
    __device__ int32_t c_gemm(int32_t k, int32_t i, int32_t j) const { return c_syrk(k, i) + 1 + (j - k - 1); }
    // ---- LU (tile(i,j) = i nb + j, generators.cpp:89-142)
    __device__ int32_t l_getrf(int32_t k) const { return static_cast<int32_t>(base(k)); }
    __device__ int32_t l_trow(int32_t k, int32_t j) const { return static_cast<int32_t>(base(k) + 1 + (j - k - 1)); }
    __device__ int32_t l_tcol(int32_t k, int32_t i) const {
        return static_cast<int32_t>(base(k) + 1 + (nb - k - 1) + (i - k - 1));
    }
    __device__ int32_t l_gemm(int32_t k, int32_t i, int32_t j) const {
        const int64_t m = nb - k - 1;
        return static_cast<int32_t>(base(k) + 1 + 2 * m + (i - k - 1) * m + (j - k - 1));
    }
    // ---- QR (GEQRT; UNMQR j>k; for i>k: TSQRT(i), TSMQR(i, j>k))
    __device__ int32_t q_geqrt(int32_t k) const { return static_cast<int32_t>(base(k)); }
    __device__ int32_t q_unmqr(int32_t k, int32_t j) const { return static_cast<int32_t>(base(k) + 1 + (j - k - 1)); }
    __device__ int32_t q_tsqrt(int32_t k, int32_t i) const {
        const int64_t m = nb - k - 1;
        return static_cast<int32_t>(base(k) + 1 + m + (i - k - 1) * (1 + m));
    }
    __device__ int32_t q_tsmqr(int32_t k, int32_t i, int32_t j) const { return q_tsqrt(k, i) + 1 + (j - k - 1); }

    __device__ Task task(int64_t t) const {
        Task r;
        int32_t k = 0;
        for (;; ++k) {
            const int64_t c = step_count(kind, nb - k - 1);
            if (t < c) break;
            t -= c;
        }
        const int32_t m = nb - k - 1;
        if (kind == TBSIM_TILED_CHOLESKY) {
            auto tile = [](int32_t i, int32_t j) { return i * (i + 1) / 2 + j; };
            if (t == 0) {  // POTRF(k): after SYRK(k-1, k)
                r.type = T_POTRF;
                if (k > 0) r.d(c_syrk(k - 1, k));
                r.in[r.ni++] = tile(k, k);
                r.out[r.no++] = tile(k, k);
            } else if (t <= m) {  // TRSM(k, i): after POTRF(k), GEMM(k-1, i, k)
                const int32_t i = k + static_cast<int32_t>(t);
                r.type = T_TRSM;
                r.d(c_potrf(k));
                if (k > 0) r.d(c_gemm(k - 1, i, k));
                r.in[r.ni++] = tile(k, k);
                r.in[r.ni++] = tile(i, k);
                r.out[r.no++] = tile(i, k);
            } else {
                int64_t u = t - 1 - m;
                int32_t row = 0;
                while (u >= 1 + row) { u -= 1 + row; ++row; }
                const int32_t i = k + 1 + row;
                if (u == 0) {  // SYRK(k, i): after TRSM(k, i), SYRK(k-1, i)
                    r.type = T_SYRK;
                    r.d(c_trsm(k, i));
                    if (k > 0) r.d(c_syrk(k - 1, i));
                    r.in[r.ni++] = tile(i, k);
                    r.in[r.ni++] = tile(i, i);
                    r.out[r.no++] = tile(i, i);
                } else {  // GEMM(k, i, j): after TRSM(k, i), TRSM(k, j), GEMM(k-1, i, j)
                    const int32_t j = k + static_cast<int32_t>(u);
                    r.type = T_GEMM;
                    r.d(c_trsm(k, i));
                    r.d(c_trsm(k, j));
                    if (k > 0) r.d(c_gemm(k - 1, i, j));
                    r.in[r.ni++] = tile(i, k);
                    r.in[r.ni++] = tile(j, k);
                    r.in[r.ni++] = tile(i, j);
                    r.out[r.no++] = tile(i, j);
                }
            }
        } else if (kind == TBSIM_TILED_LU) {
            const int32_t n = nb;
            auto tile = [n](int32_t i, int32_t j) { return i * n + j; };
            if (t == 0) {  // GETRF(k): after GEMM(k-1, k, k)
                r.type = T_GETRF;
                if (k > 0) r.d(l_gemm(k - 1, k, k));
                r.in[r.ni++] = tile(k, k);
                r.out[r.no++] = tile(k, k);
            } else if (t <= m) {  // row TRSM(k, j): after GETRF(k), GEMM(k-1, k, j)
                const int32_t j = k + static_cast<int32_t>(t);
                r.type = T_TRSM;
                r.d(l_getrf(k));
                if (k > 0) r.d(l_gemm(k - 1, k, j));
                r.in[r.ni++] = tile(k, k);
                r.in[r.ni++] = tile(k, j);
                r.out[r.no++] = tile(k, j);
            } else if (t <= 2 * m) {  // column TRSM(i, k): after GETRF(k), GEMM(k-1, i, k)
                const int32_t i = k + static_cast<int32_t>(t - m);
                r.type = T_TRSM;
                r.d(l_getrf(k));
                if (k > 0) r.d(l_gemm(k - 1, i, k));
                r.in[r.ni++] = tile(k, k);
                r.in[r.ni++] = tile(i, k);
                r.out[r.no++] = tile(i, k);
            } else {  // GEMM(k, i, j): after TRSM(i, k), TRSM(k, j), GEMM(k-1, i, j)
                const int64_t u = t - 1 - 2 * m;
                const int32_t i = k + 1 + static_cast<int32_t>(u / m), j = k + 1 + static_cast<int32_t>(u % m);
                r.type = T_GEMM;
                r.d(l_tcol(k, i));
                r.d(l_trow(k, j));
                if (k > 0) r.d(l_gemm(k - 1, i, j));
                r.in[r.ni++] = tile(i, k);
                r.in[r.ni++] = tile(k, j);
                r.in[r.ni++] = tile(i, j);
                r.out[r.no++] = tile(i, j);
            }
        } else {  // QR: every tile's last writer before step k is TSMQR(k-1, ., .)
            const int32_t n = nb;
            auto tile = [n](int32_t i, int32_t j) { return i * n + j; };
            if (t == 0) {  // GEQRT(k): after TSMQR(k-1, k, k)
                r.type = T_GEQRT;
                if (k > 0) r.d(q_tsmqr(k - 1, k, k));
                r.in[r.ni++] = tile(k, k);
                r.out[r.no++] = tile(k, k);
            } else if (t <= m) {  // UNMQR(k, j): after GEQRT(k), TSMQR(k-1, k, j)
                const int32_t j = k + static_cast<int32_t>(t);
                r.type = T_UNMQR;
                r.d(q_geqrt(k));
                if (k > 0) r.d(q_tsmqr(k - 1, k, j));
                r.in[r.ni++] = tile(k, k);
                r.in[r.ni++] = tile(k, j);
                r.out[r.no++] = tile(k, j);
            } else {
                const int64_t u = t - 1 - m;
                const int32_t i = k + 1 + static_cast<int32_t>(u / (1 + m));
                const int32_t c = static_cast<int32_t>(u % (1 + m));
                if (c == 0) {  // TSQRT(k, i): after the previous TS on (k,k), TSMQR(k-1, i, k)
                    r.type = T_TSQRT;
                    r.d(i == k + 1 ? q_geqrt(k) : q_tsqrt(k, i - 1));
                    if (k > 0) r.d(q_tsmqr(k - 1, i, k));
                    r.in[r.ni++] = tile(k, k);
                    r.in[r.ni++] = tile(i, k);
                    r.out[r.no++] = tile(k, k);
                    r.out[r.no++] = tile(i, k);
                } else {  // TSMQR(k, i, j): after TSQRT(k, i), the last writer of (k,j), TSMQR(k-1, i, j)
                    const int32_t j = k + c;
                    r.type = T_TSMQR;
                    r.d(q_tsqrt(k, i));
                    r.d(i == k + 1 ? q_unmqr(k, j) : q_tsmqr(k, i - 1, j));
                    if (k > 0) r.d(q_tsmqr(k - 1, i, j));
                    r.in[r.ni++] = tile(i, k);
                    r.in[r.ni++] = tile(k, j);
                    r.in[r.ni++] = tile(i, j);
                    r.out[r.no++] = tile(k, j);
                    r.out[r.no++] = tile(i, j);
                }
            }
        }
        return r;
    }
};

}  // namespace

int64_t tiled_task_count(int kind, int32_t nb) {
    int64_t n = 0;
    for (int32_t k = 0; k < nb; ++k) n += step_count(kind, nb - k - 1);
    return n;
}

// Per-task list lengths of one graph: off[0..3n+3) = dep, in, out counts
// (each array n+1 long, the last entry 0 for the scan).
__global__ void k_gen_tiled_count(int kind, int32_t nb, int32_t n, int32_t* off) {
    const Tiled tg{kind, nb};
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t <= n;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (t == n) {
            off[n] = off[2 * (n + 1) - 1] = off[3 * (n + 1) - 1] = 0;
            continue;
        }
        const Task r = tg.task(t);
        off[t] = r.nd;
        off[(n + 1) + t] = r.ni;
        off[2 * (n + 1) + t] = r.no;
    }
}

// One CTA: the three exclusive scans (local offsets of every copy) and
// their totals (tot[0..3) = E, I, O per graph).
__global__ void __launch_bounds__(1024) k_gen_tiled_scan(int32_t n, int32_t* off, int64_t* tot) {
    __shared__ int32_t warp_tot[32];
    for (int a = 0; a < 3; ++a) {
        const int32_t s = block_exclusive_scan_inplace(off + a * (n + 1), n + 1, warp_tot);
        if (threadIdx.x == 0) tot[a] = s;
        __syncthreads();
    }
}

// Every copy's offsets, entries, types and handle sizes.
__global__ void k_gen_tiled_fill(int kind, int32_t nb, int32_t n, int32_t n_handles, int64_t block_bytes,
                                 const int32_t* off, DevBatch b) {
    const Tiled tg{kind, nb};
    const int64_t total = b.G * static_cast<int64_t>(n + 1);
    for (int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < total;
         x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t g = x / (n + 1), t = x - g * (n + 1);
        int32_t* doff = const_cast<int32_t*>(b.dep_off) + b.task_base[g] + g;
        int32_t* ioff = const_cast<int32_t*>(b.in_off) + b.task_base[g] + g;
        int32_t* ooff = const_cast<int32_t*>(b.out_off) + b.task_base[g] + g;
        doff[t] = off[t];
        ioff[t] = off[(n + 1) + t];
        ooff[t] = off[2 * (n + 1) + t];
        if (t < n_handles) const_cast<int64_t*>(b.handle_bytes)[b.handle_base[g] + t] = block_bytes;
        if (t == n) continue;
        const Task r = tg.task(t);
        const_cast<int32_t*>(b.type)[b.task_base[g] + t] = r.type;
        int32_t* dep = const_cast<int32_t*>(b.dep) + b.edge_base[g] + off[t];
        int32_t* in = const_cast<int32_t*>(b.in) + b.in_base[g] + off[(n + 1) + t];
        int32_t* out = const_cast<int32_t*>(b.out) + b.out_base[g] + off[2 * (n + 1) + t];
        for (int q = 0; q < r.nd; ++q) dep[q] = r.dep[q];
        for (int q = 0; q < r.ni; ++q) in[q] = r.in[q];
        for (int q = 0; q < r.no; ++q) out[q] = r.out[q];
    }
}

}  // namespace tbsim_dev
