// generate.cu -- device-side replay of generate_layered_dag
// (src/generators.cpp:184-244), bit-identical to the host generator.
//
// One warp per DAG.  The std::mt19937_64 state (312 words) lives in shared
// memory; the twist runs lane-parallel in two dependency-free halves and the
// warp consumes draws 32 at a time, so the per-DAG draw sequence (one
// uniform01 per member of the previous layer, one forced uniform_below when
// none was taken, then one uniform_below(4) per handle) is exactly the
// reference's.  Pass 1 counts dependencies, degrees, types and handle sizes;
// after a scan over DAGs, pass 2 replays the dependency draws and writes the
// CSR entries.
#include <cstdint>

#include "blockscan.cuh"
#include "common.cuh"
#include "generate.cuh"

namespace tbsim_dev {

namespace {

constexpr int kNN = 312, kMM = 156;
__constant__ int64_t kTileBytes[4] = {160 * 160 * 4, 320 * 320 * 4, 640 * 640 * 4, 960 * 960 * 4};
constexpr uint64_t kMatA = 0xB5026F5AA96619E9ull, kUM = 0xFFFFFFFF80000000ull, kLM = 0x7FFFFFFFull;

struct WarpMT {
    uint64_t* mt;  // [312] in shared memory
    int idx;       // next word to temper
    int lane;

    __device__ void seed(uint64_t s) {
        if (lane == 0) {
            mt[0] = s;
            for (int i = 1; i < kNN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
        }
        __syncwarp();
        idx = kNN;
    }
    __device__ static uint64_t mix(uint64_t a, uint64_t b) {
        const uint64_t x = (a & kUM) | (b & kLM);
        return (x >> 1) ^ ((x & 1ull) ? kMatA : 0ull);
    }
    // i in [0,156): reads old mt[i+1], mt[i+156]; i in [156,311]: reads
    // old mt[i+1] (new mt[0] for i = 311) and new mt[i-156].
    __device__ void twist() {
        uint64_t v[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int i = lane + 32 * k;
            if (i < kMM) v[k] = mt[i + kMM] ^ mix(mt[i], mt[i + 1]);
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int i = lane + 32 * k;
            if (i < kMM) mt[i] = v[k];
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int i = kMM + lane + 32 * k;
            if (i < kNN) v[k] = mt[i - kMM] ^ mix(mt[i], mt[(i + 1) % kNN]);
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int i = kMM + lane + 32 * k;
            if (i < kNN) mt[i] = v[k];
        }
        __syncwarp();
        idx = 0;
    }
    __device__ static uint64_t temper(uint64_t x) {
        x ^= (x >> 29) & 0x5555555555555555ull;
        x ^= (x << 17) & 0x71D67FFFEDA60000ull;
        x ^= (x << 37) & 0xFFF7EEE000000000ull;
        x ^= x >> 43;
        return x;
    }
    // Up to 32 consecutive draws; lane j < count receives draw j.  Returns
    // the number delivered (may be less than want at a block boundary).
    __device__ int take(int want, uint64_t* out) {
        if (idx >= kNN) twist();
        const int count = min(want, min(32, kNN - idx));
        if (lane < count) *out = temper(mt[idx + lane]);
        idx += count;
        return count;
    }
    __device__ uint64_t one() {
        uint64_t x = 0;
        take(1, &x);
        return __shfl_sync(0xffffffffu, x, 0);
    }
};

// Draws for task i's dependencies: one uniform01 per member of layer-1,
// chosen when < p; a forced member when none is chosen.  emit(lane_mask of
// chosen members in this chunk, member base) is called per chunk.
// uniform01(x) < p (generators.cpp:20-22: (x >> 11) * 2^-53 < p) as one
// integer compare: k = x >> 11 < 2^53 is exact in a double and the scaling
// by 2^-53 is exact, so k * 2^-53 < p  <=>  k < p * 2^53  <=>  k < ceil(p * 2^53)
__device__ __forceinline__ uint64_t uniform01_threshold(double p) {
    const double s = p * 0x1.0p53;                  // exact (power-of-two scale)
    if (!(s > 0.0)) return 0;                       // p <= 0 or NaN: never taken
    if (s >= 0x1.0p53) return uint64_t(1) << 53;    // p >= 1: always taken
    return static_cast<uint64_t>(ceil(s));
}

template <typename Emit>
__device__ int deps_of(WarpMT& r, int i, int n, int L, uint64_t pt, Emit emit) {
    const int layer = i % L;
    if (layer == 0) return 0;
    const int prev = layer - 1;
    const int members = (n - 1 - prev) / L + 1;  // j = prev, prev+L, ... < n
    int taken = 0;
    for (int m0 = 0; m0 < members;) {
        uint64_t x = 0;
        const int got = r.take(members - m0, &x);
        const bool hit = r.lane < got && (x >> 11) < pt;
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        emit(bal, m0, prev);
        taken += __popc(bal);
        m0 += got;
    }
    if (taken == 0) {
        const uint64_t x = r.one();
        const int pick = static_cast<int>(x % static_cast<uint64_t>(members));
        emit(0u, -1 - pick, prev);  // forced member
        return 1;
    }
    return taken;
}

}  // namespace

// Pass 1: per-task dependency counts, degrees, types, handle sizes; per-DAG
// edge totals.
__global__ void __launch_bounds__(128) k_gen_layered_count(GenParams q) {
    __shared__ uint64_t mt_s[4][kNN];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t g = static_cast<int64_t>(blockIdx.x) * 4 + w;
    if (g >= q.G) return;
    const int n = q.n, L = q.L;
    WarpMT r{mt_s[w], kNN, lane};
    r.seed(q.seeds[g]);
    int32_t* ndep = q.ndep + g * n;   // dependency count per task
    int32_t* deg = q.degree + g * n;  // total degree per task
    for (int i = lane; i < n; i += 32) deg[i] = 0;
    __syncwarp();
    int64_t edges = 0;
    const uint64_t pt = uniform01_threshold(q.p);
    uint32_t* mask = q.mask + g * q.mask_per_dag;
    const int64_t period = q.wl_prefix[L];
    for (int i = 0; i < n; ++i) {
        uint32_t* mi = mask + static_cast<int64_t>(i / L) * period + q.wl_prefix[i % L];
        const int c = deps_of(r, i, n, L, pt, [&](unsigned bal, int m0, int prev) {
            if (m0 < 0) {
                if (lane == 0) {
                    atomicAdd(&deg[prev + (-1 - m0) * L], 1);
                    q.forced[g * n + i] = -1 - m0;
                }
            } else if ((bal >> lane) & 1u) {
                atomicAdd(&deg[prev + (m0 + lane) * L], 1);
                atomicOr(&mi[(m0 + lane) >> 5], 1u << ((m0 + lane) & 31));
            }
        });

        if (lane == 0) {
            ndep[i] = c;
            atomicAdd(&deg[i], c);
        }
        edges += c;
        __syncwarp();
    }
    // handle bytes: one uniform_below(4) per task, after every dependency draw
    for (int i0 = 0; i0 < n;) {
        uint64_t x = 0;
        const int got = r.take(n - i0, &x);
        if (lane < got) q.handle_bytes[g * n + i0 + lane] = kTileBytes[x % 4];
        i0 += got;
    }
    // type from total-degree quartiles: order statistics by counting
    __syncwarp();
    int32_t* hist = q.hist + g * (q.max_degree + 1);
    for (int d = lane; d <= q.max_degree; d += 32) hist[d] = 0;
    __syncwarp();
    // degrees were built with atomics (in L2): read them past L1
    for (int i = lane; i < n; i += 32) atomicAdd(&hist[min(__ldcg(&deg[i]), q.max_degree)], 1);
    __syncwarp();
    int32_t qv[3] = {0, 0, 0};
    if (lane == 0) {
        const int64_t want[3] = {static_cast<int64_t>((n - 1) * 0.25), static_cast<int64_t>((n - 1) * 0.5),
                                 static_cast<int64_t>((n - 1) * 0.75)};
        int64_t acc = 0;
        int k = 0;
        for (int d = 0; d <= q.max_degree && k < 3; ++d) {
            acc += __ldcg(&hist[d]);
            while (k < 3 && acc > want[k]) qv[k++] = d;
        }
    }
    for (int k = 0; k < 3; ++k) qv[k] = __shfl_sync(0xffffffffu, qv[k], 0);
    for (int i = lane; i < n; i += 32) {
        const int d = __ldcg(&deg[i]);
        q.type[g * n + i] = q.type_base + (d <= qv[0] ? 0 : d <= qv[1] ? 1 : d <= qv[2] ? 2 : 3);
    }
    if (lane == 0) q.edges[g] = edges;
}

// Pass 2: the CSR entries from pass 1's record -- a CTA per DAG scans the
// dependency counts into the local offsets, then a thread per task expands
// its member bits in ascending order (the draw order: members are drawn in
// ascending order, so the reference appends them in that order) or writes
// its forced pick.  Inputs alias the dependencies (same handles); output
// t is handle t.
__global__ void __launch_bounds__(256) k_gen_layered_expand(GenParams q, DevBatch b) {
    __shared__ int32_t warp_tot[32];
    const int n = q.n, L = q.L;
    const int64_t period = q.wl_prefix[L];
    for (int64_t g = blockIdx.x; g < q.G; g += gridDim.x) {
        int32_t* doff = const_cast<int32_t*>(b.dep_off) + b.task_base[g] + g;
        int32_t* ooff = const_cast<int32_t*>(b.out_off) + b.task_base[g] + g;
        int32_t* out = const_cast<int32_t*>(b.out) + b.out_base[g];
        int32_t* dep = const_cast<int32_t*>(b.dep) + b.edge_base[g];
        for (int i = threadIdx.x; i <= n; i += blockDim.x) {
            doff[i] = i < n ? q.ndep[g * n + i] : 0;
            ooff[i] = i;
            if (i < n) out[i] = i;
        }
        __syncthreads();
        block_exclusive_scan_inplace(doff, n + 1, warp_tot);
        const uint32_t* mask = q.mask + g * q.mask_per_dag;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int layer = i % L;
            if (layer == 0) continue;
            const int prev = layer - 1;
            int32_t at = doff[i];
            const int32_t f = q.forced[g * n + i];
            if (f >= 0) {
                dep[at] = prev + f * L;
                continue;
            }
            const int members = (n - 1 - prev) / L + 1;
            const uint32_t* mi = mask + static_cast<int64_t>(i / L) * period + q.wl_prefix[layer];
            for (int w = 0; w * 32 < members; ++w)
                for (uint32_t bits = mi[w]; bits; bits &= bits - 1) dep[at++] = prev + (32 * w + __ffs(bits) - 1) * L;
        }
        __syncthreads();
    }
}

}  // namespace tbsim_dev
