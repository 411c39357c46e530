// rules.cuh -- the scheduling decision rules, written once and compiled
// twice: into the device engine (simulate.cu, nvcc) and into the host policy
// API that EngineView implementations call (api/policies.cpp, abi.cpp, g++).
// Everything here is scalar FP64/integer arithmetic in the reference's
// operation order (no FMA: nvcc -fmad=false, g++ -ffp-contract=off), so the
// host functions and the kernel agree bit for bit.  The warp-parallel parts
// (argmin over lanes, argmax over queue entries, in-order sums over
// shuffles) stay in simulate.cu; they combine the values computed here.
#pragma once

#include <cstdint>

#include "tbsim_b200.h"

#ifdef __CUDACC__
#define TBSIM_HD __host__ __device__ __forceinline__
#define TBSIM_ROLLED _Pragma("unroll 1")
#else
#define TBSIM_HD inline
#define TBSIM_ROLLED
#endif

namespace tbsim_rules {

// ------------------------------------------------------------- push keys
// push_fifo / push_dm / push_dmda (src/policies.cpp:37-72): each capable
// worker's key; the argmin keeps the lowest id on ties (key < best).

// std::max(now, free_at) (src/policies.cpp:50,60)
TBSIM_HD double start_at(double now, double free_at) { return now < free_at ? free_at : now; }

TBSIM_HD double fifo_key(int64_t queue_len, bool busy) {
    return static_cast<double>(queue_len) + (busy ? 1.0 : 0.0);
}

TBSIM_HD double dm_key(double now, double free_at, double exec) { return start_at(now, free_at) + exec; }

TBSIM_HD double dmda_key(double now, double free_at, double xfer, double exec) {
    return (start_at(now, free_at) + xfer) + exec;
}

// the policy's push key; dmdap and inspirit push like dmda
TBSIM_HD double push_key(int32_t policy, int64_t queue_len, bool busy, double now, double free_at, double xfer,
                         double exec) {
    if (policy == TBSIM_POLICY_FIFO) return fifo_key(queue_len, busy);
    if (policy == TBSIM_POLICY_DM) return dm_key(now, free_at, exec);
    return dmda_key(now, free_at, xfer, exec);
}

// -------------------------------------------------------------- pop keys
// pop_adaptive (src/policies.cpp:103-137): the (k0, k1) pair compared
// lexicographically, larger first; ties fall to the static priority
// (larger first), then to the queue's insertion order.  `frac` is called
// only in the locality mode (it walks the task's inputs).
template <class Frac>
TBSIM_HD void adaptive_key(int32_t mode, double ability, double efficiency, Frac frac, double& k0, double& k1) {
    if (mode == TBSIM_MODE_ABILITY) {
        k0 = ability;
        k1 = 0.0;
    } else if (mode == TBSIM_MODE_EFFICIENCY) {
        k0 = efficiency;
        k1 = 0.0;
    } else {
        k0 = frac();
        k1 = efficiency;
    }
}

// resident_fraction (src/engine.cpp:63-74): local bytes / total bytes
TBSIM_HD double resident_fraction(int64_t local_bytes, int64_t total_bytes) {
    return static_cast<double>(local_bytes) / static_cast<double>(total_bytes);
}

// ---------------------------------------------------------- cost model
// Platform::transfer_time_ms between distinct nodes (src/platform.cpp:56-63)
TBSIM_HD double transfer_ms(double latency_ms, int64_t bytes, double bandwidth) {
    return latency_ms + static_cast<double>(bytes) / bandwidth;
}

// CostTable::mean_ms (src/platform.cpp:39-50): the mean over the kinds that
// have an entry, CPU first; 0 when neither has one (the host API throws)
TBSIM_HD double mean_cost_ms(bool has_cpu, double cpu_ms, bool has_gpu, double gpu_ms) {
    double sum = 0.0;
    int n = 0;
    if (has_cpu) { sum += cpu_ms; ++n; }
    if (has_gpu) { sum += gpu_ms; ++n; }
    return n ? sum / n : 0.0;
}

// upward_rank_priority (src/attributes.cpp:234-253): rank ms -> int64 by
// truncation of rank * 1000
TBSIM_HD int64_t rank_priority(double rank_ms) { return static_cast<int64_t>(rank_ms * 1000.0); }

// ------------------------------------------------------------- regulator
// default_regulator_config (src/policies.cpp:139-151)
TBSIM_HD tbsim_regulator_cfg default_config(int64_t n_workers, double median_gpu_ms) {
    const int64_t tw = (n_workers + 3) / 4 > 2 ? (n_workers + 3) / 4 : 2;  // max(2, ceil(n/4))
    tbsim_regulator_cfg c{};
    c.task_window = tw;
    c.s_inc = n_workers;
    c.k_inc = static_cast<double>(n_workers) / median_gpu_ms;
    c.s_dec = tw;
    c.c = (tw + 1) / 2;
    c.dec_step = tw;
    c.slope_samples = 8;
    return c;
}

// calculate_k (src/policies.cpp:153-169): two-pass least-squares slope of
// nready over time; samples oldest first through the accessors.
template <class T, class N>
TBSIM_HD double slope(int32_t n, T time_at, N nready_at) {
    if (n < 2) return 0.0;
    double sx = 0.0, sy = 0.0;
    TBSIM_ROLLED
    for (int32_t i = 0; i < n; ++i) {
        sx += time_at(i);
        sy += static_cast<double>(nready_at(i));
    }
    const double dn = static_cast<double>(n);
    const double mx = sx / dn, my = sy / dn;
    double sxx = 0.0, sxy = 0.0;
    TBSIM_ROLLED
    for (int32_t i = 0; i < n; ++i) {
        const double dx = time_at(i) - mx;
        sxx += dx * dx;
        sxy += dx * (static_cast<double>(nready_at(i)) - my);
    }
    return sxx == 0.0 ? 0.0 : sxy / sxx;
}

// regulator_step (src/policies.cpp:171-203) after the sample is recorded:
// the trigger test ...
template <class Cfg>
TBSIM_HD bool regulator_fires(int64_t cur, int64_t last_trigger, const Cfg& cfg) {
    const int64_t d = cur - last_trigger;
    return !((d < 0 ? -d : d) < cfg.task_window);
}

// ... and the update when it fires.  `k` computes the slope over the
// recorded samples; it is called only on a rise of at least s_inc.
struct RegScalars {
    int32_t mode, phase;
    int64_t peak, prev_nready, last_trigger, s_dec_count;
    double cur_k;
};

template <class Cfg, class K>
TBSIM_HD void regulator_update(RegScalars& s, const Cfg& cfg, int64_t cur, K k) {
    s.last_trigger = cur;
    s.peak = cur > s.peak ? cur : s.peak;
    s.phase = cur >= s.peak - cfg.dec_step ? TBSIM_PHASE_INC : TBSIM_PHASE_DEC;
    if (s.phase == TBSIM_PHASE_INC) {
        if (cur - s.prev_nready >= cfg.s_inc) {
            s.cur_k = k();
            if (s.cur_k < cfg.k_inc) s.mode = TBSIM_MODE_EFFICIENCY;
            else if (s.cur_k > cfg.k_inc) s.mode = TBSIM_MODE_ABILITY;
        }
    } else if (cur > s.peak - cfg.s_dec * s.s_dec_count) {
        s.mode = TBSIM_MODE_ABILITY;
    } else if (cur <= s.peak - cfg.s_dec * (s.s_dec_count + 1) + cfg.c) {
        s.mode = TBSIM_MODE_LOCALITY;
        if (cur <= s.peak - cfg.s_dec * (s.s_dec_count + 1)) s.s_dec_count += 1;
    }
    s.prev_nready = cur;
}

}  // namespace tbsim_rules
