// simulate.cu -- batched, bit-exact replay of the reference's discrete-event
// list scheduler (src/engine.cpp) with its push/pop rules and the INSPIRIT
// Nready regulator (src/policies.cpp).  One warp simulates one DAG; lane w owns
// worker w (and w+32 when the platform has more than 32 workers).
//
// Event order without a heap.  The reference orders events by (time, seq)
// with seq a global enqueue counter (engine.cpp:16-31).  TaskReady/PushDone
// are always enqueued at `now` (engine.cpp:121,183), while TransferDone and
// TaskDone are enqueued strictly in the future (transfer > 0, exec > 0,
// engine.cpp:164-165; checked below, GS_DEGENERATE_TIME otherwise).  Hence at
// each time T the reference processes (1) every worker event stamped T in
// enqueue order, then (2) the TaskReady events those created, in creation
// order, then (3) the matching PushDones in the same order.  Each worker holds
// at most one pending TransferDone and one TaskDone, so the heap collapses to
// two slots per lane plus a ready list, and "next event" is a warp-wide
// (time, seq) min done with REDUX on 32-bit halves.
//
// worker_free_at (engine.cpp:53-59) is cached per lane and extended with
// `+= exec` on every push (the same left-to-right sum the reference forms);
// after a dispatch it is recomputed from busy_until in queue order.
// Transfer estimates (engine.cpp:105-110) are computed lanes-over-inputs and
// summed in input order with shuffles, so a push costs one round of loads
// instead of one dependent chain per input.
#include <climits>
#include <cstdint>
#include <type_traits>

#include "blockscan.cuh"
#include "common.cuh"
#include "ingest.cuh"
#include "rules.cuh"
#include "simulate.cuh"

namespace tbsim_dev {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint64_t ord_f64(double x) {
    const uint64_t u = dbits(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ uint64_t ord_i64(int64_t x) {
    return static_cast<uint64_t>(x) ^ 0x8000000000000000ull;
}

// POL >= 0 fixes the policy at compile time; POL < 0 (the shipped kernels)
// reads it at run time -- specialising saved <1% of the code.
//
// Register budget: only the state every event touches lives in registers
// (time, counters, the lane's workers); regulator state, counters and graph
// ids live in the warp's SimCold record, and state sections are addressed
// from one base plus the launch's layout offsets (kernel parameters).
template <int WPL, bool COMPACT, int POL, bool MANYIN>
struct Sim {
    using UnmetT = typename std::conditional<COMPACT, int16_t, int32_t>::type;
    using ResidT = typename std::conditional<COMPACT, uint8_t, uint32_t>::type;
    using KeyT = typename std::conditional<COMPACT, int16_t, int32_t>::type;
    using PrioT = typename std::conditional<COMPACT, int32_t, int64_t>::type;
    const SimParams* P;
    // the policy-specialised kernel is launched only without trace outputs
    // (abi.cpp), so its push/pop/sample recording compiles away
    static constexpr bool kTrace = POL < 0;
    char* base;  // this warp's state memory
    // ---- graph
    int32_t n;
    // queue capacity per worker of this graph: the warp's pool of
    // qcap x max_workers entries split over the graph's own W workers (a
    // 5-worker graph in a batch with 36-worker platforms gets 7x longer queues)
    int32_t qc;
    const SimTaskHdr* hdr;  // this graph's packed records
    __device__ __forceinline__ int32_t pol() const { return POL >= 0 ? POL : P->policy; }
    // ---- state sections
    __device__ __forceinline__ SimCold& cold() const { return *reinterpret_cast<SimCold*>(base + P->layout.cold); }
    __device__ __forceinline__ UnmetT* unmet() const { return reinterpret_cast<UnmetT*>(base + P->layout.unmet); }
    __device__ __forceinline__ ResidT* resid() const { return reinterpret_cast<ResidT*>(base + P->layout.resid); }
    __device__ __forceinline__ int32_t* queue(int32_t w) const {
        return reinterpret_cast<int32_t*>(base + P->layout.queue) + w * qc;
    }
    __device__ __forceinline__ KeyT* qab(int32_t w) const { return reinterpret_cast<KeyT*>(base + P->layout.qab) + w * qc; }
    __device__ __forceinline__ KeyT* qef(int32_t w) const { return reinterpret_cast<KeyT*>(base + P->layout.qef) + w * qc; }
    __device__ __forceinline__ PrioT* qprio(int32_t w) const {
        return reinterpret_cast<PrioT*>(base + P->layout.qprio) + w * qc;
    }
    __device__ __forceinline__ double* samp_t() const { return reinterpret_cast<double*>(base + P->layout.ring); }
    __device__ __forceinline__ int64_t* samp_n() const {
        return reinterpret_cast<int64_t*>(base + P->layout.ring + 8 * P->ring);
    }
    __device__ __forceinline__ double cost(int32_t ty, int32_t k) const {
        return reinterpret_cast<const double*>(base + P->layout.costs)[2 * ty + k];
    }
    __device__ __forceinline__ double bw(int32_t i) const { return reinterpret_cast<const double*>(base + P->layout.bw)[i]; }
    // ---- lane-owned workers.  wk packs valid (w < W) | gpu kind << 1 |
    // busy << 2 | free_at dirty << 3 | memory node << 4; a pending
    // TransferDone / TaskDone is (time, seq << kSeqShift | task) -- compact
    // graphs have < 2^15 tasks and < 2^16 events, so that is one 32-bit word
    using SlotT = typename std::conditional<COMPACT, uint32_t, uint64_t>::type;
    static constexpr int kSeqShift = COMPACT ? 16 : 32;
    static constexpr SlotT kNoSlot = ~SlotT(0);
    uint32_t wk[WPL];
    int32_t qlen[WPL];
    double busy_until[WPL], fsum[WPL];
    double xt[WPL], dt[WPL];
    SlotT xs[WPL], ds[WPL];
    __device__ __forceinline__ static SlotT mk_slot(uint32_t sq, int32_t task) {
        return (static_cast<SlotT>(sq) << kSeqShift) | static_cast<SlotT>(static_cast<uint32_t>(task));
    }
    __device__ __forceinline__ static int32_t slot_task(SlotT x) {
        return static_cast<int32_t>(x & ((static_cast<SlotT>(1) << kSeqShift) - 1));
    }
    __device__ __forceinline__ int32_t kind_of(int j) const { return (wk[j] >> 1) & 1u; }
    __device__ __forceinline__ bool busy_of(int j) const { return (wk[j] >> 2) & 1u; }
    __device__ __forceinline__ int32_t node_of(int j) const { return static_cast<int32_t>(wk[j] >> 4); }
    // ---- warp-uniform hot scalars
    int lane;
    double now;
    int32_t nready;
    int32_t rcount, rhead;  // ready list: rcount tasks linked from rhead (tail in SimCold)
    uint32_t seq;
    int32_t status;
    int32_t mode;
    // the last push's transfer estimate for the worker it chose (DMDA and
    // up): an immediate dispatch of that task (the worker idle, the queue
    // holding only it, no event in between) reuses it -- same inputs, same
    // residency, the same FP64 sum
    double pxfer;

    __device__ __forceinline__ void fail(int32_t st, int32_t task) {
        status = st;
        if (lane == 0) cold().aux = task;
    }

    // static priority from the record's second half (compact queues)
    __device__ __forceinline__ int64_t prio_of(int32_t task) const {
        const int2 p = __ldg(reinterpret_cast<const int2*>(hdr + task) + 3);
        return static_cast<int64_t>((static_cast<uint64_t>(static_cast<uint32_t>(p.y)) << 32) |
                                    static_cast<uint32_t>(p.x));
    }

    // first half of a packed record: (adj4, nin, nout, nsucc | type << 24)
    __device__ __forceinline__ int4 head(int32_t task) const {
        return __ldg(reinterpret_cast<const int4*>(hdr + task));
    }
    __device__ __forceinline__ const int32_t* lists(const int4& h) const {
        return P->adj + static_cast<uint32_t>(h.x);
    }

    // size of an input's handle: its byte class, or handle_bytes (escape)
    __device__ __forceinline__ int64_t bytes_of(int32_t word) const {
        const int32_t cls = static_cast<int32_t>(static_cast<uint32_t>(word) >> kHandleBits);
        if (cls != kEscapeClass) return __ldg(&P->class_bytes[cls]);
        return __ldg(&P->b.handle_bytes[cold().hb + (word & kHandleMask)]);
    }

    // transfer_one_ms (engine.cpp:86-103): fastest resident copy, ties to the
    // lowest node; Platform::transfer_time_ms (platform.cpp:56-63) looked up
    // per byte class (k_xfer_table), computed for escaped sizes.
    __device__ __forceinline__ double transfer_one(uint32_t m, int32_t word, int32_t to) const {
        if ((m >> to) & 1u) return 0.0;
        const int32_t nn = cold().nn;
        int32_t best = 0;
        double bbw = -1.0;
        for (uint32_t mm = m; mm; mm &= mm - 1) {
            const int32_t nd = __ffs(mm) - 1;
            const double b = bw(nd * nn + to);
            if (b > bbw) { bbw = b; best = nd; }
        }
        const int32_t cls = static_cast<int32_t>(static_cast<uint32_t>(word) >> kHandleBits);
        if (cls != kEscapeClass) {
            const int32_t mn = P->max_nodes;
            return __ldg(&cold().xt[(cls * mn + best) * mn + to]);
        }
        return tbsim_rules::transfer_ms(cold().lat, bytes_of(word), bw(best * nn + to));
    }

    // transfer_total_ms (engine.cpp:105-110) for node `want` (may differ per
    // lane).  Lanes hold (node, input) pairs -- all of them at once when
    // they fit in 32 lanes, else c = 32 / (distinct nodes) inputs per node
    // per round -- so every per-input transfer is computed once and in
    // parallel; each node's lane group then adds its terms in input order.
    // Over several rounds, zero terms are skipped: a resident input
    // contributes exactly +0.0 and the sum starts at +0.0 (it can never
    // become -0.0), so the in-order chain runs over non-resident inputs only.
    // TWO: the totals for this lane's two workers' nodes (want, want2) in one
    // pass -- two workers per lane push once instead of twice (the second
    // total is returned through x2)
    template <bool TWO = false>
    __device__ __forceinline__ double transfer_total_lanes(const int32_t* inw, int32_t nin, int32_t want,
                                                           int32_t want2 = 0, double* x2 = nullptr) const {
        if (nin == 0) {
            if constexpr (TWO) *x2 = 0.0;
            return 0.0;
        }
        const unsigned want_nodes = __reduce_or_sync(kFull, TWO ? (1u << want) | (1u << want2) : 1u << want);
        const int32_t nw = __popc(want_nodes);
        const ResidT* rs = resid();
        if constexpr (!MANYIN) {
            if (nin * nw <= 32) {  // one round: every (node, input) pair on its own lane
                // r = lane / nin without an integer divide (exact: lane < 32)
                const int32_t r = __float2int_rz(__fdividef(static_cast<float>(lane) + 0.5f, static_cast<float>(nin)));
                const int32_t k = lane - r * nin;
                double t = 0.0;
                if (r < nw) {
                    unsigned m = want_nodes;  // r-th set bit (few nodes; __fns is emulated)
                    for (int32_t i = 0; i < r; ++i) m &= m - 1;
                    const int32_t to = __ffs(m) - 1;
                    const int32_t wd = __ldg(&inw[k]);
                    t = transfer_one(rs[wd & kHandleMask], wd, to);
                }
                const int32_t b0 = (r < nw ? r : 0) * nin;
                // in-order sum; the shuffles are independent and issued ahead
                double acc = 0.0;
                int32_t j = 0;
#pragma unroll 1
                for (; j + 4 <= nin; j += 4) {
                    const double a0 = __shfl_sync(kFull, t, b0 + j), a1 = __shfl_sync(kFull, t, b0 + j + 1);
                    const double a2 = __shfl_sync(kFull, t, b0 + j + 2), a3 = __shfl_sync(kFull, t, b0 + j + 3);
                    acc += a0;
                    acc += a1;
                    acc += a2;
                    acc += a3;
                }
#pragma unroll 1
                for (; j < nin; ++j) acc += __shfl_sync(kFull, t, b0 + j);
                const int32_t rw = __popc(want_nodes & ((1u << want) - 1u));
                if constexpr (TWO) *x2 = __shfl_sync(kFull, acc, __popc(want_nodes & ((1u << want2) - 1u)) * nin);
                return __shfl_sync(kFull, acc, rw * nin);
            }
            // one pass per node, 32 inputs per round
            double mine = 0.0, mine2 = 0.0;
            for (unsigned wn = want_nodes; wn; wn &= wn - 1) {
                const int32_t to = __ffs(wn) - 1;
                double acc = 0.0;
                for (int32_t b0 = 0; b0 < nin; b0 += 32) {
                    const int32_t cnt = min(32, nin - b0);
                    double t = 0.0;
                    if (lane < cnt) {
                        const int32_t wd = __ldg(&inw[b0 + lane]);
                        t = transfer_one(rs[wd & kHandleMask], wd, to);
                    }
#pragma unroll 1
                    for (int32_t j = 0; j < cnt; ++j) acc += __shfl_sync(kFull, t, j);
                }
                if (want == to) mine = acc;
                if (TWO && want2 == to) mine2 = acc;
            }
            if constexpr (TWO) *x2 = mine2;
            return mine;
        } else {
            // rounds of c inputs per node, all nodes at once
            const int32_t c = 32 / nw;
            // r = lane / c without an integer divide (exact: lane < 32)
            const int32_t r = __float2int_rz(__fdividef(static_cast<float>(lane) + 0.5f, static_cast<float>(c)));
            const int32_t k = lane - r * c;
            const bool act = r < nw;
            unsigned m = want_nodes;  // r-th set bit (few nodes; __fns is emulated)
            for (int32_t i = 0; i < r; ++i) m &= m - 1;
            const int32_t to = act ? __ffs(m) - 1 : 0;
            const unsigned gmask = (c == 32 ? kFull : ((1u << c) - 1u)) << (act ? r * c : 0);
            double acc = 0.0;
            int32_t wd = 0;
            if (act && k < nin) wd = __ldg(&inw[k]);
#pragma unroll 1
            for (int32_t b0 = 0; b0 < nin; b0 += c) {
                const bool mine = act && b0 + k < nin;
                const int32_t wc = wd;
                if (act && b0 + c + k < nin) wd = __ldg(&inw[b0 + c + k]);  // next round
                const double t = mine ? transfer_one(rs[wc & kHandleMask], wc, to) : 0.0;
                unsigned nz = __ballot_sync(kFull, t != 0.0) & gmask;
                const int32_t steps = __reduce_max_sync(kFull, static_cast<unsigned>(__popc(nz)));
                // four shuffles in flight, then four in-order adds (an exhausted
                // lane adds +0.0, which leaves its sum unchanged)
#pragma unroll 1
                for (int32_t s = 0; s < steps; s += 4) {
                    double a[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        a[u] = __shfl_sync(kFull, t, nz ? __ffs(nz) - 1 : lane);
                        a[u] = nz ? a[u] : 0.0;
                        nz &= nz - 1;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc += a[u];
                }
            }
            const int32_t rw = __popc(want_nodes & ((1u << want) - 1u));
            if constexpr (TWO) *x2 = __shfl_sync(kFull, acc, __popc(want_nodes & ((1u << want2) - 1u)) * c);
            return __shfl_sync(kFull, acc, rw * c);
        }
    }

    // resident_fraction (engine.cpp:63-74)
    __device__ __forceinline__ double resident_fraction(int32_t task, int32_t nd) const {
        const int4 hd = head(task);
        const int32_t nin = hd.y;
        if (nin == 0) return 1.0;
        const int32_t* inw = lists(hd);
        const ResidT* rs = resid();
        int64_t total = 0, local = 0;
        for (int32_t k = 0; k < nin; ++k) {
            const int32_t wd = __ldg(&inw[k]);
            const int64_t by = bytes_of(wd);
            total += by;
            if ((static_cast<uint32_t>(rs[wd & kHandleMask]) >> nd) & 1u) local += by;
        }
        return tbsim_rules::resident_fraction(local, total);
    }

    // ---------------------------------------------------------- regulator
    __device__ __forceinline__ double calculate_k(const SimCold& c) const {  // policies.cpp:153-169
        const int ring_mask = P->ring - 1, head = c.r_head;
        const double* st = samp_t();
        const int64_t* sn = samp_n();
        return tbsim_rules::slope(
            c.r_count, [&](int32_t i) { return st[(head + i) & ring_mask]; },
            [&](int32_t i) { return sn[(head + i) & ring_mask]; });
    }

    // regulator_step (policies.cpp:171-203).  Every lane computes the same
    // values; lane 0 writes them back (the reads below come after the
    // __syncwarp of the previous step).
    __device__ __forceinline__ void regulator_step(int64_t cur) {
        SimCold& c = cold();
        const int ring_mask = P->ring - 1;
        int32_t r_head = c.r_head, r_count = c.r_count;
        const int idx = (r_head + r_count) & ring_mask;
        if (r_count <= ring_mask) ++r_count;
        else r_head = (r_head + 1) & ring_mask;
        while (r_count > c.cfg.slope_samples) {
            r_head = (r_head + 1) & ring_mask;
            --r_count;
        }
        const bool fires = tbsim_rules::regulator_fires(cur, c.last_trigger, c.cfg);
        __syncwarp();
        if (lane == 0) {
            samp_t()[idx] = now;
            samp_n()[idx] = cur;
            c.r_head = r_head;
            c.r_count = r_count;
        }
        if (!fires) {
            __syncwarp();
            return;
        }
        tbsim_rules::RegScalars rs{mode, c.phase, c.peak, c.prev_nready, c.last_trigger, c.s_dec_count, c.cur_k};
        tbsim_rules::regulator_update(rs, c.cfg, cur, [&] {
            __syncwarp();  // the sample just written
            return calculate_k(c);
        });
        mode = rs.mode;
        __syncwarp();
        if (lane == 0) {
            c.last_trigger = rs.last_trigger;
            c.peak = rs.peak;
            c.phase = rs.phase;
            c.cur_k = rs.cur_k;
            c.s_dec_count = rs.s_dec_count;
            c.prev_nready = rs.prev_nready;
        }
        __syncwarp();
    }

    __device__ __forceinline__ void queue_event() {
        SimCold& c = cold();
        if (kTrace && P->sample_time) {
            const int64_t ns = c.n_samp;
            __syncwarp();
            if (lane == 0) {
                P->sample_time[2 * c.t0 + ns] = now;
                P->sample_nready[2 * c.t0 + ns] = static_cast<int64_t>(nready);
                c.n_samp = ns + 1;
            }
            __syncwarp();
        }
        if (pol() == TBSIM_POLICY_INSPIRIT) regulator_step(static_cast<int64_t>(nready));
    }

    // ---------------------------------------------------------- push rules
    __device__ __forceinline__ void refresh_free() {
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
            const int32_t w = lane + 32 * j;
            if ((wk[j] & 13u) == 13u) {  // valid, busy, dirty
                double t = busy_until[j];
                const int32_t* q = queue(w);
                const int32_t kd = kind_of(j);
                for (int32_t i = 0; i < qlen[j]; ++i) t += cost(static_cast<uint32_t>(q[i]) >> 24, kd);
                fsum[j] = t;
                wk[j] &= ~8u;
            }
        }
    }

    // push_fifo / push_dm / push_dmda (policies.cpp:37-72): argmin over
    // capable workers, strict < so ties keep the lowest id.
    __device__ __forceinline__ int32_t select_worker(const int32_t* inw, int32_t nin, int32_t ty) {
        if (pol() != TBSIM_POLICY_FIFO) refresh_free();
        double xfer[WPL];
#pragma unroll
        for (int j = 0; j < WPL; ++j) xfer[j] = 0.0;
        if (pol() >= TBSIM_POLICY_DMDA) {
            if constexpr (WPL == 2) {
                xfer[0] = transfer_total_lanes<true>(inw, nin, node_of(0), node_of(1), &xfer[1]);
            } else {
#pragma unroll
                for (int j = 0; j < WPL; ++j) xfer[j] = transfer_total_lanes(inw, nin, node_of(j));
            }
        }
        uint64_t bk = ~0ull;
        int32_t bwk = INT_MAX;
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
            const int32_t w = lane + 32 * j;
            if (!(wk[j] & 1u)) continue;
            const double ce = cost(ty, kind_of(j));
            if (!(ce > 0.0)) continue;
            double key;
            if (pol() == TBSIM_POLICY_FIFO) {
                key = tbsim_rules::fifo_key(qlen[j], busy_of(j));
            } else {
                const double fa = busy_of(j) ? fsum[j] : now;
                if (pol() == TBSIM_POLICY_DM) key = tbsim_rules::dm_key(now, fa, ce);
                else key = tbsim_rules::dmda_key(now, fa, xfer[j], ce);
            }
            const uint64_t kb = ord_f64(key);
            if (kb < bk) { bk = kb; bwk = w; }
        }
        const uint64_t mk = warp_min_u64(bk);
        const int32_t w = __reduce_min_sync(kFull, bk == mk ? bwk : INT_MAX);
        if (pol() >= TBSIM_POLICY_DMDA && mk != ~0ull) {
            double xw = 0.0;
#pragma unroll
            for (int j = 0; j < WPL; ++j)
                if (j == (w >> 5)) xw = xfer[j];
            pxfer = __shfl_sync(kFull, xw, w & 31);
        }
        return mk == ~0ull ? -1 : w;
    }

    // ----------------------------------------------------------- pop rules
    // pop_fifo / pop_priority / pop_adaptive (policies.cpp:74-137) as one
    // lexicographic argmax over (k0, k1, static priority, -seq); queue
    // position is insertion (= seq) order.
    __device__ __forceinline__ int32_t select_entry(int32_t w, int32_t ql, int32_t nd) {
        if (pol() <= TBSIM_POLICY_DMDA) return 0;
        int32_t m = TBSIM_MODE_EFFICIENCY;
        if (pol() == TBSIM_POLICY_INSPIRIT) {
            m = mode;
            if (lane == 0) {
                SimCold& c = cold();
                if (m == 0) c.pop0 += 1;
                else if (m == 1) c.pop1 += 1;
                else c.pop2 += 1;
            }
        }
        if (ql == 1) return 0;  // a single entry is its own argmax
        const int32_t* q = queue(w);
        const KeyT* ka = qab(w);
        const KeyT* ke = qef(w);
        const PrioT* kp = qprio(w);
        uint64_t b0 = 0, b1 = 0, b2 = 0;
        int32_t bpos = INT_MAX;
        for (int32_t i = lane; i < ql; i += 32) {
            uint64_t k0, k1;
            if (pol() == TBSIM_POLICY_DMDAP) {
                k0 = k1 = 1;
            } else {
                double d0, d1;
                tbsim_rules::adaptive_key(m, static_cast<double>(ka[i]), static_cast<double>(ke[i]),
                                          [&] { return resident_fraction(q[i] & 0xffffff, nd); }, d0, d1);
                k0 = ord_f64(d0);
                k1 = ord_f64(d1);
            }
            const uint64_t k2 = ord_i64(COMPACT ? prio_of(q[i] & 0xffffff) : static_cast<int64_t>(kp[i]));
            const bool better = bpos == INT_MAX || k0 > b0 ||
                                (k0 == b0 && (k1 > b1 || (k1 == b1 && k2 > b2)));
            if (better) { b0 = k0; b1 = k1; b2 = k2; bpos = i; }
        }
        const bool has = bpos != INT_MAX;
        const uint64_t m0 = warp_max_u64(has ? b0 : 0);
        const bool c0 = has && b0 == m0;
        const uint64_t m1 = warp_max_u64(c0 ? b1 : 0);
        const bool c1 = c0 && b1 == m1;
        const uint64_t m2 = warp_max_u64(c1 ? b2 : 0);
        const bool c2 = c1 && b2 == m2;
        return __reduce_min_sync(kFull, c2 ? bpos : INT_MAX);
    }

    // ------------------------------------------------------------- engine
    // pushed: a push to w just happened and its queue event (the regulator
    // step) is still due -- both queue events of a push-then-pop run through
    // one call site of queue_event, which keeps the kernel's hot code small
    // (instruction-cache stalls are the simulator's largest stall class).
    __device__ __forceinline__ void maybe_dispatch(int32_t w, bool pushed) {  // engine.cpp:143-166
        const int j = w >> 5, owner = w & 31;
        // the owner's queue length, busy flag, kind and node in one shuffle
        // (ql < 2^24 entries, < 32 nodes)
        uint32_t pk = 0;
#pragma unroll
        for (int jj = 0; jj < WPL; ++jj)
            if (jj == j) pk = (static_cast<uint32_t>(qlen[jj]) << 8) | (wk[jj] & 6u) << 5 | node_of(jj);
        pk = __shfl_sync(kFull, pk, owner);
        const int32_t ql = static_cast<int32_t>(pk >> 8), bz = (pk >> 7) & 1, kd = (pk >> 6) & 1,
                      nd = static_cast<int32_t>(pk & 31u);
        uint32_t e = 0;
        int64_t slot = 0;
        int4 hd = make_int4(0, 0, 0, 0);
#pragma unroll 1
        for (int k = pushed ? 0 : 1; k < 2; ++k) {
            if (k == 1) {
                if (bz || ql == 0) return;
                const int32_t pick = select_entry(w, ql, nd);
                int32_t* q = queue(w);
                KeyT* ka = qab(w);
                KeyT* ke = qef(w);
                PrioT* kp = qprio(w);
                e = static_cast<uint32_t>(q[pick]);
                __syncwarp();
                const bool ins = pol() == TBSIM_POLICY_INSPIRIT, pri = !COMPACT && pol() >= TBSIM_POLICY_DMDAP;
                for (int32_t b0 = pick; b0 < ql - 1; b0 += 32) {
                    const int32_t i = b0 + lane;
                    const bool mv = i < ql - 1;
                    int32_t val = 0;
                    KeyT va = 0, ve = 0;
                    PrioT vp = 0;
                    if (mv) {
                        val = q[i + 1];
                        if (ins) { va = ka[i + 1]; ve = ke[i + 1]; }
                        if (pri) vp = kp[i + 1];
                    }
                    __syncwarp();
                    if (mv) {
                        q[i] = val;
                        if (ins) { ka[i] = va; ke[i] = ve; }
                        if (pri) kp[i] = vp;
                    }
                    __syncwarp();
                }
                const int32_t task = static_cast<int32_t>(e & 0xffffffu);
                hd = head(task);  // issued before the queue bookkeeping
                nready -= 1;
                // dispatch counter and log slot: lane 0 only (cold state)
                if (lane == 0) {
                    SimCold& c = cold();
                    slot = c.t0 + c.n_pop;
                    c.n_pop += 1;
                    if (kTrace && P->pop_time) {
                        P->pop_time[slot] = now;
                        P->pop_task[slot] = task;
                        P->pop_worker[slot] = w;
                    }
                }
            }
            queue_event();
        }
        const int32_t task = static_cast<int32_t>(e & 0xffffffu);
        const int32_t ty = static_cast<int32_t>(e >> 24);
        // pushed to an idle worker with an empty queue: the push's estimate
        const bool reuse = pushed && ql == 1 && pol() >= TBSIM_POLICY_DMDA;
        const double xfer = reuse ? pxfer : transfer_total_lanes(lists(hd), hd.y, nd);
        const double exec = cost(ty, kd);
        const double start = now + xfer;
        const double end = start + exec;
        if ((xfer > 0.0 && !(start > now)) || !(end > now)) {
            fail(GS_DEGENERATE_TIME, task);
            return;
        }
        if (lane == 0) {  // dispatch log: sequential, scattered by k_sim_scatter
            SimLog* lg = P->log + slot;
            *reinterpret_cast<int2*>(lg) = make_int2(task, w);
            lg->start = start;
            lg->end = end;
        }
        const uint32_t sx = seq;
        if (xfer > 0.0) ++seq;
        const uint32_t sd = seq++;
#pragma unroll
        for (int jj = 0; jj < WPL; ++jj)
            if (jj == j && lane == owner) {
                qlen[jj] -= 1;
                wk[jj] |= 12u;  // busy, free_at dirty
                busy_until[jj] = end;
                if (xfer > 0.0) { xt[jj] = start; xs[jj] = mk_slot(sx, task); }
                dt[jj] = end; ds[jj] = mk_slot(sd, task);
            }
    }

    // push rule + queue insert; returns the chosen worker (dispatch follows
    // in run(), so the dispatch code exists once in the kernel)
    __device__ __forceinline__ int32_t on_push(int32_t task) {  // engine.cpp:124-141
        // the whole record in two 16-byte loads of one sector; the pop keys
        // ride along while the push rule runs
        const int4 hd = head(task);
        const int4 kk = __ldg(reinterpret_cast<const int4*>(hdr + task) + 1);
        const int32_t ty = static_cast<int32_t>((static_cast<uint32_t>(hd.w) >> 24) & 0x3fu);
        const int32_t ka = kk.x, ke = kk.y;
        const int64_t kp = static_cast<int64_t>((static_cast<uint64_t>(static_cast<uint32_t>(kk.w)) << 32) |
                                                static_cast<uint32_t>(kk.z));
        const bool too_large = ka < 0;  // pop keys beyond int32 or > 2^24 successor entries
        const int32_t w = select_worker(lists(hd), hd.y, ty);
        if (w < 0) { fail(GS_NO_WORKER, task); return -1; }
        if (too_large) { fail(GS_TOO_LARGE, task); return -1; }
        // compact keys: ability/efficiency < n < 2^15 always fit; the
        // static priority stays in the task record
        const int j = w >> 5, owner = w & 31;
        int32_t ovf = 0;
#pragma unroll
        for (int jj = 0; jj < WPL; ++jj)
            if (jj == j && lane == owner) {
                if (qlen[jj] >= qc) {
                    ovf = 1;
                } else {
                    const int32_t at = qlen[jj];
                    queue(w)[at] = (ty << 24) | task;
                    if (pol() == TBSIM_POLICY_INSPIRIT) {
                        qab(w)[at] = static_cast<KeyT>(ka);
                        qef(w)[at] = static_cast<KeyT>(ke);
                    }
                    if (!COMPACT && pol() >= TBSIM_POLICY_DMDAP) qprio(w)[at] = static_cast<PrioT>(kp);
                    qlen[jj] += 1;
                    if ((wk[jj] & 12u) == 4u) fsum[jj] += cost(ty, kind_of(jj));  // busy, not dirty
                }
            }
        if (__shfl_sync(kFull, ovf, owner)) { fail(GS_QUEUE_OVERFLOW, task); return -1; }
        __syncwarp();
        nready += 1;
        if (kTrace && P->push_time) {
            SimCold& c = cold();
            const int64_t np = c.n_push;
            __syncwarp();
            if (lane == 0) {
                P->push_time[c.t0 + np] = now;
                P->push_task[c.t0 + np] = task;
                c.n_push = np + 1;
            }
            __syncwarp();
        }
        return w;  // its queue event runs in maybe_dispatch(w, true)
    }

    // Appends the lanes with `rdy` (task v) to the ready list in lane order:
    // each ready task's unmet slot (now dead) links to the next ready task.
    __device__ __forceinline__ void ready_append(bool rdy, int32_t v) {
        const unsigned bal = __ballot_sync(kFull, rdy);
        if (!bal) return;
        UnmetT* um = unmet();
        const unsigned above = bal & ~((2u << lane) - 1u);  // (2u << 31) == 0: no lanes above 31
        const int32_t nv = __shfl_sync(kFull, v, above ? __ffs(above) - 1 : lane);
        const int first = __ffs(bal) - 1, last = 31 - __clz(bal);
        if (rdy && above) um[v] = static_cast<UnmetT>(nv);
        if (lane == first && rcount > 0) um[cold().rtail] = static_cast<UnmetT>(v);
        __syncwarp();
        if (lane == last) cold().rtail = v;
        const int32_t fv = __shfl_sync(kFull, v, first);
        if (rcount == 0) rhead = fv;
        rcount += __popc(bal);
    }

    __device__ __forceinline__ void run() {  // Simulation::run, engine.cpp:207-248
        // roots in position order (engine.cpp:218-221)
        UnmetT* um = unmet();
        ResidT* rs = resid();
        const int32_t* doff = P->b.dep_off + cold().t0 + cold().g;
        rcount = 0;
        for (int32_t b0 = 0; b0 < n; b0 += 32) {
            const int32_t v = b0 + lane;
            bool root = false;
            if (v < n) {
                const int32_t deg = __ldg(&doff[v + 1]) - __ldg(&doff[v]);
                um[v] = static_cast<UnmetT>(deg);
                root = deg == 0;
            }
            __syncwarp();
            ready_append(root, v);
            __syncwarp();
        }
        {
            const int64_t g = cold().g;
            const int32_t nh = static_cast<int32_t>(P->b.handle_base[g + 1] - P->b.handle_base[g]);
            for (int32_t h = lane; h < nh; h += 32) rs[h] = 1u;  // engine.cpp:215-216
        }
        __syncwarp();
        // One loop, one dispatch site: phase A pushes the tasks made ready
        // at `now` in creation order (2)+(3); phase B drains the worker
        // events stamped `now` in enqueue order (1), then time advances.
        bool events = false;
        for (;;) {
            int32_t w;
            bool pushed = false;
            if (!events) {
                if (rcount > 0) {
                    const int32_t v = rhead;
                    const int32_t nx = rcount > 1 ? static_cast<int32_t>(um[v]) : 0;
                    --rcount;
                    w = on_push(v);
                    rhead = nx;
                    if (status != GS_OK) return;
                    pushed = true;
                } else {
                    // next worker-event time
                    uint64_t lt = ~0ull;
#pragma unroll
                    for (int j = 0; j < WPL; ++j) {
                        if (xs[j] != kNoSlot) lt = min(lt, dbits(xt[j]));
                        if (ds[j] != kNoSlot) lt = min(lt, dbits(dt[j]));
                    }
                    const uint64_t mt = warp_min_u64(lt);
                    if (mt == ~0ull) break;
                    now = __longlong_as_double(static_cast<long long>(mt));
                    events = true;
                    continue;
                }
            } else {
                // the earliest-enqueued event stamped `now`: slots order by seq
                SlotT ls = kNoSlot;
                const uint64_t mt = dbits(now);
#pragma unroll
                for (int j = 0; j < WPL; ++j) {
                    if (xs[j] != kNoSlot && dbits(xt[j]) == mt) ls = min(ls, xs[j]);
                    if (ds[j] != kNoSlot && dbits(dt[j]) == mt) ls = min(ls, ds[j]);
                }
                SlotT ms;
                if constexpr (COMPACT) ms = __reduce_min_sync(kFull, ls);
                else ms = warp_min_u64(ls);
                if (ms == kNoSlot) {
                    events = false;
                    continue;
                }
                const int owner = __ffs(__ballot_sync(kFull, ls == ms)) - 1;
                int32_t info = 0;
                if (lane == owner) {
#pragma unroll
                    for (int j = 0; j < WPL; ++j) {
                        if (xs[j] == ms) { info = (j << 30) | node_of(j); xs[j] = kNoSlot; }
                        if (ds[j] == ms) { info = (1 << 29) | (j << 30) | node_of(j); ds[j] = kNoSlot; }
                    }
                }
                info = __shfl_sync(kFull, info, owner);
                const int32_t task = slot_task(ms);
                w = owner + 32 * (static_cast<uint32_t>(info) >> 30);
                const bool is_done = (info >> 29) & 1;
                const int32_t nd = info & 0xff;
                const uint32_t bit = 1u << nd;
                const int4 hd = head(task);
                const int32_t nin = hd.y, nout = hd.z;
                const int32_t* inh = lists(hd);
                if (!is_done) {  // TransferDone: inputs resident (engine.cpp:168-172)
                    for (int32_t k = lane; k < nin; k += 32) {
                        const int32_t h = __ldg(&inh[k]) & kHandleMask;
                        rs[h] = static_cast<ResidT>(rs[h] | bit);
                    }
                    __syncwarp();
                    continue;
                }
                // TaskDone (engine.cpp:174-185)
                const int32_t* outl = inh + nin;
                for (int32_t k = lane; k < nout; k += 32) {
                    const int32_t h = __ldg(&outl[k]);
                    rs[h] = static_cast<ResidT>(rs[h] | bit);
                }
#pragma unroll
                for (int j = 0; j < WPL; ++j)
                    if (j == (w >> 5) && lane == owner) wk[j] &= ~4u;
                // successors: sorted, multi-edges adjacent; the lowest lane of
                // each run of equal ids decrements by the run length
                const int32_t* succl = outl + nout;
                const int32_t s1 = static_cast<int32_t>(static_cast<uint32_t>(hd.w) & 0xffffffu);
                // multi-edges (bit 30, k_sim_pack) are adjacent in the sorted
                // list: the lowest lane of each run decrements by its length;
                // lists without them decrement by one per lane
                const bool dups = (static_cast<uint32_t>(hd.w) >> 30) & 1u;
                for (int32_t b0 = 0; b0 < s1; b0 += 32) {
                    const int32_t k = b0 + lane;
                    const bool valid = k < s1;
                    const int32_t sv = valid ? __ldg(&succl[k]) : -1 - lane;
                    int32_t dec = valid ? 1 : 0;
                    if (dups) {
                        const unsigned peers = __match_any_sync(kFull, sv);
                        dec = valid && (__ffs(peers) - 1) == lane ? __popc(peers) : 0;
                    }
                    bool rdy = false;
                    if (dec) {
                        const int32_t left = static_cast<int32_t>(um[sv]) - dec;
                        um[sv] = static_cast<UnmetT>(left);
                        rdy = left == 0;
                        // its push reads the record soon: into L1 now
                        if (rdy) asm volatile("prefetch.global.L1 [%0];" ::"l"(hdr + sv));
                    }
                    __syncwarp();
                    ready_append(rdy, sv);
                    __syncwarp();
                }
                __syncwarp();
            }
            maybe_dispatch(w, pushed);
            if (status != GS_OK) return;
        }
    }
};

// SMEM: the per-warp state lives in shared memory (provably, so every state
// access compiles to 32-bit-addressed LDS/STS); otherwise in HBM.
template <int WPL, bool COMPACT, int POL, bool MANYIN, bool SMEM>
__device__ void simulate_impl(const SimParams& p) {
    extern __shared__ __align__(16) char smem[];
    const int lane = threadIdx.x & 31;
    const int warp_in_block = threadIdx.x >> 5;
    const int warps_per_block = blockDim.x >> 5;
    char* base;
    if constexpr (SMEM) {
        // the warp's state offset passes through an opaque move so the
        // compiler keeps it in a register instead of re-deriving it from
        // %tid (S2R + shift + multiply) at every state access
        uint32_t off = static_cast<uint32_t>(warp_in_block) * static_cast<uint32_t>(p.state_bytes);
        asm volatile("mov.b32 %0, %1;" : "=r"(off) : "r"(off));
        base = smem + off;
    } else base = p.gstate + (static_cast<int64_t>(blockIdx.x) * warps_per_block + warp_in_block) * p.state_bytes;
    const DevBatch& b = p.b;
    using S = Sim<WPL, COMPACT, POL, MANYIN>;
    S s;
    s.P = &p;
    s.base = base;
    s.lane = lane;
    SimCold& c = s.cold();
    int32_t loaded_pf = -1;

    for (;;) {
        unsigned long long item = 0;
        if (lane == 0) item = atomicAdd(p.work_counter, 1ull);
        item = __shfl_sync(kFull, item, 0);
        if (item >= static_cast<unsigned long long>(p.n_items_dev ? *p.n_items_dev : p.n_items)) break;
        const int64_t g = p.graph_list ? p.graph_list[item] : static_cast<int64_t>(item);
        const int64_t t0 = b.task_base[g];
        s.n = static_cast<int32_t>(b.task_base[g + 1] - t0);
        s.hdr = p.hdr + t0;
        const int32_t pfi = p.platform_of ? p.platform_of[g] : 0;
        const DevPlatform* pf = p.platforms + pfi;
        const int32_t W = pf->n_workers, nn = pf->n_nodes;
        s.qc = static_cast<int32_t>(
            std::min<int64_t>(static_cast<int64_t>(p.qcap) * p.max_workers / (W > 0 ? W : 1), INT32_MAX / 64));
        __syncwarp();
        if (pfi != loaded_pf) {  // platform tables into this warp's state
            double* costs = reinterpret_cast<double*>(base + p.layout.costs);
            double* bw = reinterpret_cast<double*>(base + p.layout.bw);
            for (int i = lane; i < p.n_types; i += 32) {
                costs[2 * i] = pf->costs.cpu[i];
                costs[2 * i + 1] = pf->costs.gpu[i];
            }
            for (int i = lane; i < nn * nn; i += 32) bw[i] = pf->bw[(i / nn) * kMaxNodes + i % nn];
            loaded_pf = pfi;
        }
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
            const int32_t w = lane + 32 * j;
            s.wk[j] = w < W ? (1u | (pf->kind[w] ? 2u : 0u) | (static_cast<uint32_t>(pf->node[w]) << 4)) : 0u;
            s.qlen[j] = 0;
            s.busy_until[j] = 0.0;
            s.fsum[j] = 0.0;
            s.xt[j] = s.dt[j] = 0.0;
            s.xs[j] = s.ds[j] = S::kNoSlot;
        }
        s.now = 0.0;
        s.nready = 0;
        s.rcount = s.rhead = 0;
        s.seq = 0;
        s.status = GS_OK;
        if (lane == 0) {
            c.g = g;
            c.t0 = t0;
            c.nn = nn;
            c.lat = pf->latency_ms;
            c.xt = p.xtab + static_cast<int64_t>(pfi) * kByteClasses * p.max_nodes * p.max_nodes;
            c.hb = b.handle_base[g];
            c.n_push = c.n_samp = 0;
            c.n_pop = 0;
            c.pop0 = c.pop1 = c.pop2 = 0;
            c.aux = -1;
            // regulator config: explicit, or default_regulator_config
            // (policies.cpp:139-151) from the worker count and the median
            if (p.reg) {
                c.cfg = p.reg[g];
            } else {
                c.cfg = tbsim_rules::default_config(W, p.median[g * p.median_stride]);
            }
        }
        // regulator state: caller-provided (in/out) or RegulatorState{}
        if (p.reg_state) {
            const tbsim_regulator_state& rs = p.reg_state[g];
            s.mode = rs.mode;
            if (lane == 0) {
                c.phase = rs.phase; c.peak = rs.peak; c.prev_nready = rs.prev_nready;
                c.last_trigger = rs.last_trigger_nready; c.s_dec_count = rs.s_dec_count; c.cur_k = rs.cur_k;
                c.r_head = 0;
                c.r_count = rs.n_samples;
            }
            for (int i = lane; i < rs.n_samples; i += 32) { s.samp_t()[i] = rs.sample_time[i]; s.samp_n()[i] = rs.sample_nready[i]; }
        } else {
            s.mode = TBSIM_MODE_EFFICIENCY;
            if (lane == 0) {
                c.phase = TBSIM_PHASE_INC; c.peak = 0; c.prev_nready = 0;
                c.last_trigger = 0; c.s_dec_count = 1; c.cur_k = 0.0; c.r_head = 0; c.r_count = 0;
            }
        }
        __syncwarp();
        s.run();
        __syncwarp();
        // every dispatched task has completed once no event is pending, so
        // the dispatch count is the completion count (engine.cpp:235-246)
        const int32_t done = c.n_pop;
        if (s.status == GS_OK && done == s.n) {
            if (lane == 0) p.n_disp[g] = done;
        } else {
            // failed graph: outputs written here (undispatched tasks keep
            // worker -1), k_sim_scatter skips it
            for (int32_t v = lane; v < s.n; v += 32) {
                p.worker[t0 + v] = -1;
                p.start_ms[t0 + v] = 0.0;
                p.end_ms[t0 + v] = 0.0;
            }
            __syncwarp();
            for (int64_t i = lane; i < done; i += 32) {
                const SimLog e = p.log[t0 + i];
                p.worker[t0 + e.task] = e.worker;
                p.start_ms[t0 + e.task] = e.start;
                p.end_ms[t0 + e.task] = e.end;
            }
            if (lane == 0) p.n_disp[g] = -1;
        }
        if (lane == 0) {
            int32_t st = s.status;
            if (st == GS_OK && done != s.n) st = GS_STUCK;
            p.status[g] = st;
            // aux: the failing task's position, its type id in bits 24..30
            // (error texts name the type without reading the batch back)
            p.status_aux[g] = c.aux >= 0 ? (c.aux | (__ldg(&b.type[t0 + c.aux]) << 24)) : c.aux;
            // makespan: the last completion (times only grow; a completed
            // graph's last event is a TaskDone)
            p.makespan[g] = done > 0 ? s.now : 0.0;
            p.completed[g] = done;
            if (p.pop_counts) {
                p.pop_counts[3 * g + 0] = c.pop0;
                p.pop_counts[3 * g + 1] = c.pop1;
                p.pop_counts[3 * g + 2] = c.pop2;
            }
            if (p.reg_state && p.policy == TBSIM_POLICY_INSPIRIT && s.status == GS_OK) {
                tbsim_regulator_state& rs = p.reg_state[g];
                rs.mode = s.mode; rs.phase = c.phase; rs.peak = c.peak; rs.prev_nready = c.prev_nready;
                rs.last_trigger_nready = c.last_trigger; rs.s_dec_count = c.s_dec_count; rs.cur_k = c.cur_k;
                rs.n_samples = c.r_count;
            }
        }
        __syncwarp();
        if (p.reg_state && p.policy == TBSIM_POLICY_INSPIRIT && s.status == GS_OK) {
            tbsim_regulator_state& rs = p.reg_state[g];
            const int ring_mask = p.ring - 1;
            for (int i = lane; i < c.r_count; i += 32) {
                const int idx = (c.r_head + i) & ring_mask;
                rs.sample_time[i] = s.samp_t()[idx];
                rs.sample_nready[i] = s.samp_n()[idx];
            }
        }
        __syncwarp();
    }
}

__device__ __forceinline__ int64_t graph_of(const DevBatch& b, int64_t t) {
    // largest g with task_base[g] <= t (empty graphs share a base and sort first)
    int64_t lo = 0, hi = b.G;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(&b.task_base[mid]) <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}

}  // namespace

// Structural half of the packed simulation graph (record words 0-3 and the
// lists); depends only on the batch, so it is built once per batch, at
// upload (k_ingest's stream) or on first use.
template <int TL>
__global__ void __launch_bounds__(256) k_sim_pack(DevBatch b, const uint8_t* hcls, SimTaskHdr* hdr, int32_t* adj) {
    // input list word: handle | size class << 28 (k_bytes_class)
    auto word = [&](int32_t h, uint8_t c) {
        return static_cast<int32_t>(static_cast<uint32_t>(h) | (static_cast<uint32_t>(c) << kHandleBits));
    };
    // teams of TL lanes, each over a contiguous range of tasks: the team
    // loads the offsets of its next TL tasks at once (lane j: task j, one
    // coalesced load) and hands them out by shuffles, copies each task's
    // lists in parallel, and follows graph boundaries incrementally (one
    // search per team)
    const int tl = threadIdx.x & (TL - 1);
    const unsigned tmask = (TL == 32 ? 0xffffffffu : ((1u << TL) - 1u)) << ((threadIdx.x & 31) & ~(TL - 1));
    const int64_t team = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / TL;
    const int64_t nteams = static_cast<int64_t>(gridDim.x) * blockDim.x / TL;
    const int64_t per = (b.T + nteams - 1) / nteams;
    const int64_t tend = min(b.T, (team + 1) * per);
    int64_t t = team * per;
    if (t >= tend) return;
    int64_t g = graph_of(b, t);
    int64_t t0 = __ldg(&b.task_base[g]), t1 = __ldg(&b.task_base[g + 1]);
    int64_t ib = __ldg(&b.in_base[g]), ob = __ldg(&b.out_base[g]), eb = __ldg(&b.edge_base[g]);
    int64_t hb = __ldg(&b.handle_base[g]);
    while (t < tend) {
        if (t >= t1) {  // next non-empty graph
            do {
                ++g;
                t0 = t1;
                t1 = __ldg(&b.task_base[g + 1]);
            } while (t >= t1);
            ib = __ldg(&b.in_base[g]); ob = __ldg(&b.out_base[g]); eb = __ldg(&b.edge_base[g]);
            hb = __ldg(&b.handle_base[g]);
        }
        const int32_t nb = static_cast<int32_t>(min(static_cast<int64_t>(TL), min(t1, tend) - t));
        const int64_t v0 = t - t0;
        const int32_t* ioff = b.in_off + t0 + g;
        const int32_t* ooff = b.out_off + t0 + g;
        const int32_t* soff = b.succ_off + t0 + g;
        int32_t li0 = 0, li1 = 0, lo0 = 0, lo1 = 0, ls0 = 0, ls1 = 0, lty = 0;
        if (tl < nb) {
            li0 = __ldg(&ioff[v0 + tl]); li1 = __ldg(&ioff[v0 + tl + 1]);
            lo0 = __ldg(&ooff[v0 + tl]); lo1 = __ldg(&ooff[v0 + tl + 1]);
            ls0 = soff[v0 + tl]; ls1 = soff[v0 + tl + 1];  // written by k_ingest
            lty = __ldg(&b.type[t + tl]);
        }
        for (int32_t j = 0; j < nb; ++j, ++t) {
            const int32_t i0 = __shfl_sync(tmask, li0, j, TL), i1 = __shfl_sync(tmask, li1, j, TL);
            const int32_t o0 = __shfl_sync(tmask, lo0, j, TL), o1 = __shfl_sync(tmask, lo1, j, TL);
            const int32_t s0 = __shfl_sync(tmask, ls0, j, TL), s1 = __shfl_sync(tmask, ls1, j, TL);
            const int32_t ty = __shfl_sync(tmask, lty, j, TL);
            // closed-form list offset (4-byte entries, task order)
            const int64_t x = (ib + i0) + (ob + o0) + (eb + s0);
            const int32_t nin = i1 - i0, nout = o1 - o0, nsucc = s1 - s0;
            int32_t* inh = adj + x;
            int32_t* outl = inh + nin;
            int32_t* succl = outl + nout;
            const int32_t* in = b.in + ib + i0;
            const int32_t* out = b.out + ob + o0;
            const int32_t* succ = b.succ + eb + s0;
            {  // first TL entries of every list: all loads issued before any store
                const int32_t hd = tl < nin ? __ldg(&in[tl]) : 0;
                const int32_t ov = tl < nout ? __ldg(&out[tl]) : 0;
                const int32_t sv = tl < nsucc ? succ[tl] : 0;
                const uint8_t cl = tl < nin ? __ldg(&hcls[hb + hd]) : 0;
                if (tl < nin) inh[tl] = word(hd, cl);
                if (tl < nout) outl[tl] = ov;
                if (tl < nsucc) succl[tl] = sv;
            }
            for (int32_t k = tl + TL; k < nin; k += TL) {
                const int32_t hd = __ldg(&in[k]);
                inh[k] = word(hd, __ldg(&hcls[hb + hd]));
            }
            for (int32_t k = tl + TL; k < nout; k += TL) outl[k] = __ldg(&out[k]);
            for (int32_t k = tl + TL; k < nsucc; k += TL) succl[k] = succ[k];
            // record word 3: successors | type << 24 | multi-edges << 30 (the
            // sorted list holds a repeated successor)
            bool dup = false;
            for (int32_t k = tl + 1; k < nsucc; k += TL) dup = dup || succ[k] == succ[k - 1];
            dup = __any_sync(tmask, dup);
            if (tl == 0)
                reinterpret_cast<int4*>(hdr + t)[0] =
                    make_int4(static_cast<int32_t>(static_cast<uint32_t>(x)), nin, nout,
                              static_cast<int32_t>((dup ? 1u << 30 : 0u) | (static_cast<uint32_t>(ty) << 24) |
                                                   (static_cast<uint32_t>(nsucc) & 0xffffffu)));
        }
    }
}

template __global__ void k_sim_pack<8>(DevBatch, const uint8_t*, SimTaskHdr*, int32_t*);

// Uploaded batches: the successor CSR and the packed simulation graph of a
// graph in one pass of its CTA (ingest.cuh, then the k_sim_pack layout) --
// the graph's offsets and freshly sorted successor lists are still in L1/L2
// when they are packed, and one launch replaces two.  Teams of 8 lanes copy
// a task's three lists; the record follows once the team knows whether the
// successor list repeats an entry.  hcls (k_bytes_class) must be complete.
__global__ void __launch_bounds__(256) k_ingest_pack(DevBatch b, int32_t* cursor_scratch, int32_t smem_ints,
                                                     const uint8_t* hcls, SimTaskHdr* hdr, int32_t* adj) {
    __shared__ int32_t warp_tot[32];
    extern __shared__ int32_t s_ctr[];
    constexpr int TL = 8;
    const int tl = threadIdx.x & (TL - 1), team = threadIdx.x / TL, nteams = blockDim.x / TL;
    const unsigned tmask = ((1u << TL) - 1u) << ((threadIdx.x & 31) & ~(TL - 1));
    for (int64_t g = blockIdx.x; g < b.G; g += gridDim.x) {
        ingest_graph(b, g, cursor_scratch, smem_ints, s_ctr, warp_tot);
        const int64_t t0 = b.task_base[g];
        const int32_t n = static_cast<int32_t>(b.task_base[g + 1] - t0);
        const int64_t ib = b.in_base[g], ob = b.out_base[g], eb = b.edge_base[g], hb = b.handle_base[g];
        const int32_t* ioff = b.in_off + t0 + g;
        const int32_t* ooff = b.out_off + t0 + g;
        const int32_t* soff = b.succ_off + t0 + g;  // written by this CTA: plain loads
        const int32_t* in = b.in + ib;
        const int32_t* out = b.out + ob;
        const int32_t* succ = b.succ + eb;
        // a team's next TL tasks: their offsets in one load per lane, handed
        // out by shuffles; each task's first TL list entries loaded before
        // any store
        for (int32_t base = team; base < n; base += TL * nteams) {
            const int32_t vt = base + tl * nteams;
            int32_t li0 = 0, li1 = 0, lo0 = 0, lo1 = 0, ls0 = 0, ls1 = 0, lty = 0;
            if (vt < n) {
                li0 = __ldg(&ioff[vt]); li1 = __ldg(&ioff[vt + 1]);
                lo0 = __ldg(&ooff[vt]); lo1 = __ldg(&ooff[vt + 1]);
                ls0 = soff[vt]; ls1 = soff[vt + 1];
                lty = __ldg(&b.type[t0 + vt]);
            }
            for (int j = 0; j < TL; ++j) {
                const int32_t v = base + j * nteams;
                if (v >= n) break;  // uniform in the team
                const int32_t i0 = __shfl_sync(tmask, li0, j, TL), i1 = __shfl_sync(tmask, li1, j, TL);
                const int32_t o0 = __shfl_sync(tmask, lo0, j, TL), o1 = __shfl_sync(tmask, lo1, j, TL);
                const int32_t s0 = __shfl_sync(tmask, ls0, j, TL), s1 = __shfl_sync(tmask, ls1, j, TL);
                const int32_t ty = __shfl_sync(tmask, lty, j, TL);
                const int64_t x = (ib + i0) + (ob + o0) + (eb + s0);
                const int32_t nin = i1 - i0, nout = o1 - o0, nsucc = s1 - s0;
                int32_t* inh = adj + x;
                int32_t* outl = inh + nin;
                int32_t* succl = outl + nout;
                bool dup = false;
                {
                    const int32_t h = tl < nin ? __ldg(&in[i0 + tl]) : 0;
                    const int32_t ov = tl < nout ? __ldg(&out[o0 + tl]) : 0;
                    const int32_t sv = tl < nsucc ? succ[s0 + tl] : 0;
                    const int32_t sp = __shfl_up_sync(tmask, sv, 1, TL);  // the previous entry (tl > 0)
                    const uint8_t cl = tl < nin ? __ldg(&hcls[hb + h]) : 0;
                    if (tl < nin)
                        inh[tl] = static_cast<int32_t>(static_cast<uint32_t>(h) | (static_cast<uint32_t>(cl) << kHandleBits));
                    if (tl < nout) outl[tl] = ov;
                    if (tl < nsucc) succl[tl] = sv;
                    dup = tl > 0 && tl < nsucc && sp == sv;
                }
                for (int32_t k = tl + TL; k < nin; k += TL) {
                    const int32_t h = __ldg(&in[i0 + k]);
                    inh[k] = static_cast<int32_t>(static_cast<uint32_t>(h) |
                                                  (static_cast<uint32_t>(__ldg(&hcls[hb + h])) << kHandleBits));
                }
                for (int32_t k = tl + TL; k < nout; k += TL) outl[k] = __ldg(&out[o0 + k]);
                for (int32_t k = tl + TL; k < nsucc; k += TL) {
                    const int32_t sv = succ[s0 + k];
                    succl[k] = sv;
                    dup = dup || succ[s0 + k - 1] == sv;
                }
                // record words 0-3: list offset, inputs, outputs, successors |
                // type << 24 | multi-edges << 30 (as k_sim_pack)
                dup = __any_sync(tmask, dup);
                if (tl == 0)
                    reinterpret_cast<int4*>(hdr + t0 + v)[0] =
                        make_int4(static_cast<int32_t>(static_cast<uint32_t>(x)), nin, nout,
                                  static_cast<int32_t>((dup ? 1u << 30 : 0u) | (static_cast<uint32_t>(ty) << 24) |
                                                       (static_cast<uint32_t>(nsucc) & 0xffffffu)));
            }
        }
        __syncthreads();  // s_ctr / cursors are reused by the next graph
    }
}

// Every handle's size class in the batch's (final) dictionary, once per
// handle -- the pack then reads one byte per input instead of the 8-byte
// size and a dictionary search per input entry.
__global__ void __launch_bounds__(256) k_bytes_class(DevBatch b, const int64_t* dict, uint8_t* hcls) {
    __shared__ int64_t s_dict[kByteClasses];
    if (threadIdx.x < kByteClasses) s_dict[threadIdx.x] = dict[threadIdx.x];
    __syncthreads();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < b.H; i += stride) {
        const int64_t by = __ldg(&b.handle_bytes[i]);
        uint8_t c = kEscapeClass;
#pragma unroll
        for (int k = kEscapeClass - 1; k >= 0; --k)
            if (s_dict[k] == by) c = static_cast<uint8_t>(k);
        hcls[i] = c;
    }
}

// A value into a dictionary of kEscapeClass slots (first come, first
// numbered); false when it is full of other values.
__device__ __forceinline__ bool dict_insert(unsigned long long* d, unsigned long long v) {
    for (int c = 0; c < kEscapeClass; ++c) {
        const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(&d[c]);
        if (cur == v) return true;
        if (cur == static_cast<unsigned long long>(kDictEmpty)) {
            const unsigned long long old = atomicCAS(&d[c], static_cast<unsigned long long>(kDictEmpty), v);
            if (old == static_cast<unsigned long long>(kDictEmpty) || old == v) return true;
        }
    }
    return false;
}

// Each CTA collects its handles' distinct sizes in shared memory (a few
// shared-memory compares per handle), then merges them into the batch's
// dictionary -- a handful of global CAS per CTA instead of per warp.
__global__ void __launch_bounds__(256) k_bytes_dict(DevBatch b, unsigned long long* dict) {
    __shared__ unsigned long long sd[kEscapeClass];
    if (threadIdx.x < kEscapeClass) sd[threadIdx.x] = static_cast<unsigned long long>(kDictEmpty);
    __syncthreads();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < b.H; i += stride) {
        const unsigned long long v = static_cast<unsigned long long>(__ldg(&b.handle_bytes[i]));
        // this CTA's dictionary full of other values: straight to the
        // batch's (where it may still get a class)
        if (!dict_insert(sd, v)) dict_insert(dict, v);
    }
    __syncthreads();
    if (threadIdx.x < kEscapeClass && sd[threadIdx.x] != static_cast<unsigned long long>(kDictEmpty))
        dict_insert(dict, sd[threadIdx.x]);
}

__global__ void k_xfer_table(const DevPlatform* pf, int32_t n_platforms, const int64_t* dict, int32_t mn,
                             double* xtab) {
    const int64_t total = static_cast<int64_t>(n_platforms) * kByteClasses * mn * mn;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t to = static_cast<int32_t>(i % mn), from = static_cast<int32_t>((i / mn) % mn);
        const int32_t cls = static_cast<int32_t>((i / (mn * mn)) % kByteClasses);
        const DevPlatform& P = pf[i / (static_cast<int64_t>(kByteClasses) * mn * mn)];
        double t = 0.0;
        const int64_t by = dict ? dict[cls] : kDictEmpty;  // no dictionary: a batch without tasks
        if (from != to && from < P.n_nodes && to < P.n_nodes && by != kDictEmpty)
            t = tbsim_rules::transfer_ms(P.latency_ms, by, P.bw[from * kMaxNodes + to]);
        xtab[i] = t;
    }
}

// Pop keys of one simulation call (record words 4-7): ability, efficiency
// and static priority; ab = -1 flags keys beyond the queue's int32 keys or a
// task with 2^24 successor entries.
__global__ void __launch_bounds__(256) k_sim_keys(DevBatch b, const int64_t* ability, const int64_t* efficiency,
                                                  const int64_t* prio, int32_t policy, SimTaskHdr* hdr) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < b.T; t += stride) {
        int32_t ka = 0, ke = 0;
        int64_t kp = prio && policy >= TBSIM_POLICY_DMDAP ? prio[t] : 0;
        // the 24-bit field holds nsucc mod 2^24; the full count is checked here
        const int64_t g = graph_of(b, t);
        const int64_t v = t - __ldg(&b.task_base[g]);
        const int32_t* soff = b.succ_off + __ldg(&b.task_base[g]) + g;
        bool bad = soff[v + 1] - soff[v] >= (1 << 24);
        if (policy == TBSIM_POLICY_INSPIRIT) {
            const int64_t a64 = ability ? ability[t] : 0, e64 = efficiency ? efficiency[t] : 0;
            ka = static_cast<int32_t>(a64);
            ke = static_cast<int32_t>(e64);
            bad = bad || ka != a64 || ke != e64 || ka < 0;
        }
        if (bad) ka = -1;
        reinterpret_cast<int4*>(hdr + t)[1] = make_int4(ka, ke, static_cast<int32_t>(static_cast<uint64_t>(kp)),
                                                         static_cast<int32_t>(static_cast<uint64_t>(kp) >> 32));
    }
}

__global__ void __launch_bounds__(256) k_sim_scatter(DevBatch b, const SimLog* log, const int32_t* n_disp,
                                                     int32_t* worker, double* start_ms, double* end_ms) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < b.T; t += stride) {
        const int64_t g = graph_of(b, t);
        const int64_t t0 = __ldg(&b.task_base[g]);
        if (t - t0 >= __ldg(&n_disp[g])) continue;  // -1: written by the simulator
        const SimLog e = log[t];
        worker[t0 + e.task] = e.worker;
        start_ms[t0 + e.task] = e.start;
        end_ms[t0 + e.task] = e.end;
    }
}

// Graphs whose simulation overflowed a shared-memory queue, compacted into
// the rerun list (count in *n): the rerun launch reads its item count from
// the device, so no host round trip decides whether it has work.
__global__ void __launch_bounds__(1024) k_sim_collect_reruns(int64_t G, const int32_t* status, int32_t* list,
                                                            int64_t* n) {
    __shared__ int32_t warp_tot[32];
    int32_t carry = 0;
    for (int64_t base = 0; base < G; base += blockDim.x) {
        const int64_t g = base + threadIdx.x;
        const int32_t x = g < G && status[g] == GS_QUEUE_OVERFLOW ? 1 : 0;
        int32_t tot;
        const int32_t inc = block_inclusive_scan(x, warp_tot, &tot);
        if (x) list[carry + inc - 1] = static_cast<int32_t>(g);
        carry += tot;
    }
    if (threadIdx.x == 0) *n = carry;
}

#define TBSIM_SIM_KERNEL(NAME, WPL, COMPACT, POL, MANYIN, THREADS, MINB)                             \
    __global__ void __launch_bounds__(THREADS, MINB) NAME(const __grid_constant__ SimParams p) {        \
        if (p.use_smem) simulate_impl<WPL, COMPACT, POL, MANYIN, true>(p);                             \
        else simulate_impl<WPL, COMPACT, POL, MANYIN, false>(p);                                       \
    }
// <= 32 workers, compact: 4-warp CTAs, 7 per SM (<= 72 registers)
TBSIM_SIM_KERNEL(k_simulate_w1c, 1, true, -1, false, 128, 7)
// the same for inspirit only (the policy fixed at compile time)
TBSIM_SIM_KERNEL(k_simulate_w1c_ins, 1, true, TBSIM_POLICY_INSPIRIT, false, 128, 7)
// batches whose tasks read many inputs (C5: 18 per task): the multi-round
// transfer sum that skips resident inputs
TBSIM_SIM_KERNEL(k_simulate_w1c_mi, 1, true, -1, true, 128, 7)
TBSIM_SIM_KERNEL(k_simulate_w2c, 2, true, -1, false, 256, 2)
TBSIM_SIM_KERNEL(k_simulate_w2c_mi, 2, true, -1, true, 256, 2)
// inspirit-only, trace-free twins of the many-input and two-worker-per-lane
// kernels (C5's mixes, C3's 36 workers)
TBSIM_SIM_KERNEL(k_simulate_w1c_mi_ins, 1, true, TBSIM_POLICY_INSPIRIT, true, 128, 7)
TBSIM_SIM_KERNEL(k_simulate_w2c_ins, 2, true, TBSIM_POLICY_INSPIRIT, false, 256, 2)
TBSIM_SIM_KERNEL(k_simulate_w2c_mi_ins, 2, true, TBSIM_POLICY_INSPIRIT, true, 256, 2)
TBSIM_SIM_KERNEL(k_simulate_w1, 1, false, -1, false, 256, 2)
TBSIM_SIM_KERNEL(k_simulate_w2, 2, false, -1, false, 256, 2)
#undef TBSIM_SIM_KERNEL

}  // namespace tbsim_dev
