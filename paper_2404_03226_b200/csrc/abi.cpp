// abi.cpp -- implementation of include/tbsim_b200.h.
//
// Host orchestration only: argument checks, CSR ingestion into HBM, kernel
// launches, result download and the mapping of per-graph device status codes
// onto the reference's exception types and texts.  All compute runs in the
// CUDA kernels (attributes.cu, simulate.cu); there is no host fallback.
#include "tbsim_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "attributes.cuh"
#include "common.cuh"
#include "generate.cuh"
#include "hostbatch.hpp"
#include "rules.cuh"
#include "simulate.cuh"

using namespace tbsim_dev;

namespace {

thread_local std::string g_err;

struct Error {
    tbsim_status code;
    std::string msg;
};

[[noreturn]] void raise(tbsim_status code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(TBSIM_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Makes the context's device current for one ABI call and restores the
// caller's device afterwards (a host thread driving several GPUs, or a
// framework with its own current device, keeps it across our calls).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess) cur = -1;
        if (cur != dev) {
            cuda_check(cudaSetDevice(dev), "cudaSetDevice");
            prev = cur;
        }
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;
};

template <typename F>
tbsim_status guarded(F&& f) {
    try {
        f();
        return TBSIM_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return TBSIM_E_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return TBSIM_E_OUT_OF_RANGE;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return TBSIM_E_LOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TBSIM_E_RUNTIME;
    }
}

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need) {
        need = std::max<size_t>(need, 16);
        if (need > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            bytes = 0;
            cuda_check(cudaMalloc(&p, need), "cudaMalloc");
            bytes = need;
        }
        return p;
    }
    template <typename T>
    T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T))); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

}  // namespace

struct tbsim_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    int n_sms = 0;
    size_t smem_optin = 0;
    int64_t launches = 0;
    bool timing = false;
    std::map<std::string, double> last_ms;
    std::map<std::string, std::pair<cudaEvent_t, cudaEvent_t>> events;
    std::set<std::string> begun;  // timed names begun since the last collect_timing
    std::map<std::string, DevBuf> bufs;
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    cudaStream_t upload = nullptr;  // batch uploads (null: the compute stream)
    struct PoolEntry {
        void* p;
        size_t bytes;
        cudaEvent_t freed;  // compute-stream point after the last reader
    };
    std::vector<PoolEntry> batch_pool;  // freed batch allocations for reuse
    int64_t large_threshold = 65536;  // single graphs at least this large take the closure path
    int32_t sweep_tile = 0;           // forced sources per sweep tile (0: widest that fits)
    int32_t sim_warps_per_sm = 0, sim_state_smem = 0, sim_qcap = 0;  // last k_simulate launch shape
    // per-device launch facts (function attributes are per device, so they
    // live with the context, not in process-wide statics)
    bool sweep_attr = false, sweep32_attr = false;
    int structure_large_per_sm = 0, finalize_large_per_sm = 0;
    // Asynchronous results (tbsim_ctx_set_async_results): host-bound outputs
    // of tbsim_schedule are staged in one of two device buffer sets and copied
    // on the download stream, so a call's D2H overlaps the next call's
    // kernels; a set is rewritten only after its previous copies finished.
    bool async_results = false;
    cudaStream_t download = nullptr;
    cudaEvent_t set_free[2] = {nullptr, nullptr};
    bool set_pending[2] = {false, false};
    int parity = 0;
    // sharded large-graph attributes: what tbsim_attributes_shard_partial
    // left for tbsim_attributes_shard_finish (same batch, back to back)
    struct Shard {
        const tbsim_batch* b = nullptr;
        int32_t rank = -1, world = 0;
        int32_t pos_lo = 0, pos_hi = 0;
        int64_t n_words = 0;
        uint64_t gen = 0;  // scratch generation of the partial call
        AttrScratch s{};
    } shard;
    // bumped by every attribute-scratch allocation: a shard finish must
    // directly follow its partial call (no other attribute pass in between
    // reusing or regrowing the scratch it reads)
    uint64_t scratch_gen = 0;
    // uploads on the upload stream leave k_ingest / k_sim_pack to the
    // compute stream (TBSIM_INGEST_ON_UPLOAD=1: run them on the upload stream)
    bool defer_ingest = true;
    // pinned host staging (grow-only, by name)
    struct PinnedBuf {
        void* p = nullptr;
        size_t bytes = 0;
    };
    std::map<std::string, PinnedBuf> pbufs;
    template <typename T>
    T* pin(const std::string& name, size_t count) {
        PinnedBuf& b = pbufs[name];
        const size_t need = std::max<size_t>(count * sizeof(T), 16);
        if (need > b.bytes) {
            if (b.p) cudaFreeHost(b.p);
            b.p = nullptr;
            b.bytes = 0;
            cuda_check(cudaMallocHost(&b.p, need), "cudaMallocHost");
            b.bytes = need;
        }
        return static_cast<T*>(b.p);
    }
    // Deferred error checks of asynchronous schedule calls (one per result
    // set): the statuses / attribute infos are copied to pinned staging and
    // decoded at tbsim_ctx_synchronize, or when the set is reused -- no
    // host round trip inside the call.
    struct Pending {
        bool active = false;
        cudaEvent_t done = nullptr;
        int64_t G = 0;
        const GraphInfo* info = nullptr;  // compute_attributes infos (checked first)
        const int32_t* status = nullptr;
        const int32_t* aux = nullptr;
        const int64_t* completed = nullptr;
        std::vector<int64_t> task_base, task_id;
        std::vector<std::string> type_names;
        const int32_t* worker_out = nullptr;  // caller's worker array (stuck-task listing)
        bool worker_on_device = false;
        cudaEvent_t copies_done = nullptr;    // the host arrays' D2H (download stream)
    } pend[2];
    unsigned long long* relax_ctr = nullptr;  // device counter of the last timed sweep
    int64_t last_relax[2] = {0, 0};  // FP64-window, FP32-window relaxations

    DevBuf& buf(const std::string& name) { return bufs[name]; }
    void* batch_alloc(size_t bytes, size_t* got) {
        size_t best = batch_pool.size();
        for (size_t i = 0; i < batch_pool.size(); ++i)
            if (batch_pool[i].bytes >= bytes && (best == batch_pool.size() || batch_pool[i].bytes < batch_pool[best].bytes))
                best = i;
        if (best < batch_pool.size()) {
            const PoolEntry e = batch_pool[best];
            batch_pool.erase(batch_pool.begin() + static_cast<std::ptrdiff_t>(best));
            // the writer (this stream) waits for the kernels that read the
            // freed batch on the compute stream
            if (e.freed) {
                cuda_check(cudaStreamWaitEvent(stream, e.freed, 0), "cudaStreamWaitEvent(pool)");
                cudaEventDestroy(e.freed);
            }
            *got = e.bytes;
            return e.p;
        }
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(batch)");
        *got = bytes;
        return p;
    }
    void* host_stage(size_t bytes) {
        if (bytes > pinned_bytes) {
            if (pinned) cudaFreeHost(pinned);
            pinned = nullptr;
            cuda_check(cudaHostAlloc(&pinned, bytes, cudaHostAllocDefault), "cudaHostAlloc");
            pinned_bytes = bytes;
        }
        return pinned;
    }
    void begin(const char* k) {
        ++launches;
        if (!timing) return;
        auto& ev = events[k];
        if (!ev.first) {
            cudaEventCreate(&ev.first);
            cudaEventCreate(&ev.second);
        }
        // several launches under one name in one call: first begin to last end
        if (begun.insert(k).second) cudaEventRecord(ev.first, stream);
    }
    void end(const char* k) {
        cuda_check(cudaGetLastError(), k);
        if (!timing) return;
        cudaEventRecord(events[k].second, stream);
    }
    void collect_timing() {
        begun.clear();
        if (!timing) return;
        for (auto& [k, ev] : events) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ev.first, ev.second) == cudaSuccess) last_ms[k] = ms;
        }
        if (relax_ctr) {
            unsigned long long r[2] = {0, 0};
            if (cudaMemcpy(r, relax_ctr, 16, cudaMemcpyDeviceToHost) == cudaSuccess) {
                last_relax[0] = static_cast<int64_t>(r[0]);
                last_relax[1] = static_cast<int64_t>(r[1]);
            }
            relax_ctr = nullptr;
        }
    }
    void sync() { cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }
};

struct tbsim_batch {
    DevBatch d{};
    void* mem = nullptr;
    size_t mem_bytes = 0;
    void* mem2 = nullptr;  // edge-sized sections of a device-generated batch
    size_t mem2_bytes = 0;
    int64_t h2d_bytes = 0;
    std::vector<int64_t> task_base;    // host copy
    std::vector<int64_t> task_id;      // host copy (messages)
    std::vector<std::string> type_names;
    int32_t max_workers_seen = 0;
    cudaEvent_t ready = nullptr;  // recorded on the upload stream when it is not the compute stream
    // packed simulation graph (k_sim_pack): built once per batch
    void* mem3 = nullptr;
    size_t mem3_bytes = 0;
    tbsim_dev::SimTaskHdr* hdr = nullptr;
    bool needs_ingest = false;  // copied on the upload stream, derived sections not built yet
    int64_t* dict = nullptr;  // [kByteClasses] handle-size dictionary (k_bytes_dict)
    int32_t* adj = nullptr;
};

namespace {

// k_ingest with its counters in shared memory when the largest graph fits
void launch_ingest(tbsim_ctx* ctx, const DevBatch& d, int grid, int32_t* cursor) {
    const int64_t want = static_cast<int64_t>(d.max_n) + 1;
    const int32_t ints = want * 4 <= 48 * 1024 ? static_cast<int32_t>(want) : 0;
    k_ingest<<<grid, 256, static_cast<size_t>(ints) * 4, ctx->stream>>>(d, cursor, ints);
}

// The simulator's packed view of a batch (one 32-byte record per task +
// contiguous lists), built once on the stream the call runs on -- at upload,
// after k_ingest, or on a generated batch's first simulation.
// Allocation, size dictionary and per-handle size classes of the packed
// view; returns the class table the pack reads.
uint8_t* prepare_packed(tbsim_ctx* ctx, tbsim_batch* b) {
    const DevBatch& d = b->d;
    const int64_t adj_bytes = sim_adj_bytes(d.T, d.I, d.O, d.E);
    if (adj_bytes >= (int64_t(1) << 34)) raise(TBSIM_E_INVALID_ARGUMENT, "batch too large for the packed simulation graph");
    if (d.max_h > kHandleMask) raise(TBSIM_E_INVALID_ARGUMENT, "graph exceeds 2^28 handles for the simulator");
    const size_t hdr_bytes = static_cast<size_t>(d.T) * sizeof(SimTaskHdr);
    const size_t dict_at = (hdr_bytes + 255) & ~size_t(255), adj_at = dict_at + 256;
    const size_t cls_at = (adj_at + static_cast<size_t>(adj_bytes) + 255) & ~size_t(255);
    b->mem3 = ctx->batch_alloc(cls_at + static_cast<size_t>(d.H) + 256, &b->mem3_bytes);
    uint8_t* hcls = static_cast<uint8_t*>(b->mem3) + cls_at;
    b->hdr = static_cast<SimTaskHdr*>(b->mem3);
    b->dict = reinterpret_cast<int64_t*>(static_cast<char*>(b->mem3) + dict_at);
    b->adj = reinterpret_cast<int32_t*>(static_cast<char*>(b->mem3) + adj_at);
    static const int64_t empty[kByteClasses] = {kDictEmpty, kDictEmpty, kDictEmpty, kDictEmpty, kDictEmpty, kDictEmpty,
                                                kDictEmpty, kDictEmpty, kDictEmpty, kDictEmpty, kDictEmpty, kDictEmpty,
                                                kDictEmpty, kDictEmpty, kDictEmpty, kDictEmpty};
    cuda_check(cudaMemcpyAsync(b->dict, empty, sizeof empty, cudaMemcpyHostToDevice, ctx->stream), "H2D dict");
    if (d.H > 0) {
        const int grid_h = static_cast<int>(std::min<int64_t>((d.H + 255) / 256, 4LL * ctx->n_sms));
        ctx->begin("k_bytes_dict");
        k_bytes_dict<<<grid_h, 256, 0, ctx->stream>>>(d, reinterpret_cast<unsigned long long*>(b->dict));
        k_bytes_class<<<grid_h, 256, 0, ctx->stream>>>(d, b->dict, hcls);
        ctx->end("k_bytes_dict");
    }
    return hcls;
}

void ensure_packed(tbsim_ctx* ctx, tbsim_batch* b) {
    const DevBatch& d = b->d;
    if (b->hdr || d.T == 0) return;
    uint8_t* hcls = prepare_packed(ctx, b);
    const int grid = static_cast<int>(std::min<int64_t>((d.T + 255) / 256, 16LL * ctx->n_sms));
    // 8 lanes per task (measured 1/2/4/8: C2 0.90/0.68/0.58/0.55 ms,
    // 2048 C5 DAGs 6.5/4.7/3.2/2.5 ms)
    ctx->begin("k_sim_pack");
    k_sim_pack<8><<<grid, 256, 0, ctx->stream>>>(d, hcls, b->hdr, b->adj);
    ctx->end("k_sim_pack");
}

DevCosts to_dev_costs(const tbsim_costs& c, int32_t n_types_batch) {
    if (c.n_types > kMaxTypes || n_types_batch > kMaxTypes)
        raise(TBSIM_E_INVALID_ARGUMENT, "more than " + std::to_string(kMaxTypes) + " task types");
    DevCosts d{};
    d.n_types = std::max(c.n_types, 0);
    for (int i = 0; i < c.n_types; ++i) {
        d.cpu[i] = c.cpu_ms && c.cpu_ms[i] > 0.0 ? c.cpu_ms[i] : 0.0;
        d.gpu[i] = c.gpu_ms && c.gpu_ms[i] > 0.0 ? c.gpu_ms[i] : 0.0;
    }
    return d;
}

DevPlatform to_dev_platform(const tbsim_platform_desc& p, int32_t n_types_batch) {
    if (p.n_workers < 1) raise(TBSIM_E_RUNTIME, "platform has no workers");
    if (p.n_workers > kMaxWorkers)
        raise(TBSIM_E_INVALID_ARGUMENT, "device simulator supports at most " + std::to_string(kMaxWorkers) + " workers");
    if (p.n_nodes < 1 || p.n_nodes > kMaxNodes)
        raise(TBSIM_E_INVALID_ARGUMENT, "device simulator supports 1.." + std::to_string(kMaxNodes) + " memory nodes");
    DevPlatform d{};
    d.n_workers = p.n_workers;
    d.n_nodes = p.n_nodes;
    d.latency_ms = p.latency_ms;
    for (int w = 0; w < p.n_workers; ++w) {
        d.kind[w] = p.kind[w] ? 1 : 0;
        d.node[w] = p.memory_node[w];
        if (d.node[w] < 0 || d.node[w] >= p.n_nodes)
            raise(TBSIM_E_RUNTIME, "worker " + std::to_string(w) + " references unknown memory node");
    }
    for (int a = 0; a < p.n_nodes; ++a)
        for (int b = 0; b < p.n_nodes; ++b) d.bw[a * kMaxNodes + b] = p.bandwidth[a * p.n_nodes + b];
    d.costs = to_dev_costs(p.costs, n_types_batch);
    return d;
}

void check_pending(tbsim_ctx* ctx, int set);  // deferred checks of asynchronous calls (below)

// Routes a batch upload onto ctx->upload for its duration.
struct UploadStream {
    tbsim_ctx* ctx;
    cudaStream_t saved;
    explicit UploadStream(tbsim_ctx* c) : ctx(c), saved(c->stream) {
        if (c->upload) c->stream = c->upload;
    }
    ~UploadStream() { ctx->stream = saved; }
    bool active() const { return ctx->stream != saved; }
};

// Derived sections of an uploaded or generated batch: the successor CSR and the
// simulator's packed view.  Batches of many graphs build both in one pass
// per graph (k_ingest_pack); a few large graphs (C1, C3, C4) keep the
// two-kernel form, whose pack spreads every graph over the whole GPU
// (TBSIM_SPLIT_INGEST forces it).
void ingest_uploaded(tbsim_ctx* ctx, tbsim_batch* m) {
    const DevBatch& d = m->d;
    if (d.G == 0) return;
    int32_t* cursor = ctx->buf("ingest_cursor").as<int32_t>(d.T + d.G);
    const int grid = static_cast<int>(std::min<int64_t>(d.G, 8LL * ctx->n_sms));
    static const bool split = std::getenv("TBSIM_SPLIT_INGEST") != nullptr;
    if (!m->hdr && d.T > 0 && !split && d.G >= 4LL * ctx->n_sms) {
        uint8_t* hcls = prepare_packed(ctx, m);
        const int64_t want = static_cast<int64_t>(d.max_n) + 1;
        const int32_t ints = want * 4 <= 48 * 1024 ? static_cast<int32_t>(want) : 0;
        ctx->begin("k_ingest_pack");
        // a CTA per graph up to 16 per SM (C2: 8/SM 0.63 ms, 16/SM 0.53 ms)
        const int gridp = static_cast<int>(std::min<int64_t>(d.G, 16LL * ctx->n_sms));
        k_ingest_pack<<<gridp, 256, static_cast<size_t>(ints) * 4, ctx->stream>>>(d, cursor, ints, hcls, m->hdr, m->adj);
        ctx->end("k_ingest_pack");
        return;
    }
    ctx->begin("k_ingest");
    launch_ingest(ctx, d, grid, cursor);
    ctx->end("k_ingest");
    ensure_packed(ctx, m);
}

// Compute on a batch uploaded on another stream waits for its copies, then
// (first use) builds its derived sections -- successor CSR (k_ingest) and
// the simulator's packed view (k_bytes_dict, k_sim_pack) -- on the compute
// stream.  Measured on C2: overlapping those kernels with the previous
// step's attribute/simulation kernels cost that step 1.56 ms (they take
// SMs the full-GPU kernels wait for); in order they cost ~0.6 ms.
void wait_batch(tbsim_ctx* ctx, const tbsim_batch* b) {
    if (!b) return;
    if (b->ready) cuda_check(cudaStreamWaitEvent(ctx->stream, b->ready, 0), "cudaStreamWaitEvent(batch)");
    if (b->needs_ingest) {
        auto* m = const_cast<tbsim_batch*>(b);
        m->needs_ingest = false;
        ingest_uploaded(ctx, m);
    }
}

}  // namespace

extern "C" {

const char* tbsim_last_error(void) { return g_err.c_str(); }
int tbsim_abi_version(void) { return TBSIM_ABI_VERSION; }

tbsim_status tbsim_ctx_create(int device, tbsim_ctx** out) {
    return guarded([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            raise(TBSIM_E_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
        }
        if (device < 0 || device >= n) raise(TBSIM_E_INVALID_ARGUMENT, "bad device index");
        auto c = std::make_unique<tbsim_ctx>();
        c->device = device;
        DeviceScope dev_scope(device);
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major < 10)
            raise(TBSIM_E_CUDA, std::string("device ") + prop.name + " is not sm_100 (built for sm_100a)");
        c->n_sms = prop.multiProcessorCount;
        if (const char* e = std::getenv("TBSIM_INGEST_ON_UPLOAD")) c->defer_ingest = std::string(e) != "1";
        c->smem_optin = prop.sharedMemPerBlockOptin;
        cuda_check(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "cudaStreamCreate");
        c->stream = c->own;
        *out = c.release();
    });
}

tbsim_status tbsim_ctx_destroy(tbsim_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        DeviceScope dev_scope(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        for (auto& [k, b] : ctx->bufs) b.release();
        if (ctx->upload) cudaStreamSynchronize(ctx->upload);
        for (auto& pb : ctx->batch_pool) {
            cudaFree(pb.p);
            if (pb.freed) cudaEventDestroy(pb.freed);
        }
        for (auto& [k, ev] : ctx->events) {
            cudaEventDestroy(ev.first);
            cudaEventDestroy(ev.second);
        }
        if (ctx->download) {
            cudaStreamSynchronize(ctx->download);
            cudaStreamDestroy(ctx->download);
        }
        for (auto& e : ctx->set_free)
            if (e) cudaEventDestroy(e);
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        for (auto& [k, b] : ctx->pbufs)
            if (b.p) cudaFreeHost(b.p);
        for (auto& pd : ctx->pend)
            if (pd.done) cudaEventDestroy(pd.done);
        if (ctx->own) cudaStreamDestroy(ctx->own);
        delete ctx;
    });
}

tbsim_status tbsim_ctx_set_stream(tbsim_ctx* ctx, void* s) {
    return guarded([&] { ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own; });
}

tbsim_status tbsim_ctx_set_upload_stream(tbsim_ctx* ctx, void* s) {
    return guarded([&] { ctx->upload = static_cast<cudaStream_t>(s); });
}

tbsim_status tbsim_ctx_synchronize(tbsim_ctx* ctx) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        ctx->sync();
        if (ctx->download) cuda_check(cudaStreamSynchronize(ctx->download), "cudaStreamSynchronize(download)");
        // deferred checks of asynchronous calls, oldest first; both are
        // cleared, the first failure is raised
        const int first = ctx->parity;  // the set the next call would use = the older one
        std::exception_ptr err;
        for (int k = 0; k < 2; ++k) {
            try {
                check_pending(ctx, (first + k) & 1);
            } catch (...) {
                if (!err) err = std::current_exception();
            }
        }
        if (err) std::rethrow_exception(err);
    });
}

tbsim_status tbsim_ctx_set_async_results(tbsim_ctx* ctx, int enable) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        if (enable && !ctx->download) {
            cuda_check(cudaStreamCreateWithFlags(&ctx->download, cudaStreamNonBlocking), "cudaStreamCreate");
            for (auto& e : ctx->set_free)
                cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        }
        if (!enable && ctx->download) cuda_check(cudaStreamSynchronize(ctx->download), "cudaStreamSynchronize");
        ctx->async_results = enable != 0;
    });
}

int64_t tbsim_ctx_launch_count(const tbsim_ctx* ctx) { return ctx ? ctx->launches : 0; }

tbsim_status tbsim_ctx_set_large_graph_threshold(tbsim_ctx* ctx, int64_t n_tasks) {
    return guarded([&] { ctx->large_threshold = n_tasks; });
}

tbsim_status tbsim_ctx_set_sweep_tile(tbsim_ctx* ctx, int32_t sources) {
    return guarded([&] {
        if (sources != 0 && sources != 8 && sources != 16 && sources != 32 && sources != 64 && sources != 128 &&
            sources != 256)
            raise(TBSIM_E_INVALID_ARGUMENT, "sweep tile must be 0, 8, 16, 32, 64, 128 or 256 sources");
        ctx->sweep_tile = sources;
    });
}

tbsim_status tbsim_ctx_set_timing(tbsim_ctx* ctx, int enable) {
    return guarded([&] { ctx->timing = enable != 0; });
}

tbsim_status tbsim_probe_sweep_peak(tbsim_ctx* ctx, int32_t repeats, double* fp64_per_s, double* fp32_per_s) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        constexpr int32_t kRows = 128, kIters = 20000, kThreads = 512;
        double* out = ctx->buf("p_out").as<double>(ctx->n_sms);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int f32 = 0; f32 < 2; ++f32) {
            const size_t smem = static_cast<size_t>(kRows) * 128 * (f32 ? 4 : 8);
            auto kern = f32 ? tbsim_dev::k_probe_relax_f32 : tbsim_dev::k_probe_relax;
            cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                       "cudaFuncSetAttribute(k_probe_relax)");
            double best = 0.0;
            for (int32_t r = 0; r < std::max(repeats, 1) + 1; ++r) {  // first launch warms up
                cudaEventRecord(e0, ctx->stream);
                ctx->begin("k_probe_relax");
                kern<<<ctx->n_sms, kThreads, smem, ctx->stream>>>(kRows - 1, kIters, out);
                ctx->end("k_probe_relax");
                cudaEventRecord(e1, ctx->stream);
                cuda_check(cudaEventSynchronize(e1), "probe");
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                const double relax = static_cast<double>(ctx->n_sms) * kThreads * kIters * 4.0 * 4.0;
                if (r > 0 && ms > 0.f) best = std::max(best, relax / (ms * 1e-3));
            }
            *(f32 ? fp32_per_s : fp64_per_s) = best;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

tbsim_status tbsim_ctx_last_sim_shape(const tbsim_ctx* ctx, int32_t* warps_per_sm, int32_t* state_in_smem,
                                      int32_t* queue_capacity) {
    return guarded([&] {
        *warps_per_sm = ctx->sim_warps_per_sm;
        *state_in_smem = ctx->sim_state_smem;
        *queue_capacity = ctx->sim_qcap;
    });
}

tbsim_status tbsim_ctx_last_sweep_relaxations(const tbsim_ctx* ctx, int64_t* fp64, int64_t* fp32) {
    return guarded([&] {
        *fp64 = ctx->last_relax[0];
        *fp32 = ctx->last_relax[1];
    });
}

tbsim_status tbsim_ctx_last_kernel_ms(const tbsim_ctx* ctx, const char* kernel, double* ms) {
    return guarded([&] {
        auto it = ctx->last_ms.find(kernel);
        *ms = it == ctx->last_ms.end() ? 0.0 : it->second;
    });
}

// ------------------------------------------------------------------ upload

tbsim_status tbsim_batch_upload(tbsim_ctx* ctx, const tbsim_batch_desc* h, tbsim_batch** out) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        // copies + ingest on the upload stream; compute calls wait on b->ready
        UploadStream us(ctx);
        const int64_t G = h->n_graphs;
        if (G < 0) raise(TBSIM_E_INVALID_ARGUMENT, "negative graph count");
        auto b = std::make_unique<tbsim_batch>();
        const int64_t T = h->task_base[G], E = h->edge_base[G], H = h->handle_base[G];
        const int64_t I = h->in_base[G], O = h->out_base[G];
        if (h->n_type_names > kMaxTypes) raise(TBSIM_E_INVALID_ARGUMENT, "more than 64 task types");
        // per-graph maxima (device scratch sizing) and cheap sanity checks
        int32_t max_n = 0, max_e = 0, max_h = 0;
        for (int64_t g = 0; g < G; ++g) {
            const int64_t n = h->task_base[g + 1] - h->task_base[g];
            const int64_t e = h->edge_base[g + 1] - h->edge_base[g];
            const int64_t nh = h->handle_base[g + 1] - h->handle_base[g];
            if (n < 0 || e < 0 || nh < 0) raise(TBSIM_E_INVALID_ARGUMENT, "batch bases must be non-decreasing");
            if (n >= (1 << 24)) raise(TBSIM_E_INVALID_ARGUMENT, "graph exceeds 2^24 tasks");
            if (e > INT32_MAX || nh > INT32_MAX) raise(TBSIM_E_INVALID_ARGUMENT, "graph exceeds 2^31 entries");
            max_n = std::max<int32_t>(max_n, static_cast<int32_t>(n));
            max_e = std::max<int32_t>(max_e, static_cast<int32_t>(e));
            max_h = std::max<int32_t>(max_h, static_cast<int32_t>(nh));
        }
        struct Sec { const void* src; size_t bytes; void** dst; };
        DevBatch& d = b->d;
        std::vector<Sec> secs = {
            {h->task_base, static_cast<size_t>(G + 1) * 8, (void**)&d.task_base}, {h->edge_base, static_cast<size_t>(G + 1) * 8, (void**)&d.edge_base},
            {h->handle_base, static_cast<size_t>(G + 1) * 8, (void**)&d.handle_base}, {h->in_base, static_cast<size_t>(G + 1) * 8, (void**)&d.in_base},
            {h->out_base, static_cast<size_t>(G + 1) * 8, (void**)&d.out_base}, {h->dep_off, static_cast<size_t>(T + G) * 4, (void**)&d.dep_off},
            {h->dep, static_cast<size_t>(E) * 4, (void**)&d.dep}, {h->in_off, static_cast<size_t>(T + G) * 4, (void**)&d.in_off},
            {h->in, static_cast<size_t>(I) * 4, (void**)&d.in}, {h->out_off, static_cast<size_t>(T + G) * 4, (void**)&d.out_off},
            {h->out, static_cast<size_t>(O) * 4, (void**)&d.out}, {h->type, static_cast<size_t>(T) * 4, (void**)&d.type},
            {h->handle_bytes, static_cast<size_t>(H) * 8, (void**)&d.handle_bytes}};
        size_t total = 0;
        for (const auto& s : secs) total += al16(s.bytes);
        const size_t derived = al16((T + G) * 4) + al16(E * 4);
        b->mem = ctx->batch_alloc(total + derived + 16, &b->mem_bytes);
        char* p = static_cast<char*>(b->mem);
        int64_t moved = 0;
        for (size_t k = 0; k < secs.size(); ++k) {
            const Sec& s = secs[k];
            // a section that aliases an earlier one in the host descriptor
            // (e.g. inputs == dependencies, HostBatch packs them once) is
            // copied once and aliased on the device (read-only sections)
            bool aliased = false;
            for (size_t j = 0; j < k && !aliased; ++j)
                if (s.bytes && secs[j].src == s.src && secs[j].bytes == s.bytes) {
                    *s.dst = *secs[j].dst;
                    aliased = true;
                }
            if (aliased) continue;
            *s.dst = p;
            if (s.bytes) {
                cuda_check(cudaMemcpyAsync(p, s.src, s.bytes, cudaMemcpyHostToDevice, ctx->stream), "H2D batch");
                moved += static_cast<int64_t>(s.bytes);
            }
            p += al16(s.bytes);
        }
        d.succ_off = reinterpret_cast<int32_t*>(p);
        d.succ = reinterpret_cast<int32_t*>(p + al16((T + G) * 4));
        d.G = G; d.T = T; d.E = E; d.H = H; d.I = I; d.O = O;
        d.max_n = max_n; d.max_e = max_e; d.max_h = max_h;
        // type ids index the cost table; without a name table, scan them
        int32_t n_types = h->n_type_names;
        if (n_types <= 0) {
            for (int64_t t = 0; t < T; ++t) n_types = std::max(n_types, h->type[t] + 1);
            if (n_types > kMaxTypes) raise(TBSIM_E_INVALID_ARGUMENT, "more than 64 task types");
        }
        d.n_types = std::max(n_types, 1);
        b->h2d_bytes = moved;
        b->task_base.assign(h->task_base, h->task_base + G + 1);
        if (h->task_id) b->task_id.assign(h->task_id, h->task_id + T);
        for (int i = 0; i < h->n_type_names; ++i)
            b->type_names.push_back(h->type_names && h->type_names[i] ? h->type_names[i] : "type" + std::to_string(i));
        // derived successor CSR (sorted, multi-edges kept); deferred to the
        // compute stream when the copies ran on the upload stream
        if (G > 0 && us.active() && ctx->defer_ingest) {
            b->needs_ingest = true;
        } else if (G > 0) {
            ingest_uploaded(ctx, b.get());
        }
        if (us.active()) {
            cuda_check(cudaEventCreateWithFlags(&b->ready, cudaEventDisableTiming), "cudaEventCreate");
            cuda_check(cudaEventRecord(b->ready, ctx->stream), "cudaEventRecord(ready)");
        }
        *out = b.release();
    });
}

tbsim_status tbsim_batch_free(tbsim_ctx* ctx, tbsim_batch* b) {
    return guarded([&] {
        if (!b) return;
        std::unique_ptr<DeviceScope> dev_scope;
        if (ctx) dev_scope = std::make_unique<DeviceScope>(ctx->device);
        if (ctx) {
            // stream-ordered reuse: a later upload waits for every kernel
            // that reads this batch (all on the compute stream)
            for (auto [m, bytes] : {std::make_pair(b->mem, b->mem_bytes), std::make_pair(b->mem2, b->mem2_bytes),
                                    std::make_pair(b->mem3, b->mem3_bytes)}) {
                if (!m) continue;
                cudaEvent_t ev = nullptr;
                if (ctx->upload && ctx->upload != ctx->stream) {
                    cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
                    cuda_check(cudaEventRecord(ev, ctx->stream), "cudaEventRecord(freed)");
                }
                ctx->batch_pool.push_back({m, bytes, ev});
            }
        } else {
            if (b->mem) cudaFree(b->mem);
            if (b->mem2) cudaFree(b->mem2);
            if (b->mem3) cudaFree(b->mem3);
        }
        if (b->ready) cudaEventDestroy(b->ready);
        delete b;
    });
}

int64_t tbsim_batch_h2d_bytes(const tbsim_batch* b) { return b ? b->h2d_bytes : 0; }

tbsim_status tbsim_batch_sizes(const tbsim_batch* b, int64_t* s) {
    return guarded([&] {
        s[0] = b->d.G; s[1] = b->d.T; s[2] = b->d.E; s[3] = b->d.H; s[4] = b->d.I; s[5] = b->d.O;
    });
}

tbsim_status tbsim_batch_download(tbsim_ctx* ctx, const tbsim_batch* b, tbsim_batch_desc* h) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        wait_batch(ctx, b);
        const DevBatch& d = b->d;
        const int64_t G = d.G, T = d.T;
        auto cp = [&](const void* dst, const void* src, size_t bytes) {
            if (dst && bytes)
                cuda_check(cudaMemcpyAsync(const_cast<void*>(dst), src, bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H batch");
        };
        cp(h->task_base, d.task_base, (G + 1) * 8);
        cp(h->edge_base, d.edge_base, (G + 1) * 8);
        cp(h->handle_base, d.handle_base, (G + 1) * 8);
        cp(h->in_base, d.in_base, (G + 1) * 8);
        cp(h->out_base, d.out_base, (G + 1) * 8);
        cp(h->dep_off, d.dep_off, (T + G) * 4);
        cp(h->dep, d.dep, d.E * 4);
        cp(h->in_off, d.in_off, (T + G) * 4);
        cp(h->in, d.in, d.I * 4);
        cp(h->out_off, d.out_off, (T + G) * 4);
        cp(h->out, d.out, d.O * 4);
        cp(h->type, d.type, T * 4);
        cp(h->handle_bytes, d.handle_bytes, d.H * 8);
        ctx->sync();
    });
}

tbsim_status tbsim_batch_generate_layered(tbsim_ctx* ctx, int32_t n, int32_t L, double p, const uint64_t* seeds,
                                          int64_t n_seeds, tbsim_batch** out) {
    return guarded([&] {
        // generate_layered_dag's argument checks (src/generators.cpp:186-191)
        if (L < 1) raise(TBSIM_E_INVALID_ARGUMENT, "autogen: n_layers must be >= 1");
        if (n < L) raise(TBSIM_E_INVALID_ARGUMENT, "autogen: n_tasks must be >= n_layers");
        if (!(p >= 0.0 && p <= 1.0)) raise(TBSIM_E_INVALID_ARGUMENT, "autogen: edge_prob must be in [0,1]");
        if (n >= (1 << 24)) raise(TBSIM_E_INVALID_ARGUMENT, "graph exceeds 2^24 tasks");
        DeviceScope dev_scope(ctx->device);
        const int64_t G = n_seeds, T = G * n;
        auto b = std::make_unique<tbsim_batch>();
        GenParams q{};
        q.G = G;
        q.n = n;
        q.L = L;
        q.p = p;
        uint64_t* d_seeds = ctx->buf("g_seeds").as<uint64_t>(G);
        cuda_check(cudaMemcpyAsync(d_seeds, seeds, G * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D seeds");
        b->h2d_bytes = G * 8;
        q.seeds = d_seeds;
        q.ndep = ctx->buf("g_ndep").as<int32_t>(T);
        q.degree = ctx->buf("g_degree").as<int32_t>(T);
        q.max_degree = 2 * ((n + L - 1) / L) + 2;
        q.hist = ctx->buf("g_hist").as<int32_t>(G * (q.max_degree + 1));
        q.edges = ctx->buf("g_edges").as<int64_t>(G);
        q.type_base = tbsim_host::T_LAYERK0;
        // pass 1 records the draws' outcome (member bits, forced picks) so
        // pass 2 expands them without a second replay of the generator
        std::vector<int32_t> wl(static_cast<size_t>(L) + 1, 0);
        for (int32_t l = 0; l < L; ++l) {
            const int64_t members = l == 0 ? 0 : (static_cast<int64_t>(n) - 1 - (l - 1)) / L + 1;
            wl[l + 1] = wl[l] + static_cast<int32_t>((members + 31) / 32);
        }
        const int64_t per_dag = static_cast<int64_t>(n / L) * wl[L] + wl[n % L];
        int32_t* d_wl = ctx->buf("g_wl").as<int32_t>(wl.size());
        cuda_check(cudaMemcpyAsync(d_wl, wl.data(), wl.size() * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D wl");
        q.wl_prefix = d_wl;
        q.mask_per_dag = std::max<int64_t>(per_dag, 1);
        q.mask = ctx->buf("g_mask").as<uint32_t>(static_cast<size_t>(G * q.mask_per_dag));
        q.forced = ctx->buf("g_forced").as<int32_t>(std::max<int64_t>(T, 1));
        cuda_check(cudaMemsetAsync(q.mask, 0, static_cast<size_t>(G * q.mask_per_dag) * 4, ctx->stream), "memset mask");
        cuda_check(cudaMemsetAsync(q.forced, 0xff, static_cast<size_t>(T) * 4, ctx->stream), "memset forced");
        // fixed-size sections: bases, offsets, out, type, handle_bytes
        DevBatch& d = b->d;
        const size_t fixed = 5 * al16((G + 1) * 8) + 3 * al16((T + G) * 4) + al16(T * 4) + al16(T * 4) + al16(T * 8);
        b->mem = ctx->batch_alloc(fixed + 16, &b->mem_bytes);
        char* c = static_cast<char*>(b->mem);
        auto take = [&](size_t bytes) { char* r = c; c += al16(bytes); return r; };
        int64_t* task_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        int64_t* edge_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        int64_t* handle_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        int64_t* in_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        int64_t* out_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        d.dep_off = reinterpret_cast<int32_t*>(take((T + G) * 4));
        d.in_off = reinterpret_cast<int32_t*>(take((T + G) * 4));
        d.out_off = reinterpret_cast<int32_t*>(take((T + G) * 4));
        d.out = reinterpret_cast<int32_t*>(take(T * 4));
        int32_t* type = reinterpret_cast<int32_t*>(take(T * 4));
        int64_t* hbytes = reinterpret_cast<int64_t*>(take(T * 8));
        q.type = type;
        q.handle_bytes = hbytes;
        d.type = type;
        d.handle_bytes = hbytes;
        d.task_base = task_base;
        d.edge_base = edge_base;
        d.handle_base = handle_base;
        d.in_base = in_base;
        d.out_base = out_base;
        if (G > 0) {
            ctx->begin("k_gen_layered_count");
            k_gen_layered_count<<<static_cast<unsigned>((G + 3) / 4), 128, 0, ctx->stream>>>(q);
            ctx->end("k_gen_layered_count");
        }
        std::vector<int64_t> edges(G), ebase(G + 1, 0), tbase(G + 1, 0);
        if (G > 0) cuda_check(cudaMemcpyAsync(edges.data(), q.edges, G * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H edges");
        ctx->sync();
        for (int64_t g = 0; g < G; ++g) {
            ebase[g + 1] = ebase[g] + edges[g];
            tbase[g + 1] = tbase[g] + n;
        }
        const int64_t E = ebase[G];
        if (E > INT32_MAX * int64_t(G > 0 ? G : 1)) raise(TBSIM_E_INVALID_ARGUMENT, "batch too large");
        for (int64_t* dst : {task_base, handle_base, out_base})
            cuda_check(cudaMemcpyAsync(dst, tbase.data(), (G + 1) * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D bases");
        for (int64_t* dst : {edge_base, in_base})
            cuda_check(cudaMemcpyAsync(dst, ebase.data(), (G + 1) * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D bases");
        b->h2d_bytes += 5 * (G + 1) * 8;
        const size_t edge_sec = al16(E * 4) + al16((T + G) * 4) + al16(E * 4);
        b->mem2 = ctx->batch_alloc(edge_sec + 16, &b->mem2_bytes);
        c = static_cast<char*>(b->mem2);
        d.dep = reinterpret_cast<int32_t*>(take(E * 4));
        d.in = d.dep;  // inputs are the dependencies' handles (generators.cpp:239-243)
        d.in_off = d.dep_off;
        d.succ_off = reinterpret_cast<int32_t*>(take((T + G) * 4));
        d.succ = reinterpret_cast<int32_t*>(take(E * 4));
        d.G = G; d.T = T; d.E = E; d.H = T; d.I = E; d.O = T;
        d.max_n = n;
        d.max_h = n;
        d.max_e = 0;
        for (int64_t g = 0; g < G; ++g) d.max_e = std::max<int32_t>(d.max_e, static_cast<int32_t>(edges[g]));
        d.n_types = tbsim_host::T_COUNT;
        if (G > 0) {
            ctx->begin("k_gen_layered_fill");
            k_gen_layered_expand<<<static_cast<unsigned>(std::min<int64_t>(G, 8LL * ctx->n_sms)), 256, 0, ctx->stream>>>(q, d);
            ctx->end("k_gen_layered_fill");
            ingest_uploaded(ctx, b.get());  // successor CSR + packed simulation view
        }
        b->task_base = tbase;
        for (int i = 0; i < tbsim_host::T_COUNT; ++i) b->type_names.push_back(tbsim_host::kTypeNames[i]);
        *out = b.release();
    });
}

tbsim_status tbsim_batch_generate_tiled(tbsim_ctx* ctx, int32_t kind, int32_t nb, int64_t bytes, int64_t count,
                                        tbsim_batch** out) {
    return guarded([&] {
        static const char* names[3] = {"cholesky", "lu", "qr"};
        if (kind < TBSIM_TILED_CHOLESKY || kind > TBSIM_TILED_QR) raise(TBSIM_E_INVALID_ARGUMENT, "unknown tiled DAG kind");
        if (nb < 1) raise(TBSIM_E_INVALID_ARGUMENT, std::string(names[kind]) + ": nblocks must be >= 1");
        if (bytes <= 0) raise(TBSIM_E_INVALID_ARGUMENT, std::string(names[kind]) + ": block_bytes must be > 0");
        if (count < 0) raise(TBSIM_E_INVALID_ARGUMENT, "negative graph count");
        const int64_t n64 = tiled_task_count(kind, nb);
        if (n64 >= (1 << 24)) raise(TBSIM_E_INVALID_ARGUMENT, "graph exceeds 2^24 tasks");
        DeviceScope dev_scope(ctx->device);
        const int32_t n = static_cast<int32_t>(n64);
        const int32_t nh = kind == TBSIM_TILED_CHOLESKY ? nb * (nb + 1) / 2 : nb * nb;
        const int64_t G = count, T = G * n, H = G * nh;
        // one graph's list lengths -> local offsets (identical in every copy)
        int32_t* off = ctx->buf("g_tiled_off").as<int32_t>(3 * (static_cast<int64_t>(n) + 1));
        int64_t* d_tot = ctx->buf("g_tiled_tot").as<int64_t>(3);
        const int gridc = static_cast<int>(std::min<int64_t>((n + 256) / 256, 16LL * ctx->n_sms));
        ctx->begin("k_gen_tiled_count");
        k_gen_tiled_count<<<gridc, 256, 0, ctx->stream>>>(kind, nb, n, off);
        k_gen_tiled_scan<<<1, 1024, 0, ctx->stream>>>(n, off, d_tot);
        ctx->end("k_gen_tiled_count");
        int64_t tot[3];
        cuda_check(cudaMemcpyAsync(tot, d_tot, sizeof tot, cudaMemcpyDeviceToHost, ctx->stream), "D2H totals");
        ctx->sync();
        const int64_t E = G * tot[0], I = G * tot[1], O = G * tot[2];
        auto b = std::make_unique<tbsim_batch>();
        DevBatch& d = b->d;
        const size_t bytes_all = 5 * al16((G + 1) * 8) + 3 * al16((T + G) * 4) + 2 * al16(E * 4) + al16(I * 4) +
                                 al16(O * 4) + al16(T * 4) + al16(H * 8) + al16((T + G) * 4);
        b->mem = ctx->batch_alloc(bytes_all + 16, &b->mem_bytes);
        char* c = static_cast<char*>(b->mem);
        auto take = [&](size_t sz) { char* r = c; c += al16(sz); return r; };
        int64_t* task_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        int64_t* edge_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        int64_t* handle_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        int64_t* in_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        int64_t* out_base = reinterpret_cast<int64_t*>(take((G + 1) * 8));
        d.dep_off = reinterpret_cast<int32_t*>(take((T + G) * 4));
        d.in_off = reinterpret_cast<int32_t*>(take((T + G) * 4));
        d.out_off = reinterpret_cast<int32_t*>(take((T + G) * 4));
        d.dep = reinterpret_cast<int32_t*>(take(E * 4));
        d.in = reinterpret_cast<int32_t*>(take(I * 4));
        d.out = reinterpret_cast<int32_t*>(take(O * 4));
        d.type = reinterpret_cast<int32_t*>(take(T * 4));
        d.handle_bytes = reinterpret_cast<int64_t*>(take(H * 8));
        d.succ_off = reinterpret_cast<int32_t*>(take((T + G) * 4));
        d.succ = reinterpret_cast<int32_t*>(take(E * 4));
        std::vector<int64_t> tb(G + 1), eb(G + 1), hb(G + 1), ib(G + 1), ob(G + 1);
        for (int64_t g = 0; g <= G; ++g) {
            tb[g] = g * n; eb[g] = g * tot[0]; hb[g] = g * nh; ib[g] = g * tot[1]; ob[g] = g * tot[2];
        }
        const std::pair<int64_t*, const std::vector<int64_t>*> bases[5] = {
            {task_base, &tb}, {edge_base, &eb}, {handle_base, &hb}, {in_base, &ib}, {out_base, &ob}};
        for (const auto& pb : bases)
            cuda_check(cudaMemcpyAsync(pb.first, pb.second->data(), (G + 1) * 8, cudaMemcpyHostToDevice, ctx->stream),
                       "H2D bases");
        b->h2d_bytes = 5 * (G + 1) * 8;
        d.task_base = task_base; d.edge_base = edge_base; d.handle_base = handle_base;
        d.in_base = in_base; d.out_base = out_base;
        d.G = G; d.T = T; d.E = E; d.H = H; d.I = I; d.O = O;
        d.max_n = n;
        d.max_h = nh;
        d.max_e = static_cast<int32_t>(tot[0]);
        d.n_types = tbsim_host::T_COUNT;
        if (G > 0) {
            const int gridf = static_cast<int>(std::min<int64_t>((G * (n + 1) + 255) / 256, 16LL * ctx->n_sms));
            ctx->begin("k_gen_tiled_fill");
            k_gen_tiled_fill<<<gridf, 256, 0, ctx->stream>>>(kind, nb, n, nh, bytes, off, d);
            ctx->end("k_gen_tiled_fill");
            ingest_uploaded(ctx, b.get());  // successor CSR + packed simulation view
        }
        b->task_base = tb;
        for (int i = 0; i < tbsim_host::T_COUNT; ++i) b->type_names.push_back(tbsim_host::kTypeNames[i]);
        *out = b.release();
    });
}

}  // extern "C"

// ---------------------------------------------------------------- attributes

namespace {

struct AttrRun {
    AttrScratch s{};
    std::string pin_sfx;              // pinned staging name suffix (async result set)
    const GraphInfo* pinned = nullptr;  // D2H target of the per-graph infos
    std::vector<GraphInfo> info;      // host copy: fetch() after the stream reached the copy
    void fetch(int64_t G) { info.assign(pinned, pinned + G); }
};

AttrScratch alloc_attr_scratch(tbsim_ctx* ctx, const DevBatch& d) {
    ctx->scratch_gen += 1;
    AttrScratch s{};
    const int64_t T = d.T, G = d.G, E = d.E, NT = d.n_types;
    s.tmp = ctx->buf("a_tmp").as<int32_t>(T + G);
    s.tmp2 = ctx->buf("a_tmp2").as<int32_t>(T + G);
    s.order = ctx->buf("a_order").as<int32_t>(T);
    s.level = ctx->buf("a_level").as<int32_t>(T);
    s.lstart = ctx->buf("a_lstart").as<int32_t>(T + G);
    s.height = ctx->buf("a_height").as<int32_t>(T);
    s.lastuse = ctx->buf("a_lastuse").as<int32_t>(T);
    s.slot = ctx->buf("a_slot").as<int32_t>(T);
    s.rel_order = ctx->buf("a_rel").as<int32_t>(T);
    s.fstack = ctx->buf("a_fstack").as<int32_t>(T);
    s.cls = ctx->buf("a_cls").as<int32_t>(T);
    s.cls_mark = ctx->buf("a_clsmark").as<int32_t>(T * NT);
    s.om_slot = ctx->buf("a_omslot").as<int32_t>(T);
    s.om_gpu = ctx->buf("a_omgpu").as<double>(T);
    s.om_poff = ctx->buf("a_ompoff").as<int32_t>(T + G);
    s.om_pslot = ctx->buf("a_ompslot").as<int32_t>(E);
    s.rank = ctx->buf("a_rank").as<double>(T);
    s.hist = ctx->buf("a_hist").as<uint32_t>(static_cast<int64_t>(kBins) * T);
    s.info = ctx->buf("a_info").as<GraphInfo>(G);
    s.median = ctx->buf("a_median").as<double>(G);
    s.tile_base = ctx->buf("a_tilebase").as<int64_t>(G + 1);
    s.tile_s = ctx->buf("a_tiles").as<int32_t>(G);
    s.tile_graph = ctx->buf("a_tilegraph").as<int32_t>(T / 8 + G + 1);
    s.plan_fp32 = ctx->buf("a_planfp32").as<int32_t>(2);
    s.opos = ctx->buf("a_opos").as<int32_t>(T);
    s.firstuse = ctx->buf("a_firstuse").as<int32_t>(T);
    s.rslot = ctx->buf("a_rslot").as<int32_t>(T);
    return s;
}

constexpr int kSweepThreads = 512;

int64_t sweep_smem_bytes(tbsim_ctx* ctx) {
    // leave room for the kernel's static shared memory (256-source histogram)
    int64_t opt = static_cast<int64_t>(ctx->smem_optin);
    return std::max<int64_t>(0, opt - 14 * 1024);
}

// One large graph: the structure pass with the whole GPU (cooperative).
void launch_structure_large(tbsim_ctx* ctx, const DevBatch& d, const DevCosts* d_costs, const int32_t* d_cost_idx,
                            const AttrScratch& s, bool want_rank, bool sort_levels = false) {
    int& per_sm = ctx->structure_large_per_sm;
    if (!per_sm) cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_structure_large, 512, 0), "occupancy");
    // one CTA per SM: the per-level grid barriers cost less with fewer
    // participants (C4, 2 x 1024 barriers: 296 CTAs 9.3 ms, 148 8.0 ms,
    // 64 7.6 ms, 32 11.2 ms -- below ~one warp per frontier node the
    // levels' dependent memory chains dominate)
    const int grid = std::max(1, std::min(per_sm, 1)) * ctx->n_sms;
    const size_t ctl_bytes = sizeof(LargeCtl) + 4 * static_cast<size_t>(grid);
    LargeCtl* ctl = static_cast<LargeCtl*>(ctx->buf("a_large_ctl").get(ctl_bytes));
    cuda_check(cudaMemsetAsync(ctl, 0, ctl_bytes, ctx->stream), "memset");
    DevBatch dv = d;
    AttrScratch sv = s;
    int32_t wr = want_rank ? 1 : 0, so = sort_levels ? 1 : 0;
    void* args[] = {&dv, const_cast<DevCosts**>(&d_costs), const_cast<int32_t**>(&d_cost_idx), &sv, &wr, &ctl, &so};
    ctx->begin("k_structure");
    cuda_check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_structure_large), grid, 512, args, 0, ctx->stream),
               "cudaLaunchCooperativeKernel(k_structure_large)");
    ctx->end("k_structure");
}

// CTAs of a sweep whose tiles use per-CTA global windows (stride doubles
// each): one per SM while the windows total <= 8 GB, fewer for very wide
// graphs (the tile queue is persistent, any grid is correct)
int gwin_grid(const tbsim_ctx* ctx, int64_t stride) {
    const int64_t budget = (8LL << 30) / 8;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->n_sms, budget / std::max<int64_t>(stride, 1))));
}

// Launch the whole attribute pipeline on a device batch.  Returns with the
// per-graph GraphInfo copied to the host (one sync).
void run_attributes(tbsim_ctx* ctx, const tbsim_batch* b, const DevCosts* d_costs, const int32_t* d_cost_idx,
                    int32_t sweep_mode, const double* d_unit_time, bool want_rank, bool do_sweep,
                    AttrOutDev o, int32_t prio_kind, bool want_prio, AttrRun& run) {
    const DevBatch& d = b->d;
    const int64_t G = d.G;
    run.s = alloc_attr_scratch(ctx, d);
    if (G == 0) return;
    // One huge graph (C4-like): ability by the HBM bitset closure, the sweep
    // pruned at the largest window.  Batches: ability inside the sweep.
    const bool large = G == 1 && d.max_n >= ctx->large_threshold && do_sweep;
    const int grid_g = static_cast<int>(std::min<int64_t>(G, 4LL * ctx->n_sms));
    if (G == 1 && d.max_n >= ctx->large_threshold) {
        launch_structure_large(ctx, d, d_costs, d_cost_idx, run.s, want_rank);
    } else {
        // a CTA per graph, as many resident as fit (a partial second wave of
        // CTAs that each walk ~G/grid graphs would double the tail); small
        // graphs use small CTAs -- a level of a 1k-task DAG has ~100 nodes
        const int st_threads = d.max_n <= 4096 ? 128 : 512;
        // in-degrees and allocator cursors in shared memory for graphs of
        // < 2048 tasks (<= 16 KB)
        const int32_t st_ints = d.max_n < 2048 ? 2 * ((d.max_n + 1 + 31) & ~31) : 0;
        int per_sm = 0;
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_structure, st_threads, st_ints * 4),
                   "occupancy");
        const int grid_s = static_cast<int>(std::min<int64_t>(G, static_cast<int64_t>(std::max(per_sm, 1)) * ctx->n_sms));
        ctx->begin("k_structure");
        k_structure<<<grid_s, st_threads, static_cast<size_t>(st_ints) * 4, ctx->stream>>>(
            d, d_costs, d_cost_idx, run.s, want_rank ? 1 : 0, large ? 1 : 0, st_ints);
        ctx->end("k_structure");
    }
    bool ability_done = false;
    if (large && o.ability) {
        GraphInfo gi;
        cuda_check(cudaMemcpyAsync(&gi, run.s.info, sizeof gi, cudaMemcpyDeviceToHost, ctx->stream), "D2H info");
        ctx->sync();
        const int64_t nw = (static_cast<int64_t>(d.max_n) + 63) / 64;
        const size_t need = static_cast<size_t>(std::max(gi.peak_rslots, 1)) * static_cast<size_t>(nw) * 8;
        // the closure keeps one full-width set per live slot: a graph with a
        // very wide level cut (e.g. millions of sinks under one root) does
        // not fit, and its ability comes from the unpruned sweep instead
        // (free memory is queried only when the set buffer must grow:
        // cudaMemGetInfo costs milliseconds)
        const size_t have = ctx->buf("a_sets").bytes;
        bool fits = need <= have;
        if (!fits) {
            size_t free_b = 0, total_b = 0;
            cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
            fits = need <= (free_b + have) / 2;
        }
        if (gi.processed == d.max_n && fits) {  // acyclic: otherwise the error path reports it
            uint64_t* sets = ctx->buf("a_sets").as<uint64_t>(need / 8);
            cuda_check(cudaMemsetAsync(o.ability, 0, static_cast<size_t>(d.T) * 8, ctx->stream), "memset ability");
            // TMA bulk copies need 16-byte aligned set rows (an even word count)
            // TMA bulk copies of 4-KB successor chunks (k_closure_tma) need
            // 16-byte aligned set rows: an even word count
            const bool tma = nw % 2 == 0;
            const void* kern = tma ? reinterpret_cast<const void*>(k_closure_tma<3, 16, 2>)
                                   : reinterpret_cast<const void*>(k_closure<4>);
            const int threads = tma ? 64 : 256;
            int per_sm = 0;
            cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0), "occupancy");
            const int grid = std::max(1, per_sm) * ctx->n_sms;
            int64_t g0 = 0;
            int64_t wlo = 0, whi = nw;
            DevBatch dv = d;
            AttrScratch sv = run.s;
            unsigned long long* ab = reinterpret_cast<unsigned long long*>(o.ability);
            void* args[] = {&dv, &sv, &g0, &sets, &wlo, &whi, &ab};
            ctx->begin("k_closure");
            cuda_check(cudaLaunchCooperativeKernel(kern, grid, threads, args, 0, ctx->stream),
                       "cudaLaunchCooperativeKernel(k_closure)");
            ctx->end("k_closure");
            ability_done = true;
        }
    }
    // the large-graph sweep prunes at the largest window unless it must
    // count every descendant (ability requested and not from the closure)
    const bool prune = large && (ability_done || !o.ability);
    if (do_sweep && !(ability_done && sweep_mode == SWEEP_ABILITY)) {
        const int64_t smem = sweep_smem_bytes(ctx);
        ctx->begin("k_tile_plan");
        k_tile_plan<<<1, 1024, 0, ctx->stream>>>(d, run.s, smem, ctx->sweep_tile, d_costs, d_cost_idx, sweep_mode);
        ctx->end("k_tile_plan");
        // graphs whose distance window exceeds shared memory (P live slots x
        // 32 FP64 columns per CTA in HBM): k_tile_plan reports the largest P
        int64_t gwin_stride = 0;
        double* gwin = nullptr;
        int sweep_grid = ctx->n_sms;  // one 512-thread CTA per SM (smem bound)
        if (static_cast<int64_t>(d.max_n) * 8 * 8 > smem) {
            int32_t pmax = 0;
            cuda_check(cudaMemcpyAsync(&pmax, run.s.plan_fp32 + 1, 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H plan");
            ctx->sync();
            if (pmax > 0) {
                gwin_stride = static_cast<int64_t>(pmax) * 32;
                sweep_grid = gwin_grid(ctx, gwin_stride);
                gwin = ctx->buf("a_gwin").as<double>(gwin_stride * sweep_grid);
            }
        }
        unsigned long long* counter = ctx->buf("a_counter").as<unsigned long long>(1);
        cuda_check(cudaMemsetAsync(counter, 0, 8, ctx->stream), "memset");
        const int64_t total_tiles = -1;  // read on the device from tile_base[G]
        if (!ctx->sweep_attr) {
            cuda_check(cudaFuncSetAttribute(k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                       "cudaFuncSetAttribute(k_sweep)");
            ctx->sweep_attr = true;
        }
        // executed relaxations (rows x columns) when timing: the sweep's
        // achieved rate for bench.py's roofline
        unsigned long long* relax_ctr = nullptr;
        if (ctx->timing) {
            relax_ctr = ctx->buf("a_relax").as<unsigned long long>(2);
            cuda_check(cudaMemsetAsync(relax_ctr, 0, 16, ctx->stream), "memset");
            ctx->relax_ctr = relax_ctr;
        }
        if (!ctx->sweep32_attr) {
            cuda_check(cudaFuncSetAttribute(k_sweep_fp32, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                       "cudaFuncSetAttribute(k_sweep_fp32)");
            ctx->sweep32_attr = true;
        }
        // both launched: the plan (device) selects one, the other returns
        ctx->begin("k_sweep");
        k_sweep<<<sweep_grid, kSweepThreads, smem, ctx->stream>>>(d, d_costs, d_cost_idx, run.s, sweep_mode, d_unit_time,
                                                                  total_tiles, counter, smem, gwin, gwin_stride,
                                                                  prune ? 1 : 0, relax_ctr);
        k_sweep_fp32<<<sweep_grid, 1024, smem, ctx->stream>>>(d, run.s, sweep_mode, d_unit_time, counter, prune ? 1 : 0,
                                                               relax_ctr);
        ctx->end("k_sweep");
        const int64_t cls_stride = static_cast<int64_t>(d.max_n) * (3 * kWindows + 1) + 16;
        int64_t* cls_scratch = ctx->buf("a_cls_sums").as<int64_t>(cls_stride * grid_g);
        const int32_t write_ab = (prune || ability_done) ? 0 : 1;
        if (G == 1 && d.max_n >= ctx->large_threshold) {
            int& per_sm = ctx->finalize_large_per_sm;
            if (!per_sm)
                cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_finalize_large, 512, 0), "occupancy");
            const int grid = std::max(1, std::min(per_sm, 2)) * ctx->n_sms;
            int64_t tab_cap = 1;
            while (tab_cap < 2 * static_cast<int64_t>(d.max_n)) tab_cap <<= 1;
            int32_t* tab = ctx->buf("a_fin_tab").as<int32_t>(tab_cap * kWindows);
            int32_t* score = ctx->buf("a_fin_score").as<int32_t>(kWindows);
            DevBatch dv = d;
            AttrScratch sv = run.s;
            int32_t sm = sweep_mode, wa = write_ab, ph = FIN_ALL, plo = 0, phi = d.max_n;
            const int64_t* sums_in = nullptr;
            void* args[] = {&dv, &sv, &sm, &o, &cls_scratch, &tab, &tab_cap, &score, &wa, &ph, &plo, &phi, &sums_in};
            ctx->begin("k_finalize");
            cuda_check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_finalize_large), grid, 512, args, 0, ctx->stream),
                       "cudaLaunchCooperativeKernel(k_finalize_large)");
            ctx->end("k_finalize");
        } else {
            ctx->begin("k_finalize");
            k_finalize<<<grid_g, 256, 0, ctx->stream>>>(d, run.s, sweep_mode, d_unit_time, o, cls_scratch, cls_stride,
                                                        write_ab);
            ctx->end("k_finalize");
        }
    }
    if (o.layer || o.depth || (want_prio && o.static_priority)) {
        const int grid = static_cast<int>(std::min<int64_t>((d.T + 255) / 256, 16LL * ctx->n_sms));
        if (grid > 0) {
            ctx->begin("k_structure_out");
            k_structure_out<<<grid, 256, 0, ctx->stream>>>(d, run.s, o, prio_kind, want_prio ? 1 : 0);
            ctx->end("k_structure_out");
        }
    }
    GraphInfo* pinned_info = ctx->pin<GraphInfo>("p_info" + run.pin_sfx, static_cast<size_t>(G));
    run.pinned = pinned_info;
    cuda_check(cudaMemcpyAsync(pinned_info, run.s.info, G * sizeof(GraphInfo), cudaMemcpyDeviceToHost, ctx->stream),
               "D2H info");
}

// Compose the reference's exception for the first failing graph, in the
// order each reference function checks its preconditions.
std::string type_name_of(const std::vector<std::string>& names, int32_t ty) {
    if (ty >= 0 && ty < static_cast<int32_t>(names.size())) return names[ty];
    return "type" + std::to_string(ty);
}

void attr_errors(const GraphInfo* info, int64_t G, const std::vector<int64_t>& task_base,
                 const std::vector<std::string>& type_names, int32_t request, const double* unit_time) {
    for (int64_t g = 0; g < G; ++g) {
        const GraphInfo& gi = info[g];
        const int64_t n = task_base[g + 1] - task_base[g];
        const bool cyc = gi.processed != n;
        // the failing tasks' types were recorded by the structure pass
        auto ty_of = [&](int32_t pos) -> std::string {
            const int32_t ty = pos == gi.miss_gpu ? (gi.miss_types & 0xffff) : (gi.miss_types >> 16) & 0xffff;
            return type_name_of(type_names, ty);
        };
        if (request & (TBSIM_ATTR_ALL | TBSIM_ATTR_CALIBRATE)) {
            // calibrate_unit_time: topological_layers, then median_gpu_time_ms
            if (cyc) raise(TBSIM_E_RUNTIME, "graph has a dependency cycle");
            if (n == 0) raise(TBSIM_E_RUNTIME, "empty graph has no median time");
            if (gi.miss_gpu >= 0) raise(TBSIM_E_RUNTIME, "no gpu cost entry for task type " + ty_of(gi.miss_gpu));
        }
        if (request & TBSIM_ATTR_EFFICIENCY) {
            // efficiency_impl: window check, gpu times, then topological_order
            const double w = unit_time ? unit_time[g] : 0.0;
            if (!(w >= 0.0)) raise(TBSIM_E_INVALID_ARGUMENT, "unit time must be non-negative");
            if (n > 0 && gi.miss_gpu >= 0) raise(TBSIM_E_RUNTIME, "no gpu cost entry for task type " + ty_of(gi.miss_gpu));
            if (cyc) raise(TBSIM_E_RUNTIME, "graph has a dependency cycle");
        }
        if (request & TBSIM_ATTR_RANK) {
            if (gi.miss_any >= 0) raise(TBSIM_E_RUNTIME, "no cost entry for task type " + ty_of(gi.miss_any));
            if (cyc) raise(TBSIM_E_RUNTIME, "graph has a dependency cycle");
        }
        if (request & (TBSIM_ATTR_DEPTH | TBSIM_ATTR_LAYERS))
            if (cyc) raise(TBSIM_E_RUNTIME, "graph has a dependency cycle");
    }
}

void attr_errors(const tbsim_batch* b, const std::vector<GraphInfo>& info, int32_t request, const double* unit_time) {
    attr_errors(info.data(), static_cast<int64_t>(info.size()), b->task_base, b->type_names, request, unit_time);
}

// Device output staging for host-pointer outputs.
struct OutStage {
    AttrOutDev dev{};
    std::vector<std::pair<void*, std::pair<const void*, size_t>>> copies;  // host dst, (dev src, bytes)
};

template <typename T>
T* stage_out(tbsim_ctx* ctx, OutStage& st, const char* name, T* host, size_t count, bool on_device) {
    if (!host) return nullptr;
    if (on_device) return host;
    T* dev = ctx->buf(name).as<T>(count);
    st.copies.push_back({host, {dev, count * sizeof(T)}});
    return dev;
}

}  // namespace

extern "C" tbsim_status tbsim_attributes(tbsim_ctx* ctx, const tbsim_batch* b, const tbsim_costs* costs,
                                         int32_t request, int32_t priority_kind, tbsim_attr_out* out) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        wait_batch(ctx, b);
        const DevBatch& d = b->d;
        const int64_t T = d.T, G = d.G;
        const bool dev = out->on_device != 0;
        // efficiency-only: window validation happens before any device work
        if ((request & TBSIM_ATTR_EFFICIENCY) && !(request & (TBSIM_ATTR_ALL | TBSIM_ATTR_CALIBRATE))) {
            if (!out->unit_time_ms) raise(TBSIM_E_INVALID_ARGUMENT, "efficiency needs unit_time_ms");
            if (!dev)
                for (int64_t g = 0; g < G; ++g)
                    if (!(out->unit_time_ms[g] >= 0.0)) raise(TBSIM_E_INVALID_ARGUMENT, "unit time must be non-negative");
        }
        DevCosts hc = to_dev_costs(*costs, d.n_types);
        DevCosts* d_costs = ctx->buf("costs").as<DevCosts>(1);
        cuda_check(cudaMemcpyAsync(d_costs, &hc, sizeof hc, cudaMemcpyHostToDevice, ctx->stream), "H2D costs");

        OutStage st;
        AttrOutDev o{};
        const bool all = request & TBSIM_ATTR_ALL;
        const bool calib = all || (request & TBSIM_ATTR_CALIBRATE);
        const bool eff_only = (request & TBSIM_ATTR_EFFICIENCY) && !calib;
        o.ability = stage_out(ctx, st, "o_ability", out->ability, T, dev);
        if (!(all || (request & TBSIM_ATTR_ABILITY))) o.ability = nullptr;
        o.efficiency = stage_out(ctx, st, "o_eff", out->efficiency, T, dev);
        if (!(all || (request & (TBSIM_ATTR_EFFICIENCY | TBSIM_ATTR_CALIBRATE)))) o.efficiency = nullptr;
        o.static_priority = stage_out(ctx, st, "o_prio", out->static_priority, T, dev);
        o.depth = (request & TBSIM_ATTR_DEPTH) ? stage_out(ctx, st, "o_depth", out->depth, T, dev) : nullptr;
        o.layer = (request & TBSIM_ATTR_LAYERS) ? stage_out(ctx, st, "o_layer", out->layer, T, dev) : nullptr;
        o.w0_ms = calib ? stage_out(ctx, st, "o_w0", out->w0_ms, G, dev) : nullptr;
        o.best_score = calib ? stage_out(ctx, st, "o_best", out->best_score, G, dev) : nullptr;
        o.w0_score = calib ? stage_out(ctx, st, "o_w0s", out->w0_score, G, dev) : nullptr;
        o.evaluations = calib ? stage_out(ctx, st, "o_evals", out->evaluations, G, dev) : nullptr;
        double* d_unit = nullptr;
        if (out->unit_time_ms) {
            if (dev) {
                d_unit = out->unit_time_ms;
            } else {
                d_unit = ctx->buf("o_unit").as<double>(G);
                if (eff_only)
                    cuda_check(cudaMemcpyAsync(d_unit, out->unit_time_ms, G * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D unit");
                if (calib) st.copies.push_back({out->unit_time_ms, {d_unit, static_cast<size_t>(G) * 8}});
            }
        }
        o.unit_time_ms = calib ? d_unit : nullptr;
        // static priority: ALL selects by kind; RANK alone -> rank
        bool want_prio = false;
        int32_t pk = priority_kind;
        if (all) want_prio = true;
        if (request & TBSIM_ATTR_RANK) { want_prio = true; pk = TBSIM_PRIO_UPWARD_RANK; }
        if (!want_prio) o.static_priority = nullptr;
        const bool want_rank = want_prio && pk == TBSIM_PRIO_UPWARD_RANK;
        const bool do_sweep = all || (request & (TBSIM_ATTR_ABILITY | TBSIM_ATTR_EFFICIENCY | TBSIM_ATTR_CALIBRATE));
        const int32_t mode = calib ? SWEEP_CALIBRATE : eff_only ? SWEEP_SINGLE : SWEEP_ABILITY;
        AttrRun run;
        run_attributes(ctx, b, d_costs, nullptr, mode, d_unit, want_rank, do_sweep, o, pk, want_prio, run);
        for (const auto& c : st.copies)
            cuda_check(cudaMemcpyAsync(c.first, c.second.first, c.second.second, cudaMemcpyDeviceToHost, ctx->stream), "D2H out");
        ctx->sync();
        ctx->collect_timing();
        run.fetch(G);
        std::vector<double> unit_host;
        if (eff_only && dev) {
            unit_host.resize(G);
            cudaMemcpy(unit_host.data(), d_unit, G * 8, cudaMemcpyDeviceToHost);
        }
        attr_errors(b, run.info, request, eff_only ? (dev ? unit_host.data() : out->unit_time_ms) : nullptr);
    });
}

// ------------------------------------------------- sharded large graphs

namespace {

// Rank r's share of the closure's words: each word w of every set costs one
// OR per node whose set reaches down to w (its level's lower word bound <= w),
// so the split balances the cumulative per-word node count.
std::pair<int64_t, int64_t> closure_word_range(const std::vector<int32_t>& lstart, int64_t nw, int32_t rank,
                                               int32_t world) {
    std::vector<double> dens(static_cast<size_t>(nw) + 1, 0.0);
    const size_t L = lstart.size() - 1;
    for (size_t l = 0; l < L; ++l) {
        const int64_t lo = std::min<int64_t>(lstart[l + 1] >> 6, nw);
        dens[static_cast<size_t>(lo)] += static_cast<double>(lstart[l + 1] - lstart[l]);
    }
    std::vector<double> cum(static_cast<size_t>(nw) + 1, 0.0);
    double run = 0.0;
    for (int64_t w = 0; w < nw; ++w) {
        run += dens[static_cast<size_t>(w)];
        cum[static_cast<size_t>(w) + 1] = cum[static_cast<size_t>(w)] + run;
    }
    const double total = cum[static_cast<size_t>(nw)];
    auto bound = [&](int32_t r) -> int64_t {
        if (r <= 0) return 0;
        if (r >= world) return nw;
        const double want = total * r / world;
        return std::lower_bound(cum.begin(), cum.end(), want) - cum.begin();
    };
    int64_t lo = std::min(bound(rank), nw), hi = std::min(bound(rank + 1), nw);
    return {lo, std::max(lo, hi)};
}

}  // namespace

extern "C" tbsim_status tbsim_attributes_shard_partial(tbsim_ctx* ctx, const tbsim_batch* b, const tbsim_costs* costs,
                                                       int32_t rank, int32_t world, int64_t* ability_partial,
                                                       int64_t* class_sums, int64_t cap, int64_t* n_words) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        wait_batch(ctx, b);
        const DevBatch& d = b->d;
        if (d.G != 1) raise(TBSIM_E_INVALID_ARGUMENT, "sharded attributes take a batch of one graph");
        if (world < 1 || rank < 0 || rank >= world) raise(TBSIM_E_INVALID_ARGUMENT, "shard rank out of range");
        const int64_t n = d.max_n;
        ctx->shard = tbsim_ctx::Shard{};
        DevCosts hc = to_dev_costs(*costs, d.n_types);
        DevCosts* d_costs = ctx->buf("costs").as<DevCosts>(1);
        cuda_check(cudaMemcpyAsync(d_costs, &hc, sizeof hc, cudaMemcpyHostToDevice, ctx->stream), "H2D costs");
        AttrScratch s = alloc_attr_scratch(ctx, d);
        // ranks share one bit space: sort each level by task position
        launch_structure_large(ctx, d, d_costs, nullptr, s, true, world > 1);
        GraphInfo gi;
        cuda_check(cudaMemcpyAsync(&gi, s.info, sizeof gi, cudaMemcpyDeviceToHost, ctx->stream), "D2H info");
        ctx->sync();
        attr_errors(b, {gi}, TBSIM_ATTR_ALL, nullptr);
        if (world > 1 && !gi.order_det)
            raise(TBSIM_E_INVALID_ARGUMENT, "sharded attributes need levels of at most 4096 tasks (deterministic bit space)");
        // ---- ability: this rank's words of every descendant set
        std::vector<int32_t> lstart(static_cast<size_t>(gi.n_levels) + 1);
        cuda_check(cudaMemcpy(lstart.data(), s.lstart, lstart.size() * 4, cudaMemcpyDeviceToHost), "D2H lstart");
        const int64_t nw = (n + 63) / 64;
        const auto [wlo, whi] = closure_word_range(lstart, nw, rank, world);
        int64_t* d_ab = ctx->buf("o_ability").as<int64_t>(std::max<int64_t>(n, 1));
        cuda_check(cudaMemsetAsync(d_ab, 0, static_cast<size_t>(n) * 8, ctx->stream), "memset ability");
        if (whi > wlo) {
            uint64_t* sets = ctx->buf("a_sets").as<uint64_t>(static_cast<size_t>(std::max(gi.peak_rslots, 1)) * (whi - wlo));
            // TMA bulk copies when this rank's rows start 16-byte aligned
            const bool tma = wlo % 2 == 0 && (whi - wlo) % 2 == 0;
            const void* kern = tma ? reinterpret_cast<const void*>(k_closure_tma<3, 16, 2>)
                                   : reinterpret_cast<const void*>(k_closure<4>);
            const int threads = tma ? 64 : 256;
            int per_sm = 0;
            cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0), "occupancy");
            const int grid = std::max(1, per_sm) * ctx->n_sms;
            int64_t g0 = 0, lo_ = wlo, hi_ = whi;
            DevBatch dv = d;
            AttrScratch sv = s;
            unsigned long long* ab = reinterpret_cast<unsigned long long*>(d_ab);
            void* args[] = {&dv, &sv, &g0, &sets, &lo_, &hi_, &ab};
            ctx->begin("k_closure");
            cuda_check(cudaLaunchCooperativeKernel(kern, grid, threads, args, 0, ctx->stream),
                       "cudaLaunchCooperativeKernel(k_closure)");
            ctx->end("k_closure");
        }
        // ---- efficiency sweep over this rank's share of the source tiles
        const int64_t smem = sweep_smem_bytes(ctx);
        k_tile_plan<<<1, 1024, 0, ctx->stream>>>(d, s, smem, ctx->sweep_tile, d_costs, nullptr, SWEEP_CALIBRATE);
        int32_t S = 0, pmax = 0;
        int64_t tiles = 0;
        cuda_check(cudaMemcpyAsync(&S, s.tile_s, 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H tile width");
        cuda_check(cudaMemcpyAsync(&tiles, s.tile_base + 1, 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H tiles");
        cuda_check(cudaMemcpyAsync(&pmax, s.plan_fp32 + 1, 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H plan");
        ctx->sync();
        S &= kTileWidthMask;
        const int64_t t_lo = tiles * rank / world, t_hi = tiles * (rank + 1) / world;
        const int32_t pos_lo = static_cast<int32_t>(std::min<int64_t>(t_lo * S, n));
        const int32_t pos_hi = static_cast<int32_t>(std::min<int64_t>(t_hi * S, n));
        if (t_hi > t_lo) {
            int64_t gwin_stride = 0;
            double* gwin = nullptr;
            int sweep_grid = ctx->n_sms;
            if (pmax > 0) {  // global-window tiles (P x 32 FP64 per CTA)
                gwin_stride = static_cast<int64_t>(pmax) * 32;
                sweep_grid = gwin_grid(ctx, gwin_stride);
                gwin = ctx->buf("a_gwin").as<double>(gwin_stride * sweep_grid);
            }
            unsigned long long* counter = ctx->buf("a_counter").as<unsigned long long>(1);
            const unsigned long long start = static_cast<unsigned long long>(t_lo);
            cuda_check(cudaMemcpyAsync(counter, &start, 8, cudaMemcpyHostToDevice, ctx->stream), "H2D counter");
            cuda_check(cudaFuncSetAttribute(k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                       "cudaFuncSetAttribute(k_sweep)");
            ctx->begin("k_sweep");
            k_sweep<<<sweep_grid, kSweepThreads, smem, ctx->stream>>>(d, d_costs, nullptr, s, SWEEP_CALIBRATE, nullptr,
                                                                      t_hi, counter, smem, gwin, gwin_stride, 1, nullptr);
            ctx->end("k_sweep");
        }
        // ---- this shard's per-class window sums
        const int64_t C = gi.n_classes;
        *n_words = C * (kWindows + 1);
        if (cap < *n_words) raise(TBSIM_E_INVALID_ARGUMENT, "class_sums needs " + std::to_string(*n_words) + " words");
        const int64_t cls_stride = n * (3 * kWindows + 1) + 16;
        int64_t* cls_scratch = ctx->buf("a_cls_sums").as<int64_t>(cls_stride);
        {
            int& per_sm = ctx->finalize_large_per_sm;
            if (!per_sm)
                cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_finalize_large, 512, 0), "occupancy");
            const int grid = std::max(1, std::min(per_sm, 2)) * ctx->n_sms;
            int64_t tab_cap = 1;
            while (tab_cap < 2 * n) tab_cap <<= 1;
            int32_t* tab = ctx->buf("a_fin_tab").as<int32_t>(tab_cap * kWindows);
            int32_t* score = ctx->buf("a_fin_score").as<int32_t>(kWindows);
            DevBatch dv = d;
            AttrScratch sv = s;
            AttrOutDev o{};
            int32_t sm = SWEEP_CALIBRATE, wa = 0, ph = FIN_PARTIAL, plo = pos_lo, phi = pos_hi;
            const int64_t* sums_in = nullptr;
            void* args[] = {&dv, &sv, &sm, &o, &cls_scratch, &tab, &tab_cap, &score, &wa, &ph, &plo, &phi, &sums_in};
            ctx->begin("k_finalize");
            cuda_check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_finalize_large), grid, 512, args, 0, ctx->stream),
                       "cudaLaunchCooperativeKernel(k_finalize_large)");
            ctx->end("k_finalize");
        }
        cuda_check(cudaMemcpyAsync(class_sums, cls_scratch, static_cast<size_t>(*n_words) * 8, cudaMemcpyDeviceToHost,
                                   ctx->stream), "D2H class sums");
        cuda_check(cudaMemcpyAsync(ability_partial, d_ab, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx->stream),
                   "D2H ability");
        ctx->sync();
        ctx->collect_timing();
        ctx->shard.b = b;
        ctx->shard.rank = rank;
        ctx->shard.world = world;
        ctx->shard.pos_lo = pos_lo;
        ctx->shard.pos_hi = pos_hi;
        ctx->shard.n_words = *n_words;
        ctx->shard.s = s;
        ctx->shard.gen = ctx->scratch_gen;
    });
}

extern "C" tbsim_status tbsim_attributes_shard_finish(tbsim_ctx* ctx, const tbsim_batch* b, const int64_t* class_sums,
                                                      int64_t n_words, int32_t priority_kind, tbsim_attr_out* out) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        const tbsim_ctx::Shard& sh = ctx->shard;
        if (sh.b != b || n_words != sh.n_words || sh.gen != ctx->scratch_gen)
            raise(TBSIM_E_INVALID_ARGUMENT, "shard finish must follow this rank's partial call on the same batch");
        if (out->on_device) raise(TBSIM_E_INVALID_ARGUMENT, "sharded attributes return host arrays");
        const DevBatch& d = b->d;
        const int64_t n = d.max_n;
        int64_t* d_sums = ctx->buf("a_shard_sums").as<int64_t>(std::max<int64_t>(n_words, 1));
        cuda_check(cudaMemcpyAsync(d_sums, class_sums, static_cast<size_t>(n_words) * 8, cudaMemcpyHostToDevice, ctx->stream),
                   "H2D class sums");
        OutStage st;
        AttrOutDev o{};
        o.efficiency = stage_out(ctx, st, "o_eff", out->efficiency, n, false);
        if (o.efficiency) cuda_check(cudaMemsetAsync(o.efficiency, 0, static_cast<size_t>(n) * 8, ctx->stream), "memset");
        o.static_priority = stage_out(ctx, st, "o_prio", out->static_priority, n, false);
        o.unit_time_ms = stage_out(ctx, st, "o_unit", out->unit_time_ms, 1, false);
        o.w0_ms = stage_out(ctx, st, "o_w0", out->w0_ms, 1, false);
        o.best_score = stage_out(ctx, st, "o_best", out->best_score, 1, false);
        o.w0_score = stage_out(ctx, st, "o_w0s", out->w0_score, 1, false);
        o.evaluations = stage_out(ctx, st, "o_evals", out->evaluations, 1, false);
        const int64_t cls_stride = n * (3 * kWindows + 1) + 16;
        int64_t* cls_scratch = ctx->buf("a_cls_sums").as<int64_t>(cls_stride);
        int& per_sm = ctx->finalize_large_per_sm;
        if (!per_sm) cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_finalize_large, 512, 0), "occupancy");
        const int grid = std::max(1, std::min(per_sm, 2)) * ctx->n_sms;
        int64_t tab_cap = 1;
        while (tab_cap < 2 * n) tab_cap <<= 1;
        int32_t* tab = ctx->buf("a_fin_tab").as<int32_t>(tab_cap * kWindows);
        int32_t* score = ctx->buf("a_fin_score").as<int32_t>(kWindows);
        DevBatch dv = d;
        AttrScratch sv = sh.s;
        int32_t sm = SWEEP_CALIBRATE, wa = 0, ph = FIN_FINISH, plo = sh.pos_lo, phi = sh.pos_hi;
        const int64_t* sums_in = d_sums;
        void* args[] = {&dv, &sv, &sm, &o, &cls_scratch, &tab, &tab_cap, &score, &wa, &ph, &plo, &phi, &sums_in};
        ctx->begin("k_finalize");
        cuda_check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_finalize_large), grid, 512, args, 0, ctx->stream),
                   "cudaLaunchCooperativeKernel(k_finalize_large)");
        ctx->end("k_finalize");
        if (o.static_priority) {
            const int g2 = static_cast<int>(std::min<int64_t>((n + 255) / 256, 16LL * ctx->n_sms));
            ctx->begin("k_structure_out");
            k_structure_out<<<std::max(g2, 1), 256, 0, ctx->stream>>>(d, sh.s, o, priority_kind, 1);
            ctx->end("k_structure_out");
        }
        for (const auto& c : st.copies)
            cuda_check(cudaMemcpyAsync(c.first, c.second.first, c.second.second, cudaMemcpyDeviceToHost, ctx->stream), "D2H out");
        ctx->sync();
        ctx->collect_timing();
    });
}

// ---------------------------------------------------------------- simulate

namespace {

struct SimRun {
    std::vector<int32_t> status, aux;
};

int32_t pow2_at_least(int32_t x) {
    int32_t r = 1;
    while (r < x) r <<= 1;
    return r;
}

// Picks the per-warp state placement and launch shape.  Up to 32 workers
// with compact state (k_simulate_w1c, <= 72 registers) runs 4-warp CTAs, up
// to 7 per SM (28 warps: the 4096 DAGs of C2 in one wave on 148 SMs); the
// state goes to shared memory when a queue capacity of >= 32 entries fits,
// else to HBM.  Wider platforms (k_simulate_w2*) and wide state run 8-warp
// CTAs, two per SM.
void launch_sim(tbsim_ctx* ctx, SimParams& p, int32_t max_workers, int64_t n_items,
                const char* name = "k_simulate") {
    const DevBatch& d = p.b;
    const bool compact = d.max_n < 32768 && p.max_nodes <= 8;
    const bool w2 = max_workers > 32;
    const bool tight = compact && !w2;
    const int max_warps = tight ? 4 : 8;
    const int max_ctas = tight ? 7 : 2;
    // Few DAGs (e.g. two 22k-task tiled factorizations): fewer warps per CTA
    // so each warp gets more shared memory; many DAGs: full CTAs.
    int kWarps = max_warps;
    while (kWarps > 1 && n_items < static_cast<int64_t>(kWarps) * ctx->n_sms) kWarps >>= 1;
    const int kThreads = 32 * kWarps;
    const int64_t qcap_full = std::max<int32_t>(d.max_n, 1);
    auto layout = [&](int64_t qcap) {
        return sim_layout(d.max_n, d.max_h, max_workers, qcap, p.ring, p.n_types, p.max_nodes, compact, p.policy);
    };
    // HBM state with full queues: reruns of queue overflows, and batches of
    // a few large DAGs (fewer warps than SMs, so shared memory buys no
    // occupancy, and their ready queues outgrow it: C3's LU/QR overflow a
    // shared-memory queue and measured 150 ms in HBM vs 167 ms in a 1-warp
    // shared-memory CTA)
    const bool few_large = n_items < ctx->n_sms && d.max_n >= 4096;
    const bool forced = p.qcap > 0 || few_large;
    int64_t qcap = qcap_full;
    int ctas_per_sm = max_ctas;
    p.use_smem = 0;
    if (!forced) {
        // Shared-memory budgets per SM, tried in order for each CTA count:
        // 196 KB first -- the 196 KB carveout leaves 60 KB of L1 for the
        // simulator's register spills and task records (C2: 8.6 -> 8.4 ms)
        // -- then all of it (228 KB).
        const int64_t full_sm = static_cast<int64_t>(ctx->smem_optin) + 1024;
        int c = max_ctas, bi = 0;
        const int64_t budgets[2] = {tight ? std::min<int64_t>(196 * 1024, full_sm) : full_sm, full_sm};
        for (int step = 0; step < 2 * max_ctas; ++step, bi ^= 1, c -= bi == 0 ? 1 : 0) {
            const int64_t per_sm = budgets[bi];
            const int64_t per_warp = (per_sm / c - 1024) / kWarps;
            if (layout(qcap_full).total <= per_warp) {
                qcap = qcap_full;
                ctas_per_sm = c;
                p.use_smem = 1;
                break;
            }
            const int64_t cap = (per_warp - layout(0).total - 64) / ((4 + key_bytes(p.policy, compact)) * max_workers);
            // short queues are the common case (C2: <= 27 entries); a graph
            // that overflows is re-run exactly with HBM state
            if (cap >= 32) {
                qcap = std::min<int64_t>(cap & ~int64_t(3), qcap_full);
                ctas_per_sm = c;
                p.use_smem = 1;
                break;
            }
        }
    }
    // Latency-bound: DAGs in flight set the throughput.  HBM (L2-resident)
    // state costs ~1.4x per event (C5 mixes: 42 ms vs 30 ms a wave), so it
    // wins once it at least doubles the warps per SM (C5's 36-worker batch:
    // 16 vs 8), and its queues never overflow.
    if (p.use_smem && !forced && ctas_per_sm * 2 <= max_ctas) {
        p.use_smem = 0;
        ctas_per_sm = max_ctas;
    }
    if (!p.use_smem) qcap = qcap_full;
    p.qcap = static_cast<int32_t>(qcap);
    p.layout = layout(qcap);
    p.state_bytes = p.layout.total;
    p.max_workers = max_workers;
    p.n_items = n_items;
    int grid = static_cast<int>(std::min<int64_t>((n_items + kWarps - 1) / kWarps,
                                                  static_cast<int64_t>(ctas_per_sm) * ctx->n_sms));
    grid = std::max(grid, 1);
    if (std::string(name) == "k_simulate") {
        ctx->sim_warps_per_sm = ctas_per_sm * kWarps;
        ctx->sim_state_smem = p.use_smem;
        ctx->sim_qcap = p.qcap;
    }
    const size_t smem = p.use_smem ? static_cast<size_t>(p.state_bytes * kWarps) : 0;
    if (!p.use_smem) p.gstate = static_cast<char*>(ctx->buf("s_gstate").get(static_cast<size_t>(p.state_bytes) * kWarps * grid));
    unsigned long long* counter = ctx->buf("s_counter").as<unsigned long long>(1);
    cuda_check(cudaMemsetAsync(counter, 0, 8, ctx->stream), "memset");
    p.work_counter = counter;
    // tasks reading many inputs (mean inputs x memory nodes > 32, C5: 18 x
    // up to 5): the transfer sums run in rounds over every node at once and
    // skip resident inputs.  A separate kernel, because the extra code costs
    // the few-input kernel 10% (C2) even where it never runs.
    const bool many_in = d.T > 0 && d.I * p.max_nodes > 32 * d.T && p.policy >= TBSIM_POLICY_DMDA;
    // inspirit without trace outputs: the policy-specialised kernels (trace
    // recording compiled away)
    const bool ins = p.policy == TBSIM_POLICY_INSPIRIT && !p.push_time && !p.pop_time && !p.sample_time;
    auto kern = compact ? (w2 ? (many_in ? (ins ? k_simulate_w2c_mi_ins : k_simulate_w2c_mi)
                                         : (ins ? k_simulate_w2c_ins : k_simulate_w2c))
                              : many_in ? (ins ? k_simulate_w1c_mi_ins : k_simulate_w1c_mi)
                              : ins ? k_simulate_w1c_ins : k_simulate_w1c)
                        : (w2 ? k_simulate_w2 : k_simulate_w1);
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "cudaFuncSetAttribute(k_simulate)");
    // HBM (L2-resident) state: every byte of the SM's unified L1/shared
    // array as L1, which caches the warps' state lines; shared-memory state:
    // the runtime's choice for the requested size
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    p.use_smem ? -1 : static_cast<int>(cudaSharedmemCarveoutMaxL1)),
               "cudaFuncSetAttribute(k_simulate carveout)");
    ctx->begin(name);
    kern<<<grid, kThreads, smem, ctx->stream>>>(p);
    ctx->end(name);
}

// Runs the simulator over every graph, reruns queue overflows with full
// capacity in HBM, and raises the first graph's error.
struct SimKeys {
    const int64_t* ability = nullptr;
    const int64_t* efficiency = nullptr;
    const int64_t* prio = nullptr;
};

// pof_host / hp: the graphs' platforms on the host (null: all platform 0).
// A batch mixing worker counts is dispatched longest-first: graphs on the
// fewest workers (longest queues, slowest simulations) start first, so they
// do not pile up at the tail of the atomic DAG queue.
// The first failing graph's exception (engine / policy texts), from the
// simulator's statuses; aux = task position | type id << 24.  worker_of(g)
// returns the graph's per-task workers (stuck-task listing).
void sim_errors(int64_t G, const int32_t* status, const int32_t* aux, const int64_t* completed,
                const std::vector<int64_t>& task_base, const std::vector<int64_t>& task_id,
                const std::vector<std::string>& type_names,
                const std::function<std::vector<int32_t>(int64_t)>& worker_of) {
    for (int64_t g = 0; g < G; ++g) {
        if (status[g] == GS_OK) continue;
        const int64_t t0 = task_base[g], n = task_base[g + 1] - t0;
        const int32_t pos = aux[g] >= 0 ? (aux[g] & 0xffffff) : aux[g];
        const int32_t ty = aux[g] >= 0 ? (aux[g] >> 24) : 0;
        auto ident = [&](int64_t q) { return task_id.empty() ? q : task_id[t0 + q]; };
        switch (status[g]) {
            case GS_NO_WORKER: raise(TBSIM_E_RUNTIME, "no worker can run task type " + type_name_of(type_names, ty));
            case GS_TOO_LARGE:
                raise(TBSIM_E_INVALID_ARGUMENT, "task " + std::to_string(ident(pos)) +
                                                    " exceeds the device simulator's limits (ability/efficiency "
                                                    "beyond its int32 queue keys, or 2^24 successor entries)");
            case GS_DEGENERATE_TIME:
                raise(TBSIM_E_RUNTIME, "event of task " + std::to_string(ident(pos)) +
                                           " would fire at the current time (transfer/exec below FP64 resolution)");
            case GS_STUCK: {
                const std::vector<int32_t> w = worker_of(g);
                const int64_t done = completed[g];
                std::string msg = "simulation stuck with " + std::to_string(n - done) + " tasks unfinished:";
                int64_t listed = 0;
                for (int64_t i = 0; i < n && i < static_cast<int64_t>(w.size()) && listed < 20; ++i)
                    if (w[i] < 0) { msg += " " + std::to_string(ident(i)); ++listed; }
                if (listed < n - done) msg += " ...";
                raise(TBSIM_E_RUNTIME, msg);
            }
            default: raise(TBSIM_E_RUNTIME, "device simulator failed with status " + std::to_string(status[g]));
        }
    }
}

// Decodes and clears a deferred check (its copies are complete once its
// event is): compute_attributes errors first, then the simulation's.
void check_pending(tbsim_ctx* ctx, int set) {
    tbsim_ctx::Pending& pd = ctx->pend[set];
    if (!pd.active) return;
    cuda_check(cudaEventSynchronize(pd.done), "cudaEventSynchronize(pending)");
    if (pd.copies_done) cuda_check(cudaEventSynchronize(pd.copies_done), "cudaEventSynchronize(copies)");
    pd.active = false;
    if (pd.info) attr_errors(pd.info, pd.G, pd.task_base, pd.type_names, TBSIM_ATTR_ALL, nullptr);
    sim_errors(pd.G, pd.status, pd.aux, pd.completed, pd.task_base, pd.task_id, pd.type_names, [&](int64_t g) {
        const int64_t t0 = pd.task_base[g], n = pd.task_base[g + 1] - t0;
        std::vector<int32_t> w(static_cast<size_t>(n));
        if (n && pd.worker_out) {
            if (pd.worker_on_device) cudaMemcpy(w.data(), pd.worker_out + t0, n * 4, cudaMemcpyDeviceToHost);
            else std::copy(pd.worker_out + t0, pd.worker_out + t0 + n, w.begin());
        }
        return w;
    });
}

// deferred = -1: statuses are checked here (one host round trip after the
// simulation); 0/1: the result set of an asynchronous call -- queue
// overflows are re-run on the device (list built on the device) and the
// statuses are checked later (check_pending).
void run_simulation(tbsim_ctx* ctx, const tbsim_batch* b, SimParams p, int32_t max_workers, const SimKeys& keys,
                    const int32_t* pof_host = nullptr, const std::vector<DevPlatform>* hp = nullptr,
                    AttrRun* attrs_first = nullptr, int deferred = -1, const int32_t* worker_out = nullptr,
                    bool worker_on_device = false) {
    const DevBatch& d = b->d;
    const int64_t G = d.G;
    if (G == 0) return;
    // packed simulation graph (built once per batch) + this call's pop keys
    ensure_packed(ctx, const_cast<tbsim_batch*>(b));
    p.hdr = b->hdr;
    p.adj = b->adj;
    p.class_bytes = b->dict;
    {  // this call's transfer times per (platform, byte class, from, to)
        const int32_t np = hp ? static_cast<int32_t>(hp->size()) : 1;
        const int64_t nx = static_cast<int64_t>(np) * kByteClasses * p.max_nodes * p.max_nodes;
        double* xtab = ctx->buf("s_xtab").as<double>(nx);
        ctx->begin("k_xfer_table");
        k_xfer_table<<<static_cast<int>(std::min<int64_t>((nx + 255) / 256, 64)), 256, 0, ctx->stream>>>(
            p.platforms, np, b->dict, p.max_nodes, xtab);
        ctx->end("k_xfer_table");
        p.xtab = xtab;
    }
    p.log = ctx->buf("s_log").as<SimLog>(std::max<int64_t>(d.T, 1));
    p.n_disp = ctx->buf("s_ndisp").as<int32_t>(G);
    if (d.T > 0) {
        const int grid = static_cast<int>(std::min<int64_t>((d.T + 255) / 256, 16LL * ctx->n_sms));
        ctx->begin("k_sim_keys");
        k_sim_keys<<<grid, 256, 0, ctx->stream>>>(d, keys.ability, keys.efficiency, keys.prio, p.policy, b->hdr);
        ctx->end("k_sim_keys");
    }
    p.graph_list = nullptr;
    p.qcap = 0;
    int64_t n_lo = G;  // graphs of the first launch (<= 32 workers when split)
    int32_t max_lo = max_workers;
    if (pof_host && hp && hp->size() > 1 && G >= 2 * ctx->n_sms) {
        bool mixed = false;
        for (const auto& pl : *hp) mixed = mixed || pl.n_workers != (*hp)[0].n_workers;
        if (mixed) {
            std::vector<int32_t> order(G);
            for (int64_t g = 0; g < G; ++g) order[g] = static_cast<int32_t>(g);
            std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
                return (*hp)[pof_host[x]].n_workers < (*hp)[pof_host[y]].n_workers;
            });
            int32_t* d_list = ctx->buf("s_order").as<int32_t>(G);
            cuda_check(cudaMemcpyAsync(d_list, order.data(), G * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D order");
            p.graph_list = d_list;
            // graphs on <= 32 workers (a prefix of the order) run in their
            // own launch of the one-worker-per-lane kernel: ~2x the warps
            // per SM of the two-worker kernel the > 32-worker graphs need
            if (max_workers > 32) {
                int64_t lo = 0;
                while (lo < G && (*hp)[pof_host[order[lo]]].n_workers <= 32) ++lo;
                if (lo >= ctx->n_sms && G - lo >= ctx->n_sms) {
                    n_lo = lo;
                    max_lo = (*hp)[pof_host[order[lo - 1]]].n_workers;
                }
            }
        }
    }
    if (n_lo < G) {
        launch_sim(ctx, p, max_lo, n_lo);
        p.graph_list += n_lo;
        p.qcap = 0;  // (set by the first launch; 0 = choose)
        launch_sim(ctx, p, max_workers, G - n_lo);
    } else {
        launch_sim(ctx, p, max_workers, G);
    }
    p.graph_list = nullptr;
    if (deferred >= 0) {
        int32_t* list = ctx->buf("s_rerun").as<int32_t>(G);
        int64_t* count = ctx->buf("s_rerun_n").as<int64_t>(1);
        k_sim_collect_reruns<<<1, 1024, 0, ctx->stream>>>(G, p.status, list, count);
        SimParams q = p;
        q.graph_list = list;
        q.qcap = std::max<int32_t>(b->d.max_n, 1);
        q.n_items_dev = count;
        // sized for a few reruns; the launch reads the real count on the device
        launch_sim(ctx, q, max_workers, std::min<int64_t>(G, 4LL * ctx->n_sms), "k_simulate_rerun");
        if (d.T > 0) {
            const int grid = static_cast<int>(std::min<int64_t>((d.T + 255) / 256, 16LL * ctx->n_sms));
            ctx->begin("k_sim_scatter");
            k_sim_scatter<<<grid, 256, 0, ctx->stream>>>(d, p.log, p.n_disp, p.worker, p.start_ms, p.end_ms);
            ctx->end("k_sim_scatter");
        }
        const std::string sfx = deferred ? "_a1" : "_a0";
        tbsim_ctx::Pending& pd = ctx->pend[deferred];
        int32_t* st = ctx->pin<int32_t>("p_status" + sfx, static_cast<size_t>(2 * G));
        int64_t* done = ctx->pin<int64_t>("p_done" + sfx, static_cast<size_t>(G));
        cuda_check(cudaMemcpyAsync(st, p.status, G * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H status");
        cuda_check(cudaMemcpyAsync(st + G, p.status_aux, G * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H aux");
        cuda_check(cudaMemcpyAsync(done, p.completed, G * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H completed");
        if (!pd.done) cuda_check(cudaEventCreateWithFlags(&pd.done, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventRecord(pd.done, ctx->stream), "cudaEventRecord(pending)");
        pd.active = true;
        pd.G = G;
        pd.info = attrs_first ? attrs_first->pinned : nullptr;
        pd.status = st;
        pd.aux = st + G;
        pd.completed = done;
        pd.task_base = b->task_base;
        pd.task_id = b->task_id;
        pd.type_names = b->type_names;
        pd.worker_out = worker_out;
        pd.worker_on_device = worker_on_device;
        pd.copies_done = worker_on_device ? nullptr : ctx->set_free[deferred];
        return;
    }
    std::vector<int32_t> status(G), aux(G);
    cuda_check(cudaMemcpyAsync(status.data(), p.status, G * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H status");
    cuda_check(cudaMemcpyAsync(aux.data(), p.status_aux, G * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H aux");
    ctx->sync();
    if (attrs_first) {
        attrs_first->fetch(G);
        attr_errors(b, attrs_first->info, TBSIM_ATTR_ALL, nullptr);
    }
    std::vector<int32_t> rerun;
    for (int64_t g = 0; g < G; ++g)
        if (status[g] == GS_QUEUE_OVERFLOW) rerun.push_back(static_cast<int32_t>(g));
    if (!rerun.empty()) {
        int32_t* d_list = ctx->buf("s_rerun").as<int32_t>(rerun.size());
        cuda_check(cudaMemcpyAsync(d_list, rerun.data(), rerun.size() * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D rerun");
        // reset the reruns' regulator state is not needed: a graph that
        // overflowed never wrote its state back (status checked first)
        SimParams q = p;
        q.graph_list = d_list;
        q.qcap = std::max<int32_t>(b->d.max_n, 1);
        launch_sim(ctx, q, max_workers, static_cast<int64_t>(rerun.size()), "k_simulate_rerun");
        cuda_check(cudaMemcpyAsync(status.data(), p.status, G * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H status");
        cuda_check(cudaMemcpyAsync(aux.data(), p.status_aux, G * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H aux");
        ctx->sync();
    }
    if (d.T > 0) {  // dispatch logs -> per-task worker/start/end
        const int grid = static_cast<int>(std::min<int64_t>((d.T + 255) / 256, 16LL * ctx->n_sms));
        ctx->begin("k_sim_scatter");
        k_sim_scatter<<<grid, 256, 0, ctx->stream>>>(d, p.log, p.n_disp, p.worker, p.start_ms, p.end_ms);
        ctx->end("k_sim_scatter");
    }
    std::vector<int64_t> completed(G);
    if (std::any_of(status.begin(), status.end(), [](int32_t x) { return x != GS_OK; }))
        cuda_check(cudaMemcpy(completed.data(), p.completed, G * 8, cudaMemcpyDeviceToHost), "D2H completed");
    sim_errors(G, status.data(), aux.data(), completed.data(), b->task_base, b->task_id, b->type_names, [&](int64_t g) {
        const int64_t t0 = b->task_base[g], n = b->task_base[g + 1] - t0;
        std::vector<int32_t> w(static_cast<size_t>(n));
        if (n) cudaMemcpy(w.data(), p.worker + t0, n * 4, cudaMemcpyDeviceToHost);
        return w;
    });
}

struct SimStage {
    std::vector<std::pair<void*, std::pair<const void*, size_t>>> copies;
};

template <typename T>
T* sim_out_ptr(tbsim_ctx* ctx, SimStage& st, const char* name, T* host, size_t count, bool on_device, bool upload = false) {
    if (!host) return nullptr;
    if (on_device) return host;
    T* dev = ctx->buf(name).as<T>(count);
    if (upload) cuda_check(cudaMemcpyAsync(dev, host, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    st.copies.push_back({host, {dev, count * sizeof(T)}});
    return dev;
}

template <typename T>
T* scratch_if_null(tbsim_ctx* ctx, const char* name, T* p, size_t count) {
    return p ? p : ctx->buf(name).as<T>(count);
}

int32_t upload_platforms(tbsim_ctx* ctx, const tbsim_batch* b, const tbsim_platform_desc* platforms, int32_t n_platforms,
                         DevPlatform** d_out, std::vector<DevPlatform>& host, int32_t* max_nodes) {
    if (n_platforms < 1) raise(TBSIM_E_INVALID_ARGUMENT, "need at least one platform");
    int32_t maxw = 0;
    *max_nodes = 1;
    host.clear();
    for (int i = 0; i < n_platforms; ++i) {
        host.push_back(to_dev_platform(platforms[i], b->d.n_types));
        maxw = std::max(maxw, platforms[i].n_workers);
        *max_nodes = std::max(*max_nodes, platforms[i].n_nodes);
    }
    *d_out = ctx->buf("platforms").as<DevPlatform>(n_platforms);
    cuda_check(cudaMemcpyAsync(*d_out, host.data(), host.size() * sizeof(DevPlatform), cudaMemcpyHostToDevice, ctx->stream),
               "H2D platforms");
    return maxw;
}

void check_reg(const tbsim_regulator_cfg& r) {
    if (r.slope_samples < 0 || r.slope_samples > TBSIM_MAX_SLOPE_SAMPLES)
        raise(TBSIM_E_INVALID_ARGUMENT, "slope_samples must be in [0, " + std::to_string(TBSIM_MAX_SLOPE_SAMPLES) +
                                             "] on the device");
}

}  // namespace

extern "C" tbsim_status tbsim_simulate(tbsim_ctx* ctx, const tbsim_batch* b, const tbsim_platform_desc* platforms,
                                       int32_t n_platforms, const int32_t* platform_of, int32_t policy,
                                       const tbsim_regulator_cfg* reg, const tbsim_attr_in* attrs, tbsim_sim_out* out) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        wait_batch(ctx, b);
        if (policy < 0 || policy > TBSIM_POLICY_INSPIRIT) raise(TBSIM_E_RUNTIME, "unknown policy id");
        const DevBatch& d = b->d;
        const int64_t T = d.T, G = d.G;
        if (!reg) raise(TBSIM_E_INVALID_ARGUMENT, "tbsim_simulate needs a regulator config per graph");
        for (int64_t g = 0; g < G; ++g) check_reg(reg[g]);
        std::vector<DevPlatform> hp;
        DevPlatform* d_pf = nullptr;
        int32_t max_nodes = 1;
        const int32_t maxw = upload_platforms(ctx, b, platforms, n_platforms, &d_pf, hp, &max_nodes);
        SimStage st;
        const bool dev = out->on_device != 0;
        SimParams p{};
        p.b = d;
        p.platforms = d_pf;
        p.max_nodes = max_nodes;
        p.n_types = d.n_types;
        int32_t ring = 1;
        for (int64_t g = 0; g < G; ++g) ring = std::max(ring, reg[g].slope_samples);
        if (out->reg_state && !dev)
            for (int64_t g = 0; g < G; ++g) {
                if (out->reg_state[g].n_samples < 0 || out->reg_state[g].n_samples > TBSIM_MAX_SLOPE_SAMPLES)
                    raise(TBSIM_E_INVALID_ARGUMENT, "regulator state holds too many samples");
                ring = std::max(ring, out->reg_state[g].n_samples);
            }
        if (out->reg_state && dev) ring = TBSIM_MAX_SLOPE_SAMPLES;
        p.ring = pow2_at_least(ring);
        if (platform_of) {
            for (int64_t g = 0; g < G && !dev; ++g)
                if (platform_of[g] < 0 || platform_of[g] >= n_platforms) raise(TBSIM_E_INVALID_ARGUMENT, "platform index out of range");
            int32_t* dpo = ctx->buf("s_pof").as<int32_t>(G);
            cuda_check(cudaMemcpyAsync(dpo, platform_of, G * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D pof");
            p.platform_of = dpo;
        }
        p.policy = policy;
        tbsim_regulator_cfg* d_reg = ctx->buf("s_reg").as<tbsim_regulator_cfg>(G);
        cuda_check(cudaMemcpyAsync(d_reg, reg, G * sizeof(tbsim_regulator_cfg), cudaMemcpyHostToDevice, ctx->stream), "H2D reg");
        p.reg = d_reg;
        p.median_stride = 1;
        auto up_attr = [&](const int64_t* a, const char* name) -> const int64_t* {
            if (!a) return nullptr;
            if (attrs->on_device) return a;
            int64_t* dv = ctx->buf(name).as<int64_t>(T);
            cuda_check(cudaMemcpyAsync(dv, a, T * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D attrs");
            return dv;
        };
        SimKeys keys;
        if (attrs) {
            keys.ability = up_attr(attrs->ability, "s_ab");
            keys.efficiency = up_attr(attrs->efficiency, "s_ef");
            keys.prio = up_attr(attrs->static_priority, "s_pr");
        }
        p.worker = scratch_if_null(ctx, "s_worker", sim_out_ptr(ctx, st, "s_worker", out->worker, T, dev), T);
        p.start_ms = scratch_if_null(ctx, "s_start", sim_out_ptr(ctx, st, "s_start", out->start_ms, T, dev), T);
        p.end_ms = scratch_if_null(ctx, "s_end", sim_out_ptr(ctx, st, "s_end", out->end_ms, T, dev), T);
        p.makespan = scratch_if_null(ctx, "s_mk", sim_out_ptr(ctx, st, "s_mk", out->makespan_ms, G, dev), G);
        p.completed = scratch_if_null(ctx, "s_done", sim_out_ptr(ctx, st, "s_done", out->completed, G, dev), G);
        p.pop_counts = sim_out_ptr(ctx, st, "s_pops", out->pop_mode_counts, 3 * G, dev);
        p.reg_state = sim_out_ptr(ctx, st, "s_rstate", out->reg_state, G, dev, /*upload=*/true);
        p.push_time = sim_out_ptr(ctx, st, "s_pusht", out->push_time, T, dev);
        p.push_task = sim_out_ptr(ctx, st, "s_pushk", out->push_task, T, dev);
        p.pop_time = sim_out_ptr(ctx, st, "s_popt", out->pop_time, T, dev);
        p.pop_task = sim_out_ptr(ctx, st, "s_popk", out->pop_task, T, dev);
        p.pop_worker = sim_out_ptr(ctx, st, "s_popw", out->pop_worker, T, dev);
        p.sample_time = sim_out_ptr(ctx, st, "s_samt", out->sample_time, 2 * T, dev);
        p.sample_nready = sim_out_ptr(ctx, st, "s_samn", out->sample_nready, 2 * T, dev);
        if (!(p.push_time && p.push_task && p.pop_time && p.pop_task && p.pop_worker && p.sample_time && p.sample_nready)) {
            p.push_time = nullptr; p.push_task = nullptr; p.pop_time = nullptr; p.pop_task = nullptr;
            p.pop_worker = nullptr; p.sample_time = nullptr; p.sample_nready = nullptr;
        }
        p.status = ctx->buf("s_status").as<int32_t>(G);
        p.status_aux = ctx->buf("s_aux").as<int32_t>(G);
        run_simulation(ctx, b, p, maxw, keys, platform_of, &hp);
        for (const auto& c : st.copies)
            cuda_check(cudaMemcpyAsync(c.first, c.second.first, c.second.second, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ctx->sync();
        ctx->collect_timing();
    });
}

extern "C" tbsim_status tbsim_schedule(tbsim_ctx* ctx, const tbsim_batch* b, const tbsim_platform_desc* platforms,
                                       int32_t n_platforms, const int32_t* platform_of, int32_t policy,
                                       int32_t priority_kind, tbsim_attr_out* attr_out, tbsim_sim_out* out) {
    return guarded([&] {
        DeviceScope dev_scope(ctx->device);
        wait_batch(ctx, b);
        if (policy < 0 || policy > TBSIM_POLICY_INSPIRIT) raise(TBSIM_E_RUNTIME, "unknown policy id");
        const DevBatch& d = b->d;
        const int64_t T = d.T, G = d.G;
        // host-bound outputs: staged in buffer set `set`, copied on the
        // download stream when results are asynchronous
        const bool async = ctx->async_results && !out->on_device;
        const int set = async ? ctx->parity : 0;
        if (async) {
            ctx->parity ^= 1;
            // this set's previous call: its deferred checks (raised here if
            // it failed), and its copies before the staging is rewritten
            check_pending(ctx, set);
            if (ctx->set_pending[set])
                cuda_check(cudaStreamWaitEvent(ctx->stream, ctx->set_free[set], 0), "cudaStreamWaitEvent");
        }
        const std::string sfx = set ? "_1" : "";
        auto nm = [&](const char* base) { return std::string(base) + sfx; };
        std::vector<DevPlatform> hp;
        DevPlatform* d_pf = nullptr;
        int32_t max_nodes = 1;
        const int32_t maxw = upload_platforms(ctx, b, platforms, n_platforms, &d_pf, hp, &max_nodes);
        // cost tables of the platforms, one per platform (compute_attributes
        // runs on platform.costs, src/bench.cpp:104)
        std::vector<DevCosts> hc;
        for (const auto& p : hp) hc.push_back(p.costs);
        DevCosts* d_costs = ctx->buf("costs_pf").as<DevCosts>(hc.size());
        cuda_check(cudaMemcpyAsync(d_costs, hc.data(), hc.size() * sizeof(DevCosts), cudaMemcpyHostToDevice, ctx->stream),
                   "H2D costs");
        int32_t* d_pof = nullptr;
        if (platform_of) {
            d_pof = ctx->buf("s_pof").as<int32_t>(G);
            cuda_check(cudaMemcpyAsync(d_pof, platform_of, G * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D pof");
        }
        // ---- attributes (compute_attributes on every graph)
        tbsim_attr_out dummy{};
        tbsim_attr_out* ao = attr_out ? attr_out : &dummy;
        const bool adev = ao->on_device != 0;
        OutStage ast;
        AttrOutDev o{};
        o.ability = scratch_if_null(ctx, nm("f_ab").c_str(), stage_out(ctx, ast, nm("f_ab").c_str(), ao->ability, T, adev), T);
        o.efficiency = scratch_if_null(ctx, nm("f_ef").c_str(), stage_out(ctx, ast, nm("f_ef").c_str(), ao->efficiency, T, adev), T);
        o.static_priority = scratch_if_null(ctx, nm("f_pr").c_str(), stage_out(ctx, ast, nm("f_pr").c_str(), ao->static_priority, T, adev), T);
        o.unit_time_ms = scratch_if_null(ctx, nm("f_ut").c_str(), stage_out(ctx, ast, nm("f_ut").c_str(), ao->unit_time_ms, G, adev), G);
        o.w0_ms = stage_out(ctx, ast, nm("f_w0").c_str(), ao->w0_ms, G, adev);
        o.best_score = stage_out(ctx, ast, nm("f_bs").c_str(), ao->best_score, G, adev);
        o.w0_score = stage_out(ctx, ast, nm("f_ws").c_str(), ao->w0_score, G, adev);
        o.evaluations = stage_out(ctx, ast, nm("f_ev").c_str(), ao->evaluations, G, adev);
        AttrRun run;
        if (async) run.pin_sfx = set ? "_a1" : "_a0";
        run_attributes(ctx, b, d_costs, d_pof, SWEEP_CALIBRATE, nullptr, priority_kind == TBSIM_PRIO_UPWARD_RANK, true,
                       o, priority_kind, true, run);
        // no host round trip here: compute_attributes' errors are raised
        // (first, as the reference's bench cell would) at the simulation's
        // status check
        // ---- default_regulator_config + simulate
        SimStage st;
        const bool dev = out->on_device != 0;
        SimParams p{};
        p.b = d;
        p.platforms = d_pf;
        p.platform_of = d_pof;
        p.max_nodes = max_nodes;
        p.n_types = d.n_types;
        p.ring = 8;  // default_regulator_config: slope_samples = 8
        if (out->reg_state) {
            if (out->on_device) p.ring = TBSIM_MAX_SLOPE_SAMPLES;
            else
                for (int64_t g = 0; g < G; ++g) p.ring = std::max(p.ring, pow2_at_least(out->reg_state[g].n_samples));
        }
        p.policy = policy;
        p.reg = nullptr;
        p.median = run.s.median;
        p.median_stride = 1;
        SimKeys keys;
        keys.ability = o.ability;
        keys.efficiency = o.efficiency;
        keys.prio = o.static_priority;
        p.worker = scratch_if_null(ctx, nm("s_worker").c_str(), sim_out_ptr(ctx, st, nm("s_worker").c_str(), out->worker, T, dev), T);
        p.start_ms = scratch_if_null(ctx, nm("s_start").c_str(), sim_out_ptr(ctx, st, nm("s_start").c_str(), out->start_ms, T, dev), T);
        p.end_ms = scratch_if_null(ctx, nm("s_end").c_str(), sim_out_ptr(ctx, st, nm("s_end").c_str(), out->end_ms, T, dev), T);
        p.makespan = scratch_if_null(ctx, nm("s_mk").c_str(), sim_out_ptr(ctx, st, nm("s_mk").c_str(), out->makespan_ms, G, dev), G);
        p.completed = scratch_if_null(ctx, nm("s_done").c_str(), sim_out_ptr(ctx, st, nm("s_done").c_str(), out->completed, G, dev), G);
        p.pop_counts = sim_out_ptr(ctx, st, nm("s_pops").c_str(), out->pop_mode_counts, 3 * G, dev);
        p.reg_state = sim_out_ptr(ctx, st, nm("s_rstate").c_str(), out->reg_state, G, dev, true);
        p.status = ctx->buf("s_status").as<int32_t>(G);
        p.status_aux = ctx->buf("s_aux").as<int32_t>(G);
        // asynchronous results: no host round trip in the call (deferred checks)
        run_simulation(ctx, b, p, maxw, keys, platform_of, &hp, &run, async ? set : -1, out->worker, dev);
        cudaStream_t dl = ctx->stream;
        if (async) {  // the copies wait for this call's kernels, not the next call's
            cudaEvent_t done = ctx->set_free[set];
            cuda_check(cudaEventRecord(done, ctx->stream), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(ctx->download, done, 0), "cudaStreamWaitEvent");
            dl = ctx->download;
        }
        for (const auto& c : ast.copies)
            cuda_check(cudaMemcpyAsync(c.first, c.second.first, c.second.second, cudaMemcpyDeviceToHost, dl), "D2H");
        for (const auto& c : st.copies)
            cuda_check(cudaMemcpyAsync(c.first, c.second.first, c.second.second, cudaMemcpyDeviceToHost, dl), "D2H");
        if (async) {
            cuda_check(cudaEventRecord(ctx->set_free[set], ctx->download), "cudaEventRecord");
            ctx->set_pending[set] = true;
        }
        // asynchronous results: the statuses were checked after the
        // simulation; what is left on the compute stream (the dispatch-log
        // scatter) overlaps the caller's next call instead of a host wait
        if (!async || ctx->timing) ctx->sync();
        ctx->collect_timing();
    });
}

extern "C" tbsim_status tbsim_default_regulator_config(int32_t n_workers, double median, tbsim_regulator_cfg* out) {
    return guarded([&] {
        // default_regulator_config, src/policies.cpp:139-151 (shared with the
        // device's default in simulate.cu)
        *out = tbsim_rules::default_config(n_workers, median);
    });
}

// --------------------------------------------------------------- generators

struct tbsim_hostbatch {
    tbsim_host::HostBatch hb;
};

extern "C" {

tbsim_status tbsim_hostbatch_new(tbsim_hostbatch** out) {
    return guarded([&] { *out = new tbsim_hostbatch(); });
}
tbsim_status tbsim_hostbatch_free(tbsim_hostbatch* hb) {
    return guarded([&] { delete hb; });
}

tbsim_status tbsim_hostbatch_add_layered(tbsim_hostbatch* hb, int32_t n_tasks, int32_t n_layers, double p,
                                         const uint64_t* seeds, int64_t n_seeds, int32_t n_threads) {
    return guarded([&] {
        std::vector<tbsim_host::GraphCSR> gs(n_seeds);
        int nt = n_threads > 0 ? n_threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        nt = static_cast<int>(std::min<int64_t>(nt, std::max<int64_t>(n_seeds, 1)));
        std::vector<std::thread> pool;
        std::exception_ptr err;
        std::mutex mu;
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                try {
                    for (int64_t i = t; i < n_seeds; i += nt) gs[i] = tbsim_host::gen_layered(n_tasks, n_layers, p, seeds[i]);
                } catch (...) {
                    std::lock_guard<std::mutex> lk(mu);
                    err = std::current_exception();
                }
            });
        for (auto& th : pool) th.join();
        if (err) std::rethrow_exception(err);
        hb->hb.append_many(std::move(gs));
    });
}

tbsim_status tbsim_hostbatch_add_cholesky(tbsim_hostbatch* hb, int32_t nb, int64_t bytes) {
    return guarded([&] { hb->hb.append(tbsim_host::gen_cholesky(nb, bytes)); });
}
tbsim_status tbsim_hostbatch_add_lu(tbsim_hostbatch* hb, int32_t nb, int64_t bytes) {
    return guarded([&] { hb->hb.append(tbsim_host::gen_lu(nb, bytes)); });
}
tbsim_status tbsim_hostbatch_add_qr(tbsim_hostbatch* hb, int32_t nb, int64_t bytes) {
    return guarded([&] { hb->hb.append(tbsim_host::gen_qr(nb, bytes)); });
}

tbsim_status tbsim_hostbatch_add_csr(tbsim_hostbatch* hb, int32_t n, const int32_t* dep_off, const int32_t* dep,
                                     const int32_t* in_off, const int32_t* in, const int32_t* out_off,
                                     const int32_t* out, const int32_t* type, int32_t n_handles,
                                     const int64_t* handle_bytes, const int64_t* task_id) {
    return guarded([&] {
        tbsim_host::GraphCSR g;
        g.dep_off.assign(dep_off, dep_off + n + 1);
        g.dep.assign(dep, dep + dep_off[n]);
        g.in_off.assign(in_off, in_off + n + 1);
        g.in.assign(in, in + in_off[n]);
        g.out_off.assign(out_off, out_off + n + 1);
        g.out.assign(out, out + out_off[n]);
        g.type.assign(type, type + n);
        g.handle_bytes.assign(handle_bytes, handle_bytes + n_handles);
        hb->hb.append(g, task_id);
    });
}

tbsim_status tbsim_hostbatch_desc(const tbsim_hostbatch* hb, tbsim_batch_desc* out) {
    return guarded([&] { *out = const_cast<tbsim_hostbatch*>(hb)->hb.desc(); });
}

tbsim_status tbsim_hostbatch_set_type_names(tbsim_hostbatch* hb, int32_t n, const char* const* names) {
    return guarded([&] {
        if (n < 0 || n > kMaxTypes) raise(TBSIM_E_INVALID_ARGUMENT, "more than 64 task types");
        std::vector<std::string> v;
        for (int32_t i = 0; i < n; ++i) v.push_back(names[i] ? names[i] : "type" + std::to_string(i));
        hb->hb.set_type_names(v);
    });
}

tbsim_status tbsim_hostbatch_save(tbsim_hostbatch* hb, const char* path) {
    return guarded([&] { hb->hb.save(path); });
}

tbsim_status tbsim_batch_desc_save(const tbsim_batch_desc* desc, const char* path) {
    return guarded([&] { tbsim_host::save_csr_cache(*desc, path); });
}

tbsim_status tbsim_hostbatch_load(const char* path, tbsim_hostbatch** out) {
    return guarded([&] {
        auto h = std::make_unique<tbsim_hostbatch>();
        h->hb.load(path);
        *out = h.release();
    });
}

int32_t tbsim_type_count(void) { return tbsim_host::T_COUNT; }
const char* tbsim_type_name(int32_t id) {
    return id >= 0 && id < tbsim_host::T_COUNT ? tbsim_host::kTypeNames[id] : nullptr;
}

tbsim_status tbsim_default_costs(double* cpu, double* gpu) {
    return guarded([&] {
        // default_cost_table, src/platform.cpp:93-98 (GPU ms, CPU/GPU ratio);
        // QR rows are builder-chosen (no reference counterpart)
        struct Row { int32_t id; double gpu, ratio; };
        static const Row rows[] = {
            {tbsim_host::T_GEMM, 0.4, 10.0}, {tbsim_host::T_SYRK, 1.0, 10.0}, {tbsim_host::T_TRSM, 1.2, 10.0},
            {tbsim_host::T_POTRF, 2.0, 3.0}, {tbsim_host::T_GETRF, 2.0, 3.0}, {tbsim_host::T_STENCIL, 0.8, 5.0},
            {tbsim_host::T_LAYERK0, 0.5, 5.0}, {tbsim_host::T_LAYERK1, 1.0, 8.0}, {tbsim_host::T_LAYERK2, 2.0, 3.0},
            {tbsim_host::T_LAYERK3, 4.0, 6.0}, {tbsim_host::T_UNIT, 1.0, 1.0}, {tbsim_host::T_GEQRT, 2.0, 3.0},
            {tbsim_host::T_UNMQR, 0.8, 10.0}, {tbsim_host::T_TSQRT, 2.4, 3.0}, {tbsim_host::T_TSMQR, 0.8, 10.0}};
        for (int i = 0; i < tbsim_host::T_COUNT; ++i) cpu[i] = gpu[i] = 0.0;
        for (const Row& r : rows) {
            gpu[r.id] = r.gpu;
            cpu[r.id] = r.gpu * r.ratio;
        }
    });
}

}  // extern "C"
