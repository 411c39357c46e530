/*
 * tbsim_b200.h -- C-ABI of the B200-native INSPIRIT scheduling hot path.
 *
 * This is the drop-in boundary the C++ `tbsim` API (include/tbsim/*.hpp, the
 * same names and signatures as the reference's proj/include/tbsim/*.hpp) is
 * implemented on top of.  Every entry point replaces one reference function;
 * the replaced symbol is cited next to it (paths relative to
 * /root/reference/proj).  Plain pointers and sizes only -- no C++ or torch
 * types cross this line.
 *
 * Conventions
 *   - Every function returns a tbsim_status.  On failure a thread-local
 *     message is available from tbsim_last_error(); the status says which C++
 *     exception type the reference throws for the same condition, and the
 *     message text is the reference's text (the C++ shim re-throws both).
 *   - Graphs travel as a *batch* in CSR form (tbsim_batch_desc).  Positions
 *     are local to their graph (0..n_g-1), exactly the reference's "task
 *     position" (index into TaskGraph::tasks, src/taskgraph.cpp:11-43).
 *   - Host buffers are caller-owned.  Device buffers are owned by the context
 *     (tbsim_ctx) or by the caller when TBSIM_OUT_DEVICE is set.
 *   - A context is bound to one CUDA device and one stream; use one context
 *     per calling thread.  Every call makes the context's device current for
 *     its duration and restores the caller's current device before it
 *     returns, so one host thread may drive contexts on several GPUs.  There is no CPU fallback: every compute entry point
 *     runs on the GPU and fails with TBSIM_E_CUDA when no device is present.
 */
#ifndef TBSIM_B200_H
#define TBSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TBSIM_ABI_VERSION 1

typedef enum tbsim_status {
    TBSIM_OK = 0,
    TBSIM_E_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    TBSIM_E_RUNTIME = 2,          /* std::runtime_error    */
    TBSIM_E_LOGIC = 3,            /* std::logic_error      */
    TBSIM_E_OUT_OF_RANGE = 4,     /* std::out_of_range     */
    TBSIM_E_CUDA = 5              /* device/driver failure (no reference twin) */
} tbsim_status;

/* Thread-local message of the last failing call on this thread. */
const char* tbsim_last_error(void);
int tbsim_abi_version(void);

/* ------------------------------------------------------------------------
 * Graph batch (CSR).  G graphs; totals T tasks, E dependency entries,
 * H handles, I input refs, O output refs.
 *
 *   task_base[g] .. task_base[g+1]      tasks of graph g (global index)
 *   dep_off[task_base[g] + g + i]       local CSR offset of task i's deps
 *                                       (n_g + 1 entries per graph, first 0)
 *   dep[edge_base[g] + k]               local position of a predecessor, in
 *                                       TaskNode::deps order (multi-edges kept)
 *   in_off / in, out_off / out          same layout for TaskNode::inputs /
 *                                       outputs, values are local handle
 *                                       positions (index into TaskGraph::handles)
 *   type[t]                             dense task-type id (index into the
 *                                       cost table / type-name list)
 *   handle_bytes[handle_base[g] + h]    DataHandle::bytes
 *   task_id[t]                          TaskNode::id (trace/error text); may
 *                                       be NULL, then ids == positions
 *   type_names[type]                    type strings for error texts (may be
 *                                       NULL, then "type<k>" is printed)
 * ------------------------------------------------------------------------ */
typedef struct tbsim_batch_desc {
    int64_t n_graphs;
    const int64_t* task_base;   /* [G+1] */
    const int64_t* edge_base;   /* [G+1] */
    const int64_t* handle_base; /* [G+1] */
    const int64_t* in_base;     /* [G+1] */
    const int64_t* out_base;    /* [G+1] */
    const int32_t* dep_off;     /* [T+G] */
    const int32_t* dep;         /* [E]   */
    const int32_t* in_off;      /* [T+G] */
    const int32_t* in;          /* [I]   */
    const int32_t* out_off;     /* [T+G] */
    const int32_t* out;         /* [O]   */
    const int32_t* type;        /* [T]   */
    const int64_t* handle_bytes;/* [H]   */
    const int64_t* task_id;     /* [T] or NULL */
    int32_t n_type_names;
    const char* const* type_names; /* [n_type_names] or NULL */
} tbsim_batch_desc;

/* Cost table (reference: CostTable, include/tbsim/platform.hpp:23-47).
 * An entry is present iff its value is > 0 (CostTable::set rejects
 * non-positive values, src/platform.cpp:15-19). */
typedef struct tbsim_costs {
    int32_t n_types;
    const double* cpu_ms; /* [n_types] */
    const double* gpu_ms; /* [n_types] */
} tbsim_costs;

/* Machine model (reference: Platform, include/tbsim/platform.hpp:51-63).
 * kind: 0 = Cpu, 1 = Gpu.  bandwidth is row-major [from][to], bytes/ms. */
typedef struct tbsim_platform_desc {
    int32_t n_workers;
    const int32_t* kind;        /* [n_workers] */
    const int32_t* memory_node; /* [n_workers] */
    int32_t n_nodes;
    double latency_ms;
    const double* bandwidth;    /* [n_nodes * n_nodes] */
    tbsim_costs costs;
} tbsim_platform_desc;

/* ------------------------------------------------------------------------
 * Context
 * ------------------------------------------------------------------------ */
typedef struct tbsim_ctx tbsim_ctx;

tbsim_status tbsim_ctx_create(int device, tbsim_ctx** out);
tbsim_status tbsim_ctx_destroy(tbsim_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream()). NULL
 * restores the context's own stream. */
tbsim_status tbsim_ctx_set_stream(tbsim_ctx* ctx, void* cuda_stream);
/* Stream for batch uploads (H2D copies + successor ingest).  When set and
 * different from the compute stream, tbsim_batch_upload returns at once and
 * every compute call on the batch waits for its copies on the device, so the
 * next batch's upload overlaps the current batch's kernels.  Freed batch
 * memory is reused by a later upload only after the compute stream has
 * finished with it.  NULL: uploads run on the compute stream. */
tbsim_status tbsim_ctx_set_upload_stream(tbsim_ctx* ctx, void* cuda_stream);
tbsim_status tbsim_ctx_synchronize(tbsim_ctx* ctx);
/* Asynchronous results: tbsim_schedule calls with host output arrays return
 * once the results' device-to-host copies are queued on the context's
 * download stream (overlapping the next call's kernels); the host arrays are
 * valid after tbsim_ctx_synchronize.  Errors are still raised by the call.
 * Default off (results valid on return). */
tbsim_status tbsim_ctx_set_async_results(tbsim_ctx* ctx, int enable);
/* Single graphs with at least this many tasks (default 65536) take the
 * large-graph attribute path: ability by the HBM bitset closure, the
 * efficiency sweep pruned at the largest window. */
tbsim_status tbsim_ctx_set_large_graph_threshold(tbsim_ctx* ctx, int64_t n_tasks);
/* Sources per efficiency-sweep tile: 0 (default) picks the widest of
 * 256 (FP32-exact windows only)/128/64/32/16/8 whose distance window fits
 * shared memory; 8..256 forces it (tests of every tile shape; results do not
 * depend on it). */
tbsim_status tbsim_ctx_set_sweep_tile(tbsim_ctx* ctx, int32_t sources);
/* Number of kernels this context launched since creation (bench evidence). */
int64_t tbsim_ctx_launch_count(const tbsim_ctx* ctx);
/* Name/duration of the most recent launch of the dominant kernel, in ms,
 * measured with CUDA events on the launching stream (0 when not timed). */
tbsim_status tbsim_ctx_set_timing(tbsim_ctx* ctx, int enable);
tbsim_status tbsim_ctx_last_kernel_ms(const tbsim_ctx* ctx, const char* kernel,
                                      double* ms);
/* The efficiency sweep's inner-loop peak on this GPU: relaxations per
 * second of k_probe_relax (shared-memory rows + FP64 compare-select, no
 * graph) and of its FP32 twin (FMNMX), best of `repeats` launches on the
 * context's stream.  The sweep's roofline denominators (it is not
 * HBM-bound). */
tbsim_status tbsim_probe_sweep_peak(tbsim_ctx* ctx, int32_t repeats, double* fp64_per_s, double* fp32_per_s);
/* Launch shape of the last simulation: resident warps (DAGs in flight) per
 * SM, whether the per-warp state sat in shared memory, queue entries per
 * worker. */
tbsim_status tbsim_ctx_last_sim_shape(const tbsim_ctx* ctx, int32_t* warps_per_sm, int32_t* state_in_smem,
                                      int32_t* queue_capacity);
/* Relaxations (predecessor row x tile column) the last timed efficiency
 * sweep executed in FP64 and in FP32-exact windows -- the numerator of its
 * achieved rate. */
tbsim_status tbsim_ctx_last_sweep_relaxations(const tbsim_ctx* ctx, int64_t* fp64, int64_t* fp32);

/* ------------------------------------------------------------------------
 * Device-resident batch: CSR ingestion into HBM (one packed H2D copy, the
 * successor CSR is derived on the device).
 * ------------------------------------------------------------------------ */
typedef struct tbsim_batch tbsim_batch;

tbsim_status tbsim_batch_upload(tbsim_ctx* ctx, const tbsim_batch_desc* host,
                                tbsim_batch** out);
tbsim_status tbsim_batch_free(tbsim_ctx* ctx, tbsim_batch* b);
/* Bytes moved host->device by the last upload of this batch. */
int64_t tbsim_batch_h2d_bytes(const tbsim_batch* b);
/* generate_layered_dag (taskgraph.hpp:99-100) for every seed, generated on
 * the device (bit-identical to the host generator): only the seeds cross
 * PCIe.  Type ids follow tbsim_type_name(). */
tbsim_status tbsim_batch_generate_layered(tbsim_ctx* ctx, int32_t n_tasks, int32_t n_layers,
                                          double edge_prob, const uint64_t* seeds,
                                          int64_t n_seeds, tbsim_batch** out);

/* The tiled factorization DAGs built directly in HBM: `count` copies of
 * build_cholesky_dag / build_lu_dag (src/generators.cpp:30-142) or the tiled
 * QR, bit-identical to tbsim_hostbatch_add_cholesky / _lu / _qr (a thread
 * per task decodes its role and last writers in closed form). */
#define TBSIM_TILED_CHOLESKY 0
#define TBSIM_TILED_LU 1
#define TBSIM_TILED_QR 2
tbsim_status tbsim_batch_generate_tiled(tbsim_ctx* ctx, int32_t kind, int32_t nblocks,
                                        int64_t block_bytes, int64_t count, tbsim_batch** out);
/* Totals of a device batch: [G, T, E, H, I, O]. */
tbsim_status tbsim_batch_sizes(const tbsim_batch* b, int64_t* sizes6);
/* Copy a device batch back into caller buffers laid out like
 * tbsim_batch_desc; sizes from tbsim_batch_sizes, task_id/type_names unused. */
tbsim_status tbsim_batch_download(tbsim_ctx* ctx, const tbsim_batch* b, tbsim_batch_desc* host);

/* ------------------------------------------------------------------------
 * Attribute kernels (reference: include/tbsim/attributes.hpp).
 * ------------------------------------------------------------------------ */
enum {
    TBSIM_ATTR_ABILITY = 1 << 0,     /* compute_inspiring_ability     attributes.hpp:17 */
    TBSIM_ATTR_EFFICIENCY = 1 << 1,  /* compute_inspiring_efficiency  attributes.hpp:25 (window from unit_time_ms[g]) */
    TBSIM_ATTR_CALIBRATE = 1 << 2,   /* calibrate_unit_time           attributes.hpp:44 */
    TBSIM_ATTR_RANK = 1 << 3,        /* upward_rank_priority          attributes.hpp:49 */
    TBSIM_ATTR_DEPTH = 1 << 4,       /* depth_priority                attributes.hpp:53 */
    TBSIM_ATTR_LAYERS = 1 << 5,      /* topological_layers            taskgraph.hpp:71 */
    /* compute_attributes (attributes.hpp:64): ability + calibrate + efficiency
     * at the calibrated window + the selected static priority. */
    TBSIM_ATTR_ALL = 1 << 6
};

/* PriorityKind (attributes.hpp:55) */
enum { TBSIM_PRIO_UPWARD_RANK = 0, TBSIM_PRIO_DEPTH = 1, TBSIM_PRIO_ZERO = 2 };

/* Output pointers may be NULL when not requested.  Per-task arrays are [T]
 * (indexed by global task index), per-graph arrays are [G]. */
typedef struct tbsim_attr_out {
    int64_t* ability;
    int64_t* efficiency;
    int64_t* static_priority; /* rank, depth or zero per priority_kind */
    int64_t* depth;           /* TBSIM_ATTR_DEPTH */
    int32_t* layer;           /* TBSIM_ATTR_LAYERS */
    double* unit_time_ms;     /* [G] in for EFFICIENCY-only, out for CALIBRATE/ALL */
    /* CalibrationResult (attributes.hpp:32-38), [G] each */
    double* w0_ms;
    int64_t* best_score;
    int64_t* w0_score;
    int32_t* evaluations;
    int32_t on_device; /* 1: all pointers above are device pointers */
} tbsim_attr_out;

tbsim_status tbsim_attributes(tbsim_ctx* ctx, const tbsim_batch* b,
                              const tbsim_costs* costs, int32_t request,
                              int32_t priority_kind, tbsim_attr_out* out);

/* compute_attributes of ONE large graph sharded over `world` GPUs (SURVEY
 * §8(e), C4).  Every rank holds the whole graph; rank r computes the
 * descendant-set words of its share of the bit space (ability = the sum of
 * the ranks' partial counts) and the efficiency sweep of its share of the
 * sources.  Between the two calls the caller sums (all-reduces, e.g. NCCL
 * over NVLink) `ability_partial` [T] and `class_sums` [n_words] over the
 * ranks; `finish` then returns this rank's sources' efficiency (zero
 * elsewhere -- sum over ranks again), the static priority and the
 * calibration (identical on every rank).  Host arrays; back to back on the
 * same context and batch. */
tbsim_status tbsim_attributes_shard_partial(tbsim_ctx* ctx, const tbsim_batch* b, const tbsim_costs* costs,
                                            int32_t rank, int32_t world, int64_t* ability_partial,
                                            int64_t* class_sums, int64_t cap, int64_t* n_words);
tbsim_status tbsim_attributes_shard_finish(tbsim_ctx* ctx, const tbsim_batch* b, const int64_t* class_sums,
                                           int64_t n_words, int32_t priority_kind, tbsim_attr_out* out);

/* ------------------------------------------------------------------------
 * Policies, regulator and the event engine
 * (reference: include/tbsim/policies.hpp, include/tbsim/engine.hpp).
 * ------------------------------------------------------------------------ */
enum { TBSIM_POLICY_FIFO = 0, TBSIM_POLICY_DM = 1, TBSIM_POLICY_DMDA = 2,
       TBSIM_POLICY_DMDAP = 3, TBSIM_POLICY_INSPIRIT = 4 };
/* PopMode (policies.hpp:67) and RegulatorPhase (policies.hpp:87) */
enum { TBSIM_MODE_ABILITY = 0, TBSIM_MODE_EFFICIENCY = 1, TBSIM_MODE_LOCALITY = 2 };
enum { TBSIM_PHASE_INC = 0, TBSIM_PHASE_DEC = 1 };

#define TBSIM_MAX_SLOPE_SAMPLES 64

/* RegulatorConfig (policies.hpp:74-82) */
typedef struct tbsim_regulator_cfg {
    int64_t task_window, s_inc;
    double k_inc;
    int64_t s_dec, c, dec_step;
    int32_t slope_samples; /* 0..TBSIM_MAX_SLOPE_SAMPLES on the device */
    int32_t _pad;
} tbsim_regulator_cfg;

/* RegulatorState (policies.hpp:89-98); samples oldest first. */
typedef struct tbsim_regulator_state {
    int32_t mode, phase;
    int64_t peak, prev_nready, last_trigger_nready, s_dec_count;
    double cur_k;
    int32_t n_samples, _pad;
    double sample_time[TBSIM_MAX_SLOPE_SAMPLES];
    int64_t sample_nready[TBSIM_MAX_SLOPE_SAMPLES];
} tbsim_regulator_state;

/* Attribute inputs of dmdap/inspirit ([T] each; device pointers when
 * on_device).  NULL arrays are read as zeros. */
typedef struct tbsim_attr_in {
    const int64_t* ability;
    const int64_t* efficiency;
    const int64_t* static_priority;
    int32_t on_device;
} tbsim_attr_in;

/* SimTrace (engine.hpp:37-43).  Per-task arrays [T]; per-graph [G].
 * Trace arrays (optional, NULL to skip -- SimOptions::record_trace):
 * pushes/pops of graph g occupy [task_base[g], task_base[g+1]) in event
 * order; nready samples occupy [2*task_base[g], 2*task_base[g+1]). */
typedef struct tbsim_sim_out {
    int32_t* worker;
    double* start_ms;
    double* end_ms;
    double* makespan_ms;      /* [G] */
    int64_t* completed;       /* [G] tasks that finished (== n_g unless stuck) */
    int64_t* pop_mode_counts; /* [3G] inspirit only */
    tbsim_regulator_state* reg_state; /* [G] in: initial, out: final (inspirit) */
    double* push_time;  int32_t* push_task;
    double* pop_time;   int32_t* pop_task;  int32_t* pop_worker;
    double* sample_time; int64_t* sample_nready;
    int32_t on_device;
} tbsim_sim_out;

/* simulate (engine.hpp:47-48) for every graph of the batch.
 * platform_of[g] selects one of n_platforms machine models (NULL: all 0);
 * reg[g] is that graph's RegulatorConfig (NULL: default_regulator_config).
 * Results are bit-identical to the reference: same assignment, same
 * start/end doubles, same pop order. Failure statuses:
 *   runtime_error "no worker can run task type X" (policies.cpp:18-19),
 *   runtime_error "simulation stuck with K tasks unfinished: ..." (engine.cpp:235-246). */
tbsim_status tbsim_simulate(tbsim_ctx* ctx, const tbsim_batch* b,
                            const tbsim_platform_desc* platforms,
                            int32_t n_platforms, const int32_t* platform_of,
                            int32_t policy, const tbsim_regulator_cfg* reg,
                            const tbsim_attr_in* attrs, tbsim_sim_out* out);

/* One "DAG scheduled" (the bench-cell pipeline, src/bench.cpp:102-128):
 * compute_attributes(g, platform.costs, priority) + default_regulator_config
 * + simulate(policy) for every graph, fused on the device.  Attribute
 * outputs are optional (attr_out may be NULL). */
tbsim_status tbsim_schedule(tbsim_ctx* ctx, const tbsim_batch* b,
                            const tbsim_platform_desc* platforms,
                            int32_t n_platforms, const int32_t* platform_of,
                            int32_t policy, int32_t priority_kind,
                            tbsim_attr_out* attr_out, tbsim_sim_out* out);

/* default_regulator_config (policies.hpp:84-85, src/policies.cpp:139-151),
 * host-side helper; median over the graph's GPU times. */
tbsim_status tbsim_default_regulator_config(int32_t n_workers,
                                            double median_gpu_ms,
                                            tbsim_regulator_cfg* out);

/* ------------------------------------------------------------------------
 * Host-side input generators, bit-identical to the reference's
 * (src/generators.cpp).  They write a packed host batch owned by the
 * returned handle; tbsim_hostbatch_desc() exposes it as a tbsim_batch_desc.
 * ------------------------------------------------------------------------ */
typedef struct tbsim_hostbatch tbsim_hostbatch;

tbsim_status tbsim_hostbatch_new(tbsim_hostbatch** out);
tbsim_status tbsim_hostbatch_free(tbsim_hostbatch* hb);
/* generate_layered_dag (taskgraph.hpp:99-100), one graph per seed. */
tbsim_status tbsim_hostbatch_add_layered(tbsim_hostbatch* hb, int32_t n_tasks,
                                         int32_t n_layers, double edge_prob,
                                         const uint64_t* seeds, int64_t n_seeds,
                                         int32_t n_threads);
/* build_cholesky_dag / build_lu_dag (taskgraph.hpp:84,88) and a tiled QR
 * (GEQRT/UNMQR/TSQRT/TSMQR; no reference counterpart). */
tbsim_status tbsim_hostbatch_add_cholesky(tbsim_hostbatch* hb, int32_t nblocks,
                                          int64_t block_bytes);
tbsim_status tbsim_hostbatch_add_lu(tbsim_hostbatch* hb, int32_t nblocks,
                                    int64_t block_bytes);
tbsim_status tbsim_hostbatch_add_qr(tbsim_hostbatch* hb, int32_t nblocks,
                                    int64_t block_bytes);
/* Append an arbitrary graph given in the batch layout (one graph). */
tbsim_status tbsim_hostbatch_add_csr(tbsim_hostbatch* hb, int32_t n_tasks,
                                     const int32_t* dep_off, const int32_t* dep,
                                     const int32_t* in_off, const int32_t* in,
                                     const int32_t* out_off, const int32_t* out,
                                     const int32_t* type, int32_t n_handles,
                                     const int64_t* handle_bytes,
                                     const int64_t* task_id);
tbsim_status tbsim_hostbatch_desc(const tbsim_hostbatch* hb, tbsim_batch_desc* out);
/* The type-name table the batch's type ids index (default: the generators'
 * table, tbsim_type_name); set before the first tbsim_hostbatch_desc. */
tbsim_status tbsim_hostbatch_set_type_names(tbsim_hostbatch* hb, int32_t n, const char* const* names);
/* Binary CSR cache (replaces re-parsing NDJSON DAG files,
 * src/dagio.cpp:86-138): save writes the packed batch (sections + type-name
 * table) to one file; load creates a batch from such a file, reading each
 * section straight into pinned memory, ready for tbsim_batch_upload.  A
 * malformed file fails with TBSIM_E_INVALID_ARGUMENT. */
tbsim_status tbsim_hostbatch_save(tbsim_hostbatch* hb, const char* path);
tbsim_status tbsim_hostbatch_load(const char* path, tbsim_hostbatch** out);
/* The same cache file from any host batch description (e.g. graphs parsed
 * once from NDJSON by the C++ API, tbsim/csr_cache.hpp). */
tbsim_status tbsim_batch_desc_save(const tbsim_batch_desc* desc, const char* path);
/* Type-name table shared by all generated graphs (ids index it). */
int32_t tbsim_type_count(void);
const char* tbsim_type_name(int32_t type_id);
/* default_cost_table (platform.hpp:74, src/platform.cpp:80-104) over the
 * type-name table above. cpu/gpu must hold tbsim_type_count() doubles. */
tbsim_status tbsim_default_costs(double* cpu_ms, double* gpu_ms);

#ifdef __cplusplus
}
#endif
#endif /* TBSIM_B200_H */
