// hostbatch.hpp -- host-side packed graph batches (the producer side of the
// CSR ingestion path) and the synthetic input generators.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tbsim_b200.h"

namespace tbsim_host {

// Canonical type-name table of the generators (ids index it); the Python
// twin is paper_2404_03226_b200/platform.py TYPE_NAMES.
enum TypeId : int32_t {
    T_GEMM = 0, T_SYRK, T_TRSM, T_POTRF, T_GETRF, T_STENCIL,
    T_LAYERK0, T_LAYERK1, T_LAYERK2, T_LAYERK3, T_UNIT,
    T_GEQRT, T_UNMQR, T_TSQRT, T_TSMQR, T_COUNT
};
extern const char* const kTypeNames[T_COUNT];

// One graph under construction (local positions).
struct GraphCSR {
    std::vector<int32_t> dep_off{0}, dep, in_off{0}, in, out_off{0}, out, type;
    std::vector<int64_t> handle_bytes;
    int32_t add(int32_t ty, std::initializer_list<int32_t> deps, std::initializer_list<int32_t> ins,
                std::initializer_list<int32_t> outs);
    int32_t n() const { return static_cast<int32_t>(type.size()); }
};

// Bit-identical to generate_layered_dag (src/generators.cpp:184-244).
GraphCSR gen_layered(int32_t n_tasks, int32_t n_layers, double edge_prob, uint64_t seed);
GraphCSR gen_cholesky(int32_t nblocks, int64_t block_bytes);  // generators.cpp:30-87
GraphCSR gen_lu(int32_t nblocks, int64_t block_bytes);        // generators.cpp:89-142
GraphCSR gen_qr(int32_t nblocks, int64_t block_bytes);        // builder's own tiled QR

// Binary CSR cache of any host batch description (HostBatch::save's format).
void save_csr_cache(const tbsim_batch_desc& d, const std::string& path);

// Packed batch: sections in pinned memory when a CUDA runtime is present.
class HostBatch {
public:
    ~HostBatch();
    void append(const GraphCSR& g, const int64_t* task_ids = nullptr);
    void append_many(std::vector<GraphCSR>&& gs);
    const tbsim_batch_desc& desc();  // packs (once) and returns the view
    int64_t n_graphs() const { return static_cast<int64_t>(task_base_.size()) - 1; }

    // Binary CSR cache (the packed sections as one file): save writes the
    // batch (packing it), load replaces an empty batch's contents with a
    // file's -- one read per section straight into pinned memory, no
    // NDJSON parsing.  The file carries the type-name table.
    void save(const std::string& path);
    void load(const std::string& path);
    // the type-name table the ids index (default: the generators' table)
    void set_type_names(const std::vector<std::string>& names);

private:
    void pack();
    void alloc_pinned(size_t total);
    std::vector<std::string> names_;     // type names of a loaded cache (else kTypeNames)
    std::vector<const char*> name_ptrs_;
    std::vector<int64_t> task_base_{0}, edge_base_{0}, handle_base_{0}, in_base_{0}, out_base_{0};
    std::vector<int32_t> dep_off_, dep_, in_off_, in_, out_off_, out_, type_;
    std::vector<int64_t> handle_bytes_, task_id_;
    bool has_ids_ = false;
    bool packed_ = false;
    void* pinned_ = nullptr;
    bool pinned_is_cuda_ = false;
    tbsim_batch_desc desc_{};
};

}  // namespace tbsim_host
