// hostbatch.cpp -- synthetic DAG generators and packed host batches.
//
// The generators must reproduce the reference's graphs bit-for-bit (same
// edges in the same order, same types, same handle sizes), because the
// scheduling results are compared exactly.  std::mt19937_64 is fully
// specified by the C++ standard, and only raw engine draws are used, exactly
// as src/generators.cpp:18-26 does.
#include "hostbatch.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>

namespace tbsim_host {

const char* const kTypeNames[T_COUNT] = {"GEMM", "SYRK", "TRSM", "POTRF", "GETRF", "STENCIL",
                                         "LAYERK0", "LAYERK1", "LAYERK2", "LAYERK3", "UNIT",
                                         "GEQRT", "UNMQR", "TSQRT", "TSMQR"};

int32_t GraphCSR::add(int32_t ty, std::initializer_list<int32_t> deps,
                      std::initializer_list<int32_t> ins, std::initializer_list<int32_t> outs) {
    for (int32_t d : deps)
        if (d >= 0) dep.push_back(d);
    in.insert(in.end(), ins.begin(), ins.end());
    out.insert(out.end(), outs.begin(), outs.end());
    dep_off.push_back(static_cast<int32_t>(dep.size()));
    in_off.push_back(static_cast<int32_t>(in.size()));
    out_off.push_back(static_cast<int32_t>(out.size()));
    type.push_back(ty);
    return n() - 1;
}

namespace {

// generators.cpp:20-26: (x >> 11) * 2^-53 and x % n on raw 64-bit draws
inline double draw01(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
inline uint64_t draw_below(std::mt19937_64& rng, uint64_t n) { return rng() % n; }

}  // namespace

GraphCSR gen_layered(int32_t n_tasks, int32_t n_layers, double p, uint64_t seed) {
    if (n_layers < 1) throw std::invalid_argument("autogen: n_layers must be >= 1");
    if (n_tasks < n_layers) throw std::invalid_argument("autogen: n_tasks must be >= n_layers");
    if (!(p >= 0.0 && p <= 1.0)) throw std::invalid_argument("autogen: edge_prob must be in [0,1]");
    std::mt19937_64 rng(seed);
    GraphCSR g;
    const int32_t n = n_tasks, L = n_layers;
    g.dep.reserve(static_cast<size_t>(n) * (static_cast<size_t>(p * (n / L)) + 2));
    // Task i sits in layer i mod L; layer l-1's members are l-1, l-1+L, ...
    // Draw order: one uniform per member of the previous layer, then one
    // forced pick when none was taken (generators.cpp:196-203).
    for (int32_t i = 0; i < n; ++i) {
        const int32_t layer = i % L;
        if (layer > 0) {
            const size_t before = g.dep.size();
            int32_t members = 0;
            for (int32_t j = layer - 1; j < n; j += L, ++members)
                if (draw01(rng) < p) g.dep.push_back(j);
            if (g.dep.size() == before)
                g.dep.push_back(layer - 1 + static_cast<int32_t>(draw_below(rng, static_cast<uint64_t>(members))) * L);
        }
        g.dep_off.push_back(static_cast<int32_t>(g.dep.size()));
    }
    // LAYERK0..3 from total-degree quartiles (generators.cpp:206-230)
    std::vector<int32_t> degree(n, 0);
    for (int32_t i = 0; i < n; ++i) {
        degree[i] += g.dep_off[i + 1] - g.dep_off[i];
        for (int32_t k = g.dep_off[i]; k < g.dep_off[i + 1]; ++k) degree[g.dep[k]] += 1;
    }
    std::vector<int32_t> sorted = degree;
    std::sort(sorted.begin(), sorted.end());
    auto q = [&](double f) { return sorted[static_cast<size_t>((n - 1) * f)]; };
    const int32_t q1 = q(0.25), q2 = q(0.5), q3 = q(0.75);
    static const int64_t kTile[4] = {160 * 160 * 4, 320 * 320 * 4, 640 * 640 * 4, 960 * 960 * 4};
    g.handle_bytes.resize(n);
    for (int32_t i = 0; i < n; ++i) g.handle_bytes[i] = kTile[draw_below(rng, 4)];
    // handle id == task id: inputs are the deps, the output is the task itself
    g.in = g.dep;
    g.in_off = g.dep_off;
    g.out.resize(n);
    g.out_off.resize(n + 1);
    g.type.resize(n);
    for (int32_t i = 0; i < n; ++i) {
        g.out[i] = i;
        g.out_off[i + 1] = i + 1;
        const int32_t d = degree[i];
        g.type[i] = T_LAYERK0 + (d <= q1 ? 0 : d <= q2 ? 1 : d <= q3 ? 2 : 3);
    }
    return g;
}

GraphCSR gen_cholesky(int32_t nb, int64_t bytes) {
    if (nb < 1) throw std::invalid_argument("cholesky: nblocks must be >= 1");
    if (bytes <= 0) throw std::invalid_argument("cholesky: block_bytes must be > 0");
    GraphCSR g;
    // lower-triangular tiles, row-major over (i, j<=i)
    auto tile = [](int32_t i, int32_t j) { return i * (i + 1) / 2 + j; };
    std::vector<int32_t> potrf(nb, -1), trsm(nb * nb, -1), syrk(nb * nb, -1), gemm(nb * nb, -1);
    for (int32_t k = 0; k < nb; ++k) {
        potrf[k] = g.add(T_POTRF, {k > 0 ? syrk[k * nb + k - 1] : -1}, {tile(k, k)}, {tile(k, k)});
        for (int32_t i = k + 1; i < nb; ++i)
            trsm[i * nb + k] = g.add(T_TRSM, {potrf[k], k > 0 ? gemm[i * nb + k] : -1},
                                     {tile(k, k), tile(i, k)}, {tile(i, k)});
        for (int32_t i = k + 1; i < nb; ++i) {
            syrk[i * nb + k] = g.add(T_SYRK, {trsm[i * nb + k], k > 0 ? syrk[i * nb + k - 1] : -1},
                                     {tile(i, k), tile(i, i)}, {tile(i, i)});
            for (int32_t j = k + 1; j < i; ++j)
                gemm[i * nb + j] = g.add(T_GEMM, {trsm[i * nb + k], trsm[j * nb + k], k > 0 ? gemm[i * nb + j] : -1},
                                         {tile(i, k), tile(j, k), tile(i, j)}, {tile(i, j)});
        }
    }
    g.handle_bytes.assign(static_cast<size_t>(nb) * (nb + 1) / 2, bytes);
    return g;
}

GraphCSR gen_lu(int32_t nb, int64_t bytes) {
    if (nb < 1) throw std::invalid_argument("lu: nblocks must be >= 1");
    if (bytes <= 0) throw std::invalid_argument("lu: block_bytes must be > 0");
    GraphCSR g;
    auto tile = [nb](int32_t i, int32_t j) { return i * nb + j; };
    std::vector<int32_t> getrf(nb, -1), trow(nb * nb, -1), tcol(nb * nb, -1), gemm(nb * nb, -1);
    for (int32_t k = 0; k < nb; ++k) {
        getrf[k] = g.add(T_GETRF, {k > 0 ? gemm[k * nb + k] : -1}, {tile(k, k)}, {tile(k, k)});
        for (int32_t j = k + 1; j < nb; ++j)
            trow[k * nb + j] = g.add(T_TRSM, {getrf[k], k > 0 ? gemm[k * nb + j] : -1},
                                     {tile(k, k), tile(k, j)}, {tile(k, j)});
        for (int32_t i = k + 1; i < nb; ++i)
            tcol[i * nb + k] = g.add(T_TRSM, {getrf[k], k > 0 ? gemm[i * nb + k] : -1},
                                     {tile(k, k), tile(i, k)}, {tile(i, k)});
        for (int32_t i = k + 1; i < nb; ++i)
            for (int32_t j = k + 1; j < nb; ++j)
                gemm[i * nb + j] = g.add(T_GEMM, {tcol[i * nb + k], trow[k * nb + j], k > 0 ? gemm[i * nb + j] : -1},
                                         {tile(i, k), tile(k, j), tile(i, j)}, {tile(i, j)});
    }
    g.handle_bytes.assign(static_cast<size_t>(nb) * nb, bytes);
    return g;
}

// Tiled Householder QR (flat TS tree), the standard PLASMA task graph:
//   for k: GEQRT(k,k); UNMQR(k,j) j>k; for i>k: TSQRT(i,k), TSMQR(i,j) j>k.
// Dependencies follow the tile read/write sets with writers serialized; no
// reference counterpart exists (SURVEY.md §0 note 3), costs are
// builder-chosen (platform.py _QR_ROWS).  n^3/3 + O(n^2) tasks:
// sum_{m=1..n} m^2 = 22,140 at n = 40.
GraphCSR gen_qr(int32_t nb, int64_t bytes) {
    if (nb < 1) throw std::invalid_argument("qr: nblocks must be >= 1");
    if (bytes <= 0) throw std::invalid_argument("qr: block_bytes must be > 0");
    GraphCSR g;
    auto tile = [nb](int32_t i, int32_t j) { return i * nb + j; };
    // last writer of each tile (A) and of each T factor (one per (i,k) panel)
    std::vector<int32_t> last(nb * nb, -1);
    for (int32_t k = 0; k < nb; ++k) {
        const int32_t geqrt = g.add(T_GEQRT, {last[tile(k, k)]}, {tile(k, k)}, {tile(k, k)});
        last[tile(k, k)] = geqrt;
        std::vector<int32_t> unmqr(nb, -1);
        for (int32_t j = k + 1; j < nb; ++j) {
            unmqr[j] = g.add(T_UNMQR, {geqrt, last[tile(k, j)]}, {tile(k, k), tile(k, j)}, {tile(k, j)});
            last[tile(k, j)] = unmqr[j];
        }
        int32_t prev_ts = geqrt;  // TSQRT(i,k) updates the R factor in tile (k,k)
        for (int32_t i = k + 1; i < nb; ++i) {
            const int32_t tsqrt = g.add(T_TSQRT, {prev_ts, last[tile(i, k)]}, {tile(k, k), tile(i, k)},
                                        {tile(k, k), tile(i, k)});
            last[tile(i, k)] = tsqrt;
            prev_ts = tsqrt;
            for (int32_t j = k + 1; j < nb; ++j) {
                // TSMQR(i,j,k) updates tiles (k,j) and (i,j) with V(i,k)
                const int32_t ts = g.add(T_TSMQR, {tsqrt, last[tile(k, j)], last[tile(i, j)]},
                                         {tile(i, k), tile(k, j), tile(i, j)}, {tile(k, j), tile(i, j)});
                last[tile(k, j)] = ts;
                last[tile(i, j)] = ts;
            }
        }
        last[tile(k, k)] = prev_ts;
    }
    // drop duplicate dependency entries produced when two roles share a writer
    GraphCSR h;
    for (int32_t t = 0; t < g.n(); ++t) {
        std::vector<int32_t> d(g.dep.begin() + g.dep_off[t], g.dep.begin() + g.dep_off[t + 1]);
        std::vector<int32_t> uniq;
        for (int32_t x : d)
            if (std::find(uniq.begin(), uniq.end(), x) == uniq.end()) uniq.push_back(x);
        h.dep.insert(h.dep.end(), uniq.begin(), uniq.end());
        h.dep_off.push_back(static_cast<int32_t>(h.dep.size()));
    }
    g.dep = std::move(h.dep);
    g.dep_off = std::move(h.dep_off);
    g.handle_bytes.assign(static_cast<size_t>(nb) * nb, bytes);
    return g;
}

// --------------------------------------------------------------- HostBatch

HostBatch::~HostBatch() {
    if (pinned_) {
        if (pinned_is_cuda_) cudaFreeHost(pinned_);
        else std::free(pinned_);
    }
}

void HostBatch::append(const GraphCSR& g, const int64_t* task_ids) {
    if (packed_) throw std::logic_error("batch already packed");
    const int32_t n = g.n();
    if (n == 0 && task_base_.size() == 1 && !has_ids_ && task_ids) has_ids_ = true;
    if (task_ids) {
        if (!has_ids_) {
            // earlier graphs had implicit ids: materialize them
            for (int64_t gi = 0; gi + 1 < static_cast<int64_t>(task_base_.size()); ++gi)
                for (int64_t t = task_base_[gi]; t < task_base_[gi + 1]; ++t) task_id_.push_back(t - task_base_[gi]);
            has_ids_ = true;
        }
        task_id_.insert(task_id_.end(), task_ids, task_ids + n);
    } else if (has_ids_) {
        for (int32_t i = 0; i < n; ++i) task_id_.push_back(i);
    }
    dep_off_.insert(dep_off_.end(), g.dep_off.begin(), g.dep_off.end());
    in_off_.insert(in_off_.end(), g.in_off.begin(), g.in_off.end());
    out_off_.insert(out_off_.end(), g.out_off.begin(), g.out_off.end());
    dep_.insert(dep_.end(), g.dep.begin(), g.dep.end());
    in_.insert(in_.end(), g.in.begin(), g.in.end());
    out_.insert(out_.end(), g.out.begin(), g.out.end());
    type_.insert(type_.end(), g.type.begin(), g.type.end());
    handle_bytes_.insert(handle_bytes_.end(), g.handle_bytes.begin(), g.handle_bytes.end());
    task_base_.push_back(task_base_.back() + n);
    edge_base_.push_back(edge_base_.back() + static_cast<int64_t>(g.dep.size()));
    handle_base_.push_back(handle_base_.back() + static_cast<int64_t>(g.handle_bytes.size()));
    in_base_.push_back(in_base_.back() + static_cast<int64_t>(g.in.size()));
    out_base_.push_back(out_base_.back() + static_cast<int64_t>(g.out.size()));
}

void HostBatch::append_many(std::vector<GraphCSR>&& gs) {
    size_t t = 0, e = 0, h = 0, i = 0, o = 0;
    for (const auto& g : gs) { t += g.n() + 1; e += g.dep.size(); h += g.handle_bytes.size(); i += g.in.size(); o += g.out.size(); }
    dep_off_.reserve(dep_off_.size() + t); in_off_.reserve(in_off_.size() + t); out_off_.reserve(out_off_.size() + t);
    dep_.reserve(dep_.size() + e); in_.reserve(in_.size() + i); out_.reserve(out_.size() + o);
    handle_bytes_.reserve(handle_bytes_.size() + h); type_.reserve(type_.size() + t);
    for (auto& g : gs) {
        append(g);
        GraphCSR().dep.swap(g.dep);  // release as we go
    }
}

namespace {
size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
}

void HostBatch::pack() {
    // one pinned block: bases then sections, so the upload is a handful of
    // DMA copies (or one, when the device mirrors this layout)
    // inputs identical to dependencies (every generator here: a task reads
    // its predecessors' outputs) are stored once and aliased in the
    // descriptor, so the upload copies them once
    const bool in_is_dep = in_base_ == edge_base_ && in_off_ == dep_off_ && in_ == dep_;
    struct Sec { const void* src; size_t bytes; };
    std::vector<Sec> secs = {
        {task_base_.data(), task_base_.size() * 8}, {edge_base_.data(), edge_base_.size() * 8},
        {handle_base_.data(), handle_base_.size() * 8}, {in_base_.data(), in_base_.size() * 8},
        {out_base_.data(), out_base_.size() * 8}, {dep_off_.data(), dep_off_.size() * 4},
        {dep_.data(), dep_.size() * 4}, {in_off_.data(), in_off_.size() * 4}, {in_.data(), in_.size() * 4},
        {out_off_.data(), out_off_.size() * 4}, {out_.data(), out_.size() * 4}, {type_.data(), type_.size() * 4},
        {handle_bytes_.data(), handle_bytes_.size() * 8}, {task_id_.data(), task_id_.size() * 8}};
    if (in_is_dep) secs[3].bytes = secs[7].bytes = secs[8].bytes = 0;  // in_base, in_off, in
    size_t total = 0;
    for (const auto& s : secs) total += align16(s.bytes);
    alloc_pinned(total);
    char* p = static_cast<char*>(pinned_);
    std::vector<void*> dst;
    for (const auto& s : secs) {
        if (s.bytes) std::memcpy(p, s.src, s.bytes);
        dst.push_back(p);
        p += align16(s.bytes);
    }
    if (in_is_dep) {
        dst[3] = dst[1];  // in_base = edge_base
        dst[7] = dst[5];  // in_off = dep_off
        dst[8] = dst[6];  // in = dep
    }
    desc_.n_graphs = n_graphs();
    desc_.task_base = static_cast<const int64_t*>(dst[0]);
    desc_.edge_base = static_cast<const int64_t*>(dst[1]);
    desc_.handle_base = static_cast<const int64_t*>(dst[2]);
    desc_.in_base = static_cast<const int64_t*>(dst[3]);
    desc_.out_base = static_cast<const int64_t*>(dst[4]);
    desc_.dep_off = static_cast<const int32_t*>(dst[5]);
    desc_.dep = static_cast<const int32_t*>(dst[6]);
    desc_.in_off = static_cast<const int32_t*>(dst[7]);
    desc_.in = static_cast<const int32_t*>(dst[8]);
    desc_.out_off = static_cast<const int32_t*>(dst[9]);
    desc_.out = static_cast<const int32_t*>(dst[10]);
    desc_.type = static_cast<const int32_t*>(dst[11]);
    desc_.handle_bytes = static_cast<const int64_t*>(dst[12]);
    desc_.task_id = has_ids_ ? static_cast<const int64_t*>(dst[13]) : nullptr;
    if (names_.empty()) {
        desc_.n_type_names = T_COUNT;
        desc_.type_names = kTypeNames;
    } else {
        name_ptrs_.clear();
        for (const auto& nm : names_) name_ptrs_.push_back(nm.c_str());
        desc_.n_type_names = static_cast<int32_t>(names_.size());
        desc_.type_names = name_ptrs_.data();
    }
    // the vectors are no longer needed
    std::vector<int32_t>().swap(dep_); std::vector<int32_t>().swap(in_); std::vector<int32_t>().swap(out_);
    std::vector<int32_t>().swap(dep_off_); std::vector<int32_t>().swap(in_off_); std::vector<int32_t>().swap(out_off_);
    std::vector<int32_t>().swap(type_); std::vector<int64_t>().swap(handle_bytes_); std::vector<int64_t>().swap(task_id_);
    packed_ = true;
}

const tbsim_batch_desc& HostBatch::desc() {
    if (!packed_) pack();
    return desc_;
}

void HostBatch::set_type_names(const std::vector<std::string>& names) {
    if (packed_) throw std::logic_error("batch already packed");
    names_ = names;
}

void HostBatch::alloc_pinned(size_t total) {
    if (cudaHostAlloc(&pinned_, std::max<size_t>(total, 16), cudaHostAllocDefault) == cudaSuccess) {
        pinned_is_cuda_ = true;
    } else {
        cudaGetLastError();
        pinned_ = std::malloc(std::max<size_t>(total, 16));
        pinned_is_cuda_ = false;
    }
}

// ------------------------------------------------------- binary CSR cache
//
// Layout (little-endian): "TBSIMCSR" | u32 version (1) | u32 flags (bit 0:
// task ids) | i64 G, T, E, H, I, O | u32 n_names, then per name u32 length +
// bytes | the 14 sections of tbsim_batch_desc in order, each padded to 16
// bytes (bases [G+1] x i64, offsets [T+G] x i32, entries, types [T] x i32,
// handle bytes [H] x i64, task ids [T] x i64 when flagged).

namespace {

constexpr char kMagic[8] = {'T', 'B', 'S', 'I', 'M', 'C', 'S', 'R'};

struct CacheDims {
    int64_t G, T, E, H, I, O;
};

std::vector<size_t> section_bytes(const CacheDims& d, bool ids) {
    return {static_cast<size_t>(d.G + 1) * 8, static_cast<size_t>(d.G + 1) * 8, static_cast<size_t>(d.G + 1) * 8,
            static_cast<size_t>(d.G + 1) * 8, static_cast<size_t>(d.G + 1) * 8, static_cast<size_t>(d.T + d.G) * 4,
            static_cast<size_t>(d.E) * 4,     static_cast<size_t>(d.T + d.G) * 4, static_cast<size_t>(d.I) * 4,
            static_cast<size_t>(d.T + d.G) * 4, static_cast<size_t>(d.O) * 4,   static_cast<size_t>(d.T) * 4,
            static_cast<size_t>(d.H) * 8,     ids ? static_cast<size_t>(d.T) * 8 : 0};
}

void put(std::FILE* f, const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f) != n) throw std::runtime_error("csr cache: write failed");
}
void get(std::FILE* f, void* p, size_t n) {
    if (n && std::fread(p, 1, n, f) != n) throw std::invalid_argument("csr cache: truncated file");
}

}  // namespace

void HostBatch::save(const std::string& path) { save_csr_cache(desc(), path); }

void save_csr_cache(const tbsim_batch_desc& d, const std::string& path) {
    const int64_t G = d.n_graphs;
    const CacheDims dims{G, d.task_base[G], d.edge_base[G], d.handle_base[G], d.in_base[G], d.out_base[G]};
    const bool ids = d.task_id != nullptr;
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + path);
    try {
        put(f, kMagic, 8);
        const uint32_t version = 1, flags = ids ? 1u : 0u;
        const uint32_t nn = d.type_names ? static_cast<uint32_t>(d.n_type_names) : 0u;
        put(f, &version, 4);
        put(f, &flags, 4);
        put(f, &dims, sizeof dims);
        put(f, &nn, 4);
        for (uint32_t i = 0; i < nn; ++i) {
            const uint32_t len = static_cast<uint32_t>(std::strlen(d.type_names[i]));
            put(f, &len, 4);
            put(f, d.type_names[i], len);
        }
        const void* src[14] = {d.task_base, d.edge_base, d.handle_base, d.in_base, d.out_base, d.dep_off, d.dep,
                               d.in_off,    d.in,        d.out_off,     d.out,     d.type,    d.handle_bytes, d.task_id};
        const auto sz = section_bytes(dims, ids);
        static const char zeros[16] = {};
        for (int i = 0; i < 14; ++i) {
            put(f, src[i], sz[i]);
            put(f, zeros, align16(sz[i]) - sz[i]);
        }
    } catch (...) {
        std::fclose(f);
        throw;
    }
    if (std::fclose(f) != 0) throw std::runtime_error("csr cache: write failed");
}

void HostBatch::load(const std::string& path) {
    if (packed_ || n_graphs() != 0) throw std::logic_error("csr cache: load needs an empty batch");
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open " + path);
    try {
        char magic[8];
        uint32_t version = 0, flags = 0, nn = 0;
        CacheDims dims{};
        get(f, magic, 8);
        if (std::memcmp(magic, kMagic, 8) != 0) throw std::invalid_argument("csr cache: bad magic in " + path);
        get(f, &version, 4);
        if (version != 1) throw std::invalid_argument("csr cache: unsupported version");
        get(f, &flags, 4);
        get(f, &dims, sizeof dims);
        if (dims.G < 0 || dims.T < 0 || dims.E < 0 || dims.H < 0 || dims.I < 0 || dims.O < 0)
            throw std::invalid_argument("csr cache: negative section size");
        get(f, &nn, 4);
        if (nn > 4096) throw std::invalid_argument("csr cache: too many type names");
        names_.resize(nn);
        for (uint32_t i = 0; i < nn; ++i) {
            uint32_t len = 0;
            get(f, &len, 4);
            if (len > 4096) throw std::invalid_argument("csr cache: type name too long");
            names_[i].resize(len);
            get(f, names_[i].data(), len);
        }
        const bool ids = flags & 1u;
        const auto sz = section_bytes(dims, ids);
        size_t total = 0;
        for (size_t b : sz) total += align16(b);
        alloc_pinned(total);
        char* p = static_cast<char*>(pinned_);
        std::vector<void*> dst;
        for (size_t b : sz) {
            get(f, p, align16(b));  // the file pads like the pinned block
            dst.push_back(p);
            p += align16(b);
        }
        desc_ = tbsim_batch_desc{};
        desc_.n_graphs = dims.G;
        desc_.task_base = static_cast<const int64_t*>(dst[0]);
        desc_.edge_base = static_cast<const int64_t*>(dst[1]);
        desc_.handle_base = static_cast<const int64_t*>(dst[2]);
        desc_.in_base = static_cast<const int64_t*>(dst[3]);
        desc_.out_base = static_cast<const int64_t*>(dst[4]);
        desc_.dep_off = static_cast<const int32_t*>(dst[5]);
        desc_.dep = static_cast<const int32_t*>(dst[6]);
        desc_.in_off = static_cast<const int32_t*>(dst[7]);
        desc_.in = static_cast<const int32_t*>(dst[8]);
        desc_.out_off = static_cast<const int32_t*>(dst[9]);
        desc_.out = static_cast<const int32_t*>(dst[10]);
        desc_.type = static_cast<const int32_t*>(dst[11]);
        desc_.handle_bytes = static_cast<const int64_t*>(dst[12]);
        desc_.task_id = ids ? static_cast<const int64_t*>(dst[13]) : nullptr;
        if (desc_.task_base[dims.G] != dims.T || desc_.edge_base[dims.G] != dims.E ||
            desc_.handle_base[dims.G] != dims.H || desc_.in_base[dims.G] != dims.I || desc_.out_base[dims.G] != dims.O)
            throw std::invalid_argument("csr cache: bases disagree with the header");
        name_ptrs_.clear();
        for (const auto& n : names_) name_ptrs_.push_back(n.c_str());
        desc_.n_type_names = static_cast<int32_t>(nn);
        desc_.type_names = name_ptrs_.data();
        task_base_.assign(desc_.task_base, desc_.task_base + dims.G + 1);
        packed_ = true;
    } catch (...) {
        std::fclose(f);
        throw;
    }
    std::fclose(f);
}

}  // namespace tbsim_host
