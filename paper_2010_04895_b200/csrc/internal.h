// internal.h -- host-side objects shared by graph.cu, walk.cu and api.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mhw.h"
#include "mhw_device.cuh"

namespace mhw {

// Error carrying an mhw_status (errors.hpp classes -> status codes).
struct Error : std::runtime_error {
    mhw_status code;
    Error(mhw_status c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define MHW_CK(call)                                                    \
    do {                                                                \
        cudaError_t _e = (call);                                        \
        if (_e != cudaSuccess) ::mhw::throw_cuda(_e, #call, __FILE__, __LINE__); \
    } while (0)

inline void invalid(const std::string& msg) { throw Error(MHW_ERR_INVALID, msg); }

// Device allocation with a block cache for large buffers (graph.cu): blocks
// >= 32 MB are kept after a device synchronisation and reused by later calls
// (multi-GB cudaMalloc/cudaFree per generate_walks call cost tens of ms);
// on an allocation failure the cache is released and the allocation retried.
void* dev_alloc(size_t bytes, size_t* cap);
void dev_free(void* p, size_t cap);
void dev_trim();
size_t dev_cached_bytes();
size_t dev_available_bytes();  // cudaMemGetInfo free + pool memory reserved but unused

// RAII device buffer on the current device.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    size_t cap = 0;  // allocated bytes
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap) {
        o.p = nullptr;
        o.n = o.cap = 0;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p;
            n = o.n;
            cap = o.cap;
            o.p = nullptr;
            o.n = o.cap = 0;
        }
        return *this;
    }
    ~DBuf() { reset(); }
    void alloc(size_t count) {
        reset();
        if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T), &cap));
        n = count;
    }
    void reset() {
        if (p) dev_free(p, cap);
        p = nullptr;
        n = cap = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// Switches the current device for the lifetime of the guard.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) MHW_CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Device-resident CSR replica (mhw_graph).
struct Graph {
    int device = 0;
    uint32_t n = 0;
    uint64_t m = 0;
    DBuf<NodeRec> nodes;
    DBuf<uint32_t> ids;
    DBuf<float> w;           // empty: unweighted
    DBuf<uint16_t> ntype;    // empty: untyped (types are also in NodeRec)
    DBuf<uint16_t> etype;    // empty: derived
    DBuf<uint32_t> rev;      // lazily built
    DBuf<double> wtotal;     // lazily built
    DBuf<double> wblk;       // bootstrap block prefix sums, built with wtotal
    DBuf<uint32_t> tcount;   // lazily built
    DBuf<uint32_t> tperm;    // typed neighbour index (metapath2vec init), lazily built
    DBuf<uint2> tbase;
    DBuf<uint32_t> htab;     // adjacency hash sets, lazily built
    DBuf<uint32_t> bloom;    // edge Bloom filter (second-order alpha), lazily built
    uint32_t bloom_blocks = 0;
    DBuf<uint32_t> bloom2;   // the same filter at twice the blocks (bloom = its fold); compact-chain graphs
    uint32_t bloom2_blocks = 0;
    DBuf<uint4> arc;         // arc records, lazily built (m < 2^32)
    DBuf<uint4> sal;         // static-weight alias tables (alias proposal), {prob f64, alias, 0} per arc, lazily built
    uint16_t n_ntypes = 0, n_etypes = 0;
    bool symmetric = false;
    bool verified_sym = false;
    uint32_t max_deg = 0;
    uint32_t isolated = 0;
    cudaStream_t stream = nullptr;

    bool weighted() const { return w.n != 0; }
    bool has_ntypes() const { return ntype.n != 0; }
    DevGraph view() const;
    uint64_t device_bytes() const;
};

// Graph construction (graph.cu).
void graph_init_stream(Graph& g);
void graph_finalize(Graph& g, const int64_t* d_offsets, const uint16_t* d_ntypes);
void graph_upload(Graph& g, const mhw_graph_view& v);
void graph_from_edges(Graph& g, uint64_t ne, const uint32_t* src, const uint32_t* dst, const float* w,
                      bool symmetrize, uint32_t n_nodes);
void graph_generate_rmat(Graph& g, uint32_t scale, uint32_t ef, double a, double b, double c,
                         uint64_t seed, bool weighted, float wlo, float whi, uint32_t n_etypes);
void graph_generate_hetero(Graph& g, uint32_t n_nodes, uint64_t seed, float wlo, float whi);
void graph_set_node_types(Graph& g, const uint16_t* types, uint16_t num_types);
void graph_set_edge_types(Graph& g, const uint16_t* types, uint16_t num_types);
void graph_replicate(const Graph& src, Graph& dst, int device);
void graph_download(const Graph& g, int64_t* offsets, int32_t* nbr, float* w, uint16_t* ntypes,
                    uint16_t* etypes);
void graph_ensure_rev(Graph& g);
void graph_ensure_wtotal(Graph& g);
void graph_ensure_tcount(Graph& g);
void graph_ensure_typed_index(Graph& g);
void graph_ensure_hash(Graph& g, cudaStream_t st = nullptr, bool sync = true);
void graph_ensure_bloom(Graph& g, cudaStream_t st = nullptr, bool sync = true, uint32_t max_bits = 4);
// rev + wtotal, and (alpha) hash sets + edge filter concurrently.
void graph_ensure_second_order(Graph& g, bool alpha, uint32_t bloom_bits = 4);
// A separate edge filter at `bits` bits per arc into `out` (blocks out).
void graph_build_bloom(const Graph& g, uint32_t bits, DBuf<uint32_t>& out, uint32_t* blocks, cudaStream_t st);
bool graph_ensure_arcrec(Graph& g);  // deepwalk arc records (fp32 weight aux)
void graph_alias_tables(Graph& g, double* prob, uint32_t* alias);
// Same tables left on the device (prob, alias: m entries each).
void graph_alias_device(Graph& g, double* prob, uint32_t* alias);
// The same tables kept on the graph (packed {prob, alias}: sal) for the alias proposal
// of the M-H walk; unweighted graphs need none (every prob is 1.0).
void graph_ensure_static_alias(Graph& g);

// Bound model (host validation of WalkModel::bind, models.cpp:29-74).
struct Model {
    mhw_model_desc desc{};
    DBuf<uint16_t> metapath;
    DBuf<double> M;
    std::vector<uint16_t> h_metapath;
    DevModel dev{};
};
void model_bind(Model& m, Graph& g, const mhw_model_desc& d);

}  // namespace mhw

struct mhw_graph : mhw::Graph {};
