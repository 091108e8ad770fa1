// api.cu -- the extern "C" boundary (include/mhw.h). Every entry point
// converts exceptions to status codes (errors.hpp classes -> 1/2/4) and keeps
// the message in a thread-local buffer (mhw_last_error).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "jsonfmt.h"
#include "loader.h"
#include "exact.h"
#include "walk.h"

struct mhw_walks {
    std::vector<uint32_t> nodes;
    std::vector<uint32_t> lens;
    uint64_t rows = 0;
    uint32_t stride = 0;
    mhw_walk_stats stats{};
};

namespace {

thread_local std::string g_error;

void set_error(const std::string& s) { g_error = s; }

template <class F>
mhw_status guard(F&& f) {
    try {
        f();
        return MHW_OK;
    } catch (const mhw::Error& e) {
        set_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host out of memory");
        return MHW_ERR_CUDA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return MHW_ERR_CUDA;
    }
}

void need(const void* p, const char* what) {
    if (!p) mhw::invalid(std::string(what) + " must not be NULL");
}

mhw::Graph* new_graph(int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        throw mhw::Error(MHW_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
    if (device < 0 || device >= count) mhw::invalid("device index out of range");
    auto* g = new mhw_graph();
    g->device = device;
    return g;
}

template <class F>
mhw_status build_graph(int32_t device, mhw_graph** out, F&& f) {
    return guard([&] {
        need(out, "out");
        std::unique_ptr<mhw_graph> g(static_cast<mhw_graph*>(new_graph(device)));
        mhw::DeviceGuard dg(device);
        f(*g);
        *out = g.release();
    });
}

void run_into(const mhw_graph* gc, const mhw_model_desc* model, const mhw_walk_config* cfg, uint32_t* nodes,
              uint32_t* lens, uint64_t capacity, mhw_walk_stats* stats, uint64_t* rows_out) {
    need(gc, "graph");
    need(model, "model");
    need(cfg, "config");
    auto* g = const_cast<mhw_graph*>(gc);
    mhw::DeviceGuard dg(g->device);
    mhw_session s;
    mhw::session_create(s, *g, *model, *cfg);
    if ((nodes || lens) && s.rows > capacity) mhw::invalid("output buffer too small for the corpus");
    mhw::session_run(s, nullptr);
    mhw_walk_stats st{};
    mhw::session_stats(s, st);
    if (nodes || lens) mhw::session_download(s, nodes, lens, nullptr);
    if (stats) *stats = st;
    if (rows_out) *rows_out = s.rows;
}

}  // namespace

extern "C" {

const char* mhw_last_error(void) { return g_error.c_str(); }
const char* mhw_version(void) { return "mhw 0.1.0 (sm_100a)"; }

void mhw_trim_memory(void) { mhw::dev_trim(); }

int32_t mhw_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

mhw_status mhw_graph_upload(const mhw_graph_view* view, int32_t device, mhw_graph** out) {
    return build_graph(device, out, [&](mhw::Graph& g) {
        need(view, "view");
        mhw::graph_upload(g, *view);
    });
}

mhw_status mhw_graph_from_edges(uint64_t edge_count, const uint32_t* src, const uint32_t* dst,
                                const float* weights, int32_t symmetrize, uint32_t node_count,
                                int32_t device, mhw_graph** out) {
    return build_graph(device, out, [&](mhw::Graph& g) {
        if (edge_count) {
            need(src, "src");
            need(dst, "dst");
            if (weights)
                for (uint64_t i = 0; i < edge_count; ++i)
                    if (!(weights[i] >= 0)) mhw::invalid("negative edge weight");
        }
        mhw::graph_from_edges(g, edge_count, src, dst, weights, symmetrize != 0, node_count);
    });
}

mhw_status mhw_graph_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                                   uint64_t seed, int32_t weighted, float weight_lo, float weight_hi,
                                   uint32_t edge_type_count, int32_t device, mhw_graph** out) {
    return build_graph(device, out, [&](mhw::Graph& g) {
        if (weighted && !(weight_lo >= 0 && weight_hi >= weight_lo)) mhw::invalid("bad weight range");
        if (edge_type_count > 65535) mhw::invalid("too many edge types");
        mhw::graph_generate_rmat(g, scale, edge_factor, a, b, c, seed, weighted != 0, weight_lo, weight_hi,
                                 edge_type_count);
    });
}

mhw_status mhw_graph_generate_hetero(uint32_t node_count, uint64_t seed, float weight_lo, float weight_hi,
                                     int32_t device, mhw_graph** out) {
    return build_graph(device, out, [&](mhw::Graph& g) {
        if (!(weight_lo >= 0 && weight_hi >= weight_lo)) mhw::invalid("bad weight range");
        mhw::graph_generate_hetero(g, node_count, seed, weight_lo, weight_hi);
    });
}

mhw_status mhw_parse_edge_list(const char* path, int32_t weighted, int32_t symmetrize, uint64_t* n_edges,
                               uint32_t** src, uint32_t** dst, double** weights) {
    return guard([&] {
        need(path, "path");
        need(n_edges, "n_edges");
        need(src, "src");
        need(dst, "dst");
        need(weights, "weights");
        std::vector<uint32_t> s, d;
        std::vector<double> w;
        mhw::parse_edge_list(path, weighted != 0, symmetrize != 0, s, d, w);
        const size_t n = s.size();
        auto* ps = static_cast<uint32_t*>(std::malloc(std::max<size_t>(n, 1) * 4));
        auto* pd = static_cast<uint32_t*>(std::malloc(std::max<size_t>(n, 1) * 4));
        auto* pw = static_cast<double*>(std::malloc(std::max<size_t>(n, 1) * 8));
        if (!ps || !pd || !pw) {
            std::free(ps);
            std::free(pd);
            std::free(pw);
            throw std::bad_alloc();
        }
        if (n) {
            std::memcpy(ps, s.data(), n * 4);
            std::memcpy(pd, d.data(), n * 4);
            std::memcpy(pw, w.data(), n * 8);
        }
        *n_edges = n;
        *src = ps;
        *dst = pd;
        *weights = pw;
    });
}

void mhw_free_host(void* p) { std::free(p); }

mhw_status mhw_graph_load_edge_list(const char* path, int32_t weighted, int32_t symmetrize, int32_t device,
                                    mhw_graph** out) {
    // parse first (host): file and format errors take precedence, as in the
    // reference where loading precedes any walk
    std::vector<uint32_t> s, d;
    std::vector<double> w;
    const mhw_status rc = guard([&] {
        need(path, "path");
        mhw::parse_edge_list(path, weighted != 0, symmetrize != 0, s, d, w);
    });
    if (rc != MHW_OK) return rc;
    return build_graph(device, out, [&](mhw::Graph& g) { mhw::build_parsed(g, s, d, w, weighted != 0, symmetrize != 0); });
}

mhw_status mhw_graph_load_node_types(mhw_graph* g, const char* path) {
    return guard([&] {
        need(g, "graph");
        need(path, "path");
        mhw::DeviceGuard dg(g->device);
        mhw::load_node_types(*g, path);
    });
}

mhw_status mhw_graph_load_edge_types(mhw_graph* g, const char* path) {
    return guard([&] {
        need(g, "graph");
        need(path, "path");
        mhw::DeviceGuard dg(g->device);
        mhw::load_edge_types(*g, path);
    });
}

mhw_status mhw_graph_set_node_types(mhw_graph* g, const uint16_t* types, uint16_t num_types) {
    return guard([&] {
        need(g, "graph");
        need(types, "types");
        mhw::graph_set_node_types(*g, types, num_types);
    });
}

mhw_status mhw_graph_set_edge_types(mhw_graph* g, const uint16_t* types, uint16_t num_types) {
    return guard([&] {
        need(g, "graph");
        need(types, "types");
        mhw::graph_set_edge_types(*g, types, num_types);
    });
}

mhw_status mhw_graph_replicate(const mhw_graph* g, int32_t device, mhw_graph** out) {
    return build_graph(device, out, [&](mhw::Graph& d) {
        need(g, "graph");
        mhw::graph_replicate(*g, d, device);
    });
}

mhw_status mhw_graph_info_get(const mhw_graph* g, mhw_graph_info* info) {
    return guard([&] {
        need(g, "graph");
        need(info, "info");
        info->node_count = g->n;
        info->arc_count = g->m;
        info->weighted = g->weighted();
        info->symmetric = g->symmetric;
        info->verified_symmetric = g->verified_sym;
        info->num_node_types = g->n_ntypes;
        info->num_edge_types = g->n_etypes;
        info->max_degree = g->max_deg;
        info->isolated_nodes = g->isolated;
        info->device_bytes = g->device_bytes();
        info->device = g->device;
    });
}

mhw_status mhw_graph_download(const mhw_graph* g, int64_t* offsets, int32_t* neighbors, float* weights,
                              uint16_t* node_types, uint16_t* edge_types) {
    return guard([&] {
        need(g, "graph");
        mhw::graph_download(*g, offsets, neighbors, weights, node_types, edge_types);
    });
}

void mhw_graph_free(mhw_graph* g) {
    if (!g) return;
    mhw::DeviceGuard dg(g->device);
    if (g->stream) cudaStreamDestroy(g->stream);
    delete g;
}

mhw_status mhw_generate_walks(const mhw_graph* g, const mhw_model_desc* model, const mhw_walk_config* config,
                              mhw_walks** out) {
    return guard([&] {
        need(out, "out");
        need(g, "graph");
        need(model, "model");
        need(config, "config");
        auto* gg = const_cast<mhw_graph*>(g);
        mhw::DeviceGuard dg(gg->device);
        mhw_session s;
        mhw::session_create(s, *gg, *model, *config);
        std::unique_ptr<mhw_walks> w(new mhw_walks());
        w->rows = s.rows;
        w->stride = s.stride;
        w->nodes.resize(s.rows * s.stride);
        w->lens.resize(s.rows);
        mhw::session_run(s, nullptr);
        mhw::session_stats(s, w->stats);
        mhw::session_download(s, w->nodes.data(), w->lens.data(), nullptr);
        *out = w.release();
    });
}

mhw_status mhw_generate_walks_multi(const mhw_graph* const* replicas, int32_t n_replicas,
                                    const mhw_model_desc* model, const mhw_walk_config* config, mhw_walks** out) {
    return guard([&] {
        need(out, "out");
        need(replicas, "replicas");
        need(model, "model");
        need(config, "config");
        if (n_replicas <= 0) mhw::invalid("need at least one replica");
        for (int i = 0; i < n_replicas; ++i) need(replicas[i], "replica");
        const uint32_t n = replicas[0]->n;
        const uint32_t b = config->node_begin, e = config->node_end ? config->node_end : n;
        std::vector<uint32_t> cuts(n_replicas + 1);
        {
            auto* g0 = const_cast<mhw_graph*>(replicas[0]);
            mhw::partition_nodes(*g0, *model, n_replicas, cuts.data());
        }
        // clamp the balanced cuts to the requested range
        for (auto& c : cuts) c = std::min(std::max(c, b), e);
        cuts.front() = b;
        cuts.back() = e;
        std::vector<std::unique_ptr<mhw_session>> ss(n_replicas);
        std::vector<std::string> errs(n_replicas);
        std::vector<mhw_status> codes(n_replicas, MHW_OK);
        auto par = [&](auto&& body) {
            std::vector<std::thread> th;
            for (int i = 0; i < n_replicas; ++i)
                th.emplace_back([&, i] {
                    try {
                        body(i);
                    } catch (const mhw::Error& x) {
                        codes[i] = x.code;
                        errs[i] = x.what();
                    } catch (const std::exception& x) {
                        codes[i] = MHW_ERR_CUDA;
                        errs[i] = x.what();
                    }
                });
            for (auto& t : th) t.join();
            for (int i = 0; i < n_replicas; ++i)
                if (codes[i]) throw mhw::Error(codes[i], errs[i]);
        };
        par([&](int i) {
            auto* g = const_cast<mhw_graph*>(replicas[i]);
            mhw::DeviceGuard dg(g->device);
            mhw_walk_config c = *config;
            c.node_begin = cuts[i];
            c.node_end = cuts[i + 1];
            ss[i].reset(new mhw_session());
            if (cuts[i] < cuts[i + 1]) mhw::session_create(*ss[i], *g, *model, c);
        });
        std::unique_ptr<mhw_walks> w(new mhw_walks());
        std::vector<uint64_t> row0(n_replicas + 1, 0);
        for (int i = 0; i < n_replicas; ++i) row0[i + 1] = row0[i] + ss[i]->rows;
        w->rows = row0.back();
        w->stride = (config->walk_length + 1 + 3) & ~3u;
        w->nodes.resize(w->rows * w->stride);
        w->lens.resize(w->rows);
        std::vector<mhw_walk_stats> st(n_replicas);
        par([&](int i) {
            if (!ss[i]->g) return;
            mhw::DeviceGuard dg(ss[i]->g->device);
            mhw::session_run(*ss[i], nullptr);
            mhw::session_stats(*ss[i], st[i]);
            mhw::session_download(*ss[i], w->nodes.data() + row0[i] * w->stride, w->lens.data() + row0[i], nullptr);
        });
        mhw_walk_stats t{};
        double wall = 0;
        for (int i = 0; i < n_replicas; ++i) {
            t.walks += st[i].walks;
            t.early_terminations += st[i].early_terminations;
            t.skipped_starts += st[i].skipped_starts;
            t.steps += st[i].steps;
            t.slot_inits += st[i].slot_inits;
            t.chain_retries += st[i].chain_retries;
            t.rejection_trials += st[i].rejection_trials;
            wall = std::max(wall, st[i].walk_seconds);
        }
        // skipped starts outside [b, e) are not walkers of this call
        t.walk_seconds = wall;
        t.steps_per_sec = wall > 0 ? (double)t.steps / wall : 0.0;
        w->stats = t;
        *out = w.release();
    });
}

uint64_t mhw_walks_count(const mhw_walks* w) { return w ? w->rows : 0; }
uint32_t mhw_walks_stride(const mhw_walks* w) { return w ? w->stride : 0; }
const uint32_t* mhw_walks_nodes(const mhw_walks* w) { return w ? w->nodes.data() : nullptr; }
const uint32_t* mhw_walks_lengths(const mhw_walks* w) { return w ? w->lens.data() : nullptr; }

mhw_status mhw_walks_stats(const mhw_walks* w, mhw_walk_stats* stats) {
    return guard([&] {
        need(w, "walks");
        need(stats, "stats");
        *stats = w->stats;
    });
}

void mhw_walks_free(mhw_walks* w) { delete w; }

mhw_status mhw_walks_write(const mhw_walks* w, const char* path) {
    return guard([&] {
        need(w, "walks");
        need(path, "path");
        FILE* f = std::fopen(path, "wb");
        if (!f) throw mhw::Error(MHW_ERR_IO, std::string("cannot open for writing: ") + path);
        std::vector<char> buf;
        buf.reserve(1 << 20);
        char tmp[16];
        for (uint64_t r = 0; r < w->rows; ++r) {
            const uint32_t* row = w->nodes.data() + r * w->stride;
            for (uint32_t i = 0; i < w->lens[r]; ++i) {
                if (i) buf.push_back(' ');
                uint32_t x = row[i];
                int k = 0;
                do {
                    tmp[k++] = (char)('0' + x % 10);
                    x /= 10;
                } while (x);
                while (k) buf.push_back(tmp[--k]);
            }
            buf.push_back('\n');
            if (buf.size() > (1u << 20) - 1024) {
                if (std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) {
                    std::fclose(f);
                    throw mhw::Error(MHW_ERR_IO, std::string("write failed: ") + path);
                }
                buf.clear();
            }
        }
        const bool ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
        if (std::fclose(f) != 0 || !ok) throw mhw::Error(MHW_ERR_IO, std::string("write failed: ") + path);
        // stats sidecar (engine.cpp:248-259)
        const std::string side = std::string(path) + ".stats.jsonl";
        FILE* s = std::fopen(side.c_str(), "wb");
        if (!s) throw mhw::Error(MHW_ERR_IO, "cannot open for writing: " + side);
        const std::string line = mhw::stats_line(w->stats);
        const bool sok = std::fwrite(line.data(), 1, line.size(), s) == line.size();
        if (std::fclose(s) != 0 || !sok) throw mhw::Error(MHW_ERR_IO, "write failed: " + side);
    });
}

mhw_status mhw_partition_nodes(const mhw_graph* g, const mhw_model_desc* model, int32_t parts, uint32_t* cuts) {
    return guard([&] {
        need(g, "graph");
        need(model, "model");
        need(cuts, "cuts");
        mhw::partition_nodes(*const_cast<mhw_graph*>(g), *model, parts, cuts);
    });
}

mhw_status mhw_walk_rows(const mhw_graph* g, const mhw_model_desc* model, const mhw_walk_config* config,
                         uint64_t* rows, uint32_t* stride) {
    return guard([&] {
        need(g, "graph");
        need(model, "model");
        need(config, "config");
        mhw::walk_rows(*const_cast<mhw_graph*>(g), *model, *config, rows, stride);
    });
}

mhw_status mhw_generate_walks_into(const mhw_graph* g, const mhw_model_desc* model,
                                   const mhw_walk_config* config, uint32_t* h_nodes, uint32_t* h_lengths,
                                   uint64_t capacity_rows, mhw_walk_stats* stats) {
    return guard([&] { run_into(g, model, config, h_nodes, h_lengths, capacity_rows, stats, nullptr); });
}

mhw_status mhw_generate_walks_packed(const mhw_graph* g, const mhw_model_desc* model,
                                     const mhw_walk_config* config, uint32_t* h_nodes, uint64_t capacity_nodes,
                                     uint64_t* h_offsets, uint64_t capacity_rows, mhw_walk_stats* stats) {
    return guard([&] {
        need(g, "graph");
        need(model, "model");
        need(config, "config");
        need(h_nodes, "h_nodes");
        need(h_offsets, "h_offsets");
        auto* gg = const_cast<mhw_graph*>(g);
        mhw::DeviceGuard dg(gg->device);
        const bool trace = std::getenv("MHW_TRACE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        mhw_session s;
        mhw::session_create(s, *gg, *model, *config);
        const auto t1 = std::chrono::steady_clock::now();
        if (capacity_rows < s.rows + 1) mhw::invalid("offset buffer too small for the corpus");
        const char* e = std::getenv("MHW_E2E_CHUNKS");
        const int chunks = e ? std::atoi(e) : 8;
        mhw::session_run_packed(s, h_nodes, capacity_nodes, h_offsets, capacity_rows, chunks, stats);
        if (trace) {
            const auto t2 = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[mhw] packed: create %.2f ms, run+copy %.2f ms\n",
                         std::chrono::duration<double, std::milli>(t1 - t0).count(),
                         std::chrono::duration<double, std::milli>(t2 - t1).count());
        }
    });
}

mhw_status mhw_generate_walks_to_file(const mhw_graph* g, const mhw_model_desc* model,
                                      const mhw_walk_config* config, const char* path, mhw_walk_stats* stats) {
    return guard([&] {
        need(g, "graph");
        need(model, "model");
        need(config, "config");
        need(path, "path");
        auto* gg = const_cast<mhw_graph*>(g);
        mhw::DeviceGuard dg(gg->device);
        mhw_session s;
        mhw::session_create(s, *gg, *model, *config);
        mhw::session_run(s, nullptr);
        mhw_walk_stats st{};
        mhw::session_stats(s, st);
        mhw::session_write_corpus(s, path, st);
        if (stats) *stats = st;
    });
}

mhw_status mhw_session_write_corpus(mhw_session* s, const char* path) {
    return guard([&] {
        need(s, "session");
        need(path, "path");
        mhw_walk_stats st{};
        mhw::session_stats(*s, st);
        mhw::session_write_corpus(*s, path, st);
    });
}

mhw_status mhw_session_create(const mhw_graph* g, const mhw_model_desc* model, const mhw_walk_config* config,
                              mhw_session** out) {
    return guard([&] {
        need(out, "out");
        need(g, "graph");
        need(model, "model");
        need(config, "config");
        auto* gg = const_cast<mhw_graph*>(g);
        mhw::DeviceGuard dg(gg->device);
        std::unique_ptr<mhw_session> s(new mhw_session());
        mhw::session_create(*s, *gg, *model, *config);
        *out = s.release();
    });
}

mhw_status mhw_session_run(mhw_session* s, void* stream) {
    return guard([&] {
        need(s, "session");
        mhw::session_run(*s, static_cast<cudaStream_t>(stream));
    });
}

mhw_status mhw_session_select_starts(mhw_session* s, uint32_t count, const uint32_t* starts) {
    return guard([&] {
        need(s, "session");
        mhw::session_select_starts(*s, count, starts);
    });
}

mhw_status mhw_session_stats(mhw_session* s, mhw_walk_stats* stats) {
    return guard([&] {
        need(s, "session");
        need(stats, "stats");
        mhw::session_stats(*s, *stats);
    });
}

mhw_status mhw_session_buffers(mhw_session* s, uint32_t** d_nodes, uint32_t** d_lengths, uint64_t* rows,
                               uint32_t* stride) {
    return guard([&] {
        need(s, "session");
        if (d_nodes) *d_nodes = s->out.p;
        if (d_lengths) *d_lengths = s->lens.p;
        if (rows) *rows = s->rows;
        if (stride) *stride = s->stride;
    });
}

mhw_status mhw_session_download(mhw_session* s, uint32_t* h_nodes, uint32_t* h_lengths, void* stream) {
    return guard([&] {
        need(s, "session");
        mhw::session_download(*s, h_nodes, h_lengths, static_cast<cudaStream_t>(stream));
    });
}

uint32_t mhw_session_launches(const mhw_session* s) { return s ? s->launches : 0; }

mhw_status mhw_session_chain_size(const mhw_session* s, uint64_t* words) {
    return guard([&] {
        need(s, "session");
        need(words, "words");
        *words = mhw::second_order(s->model.dev.kind) ? s->g->m : 0;
    });
}

mhw_status mhw_session_init_chain(mhw_session* s, uint64_t begin, uint64_t end, uint32_t* d_words, void* stream) {
    return guard([&] {
        need(s, "session");
        if (end > begin) need(d_words, "d_words");
        mhw::session_init_chain(*s, begin, end, d_words, static_cast<cudaStream_t>(stream));
    });
}

mhw_status mhw_session_load_chain(mhw_session* s, const uint32_t* d_words, void* stream) {
    return guard([&] {
        need(s, "session");
        need(d_words, "d_words");
        mhw::session_load_chain(*s, d_words, static_cast<cudaStream_t>(stream));
    });
}

mhw_status mhw_session_shard_entry_bytes(const mhw_session* s, uint32_t* bytes) {
    return guard([&] {
        need(s, "session");
        need(bytes, "bytes");
        *bytes = mhw::session_shard_entry_bytes(*s);
    });
}

mhw_status mhw_session_init_shard(mhw_session* s, uint64_t begin, uint64_t end, void* d_out, void* stream) {
    return guard([&] {
        need(s, "session");
        if (end > begin) need(d_out, "d_out");
        mhw::session_init_shard(*s, begin, end, d_out, static_cast<cudaStream_t>(stream));
    });
}

mhw_status mhw_session_load_shard_range(mhw_session* s, uint64_t begin, uint64_t end, const void* d_in,
                                        void* stream) {
    return guard([&] {
        need(s, "session");
        if (end > begin) need(d_in, "d_in");
        mhw::session_load_shard_range(*s, begin, end, d_in, static_cast<cudaStream_t>(stream));
    });
}

mhw_status mhw_session_prepare(mhw_session* s, void* stream) {
    return guard([&] {
        need(s, "session");
        mhw::session_prepare(*s, static_cast<cudaStream_t>(stream));
    });
}

mhw_status mhw_session_export_table(mhw_session* s, uint32_t* d_words, void* stream) {
    return guard([&] {
        need(s, "session");
        need(d_words, "d_words");
        mhw::session_export_table(*s, d_words, static_cast<cudaStream_t>(stream));
    });
}

mhw_status mhw_session_init_records(mhw_session* s, uint64_t begin, uint64_t end, uint32_t* d_words, void* stream) {
    return guard([&] {
        need(s, "session");
        if (end > begin) need(d_words, "d_words");
        mhw::session_init_chain(*s, begin, end, d_words, static_cast<cudaStream_t>(stream), true);
    });
}

mhw_status mhw_session_record_width(const mhw_session* s, uint32_t* width) {
    return guard([&] {
        need(s, "session");
        need(width, "width");
        *width = mhw::session_record_width(*s);
    });
}

mhw_status mhw_session_load_records_range(mhw_session* s, uint64_t begin, uint64_t end, const uint32_t* d_words,
                                          void* stream) {
    return guard([&] {
        need(s, "session");
        if (end > begin) need(d_words, "d_words");
        mhw::session_load_records_range(*s, begin, end, d_words, static_cast<cudaStream_t>(stream));
    });
}

mhw_status mhw_session_load_records(mhw_session* s, const uint32_t* d_words, void* stream) {
    return guard([&] {
        need(s, "session");
        need(d_words, "d_words");
        mhw::session_load_chain(*s, d_words, static_cast<cudaStream_t>(stream), true);
    });
}

void mhw_session_free(mhw_session* s) {
    if (!s) return;
    int dev = s->g ? s->g->device : 0;
    mhw::DeviceGuard dg(dev);
    delete s;
}

mhw_status mhw_decide(const mhw_graph* g, const mhw_model_desc* model, uint64_t count, const uint32_t* position,
                      const uint32_t* affixture, const uint32_t* candidate, const uint32_t* last, const double* u,
                      double* w_cand, double* w_last, uint8_t* accept) {
    return guard([&] {
        need(g, "graph");
        need(model, "model");
        if (count) {
            need(position, "position");
            need(affixture, "affixture");
            need(candidate, "candidate");
            need(last, "last");
            need(u, "u");
            need(w_cand, "w_cand");
            need(w_last, "w_last");
            need(accept, "accept");
        }
        mhw::run_decide(*const_cast<mhw_graph*>(g), *model, count, position, affixture, candidate, last, u, w_cand,
                        w_last, accept);
    });
}

mhw_status mhw_decide_hastings(const mhw_graph* g, const mhw_model_desc* model, uint64_t count,
                               const uint32_t* position, const uint32_t* affixture, const uint32_t* candidate,
                               const uint32_t* last, const double* u, double* r_cand, double* r_last,
                               uint8_t* accept) {
    return guard([&] {
        need(g, "graph");
        need(model, "model");
        if (count) {
            need(position, "position");
            need(affixture, "affixture");
            need(candidate, "candidate");
            need(last, "last");
            need(u, "u");
            need(r_cand, "r_cand");
            need(r_last, "r_last");
            need(accept, "accept");
        }
        mhw::run_decide(*const_cast<mhw_graph*>(g), *model, count, position, affixture, candidate, last, u, r_cand,
                        r_last, accept, true);
    });
}

mhw_status mhw_check(const mhw_graph* g, const mhw_model_desc* model, uint64_t seed, uint64_t count,
                     const uint32_t* position, const uint32_t* affixture, uint64_t draws, double* kl,
                     uint64_t* counts) {
    return guard([&] {
        need(g, "graph");
        need(model, "model");
        if (count) {
            need(position, "position");
            need(affixture, "affixture");
            need(kl, "kl");
        }
        mhw::run_check(*const_cast<mhw_graph*>(g), *model, seed, count, position, affixture, draws, kl, counts);
    });
}

mhw_status mhw_alias_tables(const mhw_graph* g, double* prob, uint32_t* alias) {
    return guard([&] {
        need(g, "graph");
        need(prob, "prob");
        need(alias, "alias");
        mhw::graph_alias_tables(*const_cast<mhw_graph*>(g), prob, alias);
    });
}

mhw_status mhw_init_states(const mhw_graph* g, const mhw_model_desc* model, const mhw_walk_config* config,
                           uint64_t count, const uint32_t* position, const uint32_t* affixture, uint32_t* last) {
    return guard([&] {
        need(g, "graph");
        need(model, "model");
        need(config, "config");
        if (count) {
            need(position, "position");
            need(affixture, "affixture");
            need(last, "last");
        }
        mhw::run_init_states(*const_cast<mhw_graph*>(g), *model, *config, count, position, affixture, last);
    });
}

}  // extern "C"

// ------------------------------------------------------- JSON sidecars
mhw_status mhw_stats_render(const mhw_walk_stats* stats, char* out, size_t cap, size_t* len) {
    return guard([&] {
        need(stats, "stats");
        const std::string line = mhw::stats_line(*stats);
        if (len) *len = line.size();
        if (out) {
            if (cap < line.size() + 1) mhw::invalid("output buffer too small");
            std::memcpy(out, line.c_str(), line.size() + 1);
        }
    });
}

namespace {
std::string manifest_text(const mhw_manifest& m) {
    auto str = [](const char* x) { return std::string(x ? x : ""); };
    mhw::json::Value root;
    root["version"] = mhw::json::Value("0.1.0");
    mhw::json::Value& c = root["config"];
    c["input"] = str(m.input);
    c["weighted"] = m.weighted != 0;
    c["symmetrize"] = m.symmetrize != 0;
    c["model"] = str(m.model);
    c["p"] = m.p;
    c["q"] = m.q;
    c["metapath"] = str(m.metapath);
    c["edge_matrix"] = str(m.edge_matrix);
    c["node_types"] = str(m.node_types);
    c["edge_types"] = str(m.edge_types);
    c["walks_per_node"] = m.walks_per_node;
    c["walk_length"] = m.walk_length;
    c["walk_length_unit"] = mhw::json::Value("steps");
    c["sampler"] = str(m.sampler);
    c["init"] = str(m.init);
    c["burn_in_steps"] = m.burn_in_steps;
    c["hw_sample_size"] = m.hw_sample_size;
    c["threads"] = m.threads;
    c["seed"] = m.seed;
    c["output"] = str(m.output);
    mhw::json::Value& gr = root["graph"];
    gr["nodes"] = m.nodes;
    gr["arcs"] = m.arcs;
    gr["checksum"] = m.checksum;
    mhw::json::Value& t = root["timing"];
    t["T_i"] = m.T_i;
    t["T_w"] = m.T_w;
    return root.dump(2) + "\n";
}
}  // namespace

mhw_status mhw_manifest_render(const mhw_manifest* m, char* out, size_t cap, size_t* len) {
    return guard([&] {
        need(m, "manifest");
        const std::string text = manifest_text(*m);
        if (len) *len = text.size();
        if (out) {
            if (cap < text.size() + 1) mhw::invalid("output buffer too small");
            std::memcpy(out, text.c_str(), text.size() + 1);
        }
    });
}

mhw_status mhw_manifest_write(const mhw_manifest* m) {
    return guard([&] {
        need(m, "manifest");
        need(m->output, "output");
        const std::string path = std::string(m->output) + ".manifest.json";
        const std::string text = manifest_text(*m);
        FILE* f = std::fopen(path.c_str(), "wb");
        if (!f) throw mhw::Error(MHW_ERR_IO, "cannot open for writing: " + path);
        const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
        if (std::fclose(f) != 0 || !ok) throw mhw::Error(MHW_ERR_IO, "write failed: " + path);
    });
}

mhw_status mhw_graph_checksum(const mhw_graph* g, uint64_t* checksum) {
    return guard([&] {
        need(g, "graph");
        need(checksum, "checksum");
        mhw::DeviceGuard dg(g->device);
        const uint64_t m = g->m;
        std::vector<int64_t> off((size_t)g->n + 1);
        std::vector<int32_t> ids((size_t)m);
        std::vector<float> w(g->w.n ? (size_t)m : 0);
        mhw::graph_download(*g, off.data(), ids.data(), w.empty() ? nullptr : w.data(), nullptr, nullptr);
        // FNV-1a, tools/mhwalk.cpp:107-122: strictly sequential (h ^= x; h *= P)
        uint64_t h = 0xcbf29ce484222325ULL;
        auto mix = [&](uint64_t x) {
            h ^= x;
            h *= 0x100000001b3ULL;
        };
        for (const int64_t o : off) mix((uint64_t)o);
        for (const int32_t v : ids) mix((uint64_t)(uint32_t)v);
        uint64_t one = 0;
        const double d1 = 1.0;
        std::memcpy(&one, &d1, 8);
        for (uint64_t a = 0; a < m; ++a) {
            uint64_t bits = one;
            if (!w.empty()) {
                const double d = (double)w[a];
                std::memcpy(&bits, &d, 8);
            }
            mix(bits);
        }
        *checksum = h;
    });
}
