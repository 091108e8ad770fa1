// ref_driver.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. Linked against the reference sources compiled in
// place from /root/reference/proj/src (recipe: oracle/Makefile) into
// oracle/_ref/libmhwalk_ref.so. Used to pin the C restatement (mhw_oracle.c),
// to generate tests/golden fixtures, and as bench.py's CPU reference arm.
// Nothing here is on the product path.
#include "mhwalk/engine.hpp"
#include "mhwalk/errors.hpp"
#include "mhwalk/graph.hpp"
#include "mhwalk/manager.hpp"
#include "mhwalk/models.hpp"
#include "mhwalk/rng.hpp"
#include "mhwalk/samplers.hpp"

#include <nlohmann/json.hpp>

#include <chrono>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

using namespace mhwalk;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const IoError& e) {
        g_err = e.what();
        return 1;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 2;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

struct RefModel {
    WalkModel model;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- graph handles
void* ref_graph_new(uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* nbr,
                    const double* w, const uint16_t* ntype, uint16_t n_ntypes,
                    const uint16_t* etype, uint16_t n_etypes, int symmetric) {
    auto* g = new Graph();
    g->offsets.assign(offsets, offsets + n + 1);
    g->neighbors.assign(nbr, nbr + m);
    if (w) g->weights.assign(w, w + m); else g->weights.assign(m, 1.0);
    if (ntype) g->node_types.assign(ntype, ntype + n);
    if (etype) g->edge_types.assign(etype, etype + m);
    g->num_node_types = n_ntypes;
    g->num_edge_types = n_etypes;
    g->symmetric = symmetric != 0;
    return g;
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

// load_edge_list (graph.cpp:70-100) + optional type files; returns a handle.
int ref_load(const char* path, int weighted, int symmetrize, const char* ntypes_path,
             const char* etypes_path, void** out) {
    return guarded([&] {
        auto* g = new Graph(load_edge_list(path, LoadOptions{weighted != 0, symmetrize != 0}));
        try {
            if (ntypes_path && *ntypes_path) load_node_types(ntypes_path, *g);
            if (etypes_path && *etypes_path) load_edge_types(etypes_path, *g);
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

void ref_graph_sizes(void* gp, uint32_t* n, uint64_t* m, uint16_t* n_ntypes, uint16_t* n_etypes,
                     int* symmetric) {
    auto* g = static_cast<Graph*>(gp);
    *n = g->node_count();
    *m = g->arc_count();
    *n_ntypes = g->num_node_types;
    *n_etypes = g->num_edge_types;
    *symmetric = g->symmetric ? 1 : 0;
}

void ref_graph_copy(void* gp, uint64_t* offsets, uint32_t* nbr, double* w, uint16_t* ntype,
                    uint16_t* etype) {
    auto* g = static_cast<Graph*>(gp);
    std::memcpy(offsets, g->offsets.data(), g->offsets.size() * sizeof(uint64_t));
    std::memcpy(nbr, g->neighbors.data(), g->neighbors.size() * sizeof(uint32_t));
    std::memcpy(w, g->weights.data(), g->weights.size() * sizeof(double));
    if (ntype && !g->node_types.empty())
        std::memcpy(ntype, g->node_types.data(), g->node_types.size() * sizeof(uint16_t));
    if (etype && !g->edge_types.empty())
        std::memcpy(etype, g->edge_types.data(), g->edge_types.size() * sizeof(uint16_t));
}

int ref_write_edge_list(void* gp, const char* path) {
    return guarded([&] { write_edge_list(*static_cast<Graph*>(gp), path); });
}

// ---- models
int ref_model_new(void* gp, int kind, double p, double q, const uint16_t* metapath,
                  uint32_t mp_len, const double* M, uint32_t dim, void** out) {
    return guarded([&] {
        auto* rm = new RefModel();
        rm->model.kind = static_cast<ModelKind>(kind);
        rm->model.p = p;
        rm->model.q = q;
        if (metapath) rm->model.metapath.assign(metapath, metapath + mp_len);
        if (M) {
            rm->model.type_matrix.assign(dim, std::vector<double>(dim));
            for (uint32_t i = 0; i < dim; ++i)
                for (uint32_t j = 0; j < dim; ++j) rm->model.type_matrix[i][j] = M[i * dim + j];
        }
        try {
            rm->model.bind(*static_cast<Graph*>(gp));
        } catch (...) {
            delete rm;
            throw;
        }
        *out = rm;
    });
}

void ref_model_free(void* mp) { delete static_cast<RefModel*>(mp); }

// (state, cand, last, u) -> (wc, wl, accept): calculate_weight (models.cpp:82-123)
// and the verbatim accept expression of mh_transition (samplers.hpp:24).
void ref_decide(void* gp, void* mp, uint64_t count, const uint32_t* pos, const uint32_t* affix,
                const uint32_t* cand, const uint32_t* last, const double* u, double* wc,
                double* wl, uint8_t* accept) {
    const Graph& g = *static_cast<Graph*>(gp);
    const WalkModel& m = static_cast<RefModel*>(mp)->model;
    for (uint64_t i = 0; i < count; ++i) {
        const WalkerState state{pos[i], affix[i]};
        const double c = m.calculate_weight(g, state, {pos[i], cand[i]});
        const double l = m.calculate_weight(g, state, {pos[i], last[i]});
        wc[i] = c;
        wl[i] = l;
        accept[i] = (l <= 0.0 || c >= l || u[i] * l < c) ? 1 : 0;
    }
}

uint64_t ref_slot_count(void* gp, void* mp) {
    return static_cast<RefModel*>(mp)->model.state_count(*static_cast<Graph*>(gp));
}

// ---- samplers
int ref_alias_build(uint32_t n, const double* w, double* prob, uint32_t* alias) {
    return guarded([&] {
        AliasTable t = alias_build(std::span<const double>(w, n));
        std::memcpy(prob, t.prob.data(), n * sizeof(double));
        std::memcpy(alias, t.alias.data(), n * sizeof(uint32_t));
    });
}

// ---- engine: unmodified generate_walks (engine.cpp:157-234)
int ref_generate_walks(void* gp, void* mp, uint32_t K, uint32_t L, uint32_t threads, uint64_t seed,
                       int init_kind, uint32_t burn_in, uint32_t hw, int sampler, uint32_t stride,
                       uint32_t* rows, uint32_t* lens, uint64_t* n_rows, uint64_t* stats,
                       double* times) {
    return guarded([&] {
        WalkConfig cfg;
        cfg.walks_per_node = K;
        cfg.walk_length = L;
        cfg.threads = threads;
        cfg.seed = seed;
        cfg.sampler_kind = static_cast<SamplerKind>(sampler);
        cfg.init.kind = static_cast<InitStrategy::Kind>(init_kind);
        cfg.init.burn_in_steps = burn_in;
        cfg.init.hw_sample_size = hw;
        const auto t0 = std::chrono::steady_clock::now();
        WalkCorpus corpus =
            generate_walks(*static_cast<Graph*>(gp), static_cast<RefModel*>(mp)->model, cfg);
        const auto t1 = std::chrono::steady_clock::now();
        *n_rows = corpus.walks.size();
        if (rows) {
            for (size_t r = 0; r < corpus.walks.size(); ++r) {
                const auto& w = corpus.walks[r];
                std::memcpy(rows + r * stride, w.data(), w.size() * sizeof(uint32_t));
                lens[r] = static_cast<uint32_t>(w.size());
            }
        }
        stats[0] = corpus.stats.walks;
        stats[1] = corpus.stats.early_terminations;
        stats[2] = corpus.stats.skipped_starts;
        stats[3] = corpus.stats.steps;
        times[0] = std::chrono::duration<double>(t1 - t0).count();
        times[1] = corpus.stats.init_seconds;
        times[2] = corpus.stats.steps_per_sec;
    });
}

// ---- CPU baseline over a walker sample: the generate_walks worker loop
// (engine.cpp:178-205) restated over the reference's public APIs
// (SamplerManager::sample manager.hpp:35-36, initial_state/update_state,
// walker_stream rng.hpp:68-76, direct_sample samplers.cpp:133 for the
// bootstrap, engine.cpp:130-134). Walkers idx = begin + j*stride, j < count,
// statically partitioned over `threads` std::threads sharing one manager,
// exactly as generate_walks partitions its walker range.
int ref_walk_sample(void* gp, void* mp, uint32_t K, uint32_t L, uint32_t threads, uint64_t seed,
                    int init_kind, uint32_t burn_in, uint32_t hw, uint64_t begin, uint64_t stride,
                    uint64_t count, uint64_t* stats, double* times) {
    return guarded([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        const WalkModel& m = static_cast<RefModel*>(mp)->model;
        InitStrategy init;
        init.kind = static_cast<InitStrategy::Kind>(init_kind);
        init.burn_in_steps = burn_in;
        init.hw_sample_size = hw;
        SamplerManager manager(g, m);
        if (threads == 0) threads = 1;
        std::vector<uint64_t> steps(threads, 0), walks(threads, 0), early(threads, 0),
            skipped(threads, 0);
        const auto t0 = std::chrono::steady_clock::now();
        auto worker = [&](uint32_t t) {
            const uint64_t b = count * t / threads, e = count * (t + 1) / threads;
            for (uint64_t j = b; j < e; ++j) {
                const uint64_t idx = begin + j * stride;
                const NodeId v = static_cast<NodeId>(idx / K);
                Rng rng = walker_stream(seed, v, idx % K);
                auto state = m.initial_state(g, v);
                if (!state) {
                    ++skipped[t];
                    continue;
                }
                std::vector<NodeId> walk;
                walk.reserve(L + 1);
                walk.push_back(v);
                for (uint32_t step = 0; step < L; ++step) {
                    const uint32_t deg = g.degree(state->position);
                    std::optional<uint32_t> edge;
                    if (deg == 0) {
                        edge = std::nullopt;
                    } else if (m.second_order() && state->affixture == kNoAffix) {
                        auto w = g.weights_of(state->position);
                        if (std::accumulate(w.begin(), w.end(), 0.0) <= 0) edge = std::nullopt;
                        else edge = direct_sample(w, rng);
                    } else {
                        edge = manager.sample(*state, init, rng);
                    }
                    if (!edge) {
                        ++early[t];
                        break;
                    }
                    const EdgeRef chosen{state->position, *edge};
                    walk.push_back(g.neighbor(chosen.source, chosen.neighbor_index));
                    *state = m.update_state(g, *state, chosen);
                    ++steps[t];
                }
                ++walks[t];
            }
        };
        std::vector<std::thread> pool;
        for (uint32_t t = 0; t < threads; ++t) pool.emplace_back(worker, t);
        for (auto& th : pool) th.join();
        const auto t1 = std::chrono::steady_clock::now();
        stats[0] = stats[1] = stats[2] = stats[3] = 0;
        for (uint32_t t = 0; t < threads; ++t) {
            stats[0] += walks[t];
            stats[1] += early[t];
            stats[2] += skipped[t];
            stats[3] += steps[t];
        }
        times[0] = std::chrono::duration<double>(t1 - t0).count();
        times[1] = manager.init_seconds();
    });
}

// ---- the CPU reference arm over the FULL workload, in K time slices.
// One generate_walks call (engine.cpp:157-234) = one SamplerManager over all
// walkers, thread t owning walkers [T*t/threads, T*(t+1)/threads). A run
// handle keeps that manager (and the partition) alive across calls, and call
// i runs slice i of every thread's block: thread t walks
// [b_t + (e_t-b_t)*i/S, b_t + (e_t-b_t)*(i+1)/S). After all S slices every
// walker has walked exactly once against one shared manager, so the summed
// time is a full run's (lazy init amortised exactly as in generate_walks);
// each slice is a bounded step of it. The worker body is the engine loop
// (engine.cpp:186-205) over the public APIs, walks kept per thread as the
// engine keeps them (released after the slice, outside the timing).
struct RefRun {
    const Graph* g;
    const WalkModel* m;
    SamplerManager manager;
    InitStrategy init;
    uint32_t K, L, threads;
    uint64_t seed;
    RefRun(const Graph& gg, const WalkModel& mm) : g(&gg), m(&mm), manager(gg, mm) {}
};

int ref_run_new(void* gp, void* mp, uint32_t K, uint32_t L, uint32_t threads, uint64_t seed, int init_kind,
                uint32_t burn_in, uint32_t hw, void** out) {
    return guarded([&] {
        if (K == 0 || L == 0 || threads == 0)
            throw ValidationError("walks_per_node, walk_length and threads must be positive");
        auto* r = new RefRun(*static_cast<Graph*>(gp), static_cast<RefModel*>(mp)->model);
        r->init.kind = static_cast<InitStrategy::Kind>(init_kind);
        r->init.burn_in_steps = burn_in;
        r->init.hw_sample_size = hw;
        r->K = K;
        r->L = L;
        r->seed = seed;
        const uint64_t total = static_cast<uint64_t>(r->g->node_count()) * K;
        r->threads = static_cast<uint32_t>(std::min<uint64_t>(threads, std::max<uint64_t>(total, 1)));
        *out = r;
    });
}

void ref_run_free(void* h) { delete static_cast<RefRun*>(h); }

int ref_run_slice(void* h, uint32_t slice, uint32_t slices, uint64_t* stats, double* times) {
    return guarded([&] {
        RefRun& R = *static_cast<RefRun*>(h);
        const Graph& g = *R.g;
        const WalkModel& m = *R.m;
        const uint64_t total = static_cast<uint64_t>(g.node_count()) * R.K;
        const uint32_t T = R.threads;
        std::vector<uint64_t> steps(T, 0), walks(T, 0), early(T, 0), skipped(T, 0);
        std::vector<std::vector<std::vector<NodeId>>> outs(T);
        const double init0 = R.manager.init_seconds();
        const auto t0 = std::chrono::steady_clock::now();
        auto worker = [&](uint32_t t) {
            const uint64_t tb = total * t / T, te = total * (t + 1) / T;
            const uint64_t b = tb + (te - tb) * slice / slices, e = tb + (te - tb) * (slice + 1) / slices;
            for (uint64_t idx = b; idx < e; ++idx) {
                const NodeId v = static_cast<NodeId>(idx / R.K);
                Rng rng = walker_stream(R.seed, v, static_cast<uint32_t>(idx % R.K));
                auto state = m.initial_state(g, v);
                if (!state) {
                    ++skipped[t];
                    continue;
                }
                std::vector<NodeId> walk;
                walk.reserve(R.L + 1);
                walk.push_back(v);
                for (uint32_t step = 0; step < R.L; ++step) {
                    const uint32_t deg = g.degree(state->position);
                    std::optional<uint32_t> edge;
                    if (deg == 0) {
                        edge = std::nullopt;
                    } else if (m.second_order() && state->affixture == kNoAffix) {
                        auto w = g.weights_of(state->position);
                        if (std::accumulate(w.begin(), w.end(), 0.0) <= 0) edge = std::nullopt;
                        else edge = direct_sample(w, rng);
                    } else {
                        edge = R.manager.sample(*state, R.init, rng);
                    }
                    if (!edge) {
                        ++early[t];
                        break;
                    }
                    const EdgeRef chosen{state->position, *edge};
                    walk.push_back(g.neighbor(chosen.source, chosen.neighbor_index));
                    *state = m.update_state(g, *state, chosen);
                    ++steps[t];
                }
                outs[t].push_back(std::move(walk));
                ++walks[t];
            }
        };
        std::vector<std::thread> pool;
        for (uint32_t t = 0; t < T; ++t) pool.emplace_back(worker, t);
        for (auto& th : pool) th.join();
        const auto t1 = std::chrono::steady_clock::now();
        stats[0] = stats[1] = stats[2] = stats[3] = 0;
        for (uint32_t t = 0; t < T; ++t) {
            stats[0] += walks[t];
            stats[1] += early[t];
            stats[2] += skipped[t];
            stats[3] += steps[t];
        }
        times[0] = std::chrono::duration<double>(t1 - t0).count();
        times[1] = R.manager.init_seconds() - init0;
    });
}

// ---- JSON sidecars (corpus emission parity, tools/mhwalk.cpp / engine.cpp)
// nlohmann::json(x).dump() of one double (the stats line's number format).
int ref_json_double(double x, char* out, size_t cap) {
    const std::string s = nlohmann::json(x).dump();
    if (s.size() + 1 > cap) return 1;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

// The reference's own write_corpus (engine.cpp:236-259) over a corpus given
// as padded rows: corpus text + <path>.stats.jsonl.
int ref_write_corpus(const char* path, const uint32_t* rows, const uint32_t* lens, uint64_t n_rows,
                     uint32_t stride, const uint64_t* stats, const double* times) {
    return guarded([&] {
        WalkCorpus c;
        c.walks.resize(n_rows);
        for (uint64_t r = 0; r < n_rows; ++r) c.walks[r].assign(rows + r * stride, rows + r * stride + lens[r]);
        c.stats.walks = stats[0];
        c.stats.early_terminations = stats[1];
        c.stats.skipped_starts = stats[2];
        c.stats.steps = stats[3];
        c.stats.steps_per_sec = times[0];
        c.stats.init_seconds = times[1];
        c.stats.walk_seconds = times[2];
        write_corpus(c, path);
    });
}

// cmd_walk's manifest object (tools/mhwalk.cpp:142-169), restated here over
// the same nlohmann types because the CLI itself does not build (CLI11 is
// absent); strs = {input, model, metapath, edge_matrix, node_types,
// edge_types, sampler, init, output}, nums = {p, q, T_i, T_w}, ints = {K, L,
// burn_in, hw, threads, seed, nodes, arcs, checksum}, flags = {weighted,
// symmetrize}. Written with dump(2) and a newline, as cmd_walk writes it.
int ref_manifest(const char* const* strs, const double* nums, const uint64_t* ints, const int* flags,
                 char* out, size_t cap) {
    return guarded([&] {
        nlohmann::json manifest = {
            {"version", "0.1.0"},
            {"config",
             {{"input", std::string(strs[0])},
              {"weighted", flags[0] != 0},
              {"symmetrize", flags[1] != 0},
              {"model", std::string(strs[1])},
              {"p", nums[0]},
              {"q", nums[1]},
              {"metapath", std::string(strs[2])},
              {"edge_matrix", std::string(strs[3])},
              {"node_types", std::string(strs[4])},
              {"edge_types", std::string(strs[5])},
              {"walks_per_node", static_cast<uint32_t>(ints[0])},
              {"walk_length", static_cast<uint32_t>(ints[1])},
              {"walk_length_unit", "steps"},
              {"sampler", std::string(strs[6])},
              {"init", std::string(strs[7])},
              {"burn_in_steps", static_cast<uint32_t>(ints[2])},
              {"hw_sample_size", static_cast<uint32_t>(ints[3])},
              {"threads", static_cast<uint32_t>(ints[4])},
              {"seed", ints[5]},
              {"output", std::string(strs[8])}}},
            {"graph",
             {{"nodes", static_cast<uint32_t>(ints[6])},
              {"arcs", ints[7]},
              {"checksum", ints[8]}}},
            {"timing", {{"T_i", nums[2]}, {"T_w", nums[3]}}},
        };
        const std::string s = manifest.dump(2) + "\n";
        if (s.size() + 1 > cap) throw std::runtime_error("buffer too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
    });
}

}  // extern "C"
