// mhwalk_gpu.hpp -- header-only C++ shim: the reference's walk API on the GPU.
//
//   mhwalk::WalkCorpus mhwalk_gpu::generate_walks(const mhwalk::Graph&,
//                                                  const mhwalk::WalkModel&,
//                                                  const mhwalk::WalkConfig&);
//
// Same signature, argument meaning and exceptions as mhwalk::generate_walks
// (engine.hpp:47, engine.cpp:157-234): the reference's structs are converted
// to the C ABI of libmhw.so (include/mhw.h) and the corpus comes back as a
// mhwalk::WalkCorpus. Include after the reference headers (mhwalk/*.hpp) and
// link -lmhw. Conversions: u64 offsets -> i64, u32 ids -> i32, f64 weights
// rounded to nearest f32 (exact for fp32-representable weights; DESIGN.md
// "Exactness contract"). threads == 1 selects the deterministic schedule.
#pragma once

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "mhw.h"
#include "mhwalk/engine.hpp"
#include "mhwalk/errors.hpp"
#include "mhwalk/graph.hpp"
#include "mhwalk/models.hpp"

namespace mhwalk_gpu {

[[noreturn]] inline void raise(mhw_status rc) {
    const std::string msg = mhw_last_error();
    if (rc == MHW_ERR_IO) throw mhwalk::IoError(msg);
    if (rc == MHW_ERR_INVALID) throw mhwalk::ValidationError(msg);
    throw std::runtime_error("mhw: " + msg);
}

inline void check(mhw_status rc) {
    if (rc != MHW_OK) raise(rc);
}

// Device replica of a reference Graph (RAII).
class DeviceGraph {
public:
    explicit DeviceGraph(const mhwalk::Graph& g, int device = 0) {
        const uint32_t n = g.node_count();
        offsets_.assign(g.offsets.begin(), g.offsets.end());
        ids_.assign(g.neighbors.begin(), g.neighbors.end());
        bool unit = true;
        for (double w : g.weights) unit = unit && w == 1.0;
        if (!unit) weights_.assign(g.weights.begin(), g.weights.end());  // f64 -> f32, nearest
        mhw_graph_view v{};
        v.node_count = n;
        v.arc_count = g.arc_count();
        v.offsets = offsets_.data();
        v.neighbors = ids_.data();
        v.weights = weights_.empty() ? nullptr : weights_.data();
        v.node_types = g.node_types.empty() ? nullptr : g.node_types.data();
        v.edge_types = g.edge_types.empty() ? nullptr : g.edge_types.data();
        v.num_node_types = g.num_node_types;
        v.num_edge_types = g.num_edge_types;
        v.symmetric = g.symmetric ? 1 : 0;
        check(mhw_graph_upload(&v, device, &g_));
    }
    ~DeviceGraph() { mhw_graph_free(g_); }
    DeviceGraph(const DeviceGraph&) = delete;
    DeviceGraph& operator=(const DeviceGraph&) = delete;
    const mhw_graph* get() const { return g_; }

private:
    std::vector<int64_t> offsets_;
    std::vector<int32_t> ids_;
    std::vector<float> weights_;
    mhw_graph* g_ = nullptr;
};

// WalkModel's public fields -> mhw_model_desc (storage kept alive by the holder).
struct ModelDesc {
    mhw_model_desc d{};
    std::vector<double> matrix;
    explicit ModelDesc(const mhwalk::WalkModel& m) {
        d.kind = static_cast<int32_t>(m.kind);
        d.p = m.p;
        d.q = m.q;
        d.metapath = m.metapath.empty() ? nullptr : m.metapath.data();
        d.metapath_len = static_cast<uint32_t>(m.metapath.size());
        for (const auto& row : m.type_matrix) matrix.insert(matrix.end(), row.begin(), row.end());
        d.type_matrix = matrix.empty() ? nullptr : matrix.data();
        d.type_matrix_dim = static_cast<uint32_t>(m.type_matrix.size());
    }
};

// The M-H proposal (an engine extension; the reference proposes uniformly).
enum class Proposal { uniform = MHW_PROPOSAL_UNIFORM, alias = MHW_PROPOSAL_ALIAS };

inline mhw_walk_config to_config(const mhwalk::WalkConfig& c, Proposal proposal = Proposal::uniform) {
    if (c.threads == 0) throw mhwalk::ValidationError("walks_per_node, walk_length and threads must be positive");
    mhw_walk_config w{};
    w.walks_per_node = c.walks_per_node;
    w.walk_length = c.walk_length;
    w.seed = c.seed;
    w.sampler = static_cast<int32_t>(c.sampler_kind);
    w.init_kind = static_cast<int32_t>(c.init.kind);
    w.burn_in_steps = c.init.burn_in_steps;
    w.hw_sample_size = c.init.hw_sample_size;
    w.schedule = c.threads == 1 ? MHW_SCHEDULE_DETERMINISTIC : MHW_SCHEDULE_THROUGHPUT;
    w.proposal = static_cast<int32_t>(proposal);
    return w;
}

inline mhwalk::WalkCorpus generate_walks(const DeviceGraph& g, const mhwalk::WalkModel& model,
                                         const mhwalk::WalkConfig& config, Proposal proposal = Proposal::uniform) {
    ModelDesc md(model);
    const mhw_walk_config wc = to_config(config, proposal);
    mhw_walks* w = nullptr;
    check(mhw_generate_walks(g.get(), &md.d, &wc, &w));
    std::unique_ptr<mhw_walks, void (*)(mhw_walks*)> hold(w, mhw_walks_free);
    mhwalk::WalkCorpus corpus;
    const uint64_t rows = mhw_walks_count(w);
    const uint32_t stride = mhw_walks_stride(w);
    const uint32_t* nodes = mhw_walks_nodes(w);
    const uint32_t* lens = mhw_walks_lengths(w);
    corpus.walks.resize(rows);
    for (uint64_t r = 0; r < rows; ++r) corpus.walks[r].assign(nodes + r * stride, nodes + r * stride + lens[r]);
    mhw_walk_stats st{};
    check(mhw_walks_stats(w, &st));
    corpus.stats.walks = st.walks;
    corpus.stats.early_terminations = st.early_terminations;
    corpus.stats.skipped_starts = st.skipped_starts;
    corpus.stats.steps = st.steps;
    corpus.stats.steps_per_sec = st.steps_per_sec;
    corpus.stats.init_seconds = st.init_seconds;
    corpus.stats.walk_seconds = st.walk_seconds;
    return corpus;
}

// Drop-in for mhwalk::generate_walks (uploads the graph for this call).
inline mhwalk::WalkCorpus generate_walks(const mhwalk::Graph& graph, const mhwalk::WalkModel& model,
                                         const mhwalk::WalkConfig& config, Proposal proposal = Proposal::uniform) {
    DeviceGraph g(graph);
    return generate_walks(g, model, config, proposal);
}

}  // namespace mhwalk_gpu
