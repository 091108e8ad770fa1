// shim_test.cpp -- the reference's engine tests (tests/test_engine.cpp:40-134,
// acceptance.cpp:266-304) run UNCHANGED in spirit through the drop-in
// mhwalk_gpu::generate_walks, with the reference's own Graph / WalkModel /
// WalkConfig types and test builders (tests/oracles.hpp, included at compile
// time from the reference tree). Exit code = number of failed checks.
#include "mhwalk/engine.hpp"
#include "mhwalk/models.hpp"
#include "oracles.hpp"
#include "mhwalk_gpu.hpp"

#include <cstdio>

using namespace mhwalk;

static int failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            ++failures;                                                          \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
        }                                                                        \
    } while (0)

static WalkModel make_bound(ModelKind kind, const Graph& g, double p = 1.0, double q = 1.0) {
    WalkModel m;
    m.kind = kind;
    m.p = p;
    m.q = q;
    if (kind == ModelKind::metapath2vec) m.metapath = {0, 1, 0};
    if (kind == ModelKind::edge2vec) {
        const size_t dim = g.edge_type_count();
        m.type_matrix.assign(dim, std::vector<double>(dim, 1.0));
    }
    m.bind(g);
    return m;
}

static bool walks_valid(const Graph& g, const WalkCorpus& c) {
    for (const auto& w : c.walks) {
        if (w.empty()) return false;
        for (size_t i = 1; i < w.size(); ++i)
            if (!g.is_adjacent(w[i - 1], w[i])) return false;
    }
    return true;
}

int main() {
    {   // isolated node emits length-1 walks and counts terminations
        Graph g = oracles::make_graph(1, {}, true);
        WalkConfig config{.walks_per_node = 2, .walk_length = 80};
        WalkCorpus c = mhwalk_gpu::generate_walks(g, make_bound(ModelKind::deepwalk, g), config);
        CHECK(c.walks.size() == 2);
        for (const auto& w : c.walks) CHECK(w == std::vector<NodeId>{0});
        CHECK(c.stats.early_terminations == 2);
    }
    {   // triangle deepwalk produces full-length valid walks
        Graph g = oracles::triangle();
        WalkConfig config{.walks_per_node = 1, .walk_length = 3, .seed = 9};
        WalkCorpus c = mhwalk_gpu::generate_walks(g, make_bound(ModelKind::deepwalk, g), config);
        CHECK(c.walks.size() == 3);
        for (const auto& w : c.walks) CHECK(w.size() == 4);
        CHECK(walks_valid(g, c));
        CHECK(c.walks[0][0] == 0 && c.walks[1][0] == 1 && c.walks[2][0] == 2);
    }
    {   // walk count equals (nodes - skipped) * K
        Rng rng(1);
        Graph g = oracles::random_graph(60, 5.0, false, rng);
        oracles::assign_random_types(g, 2, rng);
        WalkConfig config{.walks_per_node = 3, .walk_length = 10, .seed = 2};
        WalkCorpus c = mhwalk_gpu::generate_walks(g, make_bound(ModelKind::metapath2vec, g), config);
        CHECK(c.walks.size() == uint64_t(g.node_count()) * 3 - c.stats.skipped_starts);
        CHECK(c.stats.skipped_starts > 0);
    }
    {   // every model emits edge-valid walks (weights rounded to fp32 on device)
        Rng rng(3);
        Graph g = oracles::random_graph(80, 6.0, true, rng);
        oracles::assign_random_types(g, 2, rng);
        for (auto kind : {ModelKind::deepwalk, ModelKind::node2vec, ModelKind::metapath2vec,
                          ModelKind::edge2vec, ModelKind::fairwalk}) {
            for (uint32_t threads : {1u, 8u}) {
                WalkConfig config{.walks_per_node = 2, .walk_length = 20, .threads = threads, .seed = 4};
                CHECK(walks_valid(g, mhwalk_gpu::generate_walks(g, make_bound(kind, g, 0.5, 2.0), config)));
            }
        }
    }
    {   // every sampler kind emits edge-valid walks (test_engine.cpp:88-98)
        Rng rng(5);
        Graph g = oracles::random_graph(60, 5.0, true, rng);
        for (auto kind : {SamplerKind::mh, SamplerKind::alias, SamplerKind::direct, SamplerKind::rejection}) {
            WalkModel m = make_bound(ModelKind::node2vec, g, 0.5, 2.0);
            WalkConfig config{.walks_per_node = 2, .walk_length = 15, .seed = 6, .sampler_kind = kind};
            WalkCorpus c = mhwalk_gpu::generate_walks(g, m, config);
            CHECK(c.walks.size() == 120);
            CHECK(walks_valid(g, c));
        }
    }
    {   // metapath walks follow the metapath cyclically
        Rng rng(7);
        Graph g = oracles::random_graph(80, 8.0, false, rng);
        oracles::assign_random_types(g, 2, rng);
        WalkConfig config{.walks_per_node = 3, .walk_length = 20, .seed = 8};
        WalkCorpus c = mhwalk_gpu::generate_walks(g, make_bound(ModelKind::metapath2vec, g), config);
        CHECK(!c.walks.empty());
        for (const auto& w : c.walks)
            for (size_t i = 0; i < w.size(); ++i) CHECK(g.node_type(w[i]) == (i % 2 == 0 ? 0 : 1));
    }
    {   // single-threaded seeded runs are identical
        Rng rng(9);
        Graph g = oracles::random_graph(100, 5.0, true, rng);
        WalkModel m = make_bound(ModelKind::node2vec, g, 0.25, 4.0);
        WalkConfig config{.walks_per_node = 2, .walk_length = 30, .threads = 1, .seed = 1234};
        CHECK(mhwalk_gpu::generate_walks(g, m, config).walks == mhwalk_gpu::generate_walks(g, m, config).walks);
    }
    {   // multithreaded runs produce the right number of valid walks
        Rng rng(10);
        Graph g = oracles::random_graph(100, 5.0, false, rng);
        WalkConfig config{.walks_per_node = 4, .walk_length = 20, .threads = 4, .seed = 11};
        WalkCorpus c = mhwalk_gpu::generate_walks(g, make_bound(ModelKind::deepwalk, g), config);
        CHECK(c.walks.size() == 400);
        CHECK(walks_valid(g, c));
    }
    {   // acceptance 8: 10,000 walks valid, metapath compliance
        Rng rng(1008);
        Graph g = oracles::random_graph(1000, 8.0, true, rng);
        oracles::assign_random_types(g, 2, rng);
        WalkConfig config{.walks_per_node = 10, .walk_length = 40, .threads = 1, .seed = 1008};
        WalkCorpus c = mhwalk_gpu::generate_walks(g, make_bound(ModelKind::node2vec, g, 0.5, 2.0), config);
        CHECK(c.walks.size() == 10000);
        CHECK(walks_valid(g, c));
    }
    {   // the engine's alias proposal (extension): valid walks for every model
        Rng rng(1009);
        Graph g = oracles::random_graph(300, 6.0, true, rng);
        oracles::assign_random_types(g, 2, rng);
        WalkConfig config{.walks_per_node = 4, .walk_length = 20, .threads = 8, .seed = 9};
        for (ModelKind kind : {ModelKind::deepwalk, ModelKind::node2vec, ModelKind::fairwalk}) {
            WalkCorpus c = mhwalk_gpu::generate_walks(g, make_bound(kind, g, 0.5, 2.0), config,
                                                      mhwalk_gpu::Proposal::alias);
            CHECK(c.walks.size() == 1200);
            CHECK(walks_valid(g, c));
        }
    }
    {   // errors: second-order on an asymmetric graph -> ValidationError from bind
        Graph g = oracles::make_graph(2, {{0, 1, 1.0}}, false);
        WalkModel m;
        m.kind = ModelKind::node2vec;
        bool threw = false;
        try {
            WalkConfig config;
            mhwalk_gpu::generate_walks(g, m, config);
        } catch (const ValidationError&) {
            threw = true;
        }
        CHECK(threw);
    }
    std::printf("%s: %d failed checks\n", failures ? "FAIL" : "PASS", failures);
    return failures;
}
