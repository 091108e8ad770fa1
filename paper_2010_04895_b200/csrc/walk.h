// walk.h -- walk session (one generate_walks over a start-node range on one
// device) and the kernel parameter blocks.
#pragma once

#include <memory>

#include "internal.h"

namespace mhw {

struct RunParams {
    DevGraph g;
    DevModel m;
    DevCfg cfg;
    const uint32_t* act;      // active start nodes (valid start, degree > 0)
    const uint64_t* act_row;  // first corpus row of each active start node
    uint32_t n_act;
    uint64_t n_items;         // n_act * K walkers
    uint32_t* chain;          // one packed Last word per state slot
    uint32_t rec_u32;         // u32 words per session arc record: 4 (16 B), 8 (typed 32 B), 2 (narrow 8 B)
    uint4* ac;                // node2vec throughput: arc records whose .w is the chain
                              // word of the state entered through that arc (else null)
    uint32_t* c16;            // node2vec compact chains (AR 3): one 16-bit word per forward
                              // arc s->v = state (s, v), two per u32 (else null)
    const uint2* nodes8;      // compact chains: 8-byte node records {off, deg | allpos << 31}
    const uint32_t* src;      // source node of every arc (slot-order init kernels), nullptr: owner search
    uint32_t* out;            // rows x stride walk buffer
    uint32_t stride;
    uint32_t* lens;
    unsigned long long* ctr;  // [0] work counter [1] steps [2] early [3] inits [4] error [5] error arc
};

struct DetState {
    uint32_t* v;
    uint32_t* aff;
    uint32_t* len;
    uint8_t* alive;
    uint64_t* key;
    uint32_t* idx;
    uint32_t* cand;
    uint8_t* ccls;
    double* wc;
    double* u;
    uint32_t* chosen;
};

struct ExactState;

struct Session {
    Graph* g = nullptr;
    Model model;
    DevCfg cfg{};
    mhw_walk_config wc{};
    uint32_t node_begin = 0, node_end = 0;
    DBuf<uint32_t> act, iso;
    DBuf<uint64_t> act_row, iso_row;
    uint32_t n_act = 0, n_iso = 0;
    uint64_t n_items = 0, rows = 0, skipped = 0, slots = 0;
    uint64_t rows_cap = 0, items_cap = 0;  // sizes the buffers were made for (start selections must fit)
    uint32_t stride = 0;
    DBuf<uint32_t> chain, out, lens, rep_group;
    DBuf<double> rep_scale;  // metapath2vec replica weights per node type
    DBuf<uint4> ac;          // session arc records (+ colocated chain words, second order)
    uint32_t rec_u32 = 4;    // u32 words per record: 4, 8 (typed models), 2 (narrow node2vec records)
    DBuf<uint32_t> c16;      // compact 16-bit chain words (node2vec, L2-sized), [c16 | filter copy] when pinned
    const uint32_t* bloom_copy = nullptr;  // the edge filter's copy behind c16 (one persisting window)
    DBuf<uint2> nodes8;      // compact chains: 8-byte node records (half the L2 footprint of NodeRec)
    DBuf<uint32_t> src;      // source node per arc for the slot-order init (eager second-order sessions)
    DBuf<uint32_t> init_bloom;  // compact chains: the eager init's denser edge filter (own build: MHW_INIT_BLOOM_BITS)
    const uint32_t* ib_p = nullptr;  // the init's filter: init_bloom, or the graph's dense filter (Graph::bloom2)
    size_t ib_bytes = 0;
    uint32_t init_bloom_blocks = 0;
    RunParams init_params() const;  // params() with the init's edge filter
    std::unique_ptr<ExactState> ex;  // alias / direct / rejection baselines (exact.cu)
    DBuf<unsigned long long> ctr;
    // deterministic schedule scratch
    DBuf<uint32_t> d_v, d_aff, d_len, d_idx, d_idx2, d_cand, d_chosen;
    DBuf<uint8_t> d_alive, d_ccls, sort_temp;
    DBuf<uint64_t> d_key, d_key2;
    DBuf<double> d_wc, d_u;
    int sort_bits = 1;
    int grid = 0;
    bool eager_init = false;
    bool init_rec_order = false;  // eager init in record order (k_init_rec) rather than slot order
    bool chain_loaded = false;  // mhw_session_load_chain installed the initial table
    bool l2_pin = false;        // persisting L2 window during runs (edge filter, or fairwalk group sizes)
    void* pin_p = nullptr;
    size_t pin_bytes = 0;
    float pin_ratio = 1.0f;     // hitRatio of the window (set-aside / window bytes)
    void* ipin_p = nullptr;     // window of the eager-init launch when it differs (the edge filter only)
    size_t ipin_bytes = 0;
    bool init_unpinned = false;  // the eager-init launch runs without a window
    bool use_ar = false;     // arc-record walk kernel variant
    int minb = 1;
    uint32_t launches = 0;
    cudaStream_t stream = nullptr;
    // ev0 -> evm: eager chain-table init (T_i); evm -> ev1: the walk kernels (T_w)
    cudaEvent_t ev0 = nullptr, evm = nullptr, ev1 = nullptr;

    Session() = default;
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;
    ~Session();
    RunParams params() const;
    int ar_mode() const {
        if (cfg.proposal == MHW_PROPOSAL_ALIAS) return use_ar ? 5 : 4;  // alias proposal on records / plain CSR
        return c16.n ? 3 : (use_ar ? (rec_u32 == 2 ? 2 : 1) : 0);
    }
};

uint64_t k_slots(int kind, const Graph& g);
void session_create(Session& s, Graph& g, const mhw_model_desc& md, const mhw_walk_config& wc);
void session_run(Session& s, cudaStream_t stream);
// Restricts the next runs to the given (ascending) start nodes of the session's
// range; count 0 with starts NULL restores the whole range.
void session_select_starts(Session& s, uint32_t count, const uint32_t* starts);
void walk_rows(Graph& g, const mhw_model_desc& md, const mhw_walk_config& wc, uint64_t* rows, uint32_t* stride);
void session_init_chain(Session& s, uint64_t begin, uint64_t end, uint32_t* d_words, cudaStream_t stream,
                        bool rec_order = false);
void session_load_chain(Session& s, const uint32_t* d_words, cudaStream_t stream, bool rec_order = false);
void session_prepare(Session& s, cudaStream_t stream);
void session_export_table(Session& s, uint32_t* d_words, cudaStream_t stream);
void session_load_records_range(Session& s, uint64_t begin, uint64_t end, const uint32_t* d_words,
                                cudaStream_t stream);
// u32 words per record of a record-order table (3: typed records carry w'(Last)).
uint32_t session_record_width(const Session& s);
// Sharded init in the session's best exchange format (bytes per entry: 2 =
// compact chains, slot order; else record order, 4 x record width).
uint32_t session_shard_entry_bytes(const Session& s);
void session_init_shard(Session& s, uint64_t begin, uint64_t end, void* d_out, cudaStream_t stream);
void session_load_shard_range(Session& s, uint64_t begin, uint64_t end, const void* d_in, cudaStream_t stream);
void session_stats(Session& s, mhw_walk_stats& out);
void session_download(Session& s, uint32_t* nodes, uint32_t* lens, cudaStream_t stream);
void session_write_corpus(Session& s, const char* path, const mhw_walk_stats& st);
void session_run_packed(Session& s, uint32_t* h_nodes, uint64_t cap_nodes, uint64_t* h_offsets,
                        uint64_t cap_rows, int chunks, mhw_walk_stats* stats);
void session_download_packed(Session& s, uint32_t* h_nodes, uint64_t cap_nodes, uint64_t* h_offsets,
                             uint64_t cap_rows, uint64_t* n_nodes, cudaStream_t stream);
void run_decide(Graph& g, const mhw_model_desc& md, uint64_t n, const uint32_t* pos, const uint32_t* aff,
                const uint32_t* cand, const uint32_t* last, const double* u, double* wc, double* wl,
                uint8_t* acc, bool hastings = false);
void run_init_states(Graph& g, const mhw_model_desc& md, const mhw_walk_config& wc, uint64_t n,
                     const uint32_t* pos, const uint32_t* aff, uint32_t* last);
void partition_nodes(Graph& g, const mhw_model_desc& md, int parts, uint32_t* cuts);
void run_check(Graph& g, const mhw_model_desc& md, uint64_t seed, uint64_t n, const uint32_t* pos,
               const uint32_t* aff, uint64_t draws, double* kl, uint64_t* counts);

}  // namespace mhw

struct mhw_session : mhw::Session {};
