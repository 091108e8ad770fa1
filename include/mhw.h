/*
 * mhw.h -- C ABI of the B200-native M-H random-walk engine (libmhw.so).
 *
 * Drop-in boundary for the reference's walk path (the C++ API of
 * /root/reference/proj, "mhwalk"). Plain C: POD structs, pointers and sizes,
 * no C++ or torch types. Each entry point names the reference interface it
 * replaces (file:line relative to the reference's proj/ directory).
 *
 * Status codes mirror the reference's error classes (errors.hpp:8-21, mapped
 * to exit codes at tools/mhwalk.cpp:529-541):
 *   MHW_OK 0, MHW_ERR_IO 1 (IoError), MHW_ERR_INVALID 2 (ParseError /
 *   ValidationError), MHW_ERR_CUDA 4 (device failure or out of memory).
 * The message of the last failure on the calling thread is mhw_last_error().
 *
 * Threading: every call is blocking and reentrant per handle (a graph or
 * session handle must not be used by two host threads at once). Walker
 * parallelism is internal: GPU threads, plus one host thread per device for
 * mhw_generate_walks_multi.
 */
#ifndef MHW_H
#define MHW_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MHW_API __attribute__((visibility("default")))
#else
#define MHW_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t mhw_status;
#define MHW_OK 0
#define MHW_ERR_IO 1
#define MHW_ERR_INVALID 2
#define MHW_ERR_CUDA 4

/* ModelKind order, models.hpp:13 */
typedef enum {
    MHW_DEEPWALK = 0,
    MHW_NODE2VEC = 1,
    MHW_METAPATH2VEC = 2,
    MHW_EDGE2VEC = 3,
    MHW_FAIRWALK = 4
} mhw_model_kind;

/* InitStrategy::Kind order, samplers.hpp:30 */
typedef enum { MHW_INIT_RANDOM = 0, MHW_INIT_HIGH_WEIGHT = 1, MHW_INIT_BURN_IN = 2 } mhw_init_kind;

/* SamplerKind order, engine.hpp:14. MHW_SAMPLER_MH is the product path; the
 * exact baselines of next_edge (engine.cpp:88-116) run one warp per walker
 * (alias: per-state tables, 12 B x sum of state degrees of device memory or
 * MHW_ERR_INVALID; direct: inverse CDF; rejection: static alias proposal). */
typedef enum {
    MHW_SAMPLER_MH = 0,
    MHW_SAMPLER_ALIAS = 1,
    MHW_SAMPLER_DIRECT = 2,
    MHW_SAMPLER_REJECTION = 3
} mhw_sampler_kind;

/* throughput: persistent kernel; a walker takes its state's chain word as a
 * lock (atomic exchange) for the transition, so every chain is an exact
 * sequential M-H chain (interleaving order not reproducible).
 * deterministic: step-synchronous, same-slot contenders folded in walker-id
 * order; byte-reproducible (the GPU counterpart of threads=1,
 * engine.hpp:43-46). */
typedef enum { MHW_SCHEDULE_THROUGHPUT = 0, MHW_SCHEDULE_DETERMINISTIC = 1 } mhw_schedule;

#define MHW_NO_AFFIX 0xFFFFFFFFu /* kNoAffix, models.hpp:17 */

/* Host view of a CSR graph. Replaces mhwalk::Graph (graph.hpp:15-55) with the
 * device layout's types: int64 offsets, int32 sorted ids, fp32 weights
 * (NULL = unweighted, every weight 1.0), uint16 node/edge types. */
typedef struct mhw_graph_view {
    uint32_t node_count;
    uint64_t arc_count;
    const int64_t* offsets;      /* node_count + 1 */
    const int32_t* neighbors;    /* arc_count, strictly ascending per slice */
    const float* weights;        /* arc_count or NULL */
    const uint16_t* node_types;  /* node_count or NULL */
    const uint16_t* edge_types;  /* arc_count or NULL */
    uint16_t num_node_types;
    uint16_t num_edge_types;
    int32_t symmetric;           /* Graph::symmetric */
} mhw_graph_view;

/* Replaces mhwalk::WalkModel's public fields (models.hpp:40-47). */
typedef struct mhw_model_desc {
    int32_t kind;                 /* mhw_model_kind */
    double p, q;
    const uint16_t* metapath;     /* metapath2vec */
    uint32_t metapath_len;
    const double* type_matrix;    /* edge2vec, dim x dim row-major */
    uint32_t type_matrix_dim;
} mhw_model_desc;

/* Replaces mhwalk::WalkConfig + InitStrategy (engine.hpp:19-26,
 * samplers.hpp:29-34). node_begin/node_end select the walker partition
 * (start nodes [begin, end), end == 0 means all nodes). */
typedef struct mhw_walk_config {
    uint32_t walks_per_node;   /* K, default 10 */
    uint32_t walk_length;      /* L steps, default 80 */
    uint64_t seed;
    int32_t sampler;           /* mhw_sampler_kind */
    int32_t init_kind;         /* mhw_init_kind */
    uint32_t burn_in_steps;    /* default 100 */
    uint32_t hw_sample_size;   /* default 32 */
    int32_t schedule;          /* mhw_schedule */
    uint32_t node_begin;
    uint32_t node_end;
    /* Node-keyed models (deepwalk, metapath2vec): nodes of visit weight
     * d >= D get 2^(floor(log2(d/D))+1) (at most 65536) independent chains
     * per state, picked by walker id. The weight is the degree (deepwalk) or
     * floor(deg * F[type]) (metapath2vec; F_t = share of the metapath's
     * steady cycle at type t * arcs / arcs incident to type t). 0 = auto
     * (metapath2vec: D = 32; deepwalk: the smallest power-of-two D whose
     * replica region is <= 8M chain words); 0xFFFFFFFF = one chain per state
     * exactly as SamplerManager. */
    uint32_t chain_replica_degree;
    /* Second-order slot initialisation: 0 auto, 1 lazy (first query, as
     * manager.cpp:35-56), 2 eager (all slots before the walk; identical
     * values because init randomness is keyed by the slot). */
    int32_t init_mode;
    /* M-H proposal (north star (2)): MHW_PROPOSAL_UNIFORM
     * draws the candidate uniformly over N(v) exactly as mh_transition
     * (samplers.hpp:21); MHW_PROPOSAL_ALIAS draws it from v's static-weight
     * alias table (alias_sample, samplers.hpp:65-68: index on Philox word 0,
     * coin on words 1-2; tables of alias_build, samplers.cpp:95-131) and
     * accepts with the Hastings-corrected ratio min(1, (w'(c) w(l)) / (w'(l)
     * w(c))) = min(1, r_c / r_l), r = w'/w the model's dynamic factor
     * (mhw_decide_hastings), with the unit from sub-block 0x80000000 of the
     * step's Philox block. Throughput schedule and mh sampler only. Chain
     * init (random / high_weight / burn_in) is mh_init's either way. */
    int32_t proposal;
} mhw_walk_config;

typedef enum { MHW_PROPOSAL_UNIFORM = 0, MHW_PROPOSAL_ALIAS = 1 } mhw_proposal;

/* Replaces mhwalk::RunStats (engine.hpp:28-36). init_seconds (T_i) is the
 * device time of the eager chain-table initialisation launch and walk_seconds
 * (T_w) that of the walk kernels (CUDA events on the launch stream); a lazy
 * run initialises slots on first touch inside the walk kernel, so its T_i is
 * 0 and T_w holds the init. steps_per_sec = steps / (T_i + T_w), including
 * init as engine.cpp:231-232 does. */
typedef struct mhw_walk_stats {
    uint64_t walks;
    uint64_t early_terminations;
    uint64_t skipped_starts;
    uint64_t steps;
    uint64_t slot_inits;
    uint64_t chain_retries;   /* lock retries: chain words found locked by another walker */
    double steps_per_sec;
    double init_seconds;
    double walk_seconds;
    uint64_t rejection_trials; /* rejection sampler: proposals drawn */
} mhw_walk_stats;

typedef struct mhw_graph_info {
    uint32_t node_count;
    uint64_t arc_count;
    int32_t weighted;
    int32_t symmetric;          /* the flag */
    int32_t verified_symmetric; /* every arc has its back arc (checked on device) */
    uint16_t num_node_types;
    uint16_t num_edge_types;
    uint32_t max_degree;
    uint32_t isolated_nodes;
    uint64_t device_bytes;
    int32_t device;
} mhw_graph_info;

typedef struct mhw_graph mhw_graph;
typedef struct mhw_walks mhw_walks;
typedef struct mhw_session mhw_session;

MHW_API const char* mhw_last_error(void);
MHW_API const char* mhw_version(void);
MHW_API int32_t mhw_device_count(void);
/* Releases the library's cache of large device blocks (kept between calls
 * to avoid multi-GB cudaMalloc/cudaFree per generate_walks). */
MHW_API void mhw_trim_memory(void);

/* ---- graphs (device-resident CSR) ------------------------------------ */

/* Copies a host CSR to `device`. Replaces constructing mhwalk::Graph in
 * memory (graph.hpp:15-55); validates slices like build_csr's output. */
MHW_API mhw_status mhw_graph_upload(const mhw_graph_view* view, int32_t device, mhw_graph** out);

/* Device CSR build from an edge list with build_csr semantics: sort by
 * (src, dst), duplicates summed, optional symmetrisation without self-loop
 * doubling, n = max id + 1 unless node_count is larger. Replaces
 * load_edge_list's build step (graph.cpp:35-100). */
MHW_API mhw_status mhw_graph_from_edges(uint64_t edge_count, const uint32_t* src, const uint32_t* dst,
                                const float* weights, int32_t symmetrize, uint32_t node_count,
                                int32_t device, mhw_graph** out);

/* Synthetic generators, built on device.
 * weighted = 0 -> unweighted; edge_type_count > 0 -> one uniform type per
 * undirected edge (both directions). */
MHW_API mhw_status mhw_graph_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b,
                                   double c, uint64_t seed, int32_t weighted, float weight_lo,
                                   float weight_hi, uint32_t edge_type_count, int32_t device,
                                   mhw_graph** out);
MHW_API mhw_status mhw_graph_generate_hetero(uint32_t node_count, uint64_t seed, float weight_lo,
                                     float weight_hi, int32_t device, mhw_graph** out);

/* Text ingestion (graph.cpp:70-177): "src dst [weight]" lines, '#'
 * comments, parsed by all host cores with the reference loader's acceptance
 * rules and messages (first bad line in file order: "path:LINE: expected
 * \"src dst [weight]\"", "missing edge weight", "negative edge weight";
 * unreadable file -> MHW_ERR_IO), then build_csr on the device. */
MHW_API mhw_status mhw_graph_load_edge_list(const char* path, int32_t weighted, int32_t symmetrize,
                                            int32_t device, mhw_graph** out);
MHW_API mhw_status mhw_graph_load_node_types(mhw_graph* g, const char* path);
MHW_API mhw_status mhw_graph_load_edge_types(mhw_graph* g, const char* path);
/* The parse alone, on the host (no device needed): the reference's raw edge
 * vector before build_csr (reverse arcs interleaved when symmetrize, decided
 * on the untruncated ids, graph.cpp:94-97), library-allocated arrays released
 * with mhw_free_host. */
MHW_API mhw_status mhw_parse_edge_list(const char* path, int32_t weighted, int32_t symmetrize,
                                       uint64_t* edge_count, uint32_t** src, uint32_t** dst,
                                       double** weights);
MHW_API void mhw_free_host(void* p);

/* load_node_types / load_edge_types (graph.cpp:102-177) from arrays. */
MHW_API mhw_status mhw_graph_set_node_types(mhw_graph* g, const uint16_t* types, uint16_t num_types);
MHW_API mhw_status mhw_graph_set_edge_types(mhw_graph* g, const uint16_t* types, uint16_t num_types);

/* Copy of the graph to another device (peer copy); walkers can then be
 * partitioned across replicas with mhw_generate_walks_multi. */
MHW_API mhw_status mhw_graph_replicate(const mhw_graph* g, int32_t device, mhw_graph** out);

MHW_API mhw_status mhw_graph_info_get(const mhw_graph* g, mhw_graph_info* info);

/* Parity dump of the device CSR into host arrays (any may be NULL). */
MHW_API mhw_status mhw_graph_download(const mhw_graph* g, int64_t* offsets, int32_t* neighbors,
                              float* weights, uint16_t* node_types, uint16_t* edge_types);
MHW_API void mhw_graph_free(mhw_graph* g);

/* ---- walks ------------------------------------------------------------ */

/* Replaces generate_walks (engine.hpp:47, engine.cpp:157-234): blocking,
 * returns a host corpus in the reference's order (walker idx = v*K + k,
 * skipped starts omitted). */
MHW_API mhw_status mhw_generate_walks(const mhw_graph* g, const mhw_model_desc* model,
                              const mhw_walk_config* config, mhw_walks** out);

/* Same, with walkers partitioned across replicas (one host thread per
 * device, contiguous start-node ranges balanced by active walkers). The
 * corpus is the concatenation in replica order. */
MHW_API mhw_status mhw_generate_walks_multi(const mhw_graph* const* replicas, int32_t n_replicas,
                                    const mhw_model_desc* model, const mhw_walk_config* config,
                                    mhw_walks** out);

/* Corpus size of a call (rows = walks incl. isolated starts, stride = padded
 * row length) so callers can provide their own (pinned) buffers. */
MHW_API mhw_status mhw_walk_rows(const mhw_graph* g, const mhw_model_desc* model, const mhw_walk_config* config,
                         uint64_t* rows, uint32_t* stride);

/* generate_walks into caller-owned host buffers (rows x stride nodes,
 * rows lengths); capacity_rows guards the buffer size. */
MHW_API mhw_status mhw_generate_walks_into(const mhw_graph* g, const mhw_model_desc* model,
                                   const mhw_walk_config* config, uint32_t* h_nodes,
                                   uint32_t* h_lengths, uint64_t capacity_rows,
                                   mhw_walk_stats* stats);

/* generate_walks into a packed host corpus: walk r is
 * h_nodes[h_offsets[r] .. h_offsets[r+1]) (h_offsets has rows + 1 entries).
 * The padded device rows are compacted on the device first, so the D2H
 * carries only the sum of walk lengths. */
MHW_API mhw_status mhw_generate_walks_packed(const mhw_graph* g, const mhw_model_desc* model,
                                     const mhw_walk_config* config, uint32_t* h_nodes,
                                     uint64_t capacity_nodes, uint64_t* h_offsets,
                                     uint64_t capacity_rows, mhw_walk_stats* stats);

MHW_API uint64_t mhw_walks_count(const mhw_walks* w);
MHW_API uint32_t mhw_walks_stride(const mhw_walks* w);
MHW_API const uint32_t* mhw_walks_nodes(const mhw_walks* w);   /* count x stride, row r = walk r */
MHW_API const uint32_t* mhw_walks_lengths(const mhw_walks* w); /* count */
MHW_API mhw_status mhw_walks_stats(const mhw_walks* w, mhw_walk_stats* stats);
MHW_API void mhw_walks_free(mhw_walks* w);

/* Writes the corpus like write_corpus (engine.cpp:236-259): one walk per
 * line, space separated, plus <path>.stats.jsonl. */
MHW_API mhw_status mhw_walks_write(const mhw_walks* w, const char* path);

/* The stats sidecar line of write_corpus (engine.cpp:248-259): the bytes of
 * nlohmann::json::dump() of {walks, early_terminations, skipped_starts,
 * steps, steps_per_sec, init_seconds, walk_seconds} plus '\n' (sorted keys,
 * shortest round-trip doubles). *len = bytes without the terminating NUL;
 * status 2 when cap is too small. */
MHW_API mhw_status mhw_stats_render(const mhw_walk_stats* stats, char* out, size_t cap, size_t* len);

/* cmd_walk's run manifest (tools/mhwalk.cpp:142-169), rendered like
 * nlohmann's dump(2) plus '\n'. Strings are the CLI's flag values ("" when
 * unset); checksum = graph_checksum (tools/mhwalk.cpp:107-122, see
 * mhw_graph_checksum); T_i / T_w = mhw_walk_stats init_seconds / walk_seconds. */
typedef struct mhw_manifest {
    const char* input;
    int32_t weighted;
    int32_t symmetrize;
    const char* model;        /* "deepwalk" | "node2vec" | ... */
    double p;
    double q;
    const char* metapath;     /* comma-separated type ids as given */
    const char* edge_matrix;
    const char* node_types;
    const char* edge_types;
    uint32_t walks_per_node;
    uint32_t walk_length;
    const char* sampler;      /* "mh" | "alias" | "direct" | "rejection" */
    const char* init;         /* "random" | "high_weight" | "burn_in" */
    uint32_t burn_in_steps;
    uint32_t hw_sample_size;
    uint32_t threads;
    uint64_t seed;
    const char* output;
    uint32_t nodes;
    uint64_t arcs;
    uint64_t checksum;
    double T_i;
    double T_w;
} mhw_manifest;
MHW_API mhw_status mhw_manifest_render(const mhw_manifest* m, char* out, size_t cap, size_t* len);
/* Writes <m->output>.manifest.json. */
MHW_API mhw_status mhw_manifest_write(const mhw_manifest* m);
/* graph_checksum (tools/mhwalk.cpp:107-122): FNV-1a over the reference
 * Graph's offsets (u64), neighbours and f64 weight bits (1.0 when
 * unweighted), computed from the device CSR. */
MHW_API mhw_status mhw_graph_checksum(const mhw_graph* g, uint64_t* checksum);

/* generate_walks + write_corpus with the text formatted on the device
 * (integer-to-text kernels, chunked pinned D2H overlapping fwrite); same
 * bytes as write_corpus (engine.cpp:236-259) plus <path>.stats.jsonl. */
MHW_API mhw_status mhw_generate_walks_to_file(const mhw_graph* g, const mhw_model_desc* model,
                                              const mhw_walk_config* config, const char* path,
                                              mhw_walk_stats* stats);

/* Balanced walker partition: cut points of [0, n) into `parts` contiguous
 * start-node ranges with equal active-walker counts.
 * cuts has parts + 1 entries. */
MHW_API mhw_status mhw_partition_nodes(const mhw_graph* g, const mhw_model_desc* model, int32_t parts,
                               uint32_t* cuts);

/* ---- device-resident sessions (benchmarks, repeated runs) ------------- */

MHW_API mhw_status mhw_session_create(const mhw_graph* g, const mhw_model_desc* model,
                              const mhw_walk_config* config, mhw_session** out);
/* Enqueues one full generate_walks on `stream` (cudaStream_t, NULL = the
 * session's own): chain table reset to EMPTY, then the walk kernels. The
 * corpus stays in HBM. */
MHW_API mhw_status mhw_session_run(mhw_session* s, void* stream);
/* Restricts the next runs to the given start nodes (strictly ascending,
 * inside the session's node range): the corpus holds their K walks each in
 * the reference order (engine.cpp:178-191 over that subset); count 0 with
 * starts NULL restores the whole range. Walker ids, chains and draws are the
 * ones of the full run (walker v*K + k), so a single-start selection with
 * K = 1 runs one walker alone, deterministically. */
MHW_API mhw_status mhw_session_select_starts(mhw_session* s, uint32_t count, const uint32_t* starts);
/* Synchronizes and fetches the counters of the last run. */
MHW_API mhw_status mhw_session_stats(mhw_session* s, mhw_walk_stats* stats);
/* Device pointers of the padded walk buffer (rows x stride) and lengths. */
MHW_API mhw_status mhw_session_buffers(mhw_session* s, uint32_t** d_nodes, uint32_t** d_lengths,
                               uint64_t* rows, uint32_t* stride);
/* D2H of the corpus into caller buffers (pinned for full speed). */
MHW_API mhw_status mhw_session_download(mhw_session* s, uint32_t* h_nodes, uint32_t* h_lengths,
                                void* stream);
/* Writes the last run's corpus like mhw_generate_walks_to_file. */
MHW_API mhw_status mhw_session_write_corpus(mhw_session* s, const char* path);
/* Number of kernels the last mhw_session_run enqueued. */
MHW_API uint32_t mhw_session_launches(const mhw_session* s);
/* Sharded chain initialisation (second-order models, multi-GPU): the initial
 * chain table is a pure function of (graph, model, init strategy, seed, slot)
 * (slot-keyed init draws, mh_init samplers.cpp:37-83), so ranks can each
 * initialise a slot range and all-gather the words instead of every rank
 * initialising every slot. chain_size = slots (arcs); init_chain writes the
 * initial words of slots [begin, end) to d_words (device, end - begin
 * entries) on `stream`; load_chain installs a full table (chain_size words)
 * for the NEXT mhw_session_run, which then skips its reset and eager init. */
MHW_API mhw_status mhw_session_chain_size(const mhw_session* s, uint64_t* words);
MHW_API mhw_status mhw_session_init_chain(mhw_session* s, uint64_t begin, uint64_t end, uint32_t* d_words,
                                          void* stream);
MHW_API mhw_status mhw_session_load_chain(mhw_session* s, const uint32_t* d_words, void* stream);
/* Resets and eagerly initialises the session's own chain table (what
 * mhw_session_run does before its walk) without walking; the next run starts
 * from it. Lazy sessions (init_mode 1) get an empty table. */
MHW_API mhw_status mhw_session_prepare(mhw_session* s, void* stream);
/* The installed chain table, one u32 per arc a (chain_size entries, device
 * pointer): the compact 16-bit word (node2vec compact chains), the colocated
 * word of record a, or the slot-order word a -- comparable between sessions
 * of one layout (e.g. a sharded install against a local one). */
MHW_API mhw_status mhw_session_export_table(mhw_session* s, uint32_t* d_words, void* stream);
/* The same table in RECORD order: word i belongs to arc i = (s -> v), i.e.
 * to state (s, v), slot off(v) + index of s in N(v). Sessions keep each
 * second-order chain word in the record of the arc that enters its state, so
 * a record-order table installs with one coalesced strided copy
 * (load_records) instead of a random scatter (load_chain); ranks all-gather
 * contiguous record ranges exactly as with init_chain. Entry i of
 * init_records holds word (off(v) + rev(i)) of init_chain; an entry is
 * record_width u32 words: 1, or 3 for edge2vec / fairwalk sessions, whose
 * records cache w'(Last) beside the word ({word, w'(Last) as f64 lo, hi}),
 * so the install computes nothing. d_words holds (end - begin) * width words. */
MHW_API mhw_status mhw_session_record_width(const mhw_session* s, uint32_t* width);
MHW_API mhw_status mhw_session_init_records(mhw_session* s, uint64_t begin, uint64_t end, uint32_t* d_words,
                                            void* stream);
MHW_API mhw_status mhw_session_load_records(mhw_session* s, const uint32_t* d_words, void* stream);
/* Installs entries [begin, end) only (d_words points at entry begin): lets a
 * caller install each piece of the table as soon as its all-gather lands,
 * overlapping the next piece's transfer. The next run counts the table as
 * loaded; the caller installs every piece before it. */
MHW_API mhw_status mhw_session_load_records_range(mhw_session* s, uint64_t begin, uint64_t end,
                                                  const uint32_t* d_words, void* stream);
/* Sharded chain-table initialisation in the exchange format the session
 * prefers (what bench.py's multi-GPU path uses): entries [begin, end) of
 * chain_size are computed by init_shard into d_out (entry_bytes each), the
 * ranks all-gather them, and load_shard_range installs any range. Compact
 * node2vec chains exchange 2-byte words in slot order (slot-order init keeps
 * N(v) locality; install scatters into the records); other layouts exchange
 * record-order entries (mhw_session_init_records / _load_records_range). */
MHW_API mhw_status mhw_session_shard_entry_bytes(const mhw_session* s, uint32_t* bytes);
MHW_API mhw_status mhw_session_init_shard(mhw_session* s, uint64_t begin, uint64_t end, void* d_out, void* stream);
MHW_API mhw_status mhw_session_load_shard_range(mhw_session* s, uint64_t begin, uint64_t end, const void* d_in,
                                                void* stream);
MHW_API void mhw_session_free(mhw_session* s);

/* ---- parity entry points ---------------------------------------------- */

/* (state, candidate, last, u) -> (w'(cand), w'(last), accept) on device, for
 * host arrays of `count` triples. calculate_weight (models.cpp:82-123) and
 * the accept rule of mh_transition (samplers.hpp:21-26). */
MHW_API mhw_status mhw_decide(const mhw_graph* g, const mhw_model_desc* model, uint64_t count,
                      const uint32_t* position, const uint32_t* affixture,
                      const uint32_t* candidate, const uint32_t* last, const double* u,
                      double* w_cand, double* w_last, uint8_t* accept);

/* The alias proposal's decision (engine extension, mhw_walk_config.proposal
 * = MHW_PROPOSAL_ALIAS): r = w'/w, the model's dynamic factor (calculate_weight,
 * models.cpp:82-123, without the trailing static weight), for candidate and
 * last, and the Hastings accept of a static-weight proposal:
 * w(cand) > 0 && (r_l <= 0 || r_c >= r_l || u * r_l < r_c). */
MHW_API mhw_status mhw_decide_hastings(const mhw_graph* g, const mhw_model_desc* model, uint64_t count,
                      const uint32_t* position, const uint32_t* affixture,
                      const uint32_t* candidate, const uint32_t* last, const double* u,
                      double* r_cand, double* r_last, uint8_t* accept);

/* The `check` audit (tools/mhwalk.cpp:183-264) on the GPU: for each state,
 * random init then `draws` M-H transitions counting the chain's states, and
 * KL(empirical || exact normalised w') (analysis.cpp:34-45) into kl[j] (NaN
 * when the target has no mass or init dead-ends). counts (optional) receives
 * the per-candidate visit counts, deg(position[j]) entries per state in order.
 * A caller reproduces cmd_check's exit code as max(kl) < tolerance ? 0 : 3. */
MHW_API mhw_status mhw_check(const mhw_graph* g, const mhw_model_desc* model, uint64_t seed,
                             uint64_t count, const uint32_t* position, const uint32_t* affixture,
                             uint64_t draws, double* kl, uint64_t* counts);

/* Per-node static-weight alias tables, alias_build (samplers.cpp:95-131),
 * into host arrays of arc_count entries (node v's table at offsets[v]). */
MHW_API mhw_status mhw_alias_tables(const mhw_graph* g, double* prob, uint32_t* alias);

/* Slot initialisation of (position, affixture) states under the engine's
 * slot-keyed Philox layout (mh_init, samplers.cpp:37-83); returns the initial
 * Last index or MHW_NO_AFFIX for a dead end. */
MHW_API mhw_status mhw_init_states(const mhw_graph* g, const mhw_model_desc* model,
                           const mhw_walk_config* config, uint64_t count,
                           const uint32_t* position, const uint32_t* affixture, uint32_t* last);

#ifdef __cplusplus
}
#endif
#endif /* MHW_H */
