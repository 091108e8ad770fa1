/*
 * mhw_oracle.h -- CPU restatement of the mhwalk M-H walk path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the checker the GPU engine is
 * compared against. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. The product path
 * (paper_2010_04895_b200/) never links or calls it.
 *
 * Every function restates the reference algorithm (file:line relative to the
 * reference's proj/ directory) in plain C. Two knobs make the same engine
 * reproduce either side byte for byte:
 *   rng   = OG_RNG_XOSHIRO : reference walker_stream + xoshiro256** draws
 *                            (rng.hpp:8-76), init draws from the walker stream
 *           OG_RNG_PHILOX  : the B200 engine's Philox4x32-10 layout (DESIGN.md
 *                            "Random streams"), init draws keyed by slot
 *   order = OG_ORDER_WALKER: walker-major, exactly engine.cpp:178-205 (threads=1)
 *           OG_ORDER_STEP  : step-major, walker-id order within a step (the
 *                            GPU engine's deterministic mode)
 * (XOSHIRO, WALKER) is pinned against the compiled reference in oracle/_ref and
 * against tests/golden; (PHILOX, STEP) is what the GPU deterministic mode must
 * equal byte for byte.
 */
#ifndef MHW_ORACLE_H
#define MHW_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OG_DEEPWALK = 0, OG_NODE2VEC = 1, OG_METAPATH2VEC = 2, OG_EDGE2VEC = 3, OG_FAIRWALK = 4 };
enum { OG_INIT_RANDOM = 0, OG_INIT_HIGH_WEIGHT = 1, OG_INIT_BURN_IN = 2 };
enum { OG_RNG_XOSHIRO = 0, OG_RNG_PHILOX = 1 };
enum { OG_ORDER_WALKER = 0, OG_ORDER_STEP = 1 };
enum { OG_OK = 0, OG_ERR_IO = 1, OG_ERR_INVALID = 2, OG_ERR_NOMEM = 5 };

#define OG_NO_AFFIX 0xFFFFFFFFu

/* CSR graph (graph.hpp:15-55). weights are never NULL in the oracle. */
typedef struct {
    uint32_t n;
    uint64_t m;
    const uint64_t* offsets;   /* n+1 */
    const uint32_t* nbr;       /* m, sorted per slice */
    const double* w;           /* m */
    const uint16_t* ntype;     /* n or NULL */
    const uint16_t* etype;     /* m or NULL */
    uint16_t n_ntypes;
    uint16_t n_etypes;
    int symmetric;
} og_graph;

/* Bound walk model (models.hpp:40-92). type_counts is filled by og_model_bind. */
typedef struct {
    int kind;
    double p, q;
    const uint16_t* metapath;
    uint32_t mp_len;
    const double* M;      /* dim*dim row-major */
    uint32_t M_dim;
    uint32_t* type_counts; /* n*num_types, owned by caller (fairwalk) */
    uint16_t num_types;
} og_model;

typedef struct {
    uint32_t K, L;
    uint64_t seed;
    int init_kind;
    uint32_t burn_in_steps;
    uint32_t hw_sample_size;
    int rng;
    int order;
    /* node-keyed chain replicas at hubs (engine layout, DESIGN.md "Chain
     * table"); OG_NO_REPLICAS = one chain per state like SamplerManager */
    uint32_t replica_degree;
    /* SamplerKind (engine.hpp:14): mh, or the exact baselines of
     * WalkerContext::next_edge (engine.cpp:88-116) */
    int sampler;
    /* M-H proposal (engine extension, SURVEY 8(b) proposal {uniform, alias}):
     * OG_PROPOSAL_UNIFORM = mh_transition (samplers.hpp:18-27); ALIAS = the
     * node's static-weight alias table (alias_build over weights_of(v),
     * samplers.cpp:95-131) with the Hastings-corrected accept (og_hastings) */
    int proposal;
} og_config;

enum { OG_PROPOSAL_UNIFORM = 0, OG_PROPOSAL_ALIAS = 1 };
/* Philox sub-counter of the accept unit of an alias-proposal step: block
 * (walker, step) with ctr.w = this (word 0 of that block is never a Lemire
 * retry: those use sub-counters 1, 2, ...) */
#define OG_ACCEPT_SUB 0x80000000u

enum { OG_SAMPLER_MH = 0, OG_SAMPLER_ALIAS = 1, OG_SAMPLER_DIRECT = 2, OG_SAMPLER_REJECTION = 3 };

#define OG_NO_REPLICAS 0xFFFFFFFFu

typedef struct {
    uint64_t walks, early, skipped, steps, init_calls;
    uint64_t trials;  /* rejection sampler: proposals drawn */
} og_stats;

/* ------------------------------------------------------------------ RNG */
void og_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void og_philox_key(uint64_t seed, uint32_t domain, uint32_t key[2]);
uint64_t og_splitmix64(uint64_t* state);
/* xoshiro stream of walker (seed,node,k): n draws of uniform_index(bound) */
void og_xoshiro_walker_draws(uint64_t seed, uint64_t node, uint64_t k, uint32_t bound,
                             uint32_t count, uint32_t* out);
uint32_t og_lemire_philox(const uint32_t key[2], uint64_t id, uint32_t blk, uint32_t n);
double og_unit_philox(const uint32_t key[2], uint64_t id, uint32_t blk);

/* ---------------------------------------------------------- graph build */
/* build_csr semantics (graph.cpp:35-66): sort by (src,dst), sum duplicates in
 * input order, n = max id + 1 unless n_nodes > 0. Outputs malloc'd. */
int og_build_csr(uint64_t n_edges, const uint32_t* src, const uint32_t* dst, const double* w,
                 int symmetrize, uint32_t n_nodes, uint32_t* n_out, uint64_t* m_out,
                 uint64_t** offsets, uint32_t** nbr, double** weights);
/* Synthetic generators. Undirected, deduplicated,
 * self-loop-free pair lists; weights (float) per pair; caller symmetrizes. */
int og_rmat_pairs(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                  uint64_t seed, uint64_t* n_pairs, uint32_t** lo, uint32_t** hi);
float og_pair_weight(uint64_t seed, uint32_t lo, uint32_t hi, float wlo, float whi);
uint32_t og_pair_etype(uint64_t seed, uint32_t lo, uint32_t hi, uint32_t n_types);
void og_pair_weights(uint64_t seed, uint64_t n, const uint32_t* lo, const uint32_t* hi, float wlo, float whi,
                     float* out);
void og_pair_etypes(uint64_t seed, uint64_t n, const uint32_t* lo, const uint32_t* hi, uint32_t n_types,
                    uint16_t* out);
/* graph_checksum of tools/mhwalk.cpp:107-122 (FNV-1a; w NULL = all 1.0) */
uint64_t og_graph_checksum(uint32_t n, const uint64_t* offsets, const uint32_t* nbr, const double* w);
int og_hetero_pairs(uint32_t n_nodes, uint64_t seed, uint32_t* nA, uint32_t* nP,
                    uint64_t* n_pairs, uint32_t** lo, uint32_t** hi);
void og_free(void* p);

/* ------------------------------------------------------------- models */
int og_model_bind(const og_graph* g, og_model* m, char* err, size_t errlen);
size_t og_type_counts_size(const og_graph* g);
double og_weight(const og_graph* g, const og_model* m, uint32_t v, uint32_t affix, uint32_t i);
int og_accept(double wc, double wl, double u);
/* (state, cand, last, u) -> (wc, wl, accept), samplers.hpp:21-26 verbatim */
/* Dynamic factor r = w' / w of candidate i (calculate_weight, models.cpp:82-123,
 * without the trailing static weight): deepwalk 1, metapath2vec type match ? 1
 * : 0, bootstrap 1, node2vec alpha, edge2vec alpha * M[in][out], fairwalk
 * alpha / group. */
double og_rfactor(const og_graph* g, const og_model* m, uint32_t v, uint32_t affix, uint32_t i);
/* Hastings accept of an alias (static-weight) proposal: target w' = r * w,
 * proposal q proportional to w, so min(1, w'_c q_l / (w'_l q_c)) = min(1, r_c / r_l):
 * accept iff w_c > 0 && (r_l <= 0 || r_c >= r_l || u * r_l < r_c). */
int og_hastings(double w_c, double r_c, double r_l, double u);
void og_decide_hastings(const og_graph* g, const og_model* m, uint64_t count, const uint32_t* pos,
                        const uint32_t* affix, const uint32_t* cand, const uint32_t* last, const double* u,
                        double* rc, double* rl, uint8_t* accept);
void og_decide(const og_graph* g, const og_model* m, uint64_t count, const uint32_t* pos,
               const uint32_t* affix, const uint32_t* cand, const uint32_t* last,
               const double* u, double* wc, double* wl, uint8_t* accept);

/* ----------------------------------------------------------- samplers */
/* alias_build (samplers.cpp:95-131). returns 0 ok, 2 invalid. */
int og_alias_build(uint32_t n, const double* w, double* prob, uint32_t* alias);
/* per-node alias tables of a CSR (nodes without positive weight: prob 0, alias i) */
void og_alias_tables(uint32_t n, const uint64_t* offsets, const double* w, double* prob, uint32_t* alias);
/* direct_sample given u (samplers.cpp:133-146) */
uint32_t og_direct_sample_u(uint32_t n, const double* w, double u);
/* Per-slot init under the philox layout: returns 1 and *last on success, 0 dead end. */
int og_init_philox(const og_graph* g, const og_model* m, const og_config* c, uint32_t v,
                   uint32_t affix, uint64_t slot, uint32_t* last);
uint64_t og_slot_count(const og_graph* g, const og_model* m);

/* Per-state chain audit of cmd_check (tools/mhwalk.cpp:222-247) under the
 * engine's Philox layout; counts has sum(deg(pos[j])) entries. */
void og_check(const og_graph* g, const og_model* m, uint64_t seed, uint64_t n_states, const uint32_t* pos,
              const uint32_t* affix, uint64_t draws, uint64_t* counts, double* kl);

/* ------------------------------------------------------------- engine */
/* generate_walks (engine.cpp:157-234). rows: (n*K) x stride, lens: n*K.
 * Returns status; err holds the message. */
int og_generate_walks(const og_graph* g, const og_model* m, const og_config* c, uint32_t stride,
                      uint32_t* rows, uint32_t* lens, uint64_t* n_rows, og_stats* stats,
                      char* err, size_t errlen);

/* Every walker of the given starts (K each, walker id v*K + k) run alone with a
 * fresh manager, walker-major, Philox layout (cfg->rng / order ignored). Rows:
 * count*K x stride. */
int og_walk_isolated(const og_graph* g, const og_model* m, const og_config* c, uint64_t count,
                     const uint32_t* starts, uint32_t stride, uint32_t* rows, uint32_t* lens, uint64_t* n_rows,
                     og_stats* stats, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
#endif
