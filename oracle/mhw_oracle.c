/*
 * mhw_oracle.c -- CPU restatement of the mhwalk M-H walk path.
 *
 * TEST INFRASTRUCTURE ONLY (the checker, never the product). See mhw_oracle.h.
 * Citations are file:line relative to the reference's proj/ directory.
 * Compiled with -ffp-contract=off so every double expression rounds exactly as
 * written (the decision path must not be FMA-contracted).
 */
#define _GNU_SOURCE
#include "mhw_oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <time.h>

/* ================================================================== RNG */

/* splitmix64, rng.hpp:8-13 */
uint64_t og_splitmix64(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* xoshiro256** seeded by splitmix64, rng.hpp:17-40 */
typedef struct { uint64_t s[4]; } xo_t;

static void xo_seed(xo_t* r, uint64_t seed) {
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = og_splitmix64(&sm);
}
static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t xo_next(xo_t* r) {
    const uint64_t result = rotl64(r->s[1] * 5, 7) * 9;
    const uint64_t t = r->s[1] << 17;
    r->s[2] ^= r->s[0];
    r->s[3] ^= r->s[1];
    r->s[1] ^= r->s[2];
    r->s[0] ^= r->s[3];
    r->s[2] ^= t;
    r->s[3] = rotl64(r->s[3], 45);
    return result;
}
/* uniform_index: Lemire with rejection on the high 32 bits, rng.hpp:42-55 */
static uint32_t xo_index(xo_t* r, uint32_t n) {
    uint64_t x = xo_next(r) >> 32;
    uint64_t m = x * (uint64_t)n;
    uint64_t lo = m & 0xffffffffULL;
    if (lo < n) {
        uint64_t threshold = (0x100000000ULL - n) % n;
        while (lo < threshold) {
            x = xo_next(r) >> 32;
            m = x * (uint64_t)n;
            lo = m & 0xffffffffULL;
        }
    }
    return (uint32_t)(m >> 32);
}
/* uniform_real: 53 bits, rng.hpp:58-60 */
static double xo_real(xo_t* r) { return (double)(xo_next(r) >> 11) * 0x1.0p-53; }

/* walker_stream, rng.hpp:68-76 */
static void xo_walker(xo_t* r, uint64_t seed, uint64_t node, uint64_t k) {
    uint64_t sm = seed;
    uint64_t a = og_splitmix64(&sm);
    sm ^= node * 0x9e3779b97f4a7c15ULL + 0x7f4a7c15ULL;
    uint64_t b = og_splitmix64(&sm);
    sm ^= k * 0xbf58476d1ce4e5b9ULL + 0x1ce4e5b9ULL;
    uint64_t c = og_splitmix64(&sm);
    xo_seed(r, a ^ (b + c));
}

void og_xoshiro_walker_draws(uint64_t seed, uint64_t node, uint64_t k, uint32_t bound,
                             uint32_t count, uint32_t* out) {
    xo_t r;
    xo_walker(&r, seed, node, k);
    for (uint32_t i = 0; i < count; ++i) out[i] = xo_index(&r, bound);
}

/* Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
 * 1, 2, 3"): 10 rounds of the 4x32 S-box with Weyl key schedule. */
void og_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Domain-separated key: (lo32(seed), hi32(seed) ^ domain). */
void og_philox_key(uint64_t seed, uint32_t domain, uint32_t key[2]) {
    key[0] = (uint32_t)seed;
    key[1] = (uint32_t)(seed >> 32) ^ domain;
}

#define DOM_WALK   0x00000000u
#define DOM_INIT   0x5EED1417u
#define DOM_RMAT   0x2A7E0001u
#define DOM_WEIGHT 0x3E1647u
#define DOM_ETYPE  0x7E7E0003u
#define DOM_HETERO 0x4E7E0004u
#define DOM_REJECT 0x2E1EC705u

/* One "transition block": the draws of one M-H transition / one init pick.
 * xoshiro: sequential stream (reference). philox: block (id, blk) gives
 * w0 -> candidate (Lemire), (w1,w2) -> 53-bit unit, w3 then sub-blocks
 * (ctr[3] = 1, 2, ...) -> Lemire retry words. */
typedef struct {
    int philox;
    xo_t* xo;
    uint32_t key[2];
    uint32_t ctr[4];
    uint32_t w[4];
    uint32_t rpos;
} draw_t;

static void draw_open(draw_t* d, int philox, xo_t* xo, const uint32_t key[2], uint64_t id,
                      uint32_t blk) {
    d->philox = philox;
    d->xo = xo;
    if (!philox) return;
    d->key[0] = key[0];
    d->key[1] = key[1];
    d->ctr[0] = (uint32_t)id;
    d->ctr[1] = (uint32_t)(id >> 32);
    d->ctr[2] = blk;
    d->ctr[3] = 0;
    og_philox4x32_10(d->ctr, d->key, d->w);
    d->rpos = 3;
}
/* block (id, blk) with sub-counter ctr[3] = sub (rejection trials) */
static void draw_open_sub(draw_t* d, int philox, xo_t* xo, const uint32_t key[2], uint64_t id,
                          uint32_t blk, uint32_t sub) {
    draw_open(d, philox, xo, key, id, blk);
    if (!philox) return;
    d->ctr[3] = sub;
    og_philox4x32_10(d->ctr, d->key, d->w);
}
static uint32_t draw_retry_word(draw_t* d) {
    if (d->rpos == 4) {
        d->ctr[3] += 1;
        og_philox4x32_10(d->ctr, d->key, d->w);
        d->rpos = 0;
    }
    return d->w[d->rpos++];
}
static uint32_t draw_index(draw_t* d, uint32_t n) {
    if (!d->philox) return xo_index(d->xo, n);
    uint64_t m = (uint64_t)d->w[0] * n;
    uint32_t lo = (uint32_t)m;
    if (lo < n) {
        const uint32_t threshold = (uint32_t)((0x100000000ULL - n) % n);
        while (lo < threshold) {
            m = (uint64_t)draw_retry_word(d) * n;
            lo = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}
static double draw_real(draw_t* d) {
    if (!d->philox) return xo_real(d->xo);
    const uint64_t x = ((uint64_t)d->w[1] << 32) | d->w[2];
    return (double)(x >> 11) * 0x1.0p-53;
}

uint32_t og_lemire_philox(const uint32_t key[2], uint64_t id, uint32_t blk, uint32_t n) {
    draw_t d;
    draw_open(&d, 1, NULL, key, id, blk);
    return draw_index(&d, n);
}
double og_unit_philox(const uint32_t key[2], uint64_t id, uint32_t blk) {
    draw_t d;
    draw_open(&d, 1, NULL, key, id, blk);
    return draw_real(&d);
}

/* ============================================================ graph build */

typedef struct { uint32_t src, dst; uint64_t pos; } raw_edge_t;

static int cmp_raw(const void* a, const void* b) {
    const raw_edge_t* x = (const raw_edge_t*)a;
    const raw_edge_t* y = (const raw_edge_t*)b;
    if (x->src != y->src) return x->src < y->src ? -1 : 1;
    if (x->dst != y->dst) return x->dst < y->dst ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* build_csr + load_edge_list symmetrization (graph.cpp:35-66, :94-97).
 * Duplicates are summed in input order (the reference's std::sort leaves the
 * order of >2 equal keys unspecified; for <=2 duplicates the sum is exact). */
int og_build_csr(uint64_t n_edges, const uint32_t* src, const uint32_t* dst, const double* w,
                 int symmetrize, uint32_t n_nodes, uint32_t* n_out, uint64_t* m_out,
                 uint64_t** offsets, uint32_t** nbr, double** weights) {
    uint64_t cap = symmetrize ? 2 * n_edges : n_edges;
    raw_edge_t* e = (raw_edge_t*)malloc((cap ? cap : 1) * sizeof(raw_edge_t));
    double* ew = (double*)malloc((cap ? cap : 1) * sizeof(double));
    if (!e || !ew) { free(e); free(ew); return OG_ERR_NOMEM; }
    uint64_t k = 0;
    uint32_t max_id = 0;
    for (uint64_t i = 0; i < n_edges; ++i) {
        e[k].src = src[i]; e[k].dst = dst[i]; e[k].pos = k; ew[k] = w ? w[i] : 1.0; ++k;
        if (symmetrize && src[i] != dst[i]) {
            e[k].src = dst[i]; e[k].dst = src[i]; e[k].pos = k; ew[k] = w ? w[i] : 1.0; ++k;
        }
        if (src[i] > max_id) max_id = src[i];
        if (dst[i] > max_id) max_id = dst[i];
    }
    uint32_t n = n_edges == 0 ? 0 : max_id + 1;
    if (n_nodes > n) n = n_nodes;
    qsort(e, k, sizeof(raw_edge_t), cmp_raw);
    uint64_t out = 0;
    double* sw = (double*)malloc((k ? k : 1) * sizeof(double));
    raw_edge_t* se = e;
    for (uint64_t i = 0; i < k; ++i) {
        const double wi = ew[e[i].pos];
        if (out > 0 && se[out - 1].src == e[i].src && se[out - 1].dst == e[i].dst) {
            sw[out - 1] += wi;
        } else {
            se[out] = e[i];
            sw[out] = wi;
            ++out;
        }
    }
    uint64_t* off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    uint32_t* nb = (uint32_t*)malloc((out ? out : 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < out; ++i) { off[se[i].src + 1]++; nb[i] = se[i].dst; }
    for (uint32_t v = 0; v < n; ++v) off[v + 1] += off[v];
    free(e);
    free(ew);
    *n_out = n;
    *m_out = out;
    *offsets = off;
    *nbr = nb;
    *weights = sw;
    return OG_OK;
}

static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y);
}

/* R-MAT pairs: edge e draws `scale` 32-bit words
 * from Philox block (e, level/4); quadrant by integer thresholds; MSB first.
 * Self-loops dropped, pairs canonicalized (lo<hi) and deduplicated. */
int og_rmat_pairs(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                  uint64_t seed, uint64_t* n_pairs, uint32_t** lo, uint32_t** hi) {
    const uint64_t t1 = (uint64_t)(a * 4294967296.0);
    const uint64_t t2 = (uint64_t)((a + b) * 4294967296.0);
    const uint64_t t3 = (uint64_t)((a + b + c) * 4294967296.0);
    const uint64_t ne = (uint64_t)edge_factor << scale;
    uint32_t key[2];
    og_philox_key(seed, DOM_RMAT, key);
    uint64_t* keys = (uint64_t*)malloc((ne ? ne : 1) * sizeof(uint64_t));
    if (!keys) return OG_ERR_NOMEM;
    uint64_t k = 0;
    for (uint64_t e = 0; e < ne; ++e) {
        uint32_t s = 0, d = 0, words[4] = {0, 0, 0, 0};
        for (uint32_t l = 0; l < scale; ++l) {
            if ((l & 3) == 0) {
                const uint32_t ctr[4] = {(uint32_t)e, (uint32_t)(e >> 32), l >> 2, 0};
                og_philox4x32_10(ctr, key, words);
            }
            const uint64_t r = words[l & 3];
            uint32_t bs, bd;
            if (r < t1) { bs = 0; bd = 0; }
            else if (r < t2) { bs = 0; bd = 1; }
            else if (r < t3) { bs = 1; bd = 0; }
            else { bs = 1; bd = 1; }
            s = (s << 1) | bs;
            d = (d << 1) | bd;
        }
        if (s == d) continue;
        const uint32_t x = s < d ? s : d, y = s < d ? d : s;
        keys[k++] = ((uint64_t)x << 32) | y;
    }
    qsort(keys, k, sizeof(uint64_t), cmp_u64);
    uint64_t u = 0;
    for (uint64_t i = 0; i < k; ++i) {
        if (u == 0 || keys[u - 1] != keys[i]) keys[u++] = keys[i];
    }
    *lo = (uint32_t*)malloc((u ? u : 1) * sizeof(uint32_t));
    *hi = (uint32_t*)malloc((u ? u : 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < u; ++i) {
        (*lo)[i] = (uint32_t)(keys[i] >> 32);
        (*hi)[i] = (uint32_t)keys[i];
    }
    free(keys);
    *n_pairs = u;
    return OG_OK;
}

/* fp32 weight of an undirected pair, U[wlo, whi): keyed by the pair so it is
 * independent of generation order; computed in double, rounded once to float. */
float og_pair_weight(uint64_t seed, uint32_t lo, uint32_t hi, float wlo, float whi) {
    uint32_t key[2], w[4];
    og_philox_key(seed, DOM_WEIGHT, key);
    const uint32_t ctr[4] = {lo, hi, 0, 0};
    og_philox4x32_10(ctr, key, w);
    const uint64_t x = ((uint64_t)w[0] << 32) | w[1];
    const double u = (double)(x >> 11) * 0x1.0p-53;
    return (float)((double)wlo + ((double)whi - (double)wlo) * u);
}

uint32_t og_pair_etype(uint64_t seed, uint32_t lo, uint32_t hi, uint32_t n_types) {
    uint32_t key[2];
    og_philox_key(seed, DOM_ETYPE, key);
    draw_t d;
    draw_open(&d, 1, NULL, key, ((uint64_t)hi << 32) | lo, 0);
    return draw_index(&d, n_types);
}

void og_pair_weights(uint64_t seed, uint64_t n, const uint32_t* lo, const uint32_t* hi, float wlo, float whi,
                     float* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = og_pair_weight(seed, lo[i], hi[i], wlo, whi);
}

void og_pair_etypes(uint64_t seed, uint64_t n, const uint32_t* lo, const uint32_t* hi, uint32_t n_types,
                    uint16_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint16_t)og_pair_etype(seed, lo[i], hi[i], n_types);
}

/* graph_checksum (tools/mhwalk.cpp:107-122): FNV-1a over offsets, neighbour
 * ids and the f64 bits of the weights (1.0 per arc when w is NULL). */
uint64_t og_graph_checksum(uint32_t n, const uint64_t* offsets, const uint32_t* nbr, const double* w) {
    uint64_t h = 0xcbf29ce484222325ULL;
    const uint64_t m = offsets[n];
    for (uint64_t i = 0; i <= n; ++i) { h ^= offsets[i]; h *= 0x100000001b3ULL; }
    for (uint64_t i = 0; i < m; ++i) { h ^= nbr[i]; h *= 0x100000001b3ULL; }
    for (uint64_t i = 0; i < m; ++i) {
        const double x = w ? w[i] : 1.0;
        uint64_t bits;
        memcpy(&bits, &x, sizeof bits);
        h ^= bits;
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* Heterogeneous A/P/V graph (BASELINE cfg3): types contiguous by id
 * (A = [0,nA), P = [nA,nA+nP), V = rest). A node a draws Poisson(8) (Knuth
 * product method on Philox units of block (a, j)) P targets uniformly; each P
 * links to one uniform V. Pairs deduplicated. */
int og_hetero_pairs(uint32_t n_nodes, uint64_t seed, uint32_t* nA_out, uint32_t* nP_out,
                    uint64_t* n_pairs, uint32_t** lo, uint32_t** hi) {
    const uint32_t nA = (uint32_t)((uint64_t)n_nodes * 60 / 100);
    const uint32_t nP = (uint32_t)((uint64_t)n_nodes * 35 / 100);
    const uint32_t nV = n_nodes - nA - nP;
    const double L = 0x1.5fc21041027adp-12; /* exp(-8) */
    uint32_t key[2];
    og_philox_key(seed, DOM_HETERO, key);
    uint64_t cap = (uint64_t)nA * 24 + nP + 16, k = 0;
    uint64_t* keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
    if (!keys) return OG_ERR_NOMEM;
    for (uint32_t a = 0; a < nA; ++a) {
        /* Poisson count: blocks (a, 0..): words w1,w2 -> unit; stop when product <= L */
        uint32_t cnt = 0;
        double prod = 1.0;
        for (uint32_t j = 0;; ++j) {
            prod = prod * og_unit_philox(key, a, j);
            if (prod <= L) break;
            ++cnt;
        }
        for (uint32_t j = 0; j < cnt; ++j) {
            const uint32_t p = nA + og_lemire_philox(key, ((uint64_t)1 << 40) | a, j, nP);
            if (k == cap) {
                cap *= 2;
                keys = (uint64_t*)realloc(keys, cap * sizeof(uint64_t));
            }
            keys[k++] = ((uint64_t)a << 32) | p;
        }
    }
    for (uint32_t p = 0; p < nP; ++p) {
        const uint32_t v = nA + nP + og_lemire_philox(key, ((uint64_t)2 << 40) | p, 0, nV);
        if (k == cap) {
            cap *= 2;
            keys = (uint64_t*)realloc(keys, cap * sizeof(uint64_t));
        }
        keys[k++] = ((uint64_t)(nA + p) << 32) | v;
    }
    qsort(keys, k, sizeof(uint64_t), cmp_u64);
    uint64_t u = 0;
    for (uint64_t i = 0; i < k; ++i) {
        if (u == 0 || keys[u - 1] != keys[i]) keys[u++] = keys[i];
    }
    *lo = (uint32_t*)malloc((u ? u : 1) * sizeof(uint32_t));
    *hi = (uint32_t*)malloc((u ? u : 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < u; ++i) {
        (*lo)[i] = (uint32_t)(keys[i] >> 32);
        (*hi)[i] = (uint32_t)keys[i];
    }
    free(keys);
    *n_pairs = u;
    *nA_out = nA;
    *nP_out = nP;
    return OG_OK;
}

void og_free(void* p) { free(p); }

/* ================================================================ models */

static inline uint32_t deg_of(const og_graph* g, uint32_t v) {
    return (uint32_t)(g->offsets[v + 1] - g->offsets[v]);
}

/* Graph::neighbor_index_of: lower_bound in N(v), graph.cpp:13-18 */
static int nbr_index(const og_graph* g, uint32_t v, uint32_t u, uint32_t* idx) {
    uint64_t lo = g->offsets[v], hi = g->offsets[v + 1];
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (g->nbr[mid] < u) lo = mid + 1; else hi = mid;
    }
    if (lo == g->offsets[v + 1] || g->nbr[lo] != u) return 0;
    *idx = (uint32_t)(lo - g->offsets[v]);
    return 1;
}

/* Graph::edge_type, graph.hpp:47-50 */
static inline uint16_t edge_type(const og_graph* g, uint32_t v, uint32_t idx) {
    if (g->etype) return g->etype[g->offsets[v] + idx];
    return (uint16_t)(g->ntype[v] * g->n_ntypes + g->ntype[g->nbr[g->offsets[v] + idx]]);
}
static inline uint16_t edge_type_count(const og_graph* g) {
    if (g->etype) return g->n_etypes;
    return (uint16_t)(g->n_ntypes * g->n_ntypes);
}

static inline int second_order(const og_model* m) {
    return m->kind == OG_NODE2VEC || m->kind == OG_EDGE2VEC || m->kind == OG_FAIRWALK;
}

/* metapath_next, models.hpp:82-85 */
static inline uint32_t metapath_next(const og_model* m, uint32_t affix) {
    if (affix + 1 < m->mp_len) return affix + 1;
    return (m->metapath[0] == m->metapath[m->mp_len - 1] && m->mp_len > 1) ? 1 : 0;
}
static inline uint16_t required_type(const og_model* m, uint32_t affix) {
    return m->metapath[metapath_next(m, affix)];
}

size_t og_type_counts_size(const og_graph* g) { return (size_t)g->n * g->n_ntypes; }

/* WalkModel::bind, models.cpp:29-74 */
int og_model_bind(const og_graph* g, og_model* m, char* err, size_t errlen) {
    m->num_types = g->n_ntypes;
    if (second_order(m)) {
        if (m->p <= 0 || m->q <= 0) { snprintf(err, errlen, "p and q must be positive"); return OG_ERR_INVALID; }
        if (!g->symmetric) { snprintf(err, errlen, "model requires a symmetric graph (load with symmetrize)"); return OG_ERR_INVALID; }
    }
    if (m->kind == OG_METAPATH2VEC || m->kind == OG_FAIRWALK || m->kind == OG_EDGE2VEC) {
        if (!g->ntype) { snprintf(err, errlen, "model requires node types"); return OG_ERR_INVALID; }
    }
    if (m->kind == OG_METAPATH2VEC) {
        if (m->mp_len < 2) { snprintf(err, errlen, "metapath needs at least 2 types"); return OG_ERR_INVALID; }
        for (uint32_t i = 0; i < m->mp_len; ++i) {
            if (m->metapath[i] >= m->num_types) { snprintf(err, errlen, "metapath type %u not in graph", m->metapath[i]); return OG_ERR_INVALID; }
        }
    }
    if (m->kind == OG_EDGE2VEC) {
        const uint32_t dim = edge_type_count(g);
        if (m->M_dim != dim) { snprintf(err, errlen, "edge type matrix must be %ux%u", dim, dim); return OG_ERR_INVALID; }
        for (uint32_t i = 0; i < dim * dim; ++i) {
            if (m->M[i] < 0) { snprintf(err, errlen, "edge type matrix entries must be non-negative"); return OG_ERR_INVALID; }
        }
    }
    if (m->kind == OG_FAIRWALK) {
        if (!m->type_counts) { snprintf(err, errlen, "type_counts buffer missing"); return OG_ERR_INVALID; }
        memset(m->type_counts, 0, og_type_counts_size(g) * sizeof(uint32_t));
        for (uint32_t v = 0; v < g->n; ++v) {
            for (uint64_t e = g->offsets[v]; e < g->offsets[v + 1]; ++e) {
                ++m->type_counts[(size_t)v * m->num_types + g->ntype[g->nbr[e]]];
            }
        }
    }
    return OG_OK;
}

/* WalkModel::alpha, models.cpp:76-80 */
static double alpha(const og_graph* g, const og_model* m, uint32_t prev, uint32_t cand) {
    uint32_t idx;
    if (cand == prev) return 1.0 / m->p;
    if (nbr_index(g, prev, cand, &idx)) return 1.0;
    return 1.0 / m->q;
}

/* WalkModel::calculate_weight, models.cpp:82-123 */
double og_weight(const og_graph* g, const og_model* m, uint32_t v, uint32_t affix, uint32_t i) {
    const uint64_t base = g->offsets[v];
    const double w = g->w[base + i];
    if (m->kind == OG_DEEPWALK) return w;
    if (m->kind == OG_METAPATH2VEC) {
        const uint32_t u = g->nbr[base + i];
        return g->ntype[u] == required_type(m, affix) ? w : 0.0;
    }
    if (affix == OG_NO_AFFIX) return w;
    const uint32_t s = g->nbr[base + affix];
    const uint32_t u = g->nbr[base + i];
    const double a = alpha(g, m, s, u);
    switch (m->kind) {
    case OG_NODE2VEC:
        return a * w;
    case OG_EDGE2VEC: {
        uint32_t sv = 0;
        nbr_index(g, s, v, &sv);
        const uint16_t in_t = edge_type(g, s, sv);
        const uint16_t out_t = edge_type(g, v, i);
        return a * m->M[(size_t)in_t * m->M_dim + out_t] * w;
    }
    case OG_FAIRWALK: {
        const uint32_t group = m->type_counts[(size_t)v * m->num_types + g->ntype[u]];
        return a * w / (double)group;
    }
    default:
        return w;
    }
}

double og_rfactor(const og_graph* g, const og_model* m, uint32_t v, uint32_t affix, uint32_t i) {
    const uint64_t base = g->offsets[v];
    if (m->kind == OG_DEEPWALK) return 1.0;
    if (m->kind == OG_METAPATH2VEC) return g->ntype[g->nbr[base + i]] == required_type(m, affix) ? 1.0 : 0.0;
    if (affix == OG_NO_AFFIX) return 1.0;
    const uint32_t s = g->nbr[base + affix];
    const uint32_t u = g->nbr[base + i];
    const double a = alpha(g, m, s, u);
    switch (m->kind) {
    case OG_NODE2VEC:
        return a;
    case OG_EDGE2VEC: {
        uint32_t sv = 0;
        nbr_index(g, s, v, &sv);
        return a * m->M[(size_t)edge_type(g, s, sv) * m->M_dim + edge_type(g, v, i)];
    }
    case OG_FAIRWALK:
        return a / (double)m->type_counts[(size_t)v * m->num_types + g->ntype[u]];
    default:
        return 1.0;
    }
}

int og_hastings(double w_c, double r_c, double r_l, double u) {
    return w_c > 0.0 && (r_l <= 0.0 || r_c >= r_l || u * r_l < r_c);
}

void og_decide_hastings(const og_graph* g, const og_model* m, uint64_t count, const uint32_t* pos,
                        const uint32_t* affix, const uint32_t* cand, const uint32_t* last, const double* u,
                        double* rc, double* rl, uint8_t* accept) {
    for (uint64_t i = 0; i < count; ++i) {
        rc[i] = og_rfactor(g, m, pos[i], affix[i], cand[i]);
        rl[i] = og_rfactor(g, m, pos[i], affix[i], last[i]);
        accept[i] = (uint8_t)og_hastings(g->w[g->offsets[pos[i]] + cand[i]], rc[i], rl[i], u[i]);
    }
}

/* accept rule, samplers.hpp:24 verbatim */
int og_accept(double wc, double wl, double u) { return wl <= 0.0 || wc >= wl || u * wl < wc; }

void og_decide(const og_graph* g, const og_model* m, uint64_t count, const uint32_t* pos,
               const uint32_t* affix, const uint32_t* cand, const uint32_t* last,
               const double* u, double* wc, double* wl, uint8_t* accept) {
    for (uint64_t i = 0; i < count; ++i) {
        wc[i] = og_weight(g, m, pos[i], affix[i], cand[i]);
        wl[i] = og_weight(g, m, pos[i], affix[i], last[i]);
        accept[i] = (uint8_t)og_accept(wc[i], wl[i], u[i]);
    }
}

/* ============================================================== samplers */

/* alias_build, samplers.cpp:95-131: sequential total, scaled = w*n/total,
 * LIFO small/large stacks, leftovers 1.0. */
int og_alias_build(uint32_t n, const double* w, double* prob, uint32_t* alias) {
    double total = 0.0;
    for (uint32_t i = 0; i < n; ++i) total += w[i];
    if (n == 0 || total <= 0) return OG_ERR_INVALID;
    for (uint32_t i = 0; i < n; ++i) if (w[i] < 0) return OG_ERR_INVALID;
    double* scaled = (double*)malloc(n * sizeof(double));
    uint32_t* small = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint32_t* large = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint32_t ns = 0, nl = 0;
    for (uint32_t i = 0; i < n; ++i) {
        prob[i] = 1.0;
        alias[i] = i;
        scaled[i] = w[i] * (double)n / total;
    }
    for (uint32_t i = 0; i < n; ++i) {
        if (scaled[i] < 1.0) small[ns++] = i; else large[nl++] = i;
    }
    while (ns > 0 && nl > 0) {
        const uint32_t s = small[--ns];
        const uint32_t l = large[nl - 1];
        prob[s] = scaled[s];
        alias[s] = l;
        scaled[l] -= 1.0 - scaled[s];
        if (scaled[l] < 1.0) {
            --nl;
            small[ns++] = l;
        }
    }
    for (uint32_t i = 0; i < ns; ++i) prob[small[i]] = 1.0;
    for (uint32_t i = 0; i < nl; ++i) prob[large[i]] = 1.0;
    free(scaled);
    free(small);
    free(large);
    return OG_OK;
}

/* Per-node static alias tables over a CSR (engine.cpp:136-146 builds one per
 * node); nodes without positive weight get prob 0 / alias i like the device
 * dump (mhw_alias_tables). */
void og_alias_tables(uint32_t n, const uint64_t* offsets, const double* w, double* prob, uint32_t* alias) {
    for (uint32_t v = 0; v < n; ++v) {
        const uint64_t a = offsets[v], b = offsets[v + 1];
        if (a == b) continue;
        if (og_alias_build((uint32_t)(b - a), w + a, prob + a, alias + a) != OG_OK) {
            for (uint64_t i = a; i < b; ++i) { prob[i] = 0.0; alias[i] = (uint32_t)(i - a); }
        }
    }
}

/* direct_sample with the unit supplied, samplers.cpp:133-146 */
uint32_t og_direct_sample_u(uint32_t n, const double* w, double u) {
    double total = 0.0;
    for (uint32_t i = 0; i < n; ++i) total += w[i];
    double r = u * total;
    for (uint32_t i = 0; i < n; ++i) {
        r -= w[i];
        if (r < 0) return i;
    }
    for (uint32_t i = n; i-- > 0;) {
        if (w[i] > 0) return i;
    }
    return 0;
}

/* ---- per-state sampling context */
typedef struct {
    const og_graph* g;
    const og_model* m;
    uint32_t v, affix, n;
    /* optional (og_walk_isolated): per node, every static weight > 0 and the
     * model cannot zero a weight -- then random_positive's pick-th positive is
     * simply the pick-th index, and the two O(deg) scans are skipped (the GPU
     * engine's all_positive fast path, mhw_device.cuh) */
    const uint8_t* allpos;
} st_t;

static inline double st_w(const st_t* s, uint32_t i) { return og_weight(s->g, s->m, s->v, s->affix, i); }

/* mh_transition, samplers.hpp:18-27 */
static uint32_t mh_transition(const st_t* s, uint32_t last, draw_t* d) {
    const uint32_t cand = draw_index(d, s->n);
    const double wc = st_w(s, cand);
    const double wl = st_w(s, last);
    const int accept = wl <= 0.0 || wc >= wl || draw_real(d) * wl < wc;
    return accept ? cand : last;
}

/* random_positive, samplers.cpp:22-33 */
static int random_positive(const st_t* s, draw_t* d, uint32_t* out) {
    if (s->allpos && s->allpos[s->v]) {
        *out = draw_index(d, s->n);
        return 1;
    }
    uint32_t positive = 0;
    for (uint32_t i = 0; i < s->n; ++i) if (st_w(s, i) > 0) ++positive;
    if (positive == 0) return 0;
    uint32_t pick = draw_index(d, positive);
    for (uint32_t i = 0; i < s->n; ++i) {
        if (st_w(s, i) > 0 && pick-- == 0) { *out = i; return 1; }
    }
    return 0;
}

/* Source of init draws: xoshiro = the querying walker's stream (manager.cpp:40);
 * philox = slot-keyed blocks (slot, j). */
typedef struct {
    int philox;
    xo_t* xo;
    uint32_t key[2];
    uint64_t slot;
} init_src_t;

static void init_block(const init_src_t* src, uint32_t j, draw_t* d) {
    draw_open(d, src->philox, src->xo, src->key, src->slot, j);
}

/* mh_init, samplers.cpp:37-83. Philox block plan: random -> block 0;
 * high_weight probes -> blocks 0..hw-1, fallback -> block hw; burn_in ->
 * block 0 pick, blocks 1..k transitions. */
static int mh_init(const st_t* s, const og_config* c, const init_src_t* src, uint32_t* out) {
    draw_t d;
    if (s->n == 0) return 0;
    switch (c->init_kind) {
    case OG_INIT_RANDOM:
        init_block(src, 0, &d);
        return random_positive(s, &d, out);
    case OG_INIT_HIGH_WEIGHT: {
        double best_w = 0.0;
        uint32_t best = 0;
        int found = 0;
        if (s->n <= c->hw_sample_size) {
            for (uint32_t i = 0; i < s->n; ++i) {
                const double w = st_w(s, i);
                if (w > best_w) { best_w = w; best = i; found = 1; }
            }
        } else {
            for (uint32_t probe = 0; probe < c->hw_sample_size; ++probe) {
                init_block(src, probe, &d);
                const uint32_t i = draw_index(&d, s->n);
                const double w = st_w(s, i);
                if (w > best_w || (w == best_w && found && i < best)) {
                    if (w > 0) { best_w = w; best = i; found = 1; }
                }
            }
            if (!found) {
                init_block(src, c->hw_sample_size, &d);
                return random_positive(s, &d, out);
            }
        }
        if (found) *out = best;
        return found;
    }
    case OG_INIT_BURN_IN: {
        uint32_t last;
        init_block(src, 0, &d);
        if (!random_positive(s, &d, &last)) return 0;
        for (uint32_t i = 0; i < c->burn_in_steps; ++i) {
            init_block(src, 1 + i, &d);
            last = mh_transition(s, last, &d);
        }
        *out = last;
        return 1;
    }
    }
    return 0;
}

/* slot layout, manager.cpp:14-17 + models.cpp:146-172 */
uint64_t og_slot_count(const og_graph* g, const og_model* m) {
    switch (m->kind) {
    case OG_DEEPWALK: return g->n;
    case OG_METAPATH2VEC: return (uint64_t)g->n * m->num_types;
    default: return g->m;
    }
}
static inline uint64_t slot_index(const og_graph* g, const og_model* m, uint32_t v, uint32_t affix) {
    switch (m->kind) {
    case OG_DEEPWALK: return v;
    case OG_METAPATH2VEC: return (uint64_t)v * m->num_types + required_type(m, affix);
    default: return g->offsets[v] + affix;
    }
}

/* Engine chain layout: node-keyed states of hub nodes (degree >= D) own
 * R = 2^(floor(log2(deg/D))+1) <= 65536 chains; walker w uses chain
 * (w * golden >> 40) & (R-1); chains 1..R-1 live after the n*G base slots. */
typedef struct {
    uint32_t D;
    uint32_t* group;   /* n+1 exclusive prefix of (R-1) */
    uint64_t base;     /* n*G */
    uint32_t G;
    double* scale;     /* metapath2vec: per node type visit scale (NULL: weight = degree) */
} replica_layout_t;

/* Replica weight of node v (walk.cu rep_weight): the degree, or for
 * metapath2vec floor(deg * F[type]) with F_t = (count_t * arcs) /
 * (cycle_len * arcs incident to type t) over the metapath's steady cycle. */
static uint32_t rep_weight(const og_graph* g, const replica_layout_t* rl, uint32_t v) {
    const uint32_t d = deg_of(g, v);
    if (!rl->scale) return d;
    const double x = (double)d * rl->scale[g->ntype[v]];
    return x >= 2147483647.0 ? 0x7FFFFFFFu : (uint32_t)x;
}

static double* metapath_rep_scale(const og_graph* g, const og_model* m) {
    const uint32_t T = g->n_ntypes ? g->n_ntypes : 1;
    double* F = (double*)calloc(T, sizeof(double));
    double* count = (double*)calloc(T, sizeof(double));
    uint64_t* arcs = (uint64_t*)calloc(T, sizeof(uint64_t));
    for (uint32_t v = 0; v < g->n; ++v) arcs[g->ntype[v]] += deg_of(g, v);
    const uint32_t L = m->mp_len;
    const uint32_t b = (L > 1 && m->metapath[0] == m->metapath[L - 1]) ? 1 : 0;
    for (uint32_t i = b; i < L; ++i) count[m->metapath[i]] += 1.0;
    const double cycle = (double)(L - b);
    for (uint32_t t = 0; t < T; ++t)
        if (arcs[t]) F[t] = (count[t] * (double)g->m) / (cycle * (double)arcs[t]);
    free(count);
    free(arcs);
    return F;
}

static uint32_t chain_replicas(uint32_t deg, uint32_t D) {
    if (D == OG_NO_REPLICAS || deg < D) return 1;
    uint32_t q = deg / D, lg = 0;
    while (q >>= 1) ++lg;
    const uint32_t r = lg < 16 ? 2u << lg : 65536u;
    return r < 65536 ? r : 65536;
}

static uint64_t engine_slot(const og_graph* g, const og_model* m, const replica_layout_t* rl, uint32_t v,
                            uint32_t affix, uint64_t walker) {
    const uint64_t base = slot_index(g, m, v, affix);
    if (m->kind != OG_DEEPWALK && m->kind != OG_METAPATH2VEC) return base;
    const uint32_t R = chain_replicas(rep_weight(g, rl, v), rl->D);
    if (R == 1) return base;
    const uint32_t r = (uint32_t)((walker * 0x9E3779B97F4A7C15ULL) >> 40) & (R - 1);
    if (r == 0) return base;
    const uint32_t t = m->kind == OG_METAPATH2VEC ? required_type(m, affix) : 0;
    return rl->base + ((uint64_t)rl->group[v] + r - 1) * rl->G + t;
}

int og_init_philox(const og_graph* g, const og_model* m, const og_config* c, uint32_t v,
                   uint32_t affix, uint64_t slot, uint32_t* last) {
    st_t s = {g, m, v, affix, deg_of(g, v)};
    init_src_t src;
    src.philox = 1;
    src.xo = NULL;
    og_philox_key(c->seed, DOM_INIT, src.key);
    src.slot = slot;
    return mh_init(&s, c, &src, last);
}

/* ================================================================= check */

#define DOM_CHECK 0xC4EC0005u

/* cmd_check's per-state audit (tools/mhwalk.cpp:222-247): exact target =
 * normalised w', random init, `draws` M-H transitions counting the chain's
 * states, KL(empirical || target) (analysis.cpp:34-45). Engine layout: init
 * keyed by slot = state index j, transition d from Philox block (j, d) of the
 * check domain. kl[j] = NaN when the target has no mass or init dead-ends. */
void og_check(const og_graph* g, const og_model* m, uint64_t seed, uint64_t n_states, const uint32_t* pos,
              const uint32_t* affix, uint64_t draws, uint64_t* counts, double* kl) {
    og_config c;
    memset(&c, 0, sizeof c);
    c.seed = seed;
    c.init_kind = OG_INIT_RANDOM;
    c.burn_in_steps = 100;
    c.hw_sample_size = 32;
    c.rng = OG_RNG_PHILOX;
    uint32_t key[2];
    og_philox_key(seed, DOM_CHECK, key);
    uint64_t base = 0;
    for (uint64_t j = 0; j < n_states; ++j) {
        const uint32_t v = pos[j], a = affix[j];
        const uint32_t deg = deg_of(g, v);
        uint64_t* cnt = counts + base;
        base += deg;
        for (uint32_t i = 0; i < deg; ++i) cnt[i] = 0;
        kl[j] = __builtin_nan("");
        double* w = (double*)malloc((deg ? deg : 1) * sizeof(double));
        double total = 0.0;
        for (uint32_t i = 0; i < deg; ++i) {
            w[i] = og_weight(g, m, v, a, i);
            total += w[i];
        }
        uint32_t last;
        if (total > 0 && og_init_philox(g, m, &c, v, a, j, &last)) {
            st_t s = {g, m, v, a, deg};
            for (uint64_t d = 0; d < draws; ++d) {
                draw_t dr;
                draw_open(&dr, 1, NULL, key, j, (uint32_t)d);
                last = mh_transition(&s, last, &dr);
                cnt[last]++;
            }
            double k = 0.0;
            for (uint32_t i = 0; i < deg; ++i) {
                const double p = (double)cnt[i] / (double)draws;
                if (p == 0.0) continue;
                k += p * log(p / (w[i] / total));
            }
            kl[j] = k;
        }
        free(w);
    }
}

/* ================================================================ engine */

enum { ST_EMPTY = 0, ST_READY = 2, ST_DEAD = 3 };

/* Chain table: dense arrays indexed by slot (SamplerManager's layout), or a
 * small open-addressing map of the slots one isolated walker touches
 * (og_walk_isolated: a walker alone with a fresh manager). */
typedef struct {
    uint8_t* status;
    uint32_t* last;
    uint64_t* keys;  /* sparse: slot + 1, 0 = free */
    uint32_t cap;    /* sparse capacity (power of two) */
    const uint8_t* allpos;  /* st_t.allpos for the inits of this table (NULL: scan) */
} chain_t;

static uint32_t ch_at(chain_t* ch, uint64_t slot) {
    if (!ch->keys) return (uint32_t)0;
    uint32_t h = (uint32_t)((slot * 0x9E3779B97F4A7C15ULL) >> 40) & (ch->cap - 1);
    for (;;) {
        if (ch->keys[h] == slot + 1) return h;
        if (ch->keys[h] == 0) {
            ch->keys[h] = slot + 1;
            ch->status[h] = ST_EMPTY;
            return h;
        }
        h = (h + 1) & (ch->cap - 1);
    }
}
static uint8_t* ch_status(chain_t* ch, uint64_t slot) { return ch->keys ? &ch->status[ch_at(ch, slot)] : &ch->status[slot]; }
static uint32_t* ch_last(chain_t* ch, uint64_t slot) { return ch->keys ? &ch->last[ch_at(ch, slot)] : &ch->last[slot]; }

typedef struct {
    uint32_t v, affix;
    xo_t xo;
    uint64_t walker, row;
    uint32_t len;
    int alive;
} walker_t;

/* One walker step = WalkerContext::next_edge (engine.cpp:75-87) + the push and
 * update_state of engine.cpp:201-204. Returns 1 stepped, 0 dead end, -1 error. */
/* ---- exact baseline samplers (WalkerContext::next_edge, engine.cpp:88-116) */
typedef struct {
    double* wbuf;                  /* max_deg dynamic weights */
    uint8_t* astat;                /* alias: per reference slot, 0 none 1 built */
    double** aprob;
    uint32_t** aalias;
    uint8_t* pstat;                /* rejection: per node static proposal */
    double** pprob;
    uint32_t** palias;
    double bound;
} baseline_t;

/* rejection_bound, engine.cpp:39-58 */
static double rejection_bound(const og_model* m) {
    double alpha_max = 1.0;
    if (1.0 / m->p > alpha_max) alpha_max = 1.0 / m->p;
    if (1.0 / m->q > alpha_max) alpha_max = 1.0 / m->q;
    switch (m->kind) {
    case OG_DEEPWALK:
    case OG_METAPATH2VEC: return 1.0;
    case OG_NODE2VEC:
    case OG_FAIRWALK: return alpha_max;
    default: {
        double m_max = 0.0;
        for (uint32_t i = 0; i < m->M_dim * m->M_dim; ++i) if (m->M[i] > m_max) m_max = m->M[i];
        return alpha_max * m_max;
    }
    }
}

/* dynamic_weights (engine.cpp:120-127); returns the std::accumulate total */
static double dyn_weights(const og_graph* g, const og_model* m, uint32_t v, uint32_t affix, double* w) {
    const uint32_t deg = deg_of(g, v);
    double total = 0.0;
    for (uint32_t i = 0; i < deg; ++i) {
        w[i] = og_weight(g, m, v, affix, i);
        total += w[i];
    }
    return total;
}

/* alias_sample, samplers.hpp:65-68 */
static uint32_t alias_draw(const double* prob, const uint32_t* alias, uint32_t n, draw_t* d) {
    const uint32_t i = draw_index(d, n);
    return draw_real(d) < prob[i] ? i : alias[i];
}

/* The static-weight alias table of node v (alias_build over weights_of(v),
 * engine.cpp:136-146), built on first use; 0 when the weights sum to <= 0. */
static int static_alias(const og_graph* g, baseline_t* bt, uint32_t v) {
    if (bt->pstat[v]) return 1;
    const uint32_t deg = deg_of(g, v);
    const double* ws = g->w + g->offsets[v];
    double total = 0.0;
    for (uint32_t i = 0; i < deg; ++i) total += ws[i];
    if (total <= 0) return 0;
    bt->pprob[v] = (double*)malloc(deg * sizeof(double));
    bt->palias[v] = (uint32_t*)malloc(deg * sizeof(uint32_t));
    og_alias_build(deg, ws, bt->pprob[v], bt->palias[v]);
    bt->pstat[v] = 1;
    return 1;
}

/* One M-H transition with the static alias proposal (the engine's proposal =
 * alias extension): candidate = alias_sample of v's static table on the walk
 * block (index on word 0, coin on words 1-2, as alias_sample draws,
 * samplers.hpp:65-68), accept unit from block (walker, step) with sub-counter
 * OG_ACCEPT_SUB (xoshiro: the next real of the stream, drawn only when
 * needed, as mh_transition draws it). */
static uint32_t mh_transition_alias(const st_t* s, baseline_t* bt, uint32_t last, draw_t* d, int philox,
                                    xo_t* xo, const uint32_t key[2], uint64_t walker, uint32_t step) {
    const uint32_t cand = alias_draw(bt->pprob[s->v], bt->palias[s->v], s->n, d);
    const double wc = s->g->w[s->g->offsets[s->v] + cand];
    const double rc = og_rfactor(s->g, s->m, s->v, s->affix, cand);
    const double rl = og_rfactor(s->g, s->m, s->v, s->affix, last);
    if (!(wc > 0.0)) return last;
    if (rl <= 0.0 || rc >= rl) return cand;
    double u;
    if (philox) {
        draw_t b;
        draw_open_sub(&b, 1, xo, key, walker, step, OG_ACCEPT_SUB);
        u = draw_real(&b);
    } else {
        u = draw_real(d);
    }
    return u * rl < rc ? cand : last;
}

/* One next_edge of the alias / direct / rejection sampler. Philox layout:
 * direct -> unit of the walk block; alias -> index + unit of the walk block;
 * rejection trial t -> block (walker, step) under key DOM_REJECT + (t >> 16)
 * with sub-counter (t & 0xFFFF) << 16 (index + unit of the proposal), then
 * that sub | 0x8000 (the accept unit). 1 stepped, 0 dead end, -1 error. */
static int baseline_step(const og_graph* g, const og_model* m, const og_config* c, baseline_t* bt,
                         const walker_t* w, uint32_t step, draw_t* d, uint32_t* edge, og_stats* st,
                         char* err, size_t errlen) {
    const uint32_t v = w->v, deg = deg_of(g, v);
    const int philox = c->rng == OG_RNG_PHILOX;
    if (c->sampler == OG_SAMPLER_DIRECT) {
        if (dyn_weights(g, m, v, w->affix, bt->wbuf) <= 0) return 0;
        *edge = og_direct_sample_u(deg, bt->wbuf, draw_real(d));
        return 1;
    }
    if (c->sampler == OG_SAMPLER_ALIAS) {
        const uint64_t slot = slot_index(g, m, v, w->affix);
        if (!bt->astat[slot]) {
            if (dyn_weights(g, m, v, w->affix, bt->wbuf) <= 0) return 0;
            bt->aprob[slot] = (double*)malloc(deg * sizeof(double));
            bt->aalias[slot] = (uint32_t*)malloc(deg * sizeof(uint32_t));
            if (og_alias_build(deg, bt->wbuf, bt->aprob[slot], bt->aalias[slot]) != OG_OK) {
                snprintf(err, errlen, "alias_build: negative weight");
                return -1;
            }
            bt->astat[slot] = 1;
        }
        *edge = alias_draw(bt->aprob[slot], bt->aalias[slot], deg, d);
        return 1;
    }
    /* rejection: static proposal per node (engine.cpp:136-146) */
    const double* ws = g->w + g->offsets[v];
    if (!static_alias(g, bt, v)) return 0;
    if (dyn_weights(g, m, v, w->affix, bt->wbuf) <= 0) return 0;
    /* rejection_sample, samplers.cpp:148-170 */
    for (uint32_t i = 0; i < deg; ++i) {
        if (bt->wbuf[i] > bt->bound * ws[i]) {
            snprintf(err, errlen, "rejection_sample: envelope violated at index %u", i);
            return -1;
        }
    }
    for (uint64_t t = 0;; ++t) {
        /* trial epochs of 65536 trials under distinct keys DOM_REJECT + (t >> 16):
         * the 16-bit trial field of the sub-counter never wraps onto an earlier
         * trial's draws */
        uint32_t rkey[2];
        og_philox_key(c->seed, DOM_REJECT + (uint32_t)(t >> 16), rkey);
        const uint32_t sub = (uint32_t)(t & 0xFFFFu) << 16;
        st->trials++;
        draw_t a;
        draw_open_sub(&a, philox, d->xo, rkey, w->walker, step, sub);
        const uint32_t i = alias_draw(bt->pprob[v], bt->palias[v], deg, &a);
        const double accept = bt->wbuf[i] / (bt->bound * ws[i]);
        if (accept >= 1.0) { *edge = i; return 1; }
        draw_t b;
        draw_open_sub(&b, philox, d->xo, rkey, w->walker, step, sub | 0x8000u);
        if (draw_real(&b) < accept) { *edge = i; return 1; }
    }
}

static int walker_step(const og_graph* g, const og_model* m, const og_config* c, chain_t* ch,
                       const replica_layout_t* rl, baseline_t* bt, walker_t* w, uint32_t step, uint32_t stride,
                       uint32_t* rows, og_stats* st, char* err, size_t errlen) {
    const uint32_t v = w->v;
    const uint32_t deg = deg_of(g, v);
    if (deg == 0) return 0;
    const int philox = c->rng == OG_RNG_PHILOX;
    uint32_t wkey[2];
    og_philox_key(c->seed, DOM_WALK, wkey);
    draw_t d;
    draw_open(&d, philox, &w->xo, wkey, w->walker, step);
    uint32_t edge;
    if (second_order(m) && w->affix == OG_NO_AFFIX) {
        /* bootstrap: draw_static (engine.cpp:81-83, :130-134) */
        const double* ws = g->w + g->offsets[v];
        double total = 0.0;
        for (uint32_t i = 0; i < deg; ++i) total += ws[i];
        if (total <= 0) return 0;
        edge = og_direct_sample_u(deg, ws, draw_real(&d));
    } else if (c->sampler != OG_SAMPLER_MH) {
        const int r = baseline_step(g, m, c, bt, w, step, &d, &edge, st, err, errlen);
        if (r <= 0) return r;
    } else {
        /* SamplerManager::sample, manager.cpp:30-72 */
        const uint64_t slot = engine_slot(g, m, rl, v, w->affix, w->walker);
        st_t s = {g, m, v, w->affix, deg, ch->allpos};
        uint8_t* const status = ch_status(ch, slot);
        uint32_t* const lastp = ch_last(ch, slot);
        if (*status == ST_EMPTY) {
            init_src_t src;
            src.philox = philox;
            src.xo = &w->xo;
            og_philox_key(c->seed, DOM_INIT, src.key);
            src.slot = slot;
            uint32_t init;
            st->init_calls++;
            if (mh_init(&s, c, &src, &init)) {
                *lastp = init;
                *status = ST_READY;
            } else {
                *status = ST_DEAD;
            }
        }
        if (*status == ST_DEAD) return 0;
        const uint32_t last = *lastp;
        /* the philox block is (walker, step); xoshiro continues the stream */
        if (philox) draw_open(&d, 1, NULL, wkey, w->walker, step);
        uint32_t next;
        if (c->proposal == OG_PROPOSAL_ALIAS) {
            if (!static_alias(g, bt, v)) return 0;
            next = mh_transition_alias(&s, bt, last, &d, philox, &w->xo, wkey, w->walker, step);
        } else {
            next = mh_transition(&s, last, &d);
        }
        if (next != last) *lastp = next;
        edge = next;
    }
    const uint32_t nxt = g->nbr[g->offsets[v] + edge];
    rows[w->row * stride + w->len] = nxt;
    w->len++;
    /* update_state, models.cpp:125-136 */
    if (m->kind == OG_DEEPWALK) {
        w->affix = OG_NO_AFFIX;
    } else if (m->kind == OG_METAPATH2VEC) {
        w->affix = metapath_next(m, w->affix);
    } else {
        uint32_t back;
        if (!nbr_index(g, nxt, v, &back)) {
            snprintf(err, errlen, "second-order walk on asymmetric adjacency: no back edge %u->%u", nxt, v);
            return -1;
        }
        w->affix = back;
    }
    w->v = nxt;
    st->steps++;
    return 1;
}

/* Engine chain layout of a run: base slots plus hub replicas for node-keyed
 * models (walk.cu session_create). Returns 0 when the layout is too large. */
static int layout_init(const og_graph* g, const og_model* m, const og_config* c, replica_layout_t* out,
                       uint64_t* slots_out) {
    uint64_t slots = og_slot_count(g, m);
    replica_layout_t rl;
    rl.D = c->replica_degree;
    rl.G = m->kind == OG_METAPATH2VEC ? m->num_types : 1;
    rl.base = slots;
    rl.group = NULL;
    rl.scale = NULL;
    if ((m->kind == OG_DEEPWALK || m->kind == OG_METAPATH2VEC) && rl.D != OG_NO_REPLICAS) {
        if (m->kind == OG_METAPATH2VEC) rl.scale = metapath_rep_scale(g, m);
        if (rl.D == 0) {
            /* automatic layout (walk.cu session_create): metapath2vec 32 (visit weights);
             * deepwalk the smallest power-of-two D whose replica region
             * holds at most 8M chain words */
            rl.D = 32;
            if (m->kind == OG_DEEPWALK) {
                uint64_t hist[33] = {0};
                for (uint32_t v = 0; v < g->n; ++v) {
                    uint32_t d = rep_weight(g, &rl, v), b = 0;
                    if (!d) continue;
                    while (d >>= 1) ++b;
                    ++hist[b];
                }
                for (uint32_t lg = 0; lg < 31; ++lg) {
                    uint64_t t = 0;
                    for (uint32_t b = lg; b < 33; ++b) {
                        const uint64_t r = b - lg < 16 ? (uint64_t)2 << (b - lg) : 65536;
                        t += hist[b] * ((r < 65536 ? r : 65536) - 1);
                    }
                    if (t <= ((uint64_t)8 << 20)) { rl.D = 1u << lg; break; }
                }
            }
        }
        rl.group = (uint32_t*)calloc((size_t)g->n + 1, sizeof(uint32_t));
        for (uint32_t v = 0; v < g->n; ++v) rl.group[v + 1] = rl.group[v] + chain_replicas(rep_weight(g, &rl, v), rl.D) - 1;
        slots += (uint64_t)rl.group[g->n] * rl.G;
    } else {
        rl.D = OG_NO_REPLICAS;
    }
    if (slots > ((uint64_t)1 << 40)) {
        free(rl.group);
        free(rl.scale);
        return 0;
    }
    *out = rl;
    *slots_out = slots;
    return 1;
}

int og_generate_walks(const og_graph* g, const og_model* m, const og_config* c, uint32_t stride,
                      uint32_t* rows, uint32_t* lens, uint64_t* n_rows, og_stats* stats,
                      char* err, size_t errlen) {
    memset(stats, 0, sizeof(*stats));
    if (c->K == 0 || c->L == 0) {
        snprintf(err, errlen, "walks_per_node, walk_length and threads must be positive");
        return OG_ERR_INVALID;
    }
    if (stride < c->L + 1) { snprintf(err, errlen, "row stride too small"); return OG_ERR_INVALID; }
    uint64_t slots = 0;
    replica_layout_t rl;
    if (!layout_init(g, m, c, &rl, &slots)) {
        snprintf(err, errlen, "sampler layout too large");
        return OG_ERR_INVALID;
    }
    chain_t ch;
    ch.status = (uint8_t*)calloc(slots ? slots : 1, 1);
    ch.last = (uint32_t*)calloc(slots ? slots : 1, sizeof(uint32_t));
    ch.keys = NULL;
    ch.cap = 0;
    ch.allpos = NULL;
    baseline_t bt;
    memset(&bt, 0, sizeof(bt));
    if (c->sampler != OG_SAMPLER_MH || c->proposal == OG_PROPOSAL_ALIAS) {
        uint32_t max_deg = 1;
        for (uint32_t v = 0; v < g->n; ++v) if (deg_of(g, v) > max_deg) max_deg = deg_of(g, v);
        const uint64_t rs = og_slot_count(g, m);
        bt.wbuf = (double*)malloc(max_deg * sizeof(double));
        bt.astat = (uint8_t*)calloc(rs ? rs : 1, 1);
        bt.aprob = (double**)calloc(rs ? rs : 1, sizeof(double*));
        bt.aalias = (uint32_t**)calloc(rs ? rs : 1, sizeof(uint32_t*));
        bt.pstat = (uint8_t*)calloc(g->n ? g->n : 1, 1);
        bt.pprob = (double**)calloc(g->n ? g->n : 1, sizeof(double*));
        bt.palias = (uint32_t**)calloc(g->n ? g->n : 1, sizeof(uint32_t*));
        bt.bound = rejection_bound(m);
    }
    const uint64_t total = (uint64_t)g->n * c->K;
    int rc = OG_OK;
    uint64_t row = 0;
    if (c->order == OG_ORDER_WALKER) {
        for (uint64_t idx = 0; idx < total && rc == OG_OK; ++idx) {
            walker_t w;
            w.v = (uint32_t)(idx / c->K);
            const uint32_t k = (uint32_t)(idx % c->K);
            xo_walker(&w.xo, c->seed, w.v, k);
            w.walker = idx;
            if (m->kind == OG_METAPATH2VEC) {
                if (g->ntype[w.v] != m->metapath[0]) { stats->skipped++; continue; }
                w.affix = 0;
            } else {
                w.affix = OG_NO_AFFIX;
            }
            w.row = row++;
            rows[w.row * stride] = w.v;
            w.len = 1;
            for (uint32_t step = 0; step < c->L; ++step) {
                const int r = walker_step(g, m, c, &ch, &rl, &bt, &w, step, stride, rows, stats, err, errlen);
                if (r < 0) { rc = OG_ERR_INVALID; break; }
                if (r == 0) { stats->early++; break; }
            }
            lens[w.row] = w.len;
        }
    } else {
        walker_t* ws = (walker_t*)malloc((total ? total : 1) * sizeof(walker_t));
        uint64_t nw = 0;
        for (uint64_t idx = 0; idx < total; ++idx) {
            walker_t* w = &ws[nw];
            w->v = (uint32_t)(idx / c->K);
            const uint32_t k = (uint32_t)(idx % c->K);
            if (m->kind == OG_METAPATH2VEC) {
                if (g->ntype[w->v] != m->metapath[0]) { stats->skipped++; continue; }
                w->affix = 0;
            } else {
                w->affix = OG_NO_AFFIX;
            }
            xo_walker(&w->xo, c->seed, w->v, k);
            w->walker = idx;
            w->row = row++;
            rows[w->row * stride] = w->v;
            w->len = 1;
            w->alive = 1;
            ++nw;
        }
        for (uint32_t step = 0; step < c->L && rc == OG_OK; ++step) {
            for (uint64_t i = 0; i < nw; ++i) {
                walker_t* w = &ws[i];
                if (!w->alive) continue;
                const int r = walker_step(g, m, c, &ch, &rl, &bt, w, step, stride, rows, stats, err, errlen);
                if (r < 0) { rc = OG_ERR_INVALID; break; }
                if (r == 0) { stats->early++; w->alive = 0; }
            }
        }
        for (uint64_t i = 0; i < nw; ++i) lens[ws[i].row] = ws[i].len;
        free(ws);
    }
    stats->walks = row;
    *n_rows = row;
    free(ch.status);
    free(ch.last);
    free(rl.group);
    free(rl.scale);
    if (c->sampler != OG_SAMPLER_MH || c->proposal == OG_PROPOSAL_ALIAS) {
        const uint64_t rs = og_slot_count(g, m);
        for (uint64_t i = 0; i < rs; ++i) { free(bt.aprob[i]); free(bt.aalias[i]); }
        for (uint32_t v = 0; v < g->n; ++v) { free(bt.pprob[v]); free(bt.palias[v]); }
        free(bt.wbuf); free(bt.astat); free(bt.aprob); free(bt.aalias);
        free(bt.pstat); free(bt.pprob); free(bt.palias);
    }
    return rc;
}

/* Each walker of `starts` (K walkers per start, walker id v*K + k) run ALONE
 * with a fresh SamplerManager, walker-major, under the Philox layout: the
 * corpus a GPU session restricted to that one start (mhw_session_select_starts,
 * K = 1) must produce, whatever its kernel variant. Rows in start order. */
int og_walk_isolated(const og_graph* g, const og_model* m, const og_config* cfg, uint64_t count,
                     const uint32_t* starts, uint32_t stride, uint32_t* rows, uint32_t* lens, uint64_t* n_rows,
                     og_stats* stats, char* err, size_t errlen) {
    og_config cc = *cfg;
    cc.rng = OG_RNG_PHILOX;
    const og_config* c = &cc;
    memset(stats, 0, sizeof(*stats));
    if (c->K == 0 || c->L == 0) {
        snprintf(err, errlen, "walks_per_node, walk_length and threads must be positive");
        return OG_ERR_INVALID;
    }
    if (stride < c->L + 1) { snprintf(err, errlen, "row stride too small"); return OG_ERR_INVALID; }
    if (c->sampler != OG_SAMPLER_MH) { snprintf(err, errlen, "isolated walkers: mh sampler only"); return OG_ERR_INVALID; }
    uint64_t slots = 0;
    replica_layout_t rl;
    if (!layout_init(g, m, c, &rl, &slots)) {
        snprintf(err, errlen, "sampler layout too large");
        return OG_ERR_INVALID;
    }
    chain_t ch;
    ch.cap = 1;
    while (ch.cap < 4 * (c->L + 1)) ch.cap <<= 1;
    ch.keys = (uint64_t*)malloc(ch.cap * sizeof(uint64_t));
    ch.status = (uint8_t*)malloc(ch.cap);
    ch.last = (uint32_t*)malloc(ch.cap * sizeof(uint32_t));
    /* all-positive nodes (mhw_device.cuh all_positive): every static weight
     * > 0, and a model that keeps w' > 0 (not metapath2vec; edge2vec only
     * with a positive M) */
    uint8_t* allpos = NULL;
    int model_pos = m->kind != OG_METAPATH2VEC;
    if (m->kind == OG_EDGE2VEC)
        for (uint32_t i = 0; i < m->M_dim * m->M_dim; ++i) if (!(m->M[i] > 0)) model_pos = 0;
    if (model_pos) {
        allpos = (uint8_t*)malloc(g->n ? g->n : 1);
        for (uint32_t v = 0; v < g->n; ++v) {
            uint8_t ok = 1;
            for (uint64_t a = g->offsets[v]; a < g->offsets[v + 1]; ++a) if (!(g->w[a] > 0)) { ok = 0; break; }
            allpos[v] = ok;
        }
    }
    ch.allpos = allpos;
    baseline_t bt;  /* static alias tables (proposal = alias) */
    memset(&bt, 0, sizeof(bt));
    if (c->proposal == OG_PROPOSAL_ALIAS) {
        bt.pstat = (uint8_t*)calloc(g->n ? g->n : 1, 1);
        bt.pprob = (double**)calloc(g->n ? g->n : 1, sizeof(double*));
        bt.palias = (uint32_t**)calloc(g->n ? g->n : 1, sizeof(uint32_t*));
    }
    int rc = OG_OK;
    uint64_t row = 0;
    for (uint64_t j = 0; j < count && rc == OG_OK; ++j) {
        const uint32_t v = starts[j];
        if (v >= g->n) { snprintf(err, errlen, "start node outside the graph"); rc = OG_ERR_INVALID; break; }
        for (uint32_t k = 0; k < c->K && rc == OG_OK; ++k) {
            walker_t w;
            w.v = v;
            w.walker = (uint64_t)v * c->K + k;
            xo_walker(&w.xo, c->seed, w.v, k);
            if (m->kind == OG_METAPATH2VEC) {
                if (g->ntype[w.v] != m->metapath[0]) { stats->skipped++; continue; }
                w.affix = 0;
            } else {
                w.affix = OG_NO_AFFIX;
            }
            memset(ch.keys, 0, ch.cap * sizeof(uint64_t));
            w.row = row++;
            rows[w.row * stride] = w.v;
            w.len = 1;
            for (uint32_t step = 0; step < c->L; ++step) {
                const int r = walker_step(g, m, c, &ch, &rl, &bt, &w, step, stride, rows, stats, err, errlen);
                if (r < 0) { rc = OG_ERR_INVALID; break; }
                if (r == 0) { stats->early++; break; }
            }
            lens[w.row] = w.len;
        }
    }
    stats->walks = row;
    *n_rows = row;
    if (bt.pstat) {
        for (uint32_t v = 0; v < g->n; ++v) { free(bt.pprob[v]); free(bt.palias[v]); }
        free(bt.pstat); free(bt.pprob); free(bt.palias);
    }
    free(ch.keys);
    free(ch.status);
    free(ch.last);
    free(allpos);
    free(rl.group);
    free(rl.scale);
    return rc;
}
