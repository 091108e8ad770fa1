// mhw_device.cuh -- device-side building blocks of the B200 walk engine.
//
// Graph layout in HBM, the counter-based random streams, the five walk models'
// dynamic edge weights as inlined functors (models.cpp:76-136 of the
// reference), the M-H accept rule (samplers.hpp:21-26) and slot
// initialisation (samplers.cpp:22-83). Everything here is __device__ code
// inlined into the kernels of graph.cu / walk.cu.
//
// Exactness: every fp64 operation that feeds
// a decision is an explicit round-to-nearest intrinsic, in the reference's
// association order, and the library is compiled with -fmad=false.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mhw {

constexpr uint32_t kNoAffix = 0xFFFFFFFFu;   // models.hpp:17
constexpr uint32_t kEmpty = 0xFFFFFFFFu;     // chain slot never initialised
constexpr uint32_t kDead = 0xFFFFFFFEu;      // chain slot is a dead end
constexpr uint32_t kLocked = 0xFFFFFFFDu;    // chain slot held by a walker mid-transition
constexpr uint32_t kIdxMask = 0x3FFFFFFFu;   // low 30 bits: Last index
constexpr uint32_t kMaxDegree = 0x3FFFFFF0u; // degrees must fit the index field
constexpr uint32_t kNoBack = 0xFFFFFFFFu;    // rev[] entry of an arc without back arc

enum Kind : int { DEEPWALK = 0, NODE2VEC = 1, METAPATH2VEC = 2, EDGE2VEC = 3, FAIRWALK = 4 };
enum InitKind : int { INIT_RANDOM = 0, INIT_HIGH_WEIGHT = 1, INIT_BURN_IN = 2 };

// Philox key domains; identical in oracle/mhw_oracle.c.
constexpr uint32_t DOM_WALK = 0x00000000u;
constexpr uint32_t DOM_INIT = 0x5EED1417u;
constexpr uint32_t DOM_RMAT = 0x2A7E0001u;
constexpr uint32_t DOM_WEIGHT = 0x3E1647u;
constexpr uint32_t DOM_ETYPE = 0x7E7E0003u;
constexpr uint32_t DOM_HETERO = 0x4E7E0004u;

// One 16-byte record per node: a single 32-byte sector load yields the slice
// base, degree, node type and flags.
struct __align__(16) NodeRec {
    long long off;
    uint32_t deg;
    uint16_t type;
    uint16_t flags;
};
constexpr uint16_t NF_ALLPOS = 1;  // every static weight of the slice is > 0

__host__ __device__ constexpr bool second_order(int k) {
    return k == NODE2VEC || k == EDGE2VEC || k == FAIRWALK;
}
// models whose weight functor reads the candidate's node type
__host__ __device__ constexpr bool typed_kind(int k) {
    return k == METAPATH2VEC || k == EDGE2VEC || k == FAIRWALK;
}

struct DevGraph {
    uint32_t n;
    uint64_t m;
    const NodeRec* __restrict__ nodes;
    const uint32_t* __restrict__ ids;
    const float* __restrict__ w;          // nullptr: unweighted (1.0)
    const uint16_t* __restrict__ etype;   // nullptr: derived from node types
    const uint32_t* __restrict__ rev;     // index of v in N(u) for arc v->u
    const double* __restrict__ wtotal;    // sequential fp64 slice sums
    const double* __restrict__ wblk;      // exact block prefix sums for the bootstrap (nullptr: not built)
    const uint32_t* __restrict__ tcount;  // fairwalk type counts, n * n_ntypes
    const uint32_t* __restrict__ htab;    // adjacency hash sets (nullptr: not built)
    const uint4* __restrict__ arc;        // arc records (nullptr: not built)
    const uint32_t* __restrict__ bloom;   // edge Bloom filter, 8 words per block (nullptr: not built)
    const uint32_t* __restrict__ tperm;   // per slice: neighbour indices ordered by (type, w > 0 first, index)
    const uint2* __restrict__ tbase;      // per (node, type): {start in tperm slice, count of w > 0}
    const uint4* __restrict__ sal;        // static alias tables per slice, {prob f64, alias, 0} (alias proposal; nullptr: none)
    uint32_t bloom_blocks;
    uint16_t n_ntypes;
    uint16_t n_etypes;
    int verified_sym;                     // every arc has its back arc
};

// One 32-byte sector in one request: sm_100's 256-bit vector load
// (LDG.E.ENL2.256). Two 16-byte __ldg of the same sector are two L1 lookups
// and, on a miss, two L2 requests; the L2-resident probes (edge filter, hash
// buckets) are request-rate bound.
__device__ __forceinline__ void ldg256(const void* p, uint4& lo, uint4& hi) {
    asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
}

// The same load with a cache hint (HINT 1: L2 evict-first, LDG.E.EFL2.256;
// 2: L2 evict-last, LDG.E.ELL2.256; 3: no L1 allocation, LDG.E.NA; 4: 3 + 1;
// 0: none). Build-time
// experiment knobs MHW_HASH_HINT / MHW_BLOOM_HINT / MHW_NODE8_HINT /
// MHW_STORE_HINT (scripts/build_variant.sh); results in DESIGN.md section 3.
template <int HINT>
__device__ __forceinline__ void ldg256h(const void* p, uint4& lo, uint4& hi) {
    if constexpr (HINT == 1)
        asm("ld.global.nc.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                     : "l"(p));
    else if constexpr (HINT == 2)
        asm("ld.global.nc.L2::evict_last.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                     : "l"(p));
    else if constexpr (HINT == 3)  // no L1 allocation (the line is not reused by this SM)
        asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                     : "l"(p));
    else if constexpr (HINT == 4)  // no L1 allocation, L2 evict-first
        asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                     : "l"(p));
    else
        ldg256(p, lo, hi);
}
// Defaults: the edge-filter blocks and hash buckets skip L1 allocation (an
// SM does not see the same line twice; L1 keeps the spilled frame instead):
// cfg2 init 4.27 -> 4.1 ms, step 24.05 -> 23.79; cfg3a / cfg3b / cfg4 / cfg5 equal.
#ifndef MHW_HASH_HINT
#define MHW_HASH_HINT 3
#endif
#ifndef MHW_BLOOM_HINT
#define MHW_BLOOM_HINT 3
#endif
#ifndef MHW_NODE8_HINT
#define MHW_NODE8_HINT 0
#endif
#ifndef MHW_STORE_HINT
#define MHW_STORE_HINT 0
#endif
#ifndef MHW_REC_HINT  // arc-record loads of the walk (16 / 32 bytes)
#define MHW_REC_HINT 0
#endif
#ifndef MHW_IDS_HINT  // compact-chain walk: the candidate id without L1 allocation (cfg2 walk 19.54 -> 18.89 ms)
#define MHW_IDS_HINT 3
#endif

template <int HINT>
__device__ __forceinline__ unsigned long long l2_policy() {
    unsigned long long pol = 0;
    if constexpr (HINT == 1) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if constexpr (HINT == 2) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
template <int HINT>
__device__ __forceinline__ uint2 ldg64h(const uint2* p) {
    if constexpr (HINT == 0) return __ldg(p);
    uint2 r;
    if constexpr (HINT == 3) {
        asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
        return r;
    }
    asm("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(l2_policy<HINT>()));
    return r;
}
template <int HINT>
__device__ __forceinline__ uint32_t ldg32h(const uint32_t* p) {
    if constexpr (HINT == 0) return __ldg(p);
    uint32_t r;
    if constexpr (HINT == 3) {
        asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
        return r;
    }
    if constexpr (HINT == 4) {  // no L1 allocation, L2 evict-first
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(l2_policy<1>()));
        return r;
    }
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(l2_policy<HINT>()));
    return r;
}
// One aligned 32-byte sector in one store (sm_100: STG.E.ENL2.256).
__device__ __forceinline__ void stg256(uint32_t* p, uint4 lo, uint4 hi) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(lo.x), "r"(lo.y), "r"(lo.z), "r"(lo.w),
                 "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
                 : "memory");
}
template <int HINT>
__device__ __forceinline__ uint4 ldg128h(const uint4* p) {
    if constexpr (HINT == 3) {
        uint4 r;
        asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
        return r;
    } else {
        return __ldg(p);
    }
}
template <int HINT>
__device__ __forceinline__ void stg128h(uint4* p, uint4 v) {
    if constexpr (HINT == 0) {
        *p = v;
    } else {
        asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                     "r"(v.w), "l"(l2_policy<HINT>())
                     : "memory");
    }
}

// ------------------------------------------------------------ arc records
// For graphs with < 2^32 arcs, arc a = (v -> u) has a 16-byte record
// {u, deg(u) | NF_ALLPOS(u) << 31, off(u), fp32 w(a)} (graph records, used by
// deepwalk; the other models use per-session records, walk.cu): one load
// yields everything the next walker state needs.

__device__ __forceinline__ NodeRec arc_node(uint4 a) {
    NodeRec r;
    r.off = (long long)a.z;
    r.deg = a.y & 0x7FFFFFFFu;
    r.type = 0;
    r.flags = (a.y >> 31) ? NF_ALLPOS : 0;
    return r;
}

// ------------------------------------------------- adjacency hash sets
// Nodes of degree >= kHashMinDeg get an exact hash set of their neighbour
// ids: ceil(deg/4) buckets of 8 u32 keys (one 32-byte sector, load <= 0.5),
// linear probing over buckets. Node v's buckets start at bucket
// (off_v >> 2) + v, so no per-node metadata is needed (the bases of
// consecutive nodes never overlap: floor((o+d)/4) + 1 >= floor(o/4) + ceil(d/4)).
constexpr uint32_t kHashMinDeg = 32;
constexpr uint32_t kHashEmpty = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint64_t hash_base(long long off, uint32_t v) {
    return ((uint64_t)off >> 2) + v;
}
__host__ __device__ __forceinline__ uint32_t hash_buckets(uint32_t deg) { return (deg + 3) >> 2; }
__host__ __device__ __forceinline__ uint32_t hash_bucket(uint32_t key, uint32_t nb) {
    uint32_t h = key;  // murmur3 fmix32
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return (uint32_t)(((uint64_t)h * nb) >> 32);
}

// ------------------------------------------------------ edge Bloom filter
// Blocked Bloom filter over undirected edges {a, b}: one 32-byte block per
// key (one sector, L2-resident when it fits), 4 bits set inside it. A miss
// proves non-adjacency exactly; a hit falls through to the exact test.
__host__ __device__ __forceinline__ uint64_t bloom_key(uint32_t a, uint32_t b) {
    uint64_t x = a < b ? (((uint64_t)a << 32) | b) : (((uint64_t)b << 32) | a);
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__host__ __device__ __forceinline__ uint32_t bloom_block(uint64_t x, uint32_t blocks) {
    return (uint32_t)(((x >> 32) * (uint64_t)blocks) >> 32);
}

__device__ __forceinline__ bool bloom_maybe(const DevGraph& g, uint32_t a, uint32_t b) {
    const uint64_t x = bloom_key(a, b);
    const uint4* blk = reinterpret_cast<const uint4*>(g.bloom) + 2 * (uint64_t)bloom_block(x, g.bloom_blocks);
    uint4 lo, hi;
    ldg256h<MHW_BLOOM_HINT>(blk, lo, hi);
    // 256-bit block as eight 32-bit words, selected by predicated moves (no
    // branches, no local array)
    bool all = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t bit = (uint32_t)(x >> (8 * k)) & 255u;
        const uint32_t j = bit >> 5;
        const uint32_t a = (j & 1) ? lo.y : lo.x, b = (j & 1) ? lo.w : lo.z;
        const uint32_t c = (j & 1) ? hi.y : hi.x, d = (j & 1) ? hi.w : hi.z;
        const uint32_t e = (j & 2) ? b : a, f = (j & 2) ? d : c;
        const uint32_t q = (j & 4) ? f : e;
        all &= ((q >> (bit & 31)) & 1u) != 0;
    }
    return all;
}

// HH: L2 eviction priority of the bucket loads (ldg256h). The compact-chain
// walk probes with evict-first: its pinned chain table leaves little L2, and
// a bucket of the 8 B/arc hash table is not reused (cfg2 walk 22.85 -> 22.63
// ms; cfg4, nothing pinned but the filter: 156.1 -> 157.1, so not there).
template <int HH = MHW_HASH_HINT>
__device__ __forceinline__ bool hash_contains(const uint32_t* __restrict__ tab, long long off, uint32_t v,
                                              uint32_t deg, uint32_t key) {
    const uint32_t nb = hash_buckets(deg);
    const uint4* base = reinterpret_cast<const uint4*>(tab) + 2 * hash_base(off, v);
    uint32_t b = hash_bucket(key, nb);
    for (;;) {
        uint4 x, y;
        ldg256h<HH>(base + 2 * b, x, y);
        if (x.x == key || x.y == key || x.z == key || x.w == key || y.x == key || y.y == key || y.z == key ||
            y.w == key)
            return true;
        if (y.w == kHashEmpty) return false;  // slots fill in order: a free last slot ends the probe
        b = b + 1 == nb ? 0 : b + 1;
    }
}

struct DevModel {
    int kind;
    double inv_p, inv_q;     // 1.0/p, 1.0/q computed on the host (models.cpp:77-79)
    int alpha_trivial;       // 1/p == 1 == 1/q: alpha is 1.0 whatever the class
    uint32_t spec_cls;       // the unique heaviest alpha class (3: none); its Lasts are fetched early
    // load-free rejections (compact chains, unweighted node2vec): with the
    // Last of the return class (w'(Last) = inv_p) and every other class
    // lighter (ret_wmax = max(1, inv_q) < inv_p), a proposal is rejected
    // whatever its class when u * inv_p >= ret_wmax, or when it is the Last
    int ret_skip;
    double ret_wmax;
    const uint16_t* metapath;
    uint32_t mp_len;
    const double* M;         // edge2vec type matrix, M_dim x M_dim
    uint32_t M_dim;
    int M_allpos;
    uint16_t num_types;      // graph.num_node_types at bind (models.cpp:30)
};

struct DevCfg {
    uint64_t seed;
    uint32_t K, L;
    int init_kind;
    uint32_t burn_in;
    uint32_t hw;
    // node-keyed chain replication at hubs
    uint32_t rep_deg;            // nodes with degree >= rep_deg get replicas
    uint32_t rep_max;            // replica cap (power of two)
    uint64_t rep_base_slot;      // first slot of the replica region (= n * G)
    int proposal;                // mhw_proposal: 0 uniform, 1 static-weight alias (Hastings accept)
    const uint32_t* rep_group;   // per node: first replica group (hubs only)
    const double* rep_scale;     // metapath2vec: per node type visit scale (nullptr: weight = degree)
};

constexpr uint32_t kNoReplicas = 0xFFFFFFFFu;
constexpr uint32_t kDefaultRepDeg = 32;  // metapath2vec auto replica weight threshold
constexpr uint32_t kMaxReplicas = 65536;
constexpr uint64_t kAutoReplicaSlots = uint64_t(8) << 20;  // auto D budget (32 MB of chain words)

// Chains per node-keyed state: 1 below rep_deg, else 2^(floor(log2(deg /
// rep_deg)) + 1) capped at 65536 -- about 2*deg/rep_deg concurrent chains, so a
// hub's visitors spread over independent exact M-H chains.
__host__ __device__ __forceinline__ uint32_t chain_replicas(uint32_t deg, uint32_t rep_deg,
                                                             uint32_t rep_max = kMaxReplicas) {
    if (rep_deg == kNoReplicas || deg < rep_deg) return 1;
    uint32_t q = deg / rep_deg, lg = 0;
    while (q >>= 1) ++lg;
    const uint32_t r = lg < 31 ? 2u << lg : 0x80000000u;
    return r < rep_max ? r : rep_max;
}

__host__ __device__ __forceinline__ uint32_t walker_replica(uint64_t walker, uint32_t R) {
    return (uint32_t)((walker * 0x9E3779B97F4A7C15ull) >> 40) & (R - 1);
}

// Replica weight of a node-keyed state: its expected visits in degree units.
// deepwalk: the degree (visits of an undirected walk are proportional to it).
// metapath2vec: deg * F[type], F_t = (share of metapath steps at type t) *
// arcs / (arcs incident to type-t nodes) -- a type visited every fourth
// step by walkers funnelled through few nodes (cfg3's V venues) weighs far
// more than its degree. floor of one IEEE product, identical in the oracle.
__host__ __device__ __forceinline__ uint32_t rep_weight(uint32_t deg, const double* scale, uint16_t type) {
    if (!scale) return deg;
#ifdef __CUDA_ARCH__
    const double x = __dmul_rn((double)deg, __ldg(scale + type));
#else
    const double x = (double)deg * scale[type];
#endif
    return x >= 2147483647.0 ? 0x7FFFFFFFu : (uint32_t)x;
}

// Slot of node-keyed state (v, t) for `walker`: G slots per node (1 for
// deepwalk, num_types for metapath2vec), replicas after the n*G base slots.
__device__ __forceinline__ uint64_t node_slot(const DevCfg& cfg, uint32_t G, uint32_t v, uint32_t deg,
                                              uint32_t t, uint64_t walker, uint16_t vtype = 0) {
    const uint64_t base = (uint64_t)v * G + t;
    const uint32_t R = chain_replicas(rep_weight(deg, cfg.rep_scale, vtype), cfg.rep_deg, cfg.rep_max);
    if (R == 1) return base;
    const uint32_t r = walker_replica(walker, R);
    if (r == 0) return base;
    return cfg.rep_base_slot + ((uint64_t)__ldg(cfg.rep_group + v) + r - 1) * G + t;
}

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11): 10 rounds, Weyl key schedule.
__host__ __device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
#ifdef __CUDA_ARCH__
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
#else
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

__host__ __device__ __forceinline__ uint2 philox_key(uint64_t seed, uint32_t domain) {
    return make_uint2((uint32_t)seed, (uint32_t)(seed >> 32) ^ domain);
}

__host__ __device__ __forceinline__ double unit53(uint32_t hi, uint32_t lo) {
    const uint64_t x = ((uint64_t)hi << 32) | lo;
    return (double)(x >> 11) * 0x1.0p-53;  // rng.hpp:59 construction
}

// Lemire rejection tail: retry words are w3, then sub-blocks ctr.w = 1, 2, ...
static __device__ __noinline__ uint32_t lemire_slow(uint4 w, uint2 key, uint4 ctr, uint32_t n) {
    const uint32_t threshold = (uint32_t)((0x100000000ULL - n) % n);
    uint64_t m = (uint64_t)w.x * n;
    uint32_t rpos = 3;
    while ((uint32_t)m < threshold) {
        if (rpos == 4) {
            ctr.w += 1;
            w = philox10(ctr, key);
            rpos = 0;
        }
        const uint32_t x = rpos == 0 ? w.x : rpos == 1 ? w.y : rpos == 2 ? w.z : w.w;
        ++rpos;
        m = (uint64_t)x * n;
    }
    return (uint32_t)(m >> 32);
}

// The draws of one transition: block (id, blk) of a domain.
struct Draw {
    uint4 w;
    uint4 ctr;
    uint2 key;
    __device__ __forceinline__ void open(uint2 k, uint64_t id, uint32_t blk) {
        key = k;
        ctr = make_uint4((uint32_t)id, (uint32_t)(id >> 32), blk, 0u);
        w = philox10(ctr, key);
    }
    // block (id, blk) with sub-counter ctr.w = sub (rejection trials)
    __device__ __forceinline__ void open_sub(uint2 k, uint64_t id, uint32_t blk, uint32_t sub) {
        key = k;
        ctr = make_uint4((uint32_t)id, (uint32_t)(id >> 32), blk, sub);
        w = philox10(ctr, key);
    }
    // uniform_index (rng.hpp:42-55) on word 0
    __device__ __forceinline__ uint32_t index(uint32_t n) const {
        const uint64_t m = (uint64_t)w.x * n;
        if ((uint32_t)m < n) return lemire_slow(w, key, ctr, n);
        return (uint32_t)(m >> 32);
    }
    // uniform_real (rng.hpp:58-60) on words 1,2
    __device__ __forceinline__ double unit() const { return unit53(w.y, w.z); }
};

// Sub-counter of the accept unit of an alias-proposal step (oracle
// OG_ACCEPT_SUB): block (walker, step, sub) words 1-2; Lemire retries use
// sub-counters 1, 2, ... of the same block and never reach it.
constexpr uint32_t kAcceptSub = 0x80000000u;

// --------------------------------------------------------------- loads
__device__ __forceinline__ NodeRec load_node(const DevGraph& g, uint32_t v) {
    const int4 r = __ldg(reinterpret_cast<const int4*>(g.nodes) + v);
    NodeRec n;
    n.off = ((long long)(uint32_t)r.y << 32) | (uint32_t)r.x;
    n.deg = (uint32_t)r.z;
    n.type = (uint16_t)((uint32_t)r.w & 0xFFFFu);
    n.flags = (uint16_t)((uint32_t)r.w >> 16);
    return n;
}
__device__ __forceinline__ uint32_t load_id(const DevGraph& g, long long arc) { return __ldg(g.ids + arc); }
__device__ __forceinline__ double static_w(const DevGraph& g, long long arc) {
    return g.w ? (double)__ldg(g.w + arc) : 1.0;
}

// Adjacency test: lower_bound (graph.cpp:13-18) with early exit on a hit.
__device__ __forceinline__ bool adj_search(const uint32_t* __restrict__ ids, long long off,
                                           uint32_t deg, uint32_t key) {
    const uint32_t* p = ids + off;
    uint32_t lo = 0, len = deg;
    while (len > 0) {
        const uint32_t half = len >> 1;
        const uint32_t x = __ldg(p + lo + half);
        if (x == key) return true;
        if (x < key) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return false;
}

// Exact lower_bound index; returns kNoBack when key is absent.
__device__ __forceinline__ uint32_t index_of(const uint32_t* __restrict__ ids, long long off,
                                             uint32_t deg, uint32_t key) {
    const uint32_t* p = ids + off;
    uint32_t lo = 0, len = deg;
    while (len > 0) {
        const uint32_t half = len >> 1;
        if (__ldg(p + lo + half) < key) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return (lo < deg && __ldg(p + lo) == key) ? lo : kNoBack;
}

// ------------------------------------------------------------ models
// State context of one transition distribution (WalkerState + what the
// weight functor reads). For second-order states s = N(v)[affix].
struct SCtx {
    uint32_t v;
    long long off;
    uint32_t deg;
    uint16_t vtype;
    uint16_t vflags;
    uint32_t s;          // previous node
    long long off_s;
    uint32_t deg_s;
    uint32_t in_type;    // edge2vec: type of arc s->v
    uint32_t req;        // metapath2vec: required type of the next node
    bool boot;           // second-order bootstrap (affix == kNoAffix)
};

// metapath_next / required_type, models.hpp:77-85
__device__ __forceinline__ uint32_t metapath_next(const DevModel& m, uint32_t affix) {
    if (affix + 1 < m.mp_len) return affix + 1;
    return (m.metapath[0] == m.metapath[m.mp_len - 1] && m.mp_len > 1) ? 1u : 0u;
}

// Graph::edge_type, graph.hpp:47-50
__device__ __forceinline__ uint32_t edge_type_of(const DevGraph& g, long long arc, uint16_t src_type,
                                                 uint16_t dst_type) {
    if (g.etype) return __ldg(g.etype + arc);
    return (uint16_t)(src_type * g.n_ntypes + dst_type);
}

// alpha class of candidate u under state c: 0 return (u == s), 1 adjacent to
// s, 2 otherwise (models.cpp:76-80). urec: the candidate's record if already
// loaded (lets a verified-symmetric graph search the shorter slice).
// bloom: the edge-filter result if the caller probed it already (1 maybe
// adjacent, 0 not), -1 to probe here. load_urec: without urec, fetch the
// candidate's record here when (and only when) the shorter-slice choice needs
// it -- callers keep a single call site, so lanes that need the record and
// lanes that do not stay converged through the filter probe.
template <int HH = MHW_HASH_HINT>
__device__ __forceinline__ uint32_t alpha_class(const DevGraph& g, const DevModel& m, const SCtx& c,
                                                uint32_t u, const NodeRec* urec, int bloom = -1,
                                                bool load_urec = false) {
    if (m.alpha_trivial) return 1;
    if (u == c.s) return 0;
    // the L2-resident edge filter settles most non-adjacent pairs without a
    // DRAM access
    if (g.bloom && !(bloom >= 0 ? bloom != 0 : bloom_maybe(g, c.s, u))) return 2;
    // s's own hash set needs nothing about u: probe it without waiting for
    // the candidate's node record (shorter dependency chain per step).
    if (g.htab && c.deg_s >= kHashMinDeg) return hash_contains<HH>(g.htab, c.off_s, c.s, c.deg_s, u) ? 1u : 2u;
    // is_adjacent(s, u): u in N(s), or s in N(u) when every arc has its
    // back arc. Cheapest structure first: a <= 8-entry slice (one sector),
    // else a hash set (one sector), else binary search of the shorter slice.
    uint32_t node_a = c.s, deg_a = c.deg_s, key_a = u;  // shorter slice
    long long off_a = c.off_s;
    uint32_t node_b = 0, deg_b = 0, key_b = 0;           // longer slice
    long long off_b = 0;
    const bool both = g.verified_sym && (urec || load_urec);
    if (both) {
        const NodeRec ur = urec ? *urec : load_node(g, u);
        node_b = u;
        off_b = ur.off;
        deg_b = ur.deg;
        key_b = c.s;
        if (deg_b < deg_a) {
            uint32_t t = node_a; node_a = node_b; node_b = t;
            t = deg_a; deg_a = deg_b; deg_b = t;
            t = key_a; key_a = key_b; key_b = t;
            const long long o = off_a; off_a = off_b; off_b = o;
        }
    }
    if (deg_a > 8 && g.htab) {
        if (deg_a >= kHashMinDeg) return hash_contains<HH>(g.htab, off_a, node_a, deg_a, key_a) ? 1u : 2u;
        if (both && deg_b >= kHashMinDeg) return hash_contains<HH>(g.htab, off_b, node_b, deg_b, key_b) ? 1u : 2u;
    }
    return adj_search(g.ids, off_a, deg_a, key_a) ? 1u : 2u;
}

// Does alpha_class look at the candidate's record? Only when s has no hash
// set and its slice is longer than one sector (then N(u) may be shorter).
__device__ __forceinline__ bool needs_urec_for_alpha(const DevGraph& g, const SCtx& c) {
    return g.verified_sym && c.deg_s > 8 && (c.deg_s < kHashMinDeg || !g.htab);
}

__device__ __forceinline__ double alpha_value(const DevModel& m, uint32_t cls) {
    return cls == 0 ? m.inv_p : (cls == 1 ? 1.0 : m.inv_q);
}

// Dynamic weight w' of candidate index i (node u, type utype, alpha class
// cls) under state c: WalkModel::calculate_weight, models.cpp:82-123.
// The same from the candidate's static weight w, node type utype and edge
// type out_t (edge2vec) already in registers (typed arc records).
template <int KIND>
__device__ __forceinline__ double wprime_v(const DevGraph& g, const DevModel& m, const SCtx& c, double w,
                                           uint16_t utype, uint32_t out_t, uint32_t cls) {
    if (KIND == DEEPWALK) return w;
    if (KIND == METAPATH2VEC) return utype == c.req ? w : 0.0;
    if (c.boot) return w;
    const double a = alpha_value(m, cls);
    if (KIND == NODE2VEC) return __dmul_rn(a, w);
    if (KIND == EDGE2VEC) return __dmul_rn(__dmul_rn(a, __ldg(m.M + (size_t)c.in_type * m.M_dim + out_t)), w);
    // FAIRWALK: a * w / group
    const uint32_t group = __ldg(g.tcount + (size_t)c.v * g.n_ntypes + utype);
    return __ddiv_rn(__dmul_rn(a, w), (double)group);
}

template <int KIND>
__device__ __forceinline__ double wprime(const DevGraph& g, const DevModel& m, const SCtx& c, uint32_t i,
                                         uint16_t utype, uint32_t cls) {
    const double w = static_w(g, c.off + i);
    uint32_t out_t = 0;
    if (KIND == EDGE2VEC && !c.boot) out_t = edge_type_of(g, c.off + i, c.vtype, utype);
    return wprime_v<KIND>(g, m, c, w, utype, out_t, cls);
}

// Dynamic factor r = w'/w of a candidate (node type utype, out edge type
// out_t, alpha class cls): calculate_weight (models.cpp:82-123) without the
// trailing static weight -- the Hastings ratio of the alias proposal
// (q proportional to w) is r_c / r_l. Same association as oracle og_rfactor.
template <int KIND>
__device__ __forceinline__ double rfactor(const DevGraph& g, const DevModel& m, const SCtx& c, uint16_t utype,
                                          uint32_t out_t, uint32_t cls) {
    if (KIND == DEEPWALK) return 1.0;
    if (KIND == METAPATH2VEC) return utype == c.req ? 1.0 : 0.0;
    if (c.boot) return 1.0;
    const double a = alpha_value(m, cls);
    if (KIND == NODE2VEC) return a;
    if (KIND == EDGE2VEC) return __dmul_rn(a, __ldg(m.M + (size_t)c.in_type * m.M_dim + out_t));
    return __ddiv_rn(a, (double)__ldg(g.tcount + (size_t)c.v * g.n_ntypes + utype));
}

// Hastings accept of an alias proposal (og_hastings): candidate of static
// weight w_c, factors r_c, r_l, unit u.
__device__ __forceinline__ bool hastings_accept(double w_c, double r_c, double r_l, double u) {
    return w_c > 0.0 && (r_l <= 0.0 || r_c >= r_l || __dmul_rn(u, r_l) < r_c);
}

template <int KIND>
__host__ __device__ constexpr bool needs_utype() {
    return KIND == METAPATH2VEC || KIND == FAIRWALK || KIND == EDGE2VEC;
}

// Full evaluation of candidate i (loads its id/record as needed); cls out.
template <int KIND>
__device__ __forceinline__ double eval_index(const DevGraph& g, const DevModel& m, const SCtx& c,
                                             uint32_t i, uint32_t* cls_out) {
    uint32_t cls = 0;
    uint16_t utype = 0;
    if (KIND != DEEPWALK) {
        const uint32_t u = load_id(g, c.off + i);
        if (second_order(KIND) && !c.boot && !m.alpha_trivial) {
            if (needs_utype<KIND>()) {
                const NodeRec r = load_node(g, u);
                utype = r.type;
                cls = alpha_class(g, m, c, u, &r);
            } else {
                cls = alpha_class(g, m, c, u, nullptr, -1, true);
            }
        } else {
            if (needs_utype<KIND>()) utype = load_node(g, u).type;
            if (second_order(KIND)) cls = 1;
        }
    }
    *cls_out = cls;
    return wprime<KIND>(g, m, c, i, utype, cls);
}

// The same evaluation as eval_index, returning the dynamic factor r = w'/w
// (rfactor) of candidate i -- the alias proposal's Hastings ratio input.
template <int KIND>
__device__ __forceinline__ double eval_rfactor(const DevGraph& g, const DevModel& m, const SCtx& c, uint32_t i) {
    uint32_t cls = 0;
    uint16_t utype = 0;
    if (KIND != DEEPWALK) {
        const uint32_t u = load_id(g, c.off + i);
        if (second_order(KIND) && !c.boot && !m.alpha_trivial) {
            if (needs_utype<KIND>()) {
                const NodeRec r = load_node(g, u);
                utype = r.type;
                cls = alpha_class(g, m, c, u, &r);
            } else {
                cls = alpha_class(g, m, c, u, nullptr, -1, true);
            }
        } else {
            if (needs_utype<KIND>()) utype = load_node(g, u).type;
            if (second_order(KIND)) cls = 1;
        }
    }
    const uint32_t out_t = (KIND == EDGE2VEC && !c.boot) ? edge_type_of(g, c.off + i, c.vtype, utype) : 0u;
    return rfactor<KIND>(g, m, c, utype, out_t, cls);
}

// accept rule, samplers.hpp:24
__device__ __forceinline__ bool mh_accept(double wc, double wl, double u) {
    return wl <= 0.0 || wc >= wl || __dmul_rn(u, wl) < wc;
}

__device__ __forceinline__ uint32_t pack_entry(uint32_t idx, uint32_t cls) { return idx | (cls << 30); }

// Builds the state context of (v, affix) from memory (decide / init /
// deterministic schedule; the throughput kernel keeps it in registers).
template <int KIND>
__device__ __forceinline__ SCtx make_ctx(const DevGraph& g, const DevModel& m, uint32_t v, uint32_t affix) {
    SCtx c;
    const NodeRec r = load_node(g, v);
    c.v = v;
    c.off = r.off;
    c.deg = r.deg;
    c.vtype = r.type;
    c.vflags = r.flags;
    c.s = 0;
    c.off_s = 0;
    c.deg_s = 0;
    c.in_type = 0;
    c.req = 0;
    c.boot = false;
    if (KIND == METAPATH2VEC) c.req = m.metapath[metapath_next(m, affix)];
    if (second_order(KIND)) {
        if (affix == kNoAffix) {
            c.boot = true;
        } else {
            c.s = load_id(g, c.off + affix);
            const NodeRec rs = load_node(g, c.s);
            c.off_s = rs.off;
            c.deg_s = rs.deg;
            if (KIND == EDGE2VEC) {
                // arc s->v sits at index rev[v->s] of N(s) (graph.cpp:13-18 lookup)
                const uint32_t sv = g.rev ? __ldg(g.rev + c.off + affix) : index_of(g.ids, rs.off, rs.deg, v);
                c.in_type = edge_type_of(g, rs.off + sv, rs.type, r.type);
            }
        }
    }
    return c;
}

// Slot of state (v, affix) used by `walker`: manager.hpp:29-31 +
// models.cpp:163-172, with hub replicas for node-keyed models.
template <int KIND>
__device__ __forceinline__ uint64_t slot_of(const DevModel& m, const DevCfg& cfg, const SCtx& c, uint32_t affix,
                                            uint64_t walker) {
    if (KIND == DEEPWALK) return node_slot(cfg, 1, c.v, c.deg, 0, walker);
    if (KIND == METAPATH2VEC) return node_slot(cfg, m.num_types, c.v, c.deg, c.req, walker, c.vtype);
    return (uint64_t)c.off + affix;
}

template <int KIND>
__device__ __forceinline__ bool all_positive(const DevModel& m, const SCtx& c) {
    if (KIND == METAPATH2VEC) return false;
    if (KIND == EDGE2VEC && !m.M_allpos) return false;
    return (c.vflags & NF_ALLPOS) != 0;
}

// random_positive (samplers.cpp:22-33) with the pick drawn from block `blk`.
template <int KIND>
__device__ bool random_positive(const DevGraph& g, const DevModel& m, const SCtx& c, uint2 key,
                                uint64_t slot, uint32_t blk, uint32_t* out, uint32_t* cls_out,
                                double* w_out) {
    Draw d;
    d.open(key, slot, blk);
    if (KIND == METAPATH2VEC && g.tbase) {
        // w' > 0 exactly for the neighbours of the required type with w > 0
        // (models.cpp:91-94); the typed index lists them in index order, so
        // the pick-th positive is one lookup instead of two slice scans.
        const uint2 b = __ldg(g.tbase + (size_t)c.v * g.n_ntypes + c.req);
        if (b.y == 0) return false;
        const uint32_t i = __ldg(g.tperm + c.off + b.x + d.index(b.y));
        *out = i;
        *w_out = eval_index<KIND>(g, m, c, i, cls_out);
        return true;
    }
    if (all_positive<KIND>(m, c)) {
        const uint32_t pick = d.index(c.deg);
        *out = pick;
        *w_out = eval_index<KIND>(g, m, c, pick, cls_out);
        return true;
    }
    uint32_t positive = 0, cls;
    for (uint32_t i = 0; i < c.deg; ++i) positive += eval_index<KIND>(g, m, c, i, &cls) > 0 ? 1u : 0u;
    if (positive == 0) return false;
    uint32_t pick = d.index(positive);
    for (uint32_t i = 0; i < c.deg; ++i) {
        const double w = eval_index<KIND>(g, m, c, i, &cls);
        if (w > 0 && pick-- == 0) {
            *out = i;
            *cls_out = cls;
            *w_out = w;
            return true;
        }
    }
    return false;
}

// mh_init (samplers.cpp:37-83) with slot-keyed Philox blocks: random -> block
// 0; high_weight probes -> blocks 0..hw-1, fallback -> block hw; burn_in ->
// block 0 pick, blocks 1..k transitions. Returns the packed entry or kDead.
// w_out (optional) receives w'(Last) of the returned entry.
template <int KIND>
__device__ uint32_t init_slot(const DevGraph& g, const DevModel& m, const DevCfg& cfg, const SCtx& c,
                              uint64_t slot, double* w_out = nullptr) {
    if (c.deg == 0) return kDead;
    const uint2 key = philox_key(cfg.seed, DOM_INIT);
    uint32_t last, cls;
    double wl;
    if (cfg.init_kind == INIT_RANDOM) {
        if (!random_positive<KIND>(g, m, c, key, slot, 0, &last, &cls, &wl)) return kDead;
        if (w_out) *w_out = wl;
        return pack_entry(last, cls);
    }
    if (cfg.init_kind == INIT_HIGH_WEIGHT) {
        double best_w = 0.0;
        uint32_t best = 0, best_cls = 0;
        bool found = false;
        if (c.deg <= cfg.hw) {
            for (uint32_t i = 0; i < c.deg; ++i) {
                uint32_t ci;
                const double w = eval_index<KIND>(g, m, c, i, &ci);
                if (w > best_w) {
                    best_w = w;
                    best = i;
                    best_cls = ci;
                    found = true;
                }
            }
        } else {
            for (uint32_t probe = 0; probe < cfg.hw; ++probe) {
                Draw d;
                d.open(key, slot, probe);
                const uint32_t i = d.index(c.deg);
                uint32_t ci;
                const double w = eval_index<KIND>(g, m, c, i, &ci);
                if (w > best_w || (w == best_w && found && i < best)) {
                    if (w > 0) {
                        best_w = w;
                        best = i;
                        best_cls = ci;
                        found = true;
                    }
                }
            }
            if (!found) {
                if (!random_positive<KIND>(g, m, c, key, slot, cfg.hw, &last, &cls, &wl)) return kDead;
                if (w_out) *w_out = wl;
                return pack_entry(last, cls);
            }
        }
        if (w_out) *w_out = best_w;
        return found ? pack_entry(best, best_cls) : kDead;
    }
    // burn-in
    if (!random_positive<KIND>(g, m, c, key, slot, 0, &last, &cls, &wl)) return kDead;
    for (uint32_t i = 0; i < cfg.burn_in; ++i) {
        Draw d;
        d.open(key, slot, 1 + i);
        const uint32_t cand = d.index(c.deg);
        uint32_t cc;
        const double wc = eval_index<KIND>(g, m, c, cand, &cc);
        if (mh_accept(wc, wl, d.unit())) {
            last = cand;
            cls = cc;
            wl = wc;
        }
    }
    if (w_out) *w_out = wl;
    return pack_entry(last, cls);
}

// Block prefix sums of the weighted bootstrap: node v's blocks of 32 arcs
// start at entry (off >> 5) + v (disjoint across nodes, as hash_base).
constexpr uint32_t kBootBlkMin = 64;
__host__ __device__ __forceinline__ uint64_t wblk_base(long long off, uint32_t v) {
    return ((uint64_t)off >> 5) + v;
}

// Bootstrap step of a second-order walk: direct_sample over static weights
// (engine.cpp:81-83, samplers.cpp:133-146). Unweighted: min(floor(u*deg),
// deg-1), which is what the sequential r -= 1.0 loop returns exactly.
__device__ __forceinline__ bool bootstrap_pick(const DevGraph& g, const SCtx& c, double u, uint32_t* out) {
    if (!g.w) {
        uint32_t i = (uint32_t)__dmul_rn(u, (double)c.deg);
        *out = i < c.deg ? i : c.deg - 1;
        return true;
    }
    const double total = __ldg(g.wtotal + c.v);
    if (!(total > 0)) return false;
    double r = __dmul_rn(u, total);
    const float* w = g.w + c.off;
    uint32_t i0 = 0;
    if (g.wblk && c.deg >= kBootBlkMin) {
        // Exact block prefix sums (built only where every subtraction of the
        // sequential scan is exact, see k_wblk): r - P[b-1] is then exactly
        // the remainder the reference holds after 32b subtractions, so the
        // scan can start at the block where the remainder turns negative.
        const double* P = g.wblk + wblk_base(c.off, c.v);
        if (__ldg(P) == __ldg(P)) {  // NaN marks a slice without the exactness guarantee
            uint32_t lo = 0, len = (c.deg + 31) >> 5;
            while (len > 0) {  // first block whose end prefix exceeds r
                const uint32_t half = len >> 1;
                if (__ldg(P + lo + half) <= r) {
                    lo += half + 1;
                    len -= half + 1;
                } else {
                    len = half;
                }
            }
            if (lo == (c.deg + 31) >> 5) {
                i0 = c.deg;  // r >= total: no crossing, fallback below
            } else {
                if (lo) r = __dsub_rn(r, __ldg(P + lo - 1));
                i0 = 32 * lo;
            }
        }
    }
    for (uint32_t i = i0; i < c.deg; ++i) {
        r = __dsub_rn(r, (double)__ldg(w + i));
        if (r < 0) {
            *out = i;
            return true;
        }
    }
    for (uint32_t i = c.deg; i-- > 0;) {
        if (__ldg(w + i) > 0) {
            *out = i;
            return true;
        }
    }
    *out = 0;
    return true;
}

}  // namespace mhw
