// graph.cu -- device-resident CSR: upload, build from edges, synthetic
// generators, derived per-arc/per-node arrays and alias tables.
//
// Reference semantics: build_csr / load_edge_list (graph.cpp:35-100), type
// loaders (graph.cpp:102-177), fairwalk type counts (models.cpp:66-73),
// alias_build (samplers.cpp:95-131).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace mhw {

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    cudaGetLastError();
    const mhw_status code = MHW_ERR_CUDA;
    std::string msg = std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                      std::to_string(line) + ")";
    if (e == cudaErrorMemoryAllocation) msg = "out of device memory: " + msg;
    throw Error(code, msg);
}

// ------------------------------------------------------- device allocation
// Large buffers come from the device's stream-ordered memory pool with an
// unbounded release threshold: a session's multi-GB buffers are reallocated
// on every generate_walks call, and the pool sub-allocates freed memory for
// any later size (cudaMalloc/cudaFree of such blocks cost milliseconds each
// and cudaFree synchronises the device). Allocation and free are ordered on
// the legacy stream and completed before returning, so a block is usable on
// every stream; a free first waits for in-flight work that may still read it.
namespace {
constexpr size_t kPoolMin = 1ull << 20;
std::mutex g_pool_mu;
bool g_pool_ready[64] = {};

void pool_setup(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev < 0 || dev >= 64 || g_pool_ready[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    g_pool_ready[dev] = true;
}
}  // namespace

void* dev_alloc(size_t bytes, size_t* cap) {
    int dev = 0;
    cudaGetDevice(&dev);
    void* p = nullptr;
    *cap = bytes;
    if (bytes >= kPoolMin) {
        pool_setup(dev);
        cudaError_t e = cudaMallocAsync(&p, bytes, 0);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            dev_trim();
            e = cudaMallocAsync(&p, bytes, 0);
        }
        if (e != cudaSuccess) throw_cuda(e, "cudaMallocAsync", __FILE__, __LINE__);
        MHW_CK(cudaStreamSynchronize(0));
        return p;
    }
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        dev_trim();
        e = cudaMalloc(&p, bytes);
    }
    if (e != cudaSuccess) throw_cuda(e, "cudaMalloc", __FILE__, __LINE__);
    return p;
}

void dev_free(void* p, size_t cap) {
    if (!p) return;
    if (cap < kPoolMin) {
        cudaFree(p);
        return;
    }
    // the block may still be read by in-flight work on any stream
    cudaDeviceSynchronize();
    cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
}

// Returns the pools' unused memory to the device.
void dev_trim() {
    int prev = 0, n = 0;
    cudaGetDevice(&prev);
    cudaGetDeviceCount(&n);
    for (int d = 0; d < n && d < 64; ++d) {
        if (!g_pool_ready[d]) continue;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, d) != cudaSuccess) continue;
        cudaSetDevice(d);
        cudaDeviceSynchronize();
        cudaMemPoolTrimTo(pool, 0);
    }
    cudaSetDevice(prev);
}

// Device memory available to dev_alloc: the driver's free memory plus what
// the pool holds reserved but unused (cudaMemGetInfo counts that as used;
// trimming it to make the number look bigger would only make the next
// allocations map it again).
size_t dev_available_bytes() {
    size_t f = 0, t = 0;
    MHW_CK(cudaMemGetInfo(&f, &t));
    return f + dev_cached_bytes();
}

size_t dev_cached_bytes() {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return 0;
    uint64_t reserved = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    return reserved > used ? (size_t)(reserved - used) : 0;
}

DevGraph Graph::view() const {
    DevGraph d;
    d.n = n;
    d.m = m;
    d.nodes = nodes.p;
    d.ids = ids.p;
    d.w = w.n ? w.p : nullptr;
    d.etype = etype.n ? etype.p : nullptr;
    d.rev = rev.n ? rev.p : nullptr;
    d.wtotal = wtotal.n ? wtotal.p : nullptr;
    d.wblk = wblk.n ? wblk.p : nullptr;
    d.tcount = tcount.n ? tcount.p : nullptr;
    d.tperm = tperm.n ? tperm.p : nullptr;
    d.tbase = tbase.n ? tbase.p : nullptr;
    d.htab = htab.n ? htab.p : nullptr;
    d.arc = arc.n ? arc.p : nullptr;
    d.bloom = bloom.n ? bloom.p : nullptr;
    d.sal = sal.n ? sal.p : nullptr;
    d.bloom_blocks = bloom_blocks;
    d.n_ntypes = n_ntypes;
    d.n_etypes = n_etypes;
    d.verified_sym = verified_sym ? 1 : 0;
    return d;
}

uint64_t Graph::device_bytes() const {
    return nodes.bytes() + ids.bytes() + w.bytes() + ntype.bytes() + etype.bytes() + rev.bytes() +
           wtotal.bytes() + wblk.bytes() + tcount.bytes() + tperm.bytes() + tbase.bytes() + htab.bytes() + arc.bytes() + bloom.bytes() +
           sal.bytes();
}

namespace {

constexpr int kBlock = 256;

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

unsigned grid_for(uint64_t work, int per_block = kBlock) {
    const uint64_t g = (work + per_block - 1) / per_block;
    const uint64_t cap = (uint64_t)sm_count() * 16;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, cap));
}

enum : unsigned { ERR_OFFSETS = 1, ERR_RANGE = 2, ERR_UNSORTED = 4, ERR_NEGATIVE = 8, ERR_DEGREE = 16 };

// Warp per node: NodeRec, slice validation (ids in range, strictly
// ascending, weights >= 0), NF_ALLPOS, degree statistics.
__global__ void k_nodes(const int64_t* __restrict__ off, const uint16_t* __restrict__ ntype,
                        const uint32_t* __restrict__ ids, const float* __restrict__ w, uint32_t n,
                        uint64_t m, NodeRec* __restrict__ nodes, unsigned* __restrict__ stats) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = wid; v < n; v += nw) {
        const int64_t a = off[v], b = off[v + 1];
        unsigned err = 0;
        if (a < 0 || b < a || (uint64_t)b > m) err |= ERR_OFFSETS;
        else if ((uint64_t)(b - a) >= kMaxDegree) err |= ERR_DEGREE;
        bool allpos = true;
        if (!err) {
            for (int64_t i = a + lane; i < b; i += 32) {
                const uint32_t x = ids[i];
                if (x >= n) err |= ERR_RANGE;
                if (i > a && ids[i - 1] >= x) err |= ERR_UNSORTED;
                if (w) {
                    const float wi = w[i];
                    if (!(wi > 0.0f)) allpos = false;
                    if (!(wi >= 0.0f)) err |= ERR_NEGATIVE;
                }
            }
        }
        err = __reduce_or_sync(0xffffffffu, err);
        allpos = __all_sync(0xffffffffu, allpos);
        if (lane == 0) {
            const uint32_t deg = err ? 0u : (uint32_t)(b - a);
            NodeRec r;
            r.off = a;
            r.deg = deg;
            r.type = ntype ? ntype[v] : 0;
            r.flags = (allpos && deg > 0) ? NF_ALLPOS : 0;
            nodes[v] = r;
            if (err) atomicOr(&stats[0], err);
            atomicMax(&stats[1], deg);
            if (deg == 0) atomicAdd(&stats[2], 1u);
        }
    }
}

// Warp per node: rev[arc v->u] = index of v in N(u), or kNoBack.
__global__ void k_rev(DevGraph g, uint32_t* __restrict__ rev, unsigned* __restrict__ missing) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = wid; v < g.n; v += nw) {
        const NodeRec r = load_node(g, (uint32_t)v);
        bool miss = false;
        for (uint32_t i = lane; i < r.deg; i += 32) {
            const uint32_t u = load_id(g, r.off + i);
            const NodeRec ru = load_node(g, u);
            const uint32_t b = index_of(g.ids, ru.off, ru.deg, (uint32_t)v);
            rev[r.off + i] = b;
            miss |= b == kNoBack;
        }
        if (__any_sync(0xffffffffu, miss) && lane == 0) atomicAdd(missing, 1u);
    }
}

// Source node of arc a: the last v with nodes[v].off <= a (isolated nodes
// share their successor's offset and are skipped by "last").
__device__ __forceinline__ uint32_t arc_source(const DevGraph& g, uint64_t a) {
    uint32_t lo = 0, hi = g.n;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldg(&g.nodes[mid].off) <= a) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Thread per arc: insert u into the hash set of its source (degree >=
// kHashMinDeg). Arc-parallel so hubs do not serialise on one warp; the
// bucket is read once and only the first free slot is CAS-ed.
__global__ void k_hash_build(DevGraph g, uint32_t* __restrict__ tab) {
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < g.m;
         a += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = arc_source(g, a);
        const NodeRec r = load_node(g, v);
        if (r.deg < kHashMinDeg) continue;
        const uint32_t nb = hash_buckets(r.deg);
        uint32_t* base = tab + 8 * hash_base(r.off, v);
        const uint32_t key = load_id(g, a);
        uint32_t b = hash_bucket(key, nb);
        for (;;) {
            uint32_t* bk = base + 8 * b;
            int s = 0;
            while (s < 8) {
                const uint32_t cur = __ldcg(bk + s);
                if (cur != kHashEmpty) {
                    ++s;
                    continue;
                }
                if (atomicCAS(bk + s, kHashEmpty, key) == kHashEmpty) break;
                // lost the race for slot s: it is now taken, look further
                ++s;
            }
            if (s < 8) break;
            b = b + 1 == nb ? 0 : b + 1;
        }
    }
}

// Thread per arc: arc record {u, deg(u)|allpos<<31, off(u), fp32 w(a)}.
__global__ void k_arcrec(DevGraph g, uint4* __restrict__ out) {
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < g.m;
         a += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = load_id(g, a);
        const NodeRec r = load_node(g, u);
        const uint32_t x = __float_as_uint(g.w ? __ldg(g.w + a) : 1.0f);
        out[a] = make_uint4(u, r.deg | ((r.flags & NF_ALLPOS) ? 0x80000000u : 0u), (uint32_t)r.off, x);
    }
}

// rev[] by sorting: keys (dst << bits | src) of every arc. For a symmetric
// CSR the k-th arc in (dst, src) order is the reverse of CSR arc k.
// Keys = destination u of every arc, values = (source v, index within N(v)),
// in CSR order; a stable sort by u alone then lists each u's in-arcs by
// increasing v (CSR order is v-major), i.e. in N(u) order for a symmetric
// CSR -- half the radix passes of sorting (u, v) pairs.
__global__ void k_rev_keys(DevGraph g, uint32_t* __restrict__ keys, uint64_t* __restrict__ vals) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = wid; v < g.n; v += nw) {
        const NodeRec r = load_node(g, (uint32_t)v);
        for (uint32_t i = lane; i < r.deg; i += 32) {
            keys[r.off + i] = load_id(g, r.off + i);
            vals[r.off + i] = (v << 32) | i;  // source and index of the arc within its slice
        }
    }
}

// Sorted position k holds arc (v -> u) with key u: if CSR arc k is
// (u -> v) then v sits at index k - off(u) of N(u).
__global__ void k_rev_scatter(DevGraph g, const uint32_t* __restrict__ keys, const uint64_t* __restrict__ vals,
                              uint32_t* __restrict__ rev, unsigned* __restrict__ mismatch) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = keys[k];
        const uint64_t val = vals[k];
        const uint32_t v = (uint32_t)(val >> 32);
        const NodeRec ru = load_node(g, u);
        const NodeRec rv = load_node(g, v);
        const bool ok = (uint64_t)ru.off <= k && k < (uint64_t)ru.off + ru.deg && load_id(g, k) == v;
        if (!ok) {
            atomicAdd(mismatch, 1u);
            continue;
        }
        rev[rv.off + (uint32_t)val] = (uint32_t)(k - (uint64_t)ru.off);
    }
}

// Thread per node: sequential fp64 slice sum (std::accumulate order,
// samplers.cpp:134).
__global__ void k_wtotal(DevGraph g, double* __restrict__ out) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const NodeRec r = load_node(g, (uint32_t)v);
        double t = 0.0;
        for (uint32_t i = 0; i < r.deg; ++i) t = __dadd_rn(t, (double)g.w[r.off + i]);
        out[v] = t;
    }
}

// Warp per node of degree >= kBootBlkMin: exact block prefix sums for the
// weighted bootstrap (bootstrap_pick). direct_sample subtracts the weights
// one by one from r = u * total (samplers.cpp:136-145). With weights >= 0
// that are all multiples of 2^e (e = the smallest fp32 ulp exponent in the
// slice) and total < 2^(53 + e), every remainder the scan keeps is exact
// (r - P_i, P_i the exact prefix), and the first negative one has the right
// sign; so block prefixes (exact in any summation order) locate the crossing
// block and the scan resumes there with identical arithmetic. Slices without
// that guarantee get NaN in their first entry and keep the full scan.
__global__ void k_wblk(DevGraph g, double* __restrict__ out) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = wid; v < g.n; v += nw) {
        const NodeRec r = load_node(g, (uint32_t)v);
        if (r.deg < kBootBlkMin) continue;
        const float* w = g.w + r.off;
        int emin = 1 << 20;
        double tot = 0.0;
        for (uint32_t i = lane; i < r.deg; i += 32) {
            const float x = w[i];
            if (x > 0.0f) {
                const int ex = x >= 1.17549435e-38f ? ((__float_as_int(x) >> 23) & 0xFF) - 127 - 23 : -149;
                emin = min(emin, ex);
            }
            tot += (double)x;
        }
        for (int o = 16; o; o >>= 1) {
            emin = min(emin, __shfl_xor_sync(0xFFFFFFFFu, emin, o));
            tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
        }
        double* P = out + wblk_base(r.off, (uint32_t)v);
        const uint32_t nb = (r.deg + 31) >> 5;
        // emin == 1 << 20: all weights zero (total 0, the bootstrap is a dead end)
        const bool exact = emin < (1 << 20) && emin + 53 < 1000 && tot < ldexp(1.0, emin + 53);
        if (!exact) {
            if (lane == 0) P[0] = __longlong_as_double(0x7FF8000000000000ll);
            continue;
        }
        double carry = 0.0;
        for (uint32_t b0 = 0; b0 < nb; b0 += 32) {
            const uint32_t b = b0 + lane;
            double x = 0.0;
            if (b < nb) {
                const uint32_t e = min(r.deg, 32 * b + 32);
                for (uint32_t i = 32 * b; i < e; ++i) x += (double)w[i];
            }
            for (int o = 1; o < 32; o <<= 1) {  // inclusive scan over the 32 blocks
                const double y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= (unsigned)o) x += y;
            }
            x += carry;
            if (b < nb) P[b] = x;
            carry = __shfl_sync(0xFFFFFFFFu, x, 31);
        }
    }
}

// Warp per node: type_counts[v*T + type(u)] (models.cpp:66-73).
__global__ void k_tcount(DevGraph g, uint32_t* __restrict__ tc) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t T = g.n_ntypes;
    for (uint64_t v = wid; v < g.n; v += nw) {
        const NodeRec r = load_node(g, (uint32_t)v);
        for (uint32_t i = lane; i < r.deg; i += 32) {
            const uint16_t t = load_node(g, load_id(g, r.off + i)).type;
            atomicAdd(tc + v * T + t, 1u);
        }
    }
}

// Typed neighbour index (metapath2vec's random_positive, samplers.cpp:22-33):
// each slice's indices ordered by key = 2 * type(u) + (w > 0 ? 0 : 1), index
// order kept within a key, and per (node, type) the start of its positive
// block and its length. Three passes, warp per node: key counts, exclusive
// bases (thread per node), stable scatter (match_any ranks per 32 arcs).
__device__ __forceinline__ uint32_t tidx_key(const DevGraph& g, uint64_t a) {
    const uint16_t t = load_node(g, load_id(g, a)).type;
    const bool pos = g.w ? __ldg(g.w + a) > 0.0f : true;
    return 2u * t + (pos ? 0u : 1u);
}

__global__ void k_tidx_count(DevGraph g, uint32_t* __restrict__ cnt) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t K = 2u * g.n_ntypes;
    for (uint64_t v = wid; v < g.n; v += nw) {
        const NodeRec r = load_node(g, (uint32_t)v);
        for (uint32_t i = lane; i < r.deg; i += 32) atomicAdd(cnt + v * K + tidx_key(g, r.off + i), 1u);
    }
}

__global__ void k_tidx_base(DevGraph g, uint32_t* __restrict__ cnt, uint2* __restrict__ base) {
    const uint32_t K = 2u * g.n_ntypes;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t run = 0;
        for (uint32_t k = 0; k < K; ++k) {
            const uint32_t c = cnt[v * K + k];
            cnt[v * K + k] = run;  // becomes the scatter cursor of key k
            if (!(k & 1)) base[v * g.n_ntypes + k / 2] = make_uint2(run, c);
            run += c;
        }
    }
}

__global__ void k_tidx_scatter(DevGraph g, uint32_t* __restrict__ cur, uint32_t* __restrict__ perm) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t K = 2u * g.n_ntypes;
    for (uint64_t v = wid; v < g.n; v += nw) {
        const NodeRec r = load_node(g, (uint32_t)v);
        uint32_t* cv = cur + v * K;
        for (uint32_t i0 = 0; i0 < r.deg; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool live = i < r.deg;
            const uint32_t key = live ? tidx_key(g, r.off + i) : 0xFFFFFFFFu;
            const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
            const uint32_t rank = __popc(peers & ((1u << lane) - 1));
            const uint32_t b = live ? cv[key] : 0;
            __syncwarp();
            if (live) {
                perm[r.off + b + rank] = i;
                if (rank == 0) cv[key] = b + __popc(peers);
            }
            __syncwarp();
        }
    }
}

// Edge Bloom filter: warp per node v, every arc v -> u sets the 4 bits of
// the unordered key {v, u} (a symmetric pair sets them twice; an asymmetric
// graph stays exact: any arc s -> x makes {s, x} a hit).
__global__ void k_bloom_build(DevGraph g, uint32_t* __restrict__ bloom, uint32_t blocks) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = wid; v < g.n; v += nw) {
        const NodeRec r = load_node(g, (uint32_t)v);
        for (uint32_t i = lane; i < r.deg; i += 32) {
            const uint32_t u = load_id(g, r.off + i);
            const uint64_t x = bloom_key((uint32_t)v, u);
            uint32_t* blk = bloom + 8 * (uint64_t)bloom_block(x, blocks);
            for (int k = 0; k < 4; ++k) {
                const uint32_t bit = (uint32_t)(x >> (8 * k)) & 255u;
                atomicOr(blk + (bit >> 5), 1u << (bit & 31));
            }
        }
    }
}

// Fold of a filter with 2 * blocks blocks into one with `blocks`:
// bloom_block(x, 2B) >> 1 == bloom_block(x, B) (floor(floor(y) / 2) =
// floor(y / 2)) and the in-block bits do not depend on the block count, so
// OR-ing neighbouring blocks gives exactly the filter a direct build at B
// blocks sets.
__global__ void k_bloom_fold(const uint4* __restrict__ dense, uint4* __restrict__ out, uint64_t n16) {
    // n16 = 16-byte words of `out` (2 per block); dense block 2b | 2b+1 -> block b
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = i >> 1, h = i & 1;
        const uint4 x = dense[4 * b + h], y = dense[4 * b + 2 + h];
        out[i] = make_uint4(x.x | y.x, x.y | y.y, x.z | y.z, x.w | y.w);
    }
}

// {prob, alias} of every arc in one 16-byte entry (one load per proposal).
__global__ void k_pack_alias(const double* __restrict__ prob, const uint32_t* __restrict__ alias, uint64_t m,
                             uint4* __restrict__ out) {
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < m; a += (uint64_t)gridDim.x * blockDim.x) {
        const double p = prob[a];
        out[a] = make_uint4((uint32_t)__double2loint(p), (uint32_t)__double2hiint(p), alias[a], 0u);
    }
}

// Thread per node: alias_build (samplers.cpp:95-131) bit for bit. prob holds
// `scaled` in place; the small stack grows from the front of the node's
// scratch slice, the large stack from the back (ns + nl <= deg always).
__global__ void k_alias(DevGraph g, double* __restrict__ prob, uint32_t* __restrict__ alias,
                        uint32_t* __restrict__ scratch) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const NodeRec r = load_node(g, (uint32_t)v);
        const uint32_t n = r.deg;
        if (n == 0) continue;
        double* P = prob + r.off;
        uint32_t* A = alias + r.off;
        uint32_t* S = scratch + r.off;
        double total = 0.0;
        for (uint32_t i = 0; i < n; ++i) total = __dadd_rn(total, static_w(g, r.off + i));
        if (!(total > 0)) {
            for (uint32_t i = 0; i < n; ++i) {
                P[i] = 0.0;
                A[i] = i;
            }
            continue;
        }
        const double dn = (double)n;
        uint32_t ns = 0, nl = 0;
        for (uint32_t i = 0; i < n; ++i) {
            const double sc = __ddiv_rn(__dmul_rn(static_w(g, r.off + i), dn), total);
            P[i] = sc;
            A[i] = i;
            if (sc < 1.0) S[ns++] = i;
            else S[n - 1 - nl++] = i;
        }
        while (ns > 0 && nl > 0) {
            const uint32_t s = S[--ns];
            const uint32_t l = S[n - nl];  // large.back()
            A[s] = l;
            const double pl = __dsub_rn(P[l], __dsub_rn(1.0, P[s]));
            P[l] = pl;
            if (pl < 1.0) {
                --nl;
                S[ns++] = l;
            }
        }
        for (uint32_t i = 0; i < ns; ++i) P[S[i]] = 1.0;
        for (uint32_t j = 0; j < nl; ++j) P[S[n - 1 - j]] = 1.0;
    }
}

// Arcs sorted by (src,dst) key -> ids + offsets (gaps are isolated nodes).
__global__ void k_csr_from_keys(const uint64_t* __restrict__ keys, uint64_t m, uint32_t n,
                                int64_t* __restrict__ off, uint32_t* __restrict__ ids) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[i];
        const int64_t src = (int64_t)(key >> 32);
        ids[i] = (uint32_t)key;
        const int64_t prev = i == 0 ? -1 : (int64_t)(keys[i - 1] >> 32);
        for (int64_t v = prev + 1; v <= src; ++v) off[v] = (int64_t)i;
        if (i == m - 1)
            for (int64_t v = src + 1; v <= (int64_t)n; ++v) off[v] = (int64_t)m;
    }
}

__global__ void k_fill_offsets(int64_t* off, uint32_t n, int64_t value) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
         i += (uint64_t)gridDim.x * blockDim.x)
        off[i] = value;
}

// R-MAT edge e: `scale` 32-bit words from Philox block (e, l/4); quadrant by
// integer thresholds, MSB first. Self-loops -> ~0 (dropped by unique).
__global__ void k_rmat(uint64_t ne, uint32_t scale, uint2 key, uint64_t t1, uint64_t t2, uint64_t t3,
                       uint64_t* __restrict__ out) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0, d = 0;
        uint4 w = make_uint4(0, 0, 0, 0);
        for (uint32_t l = 0; l < scale; ++l) {
            if ((l & 3) == 0) w = philox10(make_uint4((uint32_t)e, (uint32_t)(e >> 32), l >> 2, 0u), key);
            const uint32_t r = (l & 3) == 0 ? w.x : (l & 3) == 1 ? w.y : (l & 3) == 2 ? w.z : w.w;
            uint32_t bs, bd;
            if ((uint64_t)r < t1) { bs = 0; bd = 0; }
            else if ((uint64_t)r < t2) { bs = 0; bd = 1; }
            else if ((uint64_t)r < t3) { bs = 1; bd = 0; }
            else { bs = 1; bd = 1; }
            s = (s << 1) | bs;
            d = (d << 1) | bd;
        }
        out[e] = s == d ? ~0ull : (((uint64_t)min(s, d) << 32) | max(s, d));
    }
}

// Undirected pair p -> arcs 2p (lo->hi) and 2p+1 (hi->lo).
__global__ void k_symmetrize_pairs(const uint64_t* __restrict__ pairs, uint64_t np,
                                   uint64_t* __restrict__ arcs) {
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < np;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = pairs[p];
        arcs[2 * p] = k;
        arcs[2 * p + 1] = (k << 32) | (k >> 32);
    }
}

__device__ __forceinline__ float pair_weight(uint64_t seed, uint32_t lo, uint32_t hi, float wlo, float whi) {
    const uint4 w = philox10(make_uint4(lo, hi, 0u, 0u), philox_key(seed, DOM_WEIGHT));
    const double u = unit53(w.x, w.y);
    return __double2float_rn(__dadd_rn((double)wlo, __dmul_rn(__dsub_rn((double)whi, (double)wlo), u)));
}

// Per-arc weight / edge type keyed by the undirected pair (same value both ways).
__global__ void k_pair_attrs(const uint64_t* __restrict__ keys, uint64_t m, uint64_t seed, float wlo,
                             float whi, float* __restrict__ w, uint32_t n_etypes,
                             uint16_t* __restrict__ et) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = (uint32_t)(keys[i] >> 32), b = (uint32_t)keys[i];
        const uint32_t lo = min(a, b), hi = max(a, b);
        if (w) w[i] = pair_weight(seed, lo, hi, wlo, whi);
        if (et) {
            Draw d;
            d.open(philox_key(seed, DOM_ETYPE), ((uint64_t)hi << 32) | lo, 0);
            et[i] = (uint16_t)d.index(n_etypes);
        }
    }
}

// Hetero generator, pass 1: Poisson(8) out-degree of each A node (Knuth
// product on Philox units of block (a, j)).
__global__ void k_hetero_counts(uint32_t nA, uint2 key, double L, uint32_t* __restrict__ cnt) {
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < nA;
         a += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = 0;
        double prod = 1.0;
        for (uint32_t j = 0;; ++j) {
            const uint4 w = philox10(make_uint4((uint32_t)a, 0u, j, 0u), key);
            prod = __dmul_rn(prod, unit53(w.y, w.z));
            if (prod <= L) break;
            ++c;
        }
        cnt[a] = c;
    }
}

__global__ void k_hetero_edges(uint32_t nA, uint32_t nP, uint32_t nV, uint2 key,
                               const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ pos,
                               uint64_t* __restrict__ out) {
    const uint64_t total = (uint64_t)nA + nP;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        if (t < nA) {
            const uint32_t a = (uint32_t)t;
            for (uint32_t j = 0; j < cnt[a]; ++j) {
                Draw d;
                d.open(key, ((uint64_t)1 << 40) | a, j);
                const uint32_t p = nA + d.index(nP);
                out[pos[a] + j] = ((uint64_t)a << 32) | p;
            }
        } else {
            const uint32_t p = (uint32_t)(t - nA);
            Draw d;
            d.open(key, ((uint64_t)2 << 40) | p, 0);
            const uint32_t v = nA + nP + d.index(nV);
            out[pos[nA] + p] = ((uint64_t)(nA + p) << 32) | v;
        }
    }
}

__global__ void k_hetero_types(uint32_t n, uint32_t nA, uint32_t nP, uint16_t* __restrict__ t) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        t[v] = v < nA ? 0 : (v < (uint64_t)nA + nP ? 1 : 2);
}

// from_edges: expanded arc list (edge i -> 2i forward, 2i+1 reverse).
__global__ void k_expand_edges(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                               uint64_t ne, int symmetrize, uint64_t* __restrict__ keys,
                               uint64_t* __restrict__ pos, unsigned* __restrict__ maxid) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = src[i], d = dst[i];
        const uint64_t stride = symmetrize ? 2 : 1;
        keys[stride * i] = ((uint64_t)s << 32) | d;
        pos[stride * i] = stride * i;
        if (symmetrize) {
            keys[2 * i + 1] = s == d ? ~0ull : (((uint64_t)d << 32) | s);
            pos[2 * i + 1] = 2 * i + 1;
        }
        atomicMax(maxid, max(s, d));
    }
}

__global__ void k_heads(const uint64_t* __restrict__ keys, uint64_t k, uint8_t* __restrict__ flag) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (uint64_t)gridDim.x * blockDim.x)
        flag[i] = keys[i] != ~0ull && (i == 0 || keys[i] != keys[i - 1]);
}

// Run sums in input order (duplicates collapse by summation, graph.cpp:44-52).
__global__ void k_run_sums(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ pos,
                           uint64_t k, const uint64_t* __restrict__ heads, uint64_t nh,
                           const float* __restrict__ win, int symmetrize, uint64_t* __restrict__ out_keys,
                           float* __restrict__ wout, unsigned* __restrict__ dup) {
    for (uint64_t h = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nh;
         h += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i0 = heads[h];
        const uint64_t key = keys[i0];
        double s = 0.0;
        uint64_t i = i0;
        for (; i < k && keys[i] == key; ++i) {
            const uint64_t src_edge = symmetrize ? pos[i] >> 1 : pos[i];
            s = __dadd_rn(s, win ? (double)win[src_edge] : 1.0);
        }
        if (i - i0 > 1) atomicAdd(dup, 1u);
        out_keys[h] = key;
        if (wout) wout[h] = __double2float_rn(s);
    }
}

__global__ void k_iota_u64(uint64_t* p, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = i;
}

__global__ void k_extract_offsets(const NodeRec* __restrict__ nodes, uint32_t n, uint64_t m,
                                  int64_t* __restrict__ off) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
         v += (uint64_t)gridDim.x * blockDim.x)
        off[v] = v < n ? nodes[v].off : (int64_t)m;
}

__global__ void k_set_types(NodeRec* __restrict__ nodes, const uint16_t* __restrict__ t, uint32_t n) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        nodes[v].type = t[v];
}

// ---------------------------------------------------------------- helpers
void sort_keys(DBuf<uint64_t>& keys, DBuf<uint64_t>& tmp, uint64_t n, int end_bit, cudaStream_t st) {
    size_t bytes = 0;
    MHW_CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.p, tmp.p, n, 0, end_bit, st));
    DBuf<uint8_t> temp(bytes);
    MHW_CK(cub::DeviceRadixSort::SortKeys(temp.p, bytes, keys.p, tmp.p, n, 0, end_bit, st));
    std::swap(keys, tmp);
}

// Sorted keys -> unique keys (drops ~0); returns count.
uint64_t unique_keys(DBuf<uint64_t>& keys, uint64_t n, DBuf<uint64_t>& out, cudaStream_t st) {
    DBuf<int64_t> d_count(1);
    size_t bytes = 0;
    MHW_CK(cub::DeviceSelect::Unique(nullptr, bytes, keys.p, out.p, d_count.p, (int64_t)n, st));
    DBuf<uint8_t> temp(bytes);
    MHW_CK(cub::DeviceSelect::Unique(temp.p, bytes, keys.p, out.p, d_count.p, (int64_t)n, st));
    int64_t cnt = 0;
    MHW_CK(cudaMemcpyAsync(&cnt, d_count.p, sizeof(cnt), cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    uint64_t last = 0;
    if (cnt > 0) {
        MHW_CK(cudaMemcpy(&last, out.p + cnt - 1, sizeof(last), cudaMemcpyDeviceToHost));
        if (last == ~0ull) --cnt;
    }
    return (uint64_t)cnt;
}

// Pairs (lo<<32|hi, deduplicated) -> symmetric CSR with optional attributes.
void csr_from_pairs(Graph& g, DBuf<uint64_t>& pairs, uint64_t np, uint32_t n, uint64_t seed,
                    bool weighted, float wlo, float whi, uint32_t n_etypes) {
    cudaStream_t st = g.stream;
    const uint64_t m = 2 * np;
    DBuf<uint64_t> arcs(std::max<uint64_t>(m, 1)), tmp(std::max<uint64_t>(m, 1));
    if (np) k_symmetrize_pairs<<<grid_for(np), kBlock, 0, st>>>(pairs.p, np, arcs.p);
    pairs.reset();
    if (m) sort_keys(arcs, tmp, m, 64, st);
    tmp.reset();
    DBuf<int64_t> off(n + 1);
    g.n = n;
    g.m = m;
    g.ids.alloc(std::max<uint64_t>(m, 1));
    g.ids.n = m;
    if (m) k_csr_from_keys<<<grid_for(m), kBlock, 0, st>>>(arcs.p, m, n, off.p, g.ids.p);
    else k_fill_offsets<<<grid_for(n + 1), kBlock, 0, st>>>(off.p, n, 0);
    if (weighted) g.w.alloc(m);
    if (n_etypes) {
        g.etype.alloc(m);
        g.n_etypes = (uint16_t)n_etypes;
    }
    if (m && (weighted || n_etypes))
        k_pair_attrs<<<grid_for(m), kBlock, 0, st>>>(arcs.p, m, seed, wlo, whi, weighted ? g.w.p : nullptr,
                                                     n_etypes, n_etypes ? g.etype.p : nullptr);
    MHW_CK(cudaGetLastError());
    arcs.reset();
    g.symmetric = true;
    graph_finalize(g, off.p, g.ntype.n ? g.ntype.p : nullptr);
}

}  // namespace

void graph_init_stream(Graph& g) {
    if (!g.stream) MHW_CK(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
}

// NodeRec build + validation from int64 offsets already on device.
void graph_finalize(Graph& g, const int64_t* d_off, const uint16_t* d_ntypes) {
    cudaStream_t st = g.stream;
    g.nodes.alloc(std::max<uint32_t>(g.n, 1));
    g.nodes.n = g.n;
    DBuf<unsigned> stats(3);
    MHW_CK(cudaMemsetAsync(stats.p, 0, 3 * sizeof(unsigned), st));
    if (g.n)
        k_nodes<<<grid_for((uint64_t)g.n * 32), kBlock, 0, st>>>(d_off, d_ntypes, g.ids.p,
                                                                 g.w.n ? g.w.p : nullptr, g.n, g.m,
                                                                 g.nodes.p, stats.p);
    MHW_CK(cudaGetLastError());
    unsigned h[3] = {0, 0, 0};
    int64_t ends[2] = {0, 0};
    MHW_CK(cudaMemcpyAsync(h, stats.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaMemcpyAsync(&ends[0], d_off, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaMemcpyAsync(&ends[1], d_off + g.n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    if (ends[0] != 0 || (uint64_t)ends[1] != g.m) invalid("offsets must start at 0 and end at arc_count");
    if (h[0] & ERR_OFFSETS) invalid("offsets are not non-decreasing");
    if (h[0] & ERR_DEGREE) invalid("degree exceeds the engine limit of 2^30 - 16");
    if (h[0] & ERR_RANGE) invalid("neighbor id out of range");
    if (h[0] & ERR_UNSORTED) invalid("neighbor slices must be strictly ascending");
    if (h[0] & ERR_NEGATIVE) invalid("negative edge weight");
    g.max_deg = h[1];
    g.isolated = h[2];
    g.rev.reset();
    g.wtotal.reset();
    g.wblk.reset();
    g.tcount.reset();
    g.tperm.reset();
    g.tbase.reset();
    g.htab.reset();
    g.arc.reset();
    g.bloom.reset();
    g.bloom_blocks = 0;
    g.bloom2.reset();
    g.bloom2_blocks = 0;
    g.verified_sym = false;
}

void graph_upload(Graph& g, const mhw_graph_view& v) {
    if (!v.offsets || (v.arc_count && !v.neighbors)) invalid("graph view is missing offsets or neighbors");
    graph_init_stream(g);
    cudaStream_t st = g.stream;
    g.n = v.node_count;
    g.m = v.arc_count;
    g.symmetric = v.symmetric != 0;
    DBuf<int64_t> off(g.n + 1);
    MHW_CK(cudaMemcpyAsync(off.p, v.offsets, (g.n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    g.ids.alloc(std::max<uint64_t>(g.m, 1));
    g.ids.n = g.m;
    if (g.m)
        MHW_CK(cudaMemcpyAsync(g.ids.p, v.neighbors, g.m * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    if (v.weights) {
        g.w.alloc(g.m);
        if (g.m) MHW_CK(cudaMemcpyAsync(g.w.p, v.weights, g.m * sizeof(float), cudaMemcpyHostToDevice, st));
    } else {
        g.w.reset();
    }
    if (v.node_types) {
        g.ntype.alloc(std::max<uint32_t>(g.n, 1));
        g.ntype.n = g.n;
        if (g.n)
            MHW_CK(cudaMemcpyAsync(g.ntype.p, v.node_types, g.n * sizeof(uint16_t), cudaMemcpyHostToDevice, st));
        g.n_ntypes = v.num_node_types;
        if (!g.n_ntypes) {
            uint16_t mx = 0;
            for (uint32_t i = 0; i < g.n; ++i) mx = std::max(mx, v.node_types[i]);
            g.n_ntypes = (uint16_t)(mx + 1);
        }
    } else {
        g.ntype.reset();
        g.n_ntypes = 0;
    }
    if (v.edge_types) {
        g.etype.alloc(std::max<uint64_t>(g.m, 1));
        g.etype.n = g.m;
        if (g.m)
            MHW_CK(cudaMemcpyAsync(g.etype.p, v.edge_types, g.m * sizeof(uint16_t), cudaMemcpyHostToDevice, st));
        g.n_etypes = v.num_edge_types;
        if (!g.n_etypes) {
            uint16_t mx = 0;
            for (uint64_t i = 0; i < g.m; ++i) mx = std::max(mx, v.edge_types[i]);
            g.n_etypes = (uint16_t)(mx + 1);
        }
    } else {
        g.etype.reset();
        g.n_etypes = 0;
    }
    graph_finalize(g, off.p, g.ntype.n ? g.ntype.p : nullptr);
}

void graph_from_edges(Graph& g, uint64_t ne, const uint32_t* src, const uint32_t* dst, const float* w,
                      bool symmetrize, uint32_t n_nodes) {
    graph_init_stream(g);
    cudaStream_t st = g.stream;
    const uint64_t k = symmetrize ? 2 * ne : ne;
    DBuf<uint32_t> dsrc(std::max<uint64_t>(ne, 1)), ddst(std::max<uint64_t>(ne, 1));
    DBuf<float> dw(w ? std::max<uint64_t>(ne, 1) : 0);
    if (ne) {
        MHW_CK(cudaMemcpyAsync(dsrc.p, src, ne * 4, cudaMemcpyHostToDevice, st));
        MHW_CK(cudaMemcpyAsync(ddst.p, dst, ne * 4, cudaMemcpyHostToDevice, st));
        if (w) MHW_CK(cudaMemcpyAsync(dw.p, w, ne * 4, cudaMemcpyHostToDevice, st));
    }
    DBuf<uint64_t> keys(std::max<uint64_t>(k, 1)), pos(std::max<uint64_t>(k, 1));
    DBuf<unsigned> maxid(1);
    MHW_CK(cudaMemsetAsync(maxid.p, 0, sizeof(unsigned), st));
    if (ne) k_expand_edges<<<grid_for(ne), kBlock, 0, st>>>(dsrc.p, ddst.p, ne, symmetrize, keys.p, pos.p, maxid.p);
    MHW_CK(cudaGetLastError());
    unsigned mx = 0;
    MHW_CK(cudaMemcpyAsync(&mx, maxid.p, sizeof(mx), cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    uint32_t n = ne ? mx + 1 : 0;
    if (n_nodes > n) n = n_nodes;
    // stable sort by key keeps input order inside duplicate runs
    DBuf<uint64_t> k2(std::max<uint64_t>(k, 1)), p2(std::max<uint64_t>(k, 1));
    if (k) {
        size_t bytes = 0;
        MHW_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, k2.p, pos.p, p2.p, k, 0, 64, st));
        DBuf<uint8_t> temp(bytes);
        MHW_CK(cub::DeviceRadixSort::SortPairs(temp.p, bytes, keys.p, k2.p, pos.p, p2.p, k, 0, 64, st));
    }
    keys.reset();
    pos.reset();
    DBuf<uint8_t> flag(std::max<uint64_t>(k, 1));
    if (k) k_heads<<<grid_for(k), kBlock, 0, st>>>(k2.p, k, flag.p);
    DBuf<uint64_t> idx(std::max<uint64_t>(k, 1)), heads(std::max<uint64_t>(k, 1));
    DBuf<int64_t> d_nh(1);
    int64_t nh = 0;
    if (k) {
        k_iota_u64<<<grid_for(k), kBlock, 0, st>>>(idx.p, k);
        size_t bytes = 0;
        MHW_CK(cub::DeviceSelect::Flagged(nullptr, bytes, idx.p, flag.p, heads.p, d_nh.p, (int64_t)k, st));
        DBuf<uint8_t> temp(bytes);
        MHW_CK(cub::DeviceSelect::Flagged(temp.p, bytes, idx.p, flag.p, heads.p, d_nh.p, (int64_t)k, st));
        MHW_CK(cudaMemcpyAsync(&nh, d_nh.p, sizeof(nh), cudaMemcpyDeviceToHost, st));
        MHW_CK(cudaStreamSynchronize(st));
    }
    const uint64_t m = (uint64_t)nh;
    DBuf<uint64_t> arcs(std::max<uint64_t>(m, 1));
    DBuf<float> wsum(std::max<uint64_t>(m, 1));
    DBuf<unsigned> dup(1);
    MHW_CK(cudaMemsetAsync(dup.p, 0, sizeof(unsigned), st));
    if (m)
        k_run_sums<<<grid_for(m), kBlock, 0, st>>>(k2.p, p2.p, k, heads.p, m, w ? dw.p : nullptr, symmetrize,
                                                   arcs.p, wsum.p, dup.p);
    MHW_CK(cudaGetLastError());
    unsigned ndup = 0;
    MHW_CK(cudaMemcpyAsync(&ndup, dup.p, sizeof(ndup), cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    k2.reset();
    p2.reset();
    g.n = n;
    g.m = m;
    g.symmetric = symmetrize;
    g.ids.alloc(std::max<uint64_t>(m, 1));
    g.ids.n = m;
    DBuf<int64_t> off(n + 1);
    if (m) k_csr_from_keys<<<grid_for(m), kBlock, 0, st>>>(arcs.p, m, n, off.p, g.ids.p);
    else k_fill_offsets<<<grid_for(n + 1), kBlock, 0, st>>>(off.p, n, 0);
    if (w || ndup) {
        g.w = std::move(wsum);
        g.w.n = m;
    } else {
        g.w.reset();
    }
    g.ntype.reset();
    g.etype.reset();
    g.n_ntypes = g.n_etypes = 0;
    MHW_CK(cudaGetLastError());
    graph_finalize(g, off.p, nullptr);
}

void graph_generate_rmat(Graph& g, uint32_t scale, uint32_t ef, double a, double b, double c,
                         uint64_t seed, bool weighted, float wlo, float whi, uint32_t n_etypes) {
    if (scale == 0 || scale > 31) invalid("rmat scale must be in [1, 31]");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) invalid("rmat probabilities must be a valid distribution");
    graph_init_stream(g);
    cudaStream_t st = g.stream;
    const uint64_t ne = (uint64_t)ef << scale;
    // same integer thresholds as oracle/mhw_oracle.c og_rmat_pairs
    const uint64_t t1 = (uint64_t)(a * 4294967296.0);
    const uint64_t t2 = (uint64_t)((a + b) * 4294967296.0);
    const uint64_t t3 = (uint64_t)((a + b + c) * 4294967296.0);
    DBuf<uint64_t> keys(std::max<uint64_t>(ne, 1)), tmp(std::max<uint64_t>(ne, 1));
    if (ne) k_rmat<<<grid_for(ne), kBlock, 0, st>>>(ne, scale, philox_key(seed, DOM_RMAT), t1, t2, t3, keys.p);
    MHW_CK(cudaGetLastError());
    if (ne) sort_keys(keys, tmp, ne, 64, st);
    const uint64_t np = ne ? unique_keys(keys, ne, tmp, st) : 0;
    keys.reset();
    g.ntype.reset();
    g.n_ntypes = 0;
    g.etype.reset();
    g.n_etypes = 0;
    csr_from_pairs(g, tmp, np, 1u << scale, seed, weighted, wlo, whi, n_etypes);
}

void graph_generate_hetero(Graph& g, uint32_t n_nodes, uint64_t seed, float wlo, float whi) {
    if (n_nodes < 3) invalid("hetero generator needs at least 3 nodes");
    graph_init_stream(g);
    cudaStream_t st = g.stream;
    const uint32_t nA = (uint32_t)((uint64_t)n_nodes * 60 / 100);
    const uint32_t nP = (uint32_t)((uint64_t)n_nodes * 35 / 100);
    const uint32_t nV = n_nodes - nA - nP;
    if (!nA || !nP || !nV) invalid("hetero generator needs all three node types");
    const double L = 0x1.5fc21041027adp-12;  // exp(-8)
    const uint2 key = philox_key(seed, DOM_HETERO);
    DBuf<uint32_t> cnt(nA + 1);
    MHW_CK(cudaMemsetAsync(cnt.p, 0, (nA + 1) * sizeof(uint32_t), st));
    k_hetero_counts<<<grid_for(nA), kBlock, 0, st>>>(nA, key, L, cnt.p);
    DBuf<uint64_t> pos(nA + 1);
    {
        size_t bytes = 0;
        MHW_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, pos.p, (int64_t)nA + 1, st));
        DBuf<uint8_t> temp(bytes);
        MHW_CK(cub::DeviceScan::ExclusiveSum(temp.p, bytes, cnt.p, pos.p, (int64_t)nA + 1, st));
    }
    uint64_t na_edges = 0;
    MHW_CK(cudaMemcpyAsync(&na_edges, pos.p + nA, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    const uint64_t ne = na_edges + nP;
    DBuf<uint64_t> keys(ne), tmp(ne);
    k_hetero_edges<<<grid_for((uint64_t)nA + nP), kBlock, 0, st>>>(nA, nP, nV, key, cnt.p, pos.p, keys.p);
    MHW_CK(cudaGetLastError());
    sort_keys(keys, tmp, ne, 64, st);
    const uint64_t np = unique_keys(keys, ne, tmp, st);
    keys.reset();
    g.ntype.alloc(n_nodes);
    g.n_ntypes = 3;
    k_hetero_types<<<grid_for(n_nodes), kBlock, 0, st>>>(n_nodes, nA, nP, g.ntype.p);
    g.etype.reset();
    g.n_etypes = 0;
    csr_from_pairs(g, tmp, np, n_nodes, seed, true, wlo, whi, 0);
}

void graph_set_node_types(Graph& g, const uint16_t* types, uint16_t num_types) {
    DeviceGuard dg(g.device);
    uint16_t mx = 0;
    for (uint32_t i = 0; i < g.n; ++i) mx = std::max(mx, types[i]);
    if (num_types == 0) num_types = (uint16_t)(mx + 1);
    if (g.n && mx >= num_types) invalid("node type id exceeds num_types");
    g.ntype.alloc(std::max<uint32_t>(g.n, 1));
    g.ntype.n = g.n;
    if (g.n) {
        MHW_CK(cudaMemcpyAsync(g.ntype.p, types, g.n * sizeof(uint16_t), cudaMemcpyHostToDevice, g.stream));
        k_set_types<<<grid_for(g.n), kBlock, 0, g.stream>>>(g.nodes.p, g.ntype.p, g.n);
    }
    MHW_CK(cudaGetLastError());
    MHW_CK(cudaStreamSynchronize(g.stream));
    g.n_ntypes = num_types;
    g.tcount.reset();
    g.tperm.reset();
    g.tbase.reset();
}

void graph_set_edge_types(Graph& g, const uint16_t* types, uint16_t num_types) {
    DeviceGuard dg(g.device);
    uint16_t mx = 0;
    for (uint64_t i = 0; i < g.m; ++i) mx = std::max(mx, types[i]);
    if (num_types == 0) num_types = (uint16_t)(mx + 1);
    if (g.m && mx >= num_types) invalid("edge type id exceeds num_types");
    g.etype.alloc(std::max<uint64_t>(g.m, 1));
    g.etype.n = g.m;
    if (g.m) MHW_CK(cudaMemcpyAsync(g.etype.p, types, g.m * sizeof(uint16_t), cudaMemcpyHostToDevice, g.stream));
    MHW_CK(cudaStreamSynchronize(g.stream));
    g.n_etypes = num_types;
}

template <class T>
static void copy_buf(const DBuf<T>& src, int src_dev, DBuf<T>& dst, int dst_dev, cudaStream_t st) {
    dst.alloc(src.n);
    if (src.n) MHW_CK(cudaMemcpyPeerAsync(dst.p, dst_dev, src.p, src_dev, src.bytes(), st));
}

void graph_replicate(const Graph& s, Graph& d, int device) {
    d.device = device;
    graph_init_stream(d);
    copy_buf(s.nodes, s.device, d.nodes, device, d.stream);
    copy_buf(s.ids, s.device, d.ids, device, d.stream);
    copy_buf(s.w, s.device, d.w, device, d.stream);
    copy_buf(s.ntype, s.device, d.ntype, device, d.stream);
    copy_buf(s.etype, s.device, d.etype, device, d.stream);
    copy_buf(s.rev, s.device, d.rev, device, d.stream);
    copy_buf(s.wtotal, s.device, d.wtotal, device, d.stream);
    copy_buf(s.wblk, s.device, d.wblk, device, d.stream);
    copy_buf(s.tcount, s.device, d.tcount, device, d.stream);
    copy_buf(s.tperm, s.device, d.tperm, device, d.stream);
    copy_buf(s.tbase, s.device, d.tbase, device, d.stream);
    copy_buf(s.htab, s.device, d.htab, device, d.stream);
    copy_buf(s.arc, s.device, d.arc, device, d.stream);
    MHW_CK(cudaStreamSynchronize(d.stream));
    d.n = s.n;
    d.m = s.m;
    d.n_ntypes = s.n_ntypes;
    d.n_etypes = s.n_etypes;
    d.symmetric = s.symmetric;
    d.verified_sym = s.verified_sym;
    d.max_deg = s.max_deg;
    d.isolated = s.isolated;
}

void graph_download(const Graph& g, int64_t* offsets, int32_t* nbr, float* w, uint16_t* ntypes,
                    uint16_t* etypes) {
    DeviceGuard dg(g.device);
    cudaStream_t st = g.stream;
    if (offsets) {
        DBuf<int64_t> off(g.n + 1);
        k_extract_offsets<<<grid_for(g.n + 1), kBlock, 0, st>>>(g.nodes.p, g.n, g.m, off.p);
        MHW_CK(cudaGetLastError());
        MHW_CK(cudaMemcpyAsync(offsets, off.p, (g.n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        MHW_CK(cudaStreamSynchronize(st));
    }
    if (nbr && g.m) MHW_CK(cudaMemcpyAsync(nbr, g.ids.p, g.m * 4, cudaMemcpyDeviceToHost, st));
    if (w && g.m) {
        if (g.w.n) MHW_CK(cudaMemcpyAsync(w, g.w.p, g.m * 4, cudaMemcpyDeviceToHost, st));
        else {
            MHW_CK(cudaStreamSynchronize(st));
            for (uint64_t i = 0; i < g.m; ++i) w[i] = 1.0f;
        }
    }
    if (ntypes && g.n && g.ntype.n) MHW_CK(cudaMemcpyAsync(ntypes, g.ntype.p, g.n * 2, cudaMemcpyDeviceToHost, st));
    if (etypes && g.m && g.etype.n) MHW_CK(cudaMemcpyAsync(etypes, g.etype.p, g.m * 2, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
}

void graph_ensure_rev(Graph& g) {
    if (g.rev.n || !g.m) return;
    DeviceGuard dg(g.device);
    cudaStream_t st = g.stream;
    g.rev.alloc(g.m);
    DevGraph v = g.view();
    int bits = 1;
    while (bits < 32 && ((uint64_t)g.n >> bits) != 0) ++bits;
    unsigned h = 1;
    {
        // one radix sort of (dst, src) keys; valid when the CSR is symmetric
        DBuf<uint32_t> k1(g.m), k2(g.m);
        DBuf<uint64_t> v1(g.m), v2(g.m);
        DBuf<unsigned> mismatch(1);
        MHW_CK(cudaMemsetAsync(mismatch.p, 0, sizeof(unsigned), st));
        k_rev_keys<<<grid_for((uint64_t)g.n * 32), kBlock, 0, st>>>(v, k1.p, v1.p);
        size_t bytes = 0;
        MHW_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k1.p, k2.p, v1.p, v2.p, (int64_t)g.m, 0, bits, st));
        DBuf<uint8_t> temp(std::max<size_t>(bytes, 1));
        MHW_CK(cub::DeviceRadixSort::SortPairs(temp.p, bytes, k1.p, k2.p, v1.p, v2.p, (int64_t)g.m, 0, bits, st));
        k_rev_scatter<<<grid_for(g.m), kBlock, 0, st>>>(v, k2.p, v2.p, g.rev.p, mismatch.p);
        MHW_CK(cudaGetLastError());
        MHW_CK(cudaMemcpyAsync(&h, mismatch.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        MHW_CK(cudaStreamSynchronize(st));
    }
    if (h != 0) {
        // not symmetric: per-arc search, missing back arcs become kNoBack
        DBuf<unsigned> missing(1);
        MHW_CK(cudaMemsetAsync(missing.p, 0, sizeof(unsigned), st));
        k_rev<<<grid_for((uint64_t)g.n * 32), kBlock, 0, st>>>(v, g.rev.p, missing.p);
        MHW_CK(cudaGetLastError());
        MHW_CK(cudaMemcpyAsync(&h, missing.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        MHW_CK(cudaStreamSynchronize(st));
    }
    g.verified_sym = h == 0;
}

// st: the stream to build on (nullptr: the graph's); sync = wait for it.
void graph_ensure_hash(Graph& g, cudaStream_t st, bool sync) {
    if (g.htab.n || !g.m || g.max_deg < kHashMinDeg) return;
    DeviceGuard dg(g.device);
    if (!st) st = g.stream;
    const uint64_t buckets = (g.m >> 2) + g.n + 1;
    g.htab.alloc(8 * buckets);
    MHW_CK(cudaMemsetAsync(g.htab.p, 0xFF, g.htab.bytes(), st));
    k_hash_build<<<grid_for(g.m), kBlock, 0, st>>>(g.view(), g.htab.p);
    MHW_CK(cudaGetLastError());
    if (sync) MHW_CK(cudaStreamSynchronize(st));
}

// Edge Bloom filter for the alpha test. Small graphs: the densest of 4 / 3 /
// 2 bits per arc (4 bits: 8 per undirected edge, ~2.4% false positives) that
// fits 32 MB and so lives in L2 (measured on cfg2: 4 bits/arc 41.2 ms, 8 bits
// 43.2, 16 bits 46.5, none 48.8 -- residency beats a lower false-positive
// rate; cfg4: 2 bits (32 MB) 174.9 ms, 4 bits (64 MB) 176.7, none 189.8).
// Larger graphs: the filter is DRAM-resident anyway,
// and one sector probe still settles most non-adjacent pairs ahead of a hash
// probe or slice search, so it is built at 8 bits per arc when it takes at
// most 1/8 of free device memory (cfg5, 2.08 G arcs: 1185 ms without, 1111
// at 4 bits, 1099 at 8). MHW_BLOOM_MB / MHW_BLOOM_BITS override the budget
// and density; MHW_BLOOM=0 disables it.
void graph_ensure_bloom(Graph& g, cudaStream_t st, bool sync, uint32_t max_bits) {
    if (g.bloom.n || !g.m) return;
    if (!st) st = g.stream;
    const char* off = std::getenv("MHW_BLOOM");
    if (off && off[0] == '0') return;
    const char* mb = std::getenv("MHW_BLOOM_MB");
    const char* bits = std::getenv("MHW_BLOOM_BITS");
    uint64_t bytes = g.m * (uint64_t)(bits ? std::atoi(bits) : 4) / 8;  // bits per arc
    if (mb) {
        if (bytes > ((uint64_t)std::atoll(mb) << 20)) return;
    } else if (!bits) {
        // densest of 4 / 3 / 2 bits per arc within 32 MB (L2-resident),
        // else 8 bits per arc in DRAM
        for (uint64_t b = max_bits; b >= 2 && (bytes = g.m * b / 8) > (32ull << 20); --b) {
        }
        if (bytes > (32ull << 20)) bytes = g.m;
        if (bytes > dev_available_bytes() / 8) return;
    } else if (bytes > dev_available_bytes() / 8) {
        return;
    }
    if (bytes < 32) return;
    const uint64_t blocks = (bytes + 31) / 32;
    if (blocks >= (1ull << 32)) return;
    DeviceGuard dg(g.device);
    g.bloom.alloc(8 * blocks);
    g.bloom_blocks = (uint32_t)blocks;
    // compact-chain graphs (3 bits per arc asked for): the eager init probes
    // a filter of twice the density (session_create), so that one is built
    // and the walk's filter is its fold -- one scatter pass instead of two
    // (e2e session setup: k_bloom_build is 2.2 ms of cfg2's)
    const bool dense_too = max_bits == 3 && !mb && !bits && 2 * blocks < (1ull << 32) && 64 * blocks <= (33ull << 20) &&
                           !std::getenv("MHW_INIT_BLOOM_BITS");
    if (dense_too) {
        g.bloom2.alloc(16 * blocks);
        g.bloom2_blocks = (uint32_t)(2 * blocks);
        MHW_CK(cudaMemsetAsync(g.bloom2.p, 0, g.bloom2.bytes(), st));
        k_bloom_build<<<grid_for(g.n * 32ull), kBlock, 0, st>>>(g.view(), g.bloom2.p, g.bloom2_blocks);
        k_bloom_fold<<<grid_for(2 * blocks), kBlock, 0, st>>>(reinterpret_cast<const uint4*>(g.bloom2.p),
                                                             reinterpret_cast<uint4*>(g.bloom.p), 2 * blocks);
    } else {
        MHW_CK(cudaMemsetAsync(g.bloom.p, 0, g.bloom.bytes(), st));
        k_bloom_build<<<grid_for(g.n * 32ull), kBlock, 0, st>>>(g.view(), g.bloom.p, g.bloom_blocks);
    }
    MHW_CK(cudaGetLastError());
    if (sync) MHW_CK(cudaStreamSynchronize(st));
}

// A second edge filter over the same keys at `bits` bits per arc (the
// compact-chain sessions' eager init probes a denser filter than their walk).
void graph_build_bloom(const Graph& g, uint32_t bits, DBuf<uint32_t>& out, uint32_t* blocks, cudaStream_t st) {
    DeviceGuard dg(g.device);
    const uint64_t nb = (g.m * bits / 8 + 31) / 32;
    if (!g.m || nb == 0 || nb >= (1ull << 32)) {
        *blocks = 0;
        return;
    }
    out.alloc(8 * nb);
    *blocks = (uint32_t)nb;
    MHW_CK(cudaMemsetAsync(out.p, 0, out.bytes(), st));
    k_bloom_build<<<grid_for(g.n * 32ull), kBlock, 0, st>>>(g.view(), out.p, *blocks);
    MHW_CK(cudaGetLastError());
}

// The alpha-test structures of a second-order model built concurrently: the
// hash sets and the edge filter on two side streams while the reverse index
// (a radix sort) runs on the graph's stream (e2e session setup: each is a
// few scatter-bound kernels).
void graph_ensure_second_order(Graph& g, bool alpha, uint32_t bloom_bits) {
    DeviceGuard dg(g.device);
    cudaStream_t s1 = nullptr, s2 = nullptr;
    const bool side = alpha && g.m && (!g.htab.n || !g.bloom.n);
    if (side) {
        MHW_CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
        MHW_CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    }
    try {
        if (side) {
            graph_ensure_hash(g, s1, false);
            graph_ensure_bloom(g, s2, false, bloom_bits);
        }
        graph_ensure_rev(g);
        graph_ensure_wtotal(g);
        if (side) {
            MHW_CK(cudaStreamSynchronize(s1));
            MHW_CK(cudaStreamSynchronize(s2));
        }
    } catch (...) {
        if (s1) cudaStreamDestroy(s1);
        if (s2) cudaStreamDestroy(s2);
        throw;
    }
    if (s1) cudaStreamDestroy(s1);
    if (s2) cudaStreamDestroy(s2);
}

bool graph_ensure_arcrec(Graph& g) {
    if (g.arc.n) return true;
    if (!g.m || g.m >= (1ull << 32)) return false;
    DeviceGuard dg(g.device);
    if (dev_available_bytes() < 16 * g.m + (2ull << 30)) return false;  // keep headroom; the walk works without
    g.arc.alloc(g.m);
    k_arcrec<<<grid_for(g.m), kBlock, 0, g.stream>>>(g.view(), g.arc.p);
    MHW_CK(cudaGetLastError());
    MHW_CK(cudaStreamSynchronize(g.stream));
    return true;
}

void graph_ensure_wtotal(Graph& g) {
    if (g.wtotal.n || !g.w.n || !g.n) return;
    DeviceGuard dg(g.device);
    g.wtotal.alloc(g.n);
    k_wtotal<<<grid_for(g.n, 64), 64, 0, g.stream>>>(g.view(), g.wtotal.p);
    MHW_CK(cudaGetLastError());
    if (g.max_deg >= kBootBlkMin) {
        g.wblk.alloc((g.m >> 5) + g.n + 1);
        k_wblk<<<grid_for((uint64_t)g.n * 32), 256, 0, g.stream>>>(g.view(), g.wblk.p);
        MHW_CK(cudaGetLastError());
    }
    MHW_CK(cudaStreamSynchronize(g.stream));
}

void graph_ensure_static_alias(Graph& g) {
    if (g.sal.n || !g.w.n || !g.m) return;
    DeviceGuard dg(g.device);
    DBuf<double> prob(g.m);
    DBuf<uint32_t> alias(g.m);
    graph_alias_device(g, prob.p, alias.p);
    g.sal.alloc(g.m);
    k_pack_alias<<<grid_for(g.m), kBlock, 0, g.stream>>>(prob.p, alias.p, g.m, g.sal.p);
    MHW_CK(cudaGetLastError());
    MHW_CK(cudaStreamSynchronize(g.stream));
}

void graph_ensure_tcount(Graph& g) {
    if (g.tcount.n || !g.n || !g.n_ntypes) return;
    DeviceGuard dg(g.device);
    g.tcount.alloc((size_t)g.n * g.n_ntypes);
    MHW_CK(cudaMemsetAsync(g.tcount.p, 0, g.tcount.bytes(), g.stream));
    k_tcount<<<grid_for((uint64_t)g.n * 32), kBlock, 0, g.stream>>>(g.view(), g.tcount.p);
    MHW_CK(cudaGetLastError());
    MHW_CK(cudaStreamSynchronize(g.stream));
}

void graph_ensure_typed_index(Graph& g) {
    if (g.tbase.n || !g.n || !g.m || !g.n_ntypes || g.n_ntypes > 64) return;
    DeviceGuard dg(g.device);
    const uint64_t K = 2ull * g.n_ntypes;
    // index + bases + build counters; optional (inits fall back to the scan)
    const uint64_t need = 4 * g.m + 8ull * g.n * g.n_ntypes + 4 * g.n * K;
    if (need > dev_available_bytes() / 4) return;
    DBuf<uint32_t> cnt(g.n * K);
    MHW_CK(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), g.stream));
    g.tperm.alloc(g.m);
    g.tbase.alloc((size_t)g.n * g.n_ntypes);
    k_tidx_count<<<grid_for((uint64_t)g.n * 32), kBlock, 0, g.stream>>>(g.view(), cnt.p);
    k_tidx_base<<<grid_for(g.n), kBlock, 0, g.stream>>>(g.view(), cnt.p, g.tbase.p);
    k_tidx_scatter<<<grid_for((uint64_t)g.n * 32), kBlock, 0, g.stream>>>(g.view(), cnt.p, g.tperm.p);
    MHW_CK(cudaGetLastError());
    MHW_CK(cudaStreamSynchronize(g.stream));
}

void graph_alias_device(Graph& g, double* prob, uint32_t* alias) {
    DeviceGuard dg(g.device);
    if (!g.m) return;
    DBuf<uint32_t> scratch(g.m);
    k_alias<<<grid_for(g.n, 64), 64, 0, g.stream>>>(g.view(), prob, alias, scratch.p);
    MHW_CK(cudaGetLastError());
    MHW_CK(cudaStreamSynchronize(g.stream));
}

void graph_alias_tables(Graph& g, double* prob, uint32_t* alias) {
    DeviceGuard dg(g.device);
    if (!g.m) return;
    DBuf<double> dp(g.m);
    DBuf<uint32_t> da(g.m), scratch(g.m);
    k_alias<<<grid_for(g.n, 64), 64, 0, g.stream>>>(g.view(), dp.p, da.p, scratch.p);
    MHW_CK(cudaGetLastError());
    MHW_CK(cudaMemcpyAsync(prob, dp.p, g.m * sizeof(double), cudaMemcpyDeviceToHost, g.stream));
    MHW_CK(cudaMemcpyAsync(alias, da.p, g.m * sizeof(uint32_t), cudaMemcpyDeviceToHost, g.stream));
    MHW_CK(cudaStreamSynchronize(g.stream));
}

}  // namespace mhw
