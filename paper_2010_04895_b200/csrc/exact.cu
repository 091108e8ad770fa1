// exact.cu -- the exact baseline samplers of WalkerContext::next_edge
// (engine.cpp:88-116) on the GPU: one warp per walker, the O(deg) dynamic
// weights evaluated 32 candidates at a time, the reference's sequential
// fp64 sums (std::accumulate / `r -= w[i]` order) replayed lane by lane
// through warp shuffles, so every draw is bit-identical to the oracle's
// Philox layout (oracle/mhw_oracle.c baseline_step):
//   direct    : unit of the walk block (walker, step)      -- samplers.cpp:133-146
//   alias     : index + unit of the walk block, per-state tables built on
//               first visit by the visiting warp            -- samplers.cpp:95-131
//   rejection : trial t = block (walker, step) under key DOM_REJECT + (t >> 16)
//               (a fresh key every 65536 trials, so the streams never wrap),
//               sub-counter (t & 0xFFFF) << 16 (proposal index + unit), sub
//               ((t & 0xFFFF) << 16) | 0x8000 (accept unit);
//               32 trials evaluated per warp round, the first accepted wins
//                                                           -- samplers.cpp:148-170
// They are comparison baselines (tools/mhwalk.cpp:298-429), not the product.
#include <cub/cub.cuh>

#include <algorithm>
#include <string>

#include "exact.h"

namespace mhw {

namespace {

constexpr int kExBlock = 256;
constexpr uint32_t kExWarps = kExBlock / 32;
constexpr uint32_t kCache = 256;  // dynamic weights cached per warp (direct)
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t DOM_REJECT = 0x2E1EC705u;
enum : uint32_t { AS_EMPTY = 0, AS_BUILDING = 1, AS_READY = 2, AS_DEAD = 3 };

struct ExParams {
    double bound;
    uint32_t* astat;
    double* aprob;
    uint32_t* aalias;
    const uint64_t* qoff;
    uint32_t* scratch;
    uint64_t scratch_per_warp;
    const double* sprob;
    const uint32_t* salias;
};

// std::accumulate of f(0..n-1) in index order (fp64), the 32 values of a
// round reduced sequentially through shuffles (warp-uniform result). Also
// the last index with f > 0 (direct_sample's fallback) and optional copies
// of the values (shared cache / global table).
template <class F>
__device__ __forceinline__ double warp_total(const F& f, uint32_t n, uint32_t lane, double* cache, double* gout,
                                             uint32_t* lastpos) {
    double total = 0.0;
    uint32_t lp = 0;
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t i = base + lane;
        const double x = i < n ? f(i) : 0.0;
        if (i < n) {
            if (cache) cache[i] = x;
            if (gout) gout[i] = x;
        }
        const unsigned pos = __ballot_sync(kFull, i < n && x > 0);
        if (pos) lp = base + 31 - __clz(pos);
        const uint32_t cnt = n - base < 32 ? n - base : 32;
        for (uint32_t j = 0; j < cnt; ++j) total = __dadd_rn(total, __shfl_sync(kFull, x, j));
    }
    *lastpos = lp;
    return total;
}

// direct_sample's scan (samplers.cpp:138-145) with r = u * total given.
template <class F>
__device__ __forceinline__ uint32_t warp_scan(const F& f, uint32_t n, uint32_t lane, const double* cache, double r,
                                              uint32_t lastpos) {
    __syncwarp();
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t i = base + lane;
        const double x = i < n ? (cache ? cache[i] : f(i)) : 0.0;
        const uint32_t cnt = n - base < 32 ? n - base : 32;
        for (uint32_t j = 0; j < cnt; ++j) {
            r = __dsub_rn(r, __shfl_sync(kFull, x, j));
            if (r < 0) return base + j;
        }
    }
    return lastpos;
}

// alias_build's pairing (samplers.cpp:108-129) by one lane: P holds the
// scaled weights in place, S is the stack scratch (small from the front,
// large from the back).
__device__ void alias_pairs(double* P, uint32_t* A, uint32_t* S, uint32_t n) {
    uint32_t ns = 0, nl = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (P[i] < 1.0) S[ns++] = i;
        else S[n - 1 - nl++] = i;
    }
    while (ns > 0 && nl > 0) {
        const uint32_t s = S[--ns];
        const uint32_t l = S[n - nl];
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

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int KIND, int SMP>
__global__ void __launch_bounds__(kExBlock) k_walk_exact(RunParams P, ExParams X) {
    __shared__ double cache_all[kExWarps][kCache];
    const DevGraph& g = P.g;
    const DevModel& M = P.m;
    const unsigned lane = threadIdx.x & 31;
    double* cache = cache_all[threadIdx.x >> 5];
    const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t* scr = X.scratch ? X.scratch + gwarp * X.scratch_per_warp : nullptr;
    const uint2 wkey = philox_key(P.cfg.seed, DOM_WALK);
    const uint2 rkey = philox_key(P.cfg.seed, DOM_REJECT);
    const uint32_t K = P.cfg.K, L = P.cfg.L;
    unsigned long long steps = 0, early = 0, trials = 0;
    for (;;) {
        unsigned long long item = 0;
        if (lane == 0) item = atomicAdd(&P.ctr[0], 1ull);
        item = __shfl_sync(kFull, item, 0);
        if (item >= P.n_items) break;
        const uint32_t k = (uint32_t)(item / P.n_act);
        const uint32_t j = (uint32_t)(item - (uint64_t)k * P.n_act);
        const uint32_t v0 = __ldg(P.act + j);
        const uint64_t row = __ldg(P.act_row + j) + k;
        const uint64_t walker = (uint64_t)v0 * K + k;
        uint32_t* orow = P.out + row * P.stride;
        if (lane == 0) orow[0] = v0;

        const NodeRec r0 = load_node(g, v0);
        SCtx c;
        c.v = v0;
        c.off = r0.off;
        c.deg = r0.deg;
        c.vtype = r0.type;
        c.vflags = r0.flags;
        c.s = 0;
        c.off_s = 0;
        c.deg_s = 0;
        c.in_type = 0;
        c.req = 0;
        c.boot = second_order(KIND);
        uint32_t affix = second_order(KIND) ? kNoAffix : 0u;
        if (KIND == METAPATH2VEC) c.req = M.metapath[metapath_next(M, 0)];
        uint32_t len = 1;
        bool dead = false;
        for (uint32_t step = 0; step < L; ++step) {
            if (c.deg == 0) {
                dead = true;
                break;
            }
            Draw d;
            d.open(wkey, walker, step);
            uint32_t chosen = 0;
            auto fw = [&](uint32_t i) {
                uint32_t cls;
                return eval_index<KIND>(g, M, c, i, &cls);
            };
            if (second_order(KIND) && c.boot) {
                // draw_static (engine.cpp:81-83, :130-134)
                if (!g.w) {
                    uint32_t i = (uint32_t)__dmul_rn(d.unit(), (double)c.deg);
                    chosen = i < c.deg ? i : c.deg - 1;
                } else {
                    auto fs = [&](uint32_t i) { return static_w(g, c.off + i); };
                    uint32_t lp;
                    const double tot = warp_total(fs, c.deg, lane, nullptr, nullptr, &lp);
                    if (!(tot > 0)) {
                        dead = true;
                        break;
                    }
                    chosen = warp_scan(fs, c.deg, lane, nullptr, __dmul_rn(d.unit(), tot), lp);
                }
            } else if (SMP == MHW_SAMPLER_DIRECT) {
                double* cc = c.deg <= kCache ? cache : nullptr;
                uint32_t lp;
                const double tot = warp_total(fw, c.deg, lane, cc, nullptr, &lp);
                if (!(tot > 0)) {
                    dead = true;
                    break;
                }
                chosen = warp_scan(fw, c.deg, lane, cc, __dmul_rn(d.unit(), tot), lp);
            } else if (SMP == MHW_SAMPLER_ALIAS) {
                // table of the reference slot (manager.hpp:29-31)
                uint64_t slot, toff;
                if (KIND == DEEPWALK) {
                    slot = c.v;
                    toff = (uint64_t)c.off;
                } else if (KIND == METAPATH2VEC) {
                    slot = (uint64_t)c.v * M.num_types + c.req;
                    toff = (uint64_t)c.off * M.num_types + (uint64_t)c.req * c.deg;
                } else {
                    slot = (uint64_t)c.off + affix;
                    toff = __ldg(X.qoff + c.v) + (uint64_t)affix * c.deg;
                }
                uint32_t st = 0;
                if (lane == 0) st = atomicCAS(X.astat + slot, AS_EMPTY, AS_BUILDING);
                st = __shfl_sync(kFull, st, 0);
                if (st == AS_EMPTY) {
                    // alias_build(dynamic_weights) by this warp
                    double* Pp = X.aprob + toff;
                    uint32_t* Aa = X.aalias + toff;
                    uint32_t lp;
                    const double tot = warp_total(fw, c.deg, lane, nullptr, Pp, &lp);
                    if (!(tot > 0)) {
                        st = AS_DEAD;
                    } else {
                        __syncwarp();
                        const double dn = (double)c.deg;
                        for (uint32_t i = lane; i < c.deg; i += 32) {
                            Pp[i] = __ddiv_rn(__dmul_rn(Pp[i], dn), tot);
                            Aa[i] = i;
                        }
                        __syncwarp();
                        if (lane == 0) alias_pairs(Pp, Aa, scr, c.deg);
                        st = AS_READY;
                    }
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence();
                        st_release(X.astat + slot, st);
                    }
                } else {
                    unsigned ns = 32;
                    while (st == AS_BUILDING) {
                        __nanosleep(ns);
                        ns = ns < 1024 ? ns * 2 : 1024;
                        if (lane == 0) st = ld_acquire(X.astat + slot);
                        st = __shfl_sync(kFull, st, 0);
                    }
                }
                if (st == AS_DEAD) {
                    dead = true;
                    break;
                }
                // alias_sample (samplers.hpp:65-68); the table may have been
                // written by another SM in this launch: read it through L2
                const uint32_t i = d.index(c.deg);
                const double u = d.unit();
                chosen = u < __ldcg(X.aprob + toff + i) ? i : __ldcg(X.aalias + toff + i);
            } else {
                // rejection (engine.cpp:109-115): static proposal exists iff
                // the static total is positive; the target must have mass
                const double stot = g.w ? __ldg(g.wtotal + c.v) : (double)c.deg;
                if (!(stot > 0)) {
                    dead = true;
                    break;
                }
                if (!all_positive<KIND>(M, c)) {
                    bool any = false;
                    for (uint32_t base = 0; base < c.deg && !any; base += 32) {
                        const uint32_t i = base + lane;
                        any = __ballot_sync(kFull, i < c.deg && fw(i) > 0) != 0;
                    }
                    if (!any) {
                        dead = true;
                        break;
                    }
                }
                // The envelope target <= bound * w holds by construction
                // (rejection_bound; M >= 0 is enforced by bind).
                for (uint64_t t0 = 0;; t0 += 32) {
                    const uint64_t t = t0 + lane;
                    // trial epochs of 65536 under distinct keys: the 16-bit
                    // sub-counter field never wraps onto an earlier trial
                    const uint2 tkey = make_uint2(rkey.x, rkey.y ^ DOM_REJECT ^ (DOM_REJECT + (uint32_t)(t >> 16)));
                    const uint32_t sub = (uint32_t)(t & 0xFFFFu) << 16;
                    Draw a;
                    a.open_sub(tkey, walker, step, sub);
                    uint32_t i = a.index(c.deg);
                    if (!(a.unit() < __ldg(X.sprob + c.off + i))) i = __ldg(X.salias + c.off + i);
                    const double acc = __ddiv_rn(fw(i), __dmul_rn(X.bound, static_w(g, c.off + i)));
                    bool ok = acc >= 1.0;
                    if (!ok) {
                        Draw b;
                        b.open_sub(tkey, walker, step, sub | 0x8000u);
                        ok = b.unit() < acc;
                    }
                    const unsigned bal = __ballot_sync(kFull, ok);
                    if (bal) {
                        const uint32_t first = __ffs(bal) - 1;
                        chosen = __shfl_sync(kFull, i, first);
                        trials += t0 + first + 1;
                        break;
                    }
                }
            }
            const uint32_t next = load_id(g, c.off + chosen);
            const NodeRec rn = load_node(g, next);
            if (lane == 0) orow[len] = next;
            ++len;
            ++steps;
            // update_state (models.cpp:125-136)
            if (KIND == METAPATH2VEC) {
                affix = metapath_next(M, affix);
                c.req = M.metapath[metapath_next(M, affix)];
            } else if (second_order(KIND)) {
                const uint32_t back = __ldg(g.rev + c.off + chosen);
                if (back == kNoBack) {
                    if (lane == 0 && atomicCAS(&P.ctr[4], 0ull, 1ull) == 0ull)
                        P.ctr[5] = ((unsigned long long)next << 32) | c.v;
                    dead = true;
                    break;
                }
                if (KIND == EDGE2VEC) c.in_type = edge_type_of(g, c.off + chosen, c.vtype, rn.type);
                c.s = c.v;
                c.off_s = c.off;
                c.deg_s = c.deg;
                c.boot = false;
                affix = back;
            }
            c.v = next;
            c.off = rn.off;
            c.deg = rn.deg;
            c.vtype = rn.type;
            c.vflags = rn.flags;
        }
        if (lane == 0) {
            P.lens[row] = len;
            if (dead) ++early;
        }
    }
    if (lane == 0) {
        if (steps) atomicAdd(&P.ctr[1], steps);
        if (early) atomicAdd(&P.ctr[2], early);
        if (trials) atomicAdd(&P.ctr[7], trials);
    }
}

__global__ void k_deg_sq(DevGraph g, uint64_t* __restrict__ out) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t d = load_node(g, (uint32_t)v).deg;
        out[v] = d * d;
    }
}

template <class F>
void dispatch_exact(int kind, int smp, F&& f) {
    auto by_smp = [&](auto kc) {
        switch (smp) {
            case MHW_SAMPLER_ALIAS: f(kc, std::integral_constant<int, MHW_SAMPLER_ALIAS>{}); break;
            case MHW_SAMPLER_DIRECT: f(kc, std::integral_constant<int, MHW_SAMPLER_DIRECT>{}); break;
            default: f(kc, std::integral_constant<int, MHW_SAMPLER_REJECTION>{}); break;
        }
    };
    switch (kind) {
        case DEEPWALK: by_smp(std::integral_constant<int, DEEPWALK>{}); break;
        case NODE2VEC: by_smp(std::integral_constant<int, NODE2VEC>{}); break;
        case METAPATH2VEC: by_smp(std::integral_constant<int, METAPATH2VEC>{}); break;
        case EDGE2VEC: by_smp(std::integral_constant<int, EDGE2VEC>{}); break;
        default: by_smp(std::integral_constant<int, FAIRWALK>{}); break;
    }
}

unsigned grid_for(uint64_t work, int block = 256) {
    const uint64_t g = (work + block - 1) / block;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, 148ull * 16));
}

size_t free_bytes() { return dev_available_bytes(); }

}  // namespace

double exact_rejection_bound(const mhw_model_desc& md, const Model& m) {
    double alpha_max = 1.0;
    if (1.0 / md.p > alpha_max) alpha_max = 1.0 / md.p;
    if (1.0 / md.q > alpha_max) alpha_max = 1.0 / md.q;
    switch (m.dev.kind) {
        case DEEPWALK:
        case METAPATH2VEC: return 1.0;
        case NODE2VEC:
        case FAIRWALK: return alpha_max;
        default: {
            double m_max = 0.0;
            const uint64_t n = (uint64_t)md.type_matrix_dim * md.type_matrix_dim;
            for (uint64_t i = 0; i < n; ++i) m_max = std::max(m_max, md.type_matrix[i]);
            return alpha_max * m_max;
        }
    }
}

void exact_create(Session& s) {
    Graph& g = *s.g;
    ExactState& X = *s.ex;
    X.sampler = s.wc.sampler;
    cudaStream_t st = s.stream;
    const int kind = s.model.dev.kind;
    int per_sm = 0;
    dispatch_exact(kind, X.sampler, [&](auto kc, auto sc) {
        MHW_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, k_walk_exact<decltype(kc)::value, decltype(sc)::value>, kExBlock, 0));
    });
    int dev = 0, sms = 0;
    MHW_CK(cudaGetDevice(&dev));
    MHW_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    X.grid = std::max(1, per_sm) * sms;
    if (X.sampler == MHW_SAMPLER_ALIAS) {
        // tables for every reference slot (bench aux_memory, tools/mhwalk.cpp:307)
        const uint64_t slots = k_slots(kind, g);
        if (kind == DEEPWALK) {
            X.table_entries = g.m;
        } else if (kind == METAPATH2VEC) {
            X.table_entries = g.m * (uint64_t)g.n_ntypes;
        } else {
            X.qoff.alloc(g.n + 1);
            DBuf<uint64_t> sq(g.n + 1);
            MHW_CK(cudaMemsetAsync(sq.p, 0, (g.n + 1) * 8, st));
            k_deg_sq<<<grid_for(g.n), 256, 0, st>>>(g.view(), sq.p);
            MHW_CK(cudaGetLastError());
            size_t bytes = 0;
            MHW_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, sq.p, X.qoff.p, (int64_t)g.n + 1, st));
            DBuf<uint8_t> temp(std::max<size_t>(bytes, 1));
            MHW_CK(cub::DeviceScan::ExclusiveSum(temp.p, bytes, sq.p, X.qoff.p, (int64_t)g.n + 1, st));
            MHW_CK(cudaMemcpyAsync(&X.table_entries, X.qoff.p + g.n, 8, cudaMemcpyDeviceToHost, st));
            MHW_CK(cudaStreamSynchronize(st));
        }
        uint64_t warps = (uint64_t)X.grid * kExWarps;
        X.scratch_per_warp = std::max<uint64_t>(g.max_deg, 1);
        const double need = 12.0 * (double)X.table_entries + 4.0 * (double)slots;
        const size_t fb = free_bytes();
        // stack scratch: shrink the grid rather than fail
        while (warps > kExWarps && 4.0 * warps * X.scratch_per_warp > 0.25 * (double)fb) {
            X.grid = std::max(1, X.grid / 2);
            warps = (uint64_t)X.grid * kExWarps;
        }
        if (need + 4.0 * warps * X.scratch_per_warp + (2ull << 30) > (double)fb)
            invalid("alias sampler: per-state alias tables need " + std::to_string(need / 1e9) +
                    " GB (12 B x sum over states of the degree), more than the device has free");
        X.astat.alloc(std::max<uint64_t>(slots, 1));
        X.aprob.alloc(std::max<uint64_t>(X.table_entries, 1));
        X.aalias.alloc(std::max<uint64_t>(X.table_entries, 1));
        X.scratch.alloc(warps * X.scratch_per_warp);
    } else if (X.sampler == MHW_SAMPLER_REJECTION) {
        X.bound = exact_rejection_bound(s.model.desc, s.model);
        graph_ensure_wtotal(g);  // static totals (proposal existence)
        if ((double)g.m * 12.0 + (2ull << 30) > (double)free_bytes())
            invalid("rejection sampler: static proposals do not fit in device memory");
        X.sprob.alloc(std::max<uint64_t>(g.m, 1));
        X.salias.alloc(std::max<uint64_t>(g.m, 1));
        graph_alias_device(g, X.sprob.p, X.salias.p);
    }
}

void exact_launch(Session& s, const RunParams& P, cudaStream_t st) {
    ExactState& X = *s.ex;
    if (X.sampler == MHW_SAMPLER_ALIAS) {
        MHW_CK(cudaMemsetAsync(X.astat.p, 0, X.astat.bytes(), st));
    }
    ExParams E;
    E.bound = X.bound;
    E.astat = X.astat.n ? X.astat.p : nullptr;
    E.aprob = X.aprob.n ? X.aprob.p : nullptr;
    E.aalias = X.aalias.n ? X.aalias.p : nullptr;
    E.qoff = X.qoff.n ? X.qoff.p : nullptr;
    E.scratch = X.scratch.n ? X.scratch.p : nullptr;
    E.scratch_per_warp = X.scratch_per_warp;
    E.sprob = X.sprob.n ? X.sprob.p : nullptr;
    E.salias = X.salias.n ? X.salias.p : nullptr;
    dispatch_exact(s.model.dev.kind, X.sampler, [&](auto kc, auto sc) {
        k_walk_exact<decltype(kc)::value, decltype(sc)::value><<<X.grid, kExBlock, 0, st>>>(P, E);
    });
    MHW_CK(cudaGetLastError());
}

}  // namespace mhw
