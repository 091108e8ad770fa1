// walk.cu -- the M-H walk kernels and the session that drives them.
//
// Reference path: generate_walks (engine.cpp:157-234) -> next_edge
// (engine.cpp:75-118) -> SamplerManager::sample (manager.cpp:30-72) ->
// mh_transition (samplers.hpp:18-27) -> calculate_weight (models.cpp:82-123)
// -> update_state (models.cpp:125-136).
//
// Two schedules share the device functors of mhw_device.cuh:
//  * throughput: one persistent kernel; each thread owns a walker for all L
//    steps in registers; a state's chain word (one uint32 per state, HBM,
//    colocated with the session arc records for second-order models) is taken
//    as a lock with an atomic exchange for the whole transition, so every
//    state runs an exact sequential M-H chain (no lost updates);
//    slots are initialised eagerly or on first touch with slot-keyed
//    randomness, so any initialiser computes the same word.
//  * deterministic: step-synchronous; same-slot contenders are folded in
//    walker-id order; byte-reproducible and equal to the CPU oracle's
//    (philox, step-major) mode.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "exact.h"
#include "internal.h"
#include "walk.h"

namespace mhw {

namespace {

#ifndef MHW_ROWBUF_SMEM  // walk rows staged in shared memory, one 32-byte store per 8 steps
#define MHW_ROWBUF_SMEM 1
#endif
#ifndef MHW_ROWBUF_IDS  // ids staged per thread and flushed together (cfg2 walk: 8 -> 20.79 ms, 16 -> 19.52, 32 -> 19.66)
#define MHW_ROWBUF_IDS 16
#endif
constexpr uint32_t kRowGDefault = MHW_ROWBUF_IDS;
#ifndef MHW_C16_HASH_HINT
#define MHW_C16_HASH_HINT 1
#endif
#ifndef MHW_IDS_ALL_HINT  // compact chains: the Last's id loads (the candidate's: MHW_IDS_HINT)
#define MHW_IDS_ALL_HINT 3
#endif
#ifndef MHW_WALK_BLOCK
#define MHW_WALK_BLOCK 256
#endif
#ifndef MHW_REG80  // experiment: the register cap the "80" variants compile to
#define MHW_REG80 80
#endif
constexpr int kWalkBlock = MHW_WALK_BLOCK;
constexpr uint32_t kDeadMark = 0xFFFFFFFEu;

// Releases a chain slot taken with atomicExch(kLocked). The lock protects
// only the chain word itself, so a relaxed GPU-scope store suffices (no
// other data is published; a release store would add a full fence).
// u32 index of the chain word inside a session record of rw words.
__host__ __device__ __forceinline__ uint32_t chain_word_off(uint32_t rw) { return rw == 2 ? 1 : (rw == 8 ? 5 : 3); }

__device__ __forceinline__ void chain_release(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 16-byte atomic exchange (sm_90+): a typed record's chain word travels with
// the cached w'(Last) in one access, so both are always read and written
// together.
__device__ __forceinline__ uint4 atom_exch128(uint4* p, uint4 v) {
    const unsigned long long lo = ((unsigned long long)v.y << 32) | v.x, hi = ((unsigned long long)v.w << 32) | v.z;
    unsigned long long rlo, rhi;
    asm volatile(
        "{\n\t.reg .b128 d, b;\n\tmov.b128 b, {%2, %3};\n\tatom.global.exch.b128 d, [%4], b;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(rlo), "=l"(rhi)
        : "l"(lo), "l"(hi), "l"(p)
        : "memory");
    return make_uint4((uint32_t)rlo, (uint32_t)(rlo >> 32), (uint32_t)rhi, (uint32_t)(rhi >> 32));
}

// Compact chain words (AR = 3, node2vec): one 16-bit word per state, two
// per 32-bit word, so the table of a scale-20 graph (31.4 M states, 63 MB)
// stays in L2 and the lock/release traffic never reaches DRAM (the 32-bit
// words colocated in the arc records dirty one record sector per step,
// written back: cfg2 19.4 GB per launch). Encoding, by the state's degree
// deg(v): deg < 2^14: Last index | alpha class << 14; otherwise the Last index
// alone (class recomputed from the Last's id when needed). 0xFFFF = locked
// (every bit set, so an atomicOr takes the lock and returns the word),
// 0xFFFE = dead end. Requires deg(v) <= 0xFFFD and eager initialisation.
constexpr uint32_t kC16Locked = 0xFFFFu, kC16Dead = 0xFFFEu, kC16ClsDeg = 1u << 14;

__host__ __device__ __forceinline__ uint32_t c16_enc(uint32_t e, uint32_t deg) {
    if (e >= kLocked) return kC16Dead;  // kDead (kEmpty: a record no state uses)
    const uint32_t idx = e & kIdxMask;
    return deg < kC16ClsDeg ? (idx | ((e >> 30) << 14)) : idx;
}
// 32-bit chain word of a 16-bit one; class 3 = not stored (hub states)
__device__ __forceinline__ uint32_t c16_dec(uint32_t e16, uint32_t deg) {
    if (e16 == kC16Locked) return kLocked;
    if (e16 == kC16Dead) return kDead;
    return deg < kC16ClsDeg ? ((e16 & 0x3FFFu) | ((e16 >> 14) << 30)) : (e16 | (3u << 30));
}
__device__ __forceinline__ uint32_t c16_take(uint32_t* w, uint32_t sh, uint32_t deg) {
    return c16_dec((atomicOr(w, kC16Locked << sh) >> sh) & 0xFFFFu, deg);
}
// our half holds 0xFFFF while locked: AND-ing leaves the new word there and
// the neighbouring state's half untouched
__device__ __forceinline__ void c16_release(uint32_t* w, uint32_t sh, uint32_t e16) {
    atomicAnd(w, ~(kC16Locked << sh) | (e16 << sh));
}

__device__ __forceinline__ void fail_back_edge(unsigned long long* ctr, uint32_t from, uint32_t to) {
    if (atomicCAS(&ctr[4], 0ull, 1ull) == 0ull) ctr[5] = ((unsigned long long)from << 32) | to;
}

// Lazy slot initialisation out of line: keeps the rarely taken init code
// (count/select loops, burn-in) from inflating the walk kernel's registers.
template <int KIND>
__device__ __noinline__ uint32_t init_slot_ool(const DevGraph g, const DevModel m, const DevCfg cfg, const SCtx c,
                                               uint64_t slot) {
    return init_slot<KIND>(g, m, cfg, c, slot);
}

// ------------------------------------------------------ throughput kernel
// LAZY = false: every slot was initialised by k_init_all before the launch,
// so the lazy-init call (and the registers the call ABI pins) is compiled out.
// AR = true: arc records replace the id / node-record / weight / type loads
// of a step. deepwalk: graph records, aux = weight. Other models: the
// session's records (ArcRec in walk.h); for second-order models their aux
// word is the chain word of the state entered through that arc (colocated
// chains: the word a step locks sits in the sector the previous step loaded
// as its candidate record, so the lock is an L2 hit).
// AR = 2 (node2vec, small node tables): narrow 8-byte records {u, chain
// word}; the candidate's degree and offset come from its L2-resident node
// record, so the record array the walk gathers from is half as large.
// AR = 4: the plain-CSR variant (as AR = 0) with the static-weight alias
// proposal and the Hastings accept (mhw_walk_config.proposal = ALIAS).
template <int KIND, int REGS, bool LAZY, int ARV>
__global__ void __launch_bounds__(kWalkBlock) __maxnreg__(REGS == 80 ? MHW_REG80 : REGS) k_walk(RunParams P) {
    constexpr bool ALIAS = ARV == 4 || ARV == 5;  // 4: plain CSR, 5: arc records
    constexpr int AR = ARV == 4 ? 0 : (ARV == 5 ? 1 : ARV);
    const DevGraph& g = P.g;
#if MHW_ROWBUF_SMEM
    // deepwalk on L2-resident graphs is not DRAM-bound: one sector per flush (cfg1 1.00 vs 1.04 ms);
    // metapath2vec: a whole 128-byte line per flush (cfg3a 43.3 -> 43.0 ms)
    constexpr uint32_t kRowG = KIND == DEEPWALK ? 8u : (KIND == METAPATH2VEC ? 32u : kRowGDefault);
    __shared__ uint32_t rowbuf[kRowG][kWalkBlock];
#endif
    constexpr bool TYPED = AR && needs_utype<KIND>();
    constexpr bool CC = AR && second_order(KIND);
    constexpr bool NARROW = AR == 2;
    constexpr bool C16 = AR == 3;  // ids + compact 16-bit chain table (node2vec)
    constexpr int kHashHint = C16 ? MHW_C16_HASH_HINT : MHW_HASH_HINT;  // hash buckets evict-first beside the pinned table
    static_assert(!C16 || (KIND == NODE2VEC && !LAZY), "compact chains: eagerly initialised node2vec");
    // typed second-order records carry w'(Last) next to the chain word
    // (word 1 = {type | etype << 16, chain word, w'(Last) as f64}), taken and
    // released with one 16-byte exchange: the decision needs no load of the
    // Last's record, which is fetched only when the walker moves to it
    constexpr bool WLC = TYPED && CC;
    constexpr uint32_t RS = TYPED ? 2u : 1u;  // uint4 words per record (wide layouts)
    const uint4* const arcs = (AR && KIND != DEEPWALK) ? P.ac : g.arc;
    auto load_rec = [&](uint64_t arc, uint4& b) {
        if constexpr (C16) {
            const uint32_t u = ldg32h<MHW_IDS_ALL_HINT>(g.ids + arc);
            const uint2 r = __ldg(P.nodes8 + u);
            return make_uint4(u, r.y, r.x, 0u);
        }
        if constexpr (NARROW) {
            const uint2 x = __ldg(reinterpret_cast<const uint2*>(P.ac) + arc);
            const NodeRec r = load_node(g, x.x);
            return make_uint4(x.x, r.deg | ((r.flags & NF_ALLPOS) ? 0x80000000u : 0u), (uint32_t)r.off, x.y);
        }
        if constexpr (TYPED) {
            uint4 a;
            // metapath2vec: no L1 allocation (cfg3a 43.33 -> 42.77 ms; cfg5's wide records 876 -> 969, cfg1 1.00 -> 1.34)
            ldg256h<(KIND == METAPATH2VEC ? 3 : MHW_REC_HINT)>(arcs + RS * arc, a, b);  // the whole 32-byte record in one request
            return a;
        }
        return ldg128h<MHW_REC_HINT>(arcs + RS * arc);
    };
    auto rec_node = [&](const uint4& a, const uint4& b) {
        NodeRec r = arc_node(a);
        if (TYPED) r.type = (uint16_t)(b.x & 0xFFFFu);
        return r;
    };
    const uint2 wkey = philox_key(P.cfg.seed, DOM_WALK);
    const uint32_t K = P.cfg.K, L = P.cfg.L;
    const unsigned lane = threadIdx.x & 31;
    unsigned long long steps = 0, early = 0, inits = 0, retries = 0;
    for (;;) {
        // warp-aggregated work fetch (k-major item order spreads a start
        // node's K walkers over time, limiting same-slot contention)
        const unsigned mask = __activemask();
        const unsigned leader = __ffs(mask) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(&P.ctr[0], (unsigned long long)__popc(mask));
        base = __shfl_sync(mask, base, leader);
        const uint64_t item = base + __popc(mask & ((1u << lane) - 1));
        if (item >= P.n_items) break;
        const uint32_t k = (uint32_t)(item / P.n_act);
        const uint32_t j = (uint32_t)(item - (uint64_t)k * P.n_act);
        const uint32_t v0 = __ldg(P.act + j);
        const uint64_t row = __ldg(P.act_row + j) + k;
        const uint64_t walker = (uint64_t)v0 * K + k;
        uint32_t* orow = P.out + row * P.stride;

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
        uint32_t affix = 0;
        uint64_t slot = 0;
        uint64_t loc = 0;  // CC: forward arc s->v holding the chain word of state (s, v)
        uint32_t tx = 0;   // WLC: static type word of record loc (rewritten by every exchange)
        if (KIND == METAPATH2VEC) c.req = P.m.metapath[metapath_next(P.m, 0)];
        if (!second_order(KIND)) slot = slot_of<KIND>(P.m, P.cfg, c, 0, walker);
        uint32_t len = 1;
#if MHW_ROWBUF_SMEM
        // Row ids are staged in shared memory, 8 per thread (column threadIdx.x
        // of rowbuf: bank-conflict free), and leave as ONE aligned 32-byte
        // store per 8 steps: the two 16-byte halves of a sector written 4 steps
        // (~27 us) apart were evicted separately from the busy L2 (ncu: 4.76 GB
        // of DRAM writes for 2.2 GB of rows). ph: the row's first id sits at
        // slot ph (0 or 4) of its 32-byte group (rows are 16-byte aligned).
        const uint32_t ph = (uint32_t)((row * P.stride) & (kRowG - 1u));
        uint32_t* const orow_al = orow - ph;
        rowbuf[ph][threadIdx.x] = v0;
#else
        uint32_t b0 = v0, b1 = 0, b2 = 0, b3 = 0;
#endif
        bool dead = false;
        for (uint32_t step = 0; step < L; ++step) {
            if (c.deg == 0) {
                dead = true;
                break;
            }
            Draw d;
            d.open(wkey, walker, step);
            uint32_t chosen, next, back_c = 0;
            NodeRec rn;
            uint4 bn = make_uint4(0, 0, 0, 0);  // typed word of the chosen record
            if (second_order(KIND) && c.boot) {
                if (!bootstrap_pick(g, c, d.unit(), &chosen)) {
                    dead = true;
                    break;
                }
                if constexpr (AR) {
                    const uint4 a = load_rec(c.off + chosen, bn);
                    next = a.x;
                    rn = rec_node(a, bn);
                    if (!CC) back_c = a.w;
                } else {
                    next = load_id(g, c.off + chosen);
                    rn = load_node(g, next);
                    back_c = __ldg(g.rev + c.off + chosen);
                }
            } else {
                // Take the slot: the chain word itself is the lock. The
                // transition (proposal evaluation + decision) happens while
                // holding it, so the order of transitions on a chain never
                // depends on proposals or decisions -> every slot runs an
                // exact sequential M-H chain (manager.cpp:63-71 semantics
                // without lost updates).
                // The exchange is issued before any candidate-dependent work
                // (its timing cannot depend on the proposal); the candidate
                // evaluation overlaps its latency, and the chain state it
                // returns is only consumed by the decision.
                uint32_t* const cw = C16 ? P.c16 + (loc >> 1)
                                         : ((!CC || WLC) ? P.chain + slot
                                                         : (NARROW ? reinterpret_cast<uint32_t*>(P.ac) + 2 * loc + 1
                                                                   : reinterpret_cast<uint32_t*>(P.ac + RS * loc) + 3));
                const uint32_t csh = C16 ? ((uint32_t)loc & 1u) << 4 : 0u;
                uint4* const cb = WLC ? P.ac + 2 * loc + 1 : nullptr;
                uint4 E = make_uint4(0, 0, 0, 0);
                uint32_t e;
                uint32_t cand;
                double u;
                uint32_t c16_uc = 0;
                if constexpr (C16) {
                    // compact chains: the candidate id load (DRAM) is issued
                    // first and the lock right after it, with no dependency
                    // between them (the lock's timing still cannot depend on
                    // the proposal); otherwise the scheduler waits for the
                    // atomic's return before issuing the load (ncu: 13% of the
                    // stall samples on the decode of the lock word).
                    cand = d.index(c.deg);
                    u = d.unit();
                    c16_uc = ldg32h<MHW_IDS_HINT>(g.ids + c.off + cand);
                }
                if (WLC) {
                    E = atom_exch128(cb, make_uint4(tx, kLocked, 0u, 0u));
                    e = E.y;
                } else if (C16) {
                    e = c16_take(cw, csh, c.deg);
                } else {
                    e = atomicExch(cw, kLocked);
                }
                if constexpr (C16) {
                    if (P.m.ret_skip) {
                        // Last of the return class (it is s): a proposal of it,
                        // or any proposal once u * w'(Last) reaches the heaviest
                        // other class, is rejected whatever the candidate is --
                        // the decision of mh_accept (samplers.hpp:24) without
                        // the candidate's id, record or alpha probe; the walker
                        // steps back to s (id and slice in registers)
                        if (e < kLocked && (e >> 30) == 0u &&
                            (cand == (e & kIdxMask) || __dmul_rn(u, P.m.inv_p) >= P.m.ret_wmax)) {
                            c16_release(cw, csh, c16_enc(e, c.deg));
                            chosen = e & kIdxMask;
                            next = c.s;
                            rn.off = c.off_s;
                            rn.deg = c.deg_s;
                            rn.type = 0;
                            rn.flags = 0;
                            goto emit;
                        }
                    }
                } else if constexpr (ALIAS) {
                    // alias_sample (samplers.hpp:65-68) of v's static table:
                    // index on word 0, coin on words 1-2; the accept unit
                    // from sub-block kAcceptSub
                    const uint32_t i = d.index(c.deg);
                    // {prob f64, alias} of index i in one 16-byte load
                    if (g.sal) {
                        const uint4 t = __ldg(g.sal + c.off + i);
                        cand = d.unit() < __hiloint2double((int)t.y, (int)t.x) ? i : t.z;
                    } else {
                        cand = i;  // unweighted: every prob is 1.0
                    }
                    Draw da;
                    da.open_sub(wkey, walker, step, kAcceptSub);
                    u = da.unit();
                } else {
                    cand = d.index(c.deg);
                    u = d.unit();
                }
                // fairwalk: v's group sizes (one row of <= 4 types) are read
                // with the candidate's record instead of after it
                uint32_t grp0 = 0, grp1 = 0, grp2 = 0, grp3 = 0;
                const bool grp_pre = KIND == FAIRWALK && TYPED && g.n_ntypes <= 4;
                if (grp_pre) {
                    const uint32_t* row = g.tcount + (size_t)c.v * g.n_ntypes;
                    grp0 = __ldg(row);
                    if (g.n_ntypes > 1) grp1 = __ldg(row + 1);
                    if (g.n_ntypes > 2) grp2 = __ldg(row + 2);
                    if (g.n_ntypes > 3) grp3 = __ldg(row + 3);
                }
                uint32_t uc;
                uint4 ac = make_uint4(0, 0, 0, 0), bc = make_uint4(0, 0, 0, 0);
                NodeRec rc{};
                bool rc_early;
                int pre_bloom = -1;
                uint2 xl = make_uint2(0, 0);
                bool spec_l = false;
                if constexpr (NARROW || C16) {
                    // The edge-filter probe needs only the candidate id: it is
                    // computed and issued before the candidate's node record is
                    // consumed, so the two L2 accesses overlap instead of
                    // running back to back.
                    const uint2 x = C16 ? make_uint2(c16_uc, 0u)
                                        : __ldg(reinterpret_cast<const uint2*>(P.ac) + c.off + cand);
                    // A Last of the heaviest alpha class is rejected away from
                    // most of the time (cfg2: the return class, 1/p = 4): fetch
                    // its record now, beside the candidate's, instead of after
                    // the decision (cfg2 34.6 -> 34.3 ms; speculating on every
                    // Last heavier than the lightest class: 35.4).
                    // (compact chains of hub states hold no class: the Last's
                    // id is needed for it anyway)
                    // (compact chains: a Last of the return class IS s -- its
                    // id and slice are in registers, nothing to fetch)
                    if (e < kLocked && (C16 ? ((e >> 30) == 3u || ((e >> 30) == P.m.spec_cls && (e >> 30) != 0u))
                                            : (e >> 30) == P.m.spec_cls)) {
                        xl = C16 ? make_uint2(ldg32h<MHW_IDS_ALL_HINT>(g.ids + c.off + (e & kIdxMask)), 0u)
                                 : __ldg(reinterpret_cast<const uint2*>(P.ac) + c.off + (e & kIdxMask));
                        spec_l = true;
                    }
                    uc = x.x;
                    if constexpr (C16) {
                        // 8-byte node record {off, deg | allpos << 31}
                        const uint2 nr = ldg64h<MHW_NODE8_HINT>(P.nodes8 + uc);  // issued first
                        if (g.bloom && !P.m.alpha_trivial && uc != c.s) pre_bloom = bloom_maybe(g, c.s, uc) ? 1 : 0;
                        rc.off = nr.x;
                        rc.deg = nr.y & 0x7FFFFFFFu;
                        rc.type = 0;
                        rc.flags = (nr.y >> 31) ? NF_ALLPOS : 0;
                        ac = make_uint4(uc, nr.y, nr.x, 0u);
                    } else {
                        const int4 nraw = __ldg(reinterpret_cast<const int4*>(g.nodes) + uc);  // issued first
                        if (g.bloom && !P.m.alpha_trivial && uc != c.s) pre_bloom = bloom_maybe(g, c.s, uc) ? 1 : 0;
                        rc.off = ((long long)(uint32_t)nraw.y << 32) | (uint32_t)nraw.x;
                        rc.deg = (uint32_t)nraw.z;
                        rc.type = (uint16_t)((uint32_t)nraw.w & 0xFFFFu);
                        rc.flags = (uint16_t)((uint32_t)nraw.w >> 16);
                        ac = make_uint4(uc, rc.deg | ((rc.flags & NF_ALLPOS) ? 0x80000000u : 0u), (uint32_t)rc.off,
                                        x.y);
                    }
                    rc_early = true;
                } else if constexpr (AR) {
                    ac = load_rec(c.off + cand, bc);
                    uc = ac.x;
                    rc = rec_node(ac, bc);
                    rc_early = true;
                } else {
                    uc = load_id(g, c.off + cand);
                    // the candidate's record is needed before the decision
                    // only for its type or for the alpha slice choice;
                    // otherwise it is fetched after an acceptance
                    rc_early = needs_utype<KIND>() ||
                               (second_order(KIND) && !P.m.alpha_trivial && needs_urec_for_alpha(g, c));
                    if (rc_early) rc = load_node(g, uc);
                }
                const uint32_t cls_c =
                    second_order(KIND) ? alpha_class<kHashHint>(g, P.m, c, uc, rc_early ? &rc : nullptr, pre_bloom) : 0u;
                double wc;
                if (AR && KIND == DEEPWALK) wc = (double)__uint_as_float(ac.w);
                else if (grp_pre) {
                    // w' = (alpha * w) / group (models.cpp:115-119)
                    const uint32_t t = rc.type;
                    const uint32_t grp = t == 0 ? grp0 : (t == 1 ? grp1 : (t == 2 ? grp2 : grp3));
                    wc = c.boot ? (double)__uint_as_float(ac.w)
                                : __ddiv_rn(__dmul_rn(alpha_value(P.m, cls_c), (double)__uint_as_float(ac.w)),
                                            (double)grp);
                } else if (TYPED) wc = wprime_v<KIND>(g, P.m, c, (double)__uint_as_float(ac.w), rc.type, bc.x >> 16, cls_c);
                else wc = wprime<KIND>(g, P.m, c, cand, rc.type, cls_c);
                if (e == kLocked) {
                    // backoff: typed second-order chains (released by one
                    // 16-byte exchange) 8 -> 128 ns (cfg3b 90.7 -> 89.5 ms),
                    // others 32 -> 512 ns
                    constexpr unsigned kBo0 = WLC ? 8u : 32u, kBoMax = WLC ? 128u : 512u;
                    unsigned ns = kBo0;
                    do {
                        ++retries;
                        __nanosleep(ns);
                        ns = ns < kBoMax ? ns * 2 : kBoMax;
                        if (WLC) {
                            E = atom_exch128(cb, make_uint4(tx, kLocked, 0u, 0u));
                            e = E.y;
                        } else if (C16) {
                            e = c16_take(cw, csh, c.deg);
                        } else {
                            e = atomicExch(cw, kLocked);
                        }
                    } while (e == kLocked);
                }
                if (e == kEmpty) {
                    if constexpr (LAZY) {
                        // CC: slot id of (s, v) = off(v) + index of s in N(v)
                        if (CC) slot = (uint64_t)c.off + __ldg(g.rev + loc);
                        double w0 = 0.0;
                        e = init_slot<KIND>(g, P.m, P.cfg, c, slot, WLC ? &w0 : nullptr);
                        E.z = (uint32_t)__double2loint(w0);
                        E.w = (uint32_t)__double2hiint(w0);
                        ++inits;
                    } else {
                        e = kDead;  // unreachable: eager init filled every slot
                        fail_back_edge(P.ctr, 0xFFFFFFFFu, 0xFFFFFFFFu);
                    }
                }
                if (e == kDead) {
                    if (WLC) atom_exch128(cb, make_uint4(tx, kDead, 0u, 0u));
                    else if (C16) c16_release(cw, csh, kC16Dead);
                    else chain_release(cw, kDead);
                    dead = true;
                    break;
                }
                const uint32_t last = e & kIdxMask;
                uint32_t cls_l = e >> 30;
                if (C16 && cls_l == 3u) {
                    // hub state: the word holds no class; alpha(s, Last) from
                    // the Last's id (a pure function of (state, Last), as cached)
                    if (!spec_l) {
                        xl = make_uint2(ldg32h<MHW_IDS_ALL_HINT>(g.ids + c.off + last), 0u);
                        spec_l = true;
                    }
                    cls_l = alpha_class<kHashHint>(g, P.m, c, xl.x, nullptr);
                }
                // The last sample's id and record are fetched before the
                // decision where w'(last) needs its type anyway, and for
                // deepwalk (cheap, L2-resident graphs; measured win). For
                // node2vec/edge2vec the extra sectors cost more than the
                // shorter rejection path saves (profiles/, round 1).
                // (the alias proposal's Hastings ratio needs the Last's own
                // type / edge type, not the w'(Last) typed records cache)
                constexpr bool kSpec = (!WLC || ALIAS) && (needs_utype<KIND>() || KIND == DEEPWALK);
                uint32_t ul = 0;
                NodeRec rl{};
                uint4 al = make_uint4(0, 0, 0, 0), bl = make_uint4(0, 0, 0, 0);
                if (kSpec) {
                    if constexpr (AR) {
                        al = load_rec(c.off + last, bl);
                        ul = al.x;
                        rl = rec_node(al, bl);
                    } else {
                        ul = load_id(g, c.off + last);
                        rl = load_node(g, ul);
                    }
                }
                double wl;
                if (WLC) wl = __hiloint2double((int)E.w, (int)E.z);
                else if (AR && KIND == DEEPWALK) wl = (double)__uint_as_float(al.w);
                else if (TYPED) wl = wprime_v<KIND>(g, P.m, c, (double)__uint_as_float(al.w), rl.type, bl.x >> 16, cls_l);
                else wl = wprime<KIND>(g, P.m, c, last, rl.type, cls_l);
                bool acc;
                if constexpr (ALIAS) {
                    // Hastings: target w' = r w, proposal q ~ w -> min(1, r_c / r_l)
                    // records carry the edge type and the static weight
                    const uint32_t ot_c = KIND != EDGE2VEC ? 0u
                                          : (TYPED ? (bc.x >> 16) : edge_type_of(g, c.off + cand, c.vtype, rc.type));
                    const uint32_t ot_l = KIND != EDGE2VEC ? 0u
                                          : (TYPED ? (bl.x >> 16) : edge_type_of(g, c.off + last, c.vtype, rl.type));
                    const double r_c = rfactor<KIND>(g, P.m, c, rc.type, ot_c, cls_c);
                    const double r_l = rfactor<KIND>(g, P.m, c, rl.type, ot_l, cls_l);
                    const double w_c = (AR && (KIND == DEEPWALK || TYPED)) ? (double)__uint_as_float(ac.w)
                                                                           : static_w(g, c.off + cand);
                    acc = hastings_accept(w_c, r_c, r_l, u) && cand != last;
                    (void)wc;
                    (void)wl;
                } else {
                    acc = mh_accept(wc, wl, u) && cand != last;
                }
                if (WLC)
                    atom_exch128(cb, acc ? make_uint4(tx, pack_entry(cand, cls_c), (uint32_t)__double2loint(wc),
                                                      (uint32_t)__double2hiint(wc))
                                         : make_uint4(tx, e, E.z, E.w));
                else if (C16)  // (a 16-bit store release measured the same: 25.44 vs 25.25 ms)
                    c16_release(cw, csh, c16_enc(acc ? pack_entry(cand, cls_c) : e, c.deg));
                else
                    chain_release(cw, acc ? pack_entry(cand, cls_c) : e);
                chosen = acc ? cand : last;
                if constexpr (AR) {
                    const bool take_c = acc || cand == last;
                    uint4 an;
                    if (take_c) {
                        an = ac;
                        bn = bc;
                    } else if (kSpec) {
                        an = al;
                        bn = bl;
                    } else if (KIND == NODE2VEC && CC && cls_l == 0u) {
                        // return class: the Last is s itself (its id, offset and
                        // degree are the state's, no record load; the all-positive
                        // flag, left clear, only selects a lazy init's fast path,
                        // which returns the same index as the full scan)
                        an = make_uint4(c.s, c.deg_s, (uint32_t)c.off_s, 0u);
                    } else if (C16 && spec_l) {
                        const uint2 r = ldg64h<MHW_NODE8_HINT>(P.nodes8 + xl.x);
                        an = make_uint4(xl.x, r.y, r.x, 0u);
                    } else if (NARROW && spec_l && (e & kIdxMask) == last) {
                        const NodeRec r = load_node(g, xl.x);
                        an = make_uint4(xl.x, r.deg | ((r.flags & NF_ALLPOS) ? 0x80000000u : 0u), (uint32_t)r.off, xl.y);
                    } else {
                        an = load_rec(c.off + last, bn);
                    }
                    next = an.x;
                    rn = rec_node(an, bn);
                    if (!CC) back_c = an.w;
                } else {
                    if (acc || cand == last) {
                        next = uc;
                        rn = rc_early ? rc : load_node(g, uc);
                    } else if (kSpec) {
                        next = ul;
                        rn = rl;
                    } else {
                        next = load_id(g, c.off + last);
                        rn = load_node(g, next);
                    }
                    if (second_order(KIND)) back_c = __ldg(g.rev + c.off + chosen);
                }
            }
        emit:
            // emit: 4 ids buffered in registers, one 16-byte store
#if MHW_ROWBUF_SMEM
            {
                const uint32_t ab = ph + len;  // index from the aligned group base of the row
                rowbuf[ab & (kRowG - 1u)][threadIdx.x] = next;
                if ((ab & (kRowG - 1u)) == kRowG - 1u) {
                    // the whole group leaves together, sector by sector; the
                    // first group of a row starts at slot ph (a multiple of 4)
                    uint32_t* const gp = orow_al + (ab & ~(kRowG - 1u));
                    const uint32_t lo = ab < kRowG ? ph : 0u;
#pragma unroll
                    for (uint32_t k = 0; k < kRowG; k += 8) {
                        if (lo <= k) {
                            stg256(gp + k,
                                   make_uint4(rowbuf[k][threadIdx.x], rowbuf[k + 1][threadIdx.x], rowbuf[k + 2][threadIdx.x],
                                              rowbuf[k + 3][threadIdx.x]),
                                   make_uint4(rowbuf[k + 4][threadIdx.x], rowbuf[k + 5][threadIdx.x],
                                              rowbuf[k + 6][threadIdx.x], rowbuf[k + 7][threadIdx.x]));
                        } else if (lo == k + 4) {  // the row starts mid-sector: upper half only
                            *reinterpret_cast<uint4*>(gp + k + 4) =
                                make_uint4(rowbuf[k + 4][threadIdx.x], rowbuf[k + 5][threadIdx.x], rowbuf[k + 6][threadIdx.x],
                                           rowbuf[k + 7][threadIdx.x]);
                        }
                    }
                }
            }
#else
            switch (len & 3) {
                case 0: b0 = next; break;
                case 1: b1 = next; break;
                case 2: b2 = next; break;
                default:
                    b3 = next;
                    stg128h<MHW_STORE_HINT>(reinterpret_cast<uint4*>(orow + (len & ~3u)), make_uint4(b0, b1, b2, b3));
                    break;
            }
#endif
            ++len;
            ++steps;
            // update_state (models.cpp:125-136)
            if (KIND == DEEPWALK) {
                slot = node_slot(P.cfg, 1, next, rn.deg, 0, walker);
            } else if (KIND == METAPATH2VEC) {
                affix = metapath_next(P.m, affix);
                c.req = P.m.metapath[metapath_next(P.m, affix)];
                slot = node_slot(P.cfg, P.m.num_types, next, rn.deg, c.req, walker, rn.type);
            } else {
                // rev[off(v) + chosen], fetched above (CC: only checked on a
                // graph not verified symmetric; the chain word is located by
                // the forward arc itself)
                uint32_t back = back_c;
                if (CC) back = g.verified_sym ? 0u : __ldg(g.rev + c.off + chosen);
                if (back == kNoBack) {
                    fail_back_edge(P.ctr, next, c.v);
                    dead = true;
                    break;
                }
                if (KIND == EDGE2VEC)
                    c.in_type = TYPED ? (bn.x >> 16) : edge_type_of(g, c.off + chosen, c.vtype, rn.type);
                if (CC) loc = (uint64_t)c.off + chosen;
                if (WLC) tx = bn.x;
                c.s = c.v;
                c.off_s = c.off;
                c.deg_s = c.deg;
                c.boot = false;
                if (!CC) slot = (uint64_t)rn.off + back;
            }
            c.v = next;
            c.off = rn.off;
            c.deg = rn.deg;
            c.vtype = rn.type;
            c.vflags = rn.flags;
        }
#if MHW_ROWBUF_SMEM
        {
            const uint32_t ab = ph + len;              // next free index from the aligned base
            const uint32_t gb = ab & ~(kRowG - 1u);    // base of the pending group
            for (uint32_t sl = gb < ph ? ph : 0u; sl < (ab & (kRowG - 1u)); ++sl)
                orow_al[gb + sl] = rowbuf[sl][threadIdx.x];
        }
#else
        const uint32_t base4 = len & ~3u;
        const uint32_t pend = len & 3u;
        if (pend > 0) orow[base4] = b0;
        if (pend > 1) orow[base4 + 1] = b1;
        if (pend > 2) orow[base4 + 2] = b2;
#endif
        P.lens[row] = len;
        if (dead) ++early;
    }
    if (steps) atomicAdd(&P.ctr[1], steps);
    if (early) atomicAdd(&P.ctr[2], early);
    if (inits) atomicAdd(&P.ctr[3], inits);
    if (retries) atomicAdd(&P.ctr[6], retries);
}

// Node of arc a: the session's per-arc source array when it has one (one
// coalesced load; built for eagerly initialised second-order sessions), else
// the last v with nodes[v].off <= a (skips isolated nodes; ~log2(n)
// dependent loads per thread: 7-9% of k_init_all's stall samples on cfg2).
__device__ __forceinline__ uint32_t arc_owner(const RunParams& P, uint64_t a) {
    if (P.src) return __ldg(P.src + a);
    const DevGraph& g = P.g;
    uint32_t lo = 0, hi = g.n;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldg(&g.nodes[mid].off) <= a) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void k_arc_src(DevGraph g, uint32_t* __restrict__ out) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = wid; v < g.n; v += nw) {
        const NodeRec r = load_node(g, (uint32_t)v);
        for (uint32_t i = lane; i < r.deg; i += 32) out[r.off + i] = (uint32_t)v;
    }
}

// Eager chain-table initialisation of every arc-keyed slot (second-order
// models). Result-identical to the lazy path (init randomness is keyed by the
// slot), but runs with full warps and neighbouring threads share the node v.
// node2vec at 8 blocks/SM (32 registers, a few spills): the slots are
// independent random-gather chains, and occupancy wins (cfg2: 64 regs
// 40.1 ms step, 40 regs 39.6, 32 regs 39.1); the typed models spill more at
// 32 registers and keep 4 blocks/SM (cfg3b 112 vs 117 ms).
template <int KIND, int MINB = (KIND == NODE2VEC ? 6 : 4)>
__global__ void __launch_bounds__(256, MINB) k_init_all(RunParams P) {
    const DevGraph& g = P.g;
    unsigned long long inits = 0;
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < g.m;
         a += (uint64_t)gridDim.x * blockDim.x) {
        // node of arc a: the last v with nodes[v].off <= a (skips isolated nodes)
        const uint32_t lo = arc_owner(P, a);
        const NodeRec r = load_node(g, lo);
        const uint32_t affix = (uint32_t)(a - (uint64_t)r.off);
        const SCtx c = make_ctx<KIND>(g, P.m, lo, affix);
        double wl = 0.0;
        const uint32_t e = init_slot<KIND>(g, P.m, P.cfg, c, a, &wl);
        if (P.c16) {
            // compact: the 16-bit word of state (s, v) at forward arc s->v
            const uint32_t sv = __ldg(g.rev + a);
            if (sv != kNoBack)
                reinterpret_cast<uint16_t*>(P.c16)[(uint64_t)c.off_s + sv] = (uint16_t)c16_enc(e, c.deg);
        } else if (P.ac) {
            // colocated: the word lives in the record of the forward arc s->v
            const uint32_t sv = __ldg(g.rev + a);  // index of v in N(s)
            if (sv != kNoBack) {
                uint32_t* w = reinterpret_cast<uint32_t*>(P.ac) + ((uint64_t)c.off_s + sv) * P.rec_u32;
                w[chain_word_off(P.rec_u32)] = e;
                if (P.rec_u32 == 8) {  // typed: w'(Last) next to the word
                    w[6] = (uint32_t)__double2loint(wl);
                    w[7] = (uint32_t)__double2hiint(wl);
                }
            }
        } else {
            P.chain[a] = e;
        }
        ++inits;
    }
    if (inits) atomicAdd(&P.ctr[3], inits);
}

// Initial chain words of slots [b, e) (sharded init): k_init_all's work for
// a slot range, written contiguously.
template <int KIND>
__global__ void __launch_bounds__(256, KIND == NODE2VEC ? 6 : 4) k_init_range(RunParams P, uint64_t b, uint64_t e, uint32_t* __restrict__ out) {
    const DevGraph& g = P.g;
    for (uint64_t a = b + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < e;
         a += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t lo = arc_owner(P, a);
        const NodeRec r = load_node(g, lo);
        const SCtx c = make_ctx<KIND>(g, P.m, lo, (uint32_t)(a - (uint64_t)r.off));
        out[a - b] = init_slot<KIND>(g, P.m, P.cfg, c, a);
    }
}

// Shard exchange of compact chains (node2vec, AR 3): slot order (k_init_all's
// N(v) locality: a warp's slots share v), 16-bit words already encoded with
// deg(v) -- half the all-gather volume of 32-bit words -- installed by
// k_load_slot16 into the record position of each slot.
__global__ void __launch_bounds__(256, 6) k_init_range16(RunParams P, uint64_t b, uint64_t e,
                                                         uint16_t* __restrict__ out) {
    const DevGraph& g = P.g;
    for (uint64_t a = b + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < e;
         a += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t lo = arc_owner(P, a);
        const NodeRec r = load_node(g, lo);
        const SCtx c = make_ctx<NODE2VEC>(g, P.m, lo, (uint32_t)(a - (uint64_t)r.off));
        out[a - b] = (uint16_t)c16_enc(init_slot<NODE2VEC>(g, P.m, P.cfg, c, a), c.deg);
    }
}

// Slot a = (v, affix) holds state (s, v), s = N(v)[affix]; its compact word
// lives at the forward arc s -> v = off(s) + rev[a] (coalesced reads of ids /
// rev, one L2 node record, one 2-byte write into the L2-sized table).
__global__ void k_load_slot16(RunParams P, const uint16_t* __restrict__ w, uint64_t b, uint64_t e) {
    const DevGraph& g = P.g;
    for (uint64_t a = b + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < e;
         a += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t sv = __ldg(g.rev + a);
        if (sv == kNoBack) continue;
        const uint32_t src = load_id(g, a);
        reinterpret_cast<uint16_t*>(P.c16)[(uint64_t)__ldg(P.nodes8 + src).x + sv] = __ldg(w + (a - b));
    }
}

// Initial chain words in RECORD order (sharded init of colocated chains):
// record a = forward arc s->v holds the word of state (s, v), whose slot is
// off(v) + rev[a] (index of s in N(v)) -- the same slot-keyed init as
// k_init_range, permuted so that the install (k_load_rec) is a coalesced
// strided copy instead of a random scatter. out == nullptr: write straight
// into the session records (eager init in record order).
// State (s, v) of record a = arc s -> v, built from what record order gives
// for free: v, deg(v), off(v) (and v's type and the arc's edge type in typed
// records) come from the session record itself -- a coalesced load -- and s
// is the owner of arc a, shared by neighbouring threads (cached search), so
// the two random loads of make_ctx (N(v)[affix] and v's node record) go.
template <int KIND>
__device__ __forceinline__ SCtx rec_ctx(const RunParams& P, uint64_t a) {
    const DevGraph& g = P.g;
    SCtx c;
    uint32_t et = 0;
    if (P.ac && P.rec_u32 == 4) {
        const uint4 r = __ldg(P.ac + a);
        c.v = r.x;
        c.deg = r.y & 0x7FFFFFFFu;
        c.off = (long long)r.z;
        c.vtype = 0;
        c.vflags = (r.y >> 31) ? NF_ALLPOS : 0;
    } else if (P.ac && P.rec_u32 == 8) {
        uint4 r0, r1;
        ldg256(P.ac + 2 * a, r0, r1);
        c.v = r0.x;
        c.deg = r0.y & 0x7FFFFFFFu;
        c.off = (long long)r0.z;
        c.vtype = (uint16_t)(r1.x & 0xFFFFu);
        c.vflags = (r0.y >> 31) ? NF_ALLPOS : 0;
        et = r1.x >> 16;
    } else {
        c.v = load_id(g, a);
        const NodeRec r = load_node(g, c.v);
        c.off = r.off;
        c.deg = r.deg;
        c.vtype = r.type;
        c.vflags = r.flags;
    }
    uint32_t lo = 0, hi = g.n;  // s: the last node whose slice starts at or before a
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldg(&g.nodes[mid].off) <= a) lo = mid;
        else hi = mid;
    }
    const NodeRec rs = load_node(g, lo);
    c.s = lo;
    c.off_s = rs.off;
    c.deg_s = rs.deg;
    c.req = 0;
    c.boot = false;
    c.in_type = 0;
    if (KIND == EDGE2VEC) c.in_type = (P.ac && P.rec_u32 == 8) ? et : edge_type_of(g, a, rs.type, c.vtype);
    return c;
}

template <int KIND>
// node2vec at 6 blocks/SM (~40 registers): at 8 (32 registers) the record-order
// state build spills 352 bytes per thread (cfg5: 1064 ms vs 1055; 4 blocks: 1087)
__global__ void __launch_bounds__(256, KIND == NODE2VEC ? 6 : 4) k_init_rec(RunParams P, uint64_t b, uint64_t e, uint32_t* __restrict__ out) {
    const DevGraph& g = P.g;
    unsigned long long inits = 0;
    for (uint64_t a = b + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < e;
         a += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t affix = __ldg(g.rev + a);
        uint32_t w = kEmpty;  // no back arc: no state (s, v) can ever use this record
        double wl = 0.0;
        if (affix != kNoBack) {
            const SCtx c = rec_ctx<KIND>(P, a);
            w = init_slot<KIND>(g, P.m, P.cfg, c, (uint64_t)c.off + affix, &wl);
            ++inits;
        }
        if (out) {
            if (P.ac && P.rec_u32 == 8) {  // typed records: the word and w'(Last) travel together
                uint32_t* o = out + 3 * (a - b);
                o[0] = w;
                o[1] = (uint32_t)__double2loint(wl);
                o[2] = (uint32_t)__double2hiint(wl);
            } else {
                out[a - b] = w;
            }
        } else if (P.c16) {
            // record a = arc s -> v holds state (s, v); deg(v) from the state
            const uint32_t dv = affix != kNoBack ? load_node(g, load_id(g, a)).deg : 0u;
            reinterpret_cast<uint16_t*>(P.c16)[a] = (uint16_t)c16_enc(w, dv);
        } else {
            uint32_t* r = reinterpret_cast<uint32_t*>(P.ac) + a * P.rec_u32;
            r[chain_word_off(P.rec_u32)] = w;
            if (P.rec_u32 == 8) {
                r[6] = (uint32_t)__double2loint(wl);
                r[7] = (uint32_t)__double2hiint(wl);
            }
        }
    }
    if (!out && inits) atomicAdd(&P.ctr[3], inits);
}

// Installs a record-order table (k_init_rec words): one strided write per
// record; typed records take {word, w'(Last)} (3 words per record). Without
// session records the words go to their slots (chain table in slot order).
__global__ void k_load_rec(RunParams P, const uint32_t* __restrict__ w, uint32_t* __restrict__ ac, uint32_t rw,
                           uint32_t* __restrict__ chain, uint64_t b, uint64_t end) {
    const DevGraph& g = P.g;
    for (uint64_t a = b + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < end;
         a += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = a - b;  // entry of record a in w
        if (ac && rw == 8) {
            uint32_t* rec = ac + a * rw;
            rec[5] = __ldg(w + 3 * i);
            rec[6] = __ldg(w + 3 * i + 1);
            rec[7] = __ldg(w + 3 * i + 2);
            continue;
        }
        const uint32_t e = __ldg(w + i);
        if (P.c16) {  // record a = arc s -> v: the state's degree is deg(v)
            reinterpret_cast<uint16_t*>(P.c16)[a] = (uint16_t)c16_enc(e, load_node(g, load_id(g, a)).deg);
            continue;
        }
        if (ac) {
            ac[a * rw + chain_word_off(rw)] = e;
            continue;
        }
        const uint32_t affix = __ldg(g.rev + a);
        if (affix == kNoBack) continue;
        chain[(uint64_t)load_node(g, load_id(g, a)).off + affix] = e;
    }
}

// Installs a full table of slot words: colocated words go to the record of
// the forward arc s->v of slot (v, affix), s = N(v)[affix]; typed records
// also get w'(Last) of the word's Last (its class is in the word).
template <int KIND>
__global__ void k_load_chain(RunParams P, const uint32_t* __restrict__ w, uint32_t* __restrict__ ac, uint32_t rw,
                             uint32_t* __restrict__ chain) {
    const DevGraph& g = P.g;
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < g.m;
         a += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = __ldg(w + a);
        if (!ac && !P.c16) {
            chain[a] = e;
            continue;
        }
        const uint32_t s = load_id(g, a);
        const uint32_t sv = __ldg(g.rev + a);
        if (sv == kNoBack) continue;
        if (P.c16) {  // slot a = (v, affix): deg(v) of its owner v = N(s)[sv]
            const uint64_t fa = (uint64_t)load_node(g, s).off + sv;
            reinterpret_cast<uint16_t*>(P.c16)[fa] = (uint16_t)c16_enc(e, load_node(g, load_id(g, fa)).deg);
            continue;
        }
        uint32_t* rec = ac + ((uint64_t)load_node(g, s).off + sv) * rw;
        rec[chain_word_off(rw)] = e;
        if (rw == 8 && e < kLocked) {
            uint32_t lo = 0, hi = g.n;  // owner v of slot a
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if ((uint64_t)__ldg(&g.nodes[mid].off) <= a) lo = mid;
                else hi = mid;
            }
            const NodeRec r = load_node(g, lo);
            const SCtx c = make_ctx<KIND>(g, P.m, lo, (uint32_t)(a - (uint64_t)r.off));
            const uint32_t last = e & kIdxMask;
            const double wl = wprime<KIND>(g, P.m, c, last, load_node(g, load_id(g, c.off + last)).type, e >> 30);
            rec[6] = (uint32_t)__double2loint(wl);
            rec[7] = (uint32_t)__double2hiint(wl);
        }
    }
}

// Session arc records (walk.h ArcRec): word 0 = {id u, deg(u) | allpos << 31,
// off(u), chain word (second order) }, typed models add word 1 = {fp32
// weight, type(u) | edge_type(arc) << 16, 0, 0}. Warp per source node (its
// type gives the computed edge type, graph.hpp:47-50). k_ac_reset empties the
// chain words before a lazy run. rw = u32 words per record (2: narrow {u,
// chain word} records of node2vec). Typed records (rw 8): word 0 = {u,
// deg | allpos << 31, off, fp32 weight}, word 1 = {type(u) | edge_type << 16,
// chain word, w'(Last) as f64}.
__global__ void k_arc_chain(DevGraph g, uint4* __restrict__ out, uint32_t rw) {
    const uint32_t rs = rw / 4;
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = wid; v < g.n; v += nw) {
        const NodeRec rv = load_node(g, (uint32_t)v);
        for (uint32_t i = lane; i < rv.deg; i += 32) {
            const uint64_t a = (uint64_t)rv.off + i;
            const uint32_t u = load_id(g, a);
            if (rw == 2) {
                reinterpret_cast<uint2*>(out)[a] = make_uint2(u, kEmpty);
                continue;
            }
            const NodeRec r = load_node(g, u);
            const uint32_t dw = r.deg | ((r.flags & NF_ALLPOS) ? 0x80000000u : 0u);
            if (rs == 2) {
                const float w = g.w ? __ldg(g.w + a) : 1.0f;
                const uint32_t et = edge_type_of(g, a, rv.type, r.type);
                out[rs * a] = make_uint4(u, dw, (uint32_t)r.off, __float_as_uint(w));
                out[rs * a + 1] = make_uint4((uint32_t)r.type | (et << 16), kEmpty, 0u, 0u);
            } else {
                out[rs * a] = make_uint4(u, dw, (uint32_t)r.off, kEmpty);
            }
        }
    }
}

// 8-byte node records of the compact-chain walk: {off, deg | allpos << 31}
// (arcs < 2^32); half the L2 footprint of the 16-byte NodeRec.
__global__ void k_nodes8(DevGraph g, uint2* __restrict__ out) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += (uint64_t)gridDim.x * blockDim.x) {
        const NodeRec r = load_node(g, (uint32_t)v);
        out[v] = make_uint2((uint32_t)r.off, r.deg | ((r.flags & NF_ALLPOS) ? 0x80000000u : 0u));
    }
}

__global__ void k_ac_reset(uint32_t* __restrict__ ac, uint64_t m, uint32_t rw) {
    const uint32_t co = chain_word_off(rw);
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < m; a += (uint64_t)gridDim.x * blockDim.x)
        ac[a * rw + co] = kEmpty;
}

// Packed corpus: widen lengths for the 64-bit offset scan, then one warp per
// row copies the row (coalesced on both sides).
__global__ void k_len64(const uint32_t* __restrict__ lens, uint64_t rows, uint64_t* __restrict__ out) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= rows;
         r += (uint64_t)gridDim.x * blockDim.x)
        out[r] = r < rows ? lens[r] : 0;
}

__global__ void k_pack(const uint32_t* __restrict__ src, uint32_t stride, const uint64_t* __restrict__ off,
                       uint64_t rows, uint32_t* __restrict__ dst) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = wid; r < rows; r += nw) {
        const uint64_t o = off[r];
        const uint32_t len = (uint32_t)(off[r + 1] - o);
        const uint32_t* s = src + r * stride;
        for (uint32_t i = lane; i < len; i += 32) dst[o + i] = s[i];
    }
}

// Histogram of floor(log2 deg) over nodes of degree >= 1 (33 bins): with a
// power-of-two D, chain_replicas(d, D) depends on floor(log2 d) alone, so the
// host sizes the replica region for any D from it.
__global__ void k_deg_log2_hist(DevGraph g, const double* __restrict__ scale, unsigned long long* __restrict__ hist) {
    __shared__ unsigned int h[33];
    if (threadIdx.x < 33) h[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const NodeRec r = load_node(g, (uint32_t)v);
        const uint32_t d = rep_weight(r.deg, scale, r.type);
        if (d) atomicAdd(&h[31 - __clz(d)], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 33 && h[threadIdx.x]) atomicAdd(hist + threadIdx.x, (unsigned long long)h[threadIdx.x]);
}

// Replica groups per node (chain_replicas - 1).
__global__ void k_rep_counts(DevGraph g, uint32_t D, uint32_t cap, const double* __restrict__ scale,
                             uint32_t* __restrict__ cnt) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const NodeRec r = load_node(g, (uint32_t)v);
        cnt[v] = chain_replicas(rep_weight(r.deg, scale, r.type), D, cap) - 1;
    }
}

// Arcs incident to the nodes of each type (metapath2vec replica weights).
__global__ void k_type_arcs(DevGraph g, unsigned long long* __restrict__ out) {
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const NodeRec r = load_node(g, (uint32_t)v);
        if (r.deg) atomicAdd(out + r.type, (unsigned long long)r.deg);
    }
}

// Rows of valid starts on isolated nodes: [v], an early termination each.
__global__ void k_iso_rows(const uint32_t* __restrict__ iso, const uint64_t* __restrict__ iso_row,
                           uint32_t n_iso, uint32_t K, uint32_t* __restrict__ out, uint32_t stride,
                           uint32_t* __restrict__ lens) {
    const uint64_t total = (uint64_t)n_iso * K;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = t / K, k = t - j * K;
        const uint64_t row = iso_row[j] + k;
        out[row * stride] = iso[j];
        lens[row] = 1;
    }
}

// ------------------------------------------------- deterministic schedule
template <int KIND>
__global__ void k_det_setup(RunParams P, DetState S) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.n_items;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = i / P.cfg.K, k = i - j * P.cfg.K;
        const uint32_t v0 = P.act[j];
        S.v[i] = v0;
        S.aff[i] = KIND == METAPATH2VEC ? 0u : kNoAffix;
        S.len[i] = 1;
        S.alive[i] = 1;
        P.out[(P.act_row[j] + k) * P.stride] = v0;
    }
}

template <int KIND>
__global__ void k_det_propose(RunParams P, DetState S, uint32_t step, uint64_t invalid_key) {
    const uint2 wkey = philox_key(P.cfg.seed, DOM_WALK);
    unsigned long long inits = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.n_items;
         i += (uint64_t)gridDim.x * blockDim.x) {
        S.key[i] = invalid_key;
        S.idx[i] = (uint32_t)i;
        if (!S.alive[i]) continue;
        const SCtx c = make_ctx<KIND>(P.g, P.m, S.v[i], S.aff[i]);
        if (c.deg == 0) {
            S.chosen[i] = kDeadMark;
            continue;
        }
        const uint64_t j = i / P.cfg.K, k = i - j * P.cfg.K;
        const uint64_t walker = (uint64_t)P.act[j] * P.cfg.K + k;
        Draw d;
        d.open(wkey, walker, step);
        if (second_order(KIND) && c.boot) {
            uint32_t ch;
            S.chosen[i] = bootstrap_pick(P.g, c, d.unit(), &ch) ? ch : kDeadMark;
            continue;
        }
        const uint64_t slot = slot_of<KIND>(P.m, P.cfg, c, S.aff[i], walker);
        uint32_t e = __ldcg(P.chain + slot);
        if (e == kEmpty) {
            const uint32_t ie = init_slot<KIND>(P.g, P.m, P.cfg, c, slot);
            if (atomicCAS(P.chain + slot, kEmpty, ie) == kEmpty) ++inits;
        }
        const uint32_t cand = d.index(c.deg);
        const uint32_t uc = load_id(P.g, c.off + cand);
        const NodeRec rc = load_node(P.g, uc);
        const uint32_t cls = second_order(KIND) ? alpha_class(P.g, P.m, c, uc, &rc) : 0u;
        S.cand[i] = cand;
        S.ccls[i] = (uint8_t)cls;
        S.wc[i] = wprime<KIND>(P.g, P.m, c, cand, rc.type, cls);
        S.u[i] = d.unit();
        S.key[i] = slot;
    }
    if (inits) atomicAdd(&P.ctr[3], inits);
}

// One thread per run of equal slots: the sequential M-H chain in walker order.
template <int KIND>
__global__ void k_det_fold(RunParams P, DetState S, const uint64_t* __restrict__ keys,
                           const uint32_t* __restrict__ idx, uint64_t invalid_key) {
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P.n_items;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[p];
        if (key == invalid_key || (p > 0 && keys[p - 1] == key)) continue;
        uint32_t e = P.chain[key];
        const uint32_t i0 = idx[p];
        const SCtx c = make_ctx<KIND>(P.g, P.m, S.v[i0], S.aff[i0]);
        const uint32_t e0 = e;
        for (uint64_t q = p; q < P.n_items && keys[q] == key; ++q) {
            const uint32_t i = idx[q];
            if (e == kDead) {
                S.chosen[i] = kDeadMark;
                continue;
            }
            const uint32_t last = e & kIdxMask, cls_l = e >> 30;
            uint16_t ltype = 0;
            if (needs_utype<KIND>()) ltype = load_node(P.g, load_id(P.g, c.off + last)).type;
            const double wl = wprime<KIND>(P.g, P.m, c, last, ltype, cls_l);
            const uint32_t cand = S.cand[i];
            if (mh_accept(S.wc[i], wl, S.u[i]) && cand != last) {
                e = pack_entry(cand, S.ccls[i]);
                S.chosen[i] = cand;
            } else {
                S.chosen[i] = last;
            }
        }
        if (e != e0) P.chain[key] = e;
    }
}

template <int KIND>
__global__ void k_det_advance(RunParams P, DetState S) {
    unsigned long long steps = 0, early = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.n_items;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!S.alive[i]) continue;
        const uint32_t ch = S.chosen[i];
        if (ch == kDeadMark) {
            S.alive[i] = 0;
            ++early;
            continue;
        }
        const uint32_t v = S.v[i];
        const NodeRec r = load_node(P.g, v);
        const uint32_t next = load_id(P.g, r.off + ch);
        const uint64_t j = i / P.cfg.K, k = i - j * P.cfg.K;
        const uint64_t row = P.act_row[j] + k;
        P.out[row * P.stride + S.len[i]] = next;
        S.len[i] += 1;
        ++steps;
        if (KIND == DEEPWALK) {
            S.aff[i] = kNoAffix;
        } else if (KIND == METAPATH2VEC) {
            S.aff[i] = metapath_next(P.m, S.aff[i]);
        } else {
            const uint32_t back = __ldg(P.g.rev + r.off + ch);
            if (back == kNoBack) {
                fail_back_edge(P.ctr, next, v);
                S.alive[i] = 0;
                continue;
            }
            S.aff[i] = back;
        }
        S.v[i] = next;
    }
    if (steps) atomicAdd(&P.ctr[1], steps);
    if (early) atomicAdd(&P.ctr[2], early);
}

__global__ void k_det_finish(RunParams P, DetState S) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.n_items;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = i / P.cfg.K, k = i - j * P.cfg.K;
        P.lens[P.act_row[j] + k] = S.len[i];
    }
}

// --------------------------------------------------------- parity kernels
template <int KIND>
__global__ void k_decide(DevGraph g, DevModel m, uint64_t n, const uint32_t* __restrict__ pos,
                         const uint32_t* __restrict__ aff, const uint32_t* __restrict__ cand,
                         const uint32_t* __restrict__ last, const double* __restrict__ u,
                         double* __restrict__ wc, double* __restrict__ wl, uint8_t* __restrict__ acc,
                         unsigned* __restrict__ bad, int hastings) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = pos[i], a = aff[i];
        bool ok = v < g.n;
        if (ok) {
            const uint32_t deg = load_node(g, v).deg;
            ok = cand[i] < deg && last[i] < deg;
            if (KIND == METAPATH2VEC) ok = ok && a < m.mp_len;
            if (second_order(KIND)) ok = ok && (a == kNoAffix || a < deg);
        }
        if (!ok) {
            atomicAdd(bad, 1u);
            acc[i] = 2;
            continue;
        }
        const SCtx c = make_ctx<KIND>(g, m, v, a);
        if (hastings) {  // alias proposal: (r_c, r_l, Hastings accept)
            const double x = eval_rfactor<KIND>(g, m, c, cand[i]);
            const double y = eval_rfactor<KIND>(g, m, c, last[i]);
            wc[i] = x;
            wl[i] = y;
            acc[i] = hastings_accept(static_w(g, c.off + cand[i]), x, y, u[i]) ? 1 : 0;
            continue;
        }
        uint32_t cls;
        const double x = eval_index<KIND>(g, m, c, cand[i], &cls);
        const double y = eval_index<KIND>(g, m, c, last[i], &cls);
        wc[i] = x;
        wl[i] = y;
        acc[i] = mh_accept(x, y, u[i]) ? 1 : 0;
    }
}

template <int KIND>
__global__ void k_init_states(DevGraph g, DevModel m, DevCfg cfg, uint64_t n, const uint32_t* __restrict__ pos,
                              const uint32_t* __restrict__ aff, uint32_t* __restrict__ out,
                              unsigned* __restrict__ bad) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = pos[i], a = aff[i];
        bool ok = v < g.n;
        if (ok) {
            const uint32_t deg = load_node(g, v).deg;
            if (KIND == METAPATH2VEC) ok = a < m.mp_len;
            if (second_order(KIND)) ok = a < deg;
        }
        if (!ok) {
            atomicAdd(bad, 1u);
            out[i] = kNoAffix;
            continue;
        }
        const SCtx c = make_ctx<KIND>(g, m, v, a);
        const uint32_t e = init_slot<KIND>(g, m, cfg, c, slot_of<KIND>(m, cfg, c, a, 0));
        out[i] = e == kDead ? kNoAffix : (e & kIdxMask);
    }
}

// cmd_check's per-state chain audit (tools/mhwalk.cpp:222-247), one warp per
// state: the warp evaluates the state's w' table once, then runs the chain 32
// draws at a time -- lanes draw and look up their proposals in parallel, the
// fold over the 32 is done by every lane in lockstep through shuffles, each
// lane records the chain state after its own draw. Same Philox layout as
// og_check: init keyed by slot = state index, draw d from block (j, d).
constexpr uint32_t DOM_CHECK = 0xC4EC0005u;

template <int KIND>
__global__ void k_check(DevGraph g, DevModel m, DevCfg cfg, uint64_t n, const uint32_t* __restrict__ pos,
                        const uint32_t* __restrict__ aff, const uint64_t* __restrict__ base, uint64_t draws,
                        double* __restrict__ W, unsigned long long* __restrict__ counts, double* __restrict__ kl) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint2 key = philox_key(cfg.seed, DOM_CHECK);
    for (uint64_t j = wid; j < n; j += nw) {
        const SCtx c = make_ctx<KIND>(g, m, pos[j], aff[j]);
        double* w = W + base[j];
        unsigned long long* cnt = counts + base[j];
        for (uint32_t i = lane; i < c.deg; i += 32) {
            uint32_t cls;
            w[i] = eval_index<KIND>(g, m, c, i, &cls);
            cnt[i] = 0;
        }
        __syncwarp();
        double total = 0.0;
        for (uint32_t i = 0; i < c.deg; ++i) total = __dadd_rn(total, w[i]);
        if (!(total > 0)) {
            if (lane == 0) kl[j] = __longlong_as_double(0x7FF8000000000000ll);
            continue;
        }
        const uint32_t e = init_slot<KIND>(g, m, cfg, c, j);  // every lane: same value
        if (e == kDead) {
            if (lane == 0) kl[j] = __longlong_as_double(0x7FF8000000000000ll);
            continue;
        }
        uint32_t last = e & kIdxMask;
        double wl = w[last];
        for (uint64_t d0 = 0; d0 < draws; d0 += 32) {
            const uint64_t d = d0 + lane;
            uint32_t cand = 0;
            double wc = 0.0, u = 1.0;
            if (d < draws) {
                Draw dr;
                dr.open(key, j, (uint32_t)d);
                cand = dr.index(c.deg);
                u = dr.unit();
                wc = w[cand];
            }
            const uint32_t steps = draws - d0 < 32 ? (uint32_t)(draws - d0) : 32u;
            uint32_t mine = 0;
            for (uint32_t t = 0; t < steps; ++t) {
                const uint32_t ct = __shfl_sync(0xffffffffu, cand, t);
                const double wct = __shfl_sync(0xffffffffu, wc, t);
                const double ut = __shfl_sync(0xffffffffu, u, t);
                if (mh_accept(wct, wl, ut)) {
                    last = ct;
                    wl = wct;
                }
                if (t == lane) mine = last;
            }
            if (lane < steps) atomicAdd(cnt + mine, 1ull);
        }
        __syncwarp();
        if (lane == 0) {
            double k = 0.0;
            for (uint32_t i = 0; i < c.deg; ++i) {
                const double p = (double)cnt[i] / (double)draws;
                if (p == 0.0) continue;
                k += p * log(p / (w[i] / total));
            }
            kl[j] = k;
        }
    }
}

__global__ void k_state_degrees(DevGraph g, const uint32_t* __restrict__ pos, uint64_t n, uint64_t* __restrict__ d) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= n;
         j += (uint64_t)gridDim.x * blockDim.x)
        d[j] = j < n ? load_node(g, pos[j]).deg : 0;
}

// Session setup: classify start nodes of [b, e), or of the list ids[0, e - b)
// when ids is given.
__global__ void k_classify(DevGraph g, DevModel m, uint32_t b, uint32_t e, uint8_t* __restrict__ valid,
                           uint8_t* __restrict__ act, uint8_t* __restrict__ iso, const uint32_t* __restrict__ ids = nullptr) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (uint64_t)(e - b);
         t += (uint64_t)gridDim.x * blockDim.x) {
        const NodeRec r = load_node(g, ids ? ids[t] : (uint32_t)(b + t));
        const bool ok = m.kind != METAPATH2VEC || r.type == m.metapath[0];  // initial_state, models.cpp:138-144
        valid[t] = ok;
        act[t] = ok && r.deg > 0;
        iso[t] = ok && r.deg == 0;
    }
}

__global__ void k_iota_from(uint32_t* p, uint32_t n, uint32_t base) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = base + (uint32_t)i;
}

// pos: positions in the start list (selected by flag); nodes[i] = ids[pos[i]],
// rows[i] = first corpus row of that start (rank of its position among the
// valid starts, times K).
__global__ void k_rows_of(uint32_t* __restrict__ nodes, uint32_t n, const uint32_t* __restrict__ ids,
                          const uint32_t* __restrict__ rank, uint32_t K, uint64_t* __restrict__ rows) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = nodes[i];
        rows[i] = (uint64_t)rank[p] * K;
        nodes[i] = ids[p];
    }
}

int sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

unsigned grid_for(uint64_t work, int block = 256) {
    const uint64_t g = (work + block - 1) / block;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, (uint64_t)sms() * 16));
}

// Register-cap variant of the walk kernel (occupancy vs spills trade-off);
// MHW_WALK_REGS selects it at session creation. Defaults from the A/B runs of
// scripts/exp_regs.sh: deepwalk 80; node2vec uncapped
// (a 64-register cap, 4 blocks/SM: cfg2 36.8 vs 34.6 ms, no spills either way);
// eagerly initialised edge2vec / fairwalk 80.
int walk_minb(int kind, bool eager) {
    const char* e = std::getenv("MHW_WALK_REGS");
    // deepwalk: 80; eagerly initialised edge2vec / fairwalk: 80 (84-86 -> 80
    // registers without spills lifts occupancy from 2 to 3 blocks/SM: cfg3b
    // 99.5 -> 94.3 ms, cfg4 181 -> 176 ms); their lazy variants would spill.
    // metapath2vec (lazily initialised, 120 registers = 2 blocks/SM): the cap
    // spills 56 bytes, all in the first-touch init path: cfg3a 48.45 -> 45.2
    // ms at 80 (64: 48.75)
    const bool cap = kind == DEEPWALK || kind == METAPATH2VEC || (eager && (kind == EDGE2VEC || kind == FAIRWALK));
    const int v = e ? std::atoi(e) : (cap ? 80 : 255);
    return v == 64 ? 64 : (v == 80 ? 80 : 255);
}

// Calls f(REGS, LAZY, AR) with the compile-time variant of the session
// (ar: 0 none, 1 records, 2 narrow node2vec records).
template <int KIND, class F>
void with_variant(int regs, bool lazy, int ar, F&& f) {
    using T = std::true_type;
    using N = std::false_type;
    auto by_regs = [&](auto lz, auto a) {
        if (regs == 80) f(std::integral_constant<int, 80>{}, lz, a);
        else if (regs == 64) f(std::integral_constant<int, 64>{}, lz, a);
        else f(std::integral_constant<int, 255>{}, lz, a);
    };
    auto by_ar = [&](auto lz) {
        if constexpr (KIND == NODE2VEC) {
            if (ar == 2) {
                by_regs(lz, std::integral_constant<int, 2>{});
                return;
            }
            if (ar == 3) {
                if constexpr (!decltype(lz)::value) by_regs(lz, std::integral_constant<int, 3>{});
                else invalid("compact chain tables need eager initialisation");
                return;
            }
        }
        if (ar == 4) by_regs(lz, std::integral_constant<int, 4>{});
        else if (ar == 5) by_regs(lz, std::integral_constant<int, 5>{});
        else if (ar) by_regs(lz, std::integral_constant<int, 1>{});
        else by_regs(lz, std::integral_constant<int, 0>{});
    };
    if (lazy) by_ar(T{});
    else by_ar(N{});
}

template <int KIND, int REGS, bool LAZY, int AR>
int walk_grid() {
    int per_sm = 0;
    // MHW_CARVEOUT: preferred shared-memory carve-out in percent (experiment; the
    // kernel's own need, 9-17 KB per block for the row staging, is honoured)
    if (const char* cv = std::getenv("MHW_CARVEOUT"))
        MHW_CK(cudaFuncSetAttribute(k_walk<KIND, REGS, LAZY, AR>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    std::atoi(cv)));
    MHW_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_walk<KIND, REGS, LAZY, AR>, kWalkBlock, 0));
    return std::max(1, per_sm) * sms();
}

template <class F>
void dispatch(int kind, F&& f) {
    switch (kind) {
        case DEEPWALK: f(std::integral_constant<int, DEEPWALK>{}); break;
        case NODE2VEC: f(std::integral_constant<int, NODE2VEC>{}); break;
        case METAPATH2VEC: f(std::integral_constant<int, METAPATH2VEC>{}); break;
        case EDGE2VEC: f(std::integral_constant<int, EDGE2VEC>{}); break;
        case FAIRWALK: f(std::integral_constant<int, FAIRWALK>{}); break;
        default: invalid("unknown model kind");
    }
}

template <class T>
void select_flagged(const T* in, const uint8_t* flags, T* out, uint32_t n, uint32_t* count, cudaStream_t st) {
    DBuf<int64_t> d_cnt(1);
    size_t bytes = 0;
    MHW_CK(cub::DeviceSelect::Flagged(nullptr, bytes, in, flags, out, d_cnt.p, (int64_t)n, st));
    DBuf<uint8_t> temp(std::max<size_t>(bytes, 1));
    MHW_CK(cub::DeviceSelect::Flagged(temp.p, bytes, in, flags, out, d_cnt.p, (int64_t)n, st));
    int64_t h = 0;
    MHW_CK(cudaMemcpyAsync(&h, d_cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    *count = (uint32_t)h;
}

}  // namespace

// ----------------------------------------------------------- model bind
void model_bind(Model& mb, Graph& g, const mhw_model_desc& d) {
    DeviceGuard dg(g.device);
    mb.desc = d;
    const int k = d.kind;
    if (k < DEEPWALK || k > FAIRWALK) invalid("unknown model: " + std::to_string(k));
    static const char* names[] = {"deepwalk", "node2vec", "metapath2vec", "edge2vec", "fairwalk"};
    // WalkModel::bind, models.cpp:29-74
    if (second_order(k)) {
        if (!(d.p > 0) || !(d.q > 0)) invalid("p and q must be positive");
        if (!g.symmetric) invalid(std::string(names[k]) + " requires a symmetric graph (load with symmetrize)");
    }
    if ((k == METAPATH2VEC || k == FAIRWALK || k == EDGE2VEC) && !g.has_ntypes())
        invalid(std::string(names[k]) + " requires node types");
    DevModel& m = mb.dev;
    m = DevModel{};
    m.kind = k;
    m.inv_p = 1.0 / d.p;
    m.inv_q = 1.0 / d.q;
    m.alpha_trivial = (m.inv_p == 1.0 && m.inv_q == 1.0) ? 1 : 0;
    {
        const double a[3] = {m.inv_p, 1.0, m.inv_q};
        const int h = a[0] >= a[1] ? (a[0] >= a[2] ? 0 : 2) : (a[1] >= a[2] ? 1 : 2);
        const bool unique = (h == 0 || a[0] < a[h]) && (h == 1 || a[1] < a[h]) && (h == 2 || a[2] < a[h]);
        m.spec_cls = (!m.alpha_trivial && unique) ? (uint32_t)h : 3u;
    }
    m.ret_wmax = std::max(1.0, m.inv_q);
    m.ret_skip = (k == NODE2VEC && !m.alpha_trivial && !g.w.n && m.ret_wmax < m.inv_p) ? 1 : 0;
    if (const char* rs = std::getenv("MHW_RET_SKIP")) m.ret_skip = m.ret_skip && rs[0] != '0';
    m.num_types = g.n_ntypes;
    if (k == METAPATH2VEC) {
        if (d.metapath_len < 2 || !d.metapath) invalid("metapath needs at least 2 types");
        for (uint32_t i = 0; i < d.metapath_len; ++i)
            if (d.metapath[i] >= g.n_ntypes) invalid("metapath type " + std::to_string(d.metapath[i]) + " not in graph");
        mb.h_metapath.assign(d.metapath, d.metapath + d.metapath_len);
        mb.metapath.alloc(d.metapath_len);
        MHW_CK(cudaMemcpy(mb.metapath.p, d.metapath, d.metapath_len * 2, cudaMemcpyHostToDevice));
        m.metapath = mb.metapath.p;
        m.mp_len = d.metapath_len;
        graph_ensure_typed_index(g);  // O(1) random_positive for slot inits
    }
    if (k == EDGE2VEC) {
        const uint32_t dim = g.etype.n ? g.n_etypes : (uint32_t)(g.n_ntypes * g.n_ntypes);
        if (d.type_matrix_dim != dim || !d.type_matrix)
            invalid("edge type matrix must be " + std::to_string(dim) + "x" + std::to_string(dim));
        bool allpos = true;
        for (uint32_t i = 0; i < dim * dim; ++i) {
            if (d.type_matrix[i] < 0) invalid("edge type matrix entries must be non-negative");
            if (!(d.type_matrix[i] > 0)) allpos = false;
        }
        mb.M.alloc((size_t)dim * dim);
        MHW_CK(cudaMemcpy(mb.M.p, d.type_matrix, (size_t)dim * dim * sizeof(double), cudaMemcpyHostToDevice));
        m.M = mb.M.p;
        m.M_dim = dim;
        m.M_allpos = allpos ? 1 : 0;
    }
    if (second_order(k)) {
        // node2vec graphs that take the compact chain table (2 * arcs <= 96 MB,
        // node table <= 32 MB) get a 3-bit-per-arc edge filter: its 11.8 MB
        // leave more L2 beside the pinned 63 MB table (cfg2 walk 23.48 ->
        // 22.66 ms, init 4.76 -> 5.0; 2 bits: 23.41 / 5.58, 8 bits: 25.67 / 4.69)
        const bool c16_graph = k == NODE2VEC && 2ull * g.m <= (96ull << 20) && 16ull * g.n <= (32ull << 20);
        graph_ensure_second_order(g, !m.alpha_trivial, c16_graph ? 3u : 4u);
    }
    if (k == FAIRWALK) graph_ensure_tcount(g);
}

// ------------------------------------------------------------- sessions
// The persisting-L2 set-aside is a device-wide limit: the first session that
// raises it saves the previous value, the last one to go restores it and
// resets the persisting lines (nothing may outlive the sessions).
namespace {
std::mutex g_l2_mu;
int g_l2_users[64] = {};
size_t g_l2_saved[64] = {};

void l2_limit_acquire(int dev, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_l2_mu);
    // MHW_L2_PERSIST_MB: set-aside size override (experiment: slack above the window size)
    if (const char* e = std::getenv("MHW_L2_PERSIST_MB")) bytes = (size_t)std::atoll(e) << 20;
    size_t cur = 0;
    MHW_CK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
    if (g_l2_users[dev & 63]++ == 0) g_l2_saved[dev & 63] = cur;
    if (cur < bytes) MHW_CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes));
}

void l2_limit_release(int dev) {
    std::lock_guard<std::mutex> lk(g_l2_mu);
    if (g_l2_users[dev & 63] == 0 || --g_l2_users[dev & 63] != 0) return;
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_l2_saved[dev & 63]);
}
}  // namespace

Session::~Session() {
    if (l2_pin && g) {
        DeviceGuard dg(g->device);
        l2_limit_release(g->device);
    }
    if (ev0) cudaEventDestroy(ev0);
    if (evm) cudaEventDestroy(evm);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
}

static std::vector<double> metapath_rep_scale(const std::vector<uint16_t>& mp, const Graph& g, cudaStream_t st);

// Start-node lists of a session: the valid starts among ids[0, span) (device
// list, ascending) in list order (initial_state, models.cpp:138-144), split
// into active (degree > 0) and isolated starts, with their first corpus
// rows; rows, skipped and n_items follow (engine.cpp:187-191).
static void session_classify_starts(Session& s, const uint32_t* d_ids, uint32_t span) {
    cudaStream_t st = s.stream;
    const DevGraph gv = s.g->view();
    uint32_t n_valid = 0;
    s.n_act = s.n_iso = 0;
    if (span) {
        DBuf<uint8_t> valid(span), act(span), iso(span);
        DBuf<uint32_t> rank(span + 1), pos(span);
        k_classify<<<grid_for(span), 256, 0, st>>>(gv, s.model.dev, 0, span, valid.p, act.p, iso.p, d_ids);
        k_iota_from<<<grid_for(span), 256, 0, st>>>(pos.p, span, 0);
        MHW_CK(cudaGetLastError());
        size_t bytes = 0;
        MHW_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, valid.p, rank.p, (int64_t)span, st));
        DBuf<uint8_t> temp(std::max<size_t>(bytes, 1));
        MHW_CK(cub::DeviceScan::ExclusiveSum(temp.p, bytes, valid.p, rank.p, (int64_t)span, st));
        uint32_t last_rank = 0;
        uint8_t last_valid = 0;
        MHW_CK(cudaMemcpyAsync(&last_rank, rank.p + span - 1, 4, cudaMemcpyDeviceToHost, st));
        MHW_CK(cudaMemcpyAsync(&last_valid, valid.p + span - 1, 1, cudaMemcpyDeviceToHost, st));
        MHW_CK(cudaStreamSynchronize(st));
        n_valid = last_rank + last_valid;
        if (s.act.n < span) s.act.alloc(span);
        if (s.iso.n < span) s.iso.alloc(span);
        select_flagged(pos.p, act.p, s.act.p, span, &s.n_act, st);
        select_flagged(pos.p, iso.p, s.iso.p, span, &s.n_iso, st);
        if (s.act_row.n < std::max<uint32_t>(s.n_act, 1)) s.act_row.alloc(std::max<uint32_t>(s.n_act, 1));
        if (s.iso_row.n < std::max<uint32_t>(s.n_iso, 1)) s.iso_row.alloc(std::max<uint32_t>(s.n_iso, 1));
        if (s.n_act) k_rows_of<<<grid_for(s.n_act), 256, 0, st>>>(s.act.p, s.n_act, d_ids, rank.p, s.cfg.K, s.act_row.p);
        if (s.n_iso) k_rows_of<<<grid_for(s.n_iso), 256, 0, st>>>(s.iso.p, s.n_iso, d_ids, rank.p, s.cfg.K, s.iso_row.p);
        MHW_CK(cudaGetLastError());
        MHW_CK(cudaStreamSynchronize(st));
    }
    s.rows = (uint64_t)n_valid * s.cfg.K;
    s.skipped = (uint64_t)(span - n_valid) * s.cfg.K;
    s.n_items = (uint64_t)s.n_act * s.cfg.K;
}

void session_select_starts(Session& s, uint32_t count, const uint32_t* starts) {
    DeviceGuard dg(s.g->device);
    if (count && !starts) invalid("starts must not be NULL");
    for (uint32_t i = 0; i < count; ++i) {
        if (starts[i] < s.node_begin || starts[i] >= s.node_end) invalid("start node outside the session's node range");
        if (i && starts[i] <= starts[i - 1]) invalid("start nodes must be strictly ascending");
    }
    DBuf<uint32_t> ids(std::max<uint32_t>(count, 1));
    if (count) MHW_CK(cudaMemcpyAsync(ids.p, starts, count * 4ull, cudaMemcpyHostToDevice, s.stream));
    if (!count && !starts) {  // back to the whole node range
        const uint32_t span = s.node_end - s.node_begin;
        ids.alloc(std::max<uint32_t>(span, 1));
        if (span) k_iota_from<<<grid_for(span), 256, 0, s.stream>>>(ids.p, span, s.node_begin);
        MHW_CK(cudaGetLastError());
        count = span;
    }
    session_classify_starts(s, ids.p, count);
    if (s.rows > s.rows_cap || s.n_items > s.items_cap) invalid("start selection larger than the session");
}

void session_create(Session& s, Graph& g, const mhw_model_desc& md, const mhw_walk_config& wc) {
    DeviceGuard dg(g.device);
    if (wc.walks_per_node == 0 || wc.walk_length == 0)
        invalid("walks_per_node, walk_length and threads must be positive");
    if (wc.sampler < 0 || wc.sampler > 3) invalid("unknown sampler kind");
    if (wc.init_kind < 0 || wc.init_kind > 2) invalid("unknown init strategy");
    if (wc.schedule < 0 || wc.schedule > 1) invalid("unknown schedule");
    if (wc.proposal < 0 || wc.proposal > 1) invalid("unknown proposal");
    if (wc.proposal == MHW_PROPOSAL_ALIAS && wc.sampler != MHW_SAMPLER_MH)
        invalid("the alias proposal applies to the mh sampler only");
    if (wc.proposal == MHW_PROPOSAL_ALIAS && wc.schedule == MHW_SCHEDULE_DETERMINISTIC)
        invalid("the alias proposal runs on the throughput schedule only");
    s.g = &g;
    s.wc = wc;
    const bool trace = std::getenv("MHW_TRACE") != nullptr;
    const auto tc0 = std::chrono::steady_clock::now();
    auto tms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tc0).count(); };
    model_bind(s.model, g, md);
    const double t_bind = trace ? (cudaDeviceSynchronize(), tms()) : 0.0;
    const DevModel& m = s.model.dev;
    s.cfg.seed = wc.seed;
    s.cfg.K = wc.walks_per_node;
    s.cfg.L = wc.walk_length;
    s.cfg.init_kind = wc.init_kind;
    s.cfg.burn_in = wc.burn_in_steps;
    s.cfg.hw = wc.hw_sample_size;
    s.cfg.proposal = wc.proposal;
    s.node_begin = wc.node_begin;
    s.node_end = wc.node_end ? wc.node_end : g.n;
    if (s.node_end > g.n || s.node_begin > s.node_end) invalid("node range out of bounds");
    s.stride = (wc.walk_length + 1 + 3) & ~3u;
    MHW_CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    MHW_CK(cudaEventCreate(&s.ev0));
    MHW_CK(cudaEventCreate(&s.evm));
    MHW_CK(cudaEventCreate(&s.ev1));
    cudaStream_t st = s.stream;
    // slot layout (manager.cpp:14-21): base slots, then hub replicas for
    // node-keyed models
    s.slots = k_slots(m.kind, g);
    s.cfg.rep_deg = kNoReplicas;
    s.cfg.rep_max = kMaxReplicas;
    s.cfg.rep_base_slot = s.slots;
    s.cfg.rep_group = nullptr;
    s.cfg.rep_scale = nullptr;
    if (!second_order(m.kind) && wc.chain_replica_degree != kNoReplicas && g.n && g.max_deg) {
        const uint64_t G = m.kind == METAPATH2VEC ? g.n_ntypes : 1;
        if (m.kind == METAPATH2VEC) {
            // visit scale per node type (rep_weight): share of the metapath's
            // steady cycle spent at type t, times arcs / arcs incident to t
            const std::vector<double> F = metapath_rep_scale(s.model.h_metapath, g, st);
            s.rep_scale.alloc(F.size());
            MHW_CK(cudaMemcpyAsync(s.rep_scale.p, F.data(), F.size() * sizeof(double), cudaMemcpyHostToDevice, st));
            s.cfg.rep_scale = s.rep_scale.p;
        }
        // replica groups for power-of-two D from the log2-weight histogram
        DBuf<unsigned long long> hist(33);
        MHW_CK(cudaMemsetAsync(hist.p, 0, 33 * 8, st));
        k_deg_log2_hist<<<grid_for(g.n), 256, 0, st>>>(g.view(), s.cfg.rep_scale, hist.p);
        MHW_CK(cudaGetLastError());
        unsigned long long hh[33];
        MHW_CK(cudaMemcpyAsync(hh, hist.p, sizeof hh, cudaMemcpyDeviceToHost, st));
        MHW_CK(cudaStreamSynchronize(st));
        auto groups_for = [&](uint32_t lgD) {
            uint64_t t = 0;
            for (uint32_t b = lgD; b < 33; ++b) {
                const uint64_t r = std::min<uint64_t>(uint64_t(2) << (b - lgD), s.cfg.rep_max);
                t += hh[b] * (r - 1);
            }
            return t;
        };
        uint32_t D = wc.chain_replica_degree;
        if (!D) {
            // auto: metapath2vec replicates states whose visit weight
            // (rep_weight: degree scaled by how often the metapath visits
            // the node's type) reaches kDefaultRepDeg = 32 (cfg3a: the V
            // venues; D = 128 59.2 ms, 32 54.0, 16 56.1, 8 60.2 -- each
            // replica's lazy init scans the typed neighbours); deepwalk
            // takes the smallest power-of-two D whose replica region fits
            // kAutoReplicaSlots (L2-resident chain table)
            D = kDefaultRepDeg;
            if (m.kind == DEEPWALK)
                for (uint32_t lg = 0; lg < 31; ++lg)
                    if (groups_for(lg) * G <= kAutoReplicaSlots) { D = 1u << lg; break; }
        }
        if ((D & (D - 1)) == 0) {
            uint32_t lg = 0;
            while ((1u << lg) != D) ++lg;
            if (groups_for(lg) > 0xFFFFFFFEull)
                invalid("sampler layout too large: chain_replica_degree " + std::to_string(D) + " gives " +
                        std::to_string(groups_for(lg)) + " replica groups");
        }
        uint32_t top = 0;  // highest occupied log2-weight bin
        for (uint32_t b = 0; b < 33; ++b)
            if (hh[b]) top = b;
        if (((uint64_t(2) << top) - 1) >= D) {
            DBuf<uint32_t> cnt(g.n + 1);
            s.rep_group.alloc(g.n + 1);
            MHW_CK(cudaMemsetAsync(cnt.p, 0, (g.n + 1) * 4, st));
            k_rep_counts<<<grid_for(g.n), 256, 0, st>>>(g.view(), D, s.cfg.rep_max, s.cfg.rep_scale, cnt.p);
            MHW_CK(cudaGetLastError());
            size_t bytes = 0;
            MHW_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, s.rep_group.p, (int64_t)g.n + 1, st));
            DBuf<uint8_t> temp(std::max<size_t>(bytes, 1));
            MHW_CK(cub::DeviceScan::ExclusiveSum(temp.p, bytes, cnt.p, s.rep_group.p, (int64_t)g.n + 1, st));
            uint32_t groups = 0;
            MHW_CK(cudaMemcpyAsync(&groups, s.rep_group.p + g.n, 4, cudaMemcpyDeviceToHost, st));
            MHW_CK(cudaStreamSynchronize(st));
            s.cfg.rep_deg = D;
            s.cfg.rep_group = s.rep_group.p;
            s.slots += (uint64_t)groups * G;
        }
    }
    if (s.slots > (uint64_t(1) << 40)) invalid("sampler layout too large: " + std::to_string(s.slots) + " slots");
    {
        const uint32_t span = s.node_end - s.node_begin;
        DBuf<uint32_t> ids(std::max<uint32_t>(span, 1));
        if (span) k_iota_from<<<grid_for(span), 256, 0, st>>>(ids.p, span, s.node_begin);
        MHW_CK(cudaGetLastError());
        session_classify_starts(s, ids.p, span);
    }
    s.rows_cap = s.rows;
    s.items_cap = s.n_items;
    const double t_starts = trace ? tms() : 0.0;
    s.out.alloc(std::max<uint64_t>(s.rows * s.stride, 4));
    s.lens.alloc(std::max<uint64_t>(s.rows, 1));
    s.ctr.alloc(8);
    if (trace) std::fprintf(stderr, "[mhw] session_create: starts at %.2f ms, walk buffer at %.2f ms\n", t_starts, tms());
    if (wc.sampler != MHW_SAMPLER_MH) {
        // exact baselines: no chains; Philox-keyed draws make any schedule
        // deterministic
        s.chain.alloc(1);
        s.ex = std::make_unique<ExactState>();
        exact_create(s);
    } else if (wc.schedule == MHW_SCHEDULE_DETERMINISTIC) {
        s.chain.alloc(std::max<uint64_t>(s.slots, 1));
        const uint64_t n = std::max<uint64_t>(s.n_items, 1);
        if (s.n_items > 0xFFFFFFFFull) invalid("deterministic schedule supports at most 2^32 walkers");
        s.d_v.alloc(n);
        s.d_aff.alloc(n);
        s.d_len.alloc(n);
        s.d_alive.alloc(n);
        s.d_key.alloc(n);
        s.d_key2.alloc(n);
        s.d_idx.alloc(n);
        s.d_idx2.alloc(n);
        s.d_cand.alloc(n);
        s.d_ccls.alloc(n);
        s.d_wc.alloc(n);
        s.d_u.alloc(n);
        s.d_chosen.alloc(n);
        int bits = 1;
        while (bits < 64 && ((s.slots) >> bits) != 0) ++bits;
        s.sort_bits = bits;
        size_t bytes = 0;
        MHW_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, s.d_key.p, s.d_key2.p, s.d_idx.p, s.d_idx2.p,
                                               (int64_t)n, 0, bits, st));
        s.sort_temp.alloc(std::max<size_t>(bytes, 1));
    } else {
        // Eager slot init when walks will touch most arc-keyed slots anyway
        // (identical chain values: init randomness is slot-keyed).
        // Eager init order: record order builds each state from its own
        // (coalesced) session record, slot order keeps a warp on one N(v)
        // (burn-in draws ~11 candidates from it). Record order where the
        // records carry deg/off (wide or typed) and init draws few
        // candidates: cfg5 (random init, wide records) 1105 ms lazy, 1137
        // eager in slot order, 1066 in record order; cfg2 (burn-in, narrow
        // records) 34.6 slot vs 35.6 record. With the cheaper record-order
        // init, eager pays from 2 walker steps per slot (cfg5: 5) instead of 8.
        const char* io = std::getenv("MHW_INIT_ORDER");
        const char* nw0 = std::getenv("MHW_NARROW");
        const bool narrow_pred = m.kind == NODE2VEC && (nw0 ? nw0[0] == '1' : 16ull * g.n <= (32ull << 20));
        const bool rec_pred = io ? io[0] == 'r' : (!narrow_pred && s.cfg.init_kind != INIT_BURN_IN);
        // With the per-arc source array (s.src, graphs up to 2^28 arcs) the
        // slot-order init needs no owner search and beats record order there
        // too: cfg4 init 12.66 -> 11.6 ms, cfg3b 1.56 -> 1.32 (cfg5, 2.08 G
        // arcs, no source array: slot order 198 vs 136 ms)
        const char* se0 = std::getenv("MHW_ARC_SRC");
        const bool src_ok = g.m < (1ull << 28) && !(se0 && se0[0] == '0');
        s.init_rec_order = io ? rec_pred : (rec_pred && !src_ok);
        const bool dense = (double)s.n_items * s.cfg.L >= (rec_pred ? 2.0 : 8.0) * (double)s.slots;
        s.eager_init = second_order(m.kind) && (wc.init_mode == 2 || (wc.init_mode == 0 && dense));
        s.minb = walk_minb(m.kind, s.eager_init);
        // pin an L2-sized edge filter (<= 32 MB by construction) in L2
        // (cfg2: 16 MB, +3%; cfg4: 32 MB, 174.3 -> 167.5 ms; a 64 MB window
        // starves the rest of the working set: cfg4 -30%)
        // fairwalk with p = q = 1 has no alpha test (no filter): its per-
        // (node, type) group sizes, read for every candidate, take the window
        void* pin_p = nullptr;
        size_t pin_bytes = 0;
        if (g.bloom.n && !m.alpha_trivial) {
            pin_p = g.bloom.p;
            pin_bytes = g.bloom.bytes();
        } else if (m.kind == FAIRWALK && g.tcount.n) {
            pin_p = g.tcount.p;
            pin_bytes = g.tcount.bytes();
        }
        const char* pe = std::getenv("MHW_L2_PIN");
        const bool pin_ok = !(pe && pe[0] == '0');
        auto try_pin = [&](void* p, size_t bytes) {
            if (!pin_ok || !p || bytes > (33ull << 20)) return;
            int dev = 0, max_persist = 0;
            MHW_CK(cudaGetDevice(&dev));
            MHW_CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
            if ((size_t)max_persist >= bytes) {
                l2_limit_acquire(dev, bytes);
                s.l2_pin = true;
                s.pin_p = p;
                s.pin_bytes = bytes;
            }
        };
        try_pin(pin_p, pin_bytes);
        // arc records (after the session buffers, so the memory check sees them)
        const char* ar_env = std::getenv("MHW_ARC_RECORDS");
        // the alias proposal walks the plain CSR (k_walk AR = 4) with the
        // graph's static alias tables
        const bool alias_prop = wc.proposal == MHW_PROPOSAL_ALIAS;
        if (alias_prop) graph_ensure_static_alias(g);
        const bool want_ar = !(ar_env && ar_env[0] == '0');
        // node2vec compact chains (AR 3): 16-bit words in their own table when
        // it and the node table fit L2 (MHW_C16=0/1 forces)
        const char* c16e = std::getenv("MHW_C16");
        const bool c16_ok = !alias_prop && m.kind == NODE2VEC && s.eager_init && g.verified_sym && g.m && g.m < (1ull << 32) &&
                            g.max_deg <= 0xFFFDu && want_ar;
        const bool c16_want = c16_ok && (c16e ? c16e[0] == '1' : (2ull * g.m <= (96ull << 20) && 16ull * g.n <= (32ull << 20)));
        if (c16_want) {
            // MHW_C16_PIN: chain (default: the 16-bit table pinned for the
            // walk, the edge filter for the eager init) | filter | both
            // ([c16 | filter copy], one window) | none. cfg2 walk + init:
            // chain 27.65 + 5.3 ms, both 27.1 + 6.8-9.5, filter 31.6 + 4.7,
            // none 32.8 + 4.7; narrow records 29.5 + 4.7
            const char* pm = std::getenv("MHW_C16_PIN");
            const std::string mode = pm ? pm : "chain";
            const uint64_t cw = (g.m + 1) / 2;
            const uint64_t cw_al = (cw + 63) & ~63ull;  // 256-byte aligned filter copy
            const bool both = mode == "both" && g.bloom.n && !m.alpha_trivial;
            s.c16.alloc(both ? cw_al + g.bloom.n : cw);
            s.nodes8.alloc(std::max<uint32_t>(g.n, 1));
            k_nodes8<<<grid_for(g.n), 256, 0, st>>>(g.view(), s.nodes8.p);
            MHW_CK(cudaGetLastError());
            // the eager init (about 11 alpha tests per slot, issue/latency
            // bound) probes a denser filter than the walk: 6 bits per arc,
            // pinned for the init launch (cfg2 step 27.86 -> 27.71 ms: init
            // 5.0 -> 4.66, walk 22.67 -> 22.83; 8 bits 27.76; unpinned 27.81)
            if (g.bloom.n && !m.alpha_trivial) {
                const char* ib = std::getenv("MHW_INIT_BLOOM_BITS");
                const uint32_t bits = ib ? (uint32_t)std::atoi(ib) : 6u;
                if (!ib && g.bloom2.n) {
                    // built with the walk's filter (its fold), graph_ensure_bloom
                    s.ib_p = g.bloom2.p;
                    s.ib_bytes = g.bloom2.bytes();
                    s.init_bloom_blocks = g.bloom2_blocks;
                } else if (bits && (uint64_t)bits * g.m / 8 > g.bloom.bytes() && (uint64_t)bits * g.m / 8 <= (33ull << 20)) {
                    graph_build_bloom(g, bits, s.init_bloom, &s.init_bloom_blocks, st);
                    s.ib_p = s.init_bloom.p;
                    s.ib_bytes = s.init_bloom.bytes();
                }
            }
            // 64-register cap (4 blocks/SM, a 40-byte stack frame): cfg2 walk
            // 24.64 -> 23.84 ms (more walkers in flight outweigh the spills
            // and the extra lock retries, 1.97 M -> 2.35 M)
            if (!std::getenv("MHW_WALK_REGS")) s.minb = 64;
            if (both) {
                MHW_CK(cudaMemcpyAsync(s.c16.p + cw_al, g.bloom.p, g.bloom.bytes(), cudaMemcpyDeviceToDevice, st));
                s.bloom_copy = s.c16.p + cw_al;
            }
            if (s.l2_pin && mode != "filter") {  // undo the filter window taken above
                int dev = 0;
                MHW_CK(cudaGetDevice(&dev));
                l2_limit_release(dev);
                s.l2_pin = false;
                s.pin_p = nullptr;
                s.pin_bytes = 0;
            }
            if (pin_ok && (mode == "chain" || both)) {
                int dev = 0, max_persist = 0;
                MHW_CK(cudaGetDevice(&dev));
                MHW_CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
                const size_t bytes = both ? s.c16.bytes() : cw * 4;
                if (max_persist > 0) {
                    l2_limit_acquire(dev, std::min<size_t>(bytes, (size_t)max_persist));
                    s.l2_pin = true;
                    s.pin_p = s.c16.p;
                    s.pin_bytes = bytes;
                    s.pin_ratio = (float)std::min(1.0, (double)max_persist / (double)bytes);
                    // the eager init (burn-in over N(v) slices) keeps the
                    // filter-only window: pinning the chain table there
                    // starves its slice reads (cfg2 init 4.7 -> 6.8 ms)
                    const char* ip = std::getenv("MHW_C16_INITPIN");  // filter (default) | same | none
                    const std::string imode = ip ? ip : "filter";
                    if (imode == "filter" && s.ib_p && s.ib_bytes <= (33ull << 20)) {
                        s.ipin_p = const_cast<uint32_t*>(s.ib_p);
                        s.ipin_bytes = s.ib_bytes;
                    } else if (imode == "filter" && g.bloom.n && !m.alpha_trivial && g.bloom.bytes() <= (33ull << 20)) {
                        s.ipin_p = both ? (void*)s.bloom_copy : (void*)g.bloom.p;
                        s.ipin_bytes = g.bloom.bytes();
                    } else if (imode == "none") {
                        s.ipin_p = s.c16.p;
                        s.ipin_bytes = 0;
                        s.init_unpinned = true;
                    }
                }
                if (trace)
                    std::fprintf(stderr, "[mhw] compact chains: pin %s, window %zu B, max persisting %d B, ratio %.3f\n",
                                 mode.c_str(), bytes, max_persist, (double)s.pin_ratio);
            }
        }
        if (!s.c16.n && want_ar && m.kind != DEEPWALK && g.m && g.m < (1ull << 32)) {
            // session arc records (typed models: 32 B with weight and types);
            // second-order models keep their chain words in them
            // node2vec: narrow 8-byte records when the node table (16 B per
            // node) is small enough to stay in L2 (MHW_NARROW=0/1 forces)
            const char* nw = std::getenv("MHW_NARROW");
            const bool narrow = !alias_prop && m.kind == NODE2VEC && (nw ? nw[0] == '1' : 16ull * g.n <= (32ull << 20));
            s.rec_u32 = typed_kind(m.kind) ? 8 : (narrow ? 2 : 4);
            const uint64_t need = 4ull * s.rec_u32 * g.m;
            if (dev_available_bytes() >= need + (2ull << 30)) {
                s.ac.alloc((g.m * s.rec_u32 + 3) / 4);
                k_arc_chain<<<grid_for(g.n * 32ull), 256, 0, st>>>(g.view(), s.ac.p, s.rec_u32);
                MHW_CK(cudaGetLastError());
                s.use_ar = true;
            }
        }
        // per-arc source nodes for the slot-order init kernels (k_init_all,
        // k_init_range*): one coalesced load instead of an owner search per
        // slot (MHW_ARC_SRC=0 for the A/B)
        {
            const char* se = std::getenv("MHW_ARC_SRC");
            if (s.eager_init && second_order(m.kind) && !(s.init_rec_order && s.ac.n) && g.m && g.m < (1ull << 32) &&
                !(se && se[0] == '0') && dev_available_bytes() >= 4ull * g.m + (2ull << 30)) {
                s.src.alloc(g.m);
                k_arc_src<<<grid_for(g.n * 32ull), 256, 0, st>>>(g.view(), s.src.p);
                MHW_CK(cudaGetLastError());
            }
        }
        if ((!s.ac.n && !s.c16.n) || !second_order(m.kind)) s.chain.alloc(std::max<uint64_t>(s.slots, 1));
        else s.chain.alloc(1);
        // node-keyed models: the chain table itself (hub replicas included)
        if (!s.l2_pin && !second_order(m.kind)) try_pin(s.chain.p, s.chain.bytes());
        if (want_ar && m.kind == DEEPWALK) s.use_ar = graph_ensure_arcrec(g);
        dispatch(m.kind, [&](auto kc) {
            constexpr int KIND = decltype(kc)::value;
            with_variant<KIND>(s.minb, !s.eager_init, s.ar_mode(), [&](auto rg, auto lz, auto ar) {
                s.grid = walk_grid<KIND, decltype(rg)::value, decltype(lz)::value, decltype(ar)::value>();
            });
        });
    }
    MHW_CK(cudaStreamSynchronize(st));
    if (trace) std::fprintf(stderr, "[mhw] session_create: model_bind %.2f ms, total %.2f ms\n", t_bind, tms());
}

// Persisting L2 access window over [p, p + bytes) on stream st. The caller's
// own window on that stream is saved by l2_window_save and put back by
// l2_window_restore after the session's launches.
static cudaStreamAttrValue l2_window_save(cudaStream_t st) {
    cudaStreamAttrValue prev{};
    MHW_CK(cudaStreamGetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &prev));
    return prev;
}

static void l2_window_restore(cudaStream_t st, const cudaStreamAttrValue& prev) {
    MHW_CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &prev));
}

static void l2_window(cudaStream_t st, void* p, size_t bytes, float ratio = 1.0f) {
    cudaStreamAttrValue attr{};
    attr.accessPolicyWindow.base_ptr = p;
    attr.accessPolicyWindow.num_bytes = bytes;
    attr.accessPolicyWindow.hitRatio = bytes ? ratio : 0.0f;
    attr.accessPolicyWindow.hitProp = bytes ? cudaAccessPropertyPersisting : cudaAccessPropertyNormal;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    MHW_CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &attr));
}

// Per node type visit scale of metapath2vec's replica weights (rep_weight):
// the steady cycle of metapath indices (metapath_next: after the last index,
// 1 if first == last else 0, models.hpp:77-85) spends count_t of its
// cycle_len steps at type t; walkers reach a type-t node in proportion to
// its arcs among the arcs_t incident to type t.
static std::vector<double> metapath_rep_scale(const std::vector<uint16_t>& mp, const Graph& g, cudaStream_t st) {
    const uint32_t T = std::max<uint32_t>(g.n_ntypes, 1);
    DBuf<unsigned long long> arcs(T);
    MHW_CK(cudaMemsetAsync(arcs.p, 0, T * 8ull, st));
    k_type_arcs<<<grid_for(g.n), 256, 0, st>>>(g.view(), arcs.p);
    MHW_CK(cudaGetLastError());
    std::vector<unsigned long long> a(T);
    MHW_CK(cudaMemcpyAsync(a.data(), arcs.p, T * 8ull, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    const size_t L = mp.size();
    const size_t b = (L > 1 && mp[0] == mp[L - 1]) ? 1 : 0;
    std::vector<double> count(T, 0.0), F(T, 0.0);
    for (size_t i = b; i < L; ++i) count[mp[i]] += 1.0;
    const double cycle = (double)(L - b);
    for (uint32_t t = 0; t < T; ++t)
        if (a[t]) F[t] = (count[t] * (double)g.m) / (cycle * (double)a[t]);
    return F;
}

uint64_t k_slots(int kind, const Graph& g) {
    if (kind == DEEPWALK) return g.n;
    if (kind == METAPATH2VEC) return (uint64_t)g.n * g.n_ntypes;
    return g.m;
}

RunParams Session::init_params() const {
    RunParams P = params();
    if (ib_p) {
        P.g.bloom = ib_p;
        P.g.bloom_blocks = init_bloom_blocks;
    }
    return P;
}

RunParams Session::params() const {
    RunParams P;
    P.g = g->view();
    P.m = model.dev;
    P.cfg = cfg;
    P.act = act.p;
    P.act_row = act_row.p;
    P.n_act = n_act;
    P.n_items = n_items;
    P.chain = chain.p;
    P.ac = ac.n ? ac.p : nullptr;
    P.c16 = c16.n ? c16.p : nullptr;
    P.nodes8 = nodes8.n ? nodes8.p : nullptr;
    P.src = src.n ? src.p : nullptr;
    if (bloom_copy) P.g.bloom = bloom_copy;
    P.rec_u32 = rec_u32;
    P.out = out.p;
    P.stride = stride;
    P.lens = lens.p;
    P.ctr = ctr.p;
    return P;
}

// Eager init of every arc-keyed slot: slot order (k_init_all: a warp's
// threads share v, so the burn-in candidates of N(v) are local; the words
// scatter into the records) or record order (k_init_rec: coalesced writes,
// state from the record, scattered N(v) reads); chosen in session_create
// (MHW_INIT_ORDER=rec|slot overrides).
template <int KIND>
static void launch_init_all(const Session& s, const RunParams& P0, cudaStream_t st) {
    RunParams P = P0;
    if (s.ib_p) {
        P.g.bloom = s.ib_p;
        P.g.bloom_blocks = s.init_bloom_blocks;
    }
    if (s.init_rec_order && s.ac.n) k_init_rec<KIND><<<grid_for(s.g->m), 256, 0, st>>>(P, 0, s.g->m, nullptr);
    else {
        const char* e = std::getenv("MHW_INIT_MINB");  // blocks/SM of the slot-order init (A/B)
        const int mb = e ? std::atoi(e) : 0;
        if (mb == 8) k_init_all<KIND, 8><<<grid_for(s.g->m), 256, 0, st>>>(P);
        else if (mb == 4) k_init_all<KIND, 4><<<grid_for(s.g->m), 256, 0, st>>>(P);
        else if (mb == 5) k_init_all<KIND, 5><<<grid_for(s.g->m), 256, 0, st>>>(P);
        else k_init_all<KIND><<<grid_for(s.g->m), 256, 0, st>>>(P);
    }
    MHW_CK(cudaGetLastError());
}

void session_run(Session& s, cudaStream_t user) {
    DeviceGuard dg(s.g->device);
    cudaStream_t st = user ? user : s.stream;
    const RunParams P = s.params();
    s.launches = 0;
    // A small edge filter is pinned in L2 for the walk (persisting access
    // window on the launch stream, cleared again after the launches).
    const bool pin = s.l2_pin;
    cudaStreamAttrValue prev_window{};
    if (pin) {
        prev_window = l2_window_save(st);
        if (s.ipin_bytes || s.init_unpinned) l2_window(st, s.ipin_p, s.ipin_bytes);
        else l2_window(st, s.pin_p, s.pin_bytes, s.pin_ratio);
    }
    const bool preloaded = s.chain_loaded;  // mhw_session_load_chain: table already initialised
    s.chain_loaded = false;
    if (!preloaded) MHW_CK(cudaMemsetAsync(s.chain.p, 0xFF, s.chain.bytes(), st));
    MHW_CK(cudaMemsetAsync(s.ctr.p, 0, s.ctr.bytes(), st));
    if (!preloaded && s.ac.n && second_order(s.model.dev.kind) && (!s.eager_init || !s.g->verified_sym)) {
        k_ac_reset<<<grid_for(s.g->m), 256, 0, st>>>(reinterpret_cast<uint32_t*>(s.ac.p), s.g->m, s.rec_u32);
        ++s.launches;
    }
    if (s.n_iso) {
        k_iso_rows<<<grid_for((uint64_t)s.n_iso * s.cfg.K), 256, 0, st>>>(s.iso.p, s.iso_row.p, s.n_iso, s.cfg.K,
                                                                          s.out.p, s.stride, s.lens.p);
        ++s.launches;
    }
    MHW_CK(cudaEventRecord(s.ev0, st));
    bool evm_done = false;
    if (s.n_items) {
        if (s.ex) {
            exact_launch(s, P, st);
            ++s.launches;
        } else if (s.wc.schedule == MHW_SCHEDULE_DETERMINISTIC) {
            DetState S;
            S.v = s.d_v.p;
            S.aff = s.d_aff.p;
            S.len = s.d_len.p;
            S.alive = s.d_alive.p;
            S.key = s.d_key.p;
            S.idx = s.d_idx.p;
            S.cand = s.d_cand.p;
            S.ccls = s.d_ccls.p;
            S.wc = s.d_wc.p;
            S.u = s.d_u.p;
            S.chosen = s.d_chosen.p;
            const uint64_t invalid_key = s.slots;
            const unsigned gr = grid_for(s.n_items);
            dispatch(s.model.dev.kind, [&](auto kc) {
                constexpr int KIND = decltype(kc)::value;
                k_det_setup<KIND><<<gr, 256, 0, st>>>(P, S);
                ++s.launches;
                for (uint32_t step = 0; step < s.cfg.L; ++step) {
                    k_det_propose<KIND><<<gr, 256, 0, st>>>(P, S, step, invalid_key);
                    size_t bytes = s.sort_temp.n;
                    MHW_CK(cub::DeviceRadixSort::SortPairs(s.sort_temp.p, bytes, s.d_key.p, s.d_key2.p, s.d_idx.p,
                                                           s.d_idx2.p, (int64_t)s.n_items, 0, s.sort_bits, st));
                    k_det_fold<KIND><<<gr, 256, 0, st>>>(P, S, s.d_key2.p, s.d_idx2.p, invalid_key);
                    k_det_advance<KIND><<<gr, 256, 0, st>>>(P, S);
                    s.launches += 3;
                }
                k_det_finish<<<gr, 256, 0, st>>>(P, S);
                ++s.launches;
            });
        } else {
            dispatch(s.model.dev.kind, [&](auto kc) {
                constexpr int KIND = decltype(kc)::value;
                if constexpr (second_order(KIND)) {
                    if (s.eager_init && !preloaded) {
                        launch_init_all<KIND>(s, P, st);
                        ++s.launches;
                    }
                }
                MHW_CK(cudaEventRecord(s.evm, st));
                evm_done = true;
                if (pin && (s.ipin_bytes || s.init_unpinned)) l2_window(st, s.pin_p, s.pin_bytes, s.pin_ratio);
                with_variant<KIND>(s.minb, !s.eager_init, s.ar_mode(), [&](auto rg, auto lz, auto ar) {
                    k_walk<KIND, decltype(rg)::value, decltype(lz)::value, decltype(ar)::value>
                        <<<s.grid, kWalkBlock, 0, st>>>(P);
                });
            });
            ++s.launches;
        }
        MHW_CK(cudaGetLastError());
    }
    if (!evm_done) MHW_CK(cudaEventRecord(s.evm, st));  // init fused into the walk (lazy / deterministic)
    if (pin) l2_window_restore(st, prev_window);
    MHW_CK(cudaEventRecord(s.ev1, st));
}

// Corpus rows of a generate_walks call (valid starts in the node range x
// K) and the padded row stride, without building a session.
void walk_rows(Graph& g, const mhw_model_desc& md, const mhw_walk_config& wc, uint64_t* rows, uint32_t* stride) {
    DeviceGuard dg(g.device);
    if (wc.walks_per_node == 0 || wc.walk_length == 0)
        invalid("walks_per_node, walk_length and threads must be positive");
    Model mb;
    model_bind(mb, g, md);
    const uint32_t b = wc.node_begin, e = wc.node_end ? wc.node_end : g.n;
    if (e > g.n || b > e) invalid("node range out of bounds");
    uint64_t n_valid = 0;
    if (e > b) {
        cudaStream_t st = g.stream;
        const uint32_t span = e - b;
        DBuf<uint8_t> valid(span), act(span), iso(span);
        DBuf<uint32_t> rank(span);
        k_classify<<<grid_for(span), 256, 0, st>>>(g.view(), mb.dev, b, e, valid.p, act.p, iso.p);
        MHW_CK(cudaGetLastError());
        size_t bytes = 0;
        MHW_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, valid.p, rank.p, (int64_t)span, st));
        DBuf<uint8_t> temp(std::max<size_t>(bytes, 1));
        MHW_CK(cub::DeviceScan::ExclusiveSum(temp.p, bytes, valid.p, rank.p, (int64_t)span, st));
        uint32_t last_rank = 0;
        uint8_t last_valid = 0;
        MHW_CK(cudaMemcpyAsync(&last_rank, rank.p + span - 1, 4, cudaMemcpyDeviceToHost, st));
        MHW_CK(cudaMemcpyAsync(&last_valid, valid.p + span - 1, 1, cudaMemcpyDeviceToHost, st));
        MHW_CK(cudaStreamSynchronize(st));
        n_valid = (uint64_t)last_rank + last_valid;
    }
    if (rows) *rows = n_valid * wc.walks_per_node;
    if (stride) *stride = (wc.walk_length + 1 + 3) & ~3u;
}

void session_init_chain(Session& s, uint64_t begin, uint64_t end, uint32_t* d_words, cudaStream_t user,
                        bool rec_order) {
    DeviceGuard dg(s.g->device);
    if (!second_order(s.model.dev.kind) || s.ex || s.wc.schedule == MHW_SCHEDULE_DETERMINISTIC)
        invalid("chain preloading applies to second-order models on the throughput schedule");
    if (begin > end || end > s.g->m) invalid("slot range out of bounds");
    if (begin == end) return;
    cudaStream_t st = user ? user : s.stream;
    const RunParams P = s.params();
    dispatch(s.model.dev.kind, [&](auto kc) {
        constexpr int KIND = decltype(kc)::value;
        if constexpr (second_order(KIND)) {
            if (rec_order) k_init_rec<KIND><<<grid_for(end - begin), 256, 0, st>>>(P, begin, end, d_words);
            else k_init_range<KIND><<<grid_for(end - begin), 256, 0, st>>>(P, begin, end, d_words);
        }
    });
    MHW_CK(cudaGetLastError());
}

// Reset + eager initialisation of the session's chain table without a walk
// (what session_run does before its walk kernel); the next run starts from
// this table (chain_loaded). Lazy sessions get an empty table.
void session_prepare(Session& s, cudaStream_t user) {
    DeviceGuard dg(s.g->device);
    if (!second_order(s.model.dev.kind) || s.ex || s.wc.schedule == MHW_SCHEDULE_DETERMINISTIC)
        invalid("chain preloading applies to second-order models on the throughput schedule");
    cudaStream_t st = user ? user : s.stream;
    const RunParams P = s.params();
    MHW_CK(cudaMemsetAsync(s.chain.p, 0xFF, s.chain.bytes(), st));
    if (s.ac.n && (!s.eager_init || !s.g->verified_sym))
        k_ac_reset<<<grid_for(s.g->m), 256, 0, st>>>(reinterpret_cast<uint32_t*>(s.ac.p), s.g->m, s.rec_u32);
    if (s.eager_init && s.g->m) {
        dispatch(s.model.dev.kind, [&](auto kc) {
            constexpr int KIND = decltype(kc)::value;
            if constexpr (second_order(KIND)) launch_init_all<KIND>(s, P, st);
        });
    }
    MHW_CK(cudaGetLastError());
    s.chain_loaded = true;
}

// Entry of arc a of the session's chain table as installed: the 16-bit
// compact word, the colocated 32-bit word of record a, or chain[a] (slot
// order) -- for comparing tables of sessions with the same layout.
__global__ void k_export_table(RunParams P, uint64_t m, uint32_t* __restrict__ out) {
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < m; a += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t w;
        if (P.c16) w = reinterpret_cast<const uint16_t*>(P.c16)[a];
        else if (P.ac) w = reinterpret_cast<const uint32_t*>(P.ac)[a * P.rec_u32 + chain_word_off(P.rec_u32)];
        else w = P.chain[a];
        out[a] = w;
    }
}

void session_export_table(Session& s, uint32_t* d_words, cudaStream_t user) {
    DeviceGuard dg(s.g->device);
    if (!second_order(s.model.dev.kind) || s.ex || s.wc.schedule == MHW_SCHEDULE_DETERMINISTIC)
        invalid("chain tables are exported for second-order models on the throughput schedule");
    cudaStream_t st = user ? user : s.stream;
    if (s.g->m) k_export_table<<<grid_for(s.g->m), 256, 0, st>>>(s.params(), s.g->m, d_words);
    MHW_CK(cudaGetLastError());
}

void session_load_chain(Session& s, const uint32_t* d_words, cudaStream_t user, bool rec_order) {
    if (rec_order) {
        session_load_records_range(s, 0, s.g->m, d_words, user);
        return;
    }
    DeviceGuard dg(s.g->device);
    if (!second_order(s.model.dev.kind) || s.ex || s.wc.schedule == MHW_SCHEDULE_DETERMINISTIC)
        invalid("chain preloading applies to second-order models on the throughput schedule");
    cudaStream_t st = user ? user : s.stream;
    if (s.g->m) {
        const RunParams P = s.params();
        dispatch(s.model.dev.kind, [&](auto kc) {
            constexpr int KIND = decltype(kc)::value;
            uint32_t* const ac = s.ac.n ? reinterpret_cast<uint32_t*>(s.ac.p) : nullptr;
            if constexpr (second_order(KIND))
                k_load_chain<KIND><<<grid_for(s.g->m), 256, 0, st>>>(P, d_words, ac, s.rec_u32, s.chain.p);
        });
        MHW_CK(cudaGetLastError());
    }
    s.chain_loaded = true;
}

// Installs entries [begin, end) of a record-order table (d_words points at
// entry begin). A table installed piecewise (e.g. each piece as soon as its
// all-gather lands) counts as loaded for the next run once the caller has
// installed every piece.
void session_load_records_range(Session& s, uint64_t begin, uint64_t end, const uint32_t* d_words,
                                cudaStream_t user) {
    DeviceGuard dg(s.g->device);
    if (!second_order(s.model.dev.kind) || s.ex || s.wc.schedule == MHW_SCHEDULE_DETERMINISTIC)
        invalid("chain preloading applies to second-order models on the throughput schedule");
    if (begin > end || end > s.g->m) invalid("record range out of bounds");
    cudaStream_t st = user ? user : s.stream;
    if (end > begin) {
        const RunParams P = s.params();
        uint32_t* const ac = s.ac.n ? reinterpret_cast<uint32_t*>(s.ac.p) : nullptr;
        k_load_rec<<<grid_for(end - begin), 256, 0, st>>>(P, d_words, ac, s.rec_u32, s.chain.p, begin, end);
        MHW_CK(cudaGetLastError());
    }
    s.chain_loaded = true;
}

uint32_t session_record_width(const Session& s) { return (s.ac.n && s.rec_u32 == 8) ? 3u : 1u; }

// The exchange format a sharded init should use (mhw_session_init_shard /
// _load_shard_range): compact chains -> slot order, 2-byte encoded words;
// otherwise record order with session_record_width u32 words per entry.
uint32_t session_shard_entry_bytes(const Session& s) { return s.c16.n ? 2u : 4u * session_record_width(s); }

void session_init_shard(Session& s, uint64_t begin, uint64_t end, void* d_out, cudaStream_t user) {
    if (!s.c16.n) {
        session_init_chain(s, begin, end, static_cast<uint32_t*>(d_out), user, true);
        return;
    }
    DeviceGuard dg(s.g->device);
    if (begin > end || end > s.g->m) invalid("shard range out of bounds");
    if (begin == end) return;
    cudaStream_t st = user ? user : s.stream;
    k_init_range16<<<grid_for(end - begin), 256, 0, st>>>(s.init_params(), begin, end, static_cast<uint16_t*>(d_out));
    MHW_CK(cudaGetLastError());
}

void session_load_shard_range(Session& s, uint64_t begin, uint64_t end, const void* d_in, cudaStream_t user) {
    if (!s.c16.n) {
        session_load_records_range(s, begin, end, static_cast<const uint32_t*>(d_in), user);
        return;
    }
    DeviceGuard dg(s.g->device);
    if (begin > end || end > s.g->m) invalid("shard range out of bounds");
    cudaStream_t st = user ? user : s.stream;
    if (end > begin) {
        k_load_slot16<<<grid_for(end - begin), 256, 0, st>>>(s.params(), static_cast<const uint16_t*>(d_in), begin, end);
        MHW_CK(cudaGetLastError());
    }
    s.chain_loaded = true;
}

void session_stats(Session& s, mhw_walk_stats& out) {
    DeviceGuard dg(s.g->device);
    MHW_CK(cudaEventSynchronize(s.ev1));
    unsigned long long h[8];
    MHW_CK(cudaMemcpy(h, s.ctr.p, sizeof(h), cudaMemcpyDeviceToHost));
    if (h[4]) {
        const uint32_t from = (uint32_t)(h[5] >> 32), to = (uint32_t)h[5];
        invalid("second-order walk on asymmetric adjacency: no back edge " + std::to_string(from) + "->" +
                std::to_string(to));
    }
    float ms = 0.f, ms_init = 0.f;
    MHW_CK(cudaEventElapsedTime(&ms, s.ev0, s.ev1));
    MHW_CK(cudaEventElapsedTime(&ms_init, s.ev0, s.evm));
    out.walks = s.rows;
    out.early_terminations = h[2] + (uint64_t)s.n_iso * s.cfg.K;
    out.skipped_starts = s.skipped;
    out.steps = h[1];
    out.slot_inits = h[3];
    out.chain_retries = h[6];
    out.rejection_trials = h[7];
    // T_i / T_w (manager.cpp:39-44, engine.cpp:228-232): device time of the
    // eager chain-table init launch and of the walk kernels; a lazy run
    // initialises inside the walk (T_i = 0, as the reference's T_w then holds
    // it too). steps_per_sec counts both, like engine.cpp:231-232.
    out.init_seconds = ms_init * 1e-3;
    out.walk_seconds = (ms - ms_init) * 1e-3;
    out.steps_per_sec = ms > 0 ? (double)h[1] / (ms * 1e-3) : 0.0;
}

void session_download(Session& s, uint32_t* nodes, uint32_t* lens, cudaStream_t user) {
    DeviceGuard dg(s.g->device);
    cudaStream_t st = user ? user : s.stream;
    if (s.rows) {
        if (nodes) MHW_CK(cudaMemcpyAsync(nodes, s.out.p, s.rows * s.stride * 4, cudaMemcpyDeviceToHost, st));
        if (lens) MHW_CK(cudaMemcpyAsync(lens, s.lens.p, s.rows * 4, cudaMemcpyDeviceToHost, st));
    }
    MHW_CK(cudaStreamSynchronize(st));
}

// Packs the last run's corpus (rows of length lens[r]) into nodes[off[r] ..
// off[r+1]) and copies nodes + offsets to the host.
void session_download_packed(Session& s, uint32_t* h_nodes, uint64_t cap_nodes, uint64_t* h_offsets,
                             uint64_t cap_rows, uint64_t* n_nodes, cudaStream_t user) {
    DeviceGuard dg(s.g->device);
    cudaStream_t st = user ? user : s.stream;
    const uint64_t rows = s.rows;
    if (cap_rows < rows + 1) invalid("offset buffer too small for the corpus");
    DBuf<uint64_t> len64(rows + 1), off(rows + 1);
    k_len64<<<grid_for(rows + 1), 256, 0, st>>>(s.lens.p, rows, len64.p);
    size_t bytes = 0;
    MHW_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, len64.p, off.p, (int64_t)rows + 1, st));
    DBuf<uint8_t> temp(std::max<size_t>(bytes, 1));
    MHW_CK(cub::DeviceScan::ExclusiveSum(temp.p, bytes, len64.p, off.p, (int64_t)rows + 1, st));
    uint64_t total = 0;
    MHW_CK(cudaMemcpyAsync(&total, off.p + rows, 8, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    if (cap_nodes < total) invalid("node buffer too small for the corpus");
    DBuf<uint32_t> packed(std::max<uint64_t>(total, 1));
    if (rows) k_pack<<<grid_for(rows * 32), 256, 0, st>>>(s.out.p, s.stride, off.p, rows, packed.p);
    MHW_CK(cudaGetLastError());
    if (total) MHW_CK(cudaMemcpyAsync(h_nodes, packed.p, total * 4, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaMemcpyAsync(h_offsets, off.p, (rows + 1) * 8, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    if (n_nodes) *n_nodes = total;
}

// generate_walks into a packed host corpus with the D2H overlapped: the
// active start nodes are cut into `chunks` contiguous ranges (rows of a range
// are contiguous); chunk c is walked, packed on the device and copied to the
// host on a second stream while chunk c+1 walks. Every chunk shares the chain
// table (same sampler state as one launch; only the interleaving differs).
// Pinned per-chunk totals for session_run_packed: one process-wide buffer
// per host thread, grown on demand and never freed (cudaFreeHost can stall a
// call for 100+ ms).
static uint64_t* pinned_scratch(size_t n) {
    thread_local uint64_t* buf = nullptr;
    thread_local size_t cap = 0;
    if (n > cap) {
        uint64_t* p = nullptr;
        MHW_CK(cudaMallocHost(&p, std::max<size_t>(n, 64) * sizeof(uint64_t)));
        buf = p;  // the previous (smaller) buffer is kept: it may still be in use by an unfinished caller
        cap = std::max<size_t>(n, 64);
    }
    return buf;
}

void session_run_packed(Session& s, uint32_t* h_nodes, uint64_t cap_nodes, uint64_t* h_offsets,
                        uint64_t cap_rows, int chunks, mhw_walk_stats* stats) {
    DeviceGuard dg(s.g->device);
    if (s.ex || s.wc.schedule == MHW_SCHEDULE_DETERMINISTIC || s.n_act < 2 * (uint32_t)chunks || chunks < 2) {
        session_run(s, nullptr);
        mhw_walk_stats st{};
        session_stats(s, st);
        session_download_packed(s, h_nodes, cap_nodes, h_offsets, cap_rows, nullptr, nullptr);
        if (stats) *stats = st;
        return;
    }
    if (cap_rows < s.rows + 1) invalid("offset buffer too small for the corpus");
    const bool trace = std::getenv("MHW_TRACE") != nullptr;
    using clk = std::chrono::steady_clock;
    const auto ta = clk::now();
    auto ms_since = [&](clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); };
    cudaStream_t S = s.stream, T = nullptr;
    MHW_CK(cudaStreamCreateWithFlags(&T, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> ev(chunks, nullptr), cdone(chunks, nullptr);
    auto cleanup = [&] {
        for (auto* v : {&ev, &cdone})
            for (auto& e : *v)
                if (e) cudaEventDestroy(e);
        if (T) cudaStreamDestroy(T);
    };
    try {
        for (auto* v : {&ev, &cdone})
            for (auto& e : *v) MHW_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        // chunk boundaries over the active-node list and their first rows
        std::vector<uint32_t> jc(chunks + 1);
        std::vector<uint64_t> rc(chunks + 1);
        // the first chunk is a quarter of the others: the copy engine (the
        // bound of this call: the corpus leaves at ~55 GB/s) starts as soon
        // as possible after the eager init (MHW_E2E_FIRST: its weight)
        const char* fw = std::getenv("MHW_E2E_FIRST");
        const double w0 = fw ? std::atof(fw) : 0.25, wt = w0 + (chunks - 1);
        jc[0] = 0;
        for (int c = 1; c < chunks; ++c) jc[c] = (uint32_t)((double)s.n_act * (w0 + (c - 1)) / wt);
        jc[chunks] = s.n_act;
        for (int c = 1; c < chunks; ++c)  // non-empty chunks (n_act >= 2 chunks)
            jc[c] = std::min<uint32_t>(std::max<uint32_t>(jc[c], jc[c - 1] + 1), s.n_act - (uint32_t)(chunks - c));
        rc[0] = 0;
        rc[chunks] = s.rows;
        for (int c = 1; c < chunks; ++c)
            MHW_CK(cudaMemcpy(&rc[c], s.act_row.p + jc[c], 8, cudaMemcpyDeviceToHost));
        uint64_t max_rows = 0;
        for (int c = 0; c < chunks; ++c) max_rows = std::max(max_rows, rc[c + 1] - rc[c]);
        const uint64_t rowcap = (uint64_t)s.cfg.L + 1;
        // two staging buffers of one chunk each: chunk c packs into buffer
        // c & 1 once the copy of chunk c - 2 out of it has finished
        DBuf<uint32_t> stage0(std::max<uint64_t>(max_rows * rowcap, 1)), stage1(std::max<uint64_t>(max_rows * rowcap, 1));
        uint32_t* const stage[2] = {stage0.p, stage1.p};
        DBuf<uint64_t> len64(s.rows + 1), goff(s.rows + 1);
        std::vector<DBuf<uint64_t>> offc(chunks);
        uint64_t* h_tot = pinned_scratch(chunks);
        size_t scan_bytes = 0;
        MHW_CK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, len64.p, goff.p, (int64_t)s.rows + 1, S));
        DBuf<uint8_t> scan_tmp(std::max<size_t>(scan_bytes, 1));
        // sampler reset + isolated rows + eager init (as session_run); a table
        // installed with mhw_session_load_chain / _load_records is used as is
        RunParams P = s.params();
        const bool preloaded = s.chain_loaded;
        s.chain_loaded = false;
        if (!preloaded) MHW_CK(cudaMemsetAsync(s.chain.p, 0xFF, s.chain.bytes(), S));
        MHW_CK(cudaMemsetAsync(s.ctr.p, 0, s.ctr.bytes(), S));
        if (!preloaded && s.ac.n && second_order(s.model.dev.kind) && (!s.eager_init || !s.g->verified_sym))
            k_ac_reset<<<grid_for(s.g->m), 256, 0, S>>>(reinterpret_cast<uint32_t*>(s.ac.p), s.g->m, s.rec_u32);
        if (s.n_iso)
            k_iso_rows<<<grid_for((uint64_t)s.n_iso * s.cfg.K), 256, 0, S>>>(s.iso.p, s.iso_row.p, s.n_iso, s.cfg.K,
                                                                             s.out.p, s.stride, s.lens.p);
        const bool pin = s.l2_pin;
        const cudaStreamAttrValue prev_window = pin ? l2_window_save(S) : cudaStreamAttrValue{};
        if (pin) {
            if (s.ipin_bytes || s.init_unpinned) l2_window(S, s.ipin_p, s.ipin_bytes);
            else l2_window(S, s.pin_p, s.pin_bytes, s.pin_ratio);
        }
        MHW_CK(cudaEventRecord(s.ev0, S));
        const double t_setup = ms_since(ta);
        dispatch(s.model.dev.kind, [&](auto kc) {
            constexpr int KIND = decltype(kc)::value;
            if constexpr (second_order(KIND)) {
                if (s.eager_init && !preloaded) launch_init_all<KIND>(s, P, S);
            }
        });
        MHW_CK(cudaEventRecord(s.evm, S));
        if (pin && (s.ipin_bytes || s.init_unpinned)) l2_window(S, s.pin_p, s.pin_bytes, s.pin_ratio);
        uint64_t H = 0;
        auto issue_copy = [&](int c) {
            MHW_CK(cudaEventSynchronize(ev[c]));
            const uint64_t tot = h_tot[c];
            if (H + tot > cap_nodes) invalid("node buffer too small for the corpus");
            MHW_CK(cudaStreamWaitEvent(T, ev[c], 0));
            if (tot) MHW_CK(cudaMemcpyAsync(h_nodes + H, stage[c & 1], tot * 4, cudaMemcpyDeviceToHost, T));
            MHW_CK(cudaEventRecord(cdone[c], T));
            H += tot;
        };
        for (int c = 0; c < chunks; ++c) {
            RunParams Pc = P;
            Pc.act = s.act.p + jc[c];
            Pc.act_row = s.act_row.p + jc[c];
            Pc.n_act = jc[c + 1] - jc[c];
            Pc.n_items = (uint64_t)Pc.n_act * s.cfg.K;
            MHW_CK(cudaMemsetAsync(s.ctr.p, 0, sizeof(unsigned long long), S));  // work counter
            dispatch(s.model.dev.kind, [&](auto kc) {
                constexpr int KIND = decltype(kc)::value;
                with_variant<KIND>(s.minb, !s.eager_init, s.ar_mode(), [&](auto rg, auto lz, auto ar) {
                    k_walk<KIND, decltype(rg)::value, decltype(lz)::value, decltype(ar)::value>
                        <<<s.grid, kWalkBlock, 0, S>>>(Pc);
                });
            });
            // pack rows [rc[c], rc[c+1]) into staging buffer c & 1
            const uint64_t nr = rc[c + 1] - rc[c];
            offc[c].alloc(nr + 1);
            k_len64<<<grid_for(nr + 1), 256, 0, S>>>(s.lens.p + rc[c], nr, len64.p + rc[c]);
            size_t b = scan_bytes;
            MHW_CK(cub::DeviceScan::ExclusiveSum(scan_tmp.p, b, len64.p + rc[c], offc[c].p, (int64_t)nr + 1, S));
            if (c >= 2) MHW_CK(cudaStreamWaitEvent(S, cdone[c - 2], 0));
            if (nr)
                k_pack<<<grid_for(nr * 32), 256, 0, S>>>(s.out.p + rc[c] * s.stride, s.stride, offc[c].p, nr,
                                                        stage[c & 1]);
            MHW_CK(cudaMemcpyAsync(h_tot + c, offc[c].p + nr, 8, cudaMemcpyDeviceToHost, S));
            MHW_CK(cudaEventRecord(ev[c], S));
            // copy chunk c - 1 while chunk c walks
            if (c >= 1) issue_copy(c - 1);
        }
        if (pin) l2_window_restore(S, prev_window);
        MHW_CK(cudaEventRecord(s.ev1, S));
        MHW_CK(cudaGetLastError());
        issue_copy(chunks - 1);
        const double t_issued = ms_since(ta);
        // global row offsets (one scan over all lengths) and the counters
        k_len64<<<grid_for(s.rows + 1), 256, 0, S>>>(s.lens.p, s.rows, len64.p);
        size_t b = scan_bytes;
        MHW_CK(cub::DeviceScan::ExclusiveSum(scan_tmp.p, b, len64.p, goff.p, (int64_t)s.rows + 1, S));
        MHW_CK(cudaMemcpyAsync(h_offsets, goff.p, (s.rows + 1) * 8, cudaMemcpyDeviceToHost, S));
        MHW_CK(cudaStreamSynchronize(S));
        MHW_CK(cudaStreamSynchronize(T));
        s.launches = 0;
        mhw_walk_stats st{};
        session_stats(s, st);
        if (stats) *stats = st;
        if (trace)
            std::fprintf(stderr,
                         "[mhw] run_packed: %d chunks, setup %.2f ms, last copy issued %.2f ms, done %.2f ms, "
                         "device walk+pack %.2f ms\n",
                         chunks, t_setup, t_issued, ms_since(ta), st.walk_seconds * 1e3);
    } catch (...) {
        cudaStreamSynchronize(S);
        if (T) cudaStreamSynchronize(T);
        cleanup();
        throw;
    }
    if (trace) {
        const double t0 = ms_since(ta);
        cleanup();
        std::fprintf(stderr, "[mhw] run_packed: locals freed at %.2f ms, cleanup %.2f ms\n", t0, ms_since(ta) - t0);
    } else {
        cleanup();
    }
}

// ------------------------------------------------------------ parity API
void run_decide(Graph& g, const mhw_model_desc& md, uint64_t n, const uint32_t* pos, const uint32_t* aff,
                const uint32_t* cand, const uint32_t* last, const double* u, double* wc, double* wl,
                uint8_t* acc, bool hastings) {
    DeviceGuard dg(g.device);
    Model mb;
    model_bind(mb, g, md);
    if (!n) return;
    cudaStream_t st = g.stream;
    DBuf<uint32_t> dpos(n), daff(n), dc(n), dl(n);
    DBuf<double> du(n), dwc(n), dwl(n);
    DBuf<uint8_t> dacc(n);
    DBuf<unsigned> bad(1);
    MHW_CK(cudaMemcpyAsync(dpos.p, pos, n * 4, cudaMemcpyHostToDevice, st));
    MHW_CK(cudaMemcpyAsync(daff.p, aff, n * 4, cudaMemcpyHostToDevice, st));
    MHW_CK(cudaMemcpyAsync(dc.p, cand, n * 4, cudaMemcpyHostToDevice, st));
    MHW_CK(cudaMemcpyAsync(dl.p, last, n * 4, cudaMemcpyHostToDevice, st));
    MHW_CK(cudaMemcpyAsync(du.p, u, n * 8, cudaMemcpyHostToDevice, st));
    MHW_CK(cudaMemsetAsync(bad.p, 0, 4, st));
    const DevGraph gv = g.view();
    dispatch(md.kind, [&](auto kc) {
        constexpr int KIND = decltype(kc)::value;
        k_decide<KIND><<<grid_for(n), 256, 0, st>>>(gv, mb.dev, n, dpos.p, daff.p, dc.p, dl.p, du.p, dwc.p, dwl.p,
                                                   dacc.p, bad.p, hastings ? 1 : 0);
    });
    MHW_CK(cudaGetLastError());
    unsigned hbad = 0;
    MHW_CK(cudaMemcpyAsync(wc, dwc.p, n * 8, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaMemcpyAsync(wl, dwl.p, n * 8, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaMemcpyAsync(acc, dacc.p, n, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    if (hbad) invalid(std::to_string(hbad) + " decide triples reference states or indices outside the graph");
}

void run_init_states(Graph& g, const mhw_model_desc& md, const mhw_walk_config& wc, uint64_t n,
                     const uint32_t* pos, const uint32_t* aff, uint32_t* last) {
    DeviceGuard dg(g.device);
    Model mb;
    model_bind(mb, g, md);
    if (!n) return;
    DevCfg cfg{};
    cfg.seed = wc.seed;
    cfg.K = wc.walks_per_node;
    cfg.L = wc.walk_length;
    cfg.init_kind = wc.init_kind;
    cfg.burn_in = wc.burn_in_steps;
    cfg.hw = wc.hw_sample_size;
    cfg.rep_deg = kNoReplicas;  // states are queried without a walker: base slots
    cfg.rep_base_slot = 0;
    cfg.rep_group = nullptr;
    cudaStream_t st = g.stream;
    DBuf<uint32_t> dpos(n), daff(n), dout(n);
    DBuf<unsigned> bad(1);
    MHW_CK(cudaMemcpyAsync(dpos.p, pos, n * 4, cudaMemcpyHostToDevice, st));
    MHW_CK(cudaMemcpyAsync(daff.p, aff, n * 4, cudaMemcpyHostToDevice, st));
    MHW_CK(cudaMemsetAsync(bad.p, 0, 4, st));
    const DevGraph gv = g.view();
    dispatch(md.kind, [&](auto kc) {
        constexpr int KIND = decltype(kc)::value;
        k_init_states<KIND><<<grid_for(n), 256, 0, st>>>(gv, mb.dev, cfg, n, dpos.p, daff.p, dout.p, bad.p);
    });
    MHW_CK(cudaGetLastError());
    unsigned hbad = 0;
    MHW_CK(cudaMemcpyAsync(last, dout.p, n * 4, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    if (hbad) invalid(std::to_string(hbad) + " states outside the graph");
}

void run_check(Graph& g, const mhw_model_desc& md, uint64_t seed, uint64_t n, const uint32_t* pos,
               const uint32_t* aff, uint64_t draws, double* kl, uint64_t* counts) {
    DeviceGuard dg(g.device);
    Model mb;
    model_bind(mb, g, md);
    if (!n) return;
    if (!draws) invalid("draws must be positive");
    for (uint64_t j = 0; j < n; ++j)
        if (pos[j] >= g.n) invalid("state position outside the graph");
    DevCfg cfg{};
    cfg.seed = seed;
    cfg.init_kind = INIT_RANDOM;  // cmd_check uses the default InitStrategy (tools/mhwalk.cpp:235)
    cfg.burn_in = 100;
    cfg.hw = 32;
    cfg.rep_deg = kNoReplicas;
    cudaStream_t st = g.stream;
    DBuf<uint32_t> dpos(n), daff(n);
    DBuf<uint64_t> deg(n + 1), base(n + 1);
    DBuf<double> dkl(n);
    MHW_CK(cudaMemcpyAsync(dpos.p, pos, n * 4, cudaMemcpyHostToDevice, st));
    MHW_CK(cudaMemcpyAsync(daff.p, aff, n * 4, cudaMemcpyHostToDevice, st));
    k_state_degrees<<<grid_for(n + 1), 256, 0, st>>>(g.view(), dpos.p, n, deg.p);
    size_t bytes = 0;
    MHW_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, deg.p, base.p, (int64_t)n + 1, st));
    DBuf<uint8_t> temp(std::max<size_t>(bytes, 1));
    MHW_CK(cub::DeviceScan::ExclusiveSum(temp.p, bytes, deg.p, base.p, (int64_t)n + 1, st));
    uint64_t total = 0;
    MHW_CK(cudaMemcpyAsync(&total, base.p + n, 8, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
    DBuf<double> W(std::max<uint64_t>(total, 1));
    DBuf<unsigned long long> cnt(std::max<uint64_t>(total, 1));
    const DevGraph gv = g.view();
    dispatch(md.kind, [&](auto kc) {
        constexpr int KIND = decltype(kc)::value;
        k_check<KIND><<<grid_for(n * 32), 256, 0, st>>>(gv, mb.dev, cfg, n, dpos.p, daff.p, base.p, draws, W.p,
                                                        cnt.p, dkl.p);
    });
    MHW_CK(cudaGetLastError());
    MHW_CK(cudaMemcpyAsync(kl, dkl.p, n * 8, cudaMemcpyDeviceToHost, st));
    if (counts && total) MHW_CK(cudaMemcpyAsync(counts, cnt.p, total * 8, cudaMemcpyDeviceToHost, st));
    MHW_CK(cudaStreamSynchronize(st));
}

void partition_nodes(Graph& g, const mhw_model_desc& md, int parts, uint32_t* cuts) {
    DeviceGuard dg(g.device);
    if (parts <= 0) invalid("parts must be positive");
    Model mb;
    model_bind(mb, g, md);
    cudaStream_t st = g.stream;
    const uint32_t n = g.n;
    cuts[0] = 0;
    for (int i = 1; i <= parts; ++i) cuts[i] = n;
    if (!n) return;
    DBuf<uint8_t> valid(n), act(n), iso(n);
    DBuf<uint32_t> ids(n), list(n);
    k_classify<<<grid_for(n), 256, 0, st>>>(g.view(), mb.dev, 0, n, valid.p, act.p, iso.p);
    k_iota_from<<<grid_for(n), 256, 0, st>>>(ids.p, n, 0);
    MHW_CK(cudaGetLastError());
    uint32_t n_act = 0;
    select_flagged(ids.p, act.p, list.p, n, &n_act, st);
    std::vector<uint32_t> h(n_act);
    if (n_act) MHW_CK(cudaMemcpy(h.data(), list.p, n_act * 4, cudaMemcpyDeviceToHost));
    // cut i starts at the active node of rank floor(i * n_act / parts)
    for (int i = 1; i < parts; ++i) {
        const uint64_t r = (uint64_t)i * n_act / parts;
        cuts[i] = r < n_act ? h[r] : n;
        if (cuts[i] < cuts[i - 1]) cuts[i] = cuts[i - 1];
    }
}

}  // namespace mhw
