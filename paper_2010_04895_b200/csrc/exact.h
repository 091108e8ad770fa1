// exact.h -- the exact baseline samplers of WalkerContext::next_edge
// (engine.cpp:88-116): alias (per-state tables), direct (inverse CDF over the
// dynamic weights) and rejection (static alias proposal + envelope). They are
// the paper's comparison baselines, not the product path (M-H, walk.cu).
#pragma once

#include "internal.h"
#include "walk.h"

namespace mhw {

struct ExactState {
    int sampler = 0;            // MHW_SAMPLER_ALIAS / _DIRECT / _REJECTION
    double bound = 1.0;         // rejection_bound (engine.cpp:39-58)
    int grid = 0;
    // alias: one table per reference state slot (manager.hpp:29-31)
    uint64_t table_entries = 0;
    DBuf<uint32_t> astat;       // per slot: 0 empty, 1 building, 2 ready, 3 dead
    DBuf<double> aprob;
    DBuf<uint32_t> aalias;
    DBuf<uint64_t> qoff;        // second order: first entry of node v's tables
    DBuf<uint32_t> scratch;     // per warp: alias_build stacks (max degree)
    uint64_t scratch_per_warp = 0;
    // rejection: static proposal per node (alias_build of the static weights)
    DBuf<double> sprob;
    DBuf<uint32_t> salias;
};

// Validates and allocates the sampler's device state (errors before any walk).
void exact_create(Session& s);
// Resets per-run state and launches the walk kernel on `st`.
void exact_launch(Session& s, const RunParams& P, cudaStream_t st);
// rejection_bound (engine.cpp:39-58) of a bound model.
double exact_rejection_bound(const mhw_model_desc& md, const Model& m);

}  // namespace mhw
