#!/usr/bin/env python
"""Per-shard device times of an N-GPU run, measured one shard at a time on one GPU.

python scripts/shard_scaling.py --config cfg5 --parts 1 2 4 8 [--reps 3]

The walk path has no exchange: rank r of N runs the
walkers of its start-node range [cuts[r], cuts[r+1]) on its own CSR replica
with a private chain table, and its kernels never wait on another rank. So
the N-GPU walk time is max over r of rank r's time, and each rank's time can
be measured alone on one GPU. This script builds every rank's session in
turn (the exact session `bench.py --gpus N` builds on rank r), times its
steps with CUDA events (same step as bench.py: chain reset/init + walk, 256 MB
L2 flush in between, median of --reps), and prints one JSON line per N with
the max / mean shard time and the projected speed-up T(1) / max_r T_r(N).

For configs whose single-GPU run initialises every chain slot eagerly
(cfg2), bench.py shards that init (init a 1/N slot range, all-gather, load):
here rank r's step is init_chain(its range) + load_chain + run, and the
all-gather of S*4 bytes over NVLink is not included (it is reported as
bytes). This is a projection from measured per-rank device times, not a
multi-GPU measurement; bench.py under torchrun is the real one.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5", choices=sorted(bench.CONFIGS))
    ap.add_argument("--parts", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--order", default="shard", choices=["shard", "rec", "slot"],
                    help="sharded-init table order: record order (coalesced install) or slot order")
    ap.add_argument("--shard-init", action="store_true",
                    help="shard the eager chain init even where one GPU would initialise lazily")
    args = ap.parse_args()
    import torch
    import paper_2010_04895_b200 as mhw

    cfg = dict(bench.CONFIGS[args.config])
    cfg["name"] = args.config
    dev = 0
    torch.cuda.set_device(dev)
    g = bench.build_graph(cfg, device=dev)
    model = bench.make_model(cfg)
    eager1 = cfg["model"] in ("node2vec", "edge2vec", "fairwalk") and (bench.shard_init_pays(cfg, g) or args.shard_init)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    t1 = None
    for N in args.parts:
        cuts = mhw.partition_nodes(g, model, N)
        shard_init = N > 1 and eager1
        per_rank = []
        for r in range(N):
            wcfg = bench.make_config(cfg, int(cuts[r]), int(cuts[r + 1]))
            if shard_init:
                wcfg.init_mode = 2
            sess = mhw.Session(g, model, wcfg)
            S = sess.chain_size()
            if args.order == "shard":  # the session's exchange format (bench.ShardInit)
                init_fn = sess.init_shard
                load_fn = lambda ptr, st: sess.load_shard_range(0, S, ptr, st)  # noqa: E731
                B = sess.shard_entry_bytes()
            else:
                init_fn = sess.init_records if args.order == "rec" else sess.init_chain
                load_fn = sess.load_records if args.order == "rec" else sess.load_chain
                B = 4 * (sess.record_width() if args.order == "rec" else 1)
            if shard_init:
                per = (S + N - 1) // N
                lo, hi = min(S, r * per), min(S, (r + 1) * per)
                full = torch.empty(max(per * N * B, 4), dtype=torch.uint8, device=dev)
                # the all-gathered table every rank loads: built once here
                for q in range(N):
                    ql, qh = min(S, q * per), min(S, (q + 1) * per)
                    if qh > ql:
                        init_fn(ql, qh, full.data_ptr() + B * ql, stream.cuda_stream)

            def step(evs=None):
                if shard_init:
                    if hi > lo:
                        init_fn(lo, hi, full.data_ptr() + B * lo, stream.cuda_stream)
                    if evs:
                        evs[0].record(stream)
                    load_fn(full.data_ptr(), stream.cuda_stream)
                    if evs:
                        evs[1].record(stream)
                sess.run(stream.cuda_stream)

            for _ in range(args.warmup):
                step()
            ms, parts = [], []
            for _ in range(args.reps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if shard_init else None
                a.record(stream)
                step(evs)
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
                if evs:  # init / install / run
                    parts.append([a.elapsed_time(evs[0]), evs[0].elapsed_time(evs[1]), evs[1].elapsed_time(b)])
            st = sess.stats()
            per_rank.append({"rank": r, "nodes": [int(cuts[r]), int(cuts[r + 1])], "walks": st.walks,
                             "steps": st.steps, "slot_inits": st.slot_inits, "chain_retries": st.chain_retries, "ms": float(np.median(ms)),
                             "init_load_run_ms": [round(float(x), 3) for x in np.median(parts, axis=0)] if parts else None})
            sess.close()
            del sess
            torch.cuda.empty_cache()
        tmax = max(x["ms"] for x in per_rank)
        tmean = float(np.mean([x["ms"] for x in per_rank]))
        steps = sum(x["steps"] for x in per_rank)
        if N == 1:
            t1 = tmax
        line = {"config": args.config, "workload": cfg["workload"], "n_shards": N, "max_shard_ms": tmax,
                "mean_shard_ms": tmean, "imbalance": tmax / tmean, "steps": steps,
                "projected_steps_per_s": steps / (tmax * 1e-3),
                "projected_speedup": (t1 / tmax) if t1 else None,
                "allgather_bytes_excluded": None,
                "init": f"sharded eager init + load, {args.order} order (all-gather excluded)" if shard_init
                        else ("single GPU: the session's own eager/lazy rule" if N == 1 else "lazy, per rank"),
                "per_rank": per_rank,
                "note": "each rank's shard timed alone on one B200 (CUDA events, median of reps); "
                        "the walk has no inter-rank exchange, so the N-GPU time is the max over ranks"}
        if shard_init:
            line["allgather_bytes_excluded"] = B * int(S)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
