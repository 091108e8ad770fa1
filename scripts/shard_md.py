"""Writes profiles/shard_scaling_r01.md from gpurun_out/shard_<cfg>.jsonl (scripts/shard_scaling.py)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = ["# Per-shard scaling, round 1 (one B200; `python scripts/shard_scaling.py --config <cfg>`)", "",
       "Each rank's shard of an N-GPU run (start-node range balanced by active walkers, CSR replica,",
       "private chain table) timed alone on one B200: CUDA events around the bench step (chain",
       "reset/init + walk; sharded configs: init of the rank's 1/N of the records + coalesced install",
       "+ walk), 256 MB L2 flush between reps, median of 3. The walk has no inter-rank exchange, so the",
       "N-GPU step time is the max over ranks; the only collective, the all-gather of the initial",
       "chain table (bytes listed), is not included. A projection from measured per-rank device times,",
       "not a multi-GPU measurement (gpurun exposes one GPU). The last two columns add the all-gather",
       "at the profiling guide's measured NVLink bus bandwidth (725 GB/s, 8-rank all-reduce at 1 GiB):",
       "each rank receives (N-1)/N of the table. bench.py gathers the table in 4 pieces and installs",
       "piece j while piece j+1 is in flight; the last column estimates that overlap as",
       "init + max(all-gather, install) + min(all-gather, install)/4 + walk on the slowest rank.", "",
       "| config | N | max shard ms | mean shard ms | max/mean | projected speed-up | projected G steps/s | init | all-gather bytes | + all-gather ms (est.) | speed-up incl. all-gather | pipelined all-gather + install |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for c in ["cfg1", "cfg2", "cfg3a", "cfg3b", "cfg4", "cfg5"]:
    p = os.path.join(ROOT, "gpurun_out", f"shard_{c}.jsonl")
    if not os.path.exists(p):
        continue
    for line in open(p):
        d = json.loads(line)
        N = d["n_shards"]
        if N == 1:
            t1 = d["max_shard_ms"]
        ag = d.get("allgather_bytes_excluded") or 0
        t_ag = ag * (N - 1) / N / 725e9 * 1e3
        pipe = "-"
        worst = max(d["per_rank"], key=lambda r: r["ms"])
        if ag and worst.get("init_load_run_ms"):
            i0, ins, wk = worst["init_load_run_ms"]
            tp = i0 + max(t_ag, ins) + min(t_ag, ins) / 4 + wk
            pipe = f"{t1 / tp:.2f}"
        out.append(f"| {c} | {N} | {d['max_shard_ms']:.2f} | {d['mean_shard_ms']:.2f} | "
                   f"{d['imbalance']:.3f} | {d['projected_speedup']:.2f} | {d['projected_steps_per_s'] / 1e9:.2f} | "
                   f"{d['init']} | {ag or '-'} | {t_ag:.2f} | {t1 / (d['max_shard_ms'] + t_ag):.2f} | {pipe} |")
out += ["", "Per-rank detail (N = 8):", ""]
for c in ["cfg2", "cfg4", "cfg5"]:
    p = os.path.join(ROOT, "gpurun_out", f"shard_{c}.jsonl")
    if not os.path.exists(p):
        continue
    for line in open(p):
        d = json.loads(line)
        if d["n_shards"] != 8:
            continue
        out += [f"### {c}", "", "| rank | nodes | walks | steps | ms | init / install / walk ms |", "|---|---|---|---|---|---|"]
        for r in d["per_rank"]:
            out.append(f"| {r['rank']} | {r['nodes'][0]}-{r['nodes'][1]} | {r['walks']} | {r['steps']} | {r['ms']:.2f} | "
                       f"{r.get('init_load_run_ms')} |")
        out.append("")
with open(os.path.join(ROOT, "profiles", "shard_scaling_r01.md"), "w") as fh:
    fh.write("\n".join(out) + "\n")
print("wrote", len(out), "lines")
