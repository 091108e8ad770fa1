#!/usr/bin/env python
"""Benchmark: sampled walk steps/s of the M-H walk engine (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl mine|reference]

A step is one full generate_walks over the config's synthetic graph: chain
table reset (fresh sampler state, as every generate_walks call builds a new
SamplerManager, engine.cpp:167) + the walk kernel over all walkers of this
rank's start-node range. Graph generation (T_i) is outside the timed region.
Under torchrun (N > 1) walkers are partitioned into contiguous start-node
ranges balanced by active walkers; there is no collective in the walk path
(torch.distributed is used only for the barrier and the max-over-ranks time).

--impl reference times the reference's own CPU walk loop (oracle/_ref, the
unmodified reference library) on a bounded walker sample with all host
threads; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(workload="deepwalk R-MAT s16 ef16 fp32 U[1,10) K=10 L=80 random init", model="deepwalk",
                 scale=16, weighted=True, wlo=1.0, whi=10.0, K=10, L=80, init="random", p=1.0, q=1.0),
    "cfg2": dict(workload="node2vec p=0.25 q=4 R-MAT s20 ef16 unweighted K=10 L=80 burn-in 10",
                 model="node2vec", scale=20, weighted=False, K=10, L=80, init="burn_in", burn_in=10,
                 p=0.25, q=4.0),
    "cfg3a": dict(workload="metapath2vec A-P-V-P-A hetero 2M nodes fp32 U[1,5) K=10 L=80 random init",
                  model="metapath2vec", hetero=2_000_000, wlo=1.0, whi=5.0, K=10, L=80, init="random",
                  metapath=[0, 1, 2, 1, 0], p=1.0, q=1.0),
    "cfg3b": dict(workload="fairwalk p=q=1 groups=node type hetero 2M nodes K=10 L=80 random init",
                  model="fairwalk", hetero=2_000_000, wlo=1.0, whi=5.0, K=10, L=80, init="random", p=1.0, q=1.0),
    "cfg4": dict(workload="edge2vec p=1 q=2 R-MAT s22 fp32 U[1,10) 4 edge types K=10 L=80 random init",
                 model="edge2vec", scale=22, weighted=True, wlo=1.0, whi=10.0, etypes=4, K=10, L=80,
                 init="random", p=1.0, q=2.0),
    "cfg5": dict(workload="node2vec p=0.25 q=4 R-MAT s26 ef16 unweighted K=4 L=80 random init",
                 model="node2vec", scale=26, weighted=False, K=4, L=80, init="random", p=0.25, q=4.0),
}
SEED = 1
WALK_SEED = 42
METRIC = "walk steps/sec (sampled edges/s)"


def canonical_sectors(cfg, deg: np.ndarray) -> tuple[float, float]:
    """Algorithmic 32-B sectors per step S and E[sigma] over arcs."""
    d = deg[deg > 0].astype(np.float64)
    sig = np.maximum(1.0, np.ceil(np.log2(np.maximum(d, 1))) - 2)
    es = float(np.sum(d * sig) / np.sum(d)) if len(d) else 0.0
    w = 1.0 if cfg.get("weighted") or cfg.get("hetero") else 0.0
    base = 1 + 2 + (1 + w) + (1 + w) + 0.125
    m = cfg["model"]
    if m == "deepwalk":
        s = base
    elif m == "node2vec":
        s = base + 3 * es
    elif m == "metapath2vec":
        s = base + 2
    elif m == "fairwalk":
        alpha = 0 if (cfg["p"] == 1.0 and cfg["q"] == 1.0) else 2
        s = base + 4 + (alpha + 1) * es
    else:  # edge2vec
        s = base + 3 + 4 * es
    return s, es


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def type_matrix(cfg):
    r = np.random.default_rng(SEED)
    return r.uniform(0.5, 2.0, (cfg["etypes"], cfg["etypes"]))


def build_graph(cfg, device=0):
    import paper_2010_04895_b200 as mhw
    if "hetero" in cfg:
        return mhw.Graph.hetero(cfg["hetero"], seed=SEED, weight_lo=cfg["wlo"], weight_hi=cfg["whi"], device=device)
    g = mhw.Graph.rmat(cfg["scale"], 16, 0.57, 0.19, 0.19, seed=SEED, weighted=cfg["weighted"],
                       weight_lo=cfg.get("wlo", 1.0), weight_hi=cfg.get("whi", 10.0),
                       edge_types=cfg.get("etypes", 0), device=device)
    if cfg["model"] == "edge2vec":
        g.set_node_types(np.zeros(g.node_count(), dtype=np.uint16), 1)
    return g


def make_model(cfg):
    import paper_2010_04895_b200 as mhw
    return mhw.WalkModel(kind=mhw.ModelKind[cfg["model"]], p=cfg["p"], q=cfg["q"],
                         metapath=cfg.get("metapath", []),
                         type_matrix=type_matrix(cfg) if cfg["model"] == "edge2vec" else None)


def shard_init_pays(cfg, g):
    """Do the walks touch most arc-keyed slots (walker steps >= 2 x slots)?
    Then N ranks share one initialisation (each inits 1/N of the records,
    all-gather, coalesced install) instead of each rank initialising, eagerly
    or lazily, most of the table itself. cfg5 (steps = 5 x slots, lazy at N=1,
    every slot touched): 8 shards 205 -> 146 ms per rank
    (profiles/shard_scaling_r01.md)."""
    off = g.download()["offsets"]
    walkers = int(np.count_nonzero(np.diff(off))) * cfg["K"]
    return walkers * cfg["L"] >= 2 * int(off[-1])


def make_config(cfg, node_begin=0, node_end=0):
    import paper_2010_04895_b200 as mhw
    return mhw.WalkConfig(walks_per_node=cfg["K"], walk_length=cfg["L"], threads=8, seed=WALK_SEED,
                          init=mhw.InitStrategy(mhw.InitKind[cfg["init"]], cfg.get("burn_in", 100), 32),
                          schedule=mhw.Schedule.throughput, node_begin=node_begin, node_end=node_end,
                          chain_replica_degree=int(os.environ.get("MHW_REP_DEG", "0")),
                          sampler_kind=mhw.SamplerKind[cfg.get("sampler", "mh")],
                          init_mode=int(os.environ.get("MHW_INIT_MODE", "0")),
                          proposal=1 if cfg.get("proposal") == "alias" else 0)


class ShardInit:
    """Sharded chain-table initialisation of an N-rank run (the one exchange
    of the multi-GPU path; the walk itself has none). The initial table is a
    pure function of the slot (slot-keyed init draws), so each rank computes
    a contiguous 1/N of the entries in the session's exchange format
    (mhw_session_init_shard: compact node2vec chains -> 2-byte words in slot
    order; other layouts -> record-order entries, 4 or 12 bytes), the entries
    are all-gathered in PIECES pieces, and piece j of every rank is installed
    (mhw_session_load_shard_range) as soon as it lands while piece j+1 is in
    flight. Every rank ends with the table a single-GPU run builds
    (tests/test_gpu_dist_shard.py). host_coll: ranks sharing one GPU (gloo,
    through host memory; a path check, never timed)."""

    PIECES = 4

    def __init__(self, sess, rank, world, dist, dev, host_coll):
        import torch
        self.sess, self.rank, self.world, self.dist, self.host_coll = sess, rank, world, dist, host_coll
        S = self.S = sess.chain_size()
        B = self.B = sess.shard_entry_bytes()
        P = self.PIECES
        self.pc = pc = (((S + world - 1) // world) + P - 1) // P  # entries per piece per rank
        self.per = per = pc * P
        self.shard = torch.empty(max(per * B, 1), dtype=torch.uint8, device=dev)
        self.full = torch.empty(max(P * world * pc * B, 1), dtype=torch.uint8, device=dev)
        self.lo, self.hi = min(S, rank * per), min(S, (rank + 1) * per)
        self.dev = dev

    def __call__(self, stream) -> int:
        import torch
        sess, world, pc, B, S, per = self.sess, self.world, self.pc, self.B, self.S, self.per
        n_launch = 0
        if self.hi > self.lo:
            sess.init_shard(self.lo, self.hi, self.shard.data_ptr(), stream.cuda_stream)
            n_launch += 1
        works = []
        for j in range(self.PIECES):
            out_j = self.full[j * world * pc * B:(j + 1) * world * pc * B]
            src = self.shard[j * pc * B:(j + 1) * pc * B]
            if self.host_coll:
                torch.cuda.current_stream().wait_stream(stream)
                torch.cuda.synchronize(self.dev)
                parts = [torch.empty(pc * B, dtype=torch.uint8) for _ in range(world)]
                self.dist.all_gather(parts, src.cpu())
                out_j.copy_(torch.cat(parts).to(self.dev))
                torch.cuda.synchronize(self.dev)
                works.append(None)
            else:
                works.append(self.dist.all_gather_into_tensor(out_j, src, async_op=True))
        for j in range(self.PIECES):
            if works[j] is not None:
                works[j].wait()  # the install stream waits for piece j only
            base = self.full.data_ptr() + j * world * pc * B
            for q in range(world):
                b = min(S, q * per + j * pc)
                e = min(S, q * per + (j + 1) * pc)
                if e > b:
                    sess.load_shard_range(b, e, base + q * pc * B, stream.cuda_stream)
                    n_launch += 1
        return n_launch


class Clocks:
    """SM clock + throttle-reason sampling during the timed region.

    NVML from a host thread every 2 ms (a cfg1 timed region is ~10 ms, far
    shorter than nvidia-smi's 200 ms loop); nvidia-smi -lms is the fallback
    when pynvml is missing. The device is the physical index (one visible GPU)."""

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.nvml = None
        self.rows = []
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def _nvml_loop(self, h, N):
        bits = [("hw_slowdown", N.nvmlClocksEventReasonHwSlowdown),
                ("hw_thermal_slowdown", N.nvmlClocksEventReasonHwThermalSlowdown),
                ("sw_thermal_slowdown", N.nvmlClocksEventReasonSwThermalSlowdown),
                ("sw_power_cap", N.nvmlClocksEventReasonSwPowerCap)]
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((sm, mx, [n for n, b in bits if r & b]))
            except Exception:
                pass
            self.stop.wait(0.002)

    def __enter__(self):
        try:
            import threading
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() else self.device
            h = N.nvmlDeviceGetHandleByIndex(idx)
            self.stop = threading.Event()
            self.nvml = threading.Thread(target=self._nvml_loop, args=(h, N), daemon=True)
            self.nvml.start()
            return self
        except Exception:
            self.nvml = None
        return self._enter_smi()

    def _enter_smi(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.nvml.join(timeout=5)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.nvml:
            if not self.rows:
                return None
            reasons = sorted({n for _, _, rs in self.rows for n in rs})
            return {"sm_mhz": float(np.median([r[0] for r in self.rows])), "sm_max_mhz": float(self.rows[0][1]),
                    "reasons": reasons, "samples": len(self.rows), "source": "nvml 2 ms"}
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except Exception:
            return None
        rows = [[x.strip() for x in r] for r in rows if len(r) >= 9]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for i, n in enumerate(names):
                if r[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows)}


def reference_sample(cfg, threads, stride, oracle_graph=None):
    """The reference's own walk loop (oracle/_ref) over walkers idx = j*stride."""
    from oracle import oracle as O
    hg = oracle_graph or host_graph_for_reference(cfg)
    ref = O.RefLib()
    rg = ref.graph(hg)
    md = O.ModelDesc(kind=O.MODEL_NAMES.index(cfg["model"]), p=cfg["p"], q=cfg["q"],
                     metapath=cfg.get("metapath", []),
                     type_matrix=type_matrix(cfg) if cfg["model"] == "edge2vec" else None)
    rm = rg.model(md)
    wc = O.WalkCfg(K=cfg["K"], L=cfg["L"], seed=WALK_SEED, init_kind=["random", "high_weight", "burn_in"].index(cfg["init"]),
                   burn_in_steps=cfg.get("burn_in", 100), hw_sample_size=32)
    total = hg.n * cfg["K"]
    count = (total + stride - 1) // stride
    return hg, rg, rm, wc, count


def host_graph_for_reference(cfg):
    """cfg graph on the host in the reference's layout, built by the CPU
    oracle generator (identical to the device generator, see
    tests/test_gpu_parity.py::test_rmat_csr_bit_exact)."""
    from oracle import oracle as O
    o = O.Oracle()
    if "hetero" in cfg:
        lo, hi, nA, nP = o.hetero_pairs(cfg["hetero"], seed=SEED)
        w = o.pair_weights(SEED, lo, hi, cfg["wlo"], cfg["whi"]).astype(np.float64)
        hg = o.build_csr(lo, hi, w, symmetrize=True, n_nodes=cfg["hetero"])
        t = np.zeros(hg.n, dtype=np.uint16)
        t[nA:nA + nP] = 1
        t[nA + nP:] = 2
        hg.ntype, hg.n_ntypes = t, 3
        return hg
    lo, hi = o.rmat_pairs(cfg["scale"], 16, 0.57, 0.19, 0.19, seed=SEED)
    w = o.pair_weights(SEED, lo, hi, cfg["wlo"], cfg["whi"]).astype(np.float64) if cfg["weighted"] else None
    hg = o.build_csr(lo, hi, w, symmetrize=True, n_nodes=1 << cfg["scale"])
    if cfg.get("etypes"):
        src = np.repeat(np.arange(hg.n), np.diff(hg.offsets).astype(np.int64))
        a, b = np.minimum(src, hg.nbr), np.maximum(src, hg.nbr)
        hg.etype = o.pair_etypes(SEED, a, b, cfg["etypes"])
        hg.n_etypes = cfg["etypes"]
        hg.ntype, hg.n_ntypes = np.zeros(hg.n, dtype=np.uint16), 1
    return hg


def host_graph_from_device(g):
    from oracle import oracle as O
    d = g.download()
    w = d["weights"].astype(np.float64) if d["weights"] is not None else np.ones(len(d["neighbors"]))
    return O.HostGraph(d["offsets"].astype(np.uint64), d["neighbors"].astype(np.uint32), w, d["node_types"],
                       d["edge_types"], d["num_node_types"], d["num_edge_types"], True)


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def sample_stride(cfg):
    # about 10-20 s of reference CPU work on a many-core host
    return {"cfg1": 2, "cfg2": 192, "cfg3a": 16, "cfg3b": 16, "cfg4": 1024, "cfg5": 16384}[cfg["name"]]


def run_reference(args, cfg):
    """The reference's CPU walk generator on the FULL workload: one
    generate_walks-equivalent run (one SamplerManager over every walker, the
    engine's static thread partition, threads = all host cores) executed as
    `steps` time slices (oracle/ref_driver.cpp ref_run_slice): slice i walks
    the i-th 1/steps of every thread's walker block. The summed time is one
    full run's, lazy init amortised as in generate_walks; value = all sampled
    steps / summed slice time. Warm-up slices run on a separate throwaway
    manager (a 1/1000 walker sample), so the timed run starts fresh."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = cpu_threads()
    t0 = time.time()
    hg, rg, rm, wc, _ = reference_sample(cfg, threads, 1)
    setup = time.time() - t0
    warm = rm.full_run(wc, threads)
    for i in range(args.warmup):
        warm.slice(i, 1000)
    del warm
    run = rm.full_run(wc, threads)
    secs, steps_l, init_s = [], [], []
    for i in range(args.steps):
        st = run.slice(i, args.steps)
        secs.append(st["seconds"])
        steps_l.append(st["steps"])
        init_s.append(st["init_seconds"])
    del run
    value = float(np.sum(steps_l) / np.sum(secs))
    sample = (f"the full {cfg['name']} workload ({hg.n * cfg['K']} walker slots, {int(np.sum(steps_l))} steps) as "
              f"ONE generate_walks-equivalent run (one SamplerManager) in {args.steps} time slices of every "
              f"thread's walker block; {np.sum(secs):.1f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": cfg["workload"], "config": cfg["name"], "seed": SEED,
                                        "walk_seed": WALK_SEED},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": threads, "kind": "reference",
                         "sample": sample, "T_i_thread_seconds": float(np.sum(init_s)),
                         "T_w_seconds": max(0.0, float(np.sum(secs)) - float(np.sum(init_s)) / threads)},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_seconds": setup,
    }
    print(json.dumps(line), flush=True)


def run_mine(args, cfg):
    import torch
    import paper_2010_04895_b200 as mhw

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    n_dev = torch.cuda.device_count()
    dev = local % max(n_dev, 1)
    torch.cuda.set_device(dev)
    host_coll = False
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if n_dev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            # fewer GPUs than ranks (path check on one GPU): the barrier and
            # the max-over-ranks reduction go over gloo; no kernel of one rank
            # ever waits on another rank
            dist.init_process_group("gloo")
            host_coll = True
    t0 = time.time()
    g = build_graph(cfg, device=dev)
    model = make_model(cfg)
    cuts = mhw.partition_nodes(g, model, world)
    wcfg = make_config(cfg, int(cuts[rank]), int(cuts[rank + 1]))
    # Multi-GPU, second-order models whose walks touch most slots: the initial
    # table is a pure function of the slot, so each rank initialises 1/N of
    # the records (record order: the install is a coalesced strided copy) and
    # the words are all-gathered (the walk itself has no exchange).
    # --chain-init local: every rank initialises its own table (no collective
    # at all; the A/B of the exchange against the redundant per-rank init)
    shard_init = (world > 1 and args.chain_init == "sharded" and cfg["model"] in ("node2vec", "edge2vec", "fairwalk")
                  and cfg.get("sampler", "mh") == "mh" and shard_init_pays(cfg, g))
    if shard_init:
        wcfg.init_mode = 2
    sess = mhw.Session(g, model, wcfg)
    t_setup = time.time() - t0
    info = g.info()
    # a dedicated (non-legacy) stream: the walk kernels and the events that
    # time them are enqueued on the same stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    shard = ShardInit(sess, rank, world, dist, dev, host_coll) if shard_init else None

    def one_run():
        n_launch = shard(stream) if shard else 0
        sess.run(stream.cuda_stream)
        return sess.launches() + n_launch

    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    steps_total = 0
    launches = 0
    barrier()
    with Clocks(dev) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            n_launch = one_run()
            ev[i][1].record(stream)
            launches += n_launch
        barrier()
    ms = [a.elapsed_time(b) for a, b in ev]
    st = sess.stats()   # counters of the last run (identical work every run)
    steps_total = st.steps * args.steps
    t_local = sum(ms) * 1e-3
    kernel_ms = st.walk_seconds * 1e3
    args.coll_device = "cpu" if host_coll else dev
    t = torch.tensor([t_local, steps_total, launches], dtype=torch.float64, device=args.coll_device)
    if dist:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        t_job, steps_job, launches_job = float(tmax[0]), float(tsum[1]), int(tsum[2])
    else:
        t_job, steps_job, launches_job = t_local, float(steps_total), launches
    value = steps_job / t_job

    # ---- roofline of the walk kernel. frac: the kernel's measured DRAM bytes
    # per launch (ncu, profiles/traffic_<cfg>.json, same kernel variant) over
    # its live CUDA-event time, against the measured HBM copy bandwidth.
    # canonical: SURVEY 8(d)'s algorithmic sectors of the REFERENCE algorithm
    # (three binary searches per node2vec step); this design replaces those
    # searches (edge filter, hash sets, reverse index), so that figure exceeds
    # the bandwidth and is kept only for comparison. random: DRAM line fills
    # per second (128-B lines) against the measured random-access ceiling
    # (profiles/randbench_r01.md: 42-45 G independent random loads/s).
    off = g.download()["offsets"] if rank == 0 else None
    line = None
    if rank == 0:
        deg = np.diff(off)
        S, es = canonical_sectors(cfg, deg)
        peak, peak_kind = hbm_peak()
        t_k = kernel_ms * 1e-3
        canon = S * 32 * st.steps / t_k / 1e9
        tr = {}
        variant = "_alias" if cfg.get("proposal") == "alias" else ""
        prof = os.path.join(ROOT, "profiles", f"traffic_{cfg['name']}{variant}.json")
        if os.path.exists(prof):
            with open(prof) as f:
                tr = json.load(f)
        traffic = tr.get("dram_bytes_per_launch")
        achieved = traffic / t_k / 1e9 if traffic else None
        rd = tr.get("dram_read_bytes_per_launch")
        RAND_CEIL = 43e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                "traffic_source": (os.path.relpath(prof, ROOT) + f" (ncu --set full, tree {tr.get('tree')}, "
                                   f"{tr.get('ncu_ms')} ms under ncu)") if traffic else None,
                "peak_source": peak_kind,
                "dram_bytes_per_step": traffic / st.steps if traffic else None,
                "random": {"read_lines_per_s": rd / 128 / t_k, "ceiling_per_s": RAND_CEIL,
                           "frac": rd / 128 / t_k / RAND_CEIL} if rd else None,
                "canonical": {"sectors_per_step": S, "E_sigma": es, "achieved": canon, "frac": canon / peak,
                              "note": "SURVEY 8(d) reference-algorithm sectors (3 binary searches per step), "
                                      "not this kernel's traffic"},
                "kernel": "k_walk<%s>" % cfg["model"], "kernel_ms": kernel_ms,
                "init_ms": st.init_seconds * 1e3,
                "kernel_ms_note": "device time of one generate_walks' walk kernel (CUDA events on the launch "
                                  "stream, T_w); eager chain init (k_init_all / k_init_rec) is init_ms (T_i)"}
        if cfg.get("sampler", "mh") != "mh":
            roof = None  # the canonical sector count is the M-H path's
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_job / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded on-device R-MAT / hetero generators)",
            "config": {"workload": cfg["workload"], "config": cfg["name"], "nodes": info["node_count"],
                       "arcs": info["arc_count"], "walks": st.walks, "steps_per_run": st.steps,
                       "slot_inits": st.slot_inits, "chain_retries": st.chain_retries,
                       "sampler": cfg.get("sampler", "mh"), "proposal": cfg.get("proposal", "uniform"),
                       "rejection_trials": st.rejection_trials,
                       "seed": SEED, "walk_seed": WALK_SEED,
                       "l2": "explicit 256 MB L2 flush between timed steps (also inputs > L2)",
                       "parallelism": f"walker ranges x{world}, CSR replicated"
                                      + (", chain init sharded + all-gather" if shard_init else ""),
                       "chain_init": ("sharded + all-gather" if shard_init else
                                      ("per-rank" if world > 1 else "local"))},
            "roofline": roof, "clocks": clk.summary(), "gpu_launches": launches_job,
            "T_i_ms": st.init_seconds * 1e3, "T_w_ms": kernel_ms,
            "T_note": "per generate_walks (engine.cpp:228-232 split): T_i = eager chain-table init (k_init_all / "
                      "k_init_rec; 0 when init is lazy, fused into the walk), T_w = the walk kernel",
            "setup_seconds": t_setup,
        }
    # ---- e2e through the public C ABI with host buffers
    e2e = None if args.no_e2e else run_e2e(args, cfg, g, model, wcfg, dev, dist)
    if rank == 0:
        line["e2e"] = e2e
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, g)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, cfg, g, model, wcfg, dev, dist):
    """Per step: host CSR (pinned) -> mhw_graph_upload -> generate_walks into
    pinned host buffers (includes D2H) -> graph free."""
    import ctypes as C
    import torch
    import paper_2010_04895_b200 as mhw
    from paper_2010_04895_b200 import _lib as L

    d = g.download()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    off = pin(d["offsets"])
    nb = pin(d["neighbors"])
    w = pin(d["weights"]) if d["weights"] is not None else None
    nt = pin(d["node_types"]) if d["node_types"] is not None else None
    et = pin(d["edge_types"]) if d["edge_types"] is not None else None
    view = L.GraphView()
    view.node_count, view.arc_count = len(d["offsets"]) - 1, len(d["neighbors"])
    view.offsets, view.neighbors = off.data_ptr(), nb.data_ptr()
    view.weights = w.data_ptr() if w is not None else None
    view.node_types = nt.data_ptr() if nt is not None else None
    view.edge_types = et.data_ptr() if et is not None else None
    view.num_node_types, view.num_edge_types, view.symmetric = d["num_node_types"], d["num_edge_types"], 1
    md, keep = model._desc()
    c = wcfg._c()
    lib = L.lib()
    rows, stride = C.c_uint64(), C.c_uint32()
    mhw.mhwalk._check(lib.mhw_walk_rows(g.handle, C.byref(md), C.byref(c), C.byref(rows), C.byref(stride)))
    # packed corpus: walk r = nodes[offsets[r] .. offsets[r+1])
    cap = rows.value * (cfg["L"] + 1)
    out = torch.empty(max(cap, 1), dtype=torch.int32).pin_memory()
    offs = torch.empty(rows.value + 1, dtype=torch.int64).pin_memory()
    h2d = sum(x.numel() * x.element_size() for x in (off, nb, w, nt, et) if x is not None)
    steps_e2e = max(1, min(args.steps, 7))
    times, steps, d2h = [], 0, 0
    e2e_warm = max(3, args.warmup)
    for i in range(e2e_warm + steps_e2e):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        h = C.c_void_p()
        mhw.mhwalk._check(lib.mhw_graph_upload(C.byref(view), dev, C.byref(h)))
        st = L.WalkStatsC()
        try:
            mhw.mhwalk._check(lib.mhw_generate_walks_packed(h, C.byref(md), C.byref(c), C.c_void_p(out.data_ptr()),
                                                            cap, C.c_void_p(offs.data_ptr()), rows.value + 1,
                                                            C.byref(st)))
        finally:
            lib.mhw_graph_free(h)
        dt = time.perf_counter() - t0
        d2h = (st.walks + st.steps) * 4 + (rows.value + 1) * 8
        if i >= e2e_warm:
            times.append(dt)
            steps += st.steps
    # whole-run time of the calls (value); the median call is reported beside
    # it (one host hiccup in a few calls moves the mean by 10-20%)
    t_med = float(np.median(times)) * len(times)
    t_local = float(np.sum(times))
    if dist:
        tt = torch.tensor([t_med, t_local, float(steps)], dtype=torch.float64, device=args.coll_device)
        tmax = tt.clone()
        dist.all_reduce(tmax[:2], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[2:], op=dist.ReduceOp.SUM)
        t_med_job, t_job, steps_job = float(tmax[0]), float(tmax[1]), float(tt[2])
    else:
        t_med_job, t_job, steps_job = t_med, t_local, float(steps)
    return {"value": steps_job / t_job, "unit": "steps/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps_e2e, "ms_per_step": [round(1e3 * x, 2) for x in times],
            "value_median_call": steps_job / t_med_job,
            "path": "mhw_graph_upload + mhw_generate_walks_packed (pinned host buffers), wall clock"}


def cpu_baseline(cfg, g):
    """Bounded sample of the reference walk loop (about 20 s on the box) and,
    beside it, the committed full-workload measurement (scripts/cpu_full.py:
    one unmodified generate_walks over every walker, profiles/cpu_full_<cfg>.json).
    The sample runs every stride-th walker against a FRESH SamplerManager, so
    the lazy chain init (mh_init, O(deg) w' per slot; 82% of a full cfg2 run)
    is amortised over far fewer steps than in a full run: it is a lower bound
    of the reference's full-run rate, not an estimate of it."""
    full = None
    fp = os.path.join(ROOT, "profiles", f"cpu_full_{cfg['name']}.json")
    if os.path.exists(fp):
        with open(fp) as f:
            d = json.load(f)
        full = {"value": d["steps_per_sec"], "unit": "steps/s", "cores": d["threads"], "kind": "reference",
                "sample": f"the full workload, one unmodified generate_walks call ({d['steps']} steps, "
                          f"{d['seconds']:.1f} s; {os.path.relpath(fp, ROOT)}, measured by scripts/cpu_full.py)"}
    try:
        threads = cpu_threads()
        stride = sample_stride(cfg)
        hg = host_graph_from_device(g)
        _, rg, rm, wc, count = reference_sample(cfg, threads, stride, oracle_graph=hg)
        st = rm.walk_sample(wc, 0, stride, count, threads)
        return {"value": st["steps"] / st["seconds"], "unit": "steps/s", "cores": threads, "kind": "reference",
                "sample": f"every {stride}th walker ({count} walkers, {st['steps']} steps, "
                          f"{st['seconds']:.1f} s) through the unmodified reference library (oracle/_ref), "
                          "fresh SamplerManager: lazy init unamortised, a LOWER BOUND of the full-run rate",
                "full": full}
    except Exception as e:  # the reference library is optional on the box
        return {"value": full["value"] if full else None, "unit": "steps/s", "cores": cpu_threads(),
                "kind": "reference", "sample": f"sample unavailable: {e}", "full": full}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg")
    ap.add_argument("--sampler", default="mh", choices=["mh", "alias", "direct", "rejection"],
                    help="exact baseline samplers of next_edge (engine.cpp:88-116) for comparison")
    ap.add_argument("--chain-init", default="sharded", choices=["sharded", "local"],
                    help="N > 1, second-order models: sharded init + all-gather (default) or per-rank init")
    ap.add_argument("--proposal", default="uniform", choices=["uniform", "alias"],
                    help="M-H proposal: uniform (mh_transition) or the static-weight alias table + Hastings")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    cfg["name"] = args.config
    cfg["sampler"] = args.sampler
    cfg["proposal"] = args.proposal
    if args.sampler != "mh":
        args.no_cpu_baseline = True  # the CPU arm times the M-H path
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_mine(args, cfg)


if __name__ == "__main__":
    main()
