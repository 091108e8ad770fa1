"""Multi-rank host logic on CPU (gloo, world_size 2): the walker partition,
the per-rank row ranges, the corpus gather order and the max-over-ranks /
sum-over-ranks reductions bench.py performs. The per-rank walk itself is the
CPU oracle here (tests may use it); on GPUs it is libmhw.so."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2010_04895_b200.partition import balanced_cuts, imbalance, rows_in_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph():
    rng = O.XoRng(5)
    g = O.random_graph(90, 3.0, True, rng, ensure_connected=False)
    O.assign_random_types(g, 2, rng)
    return g


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oracle = O.Oracle()
        g = _graph()
        md = O.ModelDesc(O.METAPATH2VEC, metapath=[0, 1, 0])
        cfg = O.WalkCfg(K=3, L=12, seed=11, init_kind=O.INIT_RANDOM)
        rows, lens, st = oracle.generate_walks(g, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
        deg = np.diff(g.offsets).astype(np.int64)
        valid = g.ntype == md.metapath[0]
        cuts = balanced_cuts(deg, world, valid)
        a, b = rows_in_range(cuts, rank, cfg.K, valid, g.n)
        mine = torch.from_numpy(rows[a:b].astype(np.int64))
        my_len = torch.from_numpy(lens[a:b].astype(np.int64))
        # gather variable-length shards in rank order (the corpus order)
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(counts, torch.tensor([b - a]))
        mx = int(max(c.item() for c in counts))
        pad = torch.zeros((mx, rows.shape[1]), dtype=torch.int64)
        pad[:b - a] = mine
        padl = torch.zeros(mx, dtype=torch.int64)
        padl[:b - a] = my_len
        shards = [torch.zeros_like(pad) for _ in range(world)]
        lshards = [torch.zeros_like(padl) for _ in range(world)]
        dist.all_gather(shards, pad)
        dist.all_gather(lshards, padl)
        full = torch.cat([s[:int(c.item())] for s, c in zip(shards, counts)]).numpy()
        full_len = torch.cat([s[:int(c.item())] for s, c in zip(lshards, counts)]).numpy()
        # bench.py reductions: value = sum(steps) / max(time)
        steps = torch.tensor([float(np.sum(lens[a:b] - 1))], dtype=torch.float64)
        t = torch.tensor([0.5 + rank], dtype=torch.float64)
        dist.all_reduce(steps, op=dist.ReduceOp.SUM)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = (np.array_equal(full, rows.astype(np.int64)) and np.array_equal(full_len, lens)
              and steps.item() == st["steps"] and t.item() == 0.5 + world - 1)
        q.put((rank, ok, int(cuts[1]), imbalance(deg, cuts, valid)))
    finally:
        dist.destroy_process_group()


def test_two_rank_partition_and_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res), res
    assert res[0][2] == res[1][2]          # both ranks computed the same cut
    assert max(r[3] for r in res) < 1.1    # balanced by active walkers


def test_balanced_cuts_beat_equal_ranges():
    """R-MAT piles isolated nodes at high ids: equal id ranges are unbalanced,
    active-walker cuts are not."""
    oracle = O.Oracle()
    lo, hi = oracle.rmat_pairs(14, 16, seed=1)
    hg = oracle.build_csr(lo, hi, None, symmetrize=True, n_nodes=1 << 14)
    deg = np.diff(hg.offsets).astype(np.int64)
    for parts in (2, 4, 8):
        eq = np.linspace(0, len(deg), parts + 1).astype(np.int64)
        assert imbalance(deg, balanced_cuts(deg, parts)) < 1.01
        assert imbalance(deg, eq) > 1.05
