"""bench.py's multi-GPU path on libmhw.so, with two processes (gloo) sharing
one GPU: partition of the walkers by balanced start-node ranges
(engine.cpp:179-185 partitions by thread), the sharded chain-table
initialisation (each rank computes 1/N of the records, all-gather in pieces,
coalesced install: bench.ShardInit) and the walk of every rank's range.

* every rank's installed table equals the table a single-GPU session builds
  for itself (mhw_session_prepare + mhw_session_export_table), for the
  node2vec compact-chain layout and the narrow / wide record layouts and the
  typed records of edge2vec / fairwalk;
* the rank corpora, concatenated in rank order, hold exactly the single-GPU
  run's rows (reference corpus order: walker v*K + k, skipped starts
  omitted), every walk of full length or ending at a dead end, and every
  consecutive pair is an arc;
* gloo carries the exchange here; on a GPU per rank it is NCCL. No kernel of
  one rank ever waits on another rank.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = {
    "node2vec_c16": ("node2vec", {"MHW_C16": "1"}),
    "node2vec_narrow": ("node2vec", {"MHW_C16": "0", "MHW_NARROW": "1"}),
    "node2vec_wide": ("node2vec", {"MHW_C16": "0", "MHW_NARROW": "0"}),
    "edge2vec": ("edge2vec", {}),
    "fairwalk": ("fairwalk", {}),
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph(mhw, model):
    import bench
    if model == "fairwalk":
        cfg = dict(bench.CONFIGS["cfg3b"], hetero=30000)
        g = mhw.Graph.hetero(cfg["hetero"], seed=3, weight_lo=1.0, weight_hi=5.0)
    else:
        cfg = dict(bench.CONFIGS["cfg4" if model == "edge2vec" else "cfg2"], scale=12)
        g = mhw.Graph.rmat(12, 16, 0.57, 0.19, 0.19, seed=3, weighted=cfg["weighted"], weight_lo=1.0,
                           weight_hi=10.0, edge_types=cfg.get("etypes", 0))
        if model == "edge2vec":
            g.set_node_types(np.zeros(g.node_count(), dtype=np.uint16), 1)
    cfg["K"], cfg["L"] = 4, 30
    return cfg, g


def _worker(rank, world, port, model, env, out):
    for k, v in env.items():
        os.environ[k] = v
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    import bench
    import paper_2010_04895_b200 as mhw
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream(0)
    torch.cuda.set_stream(stream)
    cfg, g = _graph(mhw, model)
    mdl = bench.make_model(cfg)
    cuts = mhw.partition_nodes(g, mdl, world)
    wcfg = bench.make_config(cfg, int(cuts[rank]), int(cuts[rank + 1]))
    wcfg.init_mode = 2
    sess = mhw.Session(g, mdl, wcfg)
    shard = bench.ShardInit(sess, rank, world, dist, 0, host_coll=True)
    shard(stream)
    S = sess.chain_size()
    tab = torch.empty(S, dtype=torch.int32, device="cuda")
    sess.export_table(tab.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    sess.run(stream.cuda_stream)
    rows, lens = sess.download(stream=stream.cuda_stream)  # same stream as the walk
    out[rank] = dict(table=tab.cpu().numpy().view(np.uint32).copy(), rows=rows, lens=lens,
                     cuts=(int(cuts[rank]), int(cuts[rank + 1])))
    sess.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(CASES))
def test_two_rank_shard_path_equals_single_gpu(case):
    import torch
    import bench
    import paper_2010_04895_b200 as mhw
    model, env = CASES[case]
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        cfg, g = _graph(mhw, model)
        mdl = bench.make_model(cfg)
        wcfg = bench.make_config(cfg)
        wcfg.init_mode = 2
        s = mhw.Session(g, mdl, wcfg)
        S = s.chain_size()
        tab = torch.empty(S, dtype=torch.int32, device="cuda")
        s.prepare()
        s.export_table(tab.data_ptr())
        torch.cuda.synchronize()
        want = tab.cpu().numpy().view(np.uint32).copy()
        s.run()
        rows1, lens1 = s.download()
        s.close()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ctx = mp.get_context("spawn")
    with ctx.Manager() as man:
        out = man.dict()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, model, env, out)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(300)
            assert p.exitcode == 0
        res = [out[r] for r in range(2)]
    for r in range(2):
        assert np.array_equal(res[r]["table"], want), f"rank {r} table differs from the single-GPU table"
    assert res[0]["cuts"][1] == res[1]["cuts"][0]
    rows = np.concatenate([res[r]["rows"] for r in range(2)])
    lens = np.concatenate([res[r]["lens"] for r in range(2)])
    assert len(lens) == len(lens1)
    bad = np.nonzero(rows[:, 0] != rows1[:, 0])[0]
    assert len(bad) == 0, (case, res[0]["cuts"], bad[:5], rows[bad[:5], 0], rows1[bad[:5], 0], len(res[0]["lens"]))
    d = g.download()
    off = d["offsets"].astype(np.int64)
    nb = d["neighbors"].astype(np.int64)
    deg = np.diff(off)
    arcs = set(zip(np.repeat(np.arange(len(deg)), deg).tolist(), nb.tolist()))
    for i in range(len(lens)):
        w = rows[i, :lens[i]].astype(np.int64)
        # symmetric graphs, positive weights: no dead ends (isolated starts: the start alone)
        assert lens[i] == (cfg["L"] + 1 if deg[w[0]] else 1)
        for a, b in zip(w[:-1], w[1:]):
            assert (int(a), int(b)) in arcs
