"""Walk rows of the throughput kernel at every walk length and row phase.

k_walk stages a walker's ids in shared memory and writes them as whole
aligned sectors, 16 ids per flush (walk.cu: rowbuf); a row starts at slot
(row * stride) mod 16 of its first group, so first groups are partial for
most rows and the last group of a row is written id by id. The walk lengths
below put the end of a row at every offset of a group and the stride at every
residue, with K walkers per start node so neighbouring rows come from
different threads. Each row must be an intact walk (engine.cpp:178-205: the
start node, then an arc of the graph per step, L + 1 ids on a connected
symmetric graph); one walker alone must equal the oracle's isolated walker
byte for byte (as tests/test_gpu_kwalk_pin.py does at BASELINE scale).
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import device_graph, model_desc, typed_random_graph, walk_config, walk_model

pytestmark = pytest.mark.gpu

LENGTHS = [1, 2, 3, 4, 6, 7, 8, 11, 12, 14, 15, 16, 17, 19, 30, 31, 32, 33, 47, 48, 63, 64, 79, 80, 81, 95, 97]


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def arc_set(g):
    off = g.offsets.astype(np.int64)
    src = np.repeat(np.arange(len(off) - 1, dtype=np.int64), np.diff(off))
    return set((src << 32 | g.nbr.astype(np.int64)).tolist())


def test_metapath_rows_are_intact_walks_at_every_length(mhw):
    """metapath2vec stages 32 ids per flush and its walks end early where no
    neighbour has the required type: every row must be the start node followed
    by arcs of the graph over its own length, whatever that length is."""
    g = typed_random_graph(13, 400, 6.0)
    arcs = arc_set(g)
    deg = np.diff(g.offsets.astype(np.int64))
    dg = device_graph(g)
    md = model_desc(O.METAPATH2VEC, g)
    for L in LENGTHS:
        for K in (1, 3):
            c = mhw.generate_walks(dg, walk_model(md), walk_config(O.WalkCfg(K=K, L=L, seed=7 + L), threads=8))
            starts = np.repeat(np.nonzero((deg > 0) & (g.ntype == md.metapath[0]))[0], K)
            assert len(c.lengths) == len(starts), (L, K)
            assert np.array_equal(c.rows[:, 0], starts), (L, K)
            assert np.all((c.lengths >= 1) & (c.lengths <= L + 1))
            steps = 0
            for r in range(len(starts)):
                n = int(c.lengths[r])
                row = c.rows[r, :n].astype(np.int64)
                assert all(int(k) in arcs for k in (row[:-1] << 32 | row[1:])), (L, K, r)
                steps += n - 1
            assert c.stats.steps == steps


@pytest.mark.parametrize("kind", [O.DEEPWALK, O.NODE2VEC, O.EDGE2VEC])
def test_rows_are_intact_walks_at_every_length(mhw, kind):
    g = typed_random_graph(11, 400, 5.0)
    arcs = arc_set(g)
    deg = np.diff(g.offsets.astype(np.int64))
    dg = device_graph(g)
    md = model_desc(kind, g)
    for L in LENGTHS:
        for K in (1, 3):
            c = mhw.generate_walks(dg, walk_model(md), walk_config(O.WalkCfg(K=K, L=L, seed=5 + L), threads=8))
            starts = np.repeat(np.nonzero(deg > 0)[0], K)
            assert len(c.lengths) == len(starts), (L, K)
            assert c.rows.shape[1] == (L + 1 + 3) // 4 * 4
            assert np.array_equal(c.rows[:, 0], starts), (L, K)
            assert np.all(c.lengths == L + 1), (L, K)
            a = c.rows[:, :L].astype(np.int64)
            b = c.rows[:, 1:L + 1].astype(np.int64)
            keys = (a << 32 | b).ravel().tolist()
            assert all(k in arcs for k in keys), (kind, L, K)
            assert c.stats.steps == len(starts) * L


@pytest.mark.parametrize("L", [5, 16, 23, 80, 97])
def test_single_walkers_equal_oracle_at_odd_lengths(mhw, oracle, L):
    g = typed_random_graph(12, 300, 6.0)
    md = model_desc(O.NODE2VEC, g, p=0.25, q=4.0)
    cfg = O.WalkCfg(K=1, L=L, seed=9, init_kind=O.INIT_BURN_IN, burn_in_steps=5)
    starts = np.nonzero(np.diff(g.offsets.astype(np.int64)) > 0)[0][::7].astype(np.uint32)
    orows, olens, _ = oracle.walk_isolated(g, md, cfg, starts)
    s = mhw.Session(device_graph(g), walk_model(md), walk_config(cfg, threads=8))
    for j, v in enumerate(starts):
        s.select_starts([int(v)])
        s.run()
        rows, lens = s.download()
        assert lens[0] == olens[j] == L + 1
        assert np.array_equal(rows[0, :lens[0]], orows[j, :olens[j]]), (L, int(v))
    s.close()
