"""The static-weight alias proposal of the M-H step (north star (2): "proposes
a candidate from the uniform or static-weight alias proposal"; SURVEY 8(b)
`proposal {uniform, alias}`): the candidate comes from v's static alias table
(alias_build, samplers.cpp:95-131, sampled as alias_sample, samplers.hpp:
65-68) and is accepted with the Hastings-corrected ratio min(1, r_c / r_l),
r = w'/w. The reference has no such proposal, so the oracle's restatement
(og_hastings, mh_transition_alias) is the contract; it is pinned here by

* decisions bit for bit on identical (state, cand, last, u) triples,
* single walkers (deterministic when alone) byte for byte against the
  oracle's isolated walkers, on small graphs for every model and init and on
  the full BASELINE graphs (k_walk's AR = 4 variant),
* the chain chi-square of throughput corpora under the alias kernel
  (tests/stats.py mh_kernel with q ~ static weights).
"""
import dataclasses

import numpy as np
import pytest

import bench
from oracle import oracle as O
from tests.helpers import (INITS, KINDS, device_graph, model_desc, random_triples, typed_random_graph, walk_config,
                           walk_model)
from tests.stats import audit, gate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


@pytest.mark.parametrize("weighted", [True, False])
@pytest.mark.parametrize("kind", KINDS)
def test_hastings_decisions_bit_exact(mhw, oracle, kind, weighted):
    g = typed_random_graph(41 + kind, 300, 6.0, weighted=weighted, types=3)
    md = model_desc(kind, g, p=0.37, q=1.9, metapath=(0, 1, 2, 1, 0),
                    M=np.random.default_rng(6).uniform(0.5, 2.0, (9, 9)))
    dg = device_graph(g, weighted)
    pos, aff, cand, last, u = random_triples(g, md, 20000, seed=kind)
    orc, orl, _ = oracle.decide_hastings(g, md, pos, aff, cand, last, u)
    # unit draws at the decision boundary (u = r_c / r_l +- 1 ulp)
    ratio = np.where(orl > 0, orc / np.where(orl > 0, orl, 1), 0.5)
    k = len(u) // 4
    u[:k] = np.clip(ratio[:k], 0, np.nextafter(1, 0))
    u[k:2 * k] = np.clip(np.nextafter(ratio[k:2 * k], 2), 0, np.nextafter(1, 0))
    u[2 * k:3 * k] = np.clip(np.nextafter(ratio[2 * k:3 * k], -1), 0, np.nextafter(1, 0))
    orc, orl, oacc = oracle.decide_hastings(g, md, pos, aff, cand, last, u)
    grc, grl, gacc = mhw.decide_hastings(dg, walk_model(md), pos, aff, cand, last, u)
    assert np.array_equal(orc.view(np.uint64), grc.view(np.uint64))
    assert np.array_equal(orl.view(np.uint64), grl.view(np.uint64))
    assert np.array_equal(oacc, gacc)
    if kind == O.DEEPWALK:  # q = pi: every positive-weight proposal is accepted
        assert np.all(oacc == 1)
    else:
        assert 0 < oacc.mean() < 1


def isolated_equal(mhw, oracle, g, md, cfg, starts, weighted=True, **wkw):
    s = mhw.Session(device_graph(g, weighted), walk_model(md), walk_config(cfg, threads=8, proposal=1, **wkw))
    orows, olens, _ = oracle.walk_isolated(g, md, cfg, starts)
    for j, v in enumerate(starts):
        s.select_starts([int(v)])
        s.run()
        rows, lens = s.download()
        assert lens[0] == olens[j], (int(v), int(lens[0]), int(olens[j]))
        assert np.array_equal(rows[0, :lens[0]], orows[j, :olens[j]]), int(v)
        assert s.stats().chain_retries == 0
    s.close()


@pytest.mark.parametrize("records", ["1", "0"])
@pytest.mark.parametrize("init", INITS)
@pytest.mark.parametrize("kind", KINDS)
def test_single_walkers_equal_oracle(mhw, oracle, kind, init, records, monkeypatch):
    """Both alias variants of k_walk: on the arc records (AR 5, default) and
    on the plain CSR (AR 4, MHW_ARC_RECORDS=0)."""
    monkeypatch.setenv("MHW_ARC_RECORDS", records)
    g = typed_random_graph(60 + kind, 120, 5.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.4, q=2.5, M=np.random.default_rng(kind).uniform(0.5, 2.0, (4, 4)))
    deg = np.diff(g.offsets.astype(np.int64))
    ok = deg > 0
    if kind == O.METAPATH2VEC:
        ok &= g.ntype == md.metapath[0]
    starts = np.nonzero(ok)[0][::3].astype(np.uint32)
    for init_mode in (1, 2):  # lazy first-touch and eager tables
        cfg = O.WalkCfg(K=1, L=40, seed=13 + init, init_kind=init, burn_in_steps=6, hw_sample_size=4, proposal=1)
        isolated_equal(mhw, oracle, g, md, cfg, starts, init_mode=init_mode)


def test_unweighted_alias_equals_oracle(mhw, oracle):
    """Unweighted graphs: every alias prob is 1.0 (no table is built; the
    coin is drawn and always keeps the index)."""
    g = typed_random_graph(77, 150, 6.0, weighted=False, types=2)
    md = model_desc(O.NODE2VEC, g, p=0.25, q=4.0)
    starts = np.nonzero(np.diff(g.offsets.astype(np.int64)) > 0)[0][::2].astype(np.uint32)
    cfg = O.WalkCfg(K=1, L=40, seed=3, init_kind=O.INIT_BURN_IN, burn_in_steps=5, proposal=1)
    isolated_equal(mhw, oracle, g, md, cfg, starts, weighted=False, init_mode=2)


@pytest.mark.parametrize("kind", KINDS)
def test_throughput_alias_corpus_passes_chain_chi_square(mhw, oracle, kind):
    g = typed_random_graph(700 + kind, 40, 4.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.5, q=2.0, M=np.random.default_rng(kind).uniform(0.5, 2.0, (4, 4)))
    cfg = O.WalkCfg(K=400, L=80, seed=77, init_kind=O.INIT_RANDOM, proposal=1)
    c = mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=8, proposal=1))
    assert c.stats.chain_retries > 0  # contended chains (the lock protocol under load)
    ok, msg = gate(audit(g, oracle, md, c.rows, c.lengths, min_visits=5000, alias_proposal=True))
    assert ok, msg


def test_alias_proposal_validation(mhw):
    g = typed_random_graph(5, 30, 3.0)
    md = model_desc(O.NODE2VEC, g)
    cfg = O.WalkCfg(K=1, L=5, seed=1)
    with pytest.raises(mhw.ValidationError, match="throughput schedule"):
        mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=1, proposal=1))
    with pytest.raises(mhw.ValidationError, match="unknown proposal"):
        mhw.generate_walks(device_graph(g), walk_model(md), walk_config(cfg, threads=8, proposal=7))


@pytest.mark.parametrize("cfg_name", ["cfg1", "cfg3a", "cfg3b", "cfg4"])
def test_alias_proposal_single_walkers_on_baseline_graphs(mhw, oracle, cfg_name):
    """k_walk's alias variant on the full weighted BASELINE graphs (hub
    replicas, typed slot init, weighted bootstrap), ~600 starts each."""
    from tests.test_gpu_kwalk_pin import pin
    n, steps = pin(mhw, oracle, cfg_name, n_starts=600, proposal=1)
    assert n >= 500 and steps > 40 * n
