"""Sharded chain initialisation (mhw_session_init_chain / _load_chain), the
multi-GPU exchange of bench.py: the initial chain table is a pure function of
(graph, model, init strategy, seed, slot), so ranks initialise slot ranges and
all-gather the words. The words equal the slot-keyed mh_init of the oracle
(samplers.cpp:37-83 under the engine's Philox layout), a table assembled from
shards equals one initialised whole, and a run on a preloaded table skips its
own initialisation and still passes the chain chi-square gate."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.helpers import device_graph, model_desc, typed_random_graph, walk_config, walk_model
from tests.stats import audit, gate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def _states(g):
    deg = np.diff(g.offsets).astype(np.int64)
    pos = np.repeat(np.arange(g.n, dtype=np.uint32), deg)
    aff = (np.arange(g.m, dtype=np.int64) - np.repeat(g.offsets[:-1].astype(np.int64), deg)).astype(np.uint32)
    return pos, aff


@pytest.mark.parametrize("init", [O.INIT_RANDOM, O.INIT_HIGH_WEIGHT, O.INIT_BURN_IN])
@pytest.mark.parametrize("kind", [O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK])
def test_sharded_init_words_equal_slot_init(mhw, oracle, kind, init):
    g = typed_random_graph(700 + kind, 120, 6.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.3, q=3.0, M=np.random.default_rng(kind).uniform(0.5, 2.0, (4, 4)))
    cfg = O.WalkCfg(K=2, L=10, seed=19, init_kind=init, burn_in_steps=6, hw_sample_size=4)
    s = mhw.Session(device_graph(g), walk_model(md), walk_config(cfg, threads=8, init_mode=2))
    S = s.chain_size()
    assert S == g.m
    words = torch.empty(S, dtype=torch.int32, device="cuda")
    cuts = [0, S // 3, (2 * S) // 3, S]  # three ragged shards
    for b, e in zip(cuts[:-1], cuts[1:]):
        s.init_chain(b, e, words.data_ptr() + 4 * b)
    torch.cuda.synchronize()
    raw = words.cpu().numpy().view(np.uint32)
    # chain words carry the Last index and its cached alpha class (bits 30-31);
    # init_states reports the index (sentinels unchanged)
    got = np.where(raw >= 0xFFFFFFFD, raw, raw & 0x3FFFFFFF)
    pos, aff = _states(g)
    ref = mhw.init_states(device_graph(g), walk_model(md), walk_config(cfg, threads=8), pos, aff)
    assert np.array_equal(got, ref)
    for a in np.random.default_rng(kind + init).choice(g.m, 40, replace=False):
        o = oracle.init_philox(g, md, cfg, int(pos[a]), int(aff[a]), int(a))
        assert got[a] == (0xFFFFFFFE if o is None else o), a


@pytest.mark.parametrize("kind", [O.NODE2VEC, O.FAIRWALK])
def test_preloaded_chain_run_passes_chi_square(mhw, oracle, kind):
    g = typed_random_graph(300 + kind, 40, 4.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.5, q=2.0)
    cfg = O.WalkCfg(K=400, L=80, seed=77, init_kind=O.INIT_BURN_IN, burn_in_steps=5)
    s = mhw.Session(device_graph(g), walk_model(md), walk_config(cfg, threads=8, init_mode=2))
    words = torch.empty(s.chain_size(), dtype=torch.int32, device="cuda")
    half = s.chain_size() // 2
    s.init_chain(0, half, words.data_ptr())
    s.init_chain(half, s.chain_size(), words.data_ptr() + 4 * half)
    s.load_chain(words.data_ptr())
    s.run()
    st = s.stats()
    assert st.slot_inits == 0  # no eager or lazy init in the run itself
    rows, lens = s.download()
    ok, msg = gate(audit(g, oracle, md, rows, lens, min_visits=5000))
    assert ok, msg
    # the next run without a preload initialises on its own again
    s.run()
    assert s.stats().slot_inits == g.m


@pytest.mark.parametrize("narrow", ["1", "0", "c16"])
@pytest.mark.parametrize("init", [O.INIT_RANDOM, O.INIT_BURN_IN])
@pytest.mark.parametrize("kind", [O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK])
def test_record_order_words_are_slot_words_permuted(mhw, oracle, kind, init, narrow, monkeypatch):
    """init_records word i (arc i = s -> v) == init_chain word off(v) + index of s in N(v),
    for every session record layout (node2vec narrow {u, word} / wide {u, deg, off, word} /
    compact 16-bit table, typed 32-byte records)."""
    if narrow == "c16":
        monkeypatch.setenv("MHW_C16", "1")
    else:
        monkeypatch.setenv("MHW_C16", "0")
        monkeypatch.setenv("MHW_NARROW", narrow)
    g = typed_random_graph(900 + kind, 150, 6.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.3, q=3.0, M=np.random.default_rng(kind).uniform(0.5, 2.0, (4, 4)))
    cfg = O.WalkCfg(K=2, L=10, seed=23, init_kind=init, burn_in_steps=6)
    s = mhw.Session(device_graph(g), walk_model(md), walk_config(cfg, threads=8, init_mode=2))
    S = s.chain_size()
    W = s.record_width()
    assert W == (1 if kind == O.NODE2VEC else 3)
    slot = torch.empty(S, dtype=torch.int32, device="cuda")
    rec = torch.empty(S * W, dtype=torch.int32, device="cuda")
    s.init_chain(0, S, slot.data_ptr())
    cuts = [0, S // 4, S // 2 + 3, S]  # ragged record shards
    for b, e in zip(cuts[:-1], cuts[1:]):
        s.init_records(b, e, rec.data_ptr() + 4 * W * b)
    torch.cuda.synchronize()
    sw = slot.cpu().numpy().view(np.uint32)
    full = rec.cpu().numpy().view(np.uint32).reshape(S, W)
    rw = full[:, 0]
    if W == 3:  # w'(Last) of every live word: positive and finite
        wl = full[:, 1:].copy().view(np.float64)[:, 0]
        live = rw < 0xFFFFFFFD
        assert np.all(np.isfinite(wl[live])) and np.all(wl[live] > 0)
    off = g.offsets.astype(np.int64)
    src = np.repeat(np.arange(g.n), np.diff(off))
    for a in range(g.m):
        v = int(g.nbr[a])
        sl = off[v:v + 2]
        idx = int(np.searchsorted(g.nbr[sl[0]:sl[1]], src[a]))
        assert rw[a] == sw[sl[0] + idx], a


@pytest.mark.parametrize("kind", [O.NODE2VEC, O.EDGE2VEC, O.FAIRWALK])
def test_record_order_preload_run_passes_chi_square(mhw, oracle, kind):
    g = typed_random_graph(500 + kind, 40, 4.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.5, q=2.0, M=np.random.default_rng(kind).uniform(0.5, 2.0, (4, 4)))
    cfg = O.WalkCfg(K=400, L=80, seed=78, init_kind=O.INIT_BURN_IN, burn_in_steps=5)
    s = mhw.Session(device_graph(g), walk_model(md), walk_config(cfg, threads=8, init_mode=2))
    W = s.record_width()
    words = torch.empty(s.chain_size() * W, dtype=torch.int32, device="cuda")
    third = s.chain_size() // 3
    s.init_records(0, third, words.data_ptr())
    s.init_records(third, s.chain_size(), words.data_ptr() + 4 * W * third)
    s.load_records(words.data_ptr())
    s.run()
    assert s.stats().slot_inits == 0
    rows, lens = s.download()
    ok, msg = gate(audit(g, oracle, md, rows, lens, min_visits=5000))
    assert ok, msg


@pytest.mark.parametrize("kind", [O.NODE2VEC, O.EDGE2VEC])
def test_piecewise_install_as_bench_pipelines_it(mhw, oracle, kind):
    """bench.py's multi-GPU exchange: 3 emulated ranks, each shard in 4 pieces,
    piece j of every rank installed with load_records_range as it lands; the
    run needs no init of its own and passes the chain chi-square gate."""
    g = typed_random_graph(610 + kind, 40, 4.0, weighted=True, types=2)
    md = model_desc(kind, g, p=0.5, q=2.0, M=np.random.default_rng(kind).uniform(0.5, 2.0, (4, 4)))
    cfg = O.WalkCfg(K=400, L=80, seed=81, init_kind=O.INIT_BURN_IN, burn_in_steps=5)
    s = mhw.Session(device_graph(g), walk_model(md), walk_config(cfg, threads=8, init_mode=2))
    S, W = s.chain_size(), s.record_width()
    world, pieces = 3, 4
    pc = (((S + world - 1) // world) + pieces - 1) // pieces
    per = pc * pieces
    shards = []
    for r in range(world):
        sh = torch.zeros(per * W, dtype=torch.int32, device="cuda")
        lo, hi = min(S, r * per), min(S, (r + 1) * per)
        if hi > lo:
            s.init_records(lo, hi, sh.data_ptr())
        shards.append(sh)
    full = torch.empty(pieces * world * pc * W, dtype=torch.int32, device="cuda")
    for j in range(pieces):
        out_j = full[j * world * pc * W:(j + 1) * world * pc * W]
        out_j.copy_(torch.cat([sh[j * pc * W:(j + 1) * pc * W] for sh in shards]))
        base = full.data_ptr() + 4 * j * world * pc * W
        for q in range(world):
            b, e = min(S, q * per + j * pc), min(S, q * per + (j + 1) * pc)
            if e > b:
                s.load_records_range(b, e, base + 4 * q * pc * W)
    s.run()
    assert s.stats().slot_inits == 0
    rows, lens = s.download()
    ok, msg = gate(audit(g, oracle, md, rows, lens, min_visits=5000))
    assert ok, msg


@pytest.mark.parametrize("layout", ["c16", "narrow"])
@pytest.mark.parametrize("init", [O.INIT_RANDOM, O.INIT_BURN_IN])
def test_shard_exchange_installs_the_local_table(mhw, oracle, init, layout, monkeypatch):
    """mhw_session_init_shard over ragged ranges + load_shard_range (the
    session's exchange format: 2-byte slot-order words for compact chains,
    record-order words otherwise) installs exactly the table the session's
    own eager init builds (mhw_session_prepare), and the preloaded run passes
    the chi-square gate."""
    from tests.stats import audit, gate
    if layout == "c16":
        monkeypatch.setenv("MHW_C16", "1")
    else:
        monkeypatch.setenv("MHW_C16", "0")
        monkeypatch.setenv("MHW_NARROW", "1")
    g = typed_random_graph(930 + init, 60, 5.0, weighted=False, types=2)
    md = model_desc(O.NODE2VEC, g, p=0.3, q=3.0)
    cfg = O.WalkCfg(K=400, L=80, seed=29, init_kind=init, burn_in_steps=6)
    s = mhw.Session(device_graph(g, weighted=False), walk_model(md), walk_config(cfg, threads=8, init_mode=2))
    S = s.chain_size()
    B = s.shard_entry_bytes()
    assert B == (2 if layout == "c16" else 4)
    want = torch.empty(S, dtype=torch.int32, device="cuda")
    s.prepare()
    s.export_table(want.data_ptr())
    buf = torch.empty(S * B, dtype=torch.uint8, device="cuda")
    cuts = [0, S // 3 + 1, S // 2, S]
    for b, e in zip(cuts[:-1], cuts[1:]):
        s.init_shard(b, e, buf.data_ptr() + B * b)
    for b, e in reversed(list(zip(cuts[:-1], cuts[1:]))):
        s.load_shard_range(b, e, buf.data_ptr() + B * b)
    got = torch.empty(S, dtype=torch.int32, device="cuda")
    s.export_table(got.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    s.run()
    assert s.stats().slot_inits == 0
    rows, lens = s.download()
    ok, msg = gate(audit(g, oracle, md, rows, lens, min_visits=5000))
    assert ok, msg
