"""Device ingestion (mhw_graph_load_edge_list / _node_types / _edge_types):
the CSR equals build_csr of the same text (graph.cpp:35-100) and the type
loaders follow graph.cpp:102-177, including their errors."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mhw():
    import paper_2010_04895_b200 as m
    assert m.device_count() > 0
    return m


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("sym", [False, True])
def test_load_edge_list_csr(mhw, oracle, tmp_path, weighted, sym):
    lo, hi = oracle.rmat_pairs(12, 16, seed=5)
    w = oracle.pair_weights(5, lo, hi, 1.0, 10.0)
    lines = [f"{a} {b} {float(x):.17g}" if weighted else f"{a} {b}" for a, b, x in zip(lo, hi, w)]
    # sprinkle comments, blanks and a duplicate (summed by build_csr)
    lines.insert(10, "# comment")
    lines.insert(20, "")
    lines.append(lines[30])
    path = write(tmp_path, "g.txt", "\n".join(lines) + "\n")
    g = mhw.load_edge_list(path, weighted=weighted, symmetrize=sym)
    src = [int(l.split()[0]) for l in lines if l and not l.startswith("#")]
    dst = [int(l.split()[1]) for l in lines if l and not l.startswith("#")]
    ww = [float(l.split()[2]) for l in lines if l and not l.startswith("#")] if weighted else None
    hg = oracle.build_csr(src, dst, ww, symmetrize=sym)
    d = g.download()
    assert np.array_equal(d["offsets"].astype(np.uint64), hg.offsets)
    assert np.array_equal(d["neighbors"].astype(np.uint32), hg.nbr)
    got_w = d["weights"].astype(np.float64) if d["weights"] is not None else np.ones(len(hg.nbr))
    assert np.array_equal(got_w, hg.w.astype(np.float32).astype(np.float64))
    assert g.info()["symmetric"] == int(sym)


def test_load_errors(mhw, tmp_path):
    with pytest.raises(mhw.IoError):
        mhw.load_edge_list(str(tmp_path / "missing.txt"))
    p = write(tmp_path, "bad.txt", "0 1\nbogus\n")
    with pytest.raises(mhw.ParseError, match=":2: expected"):
        mhw.load_edge_list(p)
    p = write(tmp_path, "neg.txt", "0 1 -3\n")
    with pytest.raises(mhw.ValidationError, match="negative edge weight"):
        mhw.load_edge_list(p, weighted=True)


def test_node_and_edge_type_files(mhw, tmp_path):
    """load_node_types / load_edge_types: coverage, unknown ids, symmetric
    typing of both directions (test_graph.cpp:64-83)."""
    g = mhw.load_edge_list(write(tmp_path, "t.txt", "0 1\n1 2\n2 0\n"), symmetrize=True)
    mhw.load_node_types(g, write(tmp_path, "nt.txt", "0 0\n1 1\n2 0\n"))
    d = g.download()
    assert list(d["node_types"]) == [0, 1, 0] and d["num_node_types"] == 2
    with pytest.raises(mhw.ValidationError, match="node 2 has no type assignment"):
        mhw.load_node_types(g, write(tmp_path, "nt2.txt", "0 0\n1 1\n"))
    with pytest.raises(mhw.ValidationError, match="unknown node id 9"):
        mhw.load_node_types(g, write(tmp_path, "nt3.txt", "0 0\n1 1\n2 0\n9 1\n"))
    mhw.load_edge_types(g, write(tmp_path, "et.txt", "0 1 0\n1 2 1\n2 0 2\n"))
    d = g.download()
    # arcs in CSR order: 0->1, 0->2, 1->0, 1->2, 2->0, 2->1
    assert list(d["edge_types"]) == [0, 2, 0, 1, 2, 1] and d["num_edge_types"] == 3
    with pytest.raises(mhw.ValidationError, match="edge not present in graph"):
        mhw.load_edge_types(g, write(tmp_path, "et2.txt", "0 1 0\n0 0 1\n"))
    with pytest.raises(mhw.ValidationError, match="has no type assignment"):
        mhw.load_edge_types(g, write(tmp_path, "et3.txt", "0 1 0\n"))


def test_loaded_graph_walks(mhw, oracle, tmp_path):
    """A graph loaded from text walks like the same graph uploaded as CSR."""
    from tests.helpers import corpus_equal, model_desc, walk_config, walk_model
    rng = O.XoRng(3)
    hg = O.random_graph(60, 4.0, True, rng)
    lines = [f"{v} {u} {float(np.float32(hg.w[i])):.17g}" for v in range(hg.n)
             for i, u in zip(range(hg.offsets[v], hg.offsets[v + 1]), hg.neighbors_of(v)) if v < u]
    g = mhw.load_edge_list(write(tmp_path, "rg.txt", "\n".join(lines) + "\n"), weighted=True, symmetrize=True)
    md = model_desc(O.NODE2VEC, hg, p=0.25, q=4.0)
    cfg = O.WalkCfg(K=2, L=20, seed=7)
    orow, olen, _ = oracle.generate_walks(hg, md, cfg, rng=O.RNG_PHILOX, order=O.ORDER_STEP)
    c = mhw.generate_walks(g, walk_model(md), walk_config(cfg))
    assert corpus_equal(orow, olen, c.rows, c.lengths)
