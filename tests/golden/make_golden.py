"""Generate tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libmhwalk_ref.so, compiled in place from /root/reference by
oracle/Makefile). Run here (the reference tree does not exist on the GPU box):

    python tests/golden/make_golden.py

The fixtures pin the CPU oracle (tests/test_oracle_golden.py) without the
reference present: walk corpora of generate_walks(threads=1)
(engine.cpp:157-234), per-step decision triples (models.cpp:82-123 +
samplers.hpp:24), alias tables (samplers.cpp:95-131) and CSRs built by
load_edge_list (graph.cpp:70-100).
"""
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.helpers import model_desc, random_triples  # noqa: E402


def graph_arrays(prefix, g: O.HostGraph):
    d = {f"{prefix}offsets": g.offsets, f"{prefix}nbr": g.nbr, f"{prefix}w": g.w,
         f"{prefix}meta": np.array([g.n_ntypes, g.n_etypes, int(g.symmetric)], dtype=np.int64)}
    if g.ntype is not None:
        d[f"{prefix}ntype"] = g.ntype
    if g.etype is not None:
        d[f"{prefix}etype"] = g.etype
    return d


def walk_cases():
    """(name, graph, model desc, cfg) cases mirroring test_engine.cpp / acceptance.cpp graphs."""
    cases = []
    for gi, (seed, n, deg, weighted) in enumerate([(3, 80, 6.0, True), (9, 100, 5.0, True), (12, 60, 3.0, False)]):
        rng = O.XoRng(seed)
        g = O.random_graph(n, deg, weighted, rng, ensure_connected=gi != 2)
        O.assign_random_types(g, 2, rng)
        for kind in range(5):
            for init in range(3):
                md = model_desc(kind, g, p=0.5, q=2.0)
                cfg = O.WalkCfg(K=3, L=20, seed=4 + gi, init_kind=init, burn_in_steps=7, hw_sample_size=4)
                cases.append((f"g{gi}_k{kind}_i{init}", g, md, cfg))
    rng = O.XoRng(12)
    pa = O.preferential_attachment(50, 3, rng)
    cases.append(("pa_deepwalk", pa, model_desc(O.DEEPWALK, pa), O.WalkCfg(K=10, L=80, seed=13)))
    tri = O.triangle()
    cases.append(("triangle", tri, model_desc(O.DEEPWALK, tri), O.WalkCfg(K=1, L=3, seed=9)))
    iso = O.make_graph(1, [])
    cases.append(("isolated", iso, model_desc(O.DEEPWALK, iso), O.WalkCfg(K=2, L=80, seed=0)))
    return cases


def main():
    ref = O.RefLib()
    out = {}
    # --- walks
    names = []
    for name, g, md, cfg in walk_cases():
        rg = ref.graph(g)
        rm = rg.model(md)
        rows, lens, st = rm.generate_walks(cfg, threads=1, n_nodes=g.n)
        names.append(name)
        out.update(graph_arrays(f"{name}/g_", g))
        out[f"{name}/rows"] = rows
        out[f"{name}/lens"] = lens
        out[f"{name}/stats"] = np.array([st["walks"], st["early_terminations"], st["skipped_starts"], st["steps"]],
                                        dtype=np.int64)
        out[f"{name}/model"] = np.array([md.kind, md.p, md.q], dtype=np.float64)
        out[f"{name}/metapath"] = np.array(md.metapath, dtype=np.int64)
        out[f"{name}/M"] = md.type_matrix if md.type_matrix is not None else np.zeros((0, 0))
        out[f"{name}/cfg"] = np.array([cfg.K, cfg.L, cfg.seed, cfg.init_kind, cfg.burn_in_steps,
                                       cfg.hw_sample_size], dtype=np.int64)
    out["walk_cases"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "walks_ref.npz"), **out)

    # --- decisions
    out = {}
    rng = O.XoRng(7)
    g = O.random_graph(200, 6.0, True, rng)
    O.assign_random_types(g, 3, rng)
    out.update(graph_arrays("g_", g))
    M = np.random.default_rng(5).uniform(0.5, 2.0, (9, 9))
    for kind in range(5):
        md = model_desc(kind, g, p=0.37, q=1.9, metapath=(0, 1, 2, 1, 0), M=M)
        pos, aff, cand, last, u = random_triples(g, md, 5000, seed=100 + kind)
        wc, wl, acc = ref.graph(g).model(md).decide(pos, aff, cand, last, u)
        for k, v in dict(pos=pos, aff=aff, cand=cand, last=last, u=u, wc=wc, wl=wl, acc=acc).items():
            out[f"k{kind}/{k}"] = v
    out["M"] = M
    np.savez_compressed(os.path.join(HERE, "decide_ref.npz"), **out)

    # --- alias tables
    out = {}
    r = O.XoRng(12)
    for t in range(40):
        n = 1 + r.uniform_index(100)
        w = np.array([0.05 + r.uniform_real() for _ in range(n)])
        if t % 5 == 0:
            w[:: 3] = 0.0
            w[0] = 1.0
        prob, alias = ref.alias_build(w)
        out[f"t{t}/w"], out[f"t{t}/prob"], out[f"t{t}/alias"] = w, prob, alias
    np.savez_compressed(os.path.join(HERE, "alias_ref.npz"), **out)

    # --- CSR via load_edge_list
    out = {}
    with tempfile.TemporaryDirectory() as td:
        texts = {
            "triangle_sym": ("0 1\n1 2\n2 0\n", False, True),
            "dup_sum": ("0 1 2.5\n0 1 1.5\n", True, False),
            "comments": ("# header\n\n0 1\n# tail\n1 0\n", False, False),
        }
        o = O.Oracle()
        lo, hi = o.rmat_pairs(10, 16, seed=7)
        w = o.pair_weights(7, lo, hi, 1.0, 10.0)
        texts["rmat10_w"] = ("".join(f"{a} {b} {float(x):.17g}\n" for a, b, x in zip(lo, hi, w)), True, True)
        for name, (txt, weighted, sym) in texts.items():
            p = os.path.join(td, name + ".txt")
            with open(p, "w") as f:
                f.write(txt)
            hg = ref.load(p, weighted, sym).to_host()
            out.update(graph_arrays(f"{name}/", hg))
            out[f"{name}/text"] = np.array(txt)
            out[f"{name}/flags"] = np.array([int(weighted), int(sym)])
    np.savez_compressed(os.path.join(HERE, "csr_ref.npz"), **out)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
