"""Ingestion at scale: text edge list -> CSR.

Writes the cfg2 (or given config's) undirected edge list as text -- the
reference's own write_edge_list format (graph.cpp), weighted configs with
their weights -- then times
  * mhw_graph_load_edge_list (native multi-threaded parser + device build_csr),
  * the reference's load_edge_list (oracle/_ref, unmodified graph.cpp:70-100),
on the same file, and checks the two CSRs are identical (offsets, ids,
weights as f32). One JSON line to stdout.

python scripts/loader_bench.py [cfg2] [reps]
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = dict(bench.CONFIGS[name])
    cfg["name"] = name
    import paper_2010_04895_b200 as mhw
    from oracle import oracle as O
    weighted = bool(cfg.get("weighted") or cfg.get("hetero"))
    hg = bench.host_graph_for_reference(cfg)
    ref = O.RefLib()
    tmp = tempfile.mkdtemp(prefix="mhw_loader_")
    path = os.path.join(tmp, f"{name}.el")
    # the undirected edge list, one "src dst [w]" line per pair (src < dst);
    # both loaders symmetrise it
    src = np.repeat(np.arange(hg.n, dtype=np.int64), np.diff(hg.offsets.astype(np.int64)))
    nbr = hg.nbr.astype(np.int64)
    keep = src < nbr
    with open(path, "w") as f:
        if weighted:
            w = hg.w[keep]
            for a, b, x in zip(src[keep].tolist(), nbr[keep].tolist(), w.tolist()):
                f.write(f"{a} {b} {x!r}\n")
        else:
            for a, b in zip(src[keep].tolist(), nbr[keep].tolist()):
                f.write(f"{a} {b}\n")
    size = os.path.getsize(path)
    t_mine, t_ref = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        g = mhw.load_edge_list(path, weighted=weighted, symmetrize=True)
        g.info()
        t_mine.append(time.perf_counter() - t0)
    for _ in range(max(1, reps - 1)):
        t0 = time.perf_counter()
        rg = ref.load(path, weighted=weighted, symmetrize=True)
        t_ref.append(time.perf_counter() - t0)
    d = g.download()
    r = rg.to_host()
    same = (np.array_equal(d["offsets"].astype(np.uint64), r.offsets.astype(np.uint64))
            and np.array_equal(d["neighbors"].astype(np.uint32), r.nbr.astype(np.uint32))
            and (not weighted or np.array_equal(d["weights"], r.w.astype(np.float32))))
    os.remove(path)
    os.rmdir(tmp)
    line = {"config": name, "file_bytes": size, "arcs": int(len(d["neighbors"])), "nodes": int(len(d["offsets"]) - 1),
            "mine_s": float(np.median(t_mine)), "reference_s": float(np.median(t_ref)),
            "mine_GBps": size / float(np.median(t_mine)) / 1e9, "reference_GBps": size / float(np.median(t_ref)) / 1e9,
            "speedup": float(np.median(t_ref)) / float(np.median(t_mine)), "csr_identical": bool(same),
            "threads": bench.cpu_threads(),
            "what": "mhw_graph_load_edge_list (native parser + device build_csr) vs the reference's "
                    "load_edge_list (oracle/_ref), same text file, symmetrize=True"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
