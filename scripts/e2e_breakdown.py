"""Timing breakdown of the e2e path (upload / walk+D2H variants) for one config."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2010_04895_b200 as mhw  # noqa: E402
from paper_2010_04895_b200 import _lib as L  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1]])
cfg["name"] = sys.argv[1]
g = bench.build_graph(cfg)
model = bench.make_model(cfg)
wcfg = bench.make_config(cfg)
d = g.download()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
off, nb = pin(d["offsets"]), pin(d["neighbors"])
w = pin(d["weights"]) if d["weights"] is not None else None
view = L.GraphView()
view.node_count, view.arc_count = len(d["offsets"]) - 1, len(d["neighbors"])
view.offsets, view.neighbors = off.data_ptr(), nb.data_ptr()
view.weights = w.data_ptr() if w is not None else None
nt = pin(d["node_types"]) if d["node_types"] is not None else None
et = pin(d["edge_types"]) if d["edge_types"] is not None else None
view.node_types = nt.data_ptr() if nt is not None else None
view.edge_types = et.data_ptr() if et is not None else None
view.num_node_types, view.num_edge_types = d["num_node_types"], d["num_edge_types"]
view.symmetric = 1
md, keep = model._desc()
c = wcfg._c()
lib = L.lib()
rows, stride = C.c_uint64(), C.c_uint32()
lib.mhw_walk_rows(g.handle, C.byref(md), C.byref(c), C.byref(rows), C.byref(stride))
cap = rows.value * (cfg["L"] + 1)
out = torch.empty(cap, dtype=torch.int32).pin_memory()
offs = torch.empty(rows.value + 1, dtype=torch.int64).pin_memory()
pad = torch.empty(rows.value * stride.value, dtype=torch.int32).pin_memory()
lens = torch.empty(rows.value, dtype=torch.int32).pin_memory()
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    t0 = time.perf_counter()
    h = C.c_void_p()
    lib.mhw_graph_upload(C.byref(view), 0, C.byref(h))
    t1 = time.perf_counter()
    st = L.WalkStatsC()
    rc = lib.mhw_generate_walks_packed(h, C.byref(md), C.byref(c), C.c_void_p(out.data_ptr()), cap,
                                       C.c_void_p(offs.data_ptr()), rows.value + 1, C.byref(st))
    t2 = time.perf_counter()
    rc2 = 0
    if len(sys.argv) <= 3 or sys.argv[3] != "packed":
        rc2 = lib.mhw_generate_walks_into(h, C.byref(md), C.byref(c), C.c_void_p(pad.data_ptr()),
                                          C.c_void_p(lens.data_ptr()), rows.value, C.byref(st))
    t3 = time.perf_counter()
    lib.mhw_graph_free(h)
    t4 = time.perf_counter()
    if rc or rc2:
        print("error:", lib.mhw_last_error().decode(), flush=True)
    print(f"upload {1e3*(t1-t0):.1f} ms  packed {1e3*(t2-t1):.1f} ms (rc {rc})  padded {1e3*(t3-t2):.1f} ms "
          f"(rc {rc2})  free {1e3*(t4-t3):.1f} ms  walk {st.walk_seconds*1e3:.1f} ms", flush=True)
