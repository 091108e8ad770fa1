"""Native text ingestion (loader.cu, mhw_parse_edge_list) against the
reference's load_edge_list (graph.cpp:70-100, compiled in oracle/_ref): same
accept/reject decision and message on every line shape, and the same CSR once
build_csr semantics are applied. Host-only: runs without a GPU."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import oracle as O

CASES = [
    "0 1\n1 2\n2 0\n",
    "# header\n\n0 1\n   # indented comment\n1 0\n\t\n",
    "0 1 2.5\n0 1 1.5\n",
    "0 1 # trailing comment\n",
    "0\t1\t3\n",
    "0 1 1e2\n1 2 .5\n2 3 5.\n3 4 +7\n4 5 -0\n",
    "0 1\nbogus\n",
    "0 1 2.5e\n",
    "0 1 inf\n",
    "0 1 0x10\n",
    "1.5 2\n",
    "-1 2\n",
    "0 1 -3\n",
    "0 1\n",
    "0 1 2.5abc\n",
    "99999999999999999999 1\n",
    "4294967297 1\n",
    "0 1 2\n3",
    "",
    "\n\n\n",
    "0 +1 1\n",
]


def native_parse(path, weighted, symmetrize=False):
    from paper_2010_04895_b200 import _lib as L
    lib = L.lib()
    n = C.c_uint64()
    s, d, w = C.c_void_p(), C.c_void_p(), C.c_void_p()
    rc = lib.mhw_parse_edge_list(path.encode(), int(weighted), int(symmetrize), C.byref(n), C.byref(s),
                                 C.byref(d), C.byref(w))
    if rc:
        return rc, lib.mhw_last_error().decode(), None
    k = n.value
    src = np.ctypeslib.as_array(C.cast(s, C.POINTER(C.c_uint32)), shape=(max(k, 1),))[:k].copy()
    dst = np.ctypeslib.as_array(C.cast(d, C.POINTER(C.c_uint32)), shape=(max(k, 1),))[:k].copy()
    ww = np.ctypeslib.as_array(C.cast(w, C.POINTER(C.c_double)), shape=(max(k, 1),))[:k].copy()
    for p in (s, d, w):
        lib.mhw_free_host(p)
    return 0, "", (src, dst, ww)


@pytest.mark.parametrize("i", range(len(CASES)))
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("sym", [False, True])
def test_parse_matches_reference_loader(ref, oracle, tmp_path, i, weighted, sym):
    path = str(tmp_path / f"case{i}.txt")
    with open(path, "w") as f:
        f.write(CASES[i])
    rc, msg, arrays = native_parse(path, weighted, sym)
    try:
        rg = ref.load(path, weighted, sym)
        ref_rc, ref_msg = 0, ""
    except O.OracleError as e:
        ref_rc, ref_msg = e.code, str(e).split("] ", 1)[1]
    assert rc == ref_rc, (CASES[i], msg, ref_msg)
    if rc:
        assert msg == ref_msg
        return
    src, dst, w = arrays  # the raw edge vector, reverse arcs included
    hg = oracle.build_csr(src, dst, w, symmetrize=False)
    rh = rg.to_host()
    assert np.array_equal(hg.offsets, rh.offsets)
    assert np.array_equal(hg.nbr, rh.nbr)
    assert np.array_equal(hg.w.view(np.uint64), rh.w.view(np.uint64))


def test_missing_file_is_io_error():
    rc, msg, _ = native_parse("/nonexistent/file.txt", False)
    assert rc == 1 and "cannot open edge list" in msg


def test_large_file_multithreaded_parse_and_first_error_line(tmp_path, oracle):
    """> 1 MB: parsed by all cores; the reported line is the first bad line in
    file order even when later chunks also fail."""
    lo, hi = oracle.rmat_pairs(14, 16, seed=2)
    w = oracle.pair_weights(2, lo, hi, 1.0, 10.0)
    lines = [f"{a} {b} {float(x):.17g}" for a, b, x in zip(lo, hi, w)]
    path = str(tmp_path / "big.txt")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    assert os.path.getsize(path) > (1 << 20)
    rc, _, (src, dst, ww) = native_parse(path, True)
    assert rc == 0
    assert np.array_equal(src, lo) and np.array_equal(dst, hi)
    assert np.array_equal(ww.astype(np.float32), w)
    bad = list(lines)
    bad[len(bad) // 3] = "x y"
    bad[2 * len(bad) // 3] = "1 2 -5"
    with open(path, "w") as f:
        f.write("\n".join(bad) + "\n")
    rc, msg, _ = native_parse(path, True)
    assert rc == 2 and msg.endswith(f":{len(bad) // 3 + 1}: expected \"src dst [weight]\"")
