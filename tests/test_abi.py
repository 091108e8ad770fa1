"""C-ABI boundary checks that need no GPU: libmhw.so loads, exports exactly
the entry points include/mhw.h declares, and fails loudly (status 4, no CPU
fallback) when no CUDA device exists."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mhw.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^MHW_API\s+[\w\s\*]+?\b(mhw_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2010_04895_b200 import _lib
    return _lib.lib()


def test_header_declares_the_walk_path():
    names = declared()
    for must in ("mhw_graph_upload", "mhw_generate_walks", "mhw_decide", "mhw_alias_tables",
                 "mhw_graph_download", "mhw_last_error", "mhw_session_run"):
        assert must in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol(lib):
    for name in declared():
        assert hasattr(lib, name), name
    from paper_2010_04895_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared())


def test_library_exports_nothing_else():
    from paper_2010_04895_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted({l.split()[-1] for l in out.splitlines() if " T " in l})
    assert exported == declared()


def test_library_is_sm100a():
    from paper_2010_04895_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_strings(lib):
    assert b"sm_100a" in lib.mhw_version()
    assert isinstance(lib.mhw_last_error(), bytes)


def test_no_device_fails_loudly(lib):
    import paper_2010_04895_b200 as mhw
    if lib.mhw_device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(mhw.CudaError, match="no CUDA device"):
        mhw.Graph.from_csr(np.array([0, 1, 2]), np.array([1, 0]))
    with pytest.raises(mhw.CudaError):
        mhw.Graph.rmat(4)


def test_null_arguments_are_invalid(lib):
    from paper_2010_04895_b200 import _lib
    rc = lib.mhw_decide(None, None, 0, None, None, None, None, None, None, None, None)
    assert rc == 2
    assert b"must not be NULL" in lib.mhw_last_error()
    st = _lib.WalkStatsC()
    assert lib.mhw_walks_stats(None, C.byref(st)) == 2


def test_config_validation_messages_mirror_reference():
    """WalkConfig with threads == 0 is rejected like engine.cpp:158-160."""
    import paper_2010_04895_b200 as mhw
    with pytest.raises(mhw.ValidationError, match="must be positive"):
        mhw.WalkConfig(threads=0)._c()
    with pytest.raises(mhw.ValidationError, match="unknown model"):
        mhw.model_kind_from_string("word2vec")
    assert mhw.init_kind_from_string("burn-in") == mhw.InitKind.burn_in


def test_load_edge_list_errors(tmp_path):
    """Loader errors (graph.cpp:70-100): IoError, ParseError with line number,
    negative weight ValidationError -- raised before any device work."""
    import paper_2010_04895_b200 as mhw
    with pytest.raises(mhw.IoError):
        mhw.load_edge_list("/nonexistent/file")
    p = tmp_path / "bad.txt"
    p.write_text("0 1\nbogus\n")
    with pytest.raises(mhw.ParseError, match=":2:"):
        mhw.load_edge_list(str(p))
    p.write_text("0 1 -3\n")
    with pytest.raises(mhw.ValidationError, match="negative"):
        mhw.load_edge_list(str(p), weighted=True)
    p.write_text("0 1\n")
    with pytest.raises(mhw.ParseError, match="missing edge weight"):
        mhw.load_edge_list(str(p), weighted=True)


def test_corpus_round_trip(tmp_path):
    """write_corpus / read_corpus (engine.cpp:236-275) on the host mirror."""
    import paper_2010_04895_b200 as mhw
    rows = np.zeros((3, 4), dtype=np.uint32)
    rows[0, :3] = [0, 1, 2]
    rows[1, :1] = [5]
    rows[2, :2] = [3, 4]
    corpus = mhw.WalkCorpus(rows, np.array([3, 1, 2], dtype=np.uint32), mhw.RunStats(walks=3))
    path = str(tmp_path / "c.txt")
    mhw.write_corpus(corpus, path)
    assert open(path).readline() == "0 1 2\n"
    assert mhw.read_corpus(path) == [[0, 1, 2], [5], [3, 4]]
    assert os.path.exists(path + ".stats.jsonl")
    empty = mhw.WalkCorpus(np.zeros((0, 4), dtype=np.uint32), np.zeros(0, dtype=np.uint32), mhw.RunStats())
    mhw.write_corpus(empty, path)
    assert os.path.getsize(path) == 0 and mhw.read_corpus(path) == []
