"""Corpus emission parity for the JSON sidecars: the
`.stats.jsonl` line of write_corpus (engine.cpp:248-259) and cmd_walk's
`.manifest.json` (tools/mhwalk.cpp:142-169), rendered by libmhw.so's host
code (mhw_stats_render / mhw_manifest_render, no GPU needed) and compared
byte for byte with the reference's own nlohmann output (oracle/_ref)."""
import os
import re
import struct

import numpy as np
import pytest

from paper_2010_04895_b200 import mhwalk as M


def _doubles(n, seed=0):
    r = np.random.default_rng(seed)
    bits = r.integers(0, 1 << 63, size=n, dtype=np.uint64) | (r.integers(0, 2, size=n, dtype=np.uint64) << 63)
    x = bits.view(np.float64)
    x = x[np.isfinite(x)]
    mags = 10.0 ** r.uniform(-30, 30, n) * r.uniform(0.1, 1, n)
    rates = r.uniform(1e5, 2e10, n)                      # steps/s-like
    secs = r.uniform(0, 1000, n)                         # seconds-like
    small = r.uniform(0, 1e-3, n)
    ints = np.floor(r.uniform(0, 1e17, n))               # integral values around the 1e15 switch
    fixed = np.array([0.0, -0.0, 1.0, 0.5, 0.1, 1e-5, 1e-4, 1.5e-5, 1e15, 1e16, 1.5e16, 123456789012345.0,
                      1234567890123456.0, 0.0001, 0.00012, 2959152.659515442, 5e-324, 1.7976931348623157e308,
                      2.2250738585072014e-308, 9007199254740993.0, 0.3, 2.0 / 3.0])
    return np.concatenate([fixed, x, mags, rates, secs, small, ints])


def _render_steps_per_sec(x):
    line = M.stats_line(M.RunStats(steps_per_sec=float(x))).decode()
    return re.search(r'"steps_per_sec":([^,]+),', line).group(1)


def test_json_numbers_equal_nlohmann(ref):
    """Every double the sidecars print: shortest round-trip digits laid out as
    nlohmann's format_buffer (fixed in (-4, 15], else d.ddde+XX), 0.0 / -0.0."""
    xs = _doubles(40000)
    bad = []
    for x in xs:
        a, b = _render_steps_per_sec(x), ref.json_double(float(x))
        if a != b:
            bad.append((struct.pack("<d", x).hex(), a, b))
    assert not bad, bad[:10]


def test_json_non_finite_is_null(ref):
    for x in (float("nan"), float("inf"), -float("inf")):
        assert _render_steps_per_sec(x) == ref.json_double(x) == "null"


@pytest.mark.parametrize("seed", range(4))
def test_write_corpus_bytes_equal_reference(ref, tmp_path, seed):
    """The Python mirror's write_corpus (text + stats sidecar via
    mhw_stats_render) = the reference's write_corpus, byte for byte."""
    r = np.random.default_rng(seed)
    n, stride = int(r.integers(0, 40)), 17
    rows = r.integers(0, 1 << 32, size=(max(n, 1), stride), dtype=np.uint64).astype(np.uint32)
    lens = r.integers(1, stride + 1, size=max(n, 1)).astype(np.uint32)
    rows, lens = rows[:n], lens[:n]
    st = dict(walks=n, early_terminations=int(r.integers(0, 5)), skipped_starts=int(r.integers(0, 9)),
              steps=int(lens.astype(np.int64).sum() - n), steps_per_sec=float(r.uniform(0, 1e10)),
              init_seconds=[0.0, float(r.uniform(0, 1))][seed % 2], walk_seconds=float(r.uniform(0, 1e-3)))
    a, b = str(tmp_path / "mine.txt"), str(tmp_path / "ref.txt")
    corpus = M.WalkCorpus(rows=rows.reshape(n, stride), lengths=lens, stats=M.RunStats(**st))
    M.write_corpus(corpus, a)
    ref.write_corpus(b, rows.reshape(n, stride), lens, st)
    for suffix in ("", ".stats.jsonl"):
        assert open(a + suffix, "rb").read() == open(b + suffix, "rb").read(), suffix


@pytest.mark.parametrize("seed", range(6))
def test_manifest_equals_reference(ref, seed):
    r = np.random.default_rng(100 + seed)
    pick = lambda *xs: xs[int(r.integers(0, len(xs)))]
    f = dict(input=pick("graph.txt", "", "dir/with space/\"q\"\\x.el", "tab\there"), weighted=int(r.integers(0, 2)),
             symmetrize=int(r.integers(0, 2)), model=pick("deepwalk", "node2vec", "metapath2vec", "edge2vec",
                                                          "fairwalk"),
             p=float(pick(1.0, 0.25, r.uniform(0, 10))), q=float(pick(1.0, 4.0, r.uniform(0, 1e-6))),
             metapath=pick("", "0,1,2,1,0"), edge_matrix=pick("", "M.txt"), node_types=pick("", "nt.txt"),
             edge_types=pick("", "et.txt"), walks_per_node=int(r.integers(1, 100)),
             walk_length=int(r.integers(1, 1000)), sampler=pick("mh", "alias", "direct", "rejection"),
             init=pick("random", "high_weight", "burn_in"), burn_in_steps=int(r.integers(0, 1000)),
             hw_sample_size=int(r.integers(0, 64)), threads=int(r.integers(1, 64)),
             seed=int(r.integers(0, 1 << 63)), output=pick("walks.txt", "out/é.txt"),
             nodes=int(r.integers(0, 1 << 32)), arcs=int(r.integers(0, 1 << 40)),
             checksum=int(r.integers(0, 1 << 63)) * 2 + 1, T_i=float(pick(0.0, r.uniform(0, 100))),
             T_w=float(r.uniform(0, 1e-2)))
    assert M.render_manifest(**f) == ref.manifest(**f)
