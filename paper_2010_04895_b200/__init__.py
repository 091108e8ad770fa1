"""B200-native M-H random-walk engine (UniNet, arXiv 2010.04895).

The compute path is libmhw.so (hand-written sm_100a CUDA behind the C ABI in
include/mhw.h); this package is its Python mirror of the reference API.
"""
from .mhwalk import (  # noqa: F401
    CudaError, Graph, InitKind, InitStrategy, IoError, ModelKind, ParseError, RunStats, SamplerKind,
    Schedule, Session, ValidationError, WalkConfig, WalkCorpus, WalkModel, alias_tables, decide, decide_hastings,
    device_count, generate_walks, generate_walks_multi, init_kind_from_string, init_states, kNoAffix,
    load_edge_list, load_edge_types, load_node_types, model_kind_from_string, partition_nodes, read_corpus,
    render_manifest, stats_line, write_corpus, write_manifest,
)
