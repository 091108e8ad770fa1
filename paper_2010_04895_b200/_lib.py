"""ctypes binding of libmhw.so (include/mhw.h). The CUDA library is the only
compute path: if it cannot be loaded the import fails loudly (no CPU
fallback)."""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# MHW_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("MHW_LIB") or os.path.join(PKG, "libmhw.so")


class GraphView(C.Structure):
    _fields_ = [("node_count", C.c_uint32), ("arc_count", C.c_uint64), ("offsets", C.c_void_p),
                ("neighbors", C.c_void_p), ("weights", C.c_void_p), ("node_types", C.c_void_p),
                ("edge_types", C.c_void_p), ("num_node_types", C.c_uint16), ("num_edge_types", C.c_uint16),
                ("symmetric", C.c_int32)]


class ModelDescC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("p", C.c_double), ("q", C.c_double), ("metapath", C.c_void_p),
                ("metapath_len", C.c_uint32), ("type_matrix", C.c_void_p), ("type_matrix_dim", C.c_uint32)]


class WalkConfigC(C.Structure):
    _fields_ = [("walks_per_node", C.c_uint32), ("walk_length", C.c_uint32), ("seed", C.c_uint64),
                ("sampler", C.c_int32), ("init_kind", C.c_int32), ("burn_in_steps", C.c_uint32),
                ("hw_sample_size", C.c_uint32), ("schedule", C.c_int32), ("node_begin", C.c_uint32),
                ("node_end", C.c_uint32), ("chain_replica_degree", C.c_uint32), ("init_mode", C.c_int32),
                ("proposal", C.c_int32)]


class WalkStatsC(C.Structure):
    _fields_ = [("walks", C.c_uint64), ("early_terminations", C.c_uint64), ("skipped_starts", C.c_uint64),
                ("steps", C.c_uint64), ("slot_inits", C.c_uint64), ("chain_retries", C.c_uint64), ("steps_per_sec", C.c_double),
                ("init_seconds", C.c_double), ("walk_seconds", C.c_double), ("rejection_trials", C.c_uint64)]


class GraphInfoC(C.Structure):
    _fields_ = [("node_count", C.c_uint32), ("arc_count", C.c_uint64), ("weighted", C.c_int32),
                ("symmetric", C.c_int32), ("verified_symmetric", C.c_int32), ("num_node_types", C.c_uint16),
                ("num_edge_types", C.c_uint16), ("max_degree", C.c_uint32), ("isolated_nodes", C.c_uint32),
                ("device_bytes", C.c_uint64), ("device", C.c_int32)]


class ManifestC(C.Structure):
    _fields_ = [("input", C.c_char_p), ("weighted", C.c_int32), ("symmetrize", C.c_int32), ("model", C.c_char_p),
                ("p", C.c_double), ("q", C.c_double), ("metapath", C.c_char_p), ("edge_matrix", C.c_char_p),
                ("node_types", C.c_char_p), ("edge_types", C.c_char_p), ("walks_per_node", C.c_uint32),
                ("walk_length", C.c_uint32), ("sampler", C.c_char_p), ("init", C.c_char_p),
                ("burn_in_steps", C.c_uint32), ("hw_sample_size", C.c_uint32), ("threads", C.c_uint32),
                ("seed", C.c_uint64), ("output", C.c_char_p), ("nodes", C.c_uint32), ("arcs", C.c_uint64),
                ("checksum", C.c_uint64), ("T_i", C.c_double), ("T_w", C.c_double)]


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes)
SIGNATURES = {
    "mhw_last_error": (C.c_char_p, []),
    "mhw_version": (C.c_char_p, []),
    "mhw_device_count": (C.c_int32, []),
    "mhw_trim_memory": (None, []),
    "mhw_graph_upload": (C.c_int32, [C.POINTER(GraphView), C.c_int32, _PP]),
    "mhw_graph_from_edges": (C.c_int32, [C.c_uint64, _P, _P, _P, C.c_int32, C.c_uint32, C.c_int32, _PP]),
    "mhw_graph_generate_rmat": (C.c_int32, [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                            C.c_uint64, C.c_int32, C.c_float, C.c_float, C.c_uint32,
                                            C.c_int32, _PP]),
    "mhw_graph_generate_hetero": (C.c_int32, [C.c_uint32, C.c_uint64, C.c_float, C.c_float, C.c_int32, _PP]),
    "mhw_graph_load_edge_list": (C.c_int32, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, _PP]),
    "mhw_graph_load_node_types": (C.c_int32, [_P, C.c_char_p]),
    "mhw_graph_load_edge_types": (C.c_int32, [_P, C.c_char_p]),
    "mhw_parse_edge_list": (C.c_int32, [C.c_char_p, C.c_int32, C.c_int32, C.POINTER(C.c_uint64), _PP, _PP, _PP]),
    "mhw_free_host": (None, [_P]),
    "mhw_graph_set_node_types": (C.c_int32, [_P, _P, C.c_uint16]),
    "mhw_graph_set_edge_types": (C.c_int32, [_P, _P, C.c_uint16]),
    "mhw_graph_replicate": (C.c_int32, [_P, C.c_int32, _PP]),
    "mhw_graph_info_get": (C.c_int32, [_P, C.POINTER(GraphInfoC)]),
    "mhw_graph_download": (C.c_int32, [_P, _P, _P, _P, _P, _P]),
    "mhw_graph_free": (None, [_P]),
    "mhw_generate_walks": (C.c_int32, [_P, C.POINTER(ModelDescC), C.POINTER(WalkConfigC), _PP]),
    "mhw_generate_walks_multi": (C.c_int32, [_P, C.c_int32, C.POINTER(ModelDescC), C.POINTER(WalkConfigC), _PP]),
    "mhw_walk_rows": (C.c_int32, [_P, C.POINTER(ModelDescC), C.POINTER(WalkConfigC), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_uint32)]),
    "mhw_generate_walks_into": (C.c_int32, [_P, C.POINTER(ModelDescC), C.POINTER(WalkConfigC), _P, _P,
                                            C.c_uint64, C.POINTER(WalkStatsC)]),
    "mhw_generate_walks_packed": (C.c_int32, [_P, C.POINTER(ModelDescC), C.POINTER(WalkConfigC), _P, C.c_uint64,
                                              _P, C.c_uint64, C.POINTER(WalkStatsC)]),
    "mhw_generate_walks_to_file": (C.c_int32, [_P, C.POINTER(ModelDescC), C.POINTER(WalkConfigC), C.c_char_p,
                                               C.POINTER(WalkStatsC)]),
    "mhw_session_write_corpus": (C.c_int32, [_P, C.c_char_p]),
    "mhw_walks_count": (C.c_uint64, [_P]),
    "mhw_walks_stride": (C.c_uint32, [_P]),
    "mhw_walks_nodes": (_P, [_P]),
    "mhw_walks_lengths": (_P, [_P]),
    "mhw_walks_stats": (C.c_int32, [_P, C.POINTER(WalkStatsC)]),
    "mhw_walks_free": (None, [_P]),
    "mhw_walks_write": (C.c_int32, [_P, C.c_char_p]),
    "mhw_partition_nodes": (C.c_int32, [_P, C.POINTER(ModelDescC), C.c_int32, _P]),
    "mhw_session_create": (C.c_int32, [_P, C.POINTER(ModelDescC), C.POINTER(WalkConfigC), _PP]),
    "mhw_session_run": (C.c_int32, [_P, _P]),
    "mhw_session_select_starts": (C.c_int32, [_P, C.c_uint32, _P]),
    "mhw_session_stats": (C.c_int32, [_P, C.POINTER(WalkStatsC)]),
    "mhw_session_buffers": (C.c_int32, [_P, _PP, _PP, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]),
    "mhw_session_download": (C.c_int32, [_P, _P, _P, _P]),
    "mhw_session_launches": (C.c_uint32, [_P]),
    "mhw_session_chain_size": (C.c_int32, [_P, C.POINTER(C.c_uint64)]),
    "mhw_session_init_chain": (C.c_int32, [_P, C.c_uint64, C.c_uint64, _P, _P]),
    "mhw_session_load_chain": (C.c_int32, [_P, _P, _P]),
    "mhw_session_prepare": (C.c_int32, [_P, _P]),
    "mhw_session_shard_entry_bytes": (C.c_int32, [_P, C.POINTER(C.c_uint32)]),
    "mhw_session_init_shard": (C.c_int32, [_P, C.c_uint64, C.c_uint64, _P, _P]),
    "mhw_session_load_shard_range": (C.c_int32, [_P, C.c_uint64, C.c_uint64, _P, _P]),
    "mhw_session_export_table": (C.c_int32, [_P, _P, _P]),
    "mhw_session_init_records": (C.c_int32, [_P, C.c_uint64, C.c_uint64, _P, _P]),
    "mhw_session_load_records": (C.c_int32, [_P, _P, _P]),
    "mhw_session_record_width": (C.c_int32, [_P, _P]),
    "mhw_session_load_records_range": (C.c_int32, [_P, C.c_uint64, C.c_uint64, _P, _P]),
    "mhw_session_free": (None, [_P]),
    "mhw_decide": (C.c_int32, [_P, C.POINTER(ModelDescC), C.c_uint64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "mhw_decide_hastings": (C.c_int32, [_P, C.POINTER(ModelDescC), C.c_uint64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "mhw_alias_tables": (C.c_int32, [_P, _P, _P]),
    "mhw_check": (C.c_int32, [_P, C.POINTER(ModelDescC), C.c_uint64, C.c_uint64, _P, _P, C.c_uint64, _P, _P]),
    "mhw_init_states": (C.c_int32, [_P, C.POINTER(ModelDescC), C.POINTER(WalkConfigC), C.c_uint64, _P, _P, _P]),
    "mhw_stats_render": (C.c_int32, [C.POINTER(WalkStatsC), C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "mhw_manifest_render": (C.c_int32, [C.POINTER(ManifestC), C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "mhw_manifest_write": (C.c_int32, [C.POINTER(ManifestC)]),
    "mhw_graph_checksum": (C.c_int32, [_P, C.POINTER(C.c_uint64)]),
}

_lib = None


def build_library(force: bool = False) -> str:
    from . import build as _build
    return _build.build(force=force)


def lib() -> C.CDLL:
    """Loads libmhw.so (building it in-tree with nvcc if it is absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build_library()
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
