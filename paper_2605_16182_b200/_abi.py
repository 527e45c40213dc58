"""ctypes declarations of the C ABI in include/twg.h (libtimewalk_b200.so).

The library is built in-tree (``make lib`` / ``__graft_entry__.build()``).
There is no fallback: if the shared object is missing or fails to load,
importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TWG_LIB_PATH") or os.path.join(_HERE, "lib", "libtimewalk_b200.so")  # override: A/B builds

TWG_OK, TWG_EINVAL, TWG_ERANGE, TWG_ELOGIC, TWG_ECUDA, TWG_ENOMEM, TWG_EPARSE = range(7)


class twg_edge(C.Structure):
    _fields_ = [("src", C.c_int64), ("dst", C.c_int64), ("t", C.c_int64)]


class twg_build_opts(C.Structure):
    _fields_ = [("weights", C.c_int32), ("adjacency", C.c_int32)]


class twg_store_info(C.Structure):
    _fields_ = [
        ("edges", C.c_uint64), ("nodes", C.c_uint64), ("ts_groups", C.c_uint64),
        ("entries", C.c_uint64), ("node_groups", C.c_uint64), ("adjacency", C.c_uint64),
        ("mode", C.c_int32), ("has_weights", C.c_int32), ("has_adjacency", C.c_int32),
        ("streaming", C.c_int32), ("device_bytes", C.c_uint64),
    ]


class twg_store_layout(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("log_cap", "log_first", "ts_first", "arena_cap", "arena_used",
                                            "arena_serial", "relocated_rings", "max_ring_end")]


class twg_audit_report(C.Structure):
    _fields_ = [("walks", C.c_uint64), ("valid_walks", C.c_uint64), ("hops", C.c_uint64),
                ("valid_hops", C.c_uint64)]


class twg_batch_stats(C.Structure):
    _fields_ = [
        ("ingested", C.c_uint64), ("dropped_late", C.c_uint64), ("evicted", C.c_uint64),
        ("retained", C.c_uint64), ("rebuild_duration", C.c_double), ("peak_bytes", C.c_uint64),
    ]


class twg_thresholds(C.Structure):
    _fields_ = [
        ("w_warp", C.c_uint32), ("block_dim", C.c_uint32), ("w_max", C.c_uint32),
        ("g_warp_cap", C.c_uint32), ("g_block_cap", C.c_uint32),
    ]


class twg_walk_config(C.Structure):
    _fields_ = [
        ("walk_length", C.c_uint32), ("start_mode", C.c_int32), ("walks_per_node", C.c_uint32),
        ("_pad0", C.c_uint32), ("total_walks", C.c_uint64), ("bias", C.c_int32),
        ("start_bias", C.c_int32), ("node2vec", C.c_int32), ("temporal_adjacency", C.c_int32),
        ("p", C.c_double), ("q", C.c_double), ("direction", C.c_int32), ("rng", C.c_int32),
        ("seed", C.c_uint64), ("walk_begin", C.c_uint64), ("walk_end", C.c_uint64),
    ]


class twg_walk_stats(C.Structure):
    _fields_ = [
        ("walks", C.c_uint64), ("hops", C.c_uint64), ("steps", C.c_uint64),
        ("solo", C.c_uint64), ("warp_cached", C.c_uint64), ("warp_direct", C.c_uint64),
        ("block_cached", C.c_uint64), ("block_direct", C.c_uint64), ("multi_block", C.c_uint64),
        ("wall_seconds", C.c_double), ("ambiguous_draws", C.c_uint64), ("alg_bytes", C.c_uint64),
    ]


class twg_group_batch_stats(C.Structure):
    _fields_ = [("local", twg_batch_stats), ("replica_hash", C.c_uint64), ("replicas_agree", C.c_int32),
                ("wire_bytes_per_edge", C.c_int32), ("edges", C.c_uint64)]


VP = C.c_void_p
PP = C.POINTER(C.c_void_p)
I = C.c_int
U64 = C.c_uint64
I64 = C.c_int64

# name -> (restype, argtypes)
SIGNATURES = {
    "twg_abi_version": (I, []),
    "twg_last_error": (C.c_char_p, []),
    "twg_ctx_create": (I, [I, PP]),
    "twg_ctx_create_prio": (I, [I, I, PP]),
    "twg_ctx_destroy": (I, [VP]),
    "twg_ctx_sync": (I, [VP]),
    "twg_ctx_stream": (I, [VP, PP]),
    "twg_ctx_launch_count": (I, [VP, C.POINTER(U64)]),
    "twg_store_build": (I, [VP, VP, U64, I, VP, PP]),
    "twg_store_build_device": (I, [VP, VP, VP, VP, U64, I, VP, PP]),
    "twg_store_retain": (I, [VP]),
    "twg_store_release": (I, [VP]),
    "twg_store_get_info": (I, [VP, C.POINTER(twg_store_info)]),
    "twg_store_get_layout": (I, [VP, C.POINTER(twg_store_layout)]),
    "twg_store_download": (I, [VP, I, VP]),
    "twg_store_neighborhood": (I, [VP, VP, VP, U64, I, VP]),
    "twg_store_find_nodes": (I, [VP, VP, U64, VP, VP]),
    "twg_store_adjacent": (I, [VP, VP, VP, U64, I, VP, I, VP]),
    "twg_window_create": (I, [VP, I64, I, VP, PP]),
    "twg_window_destroy": (I, [VP]),
    "twg_window_ingest": (I, [VP, VP, U64, C.POINTER(twg_batch_stats)]),
    "twg_window_ingest_device": (I, [VP, VP, VP, VP, U64, VP]),
    "twg_stage_batch": (I, [VP, I, VP, U64]),
    "twg_window_ingest_staged": (I, [VP, I, VP]),
    "twg_walkset_download_compact_async": (I, [VP, VP, VP, VP, U64, C.POINTER(U64)]),
    "twg_walkset_wait": (I, [VP]),
    "twg_window_snapshot": (I, [VP, PP]),
    "twg_window_bounds": (I, [VP, C.POINTER(I64), C.POINTER(I64)]),
    "twg_window_state": (I, [VP, C.POINTER(I64), C.POINTER(U64), C.POINTER(twg_batch_stats)]),
    "twg_generate": (I, [VP, VP, C.POINTER(twg_walk_config), VP, I, PP, C.POINTER(twg_walk_stats)]),
    "twg_walkset_destroy": (I, [VP]),
    "twg_walkset_info": (I, [VP, C.POINTER(C.c_uint32), C.POINTER(U64), C.POINTER(U64), C.POINTER(U64)]),
    "twg_walkset_download": (I, [VP, VP, VP, VP]),
    "twg_walkset_download_compact": (I, [VP, VP, VP, VP]),
    "twg_walkset_audit": (I, [VP, VP, I, I, VP, VP]),
    "twg_walkset_text": (I, [VP, VP, U64, C.POINTER(U64)]),
    "twg_walkset_binary": (I, [VP, VP, U64, C.POINTER(U64)]),
    "twg_walkset_from_host": (I, [VP, C.c_uint32, U64, VP, VP, VP, PP]),
    "twg_parse_edges_tsv": (I, [VP, VP, U64, PP, C.POINTER(U64)]),
    "twg_synth_graph": (I, [VP, I, U64, U64, I64, U64, VP, U64, C.POINTER(U64)]),
    "twg_edges_from_host": (I, [VP, VP, U64, PP]),
    "twg_edges_info": (I, [VP, C.POINTER(U64)]),
    "twg_edges_download": (I, [VP, VP]),
    "twg_edges_device": (I, [VP, PP, PP, PP]),
    "twg_edges_format_tsv": (I, [VP, VP, U64, C.POINTER(U64)]),
    "twg_edges_destroy": (I, [VP]),
    "twg_walkset_device": (I, [VP, PP, PP, PP]),
    "twg_sample_start_edges": (I, [VP, I, VP, VP, U64, VP]),
    "twg_schedule_step": (I, [VP, VP, VP, U64, VP, VP, VP, U64, VP]),
    "twg_init_walks": (I, [VP, VP, C.POINTER(twg_walk_config), C.POINTER(C.c_uint32), C.POINTER(U64)] + [VP] * 8),
    "twg_hop_walks": (I, [VP, VP, C.POINTER(twg_walk_config), VP, U64, U64, C.c_uint32] + [VP] * 8),
    "twg_radix_sort_pairs": (I, [VP, VP, VP, U64]),
    "twg_exclusive_scan": (I, [VP, VP, VP, U64, C.POINTER(U64)]),
    "twg_run_length_encode": (I, [VP, VP, U64, VP, C.POINTER(U64)]),
    "twg_partition_flagged": (I, [VP, VP, U64, VP, U64, VP, C.POINTER(U64)]),
    "twg_pick_index": (I, [VP, I, VP, VP, U64, VP]),
    "twg_pick_weighted_range": (I, [VP, VP, VP, U64, VP, VP, VP, U64, VP]),
    "twg_rng_bits": (I, [VP, I, U64, VP, VP, VP, U64, VP]),
    "twg_synth_stream_host": (I, [U64, U64, U64, U64, VP]),
    "twg_synth_stream_device": (I, [VP, U64, U64, U64, U64, VP, VP, VP]),
    "twg_synth_uniform_device": (I, [VP, U64, U64, I64, U64, VP, VP, VP]),
    "twg_group_unique_id": (I, [VP]),
    "twg_group_create": (I, [VP, I, I, VP, PP]),
    "twg_group_destroy": (I, [VP]),
    "twg_group_info": (I, [VP, C.POINTER(I), C.POINTER(I)]),
    "twg_group_stage_device": (I, [VP, I, I, VP, VP, VP, U64]),
    "twg_group_stage_host": (I, [VP, I, I, VP, U64]),
    "twg_group_staged_edges": (I, [VP, I, C.POINTER(U64)]),
    "twg_group_ingest_staged": (I, [VP, VP, I, C.POINTER(twg_group_batch_stats)]),
    "twg_group_ingest_device": (I, [VP, VP, I, VP, VP, VP, U64, C.POINTER(twg_group_batch_stats)]),
    "twg_group_ingest": (I, [VP, VP, I, VP, U64, C.POINTER(twg_group_batch_stats)]),
    "twg_group_generate": (I, [VP, VP, C.POINTER(twg_walk_config), VP, I, PP, C.POINTER(twg_walk_stats),
                               C.POINTER(twg_walk_stats)]),
    "twg_store_replica_hash": (I, [VP, U64, C.POINTER(U64)]),
}


def header_symbols() -> list[str]:
    """Every function declared in include/twg.h (parsed, not assumed)."""
    import re

    hdr = os.path.join(os.path.dirname(_HERE), "include", "twg.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(twg_[a-z_0-9]+)\(", text, re.M)))


_lib = None


def load() -> C.CDLL:
    """Load the product library (raises if it is missing — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built: run `make lib` or __graft_entry__.build() (no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
