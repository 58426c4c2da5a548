"""ctypes binding of include/speed_c.h (the product C-ABI).

Loads the in-tree ``libspeed_b200.so``; there is no fallback — if the library
is missing the import fails loudly (run ``make`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspeed_b200.so")

EDGE_DTYPE = np.dtype([("src", "<u4"), ("dst", "<u4"), ("ts", "<f8")])
assert EDGE_DTYPE.itemsize == 16  # == speedpart::TemporalEdge (types.hpp:15-21)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `make` in the repo root (no CPU fallback)")
lib = C.CDLL(LIB_PATH)

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
u32, u64, i32, f64, f32 = C.c_uint32, C.c_uint64, C.c_int32, C.c_double, C.c_float
pu32, pu64, pi32, pf64, pf32 = (C.POINTER(t) for t in (u32, u64, i32, f64, f32))
pchar = C.c_char_p


class PartitionerConfigC(C.Structure):
    _fields_ = [("num_parts", i32), ("lambda_", f64), ("epsilon", f64), ("cent", pf64),
                ("cent_count", u32), ("hubs", pu32), ("n_hubs", u64), ("k", f64)]


class EpochReportC(C.Structure):
    _fields_ = [("batches", pu64), ("loops", pu64), ("sync_events", u64), ("digests", P),
                ("log_cap", u64), ("log_steps", pu64), ("n_log", u64), ("snap_worker", pi32),
                ("snap_digests", P), ("n_snap", u64)]


class SimConfigC(C.Structure):
    _fields_ = [("num_workers", i32), ("num_small_parts", i32), ("shuffle", i32),
                ("average", i32), ("batch_size", u64), ("epochs", i32), ("d", i32),
                ("model_seed", u64), ("shuffle_seed", u64)]


class TGNConfigC(C.Structure):
    _fields_ = [("d_mem", i32), ("d_time", i32), ("d_edge", i32), ("n_neighbors", i32),
                ("n_heads", i32), ("batch_size", u64), ("lr", f32), ("beta1", f32),
                ("beta2", f32), ("adam_eps", f32), ("seed_init", u64), ("seed_feat", u64),
                ("seed_neg", u64), ("sync_average", i32), ("gemm_mode", i32), ("backbone", i32),
                ("concurrent", i32)]


# name -> (restype, argtypes); spd_status is int32.
_SIGS = {
    "spd_last_error_code": (pchar, []),
    "spd_last_error_detail": (pchar, []),
    "spd_version": (pchar, []),
    "spd_gen_powerlaw": (i32, [u32, u64, f64, u64, P, pu32, pf64]),
    "spd_chrono_split": (i32, [u64, f64, f64, pu64, pu64, pu64]),
    "spd_compute_centrality": (i32, [P, u64, u32, f64, f64, i32, pf64, pf64]),
    "spd_compute_degree_centrality": (i32, [P, u64, u32, pf64]),
    "spd_select_hubs": (i32, [pf64, u32, f64, i32, pu32, pu64]),
    "spd_partition_stream": (i32, [P, u64, u32, C.POINTER(PartitionerConfigC), PP]),
    "spd_partition_unrestricted": (i32, [P, u64, u32, C.POINTER(PartitionerConfigC), PP]),
    "spd_score": (i32, [u32, u32, i32, C.POINTER(PartitionerConfigC), pu64, u64, u64, u32, pu64,
                        pi32, pf64]),
    "spd_assignment_from_parts": (i32, [u32, i32, pu64, pi32, pi32, u64, u64, PP]),
    "spd_assignment_destroy": (None, [P]),
    "spd_assignment_info": (i32, [P, pi32, pu32, pu64, pu64, pu64, pu64, pf64]),
    "spd_assignment_edge_part": (i32, [P, pi32]),
    "spd_assignment_node_parts": (i32, [P, pu64, pi32]),
    "spd_assignment_shared": (i32, [P, pu32]),
    "spd_free": (None, [P]),
    "spd_load_edges_csv": (i32, [pchar, i32, PP, pu64, pu32, pf64]),
    "spd_write_edges_csv": (i32, [pchar, P, u64]),
    "spd_write_edges_bin": (i32, [pchar, P, u64, u32, f64]),
    "spd_edges_bin_info": (i32, [pchar, pu64, pu32, pf64]),
    "spd_load_edges_bin": (i32, [pchar, P, u64]),
    "spd_assignment_write_json": (i32, [P, pchar, pchar]),
    "spd_assignment_read_json": (i32, [pchar, PP, PP]),
    "spd_assign_eval_edges": (i32, [P, u64, P, u64, P, PP]),
    "spd_eval_routing_counts": (i32, [P, i32, pu64, pu64]),
    "spd_eval_routing_edges": (i32, [P, i32, pu64]),
    "spd_link_metrics": (i32, [pf32, u64, pf32, u64, pf64, pf64]),
    "spd_eval_routing_destroy": (None, [P]),
    "spd_induce_subgraphs": (i32, [P, u64, u32, pu64, pi32, u32, i32, PP]),
    "spd_induce_groups": (i32, [P, u64, u32, pu64, pu32, i32, pu64, pu32, i32, PP, pu64]),
    "spd_subgraphs_from_lists": (i32, [i32, pu64, pu32, pu64, P, pu64, PP]),
    "spd_subgraphs_count": (i32, [P, pi32]),
    "spd_subgraph_sizes": (i32, [P, i32, pu64, pu64]),
    "spd_subgraph_nodes": (i32, [P, i32, pu32]),
    "spd_subgraph_edges": (i32, [P, i32, P, pu64]),
    "spd_subgraphs_destroy": (None, [P]),
    "spd_shuffle_combine": (i32, [pu64, pu32, u64, i32, u64, pu64, pu32]),
    "spd_lockstep_schedule": (i32, [P, u64, pu64, pu64, u64, pu64, pu64, pu64]),
    "spd_model_seeded": (i32, [i32, u64, pf64, pf64, pf64]),
    "spd_memstore_create": (i32, [u32, i32, i32, PP]),
    "spd_memstore_destroy": (None, [P]),
    "spd_memstore_upload": (i32, [P, pf64, pf64]),
    "spd_memstore_download": (i32, [P, pf64, pf64]),
    "spd_memstore_reset": (i32, [P]),
    "spd_memstore_copy": (i32, [P, P]),
    "spd_memstore_digest": (i32, [P, P]),
    "spd_model_update": (i32, [P, P, u64, pf64, pf64, f64]),
    "spd_sync_shared": (i32, [PP, i32, pu32, u64, i32]),
    "spd_run_epoch": (i32, [P, PP, i32, pf64, pf64, f64, pu32, u64, i32, u64,
                            C.POINTER(EpochReportC)]),
    "spd_simulate": (i32, [P, u64, u32, P, C.POINTER(SimConfigC), i32, pu64, pu64, pu64, P,
                           pu64]),
    "spd_tgn_create": (i32, [C.POINTER(TGNConfigC), P, pi32, i32, pu32, u64, u32, i32, i32, P,
                             i32, PP]),
    "spd_tgn_destroy": (None, [P]),
    "spd_nccl_unique_id": (i32, [P]),
    "spd_tgn_peer_blob_bytes": (u64, []),
    "spd_tgn_set_surrogate": (i32, [P, i32, P, P, f64]),
    "spd_tgn_attach_stream": (i32, [P, P, u64, u32, P, P, i32]),
    "spd_tgn_shuffle_epoch": (i32, [P, u64, P]),
    "spd_tgn_worker_event_count": (i32, [P, i32, P]),
    "spd_tgn_peer_export": (i32, [P, P]),
    "spd_tgn_peer_connect": (i32, [P, P]),
    "spd_tgn_epoch_steps": (i32, [P, pu64]),
    "spd_tgn_begin_epoch": (i32, [P, i32]),
    "spd_tgn_seek": (i32, [P, u64]),
    "spd_tgn_step": (i32, [P, pf32]),
    "spd_tgn_end_epoch": (i32, [P]),
    "spd_tgn_run_epoch": (i32, [P, i32, pf64]),
    "spd_tgn_set_eval_events": (i32, [P, i32, P, pu64, u64]),
    "spd_tgn_evaluate": (i32, [P, i32, u64, u64, u64, pf32, pf32]),
    "spd_tgn_param_count": (i32, [P, pu64]),
    "spd_tgn_get_params": (i32, [P, pf32]),
    "spd_tgn_set_params": (i32, [P, pf32]),
    "spd_tgn_get_grads": (i32, [P, pf32]),
    "spd_tgn_local_nodes": (i32, [P, i32, pu64, pu32]),
    "spd_tgn_get_memory": (i32, [P, i32, pf32, pf64]),
    "spd_tgn_set_memory": (i32, [P, i32, pf32, pf64]),
    "spd_tgn_last_step": (i32, [P, i32, pu64, pf32, pu32, pu32, pf32]),
    "spd_tgn_kernel_times": (i32, [P, pf32, pi32, P, i32, i32]),
    "spd_tgn_run_steps": (i32, [P, u64, pf32]),
    "spd_tgn_step_host": (i32, [P, PP, PP, pf32]),
    "spd_tgn_next_batch": (i32, [P, i32, pu64, pu64, pi32]),
    "spd_tgn_worker_events": (i32, [P, i32, P]),
    "spd_tgn_io_bytes": (i32, [P, pu64, pu64]),
    "spd_kernel_launches": (u64, []),
    "spd_edge_features_bf16": (i32, [u64, pu64, u64, i32, i32, P]),
    "spd_debug_gemm": (i32, [i32, i32, P, i32, P, i32, P, i32, i32, i32, i32, P, u64]),
    "spd_tgn_set_debug": (i32, [P, i32]),
    "spd_tgn_rebind": (i32, [P, P]),
    "spd_tgn_step_host_async": (i32, [P, PP, PP, P]),
    "spd_tgn_sync": (i32, [P]),
    "spd_tgn_set_graph": (i32, [P, i32]),
    "spd_tgn_set_gemm_mode": (i32, [P, i32]),
    "spd_tgn_debug_scratch": (i32, [P, C.c_char_p, pf32, u64, pu64]),
    "spd_tgn_set_profile": (i32, [P, i32]),
    "spd_edge_feature": (f32, [u64, u64, u32]),
}

MISSING = []
for _name, (_res, _args) in _SIGS.items():
    try:
        _fn = getattr(lib, _name)
    except AttributeError:
        MISSING.append(_name)
        continue
    _fn.restype = _res
    _fn.argtypes = _args


def ptr(a: np.ndarray | None, ctype=None):
    """numpy array -> ctypes pointer (None -> NULL)."""
    if a is None:
        return None
    if ctype is None:
        return a.ctypes.data_as(C.c_void_p)
    return a.ctypes.data_as(C.POINTER(ctype))
