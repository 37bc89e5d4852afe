"""ctypes binding of librsgpu.so (the C-ABI declared in include/rsgpu.h).

The shared library is built in-tree by ``paper_2505_12663_b200/csrc/Makefile``
(nvcc, sm_100a only).  There is no CPU fallback: if the library cannot be
loaded, importing the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# RS_LIB_PATH: load another build (kernel-variant experiments)
LIB_PATH = os.environ.get("RS_LIB_PATH") or os.path.join(HERE, "_lib", "librsgpu.so")
CSRC = os.path.join(HERE, "csrc")

RS_OK, RS_ERR_CONFIG, RS_ERR_INVARIANT, RS_ERR_IO, RS_ERR_CUDA, RS_ERR_CAPACITY, RS_ERR_RANGE = range(7)
RS_OPT_NONE, RS_OPT_ADAM, RS_OPT_ADAGRAD = 0, 1, 2


# Exception taxonomy of the reference (common.hpp:24-39) + the GPU build's.
class RecsparseError(RuntimeError):
    status = -1


class ConfigError(RecsparseError):
    status = RS_ERR_CONFIG


class InvariantError(RecsparseError):
    status = RS_ERR_INVARIANT


class IoError(RecsparseError):
    status = RS_ERR_IO


class CudaError(RecsparseError):
    status = RS_ERR_CUDA


class CapacityError(RecsparseError):
    status = RS_ERR_CAPACITY


class RangeError(RecsparseError, OverflowError):
    status = RS_ERR_RANGE


_ERR = {c.status: c for c in (ConfigError, InvariantError, IoError, CudaError, CapacityError, RangeError)}


class rs_table_config(C.Structure):
    _fields_ = [("capacity", C.c_uint64), ("embedding_dim", C.c_uint32), ("thread_groups", C.c_uint32),
                ("max_load_factor", C.c_double), ("chunk_rows", C.c_uint32), ("optimizer", C.c_uint32),
                ("initial_rows", C.c_uint64), ("max_keys", C.c_uint64)]


class rs_feature_config(C.Structure):
    _fields_ = [("feature_name", C.c_char_p), ("embedding_dim", C.c_uint32),
                ("lookup_tables", C.POINTER(C.c_char_p)), ("n_lookup_tables", C.c_uint32), ("pooling", C.c_uint32)]


class rs_ckpt_header(C.Structure):
    _fields_ = [("version", C.c_uint32), ("world_size", C.c_uint32), ("shard_rank", C.c_uint32),
                ("embedding_dim", C.c_uint32), ("capacity", C.c_uint64), ("entry_count", C.c_uint64)]


class rs_optimizer_params(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double)]


class rs_table_info(C.Structure):
    _fields_ = [("capacity", C.c_uint64), ("occupied", C.c_uint64), ("tombstones", C.c_uint64),
                ("rows_allocated", C.c_uint64), ("rows_free", C.c_uint64), ("row_capacity", C.c_uint64),
                ("tick", C.c_uint64), ("embedding_dim", C.c_uint32), ("optimizer", C.c_uint32),
                ("host_syncs", C.c_uint64)]


vp = C.c_void_p
u64, u32, i32 = C.c_uint64, C.c_uint32, C.c_int32
rs_chunk_source = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_uint64,
                              C.POINTER(C.c_uint64))

# name -> (restype, argtypes)
_SIGS = {
    "rs_abi_version": (C.c_int, []),
    "rs_status_string": (C.c_char_p, [C.c_int]),
    "rs_last_error": (C.c_char_p, []),
    "rs_kernel_launches": (u64, []),
    "rs_buffer_alloc": (C.c_int, [u64, C.POINTER(vp)]),
    "rs_buffer_free": (C.c_int, [vp]),
    "rs_copy_to_device": (C.c_int, [vp, vp, u64]),
    "rs_copy_to_host": (C.c_int, [vp, vp, u64]),
    "rs_table_bump_tick": (C.c_int, [vp, u64]),
    "rs_table_clone": (C.c_int, [vp, C.POINTER(vp)]),
    "rs_table_read_entries": (C.c_int, [vp, vp, u64, vp, vp, vp, vp, vp, vp]),
    "rs_hash64_batch": (C.c_int, [vp, u64, vp, vp]),
    "rs_shard_of_batch": (C.c_int, [vp, u64, u32, vp, vp]),
    "rs_table_create": (C.c_int, [C.POINTER(rs_table_config), C.POINTER(vp)]),
    "rs_table_destroy": (C.c_int, [vp]),
    "rs_table_stats": (C.c_int, [vp, C.POINTER(rs_table_info)]),
    "rs_table_insert": (C.c_int, [vp, vp, u64, vp, vp]),
    "rs_table_find": (C.c_int, [vp, vp, u64, vp, vp]),
    "rs_table_lookup": (C.c_int, [vp, vp, u64, vp, vp]),
    "rs_table_ensure": (C.c_int, [vp, vp, u64, vp, vp]),
    "rs_table_remove": (C.c_int, [vp, vp, u64, vp, vp]),
    "rs_table_expand": (C.c_int, [vp, C.POINTER(u64), vp]),
    "rs_table_evict": (C.c_int, [vp, u64, C.POINTER(u64), vp]),
    "rs_table_gather_rows": (C.c_int, [vp, vp, u64, vp, vp]),
    "rs_table_export": (C.c_int, [vp, u64, vp, vp, vp, vp, vp, vp, C.POINTER(u64)]),
    "rs_table_import": (C.c_int, [vp, u64, vp, vp, vp, vp, vp, vp]),
    "rs_workspace_create": (C.c_int, [u64, C.POINTER(vp)]),
    "rs_workspace_destroy": (C.c_int, [vp]),
    "rs_dedup": (C.c_int, [vp, vp, u64, vp, vp, vp, vp]),
    "rs_forward": (C.c_int, [vp, vp, vp, u64, vp, vp]),
    "rs_backward": (C.c_int, [vp, vp, vp, u64, C.POINTER(rs_optimizer_params), vp]),
    "rs_step": (C.c_int, [vp, vp, vp, u64, vp, vp, C.POINTER(rs_optimizer_params), vp]),
    "rs_step_checksum": (C.c_int, [vp, vp, vp, u64, vp, vp, C.POINTER(rs_optimizer_params), vp, vp]),
    "rs_sparse_update": (C.c_int, [vp, vp, vp, u64, vp, C.POINTER(rs_optimizer_params), vp]),
    "rs_workspace_results": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    "rs_workspace_set_profiling": (C.c_int, [vp, C.c_int]),
    "rs_workspace_trace": (C.c_int, [vp, vp, u64, C.POINTER(u64)]),
    "rs_workspace_phase_ms": (C.c_int, [vp, vp, u32, C.POINTER(u64)]),
    "rs_workspace_unique": (C.c_int, [vp, vp, u64, C.POINTER(u64)]),
    "rs_workspace_n_unique": (C.c_int, [vp, C.POINTER(u64)]),
    "rs_accumulate": (C.c_int, [vp, vp, u64, vp, vp]),
    "rs_apply_aggregated": (C.c_int, [vp, vp, u64, vp, C.POINTER(rs_optimizer_params), vp]),
    "rs_comm_create": (C.c_int, [C.c_int, C.c_int, u64, u32, C.POINTER(vp)]),
    "rs_comm_ipc_handle": (C.c_int, [vp, vp]),
    "rs_comm_open": (C.c_int, [vp, vp]),
    "rs_comm_destroy": (C.c_int, [vp]),
    "rs_dist_forward": (C.c_int, [vp, vp, vp, u64, vp, vp]),
    "rs_dist_backward": (C.c_int, [vp, vp, vp, u64, C.POINTER(rs_optimizer_params), vp]),
    "rs_dist_step": (C.c_int, [vp, vp, vp, u64, vp, vp, C.POINTER(rs_optimizer_params), vp]),
    "rs_dist_step_checksum": (C.c_int, [vp, vp, vp, u64, vp, vp, C.POINTER(rs_optimizer_params), vp, vp]),
    "rs_comm_set_profiling": (C.c_int, [vp, C.c_int]),
    "rs_comm_barrier": (C.c_int, [vp, vp]),
    "rs_comm_phase_ms": (C.c_int, [vp, C.POINTER(C.c_double), C.c_int, C.POINTER(u64)]),
    "rs_comm_trace": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "rs_comm_timeline": (C.c_int, [vp, vp, u64, C.POINTER(u64)]),
    "rs_comm_create_local": (C.c_int, [C.c_int, u64, u32, vp]),
    "rs_dist_group_forward": (C.c_int, [vp, vp, C.c_int, vp, vp, vp, vp]),
    "rs_dist_group_backward": (C.c_int, [vp, vp, C.c_int, vp, vp, C.POINTER(rs_optimizer_params), vp]),
    "rs_dist_group_step": (C.c_int, [vp, vp, C.c_int, vp, vp, vp, vp, C.POINTER(rs_optimizer_params), vp]),
    "rs_plan_merge": (C.c_int, [C.POINTER(rs_feature_config), u32, C.POINTER(vp)]),
    "rs_merge_plan_destroy": (C.c_int, [vp]),
    "rs_merge_plan_groups": (u32, [vp]),
    "rs_merge_plan_group": (C.c_int, [vp, u32, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]),
    "rs_merge_plan_member": (C.c_char_p, [vp, u32, u32]),
    "rs_merge_plan_find": (C.c_int, [vp, C.c_char_p, C.POINTER(u32), C.POINTER(u32)]),
    "rs_collection_create": (C.c_int, [vp, C.POINTER(rs_table_config), C.POINTER(vp)]),
    "rs_collection_destroy": (C.c_int, [vp]),
    "rs_collection_table": (vp, [vp, u32]),
    "rs_collection_lookup": (C.c_int, [vp, C.POINTER(rs_feature_config), vp, u64, vp, vp]),
    "rs_router_create": (C.c_int, [vp, C.POINTER(C.c_char_p), u32, C.POINTER(vp)]),
    "rs_router_destroy": (C.c_int, [vp]),
    "rs_route_tagged": (C.c_int, [vp, vp, u64, vp, vp, vp, vp]),
    "rs_closest_prefix": (C.c_int, [vp, u64, u64, C.POINTER(u64)]),
    "rs_seq_batcher_create": (C.c_int, [u64, rs_chunk_source, vp, u64, C.POINTER(vp)]),
    "rs_seq_batcher_destroy": (C.c_int, [vp]),
    "rs_seq_batcher_next": (C.c_int, [vp, vp, vp, u64, C.POINTER(u64)]),
    "rs_seq_batcher_buffered_tokens": (u64, [vp]),
    "rs_seq_batcher_buffered_samples": (u64, [vp]),
    "rs_partition_sequences": (C.c_int, [vp, u64, u32, u32, C.c_double, C.c_double, vp, vp]),
    "rs_imbalance_report": (C.c_int, [vp, u64, C.POINTER(u64), C.POINTER(u64), C.POINTER(C.c_double)]),
    "rs_weighted_grad_combine": (C.c_int, [vp, vp, u64, u64, vp]),
    "rs_pseudo_grads_jagged": (C.c_int, [vp, u64, u64, u64, u32, u64, vp, vp]),
    "rs_checksum": (C.c_int, [vp, u64, vp, vp]),
    "rs_pseudo_grads_offsets": (C.c_int, [vp, u64, u64, u64, u32, vp, vp]),
    "rs_pseudo_grads_chunks": (C.c_int, [vp, u32, u64, u64, u32, vp, vp]),
    "rs_feeder_create": (C.c_int, [u64, u64, u32, C.POINTER(vp)]),
    "rs_feeder_destroy": (C.c_int, [vp]),
    "rs_feeder_out": (vp, [vp, C.c_int]),
    "rs_feeder_step": (C.c_int, [vp, vp, vp, vp, u64, vp, u64, u64, u64, C.POINTER(rs_optimizer_params), vp, vp]),
    "rs_feeder_dist_step": (C.c_int, [vp, vp, vp, vp, u64, vp, u64, u64, u64, C.POINTER(rs_optimizer_params), vp,
                                      vp]),
    "rs_ckpt_shard_file_name": (C.c_int, [u32, u32, C.c_char_p, u64]),
    "rs_ckpt_save_shard": (C.c_int, [vp, u32, u32, C.c_char_p]),
    "rs_ckpt_read_header": (C.c_int, [C.c_char_p, C.POINTER(rs_ckpt_header)]),
    "rs_ckpt_load_shard": (C.c_int, [vp, C.c_char_p, u32, u32, u32]),
    "rs_encode_ids": (C.c_int, [vp, u64, u32, u32, u32, vp, vp]),
    "rs_workload_generate": (C.c_int, [u64, u64, C.c_double, u64, C.c_double, C.c_double, u32, vp, vp, vp,
                                       u64, C.POINTER(u64)]),
    "rs_pseudo_grads": (C.c_int, [vp, u64, u64, u32, vp, vp]),
    "rs_workload_write": (C.c_int, [C.c_char_p, u64, u64, C.c_double, u64, C.c_double, C.c_double, u32, vp]),
    "rs_workload_read": (C.c_int, [C.c_char_p, u64, u64, vp, vp, vp, vp, C.POINTER(u64), C.POINTER(u64)]),
}

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile librsgpu.so for sm_100a in-tree (nvcc).  Returns its path."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", CSRC, "-j8"], check=True)
    return LIB_PATH


def lib():
    """Load (building if needed) librsgpu.so.  Raises if it cannot be loaded."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name, None)
                if fn is None:
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = L
        return _lib


def check(status: int, what: str = "") -> None:
    if status == RS_OK:
        return
    L = lib()
    msg = (L.rs_last_error() or b"").decode(errors="replace")
    cls = _ERR.get(status, RecsparseError)
    raise cls(f"{what}: {L.rs_status_string(status).decode()}: {msg}")


def exported_symbols():
    return [n for n in _SIGS if getattr(lib(), n, None) is not None]
