"""ctypes binding of ``include/ds_cuda.h`` (``lib/libds_cuda.so``).

The shared library is built in-tree by ``paper_1602_08191_b200/Makefile`` (``build()``
in ``__graft_entry__``). There is no CPU fallback: if the library is missing this
module raises ImportError at import time, and every entry point reports a CUDA failure
as :class:`CudaError`.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DS_LIB_PATH: load an instrumented build of the same library (tools/ experiments)
LIB_PATH = os.environ.get("DS_LIB_PATH") or os.path.join(HERE, "lib", "libds_cuda.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C paper_1602_08191_b200` "
        "(or __graft_entry__.build()); the B200 hot path has no CPU fallback")

lib = C.CDLL(LIB_PATH)

DS_OK, DS_E_CONTRACT, DS_E_NUMERIC, DS_E_CUDA, DS_E_NOMEM, DS_E_STATE, DS_E_FORMAT, DS_E_IO = range(8)
DS_MODE_LOCKED, DS_MODE_LOCKFREE = 0, 1
DS_ENGINE_AUTO, DS_ENGINE_LAYERED, DS_ENGINE_FUSED, DS_ENGINE_TC = 0, 1, 2, 3
DS_IPC_RECORD_BYTES = 256
DS_STREAM_RING = 8  # include/ds_cuda.h

FLAG_X_NONFINITE = 1
FLAG_G_NONFINITE = 2
FLAG_OUT_NONFINITE = 4
FLAG_LOSS_NONFINITE = 8
FLAG_GRAD_NONFINITE = 16
FLAG_LABEL_RANGE = 32


class DsError(RuntimeError):
    code = -1


class ContractError(DsError):
    """deepspark::ContractError (errors.hpp:10-13)."""
    code = DS_E_CONTRACT


class NumericError(DsError):
    """deepspark::NumericError (errors.hpp:16-19)."""
    code = DS_E_NUMERIC


class CudaError(DsError):
    code = DS_E_CUDA


class StateError(DsError):
    code = DS_E_STATE


class FormatError(DsError):
    """deepspark::FormatError (errors.hpp:33-36): a malformed DSHD shard."""
    code = DS_E_FORMAT


class IoError(DsError):
    """deepspark::IoError (errors.hpp:56-59)."""
    code = DS_E_IO


_ERRS = {DS_E_CONTRACT: ContractError, DS_E_NUMERIC: NumericError, DS_E_CUDA: CudaError,
         DS_E_NOMEM: CudaError, DS_E_STATE: StateError, DS_E_FORMAT: FormatError, DS_E_IO: IoError}


def check(rc: int) -> None:
    if rc != DS_OK:
        msg = lib.ds_last_error().decode(errors="replace")
        raise _ERRS.get(rc, DsError)(msg)


class ds_model_desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_features", C.c_uint32), ("n_classes", C.c_uint32),
                ("n_hidden", C.c_uint32), ("hidden", C.POINTER(C.c_uint32))]


class ds_shard_info(C.Structure):
    _fields_ = [("n_samples", C.c_uint32), ("n_features", C.c_uint32), ("n_classes", C.c_uint32),
                ("seed", C.c_uint64)]


class ds_hyper(C.Structure):
    _fields_ = [("eta", C.c_double), ("alpha", C.c_double), ("tau", C.c_uint32),
                ("batch_size", C.c_uint32), ("i_max", C.c_uint64), ("loss_cut", C.c_double),
                ("weight_decay", C.c_double), ("adaptive", C.c_int32)]


VP = C.c_void_p
U64 = C.c_uint64
U32 = C.c_uint32
P_U64 = C.POINTER(C.c_uint64)
P_U32 = C.POINTER(C.c_uint32)
P_F = C.POINTER(C.c_float)
P_D = C.POINTER(C.c_double)


def _sig(name, *args, res=C.c_int):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)
    return fn


_sig("ds_last_error", res=C.c_char_p)
_sig("ds_version", res=C.c_char_p)
_sig("ds_device_count", C.POINTER(C.c_int))
_sig("ds_elastic_update", VP, VP, U64, C.c_float, VP)
_sig("ds_elastic_exchange", VP, VP, VP, U64, C.c_float, VP)
_sig("ds_sgd_update", VP, VP, VP, U64, C.c_float, C.c_float, VP, VP)
_sig("ds_sgd_step_checked", VP, VP, VP, U64, C.c_double, VP)
_sig("ds_grad_accumulate", VP, VP, U64, VP)
_sig("ds_sgd_momentum_update", VP, VP, VP, VP, U64, C.c_float, C.c_float, C.c_float, VP, VP)
_sig("ds_engine_set_momentum", VP, C.c_float)
_sig("ds_engine_attach_sync", VP, VP)
_sig("ds_grad_average", VP, VP, U64, U32, C.c_float, VP, VP)
_sig("ds_device_alloc", C.c_int, U64, C.POINTER(VP))
_sig("ds_device_free", VP)
_sig("ds_memcpy", VP, VP, U64, VP)
_sig("ds_memset", VP, C.c_int, U64, VP)
_sig("ds_stream_create", C.c_int, C.POINTER(VP))
_sig("ds_stream_destroy", VP)
_sig("ds_stream_sync", VP)
_sig("ds_param_dim", C.POINTER(ds_model_desc), P_U64)
_sig("ds_loss_and_grad_workspace", C.POINTER(ds_model_desc), U32, P_U64)
_sig("ds_loss_and_grad", C.POINTER(ds_model_desc), VP, VP, VP, U32, VP, VP, VP, VP, VP)
_sig("ds_predict", C.POINTER(ds_model_desc), VP, VP, U64, VP, VP)
_sig("ds_count_hits", C.POINTER(ds_model_desc), VP, VP, VP, U64, VP, VP)
_sig("ds_master_create", C.POINTER(VP), C.c_int, U64, C.c_float, C.c_int, VP)
_sig("ds_master_create_sharded", C.POINTER(VP), C.c_int, U64, C.c_float, C.c_int, C.c_int, C.c_int, VP)
_sig("ds_master_export", VP, VP)
_sig("ds_master_attach", VP, VP)
_sig("ds_master_destroy", VP)
_sig("ds_master_exchange", VP, VP, VP, VP)
_sig("ds_master_exchange_ticketed", VP, VP, VP, U64, VP)
_sig("ds_master_snapshot", VP, VP)
_sig("ds_master_local_slice", VP, C.POINTER(VP), P_U64, P_U64)
_sig("ds_master_exchange_count", VP, P_U64)
_sig("ds_master_dim", VP, P_U64)
_sig("ds_master_reset_tickets", VP)
_sig("ds_engine_create", C.POINTER(VP), C.c_int, C.POINTER(ds_model_desc), VP, VP, U64, U32,
     C.POINTER(ds_hyper), U64, VP, C.c_int)
_sig("ds_engine_destroy", VP)
_sig("ds_engine_attach_master", VP, VP)
_sig("ds_engine_set_tickets", VP, VP, U64)
_sig("ds_engine_run", VP, U64, C.c_int, P_U64)
_sig("ds_engine_run_group", C.POINTER(VP), U32, U64)
_sig("ds_engine_stream_begin_group", C.POINTER(VP), U32, U64, C.POINTER(VP))
_sig("ds_engine_reserve", VP, U64)
_sig("ds_engine_step_host", VP, VP, VP, U32, VP)
_sig("ds_engine_step_host_async", VP, VP, VP, U32, VP)
_sig("ds_engine_stream_begin", VP, U64, VP)
_sig("ds_engine_stream_push", VP, VP, VP, U32)
_sig("ds_engine_stream_push_rows", VP, VP, VP, VP, U32)
_sig("ds_engine_stream_push_rows_n", VP, VP, VP, VP, VP, U64)
_sig("ds_engine_stream_cache_host_shard", VP, VP, U64)
_sig("ds_host_rows_to_bf16", VP, U32, VP, U32, VP, U64)
_sig("ds_engine_stream_end", VP)
_sig("ds_engine_sync", VP)
_sig("ds_engine_stream", VP, C.POINTER(VP))
_sig("ds_engine_log", VP, U64, U64, VP, VP, VP, VP)
_sig("ds_engine_iterations", VP, P_U64)
_sig("ds_engine_get_params", VP, VP)
_sig("ds_engine_set_params", VP, VP)
_sig("ds_engine_params_device", VP, C.POINTER(VP))
_sig("ds_engine_policy", VP, P_D, P_U32, P_D)
_sig("ds_engine_launches", VP, P_U64)
_sig("ds_sync_create", C.POINTER(VP), C.c_int, U64, C.c_int, C.c_int)
_sig("ds_sync_export", VP, VP)
_sig("ds_sync_attach", VP, VP)
_sig("ds_sync_begin", VP, C.POINTER(VP), VP)
_sig("ds_sync_reduce_update", VP, VP, C.c_float, C.c_float, VP, VP)
_sig("ds_sync_easgd_update", VP, VP, VP, C.c_float, VP, VP)
_sig("ds_sync_reduce_update_group", C.POINTER(VP), U32, C.POINTER(VP), C.c_float, C.c_float, VP, VP)
_sig("ds_sync_easgd_update_group", C.POINTER(VP), U32, C.POINTER(VP), C.POINTER(VP), C.c_float, VP, VP)
_sig("ds_sync_peer_read", VP, VP, U64, VP)
_sig("ds_sync_rounds", VP, P_U64)
_sig("ds_sync_destroy", VP)
_sig("ds_gather_rows", VP, VP, VP, VP, VP, U32, U32, VP)
_sig("ds_gemm_tf32", VP, U64, VP, U64, VP, U64, U32, U32, U32, C.c_float, VP, VP, C.c_int, U32, VP, VP)
_sig("ds_shard_info_read", C.c_char_p, C.POINTER(ds_shard_info))
_sig("ds_shard_load", C.c_char_p, VP, VP, U64, C.POINTER(ds_shard_info), VP)
_sig("ds_engine_create_from_shard", C.POINTER(VP), C.c_int, C.POINTER(ds_model_desc), C.c_char_p,
     C.POINTER(ds_hyper), U64, VP, C.c_int)

EXPORTED = [
    "ds_gemm_tf32", "ds_shard_info_read", "ds_shard_load", "ds_engine_create_from_shard",
    "ds_last_error", "ds_version", "ds_device_count", "ds_elastic_update", "ds_elastic_exchange",
    "ds_sgd_update", "ds_sgd_step_checked", "ds_sgd_momentum_update", "ds_engine_set_momentum", "ds_engine_attach_sync", "ds_grad_accumulate", "ds_grad_average", "ds_device_alloc",
    "ds_device_free", "ds_memcpy", "ds_memset", "ds_stream_create", "ds_stream_destroy", "ds_stream_sync",
    "ds_param_dim", "ds_loss_and_grad_workspace",
    "ds_loss_and_grad", "ds_predict", "ds_count_hits", "ds_master_create", "ds_master_create_sharded",
    "ds_master_export", "ds_master_attach", "ds_master_destroy", "ds_master_exchange",
    "ds_master_exchange_ticketed", "ds_master_snapshot", "ds_master_local_slice",
    "ds_master_exchange_count", "ds_master_dim", "ds_master_reset_tickets", "ds_engine_create",
    "ds_engine_destroy", "ds_engine_attach_master", "ds_engine_set_tickets", "ds_engine_run", "ds_engine_run_group", "ds_engine_stream_begin_group", "ds_engine_reserve", "ds_engine_step_host", "ds_engine_step_host_async",
    "ds_engine_stream_begin", "ds_engine_stream_push", "ds_engine_stream_push_rows", "ds_engine_stream_push_rows_n", "ds_engine_stream_cache_host_shard", "ds_host_rows_to_bf16",
    "ds_engine_stream_end",
    "ds_engine_sync", "ds_engine_stream", "ds_engine_log", "ds_engine_iterations",
    "ds_engine_get_params", "ds_engine_set_params", "ds_engine_params_device", "ds_engine_policy",
    "ds_engine_launches", "ds_sync_create", "ds_sync_export", "ds_sync_attach", "ds_sync_begin",
    "ds_sync_reduce_update", "ds_sync_easgd_update", "ds_sync_reduce_update_group",
    "ds_sync_easgd_update_group", "ds_sync_peer_read", "ds_sync_rounds", "ds_sync_destroy", "ds_gather_rows",
]


def version() -> str:
    return lib.ds_version().decode()


def device_count() -> int:
    n = C.c_int(0)
    check(lib.ds_device_count(C.byref(n)))
    return n.value
