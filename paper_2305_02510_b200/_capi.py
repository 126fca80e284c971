"""ctypes binding of the engine's C ABI (include/superneuro_mat.h).

The shared library ``libsnmat.so`` is built in-tree by ``__graft_entry__.build()``
(nvcc, sm_100a).  There is no fallback: if the library is missing this module
raises at import, and every compute call needs a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SNB_LIB") or os.path.join(_HERE, "libsnmat.so")  # SNB_LIB: A/B builds

SN_OK = 0
SN_ERR_INVALID_ARGUMENT = 1
SN_ERR_LOGIC = 2
SN_ERR_CUDA = 3
SN_ERR_NCCL = 4
SN_ERR_OOM = 5
SN_ERR_UNSUPPORTED = 6

SN_STORAGE_AUTO, SN_STORAGE_DENSE, SN_STORAGE_SPARSE = 0, 1, 2
SN_WEIGHTS_F32, SN_WEIGHTS_F64 = 0, 1
SN_MODE_MAT, SN_MODE_ABM = 0, 1
SN_ABI_VERSION = 2


class Options(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32),
        ("device", C.c_int32),
        ("storage", C.c_int32),
        ("precision", C.c_int32),
        ("exact_order", C.c_int32),
        ("record_membrane", C.c_int32),
        ("stream_io", C.c_int32),
        ("use_graphs", C.c_int32),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("profile", C.c_int32),
        ("persistent", C.c_int32),
        ("mode", C.c_int32),
        ("reserved", C.c_int32 * 3),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("steps_done", C.c_int64),
        ("spike_count", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("synapses_local", C.c_int64),
        ("dense", C.c_int32),
        ("n_local", C.c_int32),
        ("first_local", C.c_int32),
        ("max_delay", C.c_int32),
        ("sweep_ms", C.c_double),
        ("sweep_launches", C.c_int64),
        ("neuron_ms", C.c_double),
        ("neuron_launches", C.c_int64),
        ("exchange_ms", C.c_double),
        ("last_simulate_ms", C.c_double),
        ("sweep_bytes_per_launch_last", C.c_double),
        ("sweep_bytes_total", C.c_double),
        ("sweep_kernel", C.c_int32),
        ("sweep_ctas", C.c_int32),
        ("h2d_bytes_last", C.c_double),
        ("d2h_bytes_last", C.c_double),
    ]

    KERNEL_NAMES = {1: "k_dense_stream", 2: "k_dense_tma", 3: "k_dense_sweep<exact>",
                    4: "k_persistent_dense", 5: "k_sparse_pull", 6: "k_sparse_pull<dict>",
                    7: "k_sparse_stream", 8: "k_sparse_exact", 9: "k_tiny",
                    10: "k_sparse_tma", 11: "k_sparse_count", 12: "k_persistent_cols",
                    13: "k_sparse_count16", 14: "k_cluster_count", 15: "k_sparse_count8"}

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the engine."""


class NcclError(RuntimeError):
    """An NCCL failure inside the engine."""


_P = C.c_void_p
_i32, _i64, _u64, _dbl = C.c_int32, C.c_int64, C.c_uint64, C.c_double
_pi32, _pi64, _pdbl, _pu8, _pu32 = (C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                                    C.POINTER(C.c_uint32))

# name -> (restype, argtypes); the list is also the export contract checked by
# tests/test_capi_symbols.py against include/superneuro_mat.h
SIGNATURES = {
    "sn_options_init": (_i32, [C.POINTER(Options)]),
    "sn_engine_create": (_i32, [C.POINTER(Options), C.POINTER(_P)]),
    "sn_engine_destroy": (None, [_P]),
    "sn_last_error": (C.c_char_p, []),
    "sn_abi_version": (_i32, []),
    "sn_device_count": (_i32, []),
    "sn_add_neurons": (_i32, [_P, _i64, _pdbl, _pdbl, _pdbl, _pi32, _pi32, _pi64]),
    "sn_add_synapses": (_i32, [_P, _i64, _pi32, _pi32, _pdbl, _pi32, _pu8]),
    "sn_add_stimulus": (_i32, [_P, _i64, _pi32, _pi32, _pdbl]),
    "sn_clear_stimulus": (_i32, [_P]),
    "sn_set_stdp": (_i32, [_P, _i32, _pdbl, _pdbl, _dbl, _dbl]),
    "sn_stdp_defaults": (_i32, [_pi32, _pdbl, _pdbl, _pdbl, _pdbl]),
    "sn_generate_erdos_renyi": (_i32, [_P, _i32, _dbl, _u64, _dbl, _i32, _u64, _i32, _i32]),
    "sn_set_seed": (_i32, [_P, _u64]),
    "sn_set_fire_probability": (_i32, [_P, _i64, _i64, _pdbl]),
    "sn_setup": (_i32, [_P]),
    "sn_simulate": (_i32, [_P, _i32]),
    "sn_synchronize": (_i32, [_P]),
    "sn_step": (_i32, [_P, _pdbl, _i64, _pi32, _i64, _pi64]),
    "sn_simulate_raster": (_i32, [_P, _i32, _pi32, _pi32, _i64, _pi64]),
    "sn_set_plasticity": (_i32, [_P, _i32]),
    "sn_raster_size": (_i32, [_P, _pi64]),
    "sn_get_raster": (_i32, [_P, _pi32, _pi32, _i64]),
    "sn_clear_raster": (_i32, [_P]),
    "sn_get_membrane": (_i32, [_P, _pdbl, _i64]),
    "sn_membrane_trace_rows": (_i32, [_P, _pi64]),
    "sn_get_membrane_trace": (_i32, [_P, _pdbl, _i64]),
    "sn_get_synapse_weights": (_i32, [_P, _pdbl, _i64]),
    "sn_get_weight_matrix": (_i32, [_P, _pdbl, _i64]),
    "sn_weight_value_counts": (_i32, [_P, _pdbl, _i32, _pi64]),
    "sn_get_stats": (_i32, [_P, C.POINTER(Stats)]),
    "sn_reset_stats": (_i32, [_P]),
    "sn_comm_id_size": (_i32, []),
    "sn_comm_create_id": (_i32, [_pu8]),
    "sn_comm_init": (_i32, [_P, _pu8, _i32, _i32]),
    "sn_partition_range": (_i32, [_i32, _i32, _i32, _pi32, _pi32]),
    "sn_step_local": (_i32, [_P]),
    "sn_get_spike_words": (_i32, [_P, _pu32, _i64]),
    "sn_put_spike_words": (_i32, [_P, _i32, _pu32, _i64]),
    "sn_step_finish": (_i32, [_P]),
    "sn_p2p_handle_size": (_i32, []),
    "sn_p2p_get_handles": (_i32, [_P, _pu8, _i64]),
    "sn_p2p_open": (_i32, [_P, _pu8, _i32]),
    "sn_p2p_connect_local": (_i32, [C.POINTER(_P), _i32]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA engine first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback."
        )
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sn_abi_version() != SN_ABI_VERSION:
        raise ImportError("libsnmat.so ABI version mismatch; rebuild")
    return lib


lib = _load()


def check(status: int, what: str = "") -> None:
    """Map an sn_status to the exception the reference's bindings raise."""
    if status == SN_OK:
        return
    msg = lib.sn_last_error().decode("utf-8", "replace") or what
    if status == SN_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)          # pybind11: std::invalid_argument -> ValueError
    if status == SN_ERR_LOGIC:
        raise RuntimeError(msg)        # std::logic_error -> RuntimeError
    if status == SN_ERR_OOM:
        raise MemoryError(msg)
    if status == SN_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if status == SN_ERR_NCCL:
        raise NcclError(msg)
    raise CudaError(msg)


def ptr(arr, ctype):
    """ctypes pointer to a contiguous numpy array (or None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(C.POINTER(ctype))
