"""ctypes binding of libdiscomatch_b200.so (include/discomatch_b200.h).

The product path has no fallback: if the shared library is missing or fails
to load, every solver entry point raises.  Device vectors are torch CUDA
tensors passed by data pointer on the current torch stream.
"""

from __future__ import annotations

import ctypes
import os

from .errors import EmptyFeasibleSet, NativeLibraryError, ProdmatchError, UnsupportedInstance

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DM_LIB_PATH") or os.path.join(_HERE, "libdiscomatch_b200.so")

DM_OK = 0
DM_ERR_INVALID = -1
DM_ERR_INFEASIBLE = -2
DM_ERR_CUDA = -3
DM_ERR_UNSUPPORTED = -4

_P = ctypes.c_void_p
_I = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int


class InstanceInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "num_variables", "num_bdds", "num_layers", "num_nodes", "max_width", "max_degree",
        "max_layers")]


class FlatDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("num_bdds", "num_layers", "num_nodes", "num_positions")] + [
        (n, ctypes.c_void_p) for n in ("bdd_layer_lo", "layer_node_lo", "layer_var", "zero_t", "one_t",
                                       "proc_ptr", "proc_layers")]


class FlatInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "fw_depth", "bw_depth", "fw_tasks", "bw_tasks", "mma_grid", "mma_block", "max_width",
        "max_degree", "device_bytes", "lanes_per_task", "dfr_node_parallel")]


# name -> (argtypes, restype); kept in sync with include/discomatch_b200.h
SIGNATURES = {
    "dm_last_error": ([], ctypes.c_char_p),
    "dm_version": ([], ctypes.c_char_p),
    "dm_instance_from_rows": ([_I, _P, _I, _P, _P, _P, _P, _I, ctypes.POINTER(_P)], _INT),
    "dm_instance_from_bdds": ([_I, _P, _P, _I, _P, _P, _P, _P, _P, _I, ctypes.POINTER(_P)], _INT),
    "dm_condition_flat": ([_I, _P, _P, _I, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_I), ctypes.POINTER(_P)], _INT),
    "dm_row_colouring": ([_I, _I, _P, _P, _P], _INT),
    "dm_instance_get_info": ([_P, ctypes.POINTER(InstanceInfo)], _INT),
    "dm_instance_export": ([_P] + [_P] * 11, _INT),
    "dm_instance_free": ([_P], None),
    "dm_flat_create": ([ctypes.POINTER(FlatDesc), _INT, _P, ctypes.POINTER(_P)], _INT),
    "dm_flat_create_ex": ([ctypes.POINTER(FlatDesc), _INT, _P, _INT, ctypes.POINTER(_P)], _INT),
    "dm_flat_get_info": ([_P, ctypes.POINTER(FlatInfo)], _INT),
    "dm_flat_status": ([_P, _P], _INT),
    "dm_flat_set_mma_config": ([_P, _INT, _INT, _INT, _INT, _INT], _INT),
    "dm_flat_set_trace": ([_P, _P], _INT),
    "dm_flat_task_levels": ([_P, _INT, _P, _P], _INT),
    "dm_flat_destroy": ([_P], None),
    "dm_k_backward": ([_P, _P, _P, _P, _P], _INT),
    "dm_qn_move": ([_P, _P, _P, _D, _P, _P, _P, _P, _P], _INT),
    "dm_k_backward_trial": ([_P, _P, _P, _D, _P, _P, _P], _INT),
    "dm_debug_div_check": ([_INT, ctypes.c_uint64, ctypes.c_uint64, _P], _INT),
    "dm_flat_status_to": ([_P, _P, _P], _INT),
    "dm_step_search": ([_P, _P, _P, _D, _D, _D, _D, _D, _INT, _P, _P, _P], _INT),
    "dm_k_forward": ([_P, _P, _P, _P, _P], _INT),
    "dm_k_mma_forward": ([_P, _P, _P, _P, _P, _P], _INT),
    "dm_k_mma_backward": ([_P, _P, _P, _P, _P, _P], _INT),
    "dm_k_min_marginals": ([_P, _P, _P, _P, _P, _P, _P], _INT),
    "dm_k_argmin": ([_P, _P, _P, _P, _P], _INT),
    "dm_k_argmin_from_pass": ([_P, _P, _P, _P], _INT),
    "dm_dfr_table_size": ([_P, ctypes.POINTER(_I)], _INT),
    "dm_dfr_forward": ([_P, _D, _P, _P, _P, _P, _P, _P, _P], _INT),
    "dm_dfr_backward": ([_P, _D, _P, _P, _P, _P, _P, _P, _INT, _P], _INT),
    "dm_dfr_np_forward": ([_P, _D, _P, _P, _P, _P, _P, _P, _P], _INT),
    "dm_dfr_np_backward": ([_P, _D, _P, _P, _P, _P, _P, _P, _INT, _P], _INT),
    "dm_dfr_average": ([_P, _P, _P, _P], _INT),
    "dm_dfr_flush": ([_P, _P, _P, _P], _INT),
    "dm_dfr_average_csr": ([_I, _P, _P, _P, _P, _INT, _P], _INT),
    "dm_dfr_boundary_gather": ([_I, _P, _P, _P, _P, _P], _INT),
    "dm_dfr_boundary_average": ([_I, _P, _P, _P, _P, _P, _P, _INT, _P], _INT),
    "dm_dfr_to_nodes": ([_P, _P, _P, _P], _INT),
    "dm_perturb_round": ([_P, _P, _P, _P, _D, _D, ctypes.c_uint64, _INT, _P, _P, _P, _P], _INT),
    "dm_batch_create": ([_P, _INT, _P, _P, _P, ctypes.POINTER(_P)], _INT),
    "dm_batch_destroy": ([_P], None),
    "dm_batch_sum": ([_P, _P, _P, _P], _INT),
    "dm_batch_dot": ([_P, _P, _P, _P, _P, _P], _INT),
    "dm_batch_update": ([_P, _INT, _P, _P, _P, _P, _P, _P, _P, _P], _INT),
    "dm_batch_curvature": ([_P, _P, _P, _P, _P, _P, _P, _P, _P], _INT),
    "dm_batch_step_search": ([_P, _P, _P, _P, _P, _P, _P, _D, _D, _INT, _P, _P, _P, _P, _P], _INT),
    "dm_init_duals": ([_P, _P, _P, _P], _INT),
    "dm_project_direction": ([_P, _P, _P, _P], _INT),
    "dm_lambda_sums": ([_P, _P, _P, _P], _INT),
    "dm_agreement_scores": ([_P, _P, _P, _P, _P, _P, _P], _INT),
    "dm_sum": ([_P, _I, _P, _P], _INT),
    "dm_release_caches": ([], _INT),
    "dm_dot": ([_P, _P, _I, _P, _P], _INT),
    "dm_axpy_dev": ([_P, _P, _D, _P, _P, _I, _P], _INT),
    "dm_scale_dev": ([_P, _D, _P, _I, _P], _INT),
    "dm_lbfgs_up": ([_P, _P, _P, _D, _P, _I, _P], _INT),
    "dm_lbfgs_direction": ([_P, _P, _P, _P, _P, _INT, _I, _P, _P], _INT),
    "dm_curvature_pair": ([_P, _P, _P, _P, _P, _P, _I, _P, _P], _INT),
    "dm_axpy_host": ([_P, _D, _P, _I, _P], _INT),
    "dm_sub": ([_P, _P, _P, _I, _P], _INT),
    "dm_host_pairwise_sum": ([_P, _I, _P], _INT),
    "dm_debug_emulate_mma": ([ctypes.POINTER(FlatDesc), _INT, _P, _P, _P, _P, ctypes.POINTER(_I)], _INT),
}

_lib = None


def load():
    """Load the native library (raises NativeLibraryError when absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - environment specific
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def last_error() -> str:
    return load().dm_last_error().decode()


def check(rc: int, what: str = "") -> None:
    if rc == DM_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == DM_ERR_INFEASIBLE:
        raise EmptyFeasibleSet(msg)
    if rc == DM_ERR_INVALID:
        raise ValueError(msg)
    if rc == DM_ERR_UNSUPPORTED:
        raise UnsupportedInstance(msg)
    raise ProdmatchError(msg)


# kernels each entry point launches (for the bench's gpu_launches claim)
LAUNCHES = {"dm_k_mma_forward": 3, "dm_k_mma_backward": 2, "dm_sum": 2, "dm_curvature_pair": 2, "dm_qn_move": 2}
KERNEL_ENTRIES = {"dm_k_backward", "dm_k_backward_trial", "dm_qn_move", "dm_k_forward", "dm_k_mma_forward",
                  "dm_k_mma_backward", "dm_k_min_marginals", "dm_k_argmin", "dm_init_duals",
                  "dm_project_direction", "dm_lambda_sums", "dm_agreement_scores", "dm_sum", "dm_dot",
                  "dm_axpy_dev", "dm_scale_dev", "dm_lbfgs_up", "dm_axpy_host", "dm_sub",
                  "dm_lbfgs_direction", "dm_k_argmin_from_pass", "dm_curvature_pair", "dm_step_search",
                  "dm_flat_status_to", "dm_dfr_forward", "dm_dfr_backward", "dm_dfr_np_forward", "dm_dfr_np_backward", "dm_dfr_average", "dm_dfr_flush", "dm_dfr_to_nodes",
                  "dm_dfr_average_csr", "dm_dfr_boundary_gather", "dm_dfr_boundary_average",
                  "dm_perturb_round", "dm_batch_sum", "dm_batch_dot", "dm_batch_update", "dm_batch_curvature",
                  "dm_batch_step_search"}
launch_count = 0


def call(name: str, *args, launches: int | None = None) -> None:
    global launch_count
    check(getattr(load(), name)(*args), name)
    if name in KERNEL_ENTRIES:
        launch_count += launches if launches is not None else LAUNCHES.get(name, 1)
