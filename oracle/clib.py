"""ORACLE — TEST INFRASTRUCTURE ONLY.  ctypes binding of oracle/ckernels.c."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "liboracle.so")


def build_oracle(force: bool = False) -> str:
    src = os.path.join(_HERE, "ckernels.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_P = ctypes.c_void_p
_I = ctypes.c_int64
_D = ctypes.c_double


class _Lib:
    def __init__(self):
        self._h = None

    def _load(self):
        if self._h is None:
            build_oracle()
            h = ctypes.CDLL(_SO)
            sig = {
                "oracle_set_threads": ([ctypes.c_int], ctypes.c_int),
                "oracle_max_threads": ([], ctypes.c_int),
                "oracle_k_backward": ([_I, _P, _P, _P, _P, _P, _P, _P], None),
                "oracle_k_backward_trial": ([_I, _P, _P, _P, _P, _P, _P, _D, _P, _P], None),
                "oracle_k_forward": ([_I, _P, _P, _P, _P, _P, _P, _P], None),
                "oracle_k_mma_forward": ([_I, _I] + [_P] * 13, None),
                "oracle_k_mma_backward": ([_I, _I] + [_P] * 13, None),
                "oracle_k_min_marginals": ([_I] + [_P] * 8, None),
                "oracle_k_argmin": ([_I] + [_P] * 7, None),
                "oracle_equality_tables": ([_I, _P, _I, _P, _P, _P], _I),
                "oracle_dfr_forward": ([_I, _P, _P, _P, _P, _D] + [_P] * 6, None),
                "oracle_dfr_backward": ([_I, _P, _P, _P, _P, _D] + [_P] * 6, None),
                "oracle_dfr_average": ([_I, _P, _P, _P, _P], None),
                "oracle_row_colouring": ([_I, _I, _P, _P, _P], _I),
            }
            for name, (args, res) in sig.items():
                fn = getattr(h, name)
                fn.argtypes = args
                fn.restype = res
            self._h = h
        return self._h

    def __getattr__(self, name):
        return getattr(self._load(), name)


lib = _Lib()


def ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be contiguous"
    return a.ctypes.data


def row_colouring(p) -> np.ndarray:
    """Greedy row colouring of a ProductSpace (oracle_row_colouring): the CPU
    arm's copy of the product's dm_row_colouring."""
    colour = np.empty(p.num_variables, np.int64)
    rp = np.ascontiguousarray(p.row_ptr, dtype=np.int64)
    rv = np.ascontiguousarray(p.row_var, dtype=np.int64)
    if lib.oracle_row_colouring(p.num_variables, p.num_rows, ptr(rp), ptr(rv), ptr(colour)) < 0:
        raise ValueError("oracle_row_colouring: invalid rows")
    return colour
