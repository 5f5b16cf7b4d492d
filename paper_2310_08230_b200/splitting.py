"""Constraint splitting (splitting.py:25-155 of the reference).

The split itself runs in the native lowering (csrc/dm_host.cpp
``split_bdd``/``split_and_flatten``); this module keeps the reference's
entry points.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .ilp import FlatTable, IlpInstance

DEFAULT_CHUNK_SIZE = 128


def plan_chunks(instance: IlpInstance, chunk_size: int) -> list[tuple[int, list[int]]]:
    """Which constraints get cut, and after which original layers (splitting.py:99-113)."""
    if chunk_size < 2:
        raise ValueError("chunk_size must be at least 2")
    f = instance.flat
    per = np.diff(f.bdd_layer_lo)
    return [(int(j), list(range(chunk_size, int(n), chunk_size))) for j, n in enumerate(per) if n > chunk_size]


def _local_tables(f: FlatTable):
    widths = np.diff(f.layer_node_lo)
    nxt = np.repeat(f.layer_node_lo[1:], widths)
    z = np.where(f.zero_t >= 0, f.zero_t - nxt, f.zero_t).astype(np.int32)
    o = np.where(f.one_t >= 0, f.one_t - nxt, f.one_t).astype(np.int32)
    return z, o


def split_instance(instance: IlpInstance, chunk_size: int = DEFAULT_CHUNK_SIZE) -> IlpInstance:
    """Cut every diagram longer than ``chunk_size`` layers every ``chunk_size``
    layers; auxiliary ids follow all originals and are visited right after
    their split anchor.  Returns the instance unchanged if nothing is cut."""
    if chunk_size < 2:
        raise ValueError("chunk_size must be at least 2")
    f = instance.flat
    if f.num_bdds == 0 or int(np.diff(f.bdd_layer_lo).max()) <= chunk_size:
        return instance
    z, o = _local_tables(f)
    lib = _native.load()
    h = ctypes.c_void_p()
    arrs = [np.ascontiguousarray(a) for a in (instance.costs, instance.variable_order, f.bdd_layer_lo,
                                              f.layer_var, f.layer_node_lo, z, o)]
    _native.check(lib.dm_instance_from_bdds(len(instance.costs), arrs[0].ctypes.data, arrs[1].ctypes.data,
                                            f.num_bdds, arrs[2].ctypes.data, arrs[3].ctypes.data,
                                            arrs[4].ctypes.data, arrs[5].ctypes.data, arrs[6].ctypes.data,
                                            int(chunk_size), ctypes.byref(h)), "split_instance")
    try:
        flat = FlatTable.from_native(h)
    finally:
        lib.dm_instance_free(h)
    return IlpInstance(flat.costs, flat=flat)
