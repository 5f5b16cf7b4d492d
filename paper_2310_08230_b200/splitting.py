"""Constraint splitting (splitting.py:25-155 of the reference).

The split itself runs in the native lowering (csrc/dm_host.cpp
``split_bdd``/``split_and_flatten``); this module keeps the reference's
entry points.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterator

import numpy as np

from . import _native
from .errors import SplitAtTerminalLayer
from .ilp import Bdd, FlatTable, IlpInstance

DEFAULT_CHUNK_SIZE = 128
_F, _T = -1, -2  # FALSE / TRUE terminals (bdd.py:24-25)


@dataclass(frozen=True)
class SplitResult:
    """The two coupled halves of a cut diagram and the coupling variables
    (splitting.py:28-32)."""

    left: Bdd
    right: Bdd
    aux_ids: list


def split_bdd(bdd: Bdd, split_after_layer: int, fresh_ids: Iterator[int]) -> SplitResult:
    """Cut one diagram after its first ``split_after_layer`` layers into two
    coupled by k fresh one-hot variables, k = width of the crossing layer
    (splitting.py:35-96; the same construction the native lowering applies,
    csrc/dm_host.cpp).  The left half reads the prefix and then y = e_t for
    the crossing node t it reached; the right half decodes y and resumes the
    suffix at node t.  Per-diagram API; instances are split natively by
    split_instance."""
    n = bdd.num_variables
    cut = int(split_after_layer)
    if not 1 <= cut < n:
        raise SplitAtTerminalLayer(f"split index {cut} outside [1, {n - 1}]")
    k = len(bdd.zeros[cut])
    aux = [next(fresh_ids) for _ in range(k)]

    def layer(width):
        return np.full(width, _F, np.int32), np.full(width, _F, np.int32)

    # left tail, layer q over y_q: slots 0..k-q-1 = crossing nodes q.. still
    # waiting for their bit, slot k-q (q > 0) = "bit already placed"
    lz, lo = [z.copy() for z in bdd.zeros[:cut]], [o.copy() for o in bdd.ones[:cut]]
    for q in range(k):
        waiting, final = k - q, q == k - 1
        z, o = layer(waiting + (q > 0))
        o[0] = _T if final else waiting - 1  # node q places its bit here -> "placed"
        z[1:waiting] = np.arange(waiting - 1)  # the others wait one more layer
        if q > 0:
            z[waiting] = _T if final else waiting - 1  # "placed" passes zeros
        lz.append(z)
        lo.append(o)
    # right head, layer q over y_q: slot 0 = nothing placed yet, slot t+1 =
    # placed at t; the last layer hands over to crossing node t of the suffix
    rz, ro = [], []
    for q in range(k):
        final = q == k - 1
        z, o = layer(q + 1)
        o[0] = q if final else q + 1
        if not final:
            z[0] = 0
        z[1:] = np.arange(q) + (0 if final else 1)
        rz.append(z)
        ro.append(o)
    rz += [z.copy() for z in bdd.zeros[cut:]]
    ro += [o.copy() for o in bdd.ones[cut:]]
    left = Bdd(list(bdd.variables[:cut]) + aux, lz, lo)
    right = Bdd(aux + list(bdd.variables[cut:]), rz, ro)
    return SplitResult(left, right, aux)


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
