"""0-1 equality ILPs whose constraints are layered decision diagrams.

Mirrors the reference containers (ilp.py:13-117, bdd.py:55-87) with the
same constructor signatures, but an instance built from rows lives as the
flat node table from the start: rows are compiled, split and flattened by
the native lowering (csrc/dm_host.cpp), never as per-row Python objects.
Per-diagram ``Bdd`` objects are materialised only on request.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from .errors import EmptyFeasibleSet

FALSE_T = -1
TRUE_T = -2


@dataclass(frozen=True)
class LinearRow:
    """One integer equality row (ilp.py:13-27)."""

    variables: np.ndarray
    coefficients: np.ndarray
    rhs: int
    tag: str = ""

    def residual(self, x: np.ndarray) -> int:
        return int(self.coefficients @ x[self.variables]) - self.rhs


def make_row(variables, coefficients, rhs, tag="") -> LinearRow:
    return LinearRow(np.asarray(variables, dtype=np.int64), np.asarray(coefficients, dtype=np.int64),
                     int(rhs), tag)


class Bdd:
    """Read-only view of one diagram in the reference layout (bdd.py:55-87)."""

    __slots__ = ("variables", "zeros", "ones")

    def __init__(self, variables, zeros, ones):
        variables = np.asarray(variables, dtype=np.int64)
        if variables.ndim != 1 or len(variables) == 0:
            raise ValueError("a diagram needs at least one variable")
        if len(set(variables.tolist())) != len(variables):
            raise ValueError("duplicate variable in constraint")
        if len(zeros) != len(variables) or len(ones) != len(variables):
            raise ValueError("layer count must match variable count")
        zeros = [np.asarray(z, dtype=np.int32) for z in zeros]
        ones = [np.asarray(o, dtype=np.int32) for o in ones]
        if len(zeros[0]) != 1:
            raise ValueError("first layer must hold exactly the root node")
        for z, o in zip(zeros, ones):
            if len(z) != len(o) or len(z) == 0:
                raise ValueError("malformed layer")
        self.variables, self.zeros, self.ones = variables, zeros, ones

    @property
    def num_variables(self) -> int:
        return len(self.variables)

    @property
    def widths(self) -> list[int]:
        return [len(z) for z in self.zeros]

    @property
    def num_nodes(self) -> int:
        return sum(len(z) for z in self.zeros)

    def __repr__(self) -> str:
        return f"Bdd({self.num_variables} vars, {self.num_nodes} nodes)"

    def accepts(self, bits) -> bool:
        if len(bits) != self.num_variables:
            raise ValueError("assignment length mismatch")
        node = 0
        for layer, bit in enumerate(bits):
            t = int((self.ones if bit else self.zeros)[layer][node])
            if t == FALSE_T:
                return False
            if t == TRUE_T:
                return layer == self.num_variables - 1
            node = t
        raise AssertionError("last layer must end in a terminal")

    def enumerate_accepted(self):
        stack = [(0, 0, ())]
        while stack:
            layer, node, prefix = stack.pop()
            for bit in (1, 0):
                t = int((self.ones if bit else self.zeros)[layer][node])
                if t == FALSE_T:
                    continue
                if t == TRUE_T:
                    yield prefix + (bit,)
                else:
                    stack.append((layer + 1, t, prefix + (bit,)))

    def count_accepting_paths(self) -> int:
        counts = None
        for layer in range(self.num_variables - 1, -1, -1):
            new = []
            for z, o in zip(self.zeros[layer], self.ones[layer]):
                c = 0
                for t in (int(z), int(o)):
                    c += 1 if t == TRUE_T else (counts[t] if t >= 0 else 0)
                new.append(c)
            counts = new
        return counts[0]


class FlatTable:
    """The FlatBdds arrays (kernels.py:35-92) of one instance, int64 host."""

    __slots__ = ("costs", "variable_order", "bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd",
                 "zero_t", "one_t", "proc_ptr", "proc_layers", "constraint_counts", "max_width",
                 "max_degree", "max_layers")

    @classmethod
    def from_native(cls, handle) -> "FlatTable":
        lib = _native.load()
        info = _native.InstanceInfo()
        _native.check(lib.dm_instance_get_info(handle, ctypes.byref(info)), "instance info")
        V, nb, L, N = info.num_variables, info.num_bdds, info.num_layers, info.num_nodes
        t = cls()
        t.costs = np.empty(V, np.float64)
        t.variable_order = np.empty(V, np.int64)
        t.bdd_layer_lo = np.empty(nb + 1, np.int64)
        t.layer_node_lo = np.empty(L + 1, np.int64)
        t.layer_var = np.empty(L, np.int64)
        t.layer_bdd = np.empty(L, np.int64)
        t.zero_t = np.empty(N, np.int64)
        t.one_t = np.empty(N, np.int64)
        t.proc_ptr = np.empty(V + 1, np.int64)
        t.proc_layers = np.empty(L, np.int64)
        t.constraint_counts = np.empty(V, np.int64)
        arrs = [t.costs, t.variable_order, t.bdd_layer_lo, t.layer_node_lo, t.layer_var, t.layer_bdd,
                t.zero_t, t.one_t, t.proc_ptr, t.proc_layers, t.constraint_counts]
        _native.check(lib.dm_instance_export(handle, *[a.ctypes.data for a in arrs]), "instance export")
        t.max_width, t.max_degree, t.max_layers = info.max_width, info.max_degree, info.max_layers
        return t

    @property
    def num_bdds(self) -> int:
        return len(self.bdd_layer_lo) - 1

    @property
    def num_layers(self) -> int:
        return len(self.layer_var)

    @property
    def num_nodes(self) -> int:
        return int(self.layer_node_lo[-1])


def _lower_rows(costs, row_ptr, row_var, row_coef, row_rhs, chunk_size: int) -> FlatTable:
    lib = _native.load()
    costs = np.ascontiguousarray(costs, dtype=np.float64)
    arrs = [np.ascontiguousarray(a, dtype=np.int64) for a in (row_ptr, row_var, row_coef, row_rhs)]
    h = ctypes.c_void_p()
    _native.check(lib.dm_instance_from_rows(len(costs), costs.ctypes.data, len(arrs[3]),
                                            *[a.ctypes.data for a in arrs], int(chunk_size),
                                            ctypes.byref(h)), "lower rows")
    try:
        return FlatTable.from_native(h)
    finally:
        lib.dm_instance_free(h)


def _lower_bdds(costs, bdds: Sequence, order, chunk_size: int) -> FlatTable:
    lib = _native.load()
    costs = np.ascontiguousarray(costs, dtype=np.float64)
    nb = len(bdds)
    per = np.array([len(b.variables) for b in bdds], np.int64)
    bdd_layer_lo = np.concatenate([[0], np.cumsum(per)]).astype(np.int64)
    layer_var = np.concatenate([np.asarray(b.variables, np.int64) for b in bdds]) if nb else np.zeros(0, np.int64)
    widths = np.array([len(z) for b in bdds for z in b.zeros], np.int64)
    layer_node_lo = np.concatenate([[0], np.cumsum(widths)]).astype(np.int64)
    zeros = np.concatenate([np.asarray(z, np.int32) for b in bdds for z in b.zeros]) if nb else np.zeros(0, np.int32)
    ones = np.concatenate([np.asarray(o, np.int32) for b in bdds for o in b.ones]) if nb else np.zeros(0, np.int32)
    order = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
    h = ctypes.c_void_p()
    _native.check(lib.dm_instance_from_bdds(
        len(costs), costs.ctypes.data, None if order is None else order.ctypes.data, nb,
        bdd_layer_lo.ctypes.data, layer_var.ctypes.data, layer_node_lo.ctypes.data,
        np.ascontiguousarray(zeros).ctypes.data, np.ascontiguousarray(ones).ctypes.data,
        int(chunk_size), ctypes.byref(h)), "lower diagrams")
    try:
        return FlatTable.from_native(h)
    finally:
        lib.dm_instance_free(h)


class IlpInstance:
    """Objective vector plus one diagram per constraint (ilp.py:30-87).

    Constructed either like the reference from ``Bdd`` objects, or (fast
    path) from a lowered ``FlatTable``.  ``variable_order`` is the
    visitation order of the averaging passes; every diagram lists its
    variables in that order.
    """

    def __init__(self, costs, constraints=None, rows=None, variable_order=None, *, flat: FlatTable | None = None):
        self.costs = np.asarray(costs, dtype=np.float64)
        if self.costs.ndim != 1:
            raise ValueError("costs must be a flat vector")
        self.rows = list(rows) if rows is not None else None
        self._bdds = list(constraints) if constraints is not None else None
        n = len(self.costs)
        if flat is not None:
            self._flat = flat
            self.variable_order = flat.variable_order
        else:
            if variable_order is None:
                variable_order = np.arange(n, dtype=np.int64)
            self.variable_order = np.asarray(variable_order, dtype=np.int64)
            if len(self.variable_order) != n or not np.array_equal(np.sort(self.variable_order), np.arange(n)):
                raise ValueError("variable_order must be a permutation of all variables")
            # validation + flattening in one native pass (no splitting)
            self._flat = _lower_bdds(self.costs, self._bdds or [], self.variable_order, 0)
        self.positions = np.empty(n, dtype=np.int64)
        self.positions[self.variable_order] = np.arange(n, dtype=np.int64)
        self.constraint_counts = self._flat.constraint_counts

    @property
    def flat(self) -> FlatTable:
        return self._flat

    @property
    def constraints(self) -> list[Bdd]:
        if self._bdds is None:
            f = self._flat
            out = []
            for j in range(f.num_bdds):
                l0, l1 = f.bdd_layer_lo[j], f.bdd_layer_lo[j + 1]
                zs, os_ = [], []
                for l in range(l0, l1):
                    a, b = f.layer_node_lo[l], f.layer_node_lo[l + 1]
                    nxt = f.layer_node_lo[l + 1]
                    z, o = f.zero_t[a:b], f.one_t[a:b]
                    zs.append(np.where(z >= 0, z - nxt, z).astype(np.int32))
                    os_.append(np.where(o >= 0, o - nxt, o).astype(np.int32))
                out.append(Bdd(f.layer_var[l0:l1], zs, os_))
            self._bdds = out
        return self._bdds

    @property
    def num_variables(self) -> int:
        return len(self.costs)

    @property
    def num_constraints(self) -> int:
        return self._flat.num_bdds

    def unconstrained_variables(self) -> np.ndarray:
        return np.flatnonzero(self.constraint_counts == 0)

    def __repr__(self) -> str:
        return f"IlpInstance({self.num_variables} vars, {self.num_constraints} constraints)"

    @classmethod
    def from_rows(cls, costs, rows: Sequence[LinearRow], chunk_size: int = 0) -> "IlpInstance":
        """Compile rows into diagrams (ilp.py:89-108); ``chunk_size > 0``
        also applies split_instance (splitting.py:116-155) in the same pass."""
        rows = list(rows)
        row_ptr = np.zeros(len(rows) + 1, np.int64)
        row_ptr[1:] = np.cumsum([len(r.variables) for r in rows])
        var = np.concatenate([np.asarray(r.variables, np.int64) for r in rows]) if rows else np.zeros(0, np.int64)
        coef = np.concatenate([np.asarray(r.coefficients, np.int64) for r in rows]) if rows else np.zeros(0, np.int64)
        rhs = np.array([int(r.rhs) for r in rows], np.int64)
        for r in rows:
            if len(r.variables) != len(r.coefficients):
                raise ValueError("one coefficient per variable required")
        inst = cls.from_csr(costs, row_ptr, var, coef, rhs, chunk_size)
        canon = []
        for r in rows:
            v = np.asarray(r.variables, np.int64)
            o = np.argsort(v, kind="stable")
            canon.append(LinearRow(v[o], np.asarray(r.coefficients, np.int64)[o], int(r.rhs), r.tag))
        inst.rows = canon
        return inst

    @classmethod
    def from_csr(cls, costs, row_ptr, row_var, row_coef, row_rhs, chunk_size: int = 0) -> "IlpInstance":
        """Rows given as CSR arrays (the product-space builder's output)."""
        costs = np.asarray(costs, dtype=np.float64)
        flat = _lower_rows(costs, row_ptr, row_var, row_coef, row_rhs, chunk_size)
        return cls(flat.costs, flat=flat)


def build_equality_bdd(coefficients, rhs, variables) -> Bdd:
    """bdd.py:478-501 through the native compiler."""
    coeffs = np.asarray(list(coefficients), dtype=np.int64)
    variables = list(variables)
    if len(coeffs) != len(variables):
        raise ValueError("one coefficient per variable required")
    if len(coeffs) == 0:
        raise ValueError("empty constraint row")
    # compile under the row's own order: ids are renamed to 0..k-1 in the
    # given sequence so the native stable sort keeps that order
    k = len(variables)
    flat = _lower_rows(np.zeros(k), [0, k], np.arange(k), coeffs, [int(rhs)], 0)
    inst = IlpInstance(flat.costs, flat=flat)
    b = inst.constraints[0]
    return Bdd(np.asarray(variables, np.int64), b.zeros, b.ones)


__all__ = ["Bdd", "FlatTable", "IlpInstance", "LinearRow", "make_row", "build_equality_bdd",
           "EmptyFeasibleSet", "FALSE_T", "TRUE_T"]
