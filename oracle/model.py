"""ORACLE — TEST INFRASTRUCTURE ONLY.

Restatement of the reference's instance pipeline:
rows -> equality diagrams (bdd.py:478-501, ilp.py:89-108) -> optional
chunk splitting (splitting.py:35-155) -> flat node table (kernels.py:35-92).

Diagrams are plain tuples ``(variables, zeros, ones)``: ``zeros[l]`` and
``ones[l]`` are int32 arrays of local next-layer indices with sentinels
-1 (FALSE) and -2 (TRUE), exactly the reference's ``Bdd`` fields.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from .clib import lib, ptr

FALSE_T = -1
TRUE_T = -2


class OracleInfeasibleRow(Exception):
    """A row has no 0-1 solution (reference: EmptyFeasibleSet, bdd.py:493-494)."""


def equality_bdd(coeffs, rhs, variables):
    """bdd.py:478-501 via the C restatement of _equality_tables."""
    c = np.ascontiguousarray(np.asarray(list(coeffs), dtype=np.int64))
    n = len(c)
    if n == 0:
        raise ValueError("empty constraint row")
    widths = np.zeros(n, dtype=np.int64)
    total = lib.oracle_equality_tables(n, ptr(c), int(rhs), ptr(widths), None, None)
    if total == 0:
        raise OracleInfeasibleRow(f"no 0-1 solution of row == {rhs}")
    z = np.empty(total, np.int32)
    o = np.empty(total, np.int32)
    lib.oracle_equality_tables(n, ptr(c), int(rhs), ptr(widths), ptr(z), ptr(o))
    zeros, ones, pos = [], [], 0
    for w in widths:
        zeros.append(z[pos : pos + w])
        ones.append(o[pos : pos + w])
        pos += int(w)
    return (np.asarray(list(variables), dtype=np.int64), zeros, ones)


def split_bdd(bdd, cut, fresh):
    """splitting.py:35-96: cut after ``cut`` layers, one-hot coupling."""
    variables, zeros, ones = bdd
    n = len(variables)
    if not 1 <= cut < n:
        raise ValueError("split index outside the interior")
    k = len(zeros[cut])
    aux = [next(fresh) for _ in range(k)]
    lz = [a.copy() for a in zeros[:cut]]
    lo = [a.copy() for a in ones[:cut]]
    # left tail: layer q tracks the k-q crossing nodes whose bit is still
    # pending (slot t-q), plus one "already chose" slot once q > 0.
    for q in range(k):
        pend = k - q
        z = np.full(pend + (q > 0), FALSE_T, np.int32)
        o = np.full(pend + (q > 0), FALSE_T, np.int32)
        final = q == k - 1
        o[0] = TRUE_T if final else pend - 1
        if not final:
            z[1:pend] = np.arange(0, pend - 1, dtype=np.int32)
        if q > 0:
            z[pend] = TRUE_T if final else pend - 1
        lz.append(z)
        lo.append(o)
    left = (np.concatenate([variables[:cut], np.asarray(aux, np.int64)]), lz, lo)
    # right head: slot 0 = nothing placed yet, slot t+1 = bit placed at t.
    rz, ro = [], []
    for q in range(k):
        z = np.full(q + 1, FALSE_T, np.int32)
        o = np.full(q + 1, FALSE_T, np.int32)
        final = q == k - 1
        o[0] = q if final else q + 1
        if not final:
            z[0] = 0
        if q:
            t = np.arange(q, dtype=np.int32)
            z[1:] = t if final else t + 1
        rz.append(z)
        ro.append(o)
    rz += [a.copy() for a in zeros[cut:]]
    ro += [a.copy() for a in ones[cut:]]
    right = (np.concatenate([np.asarray(aux, np.int64), variables[cut:]]), rz, ro)
    return left, right, aux


@dataclass
class OracleInstance:
    costs: np.ndarray
    bdds: list
    order: np.ndarray  # visitation order (ilp.py:42-71)

    @property
    def num_variables(self) -> int:
        return len(self.costs)

    def positions(self) -> np.ndarray:
        pos = np.empty(len(self.order), np.int64)
        pos[self.order] = np.arange(len(self.order))
        return pos

    def counts(self) -> np.ndarray:
        if self.bdds is None:  # built from a flat table (see from_flat_table)
            return self._counts
        cnt = np.zeros(self.num_variables, np.int64)
        for v, _, _ in self.bdds:
            cnt[v] += 1
        return cnt


def instance_from_rows(costs, rows):
    """ilp.py:89-108: canonicalise each row (stable sort by id), compile it."""
    bdds = []
    for variables, coeffs, rhs in rows:
        variables = np.asarray(variables, np.int64)
        coeffs = np.asarray(coeffs, np.int64)
        perm = np.argsort(variables, kind="stable")
        bdds.append(equality_bdd(coeffs[perm], int(rhs), variables[perm]))
    costs = np.asarray(costs, np.float64)
    return OracleInstance(costs, bdds, np.arange(len(costs), dtype=np.int64))


def split_instance(inst: OracleInstance, chunk: int = 128) -> OracleInstance:
    """splitting.py:99-155: cut every ``chunk`` original layers."""
    if chunk < 2:
        raise ValueError("chunk_size must be at least 2")
    if not any(len(b[0]) > chunk for b in inst.bdds):
        return inst
    fresh = itertools.count(inst.num_variables)
    after = {}
    out = []
    for bdd in inst.bdds:
        n = len(bdd[0])
        if n <= chunk:
            out.append(bdd)
            continue
        rest, prev, carried = bdd, 0, 0
        for cut in range(chunk, n, chunk):
            left, rest, aux = split_bdd(rest, carried + cut - prev, fresh)
            after.setdefault(int(bdd[0][cut - 1]), []).extend(aux)
            out.append(left)
            carried, prev = len(aux), cut
        out.append(rest)
    n_aux = next(fresh) - inst.num_variables
    order = []
    for v in inst.order.tolist():
        order.append(v)
        order.extend(after.get(v, ()))
    return OracleInstance(
        np.concatenate([inst.costs, np.zeros(n_aux)]), out, np.asarray(order, np.int64)
    )


@dataclass
class OracleFlat:
    """kernels.py:35-92 FlatBdds, int64 arrays."""

    bdd_layer_lo: np.ndarray
    layer_node_lo: np.ndarray
    layer_var: np.ndarray
    layer_bdd: np.ndarray
    zero_t: np.ndarray
    one_t: np.ndarray
    proc_ptr: np.ndarray
    proc_layers: np.ndarray
    max_degree: int

    @property
    def num_bdds(self):
        return len(self.bdd_layer_lo) - 1

    @property
    def num_layers(self):
        return len(self.layer_var)

    @property
    def num_nodes(self):
        return int(self.layer_node_lo[-1])


def flatten(inst: OracleInstance) -> OracleFlat:
    nl_per = np.array([len(b[0]) for b in inst.bdds], np.int64)
    bdd_layer_lo = np.concatenate([[0], np.cumsum(nl_per)]).astype(np.int64)
    widths = np.array([len(z) for b in inst.bdds for z in b[1]], np.int64)
    layer_node_lo = np.concatenate([[0], np.cumsum(widths)]).astype(np.int64)
    L = int(bdd_layer_lo[-1])
    layer_var = (
        np.concatenate([b[0] for b in inst.bdds]).astype(np.int64) if L else np.zeros(0, np.int64)
    )
    layer_bdd = np.repeat(np.arange(len(inst.bdds), dtype=np.int64), nl_per)
    zl = np.concatenate([z for b in inst.bdds for z in b[1]]).astype(np.int64) if L else np.zeros(0, np.int64)
    ol = np.concatenate([o for b in inst.bdds for o in b[2]]).astype(np.int64) if L else np.zeros(0, np.int64)
    base = np.repeat(layer_node_lo[1:], widths)  # start of the next layer
    zero_t = np.where(zl >= 0, zl + base, zl)
    one_t = np.where(ol >= 0, ol + base, ol)
    pos = inst.positions()[layer_var]
    proc_layers = np.argsort(pos, kind="stable").astype(np.int64)
    cnt = np.bincount(pos, minlength=inst.num_variables)
    proc_ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    return OracleFlat(
        bdd_layer_lo, layer_node_lo, layer_var, layer_bdd, zero_t, one_t, proc_ptr,
        proc_layers, int(cnt.max()) if len(cnt) else 0,
    )


def from_flat_table(costs, order, counts, arrays: dict):
    """Wrap an already-lowered flat table (int64 arrays keyed like FlatBdds)
    so the oracle kernels can run on it; used for full-size checks where
    the Python diagram builder would be slow.  Parity of the lowering itself
    is established separately against the reference's golden hashes."""
    inst = OracleInstance(np.asarray(costs, np.float64), None, np.asarray(order, np.int64))
    inst._counts = np.asarray(counts, np.int64)
    a = {k: np.ascontiguousarray(arrays[k], dtype=np.int64) for k in (
        "bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd", "zero_t", "one_t", "proc_ptr", "proc_layers")}
    deg = int(np.diff(a["proc_ptr"]).max()) if len(a["proc_ptr"]) > 1 else 0
    return inst, OracleFlat(max_degree=deg, **a)
