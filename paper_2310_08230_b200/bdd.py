"""Per-diagram operations of the reference's ``prodmatch.bdd`` module
(bdd.py:24-359): distances, cheapest assignment, min-marginals, conditioning,
reduction and the structural check — the API a caller uses on single
``Bdd`` objects.  The solver never runs these (its kernels work on the flat
table in HBM); they exist so code written against ``prodmatch.bdd`` runs
unchanged, and the reference's own tests (pkg/tests/test_bdd.py,
test_split.py) pass against this package by import alias
(tests/test_reference_api.py).

Semantics follow the reference (distances with the zero arc free and the one
arc costing ``costs[layer]``; ties to the zero arc; first-occurrence node
order in reductions); the implementation is written over whole layers with
numpy.  The equality-row compiler is the native one (ilp.build_equality_bdd).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from .errors import EmptyFeasibleSet
from .ilp import Bdd, build_equality_bdd

FALSE_T = -1  # bdd.py:24
TRUE_T = -2  # bdd.py:25
ArcCosts = Sequence[float]  # one-arc cost per layer

__all__ = ["FALSE_T", "TRUE_T", "ArcCosts", "MinMarginalPair", "Bdd", "build_equality_bdd", "reduce_bdd",
           "check_structure"]


@dataclass(frozen=True)
class MinMarginalPair:
    """Best accepted-path cost with the layer's variable clamped to 0 / 1
    (bdd.py:33-52); a side without any accepting path is inf."""

    m0: float
    m1: float

    @property
    def difference(self) -> float:
        """m1 - m0, with a clamped side kept symbolic (+-inf, never inf - inf)."""
        inf0, inf1 = np.isinf(self.m0), np.isinf(self.m1)
        if inf0 and inf1:
            raise ValueError("min-marginal pair with no feasible branch")
        if inf1:
            return np.inf
        if inf0:
            return -np.inf
        return self.m1 - self.m0


def _follow(targets: np.ndarray, below: np.ndarray | None) -> np.ndarray:
    """Value of taking each arc in ``targets``: the next layer's value at a
    node target, 0 at TRUE, inf at FALSE."""
    out = np.where(targets == TRUE_T, 0.0, np.inf)
    if below is not None:
        inner = targets >= 0
        out[inner] = below[targets[inner]]
    return out


def backward_distances(bdd: Bdd, costs: ArcCosts) -> list:
    """Least cost from each node to TRUE, [layer][node] (bdd.py:131-142)."""
    c = np.asarray(costs, dtype=np.float64)
    out = [None] * bdd.num_variables
    below = None
    for layer in reversed(range(bdd.num_variables)):
        below = np.minimum(_follow(bdd.zeros[layer], below), c[layer] + _follow(bdd.ones[layer], below))
        out[layer] = below
    return out


def forward_distances(bdd: Bdd, costs: ArcCosts) -> tuple[list, float]:
    """Least cost from the root to each node, and to TRUE (bdd.py:144-164)."""
    c = np.asarray(costs, dtype=np.float64)
    n = bdd.num_variables
    dist = [np.zeros(1)]
    to_true = np.inf
    for layer in range(n):
        here = dist[layer]
        nxt = np.full(len(bdd.zeros[layer + 1]), np.inf) if layer + 1 < n else None
        for arcs, value in ((bdd.zeros[layer], here), (bdd.ones[layer], here + c[layer])):
            if nxt is not None:
                inner = arcs >= 0
                np.minimum.at(nxt, arcs[inner], value[inner])
            hit = arcs == TRUE_T
            if hit.any():
                to_true = min(to_true, float(value[hit].min()))
        if nxt is not None:
            dist.append(nxt)
    return dist, to_true


def min_assignment(bdd: Bdd, costs: ArcCosts) -> tuple[float, tuple]:
    """Cheapest accepted assignment; ties take the zero arc (bdd.py:166-189)."""
    c = np.asarray(costs, dtype=np.float64)
    back = backward_distances(bdd, c)
    n = bdd.num_variables
    node, bits = 0, []
    for layer in range(n):
        below = back[layer + 1] if layer + 1 < n else None
        z = int(bdd.zeros[layer][node])
        o = int(bdd.ones[layer][node])
        cz = float(_follow(np.array([z]), below)[0])
        co = c[layer] + float(_follow(np.array([o]), below)[0])
        take_one = not cz <= co
        bits.append(int(take_one))
        node = o if take_one else z
    return float(back[0][0]), tuple(bits)


def min_marginals(bdd: Bdd, costs: ArcCosts) -> list:
    """Per layer, (m0, m1) from one forward and one backward sweep (bdd.py:191-207)."""
    c = np.asarray(costs, dtype=np.float64)
    fwd, _ = forward_distances(bdd, c)
    back = backward_distances(bdd, c)
    n = bdd.num_variables
    out = []
    for layer in range(n):
        below = back[layer + 1] if layer + 1 < n else None
        m0 = (fwd[layer] + _follow(bdd.zeros[layer], below)).min()
        m1 = (fwd[layer] + c[layer] + _follow(bdd.ones[layer], below)).min()
        out.append(MinMarginalPair(float(m0), float(m1)))
    return out


def condition(bdd: Bdd, fixes: Mapping[int, int]) -> Bdd:
    """Clamp this diagram's fixed variables (the layer stays, its other arc
    goes to FALSE) and re-reduce; the same object when no fix applies
    (bdd.py:243-264)."""
    layer_of = {int(v): i for i, v in enumerate(bdd.variables)}
    hits = [(layer_of[int(v)], int(b)) for v, b in fixes.items() if int(v) in layer_of]
    if not hits:
        return bdd
    zeros = [z.copy() for z in bdd.zeros]
    ones = [o.copy() for o in bdd.ones]
    for layer, bit in hits:
        (zeros if bit else ones)[layer][:] = FALSE_T
    return reduce_bdd(Bdd(bdd.variables, zeros, ones))


def is_constant_true(bdd: Bdd) -> bool:
    """Every assignment accepted: each layer one node whose two arcs agree and
    are not FALSE (bdd.py:266-275)."""
    for z, o in zip(bdd.zeros, bdd.ones):
        if len(z) != 1 or int(z[0]) != int(o[0]) or int(z[0]) == FALSE_T:
            return False
    return True


def reduce_bdd(bdd: Bdd) -> Bdd:
    """Drop nodes that cannot reach TRUE or be reached from the root, then
    merge nodes with identical arcs, keeping first occurrences in layer order
    (reducing a reduced diagram is the identity; bdd.py:278-333).  Raises
    EmptyFeasibleSet when the root cannot reach TRUE."""
    n = bdd.num_variables
    zeros = [z.astype(np.int64) for z in bdd.zeros]
    ones = [o.astype(np.int64) for o in bdd.ones]
    live = [None] * n
    for layer in reversed(range(n)):  # co-reachability; arcs into dead nodes -> FALSE
        for arcs in (zeros[layer], ones[layer]):
            if layer + 1 < n:
                inner = np.flatnonzero(arcs >= 0)
                arcs[inner[~live[layer + 1][arcs[inner]]]] = FALSE_T
        live[layer] = (zeros[layer] != FALSE_T) | (ones[layer] != FALSE_T)
    if not live[0][0]:
        raise EmptyFeasibleSet("constraint has no accepting assignment")
    seen = [np.ones(1, bool)]
    for layer in range(n - 1):  # reachability over the surviving arcs
        nxt = np.zeros(len(zeros[layer + 1]), bool)
        for arcs in (zeros[layer], ones[layer]):
            nxt[arcs[seen[layer] & (arcs >= 0)]] = True
        seen.append(nxt)
    new_z, new_o = [None] * n, [None] * n
    rename = None  # next layer: old node id -> new id (FALSE_T when dropped)
    for layer in reversed(range(n)):
        keep = np.flatnonzero(live[layer] & seen[layer])
        pairs = {}
        ids = np.full(len(zeros[layer]), FALSE_T, np.int64)
        zl, ol = [], []
        for v in keep:
            z, o = int(zeros[layer][v]), int(ones[layer][v])
            if rename is not None:
                z = int(rename[z]) if z >= 0 else z
                o = int(rename[o]) if o >= 0 else o
            new = pairs.setdefault((z, o), len(zl))
            if new == len(zl):
                zl.append(z)
                ol.append(o)
            ids[v] = new
        new_z[layer] = np.asarray(zl, np.int32)
        new_o[layer] = np.asarray(ol, np.int32)
        rename = ids
    return Bdd(bdd.variables, new_z, new_o)


def check_structure(bdd: Bdd) -> None:
    """Raise ValueError unless the diagram is layered (inner arcs only into
    the next layer, terminals only from the last), reduced and free of dead
    or unreachable nodes (bdd.py:336-359)."""
    n = bdd.num_variables
    if len(bdd.zeros[0]) != 1:
        raise ValueError("root layer width must be 1")
    for layer in range(n):
        below = len(bdd.zeros[layer + 1]) if layer + 1 < n else 0
        for arcs in (bdd.zeros[layer], bdd.ones[layer]):
            if len(arcs) and int(arcs.min()) < TRUE_T:
                raise ValueError("arc target below sentinel range")
            if layer + 1 < n and (arcs == TRUE_T).any():
                raise ValueError("inner arc to TRUE (skip arcs are forbidden)")
            if layer + 1 < n and len(arcs) and int(arcs.max()) >= below:
                raise ValueError("arc target beyond next layer")
            if layer + 1 == n and (arcs >= 0).any():
                raise ValueError("last layer must target terminals only")
        pairs = set(zip(bdd.zeros[layer].tolist(), bdd.ones[layer].tolist()))
        if len(pairs) != len(bdd.zeros[layer]):
            raise ValueError(f"layer {layer} holds isomorphic nodes (not reduced)")
    if reduce_bdd(bdd).widths != bdd.widths:
        raise ValueError("diagram contains dead or unreachable nodes")


# the reference's Bdd methods (bdd.py:131-275) on this package's Bdd
Bdd.backward_distances = backward_distances
Bdd.forward_distances = forward_distances
Bdd.min_assignment = min_assignment
Bdd.min_marginals = min_marginals
Bdd.condition = condition
Bdd.is_constant_true = is_constant_true
