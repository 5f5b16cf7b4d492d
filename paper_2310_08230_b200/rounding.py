"""Perturbation-based primal rounding on the GPU (north star: "perturbation-
based primal rounding"; the paper's full-instance primal heuristic is
FastDOG's, PAPER.md:282,5031-5043 — the reference package replaced it by
agreement fixing + an exact search, primal.py:380-429, which stays
available as primal.recover_primal).

Round r, on the current duals: fresh min-marginals (k_min_marginals), then
per variable the copies' votes give a direction — a unanimous strict vote,
else the sign of the summed differences, else a hashed coin — and its cost
moves by dir * delta_r * (1 + u) (u hashed in [0, 1); variables whose vote is
already unanimous move ``boost`` times further, which all but fixes them),
spread evenly over the
copies' duals (dm_perturb_round; feasibility for the perturbed costs is
kept).  A few averaging iterations then re-equilibrate the duals.  When
every constrained variable has a unanimous strict vote, each diagram's
unique optimum sets every variable to its voted value, so the voted
assignment satisfies every constraint: it is returned (after a host check of
every diagram) with its ORIGINAL cost and the gap to the unperturbed best
bound.  delta_r grows geometrically, so the loop terminates.

Deterministic for a given (seed, schedule, iteration counts): the hash is
splitmix64 on (seed, round, variable), and every kernel on the way is
bit-exact against the C oracle (tests/test_rounding.py restates the loop).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from .dual import BACKWARD, FORWARD, DualState, mma_pass
from .primal import GapReport, make_gap_report


@dataclass
class RoundingResult:
    status: str  # "certified" | "feasible" | "unrounded"
    assignment: np.ndarray | None
    objective: float | None
    report: GapReport | None
    rounds: int
    iterations: int
    seconds: float
    disagree_history: list


def diagrams_accept(flat, x: np.ndarray) -> np.ndarray:
    """Per diagram, whether it accepts the assignment ``x`` (by variable id):
    all diagrams walked in lock step, one layer at a time (host check)."""
    bl = flat.bdd_layer_lo
    nb = flat.num_bdds
    node = flat.layer_node_lo[bl[:-1]].copy()
    ok = np.ones(nb, bool)
    nl = np.diff(bl)
    for k in range(int(nl.max()) if nb else 0):
        act = np.flatnonzero(ok & (k < nl))
        if not len(act):
            break
        layer = bl[act] + k
        bit = x[flat.layer_var[layer]]
        tgt = np.where(bit == 1, flat.one_t[node[act]], flat.zero_t[node[act]])
        last = k + 1 == nl[act]
        ok[act[(tgt == -1) | (last & (tgt != -2)) | (~last & (tgt < 0))]] = False
        node[act] = np.where(tgt >= 0, tgt, node[act])
    return ok


def perturbation_rounding(state: DualState, seed: int = 0, max_rounds: int = 80, iterations_per_round: int = 3,
                          delta0: float | None = None, growth: float = 1.2, boost: float = 10.0, damping: float = 0.5,
                          clock=time.perf_counter) -> RoundingResult:
    """Round the solved duals of ``state`` to a feasible assignment (the state's
    duals end perturbed; its instance and best bound are untouched)."""
    t0 = clock()
    inst = state.instance
    best_bound = state.best_bound
    costs = inst.costs
    nv = inst.num_variables
    if delta0 is None:
        nz = np.abs(costs[costs != 0])
        delta0 = 1e-3 * float(np.median(nz)) if len(nz) else 1e-3
    dev = state.device
    values = torch.zeros(nv, dtype=torch.int8, device=dev)
    agrees = torch.zeros(nv, dtype=torch.int8, device=dev)
    disagree = torch.zeros(1, dtype=torch.int32, device=dev)
    history, iters = [], 0
    x = None
    r = 0
    for r in range(max_rounds):
        m0, m1 = state.min_marginal_table_device()
        state.dev.perturb_round(m0, m1, state.lam_d, delta0 * growth ** r, boost, seed, r, values, agrees, disagree)
        n_dis = int(disagree.item())
        history.append(n_dis)
        state.f_valid = state.b_valid = False  # duals moved
        if n_dis == 0:
            x = values.cpu().numpy().astype(np.int8)
            break
        for _ in range(iterations_per_round):
            if state.deferred:
                state.deferred_round(damping)
            else:
                mma_pass(state, FORWARD)
                mma_pass(state, BACKWARD)
            iters += 1
    free = inst.unconstrained_variables()
    if x is None:
        return RoundingResult("unrounded", None, None, None, r + 1, iters, clock() - t0, history)
    x[free] = (costs[free] < 0).astype(np.int8)
    if not diagrams_accept(inst.flat, x).all():  # cannot happen for strict unanimous votes; checked anyway
        return RoundingResult("unrounded", None, None, None, r + 1, iters, clock() - t0, history)
    obj = float(costs @ x)
    rep = make_gap_report(obj, best_bound)
    return RoundingResult("certified" if rep.certified else "feasible", x, obj, rep, r + 1, iters, clock() - t0,
                          history)
