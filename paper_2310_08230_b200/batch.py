"""Independent instances solved as ONE merged instance (BASELINE config C5:
a batch of 64 independent ~500-triangle pairs).

No reference counterpart (the reference solves one instance per call,
qn.py:211-259).  The batch's flat tables are concatenated block-diagonally
(variables, diagrams, layers and nodes offset; visitation orders appended),
so one upload, one set of plans and one launch per kernel serve every
instance: the exact passes' persistent grid walks the interleaved DAG levels
of all instances at once (depth = the deepest instance, not the sum), the
sweeps and vector kernels see one long vector.  Diagrams of different
instances never share a variable, so every averaging pass acts on each
instance exactly as on its own — in mode "mma-only" the per-instance duals
after n iterations are bit-identical to n-iteration solves of the instances
one by one (tests/test_batch.py); the batch stops when every instance's own
stopping rule has fired.  In hybrid mode the L-BFGS direction and step size
are those of the merged dual (one quasi-Newton step for the whole block-
diagonal problem), so per-instance trajectories differ from separate solves
(every instance's duals stay feasible and its bound valid; parity at
convergence, tests/test_batch.py) and the coupled step converges more
slowly than separate solves — the C5 bench line uses averaging-only batches.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from .config import SolveConfig
from .ilp import FlatTable, IlpInstance

_FIELDS = ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd", "zero_t", "one_t", "proc_ptr", "proc_layers")


@dataclass
class BatchIndex:
    """Offsets of each instance in the merged arrays (length n + 1 each)."""

    var: np.ndarray
    bdd: np.ndarray
    layer: np.ndarray
    node: np.ndarray

    def __len__(self) -> int:
        return len(self.var) - 1


_REUSE: dict = {}  # (V, nb, L, N) -> the FlatTable last merged with reuse_buffers


def merge_instances(instances, threads: int = 8, reuse_buffers: bool = False) -> tuple[IlpInstance, BatchIndex]:
    """Block-diagonal concatenation of lowered instances (their FlatTables):
    outputs preallocated, each instance's slices filled by a worker thread
    (numpy releases the GIL on these copies).  ``reuse_buffers`` refills the
    host arrays of the previous merge of the same sizes instead of faulting
    in gigabytes of fresh pages (the previous merged instance is then
    overwritten: a serving loop's staging arena)."""
    from concurrent.futures import ThreadPoolExecutor

    flats = [i.flat for i in instances]
    if not flats:
        raise ValueError("empty batch")
    off = lambda xs: np.concatenate([[0], np.cumsum(xs)]).astype(np.int64)  # noqa: E731
    vo = off([len(i.costs) for i in instances])
    bo = off([f.num_bdds for f in flats])
    lo = off([f.num_layers for f in flats])
    no = off([f.num_nodes for f in flats])
    V, nb, L, N = int(vo[-1]), int(bo[-1]), int(lo[-1]), int(no[-1])
    if reuse_buffers and (V, nb, L, N) in _REUSE:
        t = _REUSE[(V, nb, L, N)]
    else:
        t = _new_table(V, nb, L, N)
        if reuse_buffers:
            _REUSE.clear()
            _REUSE[(V, nb, L, N)] = t
    t.bdd_layer_lo[nb] = L
    t.layer_node_lo[L] = N
    t.proc_ptr[V] = L

    def shifted(dst, src, by, nodes=False):
        np.copyto(dst, src)
        if by:
            if nodes:  # node targets move, the terminal sentinels (-1, -2) stay
                np.add(dst, by, out=dst, where=src >= 0)
            else:
                dst += by

    def fill(k):
        i, f = instances[k], flats[k]
        v0, v1, b0, b1 = vo[k], vo[k + 1], bo[k], bo[k + 1]
        l0, l1, n0, n1 = lo[k], lo[k + 1], no[k], no[k + 1]
        t.costs[v0:v1] = i.costs
        shifted(t.variable_order[v0:v1], i.variable_order, v0)
        t.constraint_counts[v0:v1] = f.constraint_counts
        shifted(t.bdd_layer_lo[b0:b1], f.bdd_layer_lo[:-1], l0)
        shifted(t.layer_node_lo[l0:l1], f.layer_node_lo[:-1], n0)
        shifted(t.layer_var[l0:l1], f.layer_var, v0)
        shifted(t.layer_bdd[l0:l1], f.layer_bdd, b0)
        shifted(t.zero_t[n0:n1], f.zero_t, n0, nodes=True)
        shifted(t.one_t[n0:n1], f.one_t, n0, nodes=True)
        # visitation positions appended instance after instance (copies stay in ascending layer order)
        shifted(t.proc_ptr[v0:v1], f.proc_ptr[:-1], l0)
        shifted(t.proc_layers[l0:l1], f.proc_layers, l0)

    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(fill, range(len(instances))))
    t.max_width = max(int(f.max_width) for f in flats)
    t.max_degree = max(int(f.max_degree) for f in flats)
    t.max_layers = max(int(f.max_layers) for f in flats)
    return IlpInstance(t.costs, flat=t), BatchIndex(vo, bo, lo, no)


def _new_table(V, nb, L, N) -> FlatTable:
    t = FlatTable()
    t.costs = np.empty(V)
    t.variable_order = np.empty(V, np.int64)
    t.constraint_counts = np.empty(V, np.int64)
    t.bdd_layer_lo = np.empty(nb + 1, np.int64)
    t.layer_node_lo = np.empty(L + 1, np.int64)
    t.layer_var = np.empty(L, np.int64)
    t.layer_bdd = np.empty(L, np.int64)
    t.zero_t = np.empty(N, np.int64)
    t.one_t = np.empty(N, np.int64)
    t.proc_ptr = np.empty(V + 1, np.int64)
    t.proc_layers = np.empty(L, np.int64)
    return t


@dataclass
class BatchResult:
    merged: object  # qn.SolveResult of the merged instance
    index: BatchIndex
    bounds: list  # per instance: bound of its final duals (its diagrams' optima, numpy order, + free part)
    iterations: int
    seconds: float

    def lam(self, k: int) -> np.ndarray:
        """Final duals of instance k (host copy)."""
        i = self.index
        return self.merged.state.lam[i.layer[k]:i.layer[k + 1]]


def instance_bounds(state, index: BatchIndex, instances) -> list:
    """Per-instance bound of the merged state's current duals: each
    instance's diagram optima summed in numpy's order (dual.py:66-69) plus
    its unconstrained variables' part."""
    F, B = state.node_tables(need_f=False)
    del F
    opt = torch.empty(state.flat.num_bdds, dtype=torch.float64, device=state.device)
    # per-diagram optimum = B at its root (kernels.py:359-361 / 104-120)
    roots = torch.as_tensor(state.flat.layer_node_lo[state.flat.bdd_layer_lo[:-1]], device=state.device)
    opt.copy_(B[roots])
    host = opt.cpu().numpy()
    out = []
    for k, inst in enumerate(instances):
        free = inst.unconstrained_variables()
        fc = float(np.minimum(inst.costs[free], 0.0).sum()) if len(free) else 0.0
        out.append(float(np.sum(host[index.bdd[k]:index.bdd[k + 1]])) + fc)
    return out


def solve_merged(instances, cfg: SolveConfig | None = None, device=None, clock=time.perf_counter,
                 per_instance_stop: bool = True, reuse_buffers: bool = False) -> BatchResult:
    """Solve a batch of independent instances as one merged instance (from
    their lowered host tables: merge, upload, plans and solve all timed).

    ``per_instance_stop`` (averaging-only mode): the batch runs until EVERY
    instance's own stopping rule (bound gain below dual_tolerance, qn.py:252)
    has fired once, each instance's bound taken from the device per-diagram
    optima after every iteration; instances that stopped earlier keep being
    averaged (monotone) — their duals equal a separate solve run to the
    batch's iteration count.  Otherwise (and always in hybrid mode) the
    merged instance's own stopping rule applies."""
    from .dual import init_duals
    from .qn import DualSolver

    instances = list(instances)
    cfg = cfg or SolveConfig()
    t0 = clock()
    merged, index = merge_instances(instances, reuse_buffers=reuse_buffers)
    state = init_duals(merged, device=device, schedule=cfg.mma_schedule)
    if not per_instance_stop or cfg.mode != "mma-only":
        from .qn import solve

        res = solve(merged, cfg, device=device, state=state, clock=clock)
        bounds = instance_bounds(res.state, index, instances)
        return BatchResult(res, index, bounds, res.iterations, clock() - t0)
    run = DualSolver(merged, cfg, clock=clock, device=device, state=state).start()
    ends = torch.as_tensor(index.bdd[1:] - 1, device=state.device)
    fcs = torch.as_tensor([float(np.minimum(i.costs[i.unconstrained_variables()], 0.0).sum()) for i in instances],
                          dtype=torch.float64, device=state.device)
    n = len(instances)

    def per_instance():  # deterministic segment sums (an inclusive scan, differenced)
        c = torch.cumsum(state._bounds, 0)[ends]
        return torch.cat([c[:1], c[1:] - c[:-1]]) + fcs

    prev = per_instance()
    stopped = torch.zeros(n, dtype=torch.bool, device=state.device)
    reason = "max_iterations"
    for _ in range(cfg.max_iterations):
        run.step()
        cur = per_instance()
        stopped |= (cur - prev) < cfg.dual_tolerance * torch.clamp(cur.abs(), min=1.0)
        prev = cur
        if bool(stopped.all()):
            reason = "dual_tolerance"
            break
        if cfg.max_seconds is not None and clock() - t0 > cfg.max_seconds:
            reason = "max_seconds"
            break
    res = run.result(reason)
    bounds = instance_bounds(res.state, index, instances)
    return BatchResult(res, index, bounds, res.iterations, clock() - t0)
