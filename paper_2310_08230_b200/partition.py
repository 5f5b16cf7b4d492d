"""One instance split over several GPUs (BASELINE config C4: "BDDs partitioned
across 1/2/4/8 B200 with NCCL marginal allreduce").

No reference counterpart: the reference is single-process;
the plan is SURVEY.md §5(b).  The diagrams are cut into k compact blocks
(slabs of a breadth-first diagram order, balanced by node count); each rank
owns its block's diagrams, their nodes,
duals and distance tables, and runs the DEFERRED averaging schedule
(dm_deferred.cu) on them — within a pass every diagram is independent, so
the only data-plane exchange is, per pass, the escrow of the variables whose
copies span ranks: one allreduce-sum over a packed buffer with one slot per
boundary copy, in global copy order (each slot has exactly one writer, so
the sum is exact), plus an all-gather of the per-diagram optima for the
bound.  Averages of boundary variables are then taken from the buffer with
the same arithmetic as dm_dfr_average, so a k-rank solve is bit-identical
to the one-GPU ``qn.solve(..., SolveConfig(mode="mma-only",
mma_schedule="deferred"))`` (tests/test_partition.py: world size 2 over gloo
on the CPU, and k logical partitions on one GPU).

Scope: averaging-only solves (mode "mma-only") — the north star's "NCCL
allreducing only the min-marginal sums of variables that span partitions".
The hybrid (L-BFGS) mode would add global inner products per two-loop step
and a bound exchange per step-search trial; it is not partitioned.

Roles:
  * ``plan_partition`` — host plan: diagram cut points, the per-rank local
    FlatBdds tables (global ids renumbered), local-only visitation CSRs and
    the boundary slot layout (identical on every rank);
  * ``DeviceEngine`` — one rank's device state and kernels (C-ABI);
  * ``Comm`` implementations — ``DistComm`` (torch.distributed: NCCL on
    GPUs, gloo on CPUs, one part per process) and ``LoopbackComm`` (all parts
    in one process: logical partitions on one GPU);
  * ``PartitionedSolver`` — the solve loop over the parts a process owns.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from .config import SolveConfig
from .ilp import FlatTable, IlpInstance

_F64 = torch.float64


# --------------------------------------------------------------------------- host plan
@dataclass
class PartPlan:
    """What one rank owns and how its boundary copies map into the buffer."""

    rank: int
    bdds: np.ndarray  # global ids of the diagrams this rank owns (ascending)
    layers: np.ndarray  # global ids of their layers (local layer i = global layers[i])
    table: FlatTable  # local FlatBdds arrays (local diagram / layer / node ids, global variable ids)
    local_ptr: np.ndarray  # visitation CSR of the variables whose copies are all on this rank (int32)
    local_layers: np.ndarray
    b_layer: np.ndarray  # boundary copies on this rank: local layer, slot, and their variable's slot range
    b_slot: np.ndarray
    b_lo: np.ndarray
    b_hi: np.ndarray
    lam0: np.ndarray  # initial duals of the local layers (dual.py:137-144, global counts)


@dataclass
class PartitionPlan:
    k: int
    parts: list
    bdd_order: np.ndarray  # the parts' diagrams concatenated in rank order (global ids)
    slots: int  # boundary exchange buffer length (copies of boundary variables)
    boundary_variables: int
    variables_with_copies: int
    free_contribution: float

    @property
    def boundary_fraction(self) -> float:
        return self.boundary_variables / max(self.variables_with_copies, 1)


def _diagram_graph(flat):
    """CSR of diagram -> diagrams sharing a variable with it (through the
    visitation CSR), as (ptr, nbr) int64 arrays; duplicates kept."""
    ptr, pl = flat.proc_ptr, flat.proc_layers
    cnt = np.diff(ptr)
    pos = np.repeat(np.arange(len(cnt)), cnt)
    bdd_of_copy = flat.layer_bdd[pl]
    # every ordered pair of copies of one variable (degrees are small: <= 32)
    src, dst = [], []
    for d in range(1, int(cnt.max()) if len(cnt) else 1):
        ok = np.flatnonzero((np.arange(len(pl)) - ptr[pos] + d) < cnt[pos])
        src.append(bdd_of_copy[ok])
        dst.append(bdd_of_copy[ok + d])
    src = np.concatenate(src + [np.zeros(0, np.int64)])
    dst = np.concatenate(dst + [np.zeros(0, np.int64)])
    u = np.concatenate([src, dst])
    v = np.concatenate([dst, src])
    order = np.argsort(u, kind="stable")
    nb = flat.num_bdds
    gptr = np.zeros(nb + 1, np.int64)
    np.add.at(gptr, u + 1, 1)
    return np.cumsum(gptr), v[order]


def diagram_order(flat) -> np.ndarray:
    """Breadth-first order of the diagram graph (diagrams adjacent when they
    share a variable) from a far corner: consecutive runs of it are compact
    regions of the instance, so cutting it into k slabs leaves few variables
    with copies on two sides (a bandwidth-reducing, Cuthill-McKee-like order;
    every component is walked in turn)."""
    nb = flat.num_bdds
    gptr, nbr = _diagram_graph(flat)
    seen = np.zeros(nb, bool)
    out = []

    def bfs(start):
        lvl = np.array([start])
        seen[start] = True
        order = [lvl]
        while len(lvl):
            lo, hi = gptr[lvl], gptr[lvl + 1]
            idx = np.repeat(lo - np.cumsum(np.concatenate([[0], (hi - lo)[:-1]])), hi - lo) + np.arange((hi - lo).sum())
            cand = np.unique(nbr[idx]) if len(idx) else np.zeros(0, np.int64)
            cand = cand[~seen[cand]]
            seen[cand] = True
            lvl = cand
            if len(cand):
                order.append(cand)
        return np.concatenate(order)

    for root in range(nb):
        if seen[root]:
            continue
        first = bfs(root)  # pseudo-peripheral start: the last diagram reached from an arbitrary one
        seen[first] = False
        out.append(bfs(int(first[-1])))
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def plan_partition(instance: IlpInstance, k: int, order: np.ndarray | None = None) -> PartitionPlan:
    """Cut the diagrams into k parts of (nearly) equal node counts along
    ``order`` (default: diagram_order, compact slabs) and build each rank's
    local table, averaging CSR and boundary slots."""
    flat = instance.flat
    nb = flat.num_bdds
    if not 1 <= k <= max(nb, 1):
        raise ValueError(f"cannot split {nb} diagrams into {k} parts")
    bl, lnl = flat.bdd_layer_lo, flat.layer_node_lo
    order = diagram_order(flat) if order is None else np.asarray(order, np.int64)
    sizes = lnl[bl[order + 1]] - lnl[bl[order]]
    ends = np.cumsum(sizes)
    cut = [0] + [int(np.searchsorted(ends, ends[-1] * r / k, side="left")) + 1 for r in range(1, k)] + [nb]
    for r in range(1, k):  # every part non-empty
        cut[r] = min(max(cut[r], cut[r - 1] + 1), nb - (k - r))
    bdd_rank = np.empty(nb, np.int64)
    for r in range(k):
        bdd_rank[order[cut[r]:cut[r + 1]]] = r
    layer_rank = bdd_rank[flat.layer_bdd]
    ptr, pl = flat.proc_ptr, flat.proc_layers
    P = len(ptr) - 1
    cnt = np.diff(ptr)
    pos_of_copy = np.repeat(np.arange(P), cnt)
    copy_rank = layer_rank[pl]
    first_rank = np.full(P, -1, np.int64)
    first_rank[cnt > 0] = copy_rank[ptr[:-1][cnt > 0]]
    mixed = np.zeros(P, bool)
    np.logical_or.at(mixed, pos_of_copy, copy_rank != first_rank[pos_of_copy])
    bpos = np.flatnonzero(mixed)
    bptr = np.zeros(len(bpos) + 1, np.int64)
    bptr[1:] = np.cumsum(cnt[bpos])
    slot_base = np.full(P, -1, np.int64)
    slot_base[bpos] = bptr[:-1]
    copy_slot = np.where(mixed[pos_of_copy], slot_base[pos_of_copy] + (np.arange(len(pl)) - ptr[pos_of_copy]), -1)
    counts = flat.constraint_counts
    lam_all = instance.costs[flat.layer_var] / counts[flat.layer_var]
    free = np.flatnonzero(counts == 0)
    free_contribution = float(np.minimum(instance.costs[free], 0.0).sum()) if len(free) else 0.0

    def ranges(lo, hi):  # concatenation of [lo_i, hi_i)
        n = hi - lo
        return np.repeat(lo - np.concatenate([[0], np.cumsum(n)[:-1]]), n) + np.arange(n.sum())

    parts = []
    for r in range(k):
        sel = np.sort(order[cut[r]:cut[r + 1]])
        nl = bl[sel + 1] - bl[sel]
        g_layers = ranges(bl[sel], bl[sel + 1])
        g_nodes = ranges(lnl[g_layers], lnl[g_layers + 1])
        t = FlatTable()
        t.costs = instance.costs
        t.variable_order = instance.variable_order
        t.constraint_counts = counts
        t.bdd_layer_lo = np.concatenate([[0], np.cumsum(nl)]).astype(np.int64)
        t.layer_node_lo = np.concatenate([[0], np.cumsum(lnl[g_layers + 1] - lnl[g_layers])]).astype(np.int64)
        t.layer_var = flat.layer_var[g_layers]
        t.layer_bdd = np.repeat(np.arange(len(sel), dtype=np.int64), nl)
        z, o = flat.zero_t[g_nodes], flat.one_t[g_nodes]
        t.zero_t = np.where(z >= 0, np.searchsorted(g_nodes, np.maximum(z, 0)), z).astype(np.int64)
        t.one_t = np.where(o >= 0, np.searchsorted(g_nodes, np.maximum(o, 0)), o).astype(np.int64)
        mine = copy_rank == r
        # full local visitation CSR (every local layer visited, global copy order kept)
        lcnt = np.bincount(pos_of_copy[mine], minlength=P)
        t.proc_ptr = np.concatenate([[0], np.cumsum(lcnt)]).astype(np.int64)
        t.proc_layers = np.searchsorted(g_layers, pl[mine]).astype(np.int64)
        widths = np.diff(t.layer_node_lo)
        t.max_width = int(widths.max()) if len(widths) else 0
        t.max_degree = int(lcnt.max()) if P else 0
        t.max_layers = int(nl.max()) if len(nl) else 0
        # averaging CSR over the variables whose copies are all here
        only = mine & ~mixed[pos_of_copy]
        ocnt = np.bincount(pos_of_copy[only], minlength=P)
        local_ptr = np.concatenate([[0], np.cumsum(ocnt[ocnt > 0])]).astype(np.int32)
        local_layers = np.searchsorted(g_layers, pl[only]).astype(np.int32)
        bm = mine & mixed[pos_of_copy]
        bpos_idx = np.searchsorted(bpos, pos_of_copy[bm])
        parts.append(PartPlan(r, sel, g_layers, t, local_ptr, local_layers,
                              np.searchsorted(g_layers, pl[bm]).astype(np.int32), copy_slot[bm].astype(np.int32),
                              bptr[bpos_idx].astype(np.int32), bptr[bpos_idx + 1].astype(np.int32),
                              np.ascontiguousarray(lam_all[g_layers])))
    return PartitionPlan(k, parts, np.concatenate([p.bdds for p in parts]), int(bptr[-1]), len(bpos),
                         int((cnt > 0).sum()), free_contribution)


def scatter_duals(plan: PartitionPlan, lam_parts: list, num_layers: int) -> np.ndarray:
    """The global dual vector (FlatBdds layer order) from the parts' duals."""
    lam = np.empty(num_layers)
    for p, x in zip(plan.parts, lam_parts):
        lam[p.layers] = x.cpu().numpy() if isinstance(x, torch.Tensor) else x
    return lam


# --------------------------------------------------------------------------- communicators
class LoopbackComm:
    """Collectives over the parts of ONE process (logical partitions)."""

    def allreduce_sum(self, bufs: list) -> None:
        total = bufs[0].clone()
        for b in bufs[1:]:
            total += b
        for b in bufs:
            b.copy_(total)

    def allgather_cat(self, pieces: list) -> list:
        whole = torch.cat(pieces)
        return [whole for _ in pieces]


class DistComm:
    """torch.distributed, one part per process (NCCL for CUDA tensors, gloo on CPUs)."""

    def __init__(self, sizes: list):
        import torch.distributed as dist

        self.dist = dist
        self.sizes = sizes  # per-rank piece lengths of allgather_cat
        self.width = max(sizes) if sizes else 0

    def allreduce_sum(self, bufs: list) -> None:
        (b,) = bufs
        if b.numel():
            self.dist.all_reduce(b, op=self.dist.ReduceOp.SUM)

    def allgather_cat(self, pieces: list) -> list:
        (p,) = pieces
        pad = torch.zeros(self.width, dtype=p.dtype, device=p.device)
        pad[: p.numel()] = p
        outs = [torch.empty_like(pad) for _ in self.sizes]
        self.dist.all_gather(outs, pad)
        return [torch.cat([o[:n] for o, n in zip(outs, self.sizes)])]


# --------------------------------------------------------------------------- device engine
class DeviceEngine:
    """One rank's part on a GPU: its diagrams through dm_flat + dm_dfr_* kernels."""

    def __init__(self, part: PartPlan, device):
        from .kernels import DeviceFlat

        self.part = part
        self.device = torch.device(device)
        self.dev = DeviceFlat(part.table, self.device, exact_plans=False)
        t = part.table
        n = self.dev.dfr_table_size()
        z = lambda m: torch.zeros(m, dtype=_F64, device=self.device)  # noqa: E731
        self.lam = torch.as_tensor(part.lam0, device=self.device).clone()
        self.F, self.B = z(n), z(n)
        self.mbar, self.avg = z(t.num_layers), z(t.num_layers)
        self.bounds = z(t.num_bdds)
        i32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.int32), device=self.device)  # noqa: E731
        self.local_ptr, self.local_layers = i32(part.local_ptr), i32(part.local_layers)
        self.b = [i32(a) for a in (part.b_layer, part.b_slot, part.b_lo, part.b_hi)]

    def new_buffer(self, n: int) -> torch.Tensor:
        return torch.zeros(n, dtype=_F64, device=self.device)

    def sweep(self):
        self.dev.dfr_backward(0.0, self.lam, None, None, self.B, None, self.bounds)

    def forward_pass(self, omega):
        self.dev.dfr_forward(omega, self.lam, None, self.B, self.F, self.mbar, self.bounds)

    def backward_pass(self, omega):
        self.dev.dfr_backward(omega, self.lam, self.avg, self.F, self.B, self.mbar, self.bounds)

    def average_local(self, apply: bool):
        from . import _native
        from .kernels import _ptr, _stream

        out = self.lam if apply else self.avg
        _native.call("dm_dfr_average_csr", len(self.part.local_ptr) - 1, _ptr(self.local_ptr),
                     _ptr(self.local_layers), _ptr(self.mbar), _ptr(out), int(apply), _stream(self.device))

    def gather_boundary(self, buf):
        from . import _native
        from .kernels import _ptr, _stream

        buf.zero_()
        layer, slot = self.b[0], self.b[1]
        _native.call("dm_dfr_boundary_gather", layer.numel(), _ptr(layer), _ptr(slot), _ptr(self.mbar), _ptr(buf),
                     _stream(self.device))

    def average_boundary(self, buf, apply: bool):
        from . import _native
        from .kernels import _ptr, _stream

        layer, slot, lo, hi = self.b
        out = self.lam if apply else self.avg
        _native.call("dm_dfr_boundary_average", layer.numel(), _ptr(layer), _ptr(slot), _ptr(lo), _ptr(hi),
                     _ptr(buf), _ptr(out), int(apply), _stream(self.device))

    def global_bound(self, all_bounds) -> float:
        from .kernels import dev_sum

        out = torch.empty(1, dtype=_F64, device=self.device)
        dev_sum(all_bounds, out)
        return float(out.item())


# --------------------------------------------------------------------------- solve loop
@dataclass
class PartitionedResult:
    bounds: list
    best_bound: float
    iterations: int
    stop_reason: str
    lam_parts: list  # per owned part, device tensors
    times: list


class PartitionedSolver:
    """Deferred-schedule averaging solve of a partitioned instance over the
    parts this process owns (``engines``), with ``comm`` for the exchange."""

    def __init__(self, plan: PartitionPlan, engines: list, comm, cfg: SolveConfig | None = None):
        self.plan, self.engines, self.comm = plan, engines, comm
        self.cfg = cfg or SolveConfig(mode="mma-only", mma_schedule="deferred")
        if self.cfg.mode != "mma-only":
            raise ValueError("partitioned solves run the averaging-only mode (mode='mma-only')")
        self.bufs = [e.new_buffer(plan.slots) for e in engines]
        self._perm = torch.as_tensor(plan.bdd_order)

    def _exchange(self, apply: bool):
        for e in self.engines:
            e.average_local(apply)
        for e, b in zip(self.engines, self.bufs):
            e.gather_boundary(b)
        self.comm.allreduce_sum(self.bufs)
        for e, b in zip(self.engines, self.bufs):
            e.average_boundary(b, apply)

    def _bound(self) -> float:
        alls = self.comm.allgather_cat([e.bounds for e in self.engines])[0]
        ordered = torch.empty_like(alls)
        ordered[self._perm.to(alls.device)] = alls  # back to global diagram order: numpy's summation order
        return self.engines[0].global_bound(ordered) + self.plan.free_contribution

    def start(self, clock=time.perf_counter) -> "PartitionedSolver":
        self.clock = clock
        self.t0 = clock()
        for e in self.engines:
            e.sweep()
        self.bounds, self.times = [self._bound()], [clock() - self.t0]
        self.iterations = 0
        return self

    def step(self) -> str | None:
        """One deferred averaging round over all parts; the stop reason or None."""
        cfg, omega = self.cfg, self.cfg.mma_damping
        for e in self.engines:
            e.forward_pass(omega)
        self._exchange(apply=False)
        for e in self.engines:
            e.backward_pass(omega)
        self._exchange(apply=True)  # the flush: escrow straight into the duals
        for e in self.engines:
            e.sweep()
        b = self._bound()
        self.bounds.append(b)
        self.times.append(self.clock() - self.t0)
        self.iterations += 1
        it, k, bounds = self.iterations, cfg.effective_stall_window, self.bounds
        if k == 1:
            if b - bounds[-2] < cfg.dual_tolerance * max(1.0, abs(b)):
                return "dual_tolerance"
        elif it >= k and max(bounds[-k:]) - max(bounds[:-k]) < cfg.dual_tolerance * max(1.0, abs(b)):
            return "dual_tolerance"
        if cfg.max_seconds is not None and self.times[-1] > cfg.max_seconds:
            return "max_seconds"
        return None

    def solve(self, clock=time.perf_counter) -> PartitionedResult:
        self.start(clock)
        reason = "max_iterations"
        for _ in range(self.cfg.max_iterations):
            r = self.step()
            if r is not None:
                reason = r
                break
        return PartitionedResult(self.bounds, max(self.bounds), self.iterations, reason,
                                 [e.lam for e in self.engines], self.times)
