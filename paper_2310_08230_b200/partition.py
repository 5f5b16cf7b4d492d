"""One instance split over several GPUs (BASELINE config C4: "BDDs partitioned
across 1/2/4/8 B200 with NCCL marginal allreduce").

No reference counterpart: the reference is single-process;
the plan is SURVEY.md §5(b).  The diagrams are cut into k contiguous blocks
(balanced by node count); each rank owns its block's diagrams, their nodes,
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
    bdd_lo: int
    bdd_hi: int
    layer_lo: int
    layer_hi: int
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
    cuts: list  # diagram ids: part r owns [cuts[r], cuts[r+1])
    parts: list
    slots: int  # boundary exchange buffer length (copies of boundary variables)
    boundary_variables: int
    variables_with_copies: int
    free_contribution: float

    @property
    def boundary_fraction(self) -> float:
        return self.boundary_variables / max(self.variables_with_copies, 1)


def diagram_cuts(flat, k: int) -> list:
    """k contiguous diagram blocks with (nearly) equal node counts."""
    nb = flat.num_bdds
    if not 1 <= k <= max(nb, 1):
        raise ValueError(f"cannot split {nb} diagrams into {k} parts")
    node_end = flat.layer_node_lo[flat.bdd_layer_lo[1:]]  # nodes up to the end of each diagram
    total = flat.num_nodes
    cuts = [0]
    for r in range(1, k):
        c = int(np.searchsorted(node_end, total * r / k, side="left")) + 1
        cuts.append(min(max(c, cuts[-1] + 1), nb - (k - r)))
    cuts.append(nb)
    return cuts


def plan_partition(instance: IlpInstance, k: int) -> PartitionPlan:
    flat = instance.flat
    cuts = diagram_cuts(flat, k)
    bl, lnl = flat.bdd_layer_lo, flat.layer_node_lo
    layer_rank = np.repeat(np.arange(k), [int(bl[cuts[r + 1]] - bl[cuts[r]]) for r in range(k)])
    ptr, pl = flat.proc_ptr, flat.proc_layers
    P = len(ptr) - 1
    cnt = np.diff(ptr)
    pos_of_copy = np.repeat(np.arange(P), cnt)
    copy_rank = layer_rank[pl]
    # a position is on the boundary when its copies are not all on one rank
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
    parts = []
    for r in range(k):
        b0, b1 = cuts[r], cuts[r + 1]
        L0, L1 = int(bl[b0]), int(bl[b1])
        N0, N1 = int(lnl[L0]), int(lnl[L1])
        t = FlatTable()
        t.costs = instance.costs
        t.variable_order = instance.variable_order
        t.constraint_counts = counts
        t.bdd_layer_lo = bl[b0:b1 + 1] - L0
        t.layer_node_lo = lnl[L0:L1 + 1] - N0
        t.layer_var = flat.layer_var[L0:L1].copy()
        t.layer_bdd = flat.layer_bdd[L0:L1] - b0
        z, o = flat.zero_t[N0:N1], flat.one_t[N0:N1]
        t.zero_t = np.where(z >= 0, z - N0, z)
        t.one_t = np.where(o >= 0, o - N0, o)
        mine = copy_rank == r
        # full local visitation CSR (every local layer visited, global copy order kept)
        lcnt = np.bincount(pos_of_copy[mine], minlength=P)
        t.proc_ptr = np.concatenate([[0], np.cumsum(lcnt)]).astype(np.int64)
        t.proc_layers = (pl[mine] - L0).astype(np.int64)
        widths = np.diff(t.layer_node_lo)
        t.max_width = int(widths.max()) if len(widths) else 0
        t.max_degree = int(lcnt.max()) if P else 0
        t.max_layers = int(np.diff(t.bdd_layer_lo).max()) if b1 > b0 else 0
        # averaging CSR over the variables whose copies are all here
        only = mine & ~mixed[pos_of_copy]
        ocnt = np.bincount(pos_of_copy[only], minlength=P)
        keep = ocnt > 0
        local_ptr = np.concatenate([[0], np.cumsum(ocnt[keep])]).astype(np.int32)
        local_layers = (pl[only] - L0).astype(np.int32)
        bm = mine & mixed[pos_of_copy]
        bpos_idx = np.searchsorted(bpos, pos_of_copy[bm])
        parts.append(PartPlan(r, b0, b1, L0, L1, t, local_ptr, local_layers,
                              (pl[bm] - L0).astype(np.int32), copy_slot[bm].astype(np.int32),
                              bptr[bpos_idx].astype(np.int32), bptr[bpos_idx + 1].astype(np.int32),
                              np.ascontiguousarray(lam_all[L0:L1])))
    return PartitionPlan(k, cuts, parts, int(bptr[-1]), len(bpos), int((cnt > 0).sum()), free_contribution)


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
        self.dev = DeviceFlat(part.table, self.device)
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

    def _exchange(self, apply: bool):
        for e in self.engines:
            e.average_local(apply)
        for e, b in zip(self.engines, self.bufs):
            e.gather_boundary(b)
        self.comm.allreduce_sum(self.bufs)
        for e, b in zip(self.engines, self.bufs):
            e.average_boundary(b, apply)

    def _bound(self) -> float:
        alls = self.comm.allgather_cat([e.bounds for e in self.engines])
        return self.engines[0].global_bound(alls[0]) + self.plan.free_contribution

    def solve(self, clock=time.perf_counter) -> PartitionedResult:
        cfg, omega = self.cfg, self.cfg.mma_damping
        t0 = clock()
        for e in self.engines:
            e.sweep()
        bounds, times = [self._bound()], [clock() - t0]
        reason = "max_iterations"
        k = cfg.effective_stall_window
        for it in range(1, cfg.max_iterations + 1):
            for e in self.engines:
                e.forward_pass(omega)
            self._exchange(apply=False)
            for e in self.engines:
                e.backward_pass(omega)
            self._exchange(apply=True)  # the flush: escrow straight into the duals
            for e in self.engines:
                e.sweep()
            b = self._bound()
            bounds.append(b)
            times.append(clock() - t0)
            if k == 1:
                if b - bounds[-2] < cfg.dual_tolerance * max(1.0, abs(b)):
                    reason = "dual_tolerance"
                    break
            elif it >= k and max(bounds[-k:]) - max(bounds[:-k]) < cfg.dual_tolerance * max(1.0, abs(b)):
                reason = "dual_tolerance"
                break
            if cfg.max_seconds is not None and clock() - t0 > cfg.max_seconds:
                reason = "max_seconds"
                break
        return PartitionedResult(bounds, max(bounds), len(bounds) - 1, reason, [e.lam for e in self.engines], times)
