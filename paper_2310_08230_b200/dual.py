"""Lagrangian dual state and exact min-marginal-averaging passes on the GPU.

Same API and semantics as the reference (dual.py:29-201): ``lam`` has one
entry per (variable, constraint) incidence indexed by global layer id, the
forward/backward distance caches carry validity flags, and every bound is
the numpy-pairwise sum of the per-diagram optima plus the contribution of
unconstrained variables.  All vectors live in HBM (``lam_d``, ``F``, ``B``);
``lam`` and the table accessors return host copies for API compatibility.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from .config import SCHEDULE_DEFERRED, SCHEDULE_EXACT
from .ilp import IlpInstance
from .kernels import DeviceFlat, FlatBdds, dev_axpy_host, dev_sum

FORWARD = "forward"
BACKWARD = "backward"
NP_MAX_DIAGRAMS = 200_000  # deferred schedule: node-parallel passes up to this many diagrams ...
NP_MIN_LAYERS = 256  # ... or when some diagram is longer than this

_F64 = torch.float64


def as_device(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=_F64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=device)


def to_host(x: torch.Tensor) -> np.ndarray:
    """Device -> host copy through page-locked memory (torch's caching host
    allocator reuses the block): a pageable read-back of the 75 MB C2 dual
    vector runs at a fraction of the copy engine's rate."""
    if x.device.type != "cuda":
        return x.numpy()
    h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    h.copy_(x)  # synchronous for the host: the values are there on return
    return h.numpy()


class KernelTimer:
    """CUDA-event timing of individual kernel launches on the launching
    (current torch) stream; used by bench.py for the roofline numbers."""

    def __init__(self):
        self.events: dict[str, list] = {}
        self.counts: dict[str, int] = {}

    def begin(self, name):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        return (name, a, b)

    def end(self, ev):
        name, a, b = ev
        b.record()
        self.events.setdefault(name, []).append((a, b))

    def count(self, name, n):
        self.counts[name] = self.counts.get(name, 0) + int(n)

    def summary(self) -> dict[str, dict]:
        torch.cuda.synchronize()
        out = {}
        for name, evs in self.events.items():
            ms = [a.elapsed_time(b) for a, b in evs]
            out[name] = {"launches": len(ms), "total_ms": float(sum(ms)), "avg_ms": float(sum(ms) / len(ms))}
        return out


class DualState:
    """Per-constraint duals plus cached sweep distances, resident on a GPU."""

    def __init__(self, instance: IlpInstance, flat: FlatBdds | None = None, device=None,
                 schedule: str = SCHEDULE_EXACT):
        if schedule not in (SCHEDULE_EXACT, SCHEDULE_DEFERRED):
            raise ValueError(f"unknown averaging schedule {schedule!r}")
        self.schedule = schedule
        self.instance = instance
        self.flat = flat if flat is not None else FlatBdds(instance)
        self.dev: DeviceFlat = self.flat.device(device, exact_plans=schedule == SCHEDULE_EXACT)
        d = self.dev.device
        self.device = d
        f = self.flat
        self.lam_d = torch.zeros(f.num_layers, dtype=_F64, device=d)
        self.F = torch.zeros(f.num_nodes, dtype=_F64, device=d)
        self.B = torch.zeros(f.num_nodes, dtype=_F64, device=d)
        self._bounds = torch.zeros(f.num_bdds, dtype=_F64, device=d)
        self._scratch_B: torch.Tensor | None = None
        self._scratch_bounds = torch.zeros(f.num_bdds, dtype=_F64, device=d)
        self._scal = torch.zeros(8, dtype=_F64, device=d)
        # device scalars read back together: bound sums [0, 8), the passes'
        # watchdog word [8], the curvature product s.y [9]
        self._slots = torch.zeros(16, dtype=_F64, device=d)
        self._pending: list[int] = []  # bound slots not yet read, in order
        self._status_pending = False
        self._step_state = None
        self._move_pending = False
        self.f_valid = False
        self.b_valid = False
        self._bound = -np.inf
        self._best_bound = -np.inf
        self.sweeps = 0  # full-table sweep equivalents (2 arcs per node each)
        self.pass_timer: KernelTimer | None = None
        self._bgen = 0  # generation of the distance-to-TRUE table B
        self._argmin_cache = None
        self._dec_gen = -1  # B generation whose argmin decisions the last backward pass recorded
        self._np = False
        if schedule == SCHEDULE_DEFERRED:
            # node-parallel passes on the node-order F / B when the instance
            # allows them (dm_dfr_np_*); otherwise lane-per-diagram passes on
            # tables in the sweep layout (dm_dfr_*): f_valid / b_valid then
            # refer to F_il / B_il, and the node-order F / B are filled from
            # them on demand
            # node-parallel passes pay off when few diagrams leave most lanes
            # idle or long diagrams set a serial floor (C4: 125 k diagrams,
            # passes 1.3-1.5x faster; unsplit C2: 4,002-layer diagrams, 1.4-1.7x),
            # lane-per-diagram passes when there are many short diagrams (C2:
            # 637 k, 2-2.7x faster); DM_DFR_NP=1/0 forces either
            env = os.environ.get("DM_DFR_NP")
            auto = f.num_bdds <= NP_MAX_DIAGRAMS or int(f.table.max_layers) > NP_MIN_LAYERS
            self._np = self.dev.dfr_node_parallel and (auto if env is None else env != "0")
            if not self._np:
                n = self.dev.dfr_table_size()
                self.F_il = torch.zeros(n, dtype=_F64, device=d)
                self.B_il = torch.zeros(n, dtype=_F64, device=d)
            self.mbar = torch.zeros(f.num_layers, dtype=_F64, device=d)  # escrow of the last pass
            self.avg = torch.zeros(f.num_layers, dtype=_F64, device=d)  # its per-copy average
        free = instance.unconstrained_variables()
        self.free_values = {int(v): (0 if instance.costs[v] >= 0 else 1) for v in free}
        self.free_contribution = float(np.minimum(instance.costs[free], 0.0).sum()) if len(free) else 0.0

    # -- host views -------------------------------------------------------
    @property
    def lam(self) -> np.ndarray:
        if self._status_pending:
            self.read_scalars()  # never hand out duals of an aborted pass
        return to_host(self.lam_d)

    @property
    def arc_updates(self) -> int:
        return self.sweeps * 2 * self.flat.num_nodes

    # -- cache management (dual.py:66-106) ---------------------------------
    def _sum_bounds(self, bounds: torch.Tensor) -> float:
        dev_sum(bounds, self._scal[0:1])
        return float(self._scal[0].item()) + self.free_contribution

    def _set_bound(self) -> None:
        """Queue the bound of the current distance table (numpy-order sum on
        the device); the host reads it, with the other queued scalars, the
        next time one is needed (``read_scalars``)."""
        if len(self._pending) == 8:
            self.read_scalars()
        i = len(self._pending)
        dev_sum(self._bounds, self._slots[i:i + 1])
        self._pending.append(i)

    def _check_status_later(self) -> None:
        """Queue the exact passes' watchdog word (read by ``read_scalars``)."""
        self.dev.status_to(self._slots[8:9])
        self._status_pending = True

    def read_scalars(self) -> np.ndarray:
        """One read-back of the queued device scalars: applies the queued
        bounds in order (bound = latest, best_bound = running max, as the
        eager bookkeeping would) and raises if a pass's watchdog fired."""
        vals = self._slots.cpu().numpy()
        if self._status_pending:
            self._status_pending = False
            if vals[8] != 0.0:
                self._pending = []
                self.dev.check_status()  # raises with the library's message (and clears the word)
        for i in self._pending:
            b = float(vals[i]) + self.free_contribution
            self._bound = b
            if b > self._best_bound:
                self._best_bound = b
        self._pending = []
        return vals

    @property
    def bound(self) -> float:
        if self._pending or self._status_pending:
            self.read_scalars()
        return self._bound

    @bound.setter
    def bound(self, v: float) -> None:
        self._pending = []
        self._bound = v

    @property
    def best_bound(self) -> float:
        if self._pending or self._status_pending:
            self.read_scalars()
        return self._best_bound

    @best_bound.setter
    def best_bound(self, v: float) -> None:
        self._pending = []
        self._best_bound = v

    @property
    def deferred(self) -> bool:
        return self.schedule == SCHEDULE_DEFERRED

    # the deferred schedule's two passes, on whichever tables it keeps
    def _dfr_fw(self, omega, avg, mbar) -> None:
        if self._np:
            self.dev.dfr_np_forward(omega, self.lam_d, avg, self.B, self.F, mbar, self._bounds)
        else:
            self.dev.dfr_forward(omega, self.lam_d, avg, self.B_il, self.F_il, mbar, self._bounds)

    def _dfr_bw(self, omega, avg, mbar, record_decisions=False) -> None:
        if self._np:
            self.dev.dfr_np_backward(omega, self.lam_d, avg, self.F, self.B, mbar, self._bounds, record_decisions)
        else:
            self.dev.dfr_backward(omega, self.lam_d, avg, self.F_il, self.B_il, mbar, self._bounds, record_decisions)

    @property
    def _dec_table(self) -> torch.Tensor:
        """The distance table the recorded argmin decisions belong to."""
        return self.B_il if self.deferred and not self._np else self.B

    def refresh_backward(self) -> None:
        if self.deferred:
            self._dfr_bw(0.0, None, None, record_decisions=True)
            self._bgen += 1
            if self.dev.dfr_records_decisions:
                self._dec_gen = self._bgen
        else:
            self.dev.k_backward(self.lam_d, self.B, self._bounds)
            self._bgen += 1
        self.sweeps += 1
        self.b_valid = True
        self._set_bound()

    def refresh_forward(self) -> None:
        if self.deferred:
            self._dfr_fw(0.0, None, None)
        else:
            self.dev.k_forward(self.lam_d, self.F, self._bounds)
        self.sweeps += 1
        self.f_valid = True
        self._set_bound()

    def node_tables(self, need_f: bool = True, need_b: bool = True) -> tuple[torch.Tensor, torch.Tensor]:
        """Node-order (FlatBdds) F and B valid for the current duals; under
        the deferred schedule they are converted from the interleaved tables."""
        if need_f and not self.f_valid:
            self.refresh_forward()
        if need_b and not self.b_valid:
            self.refresh_backward()
        if self.deferred and not self._np:
            if need_f:
                self.dev.dfr_to_nodes(self.F_il, self.F)
            if need_b:
                self.dev.dfr_to_nodes(self.B_il, self.B)
        return self.F, self.B

    def deferred_round(self, omega: float) -> None:
        """One round of the deferred (FastDOG) schedule: a forward and a
        backward averaging pass over all diagrams in parallel, each copy's
        escrow redistributed by the next pass, and a final sweep that adds the
        backward pass's escrow and rebuilds B (dm_deferred.cu).  The duals are
        feasible again afterwards; the bound of the new duals is queued."""
        if not self.deferred:
            raise ValueError("deferred_round needs a state built with schedule='deferred'")
        timer = self.pass_timer
        if not self.b_valid:
            self.refresh_backward()
        ev = timer.begin("dfr_forward") if timer else None
        self._dfr_fw(omega, None, self.mbar)
        if ev:
            timer.end(ev)
        ev = timer.begin("dfr_average") if timer else None
        self.dev.dfr_average(self.mbar, self.avg)
        if ev:
            timer.end(ev)
        ev = timer.begin("dfr_backward") if timer else None
        self._dfr_bw(omega, self.avg, self.mbar)
        if ev:
            timer.end(ev)
        # flush: the backward pass's escrow straight into the duals, then a
        # plain sweep rebuilds B (and the argmin decisions) for them
        ev = timer.begin("dfr_flush") if timer else None
        self.dev.dfr_flush(self.mbar, self.lam_d)
        if ev:
            timer.end(ev)
        ev = timer.begin("dfr_sweep") if timer else None
        self._dfr_bw(0.0, None, None, record_decisions=True)
        if ev:
            timer.end(ev)
        self._bgen += 1
        if self.dev.dfr_records_decisions:
            self._dec_gen = self._bgen
        self.sweeps += 5
        self.b_valid = True
        self.f_valid = False
        self._set_bound()

    def shift_lambda(self, delta) -> None:
        """Move the duals along a feasibility-preserving direction."""
        self.lam_d += as_device(delta, self.device)
        self.f_valid = False
        self.b_valid = False

    def shift_lambda_scaled(self, gamma: float, d: torch.Tensor) -> None:
        """lam += gamma * d with numpy's two roundings (qn.py:206)."""
        dev_axpy_host(self.lam_d, gamma, d)
        self.f_valid = False
        self.b_valid = False

    def set_lambda(self, lam) -> None:
        lam_t = as_device(lam, self.device)
        if lam_t.shape != self.lam_d.shape:
            raise ValueError("dual vector length mismatch")
        self.lam_d.copy_(lam_t)
        self.f_valid = False
        self.b_valid = False
        self.refresh_backward()

    def _scratch(self) -> torch.Tensor:
        if self._scratch_B is None:
            self._scratch_B = torch.zeros(self.flat.num_nodes, dtype=_F64, device=self.device)
        return self._scratch_B

    def eval_lambda(self, lam_trial) -> float:
        """Dual objective of a trial vector; caches are left untouched."""
        self.dev.k_backward(as_device(lam_trial, self.device), self._scratch(), self._scratch_bounds)
        self.sweeps += 1
        return self._sum_bounds(self._scratch_bounds)

    def eval_step(self, d: torch.Tensor, gamma: float) -> float:
        """Objective at lam + gamma*d without materialising it (fused trial)."""
        ev = self.pass_timer.begin("backward_trial") if self.pass_timer else None
        # trial distances are scratch in the reference (dual.py:99-106): only
        # the per-diagram optima are produced, no distance table is written
        self.dev.k_backward_trial(self.lam_d, d, gamma, None, self._scratch_bounds)
        if ev:
            self.pass_timer.end(ev)
        self.sweeps += 1
        return self._sum_bounds(self._scratch_bounds)

    def search_step(self, d: torch.Tensor, gamma_prev: float, shrink: float, grow: float, min_ascent: float,
                    max_trials: int) -> tuple[float, float, int]:
        """find_step_size's trial sequence on the device (dm_step_search):
        returns (gamma_best, e_best, trials run); one read-back at the end."""
        if self._step_state is None:
            self._step_state = torch.zeros(8, dtype=_F64, device=self.device)
        ev = self.pass_timer.begin("step_search") if self.pass_timer else None
        self.dev.step_search(self.lam_d, d, gamma_prev, self.free_contribution, shrink, grow, min_ascent,
                             max_trials, self._scratch_bounds, self._step_state)
        if ev:
            self.pass_timer.end(ev)
        st = self._step_state.cpu().numpy()
        trials = int(st[6])
        self.sweeps += trials
        if self.pass_timer:
            self.pass_timer.count("step_search_trials", trials)
        return float(st[3]), float(st[2]), trials

    def search_and_move(self, d: torch.Tensor, gamma_prev: float, shrink: float, grow: float, min_ascent: float,
                        max_trials: int) -> None:
        """find_step_size, the move it decides and the refresh of B (qn.py:203-206,
        dual.py:164-165), all queued on the device (exact schedule, B valid):
        dm_step_search, then dm_qn_move — lam += gamma_best * d and B rebuilt
        iff the best trial beat the current objective.  No read-back: the
        verdict {gamma_best, used, trials} lands in _slots[10:13] for the
        next ``read_scalars`` (``take_move``)."""
        if self.deferred or not self.b_valid:
            raise ValueError("search_and_move needs the exact schedule and a valid B")
        base = self.bound  # known on the host: the last read-back left nothing queued
        if self._step_state is None:
            self._step_state = torch.zeros(8, dtype=_F64, device=self.device)
        ev = self.pass_timer.begin("step_search") if self.pass_timer else None
        self.dev.step_search(self.lam_d, d, gamma_prev, self.free_contribution, shrink, grow, min_ascent,
                             max_trials, self._scratch_bounds, self._step_state)
        if ev:
            self.pass_timer.end(ev)
        self.dev.qn_move(self.lam_d, d, base, self._step_state, self._slots[10:13], self.B, self._bounds)
        self._bgen += 1  # B rebuilt, or unchanged for unchanged duals
        self.f_valid = False
        self.b_valid = True
        self._set_bound()
        self._move_pending = True

    def take_move(self, vals: np.ndarray) -> tuple[float, bool]:
        """(gamma_best, used) of the last ``search_and_move`` from a read-back."""
        self._move_pending = False
        used = bool(vals[11] != 0.0)
        trials = int(vals[12])
        self.sweeps += trials + (1 if used else 0)
        if self.pass_timer:
            self.pass_timer.count("step_search_trials", trials)
        return float(vals[10]), used

    # -- dual vectors per constraint ------------------------------------------
    def lambda_of(self, constraint: int) -> np.ndarray:
        lo, hi = self.flat.bdd_layer_lo[constraint], self.flat.bdd_layer_lo[constraint + 1]
        return self.lam_d[lo:hi].cpu().numpy()

    def lambda_sums(self) -> np.ndarray:
        """Per-variable sum of dual entries (== costs when feasible)."""
        out = torch.zeros(self.instance.num_variables, dtype=_F64, device=self.device)
        self.dev.lambda_sums(self.lam_d, out)
        res = out.cpu().numpy()
        fv = list(self.free_values)
        res[fv] = self.instance.costs[fv]
        return res

    def min_marginal_table_device(self) -> tuple[torch.Tensor, torch.Tensor]:
        F, B = self.node_tables()
        m0 = torch.empty(self.flat.num_layers, dtype=_F64, device=self.device)
        m1 = torch.empty_like(m0)
        self.dev.k_min_marginals(self.lam_d, F, B, m0, m1)
        return m0, m1

    def min_marginal_table(self) -> tuple[np.ndarray, np.ndarray]:
        """Fresh (m0, m1) per layer at the current duals."""
        m0, m1 = self.min_marginal_table_device()
        return m0.cpu().numpy(), m1.cpu().numpy()


def init_duals(instance: IlpInstance, device=None, flat: FlatBdds | None = None,
               schedule: str = SCHEDULE_EXACT) -> DualState:
    """Spread every cost uniformly over the constraints containing it (dual.py:137-144)."""
    state = DualState(instance, flat=flat, device=device, schedule=schedule)
    costs = torch.as_tensor(np.ascontiguousarray(instance.costs, dtype=np.float64), device=state.device)
    state.dev.init_duals(costs, state.lam_d)
    state.refresh_backward()
    return state


def dual_objective(state: DualState) -> float:
    """Sum of subproblem optima; a lower bound for the integer program."""
    if not (state.b_valid or state.f_valid):
        state.refresh_backward()
    return state.bound


def mma_pass(state: DualState, direction: str) -> DualState:
    """One exact averaging pass over all variables (dual.py:154-186)."""
    if state.deferred:
        raise ValueError("mma_pass is the exact schedule; a deferred-schedule state averages with deferred_round")
    timer = state.pass_timer
    if direction == FORWARD:
        if not state.b_valid:
            state.refresh_backward()
        ev = timer.begin("mma_forward") if timer else None
        state.dev.k_mma_forward(state.lam_d, state.F, state.B, state._bounds)
        if ev:
            timer.end(ev)
        state.f_valid = True
        state.b_valid = False
    elif direction == BACKWARD:
        if not state.f_valid:
            state.refresh_forward()
        ev = timer.begin("mma_backward") if timer else None
        state.dev.k_mma_backward(state.lam_d, state.F, state.B, state._bounds)
        if ev:
            timer.end(ev)
        state._bgen += 1
        if state.dev.records_decisions:
            state._dec_gen = state._bgen
        state.b_valid = True
        state.f_valid = False
    else:
        raise ValueError(f"unknown pass direction {direction!r}")
    state.sweeps += 2
    state._set_bound()
    state._check_status_later()  # a fired watchdog raises at the next read-back
    return state


def subgradient_device(state: DualState) -> torch.Tensor:
    """Argmin bits for the current duals.  The reference recomputes them at
    the end of one iteration and again at the start of the next on the same
    duals (qn.py:201,249); the walk is cached per distance-table generation,
    so the second call returns the identical tensor without a launch.
    Callers must not modify the returned tensor."""
    if not state.b_valid:
        state.refresh_backward()
    cached = state._argmin_cache
    if cached is not None and cached[0] == state._bgen:
        return cached[1]
    bits = torch.empty(state.flat.num_layers, dtype=_F64, device=state.device)
    if state._dec_gen == state._bgen:
        # decisions of the pass that wrote B
        state.dev.k_argmin_from_pass(state._dec_table, bits)
    else:
        _, B = state.node_tables(need_f=False)
        state.dev.k_argmin(state.lam_d, B, bits)
    state._argmin_cache = (state._bgen, bits)
    return bits


def subgradient(state: DualState) -> np.ndarray:
    """Concatenated minimising assignments of all subproblems (dual.py:189-201)."""
    return subgradient_device(state).cpu().numpy()
