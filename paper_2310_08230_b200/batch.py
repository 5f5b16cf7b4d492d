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


# --------------------------------------------------------------------------- batched hybrid solves
class _Handle:
    """dm_batch handle: per-instance reduction plans of a merged flat."""

    def __init__(self, state, index: BatchIndex):
        import ctypes

        from . import _native
        from .kernels import _stream

        self.lib = _native.load()
        self.device = state.device
        bo = np.ascontiguousarray(index.bdd, dtype=np.int64)
        lo = np.ascontiguousarray(index.layer, dtype=np.int64)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(self.lib.dm_batch_create(state.dev.handle, len(index), bo.ctypes.data, lo.ctypes.data,
                                                   _stream(self.device), ctypes.byref(h)), "dm_batch_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self.lib.dm_batch_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None


def _ptrs(tensors, device) -> torch.Tensor:
    """Device array of the tensors' data pointers (int64)."""
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64, device=device)


class BatchedSolver:
    """Every instance's OWN hybrid ``qn.solve`` (qn.py:211-259), side by side
    on one merged block-diagonal instance: the averaging passes and sweeps run
    once for the whole batch, and each instance keeps its own L-BFGS history,
    step size, step search, curvature test and stopping rule, with reductions
    taken over its own ranges in the order a separate solve takes them
    (dm_batch.cu) — so every instance's bounds and duals are bit-identical to
    ``qn.solve(instance, cfg)`` (tests/test_batch.py).  An instance whose
    stopping rule fires is frozen: its duals and records are snapshotted
    (the merged passes keep running over it, unobserved)."""

    def __init__(self, instances, cfg: SolveConfig | None = None, device=None, clock=time.perf_counter,
                 reuse_buffers: bool = False):
        from .dual import init_duals

        self.instances = list(instances)
        self.cfg = cfg or SolveConfig()
        if self.cfg.mode != "hybrid":
            raise ValueError("BatchedSolver runs hybrid solves (mode='mma-only' batches: solve_merged)")
        self.clock = clock
        self.t0 = clock()
        self.merged, self.index = merge_instances(self.instances, reuse_buffers=reuse_buffers)
        self.state = init_duals(self.merged, device=device, schedule=self.cfg.mma_schedule)
        self.device = self.state.device
        self.h = _Handle(self.state, self.index)
        self.n = len(self.instances)

    # -- device helpers ----------------------------------------------------------
    def _call(self, name, *args):
        from . import _native
        from .kernels import _stream

        _native.call(name, self.h._h, *args, _stream(self.device))

    def _sums(self, out):
        """Per-instance numpy-order sums of the state's per-diagram optima."""
        self._call("dm_batch_sum", self.state._bounds.data_ptr(), out.data_ptr())

    # -- the solve -----------------------------------------------------------------
    def solve(self):
        from .dual import BACKWARD, FORWARD, mma_pass, subgradient_device
        from .qn import IterationRecord, StepConfig

        cfg, n, dev, st = self.cfg, self.n, self.device, self.state
        f64 = dict(dtype=torch.float64, device=dev)
        m = cfg.history_size
        L = self.merged.flat.num_layers
        scfg = StepConfig.from_solve_config(cfg)
        free_c = np.array([float(np.minimum(i.costs[i.unconstrained_variables()], 0.0).sum()) for i in self.instances])
        free_c_d = torch.as_tensor(free_c, **f64)
        # per-instance bookkeeping (host)
        records = [[] for _ in range(n)]
        bound = np.zeros(n)
        best = np.full(n, -np.inf)
        gamma = np.full(n, scfg.initial_step)
        min_ascent = np.zeros(n)
        stopped = np.zeros(n, bool)
        stop_reason = ["max_iterations"] * n
        iters = np.zeros(n, np.int64)
        lam_final = [None] * n
        rings = [[] for _ in range(n)]  # newest first: (slot, rho, sy)
        free_slots = [list(range(m + 1)) for _ in range(n)]
        pool_s = [torch.empty(L, **f64) for _ in range(m + 1)]
        pool_y = [torch.empty(L, **f64) for _ in range(m + 1)]
        sums = torch.empty(n, **f64)
        nb_scratch = torch.empty(self.merged.flat.num_bdds, **f64)
        state_d = torch.empty(8 * n, **f64)

        def note(b_host, ks):
            for k in ks:
                bound[k] = b_host[k] + free_c[k]
                best[k] = max(best[k], bound[k])

        every = np.arange(n)
        self._sums(sums)  # init_duals' refresh (dual.py:137-144)
        note(sums.cpu().numpy(), every)
        t = self.clock() - self.t0
        for k in range(n):
            records[k].append(IterationRecord(0, "init", bound[k], t))
        initial = bound.copy()
        lam_prev = st.lam_d.clone()
        g_prev = subgradient_device(st).clone()
        d = torch.zeros(L, **f64)
        dots = torch.empty((2 * m + 1, n), **f64)
        alphas = torch.empty((m, n), **f64)
        for it in range(1, cfg.max_iterations + 1):
            live = ~stopped
            qn_on = live & np.array([len(r) > 0 for r in rings])
            used = np.zeros(n, bool)
            refreshed = np.zeros(n, bool)
            if qn_on.any():
                g = subgradient_device(st)
                self._two_loop(g, d, rings, qn_on, pool_s, pool_y, dots, alphas)
                dh = d
                d = torch.empty(L, **f64)
                st.dev.project_direction(dh, d)  # per variable: independent per instance
                active = torch.as_tensor(qn_on.astype(np.int8), device=dev)
                base = bound.copy()
                from . import _native
                from .kernels import _stream

                # (the argument tensors are bound to names: a temporary's block could be
                # reused by the next temporary before the kernels read it)
                gamma_d = torch.as_tensor(gamma, **f64)
                ascent_d = torch.as_tensor(min_ascent, **f64)
                _native.call("dm_batch_step_search", st.dev.handle, self.h._h, st.lam_d.data_ptr(), d.data_ptr(),
                             gamma_d.data_ptr(), free_c_d.data_ptr(), ascent_d.data_ptr(), float(scfg.shrink),
                             float(scfg.grow), int(scfg.max_trials), active.data_ptr(), nb_scratch.data_ptr(),
                             sums.data_ptr(), state_d.data_ptr(), _stream(dev))
                ctl = state_d.cpu().numpy().reshape(n, 8)
                st.sweeps += int(ctl[qn_on, 6].max()) if qn_on.any() else 0
                for k in np.flatnonzero(qn_on):
                    gamma[k] = ctl[k, 3]  # qn.py:159 returns the best trial's step
                    used[k] = ctl[k, 2] > base[k]
                if used.any():
                    coef = torch.as_tensor(np.where(used, gamma, 0.0), **f64)
                    self._update(4, st.lam_d, [d] * n, coef, None, None, None, used)
                    st.f_valid = st.b_valid = False
                    st.refresh_backward()  # the averaging pass's refresh (dual.py:164-165), all at once
                    self._sums(sums)
                    refreshed = used
                    note(sums.cpu().numpy(), np.flatnonzero(used))
            if st.deferred:
                st.deferred_round(cfg.mma_damping)
                self._sums(sums)
                note(sums.cpu().numpy(), np.flatnonzero(live))
            else:
                mma_pass(st, FORWARD)
                self._sums(sums)
                fw = sums.clone()
                mma_pass(st, BACKWARD)
                self._sums(sums)
                note(fw.cpu().numpy(), np.flatnonzero(live))
                note(sums.cpu().numpy(), np.flatnonzero(live))
            del refreshed
            g_now = subgradient_device(st).clone()
            # curvature pair into each live instance's free slot, and s . y per instance
            slots = [free_slots[k][-1] if live[k] else 0 for k in range(n)]
            s_p = _ptrs([pool_s[slots[k]] for k in range(n)], dev)
            y_p = _ptrs([pool_y[slots[k]] for k in range(n)], dev)
            act = torch.as_tensor(live.astype(np.int8), device=dev)
            self._call_curv(st.lam_d, lam_prev, g_now, g_prev, s_p, y_p, act)
            self._call("dm_batch_dot", s_p.data_ptr(), y_p.data_ptr(), act.data_ptr(), sums.data_ptr())
            sy = sums.cpu().numpy()
            st.read_scalars()  # the passes' watchdog word (raises if an exact pass was aborted)
            t = self.clock() - self.t0
            for k in np.flatnonzero(live):
                iters[k] = it
                records[k].append(IterationRecord(it, "hybrid" if used[k] else "mma", bound[k], t))
                if it == 1:
                    min_ascent[k] = cfg.ascent_rel_threshold * (bound[k] - initial[k])
                if sy[k] >= scfg.curvature_eps:  # qn.py:85-92
                    slot = free_slots[k].pop()
                    rings[k].insert(0, (slot, 1.0 / sy[k], float(sy[k])))
                    if len(rings[k]) > m:
                        free_slots[k].append(rings[k].pop()[0])
                if self._tolerance_met(records[k], bound[k], it, cfg):
                    stop_reason[k] = "dual_tolerance"
                elif cfg.max_seconds is not None and t > cfg.max_seconds:
                    stop_reason[k] = "max_seconds"
                else:
                    continue
                stopped[k] = True
                lo, hi = self.index.layer[k], self.index.layer[k + 1]
                lam_final[k] = st.lam_d[lo:hi].cpu().numpy()
            g_prev = g_now
            if stopped.all():
                break
        for k in np.flatnonzero(~stopped):
            lo, hi = self.index.layer[k], self.index.layer[k + 1]
            lam_final[k] = st.lam_d[lo:hi].cpu().numpy()
        return [BatchedResult(records[k], float(best[k]), int(iters[k]), stop_reason[k], lam_final[k])
                for k in range(n)]

    @staticmethod
    def _tolerance_met(recs, bound, it, cfg) -> bool:
        """DualSolver.step's dual-tolerance rule (one iteration's gain, or the
        best bound over the stall window for the deferred schedule)."""
        k = cfg.effective_stall_window
        if k == 1:
            return bound - recs[-2].dual_objective < cfg.dual_tolerance * max(1.0, abs(bound))
        if it < k:
            return False
        recent = max(r.dual_objective for r in recs[-k:])
        before = max(r.dual_objective for r in recs[:-k])
        return recent - before < cfg.dual_tolerance * max(1.0, abs(bound))

    def _call_curv(self, lam, lam_prev, g, g_prev, s_p, y_p, act):
        self._call("dm_batch_curvature", lam.data_ptr(), lam_prev.data_ptr(), g.data_ptr(), g_prev.data_ptr(),
                   s_p.data_ptr(), y_p.data_ptr(), act.data_ptr())

    def _update(self, mode, x, u_list, coef, dot, alpha, alpha_out, active):
        dev = self.device
        u_p = _ptrs(u_list, dev)
        act = torch.as_tensor(np.asarray(active).astype(np.int8), device=dev)
        p = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        self._call("dm_batch_update", int(mode), x.data_ptr(), u_p.data_ptr(), p(coef), p(dot), p(alpha),
                   p(alpha_out), act.data_ptr())

    def _two_loop(self, g, d, rings, qn_on, pool_s, pool_y, dots, alphas):
        """lbfgs_direction per instance (qn.py:95-115) in the unfused order of
        qn.lbfgs_direction(fused=False), which equals the fused two-loop bit
        for bit: d = two-loop(g) on each QN-active instance's segment."""
        n, dev = self.n, self.device
        f64 = dict(dtype=torch.float64, device=dev)
        ms = [len(r) if qn_on[k] else 0 for k, r in enumerate(rings)]
        M = max(ms)
        self._update(0, d, [g] * n, None, None, None, None, qn_on)  # q = g.copy()
        rho = np.zeros((M, n))
        for i in range(M):
            act = np.array([i < ms[k] for k in range(n)])
            sl = [rings[k][i][0] if act[k] else 0 for k in range(n)]
            rho[i] = [rings[k][i][1] if act[k] else 0.0 for k in range(n)]
            s_p = _ptrs([pool_s[x] for x in sl], dev)
            d_p = _ptrs([d] * n, dev)
            a_t = torch.as_tensor(act.astype(np.int8), device=dev)
            self._call("dm_batch_dot", s_p.data_ptr(), d_p.data_ptr(), a_t.data_ptr(), dots[i].data_ptr())
            self._update(1, d, [pool_y[x] for x in sl], torch.as_tensor(rho[i], **f64), dots[i], None, alphas[i],
                         act)  # q -= (rho s.q) y
        act = np.array([ms[k] > 0 for k in range(n)])
        y0 = [pool_y[rings[k][0][0]] if act[k] else pool_y[0] for k in range(n)]
        y_p = _ptrs(y0, dev)
        a_t = torch.as_tensor(act.astype(np.int8), device=dev)
        self._call("dm_batch_dot", y_p.data_ptr(), y_p.data_ptr(), a_t.data_ptr(), dots[M].data_ptr())
        sy0 = torch.as_tensor([rings[k][0][2] if act[k] else 0.0 for k in range(n)], **f64)
        self._update(2, d, [d] * n, sy0, dots[M], None, None, act)  # d = (s0.y0 / y0.y0) q
        for j in range(M):
            act = np.array([j < ms[k] for k in range(n)])
            idx = [ms[k] - 1 - j if act[k] else 0 for k in range(n)]  # oldest first
            y_p = _ptrs([pool_y[rings[k][idx[k]][0]] if act[k] else pool_y[0] for k in range(n)], dev)
            d_p = _ptrs([d] * n, dev)
            a_t = torch.as_tensor(act.astype(np.int8), device=dev)
            self._call("dm_batch_dot", y_p.data_ptr(), d_p.data_ptr(), a_t.data_ptr(), dots[M + 1 + j].data_ptr())
            rho_j = torch.as_tensor([rings[k][idx[k]][1] if act[k] else 0.0 for k in range(n)], **f64)
            al = alphas[torch.as_tensor(idx, device=dev), torch.arange(n, device=dev)]
            self._update(3, d, [pool_s[rings[k][idx[k]][0]] if act[k] else pool_s[0] for k in range(n)], rho_j,
                         dots[M + 1 + j], al, None, act)  # d += s (alpha - rho y.d)


@dataclass
class BatchedResult:
    """One instance's part of a batched solve (qn.SolveResult's fields)."""

    records: list
    best_bound: float
    iterations: int
    stop_reason: str
    lam: np.ndarray

    @property
    def bounds(self) -> list:
        return [r.dual_objective for r in self.records]


def solve_batched(instances, cfg: SolveConfig | None = None, device=None, clock=time.perf_counter,
                  reuse_buffers: bool = False) -> list:
    """qn.solve for each instance, run together on one merged instance
    (BatchedSolver): per-instance results equal to separate solves."""
    return BatchedSolver(instances, cfg, device, clock, reuse_buffers).solve()
