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


def merge_instances(instances, threads: int = 8, reuse_buffers: bool = False,
                    into: FlatTable | None = None) -> tuple[IlpInstance, BatchIndex]:
    """Block-diagonal concatenation of lowered instances (their FlatTables):
    outputs preallocated, each instance's slices filled by a worker thread
    (numpy releases the GIL on these copies).  ``reuse_buffers`` refills the
    host arrays of the previous merge of the same sizes instead of faulting
    in gigabytes of fresh pages (the previous merged instance is then
    overwritten: a serving loop's staging arena).  ``into``: a larger merged
    table whose host arrays are no longer needed (a compaction's previous
    pack, already resident on the device) — the new table is written into
    prefixes of its arrays."""
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
    if into is not None and len(into.costs) >= V and len(into.zero_t) >= N and len(into.bdd_layer_lo) > nb \
            and len(into.layer_var) >= L:
        t = _prefix_table(into, V, nb, L, N)
    elif reuse_buffers and (V, nb, L, N) in _REUSE:
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


def _prefix_table(big: FlatTable, V, nb, L, N) -> FlatTable:
    t = FlatTable()
    for name, size in (("costs", V), ("variable_order", V), ("constraint_counts", V), ("bdd_layer_lo", nb + 1),
                       ("layer_node_lo", L + 1), ("layer_var", L), ("layer_bdd", L), ("zero_t", N), ("one_t", N),
                       ("proc_ptr", V + 1), ("proc_layers", L)):
        setattr(t, name, getattr(big, name)[:size])
    return t


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


class _Staging:
    """Host -> device staging of one iteration's small tables (pointer
    arrays, masks, per-instance coefficients): appended to a pinned host
    buffer, uploaded with ONE copy per ``flush``; ``put`` returns the device
    address the table will have."""

    def __init__(self, device, nbytes: int = 1 << 18):
        self.device = device
        self._alloc(nbytes)
        self.lo = self.hi = 0
        self.done = None

    def _alloc(self, nbytes):
        self.host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        self.hview = self.host.numpy()
        self.dev = torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    def reset(self, need: int = 0):
        """Start an iteration's tables (``need``: an upper bound of their bytes)."""
        if self.done is not None:
            self.done.synchronize()  # the last upload has left the host buffer
        if need > len(self.hview):
            self._alloc(2 * need)
        self.lo = self.hi = 0

    def put(self, arr) -> int:
        a = np.ascontiguousarray(arr)
        off = (self.hi + 15) & ~15
        if off + a.nbytes > len(self.hview):
            raise RuntimeError("staging buffer overflow (reset's size bound too small)")
        self.hview[off:off + a.nbytes] = a.reshape(-1).view(np.uint8)
        self.hi = off + a.nbytes
        return self.dev.data_ptr() + off

    def ptrs(self, tensors) -> int:
        return self.put(np.array([t.data_ptr() for t in tensors], dtype=np.int64))

    def flush(self, stream_ptr=None):
        if self.hi > self.lo:
            self.dev[self.lo:self.hi].copy_(self.host[self.lo:self.hi], non_blocking=True)
            self.done = torch.cuda.Event()
            self.done.record()
        self.lo = self.hi


class _Pack:
    """The live instances' merged block-diagonal instance and their device
    vectors (duals, L-BFGS pair pool, previous duals and subgradient).
    Built, then filled by ``start`` (a new batch) or ``adopt`` (a
    compaction)."""

    def __init__(self, solver, ids, reuse_buffers: bool = False, into: FlatTable | None = None):
        from .dual import DualState

        cfg, m = solver.cfg, solver.cfg.history_size
        self.m = m
        self.stream_ptr = solver.stream_ptr
        self.ids = list(ids)
        self.n = len(self.ids)
        c = time.perf_counter
        t0 = c()
        self.merged, self.index = merge_instances([solver.instances[i] for i in self.ids],
                                                  reuse_buffers=reuse_buffers, into=into)
        t1 = c()
        self.state = st = DualState(self.merged, device=solver.device, schedule=cfg.mma_schedule)
        t2 = c()
        f64 = dict(dtype=torch.float64, device=st.device)
        self.h = _Handle(st, self.index)
        self.phases = {"merge": t1 - t0, "state": t2 - t1, "handle": c() - t2}
        self.free_c = solver.free_c[self.ids]
        self.free_c_d = torch.as_tensor(self.free_c, **f64)
        self.sums = torch.empty(self.n, **f64)
        self.nb_scratch = torch.empty(self.merged.flat.num_bdds, **f64)
        self.state_d = torch.empty(8 * self.n, **f64)
        self.dots = torch.empty((2 * m + 1, self.n), **f64)
        self.alphas = torch.empty((m, self.n), **f64)
        self.d = torch.zeros(self.merged.flat.num_layers, **f64)
        self.d2 = torch.empty_like(self.d)

    def start(self):
        """init_duals (dual.py:137-144) and an empty pair pool."""
        from .dual import subgradient_device

        st = self.state
        costs = torch.as_tensor(np.ascontiguousarray(self.merged.costs, dtype=np.float64), device=st.device)
        st.dev.init_duals(costs, st.lam_d)
        st.refresh_backward()
        self.pool_s = [torch.empty_like(self.d) for _ in range(self.m + 1)]
        self.pool_y = [torch.empty_like(self.d) for _ in range(self.m + 1)]
        self.lam_prev = st.lam_d.clone()
        self.g_prev = subgradient_device(st).clone()
        return self

    def adopt(self, prev: "_Pack"):
        """Carry every instance's device vectors over from ``prev``, segment by
        segment (one gather per vector); the distance tables are rebuilt from
        the duals by the next pass."""
        pos = {k: p for p, k in enumerate(prev.ids)}
        src = np.concatenate([np.arange(prev.index.layer[pos[k]], prev.index.layer[pos[k] + 1]) for k in self.ids])
        src = torch.as_tensor(src, device=self.state.device)
        st = self.state
        st.lam_d.copy_(prev.state.lam_d[src])
        st.f_valid = st.b_valid = False
        self.lam_prev = prev.lam_prev[src]
        self.g_prev = prev.g_prev[src]
        self.pool_s = [t[src] for t in prev.pool_s]
        self.pool_y = [t[src] for t in prev.pool_y]
        return self

    def call(self, name, *args):
        from . import _native

        _native.call(name, self.h._h, *args, self.stream_ptr)

    def instance_sums(self):
        """Per-instance numpy-order sums of the per-diagram optima."""
        self.call("dm_batch_sum", self.state._bounds.data_ptr(), self.sums.data_ptr())
        return self.sums


class BatchedSolver:
    """Every instance's OWN hybrid ``qn.solve`` (qn.py:211-259), side by side
    on one merged block-diagonal instance: the averaging passes and sweeps run
    once for the batch, and each instance keeps its own L-BFGS history, step
    size, step search, curvature test and stopping rule, with reductions
    taken over its own ranges in the order a separate solve takes them
    (dm_batch.cu) — so every instance's bounds and duals are bit-identical to
    ``qn.solve(instance, cfg)`` (tests/test_batch.py).

    An instance whose stopping rule fires leaves the batch: its duals and
    records are snapshotted, and once at most a fraction ``compact`` of the
    merged instances is still live (or one; 0 = never), the live instances
    are re-merged into a smaller instance and their duals, curvature pairs,
    previous duals and subgradient carried over segment by segment — the
    passes then only walk live instances; the last one continues in its own
    ``qn.DualSolver`` loop.  Diagrams of different instances never interact,
    so the carried state continues each instance's trajectory unchanged."""

    def __init__(self, instances, cfg: SolveConfig | None = None, device=None, clock=time.perf_counter,
                 reuse_buffers: bool = False, compact: float = 0.25):
        self.instances = list(instances)
        self.cfg = cfg or SolveConfig()
        if self.cfg.mode != "hybrid":
            raise ValueError("BatchedSolver runs hybrid solves (mode='mma-only' batches: solve_merged)")
        self.clock = clock
        self.compact = compact
        self.t0 = clock()
        self.n = len(self.instances)
        self.free_c = np.array([float(np.minimum(i.costs[i.unconstrained_variables()], 0.0).sum())
                                for i in self.instances])
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())
        self.stream_ptr = torch.cuda.current_stream(self.device).cuda_stream
        self.pack = _Pack(self, range(self.n), reuse_buffers=reuse_buffers).start()
        self.repacks = 0
        self.arc_updates = 0
        self.pack_phases = [(self.n, self.pack.phases)]
        self.trace = [(0, self.n, self.n, clock() - self.t0)]  # (iteration, pack size, live, seconds)

    # -- the solve -----------------------------------------------------------------
    def solve(self):
        from . import _native
        from .dual import BACKWARD, FORWARD, mma_pass, subgradient_device
        from .qn import IterationRecord, StepConfig

        cfg, n = self.cfg, self.n
        m = cfg.history_size
        scfg = StepConfig.from_solve_config(cfg)
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
        stage = _Staging(self.device)
        pk = self.pack

        def note(ids, vals, mask):
            for p in np.flatnonzero(mask):
                k = ids[p]
                bound[k] = vals[p] + self.free_c[k]
                best[k] = max(best[k], bound[k])

        every = np.ones(n, bool)
        note(pk.ids, pk.instance_sums().cpu().numpy(), every)  # init_duals' refresh (dual.py:137-144)
        t = self.clock() - self.t0
        for k in range(n):
            records[k].append(IterationRecord(0, "init", bound[k], t))
        initial = bound.copy()
        for it in range(1, cfg.max_iterations + 1):
            st, ids, np_ = pk.state, np.asarray(pk.ids), pk.n
            live = ~stopped[ids]
            qn_on = live & np.array([len(rings[k]) > 0 for k in ids])
            used = np.zeros(np_, bool)
            stage.reset((4 * m + 16) * (25 * np_ + 64))
            # this iteration's tables, known up front: the two-loop's, the step
            # search's and the curvature pair's
            loop = self._stage_two_loop(stage, pk, rings, qn_on) if qn_on.any() else None
            slots = [free_slots[k][-1] if live[p] else 0 for p, k in enumerate(ids)]
            curv = (stage.ptrs([pk.pool_s[s] for s in slots]), stage.ptrs([pk.pool_y[s] for s in slots]),
                    stage.put(live.astype(np.int8)))
            if loop is not None:
                srch = (stage.put(gamma[ids]), stage.put(min_ascent[ids]), stage.put(qn_on.astype(np.int8)))
            stage.flush()
            if loop is not None:
                # g = the subgradient cached at the end of the last iteration (qn.py:201,249)
                self._run_two_loop(pk, pk.g_prev, pk.d, loop)
                st.dev.project_direction(pk.d, pk.d2)  # per variable: independent per instance
                d = pk.d2
                _native.call("dm_batch_step_search", st.dev.handle, pk.h._h, st.lam_d.data_ptr(), d.data_ptr(),
                             srch[0], pk.free_c_d.data_ptr(), srch[1], float(scfg.shrink), float(scfg.grow),
                             int(scfg.max_trials), srch[2], pk.nb_scratch.data_ptr(), pk.sums.data_ptr(),
                             pk.state_d.data_ptr(), self.stream_ptr)
                ctl = pk.state_d.cpu().numpy().reshape(np_, 8)
                st.sweeps += int(ctl[qn_on, 6].max())
                for p in np.flatnonzero(qn_on):
                    k = ids[p]
                    gamma[k] = ctl[p, 3]  # qn.py:159 returns the best trial's step
                    used[p] = ctl[p, 2] > bound[k]
                if used.any():
                    coef = stage.put(np.where(used, gamma[ids], 0.0))
                    act = stage.put(used.astype(np.int8))
                    u = stage.ptrs([d] * np_)
                    stage.flush()
                    pk.call("dm_batch_update", 4, st.lam_d.data_ptr(), u, coef, None, None, None, act)
                    st.f_valid = st.b_valid = False
                    st.refresh_backward()  # the averaging pass's refresh (dual.py:164-165), all at once
                    note(ids, pk.instance_sums().cpu().numpy(), used)
            if st.deferred:
                st.deferred_round(cfg.mma_damping)
                note(ids, pk.instance_sums().cpu().numpy(), live)
            else:
                mma_pass(st, FORWARD)
                fw = pk.instance_sums().clone()
                mma_pass(st, BACKWARD)
                both = torch.stack([fw, pk.instance_sums()]).cpu().numpy()
                note(ids, both[0], live)
                note(ids, both[1], live)
            g_now = subgradient_device(st).clone()
            # curvature pair into each live instance's free slot, and s . y per instance
            pk.call("dm_batch_curvature", st.lam_d.data_ptr(), pk.lam_prev.data_ptr(), g_now.data_ptr(),
                    pk.g_prev.data_ptr(), curv[0], curv[1], curv[2])
            pk.call("dm_batch_dot", curv[0], curv[1], curv[2], pk.sums.data_ptr())
            sy = pk.sums.cpu().numpy()
            st.read_scalars()  # the passes' watchdog word (raises if an exact pass was aborted)
            pk.g_prev = g_now
            t = self.clock() - self.t0
            for p in np.flatnonzero(live):
                k = ids[p]
                iters[k] = it
                records[k].append(IterationRecord(it, "hybrid" if used[p] else "mma", bound[k], t))
                if it == 1:
                    min_ascent[k] = cfg.ascent_rel_threshold * (bound[k] - initial[k])
                if sy[p] >= scfg.curvature_eps:  # qn.py:85-92
                    slot = free_slots[k].pop()
                    rings[k].insert(0, (slot, 1.0 / sy[p], float(sy[p])))
                    if len(rings[k]) > m:
                        free_slots[k].append(rings[k].pop()[0])
                if self._tolerance_met(records[k], bound[k], it, cfg):
                    stop_reason[k] = "dual_tolerance"
                elif cfg.max_seconds is not None and t > cfg.max_seconds:
                    stop_reason[k] = "max_seconds"
                else:
                    continue
                stopped[k] = True
                lo, hi = pk.index.layer[p], pk.index.layer[p + 1]
                lam_final[k] = st.lam_d[lo:hi].cpu().numpy()
            self.trace.append((it, pk.n, int(live.sum()), t))
            if stopped.all():
                break
            n_live = int((~stopped[ids]).sum())
            if self.compact and n_live < np_ and (n_live <= self.compact * np_ or n_live == 1):
                # the old pack's host tables are dead weight once it is on the device: reused
                new = _Pack(self, [k for k in ids if not stopped[k]], into=pk.merged.flat).adopt(pk)
                self.arc_updates += st.arc_updates
                c = time.perf_counter()
                pk = self.pack = new
                del st, new
                torch.cuda.synchronize(self.device)
                pk.phases["drop"] = time.perf_counter() - c
                self.pack_phases.append((pk.n, pk.phases))
                self.repacks += 1
            if self.compact and pk.n == 1:
                k = pk.ids[0]  # the last live instance: its own solver loop from here (fused two-loop)
                run = self._alone(pk, records[k], rings[k], gamma[k], min_ascent[k], initial[k], it)
                while run.iterations < cfg.max_iterations:
                    reason = run.step()
                    if reason is not None:
                        stop_reason[k] = reason
                        break
                iters[k] = run.iterations
                best[k] = max(best[k], run.state.best_bound)
                stopped[k] = True
                lam_final[k] = pk.state.lam
                self.trace.append((run.iterations, 1, 1, self.clock() - self.t0))
                break
        self.arc_updates += pk.state.arc_updates
        for k in np.flatnonzero(~stopped):
            p = pk.ids.index(k)
            lo, hi = pk.index.layer[p], pk.index.layer[p + 1]
            lam_final[k] = pk.state.lam_d[lo:hi].cpu().numpy()
        return [BatchedResult(records[k], float(best[k]), int(iters[k]), stop_reason[k], lam_final[k])
                for k in range(n)]

    def _alone(self, pk, recs, ring, gamma, min_ascent, initial, it):
        """A qn.DualSolver continuing a one-instance pack's solve after
        iteration ``it``: the carried duals, curvature pairs (oldest pushed
        first), step size, ascent threshold and records; the subgradient of
        the current duals is the carried one (the last pass's decisions)."""
        from .qn import DualSolver, LbfgsHistory, StepConfig

        st = pk.state
        run = DualSolver(self.instances[pk.ids[0]], self.cfg, self.clock, self.device, st)
        run.t0 = self.t0
        run.state = st
        run.step_cfg = StepConfig.from_solve_config(self.cfg)
        run.step_cfg.min_ascent = min_ascent
        run.history = LbfgsHistory(run.step_cfg.memory)
        for slot, rho, sy in reversed(ring):
            run.history.push(pk.pool_s[slot], pk.pool_y[slot], rho, sy)
        run.records = recs
        run.initial_bound = initial
        run.lam_prev = pk.lam_prev
        st.refresh_backward()
        st._argmin_cache = (st._bgen, pk.g_prev)
        run.g_prev = pk.g_prev
        run.gamma = gamma
        run.iterations = it
        return run

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

    @staticmethod
    def _stage_two_loop(stage, pk, rings, qn_on):
        """The two-loop's per-step tables (qn.py:95-115, qn.lbfgs_direction's
        unfused order): per step, the pair pointers, the active mask and rho."""
        n, ids = pk.n, pk.ids
        ms = [len(rings[k]) if qn_on[p] else 0 for p, k in enumerate(ids)]
        M = max(ms)
        d_p = stage.ptrs([pk.d] * n)
        g_p = stage.ptrs([pk.g_prev] * n)
        first = []
        for i in range(M):  # newest first
            act = np.array([i < ms[p] for p in range(n)])
            sl = [rings[ids[p]][i][0] if act[p] else 0 for p in range(n)]
            rho = np.array([rings[ids[p]][i][1] if act[p] else 0.0 for p in range(n)])
            first.append((stage.ptrs([pk.pool_s[x] for x in sl]), stage.ptrs([pk.pool_y[x] for x in sl]),
                          stage.put(act.astype(np.int8)), stage.put(rho)))
        act0 = np.array([ms[p] > 0 for p in range(n)])
        y0 = stage.ptrs([pk.pool_y[rings[ids[p]][0][0]] if act0[p] else pk.pool_y[0] for p in range(n)])
        sy0 = stage.put(np.array([rings[ids[p]][0][2] if act0[p] else 0.0 for p in range(n)]))
        mid = (y0, sy0, stage.put(act0.astype(np.int8)))
        second = []
        for j in range(M):  # oldest first
            act = np.array([j < ms[p] for p in range(n)])
            idx = np.array([ms[p] - 1 - j if act[p] else 0 for p in range(n)])
            sl = [rings[ids[p]][idx[p]][0] if act[p] else 0 for p in range(n)]
            rho = np.array([rings[ids[p]][idx[p]][1] if act[p] else 0.0 for p in range(n)])
            second.append((stage.ptrs([pk.pool_s[x] for x in sl]), stage.ptrs([pk.pool_y[x] for x in sl]),
                           stage.put(act.astype(np.int8)), stage.put(rho), idx))
        return d_p, g_p, qn_on.astype(np.int8), stage.put(qn_on.astype(np.int8)), first, mid, second

    @staticmethod
    def _run_two_loop(pk, g, d, loop):
        """d = two-loop(g) on each QN-active instance's segment."""
        d_p, g_p, _, on, first, (y0, sy0, act0), second = loop
        dots, alphas = pk.dots, pk.alphas
        stride = alphas.stride(0) * 8
        pk.call("dm_batch_update", 0, d.data_ptr(), g_p, None, None, None, None, on)  # q = g.copy()
        for i, (s_p, y_p, act, rho) in enumerate(first):
            pk.call("dm_batch_dot", s_p, d_p, act, dots[i].data_ptr())
            pk.call("dm_batch_update", 1, d.data_ptr(), y_p, rho, dots[i].data_ptr(), None,
                    alphas.data_ptr() + i * stride, act)  # q -= (rho s.q) y
        M = len(first)
        pk.call("dm_batch_dot", y0, y0, act0, dots[M].data_ptr())
        pk.call("dm_batch_update", 2, d.data_ptr(), d_p, sy0, dots[M].data_ptr(), None, None, act0)
        # d = (s0.y0 / y0.y0) q
        for j, (s_p, y_p, act, rho, idx) in enumerate(second):
            pk.call("dm_batch_dot", y_p, d_p, act, dots[M + 1 + j].data_ptr())
            al = alphas[torch.as_tensor(idx, device=alphas.device), torch.arange(pk.n, device=alphas.device)]
            pk.call("dm_batch_update", 3, d.data_ptr(), s_p, rho, dots[M + 1 + j].data_ptr(), al.data_ptr(), None,
                    act)  # d += s (alpha - rho y.d)
            del al


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
                  reuse_buffers: bool = False, compact: float = 0.25) -> list:
    """qn.solve for each instance, run together on one merged instance
    (BatchedSolver): per-instance results equal to separate solves."""
    return BatchedSolver(instances, cfg, device, clock, reuse_buffers, compact).solve()
