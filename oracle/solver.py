"""ORACLE — TEST INFRASTRUCTURE ONLY.

Restatement of the reference dual state and quasi-Newton loop
(/root/reference/pkg/src/prodmatch/dual.py:33-201, qn.py:30-259) and of the
agreement scores (primal.py:83-111) on top of the C kernels in ckernels.c.

Reductions: the reference sums per-diagram optima with ``ndarray.sum``
(numpy pairwise summation, dual.py:67,106) — reused here unchanged.  Its
inner products go through OpenBLAS ``ddot`` (qn.py:89,107,111,113), whose
summation order depends on the host's thread count; ``dot="blas"`` keeps
that (used to pin against the reference), ``dot="chunked"`` uses the
B200 path's fixed order (numpy pairwise per 4096-element chunk, then over
the chunk totals) so GPU and oracle agree bit-for-bit in hybrid mode too.
"""

from __future__ import annotations

import time
from collections import deque

import numpy as np

from .clib import lib, ptr
from .model import OracleFlat, OracleInstance, flatten

INF = np.inf


def _dot_blas(a, b):
    return float(a @ b)


DOT_CHUNK = 4096


def _dot_chunked(a, b):
    """The B200 path's inner-product order (csrc/dm_sweep.cu chunk_dot):
    numpy pairwise over 4096-element chunks of a*b, then numpy pairwise over
    the chunk totals."""
    p = a * b
    n = len(p)
    if n == 0:
        return 0.0
    full = n // DOT_CHUNK
    sums = list(np.sum(p[: full * DOT_CHUNK].reshape(-1, DOT_CHUNK), axis=1)) if full else []
    if n % DOT_CHUNK:
        sums.append(np.sum(p[full * DOT_CHUNK:]))
    return float(np.sum(np.asarray(sums, dtype=np.float64)))


_dot_pairwise = _dot_chunked  # name kept for callers of the previous order


class OracleDual:
    """dual.py:33-134 — duals, cached distances and validity flags."""

    def __init__(self, inst: OracleInstance, flat: OracleFlat | None = None):
        self.inst = inst
        self.flat = flat if flat is not None else flatten(inst)
        f = self.flat
        self.lam = np.zeros(f.num_layers)
        self.F = np.zeros(f.num_nodes)
        self.B = np.zeros(f.num_nodes)
        self.bounds = np.zeros(f.num_bdds)
        self.m0s = np.zeros(max(f.max_degree, 1))
        self.m1s = np.zeros(max(f.max_degree, 1))
        self.scratch = np.zeros(f.num_nodes)
        self.f_valid = self.b_valid = False
        self.bound = -INF
        self.best_bound = -INF
        self.counts = inst.counts()
        free = np.flatnonzero(self.counts == 0)
        self.free_values = {int(v): (0 if inst.costs[v] >= 0 else 1) for v in free}
        self.free_contribution = float(np.minimum(inst.costs[free], 0.0).sum()) if len(free) else 0.0
        self.sweeps = 0  # full-diagram sweeps executed (for arc-update accounting)

    # dual.py:66-69
    def _set_bound(self):
        self.bound = float(self.bounds.sum()) + self.free_contribution
        if self.bound > self.best_bound:
            self.best_bound = self.bound

    def refresh_backward(self):
        f = self.flat
        lib.oracle_k_backward(f.num_bdds, ptr(f.bdd_layer_lo), ptr(f.layer_node_lo), ptr(f.zero_t),
                              ptr(f.one_t), ptr(self.lam), ptr(self.B), ptr(self.bounds))
        self.sweeps += 1
        self.b_valid = True
        self._set_bound()

    def refresh_forward(self):
        f = self.flat
        lib.oracle_k_forward(f.num_bdds, ptr(f.bdd_layer_lo), ptr(f.layer_node_lo), ptr(f.zero_t),
                             ptr(f.one_t), ptr(self.lam), ptr(self.F), ptr(self.bounds))
        self.sweeps += 1
        self.f_valid = True
        self._set_bound()

    def shift(self, delta):
        self.lam += delta
        self.f_valid = self.b_valid = False

    def set_lambda(self, lam):
        lam = np.asarray(lam, np.float64)
        if lam.shape != self.lam.shape:
            raise ValueError("dual vector length mismatch")
        self.lam[:] = lam
        self.f_valid = self.b_valid = False
        self.refresh_backward()

    def eval_trial(self, d, gamma):
        """dual.py:99-106 on lam + gamma*d (qn.py:147,153), caches untouched."""
        f = self.flat
        b = np.zeros(f.num_bdds)
        lib.oracle_k_backward_trial(f.num_bdds, ptr(f.bdd_layer_lo), ptr(f.layer_node_lo),
                                    ptr(f.zero_t), ptr(f.one_t), ptr(self.lam), ptr(d),
                                    float(gamma), ptr(self.scratch), ptr(b))
        self.sweeps += 1
        return float(b.sum()) + self.free_contribution

    def objective(self):
        """dual.py:147-151"""
        if not (self.b_valid or self.f_valid):
            self.refresh_backward()
        return self.bound

    def mma(self, forward: bool):
        """dual.py:154-186"""
        f = self.flat
        args = (f.num_bdds, len(f.proc_ptr) - 1, ptr(f.bdd_layer_lo), ptr(f.layer_node_lo),
                ptr(f.layer_bdd), ptr(f.zero_t), ptr(f.one_t), ptr(f.proc_ptr), ptr(f.proc_layers),
                ptr(self.lam), ptr(self.F), ptr(self.B), ptr(self.bounds), ptr(self.m0s), ptr(self.m1s))
        if forward:
            if not self.b_valid:
                self.refresh_backward()
            lib.oracle_k_mma_forward(*args)
            self.f_valid, self.b_valid = True, False
        else:
            if not self.f_valid:
                self.refresh_forward()
            lib.oracle_k_mma_backward(*args)
            self.f_valid, self.b_valid = False, True
        self.sweeps += 2
        self._set_bound()

    def deferred_round(self, omega):
        """The B200 path's deferred (FastDOG) averaging round
        (DualState.deferred_round, csrc/dm_deferred.cu) on node-order tables:
        forward pass (escrow), average, backward pass (adds it, new escrow),
        average, flush sweep."""
        f = self.flat
        if not self.b_valid:
            self.refresh_backward()
        P = len(f.proc_ptr) - 1
        mbar = np.zeros(f.num_layers)
        avg = np.zeros(f.num_layers)
        geo = (f.num_bdds, ptr(f.bdd_layer_lo), ptr(f.layer_node_lo), ptr(f.zero_t), ptr(f.one_t))
        lib.oracle_dfr_forward(*geo, float(omega), ptr(self.lam), None, ptr(self.B), ptr(self.F), ptr(mbar),
                               ptr(self.bounds))
        lib.oracle_dfr_average(P, ptr(f.proc_ptr), ptr(f.proc_layers), ptr(mbar), ptr(avg))
        lib.oracle_dfr_backward(*geo, float(omega), ptr(self.lam), ptr(avg), ptr(self.F), ptr(self.B), ptr(mbar),
                                ptr(self.bounds))
        lib.oracle_dfr_average(P, ptr(f.proc_ptr), ptr(f.proc_layers), ptr(mbar), ptr(avg))
        lib.oracle_dfr_backward(*geo, 0.0, ptr(self.lam), ptr(avg), None, ptr(self.B), None, ptr(self.bounds))
        self.sweeps += 5
        self.f_valid, self.b_valid = False, True
        self._set_bound()
        return mbar, avg

    def subgradient(self):
        """dual.py:189-201"""
        f = self.flat
        if not self.b_valid:
            self.refresh_backward()
        bits = np.zeros(f.num_layers)
        lib.oracle_k_argmin(f.num_bdds, ptr(f.bdd_layer_lo), ptr(f.layer_node_lo), ptr(f.zero_t),
                            ptr(f.one_t), ptr(self.lam), ptr(self.B), ptr(bits))
        return bits

    def min_marginals(self):
        """dual.py:121-134"""
        f = self.flat
        if not self.f_valid:
            self.refresh_forward()
        if not self.b_valid:
            self.refresh_backward()
        m0 = np.zeros(f.num_layers)
        m1 = np.zeros(f.num_layers)
        lib.oracle_k_min_marginals(f.num_layers, ptr(f.layer_node_lo), ptr(f.zero_t), ptr(f.one_t),
                                   ptr(self.lam), ptr(self.F), ptr(self.B), ptr(m0), ptr(m1))
        return m0, m1

    def lambda_sums(self):
        """dual.py:114-119"""
        out = np.zeros(self.inst.num_variables)
        np.add.at(out, self.flat.layer_var, self.lam)
        fv = list(self.free_values)
        out[fv] = self.inst.costs[fv]
        return out


def init_duals(inst: OracleInstance, flat: OracleFlat | None = None) -> OracleDual:
    """dual.py:137-144"""
    st = OracleDual(inst, flat)
    lv = st.flat.layer_var
    st.lam[:] = inst.costs[lv] / st.counts[lv]
    st.refresh_backward()
    return st


def project(d_hat, st: OracleDual):
    """qn.py:118-129"""
    lv = st.flat.layer_var
    sums = np.bincount(lv, weights=d_hat, minlength=st.inst.num_variables)
    return d_hat - (sums / np.maximum(st.counts, 1))[lv]


def lbfgs(g, pairs, dot):
    """qn.py:95-115 two-loop recursion; ``pairs`` newest first (s, y, rho, sy)."""
    q = np.array(g, dtype=np.float64, copy=True)
    alphas = []
    for s, y, rho, _ in pairs:
        a = rho * dot(s, q)
        q -= a * y
        alphas.append(a)
    s0, y0, _, _ = pairs[0]
    d = (dot(s0, y0) / dot(y0, y0)) * q
    for (s, y, rho, _), a in zip(reversed(pairs), reversed(alphas)):
        b = rho * dot(y, d)
        d += s * (a - b)
    return d


def step_search(st: OracleDual, d, gamma_prev, shrink, grow, trials, min_ascent):
    """qn.py:132-159"""
    base = st.objective()
    gamma = float(gamma_prev)
    e_init = st.eval_trial(d, gamma)
    g_best, e_best, e_cur = gamma, e_init, e_init
    for _ in range(trials):
        gamma *= shrink if e_cur <= e_init else grow
        e_cur = st.eval_trial(d, gamma)
        if e_cur >= e_best:
            g_best, e_best = gamma, e_cur
        if e_cur - e_init >= min_ascent:
            break
    return g_best, bool(e_best > base)


def solve(inst: OracleInstance, mode="hybrid", max_iterations=2000, dual_tolerance=1e-10,
          curvature_eps=1e-8, grow=1.1, shrink=0.8, trials=5, ascent_rel=1e-6,
          initial_step=1.0, memory=10, max_seconds=None, dot="blas", flat=None,
          clock=time.perf_counter, threads=None, schedule="exact", damping=0.5, stall_window=None):
    """qn.py:184-259; returns (state, records[(it, kind, bound, t)], stop_reason).
    ``schedule="deferred"`` replaces the two exact passes of every iteration by
    the B200 path's deferred averaging round (OracleDual.deferred_round)."""
    if threads is not None:
        lib.oracle_set_threads(int(threads))
    dotf = _dot_blas if dot == "blas" else _dot_chunked
    hybrid = mode == "hybrid"
    t0 = clock()
    st = init_duals(inst, flat)
    hist = deque(maxlen=memory)  # newest first
    records = [(0, "init", st.objective(), clock() - t0)]
    first = records[0][2]
    min_ascent = 0.0
    lam_prev = st.lam.copy()
    g_prev = st.subgradient()
    gamma = initial_step
    reason = "max_iterations"
    for it in range(1, max_iterations + 1):
        used = False
        if hybrid and len(hist) > 0:
            g = st.subgradient()
            d = project(lbfgs(g, list(hist), dotf), st)
            gamma, better = step_search(st, d, gamma, shrink, grow, trials, min_ascent)
            if better:
                st.shift(gamma * d)
                used = True
        if schedule == "deferred":
            st.deferred_round(damping)
        else:
            st.mma(True)
            st.mma(False)
        bound = st.objective()
        records.append((it, "hybrid" if used else "mma", bound, clock() - t0))
        if it == 1:
            min_ascent = ascent_rel * (bound - first)
        if hybrid:
            g_now = st.subgradient()
            s = st.lam - lam_prev
            y = g_prev - g_now
            sy = dotf(s, y)
            if sy >= curvature_eps:
                hist.appendleft((s, y, 1.0 / sy, sy))
            lam_prev = st.lam.copy()
            g_prev = g_now
        k = stall_window if stall_window is not None else (32 if schedule == "deferred" else 1)
        if k == 1:
            if bound - records[-2][2] < dual_tolerance * max(1.0, abs(bound)):
                reason = "dual_tolerance"
                break
        elif it >= k:  # best-bound gain over the last k iterations (SolveConfig.stall_window)
            recent = max(r[2] for r in records[-k:])
            before = max(r[2] for r in records[:-k])
            if recent - before < dual_tolerance * max(1.0, abs(bound)):
                reason = "dual_tolerance"
                break
        if max_seconds is not None and clock() - t0 > max_seconds:
            reason = "max_seconds"
            break
    return st, records, reason


def agreement_scores(st: OracleDual):
    """primal.py:83-111 -> (agrees, score, preferred)."""
    m0, m1 = st.min_marginals()
    diff = np.empty_like(m0)
    both = np.isfinite(m0) & np.isfinite(m1)
    diff[both] = m1[both] - m0[both]
    diff[np.isinf(m1) & ~np.isinf(m0)] = np.inf
    diff[np.isinf(m0) & ~np.isinf(m1)] = -np.inf
    nv = st.inst.num_variables
    vote = np.sign(diff)
    vmax = np.full(nv, -2.0)
    vmin = np.full(nv, 2.0)
    lv = st.flat.layer_var
    np.maximum.at(vmax, lv, vote)
    np.minimum.at(vmin, lv, vote)
    agrees = (vmax == vmin) & (vmax != 0.0) & (st.counts > 0)
    total = np.zeros(nv)
    np.add.at(total, lv, diff)
    score = np.abs(np.nan_to_num(total, nan=0.0, posinf=np.inf, neginf=-np.inf))
    preferred = np.where(vmax > 0, 0, 1).astype(np.int8)
    return agrees, score, preferred


# ---------------------------------------------------------------------------
# Perturbation rounding (restates paper_2310_08230_b200/rounding.py and the
# dm_perturb_round kernel, csrc/dm_device.cu: same votes, same splitmix64
# hash, same roundings) — for the GPU-vs-oracle rounding test.
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(seed, rnd, v):
    """splitmix64 of (seed, round, variable ids v) as uint64 numpy."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * (
            (np.uint64(rnd & 0xFFFFFFFF) << np.uint64(32)) + np.asarray(v, np.uint64) + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def perturb_round(st: OracleDual, delta, seed, rnd, boost=10.0):
    """One round on fresh min-marginals: returns (values, agrees, disagree
    count) and moves st.lam (caches invalidated)."""
    m0, m1 = st.min_marginals()
    f = st.flat
    nv = st.inst.num_variables
    values = np.zeros(nv, np.int8)
    agrees = np.zeros(nv, np.int8)
    dis = 0
    for p in range(len(f.proc_ptr) - 1):
        lo, hi = int(f.proc_ptr[p]), int(f.proc_ptr[p + 1])
        if hi == lo:
            continue
        ls = f.proc_layers[lo:hi]
        vmax, vmin, total = -2.0, 2.0, 0.0
        for l in ls:
            a, b = m0[l], m1[l]
            fa, fb = a != INF, b != INF
            diff = (b - a) if (fa and fb) else (INF if fa else -INF)
            vote = 1.0 if diff > 0.0 else (-1.0 if diff < 0.0 else 0.0)
            vmax, vmin = max(vmax, vote), min(vmin, vote)
            total = total + diff
        v = int(f.layer_var[ls[0]])
        agree = vmax == vmin and vmax != 0.0
        h = int(mix64(seed, rnd, v))
        if agree:
            d = vmax
        elif total > 0.0:
            d = 1.0
        elif total < 0.0:
            d = -1.0
        else:
            d = 1.0 if (h >> 10) & 1 else -1.0
        u = float(h >> 11) * 2.0 ** -53
        mag = delta * boost if agree else delta
        share = ((d * mag) * (1.0 + u)) / float(hi - lo)
        st.lam[ls] = st.lam[ls] + share
        values[v] = 0 if d > 0.0 else 1
        agrees[v] = agree
        dis += not agree
    st.f_valid = st.b_valid = False
    return values, agrees, dis
