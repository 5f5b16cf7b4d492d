"""Flat diagram table (FlatBdds, kernels.py:35-92 of the reference) and its
device-resident twin.

``FlatBdds(instance)`` exposes the same int64 host arrays as the reference;
``FlatBdds.device()`` uploads them once (int32 SoA + the level schedules of
the exact averaging passes) and returns a ``DeviceFlat`` whose methods are
the reference kernels (k_backward, k_forward, k_mma_forward,
k_mma_backward, k_min_marginals, k_argmin) on torch CUDA tensors.  Every
call goes through the C-ABI of libdiscomatch_b200.so; there is no CPU path.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .errors import NativeLibraryError
from .ilp import FlatTable, IlpInstance, _lower_bdds


def set_threads(n: int) -> int:
    """Reference knob (kernels.py:27-32); the device path has no host threads."""
    return max(1, int(n))


def _ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("device vectors must be contiguous")
    return t.data_ptr()


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class DeviceFlat:
    """dm_flat handle: topology + schedules resident in HBM."""

    def __init__(self, table: FlatTable, device: torch.device, exact_plans: bool = True):
        if not torch.cuda.is_available():
            raise NativeLibraryError("a CUDA device is required (there is no CPU path)")
        self.device = torch.device(device)
        self.table = table
        lib = _native.load()
        desc = _native.FlatDesc()
        desc.num_bdds = table.num_bdds
        desc.num_layers = table.num_layers
        desc.num_nodes = table.num_nodes
        desc.num_positions = len(table.proc_ptr) - 1
        keep = {}
        for name in ("bdd_layer_lo", "layer_node_lo", "layer_var", "zero_t", "one_t", "proc_ptr", "proc_layers"):
            a = np.ascontiguousarray(getattr(table, name), dtype=np.int64)
            keep[name] = a
            setattr(desc, name, a.ctypes.data)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(lib.dm_flat_create_ex(ctypes.byref(desc), self.device.index or 0, _stream(self.device),
                                                0 if exact_plans else 1, ctypes.byref(h)), "dm_flat_create")
        self._h = h
        self.exact_plans = exact_plans
        info = _native.FlatInfo()
        _native.check(lib.dm_flat_get_info(h, ctypes.byref(info)), "dm_flat_get_info")
        self.info = {k: getattr(info, k) for k, _ in _native.FlatInfo._fields_}
        self.num_bdds, self.num_layers, self.num_nodes = table.num_bdds, table.num_layers, table.num_nodes
        self.num_positions = desc.num_positions

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _native.load().dm_flat_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def _s(self) -> int:
        return _stream(self.device)

    # --- reference kernels -------------------------------------------------
    def k_backward(self, lam, B, bounds):
        _native.call("dm_k_backward", self._h, _ptr(lam), _ptr(B), _ptr(bounds), self._s())

    def qn_move(self, lam, d, base, state, out, B, bounds):
        """Device-side quasi-Newton move + gated refresh of B (dm_qn_move)."""
        _native.call("dm_qn_move", self._h, _ptr(lam), _ptr(d), float(base), _ptr(state), _ptr(out), _ptr(B),
                     _ptr(bounds), self._s())

    def k_backward_trial(self, lam, d, gamma, B, bounds):
        _native.call("dm_k_backward_trial", self._h, _ptr(lam), _ptr(d), float(gamma), _ptr(B), _ptr(bounds),
                     self._s())

    def step_search(self, lam, d, gamma_prev, free_contribution, shrink, grow, min_ascent, max_trials, bounds,
                    state):
        """The whole find_step_size trial sequence on the device (dm_step_search)."""
        sweep_launches = 3  # per trial: sweep, pairwise leaves, pairwise combine + decision
        _native.call("dm_step_search", self._h, _ptr(lam), _ptr(d), float(gamma_prev), float(free_contribution),
                     float(shrink), float(grow), float(min_ascent), int(max_trials), _ptr(bounds), _ptr(state),
                     self._s(), launches=1 + sweep_launches * (int(max_trials) + 1))

    def k_forward(self, lam, F, bounds):
        _native.call("dm_k_forward", self._h, _ptr(lam), _ptr(F), _ptr(bounds), self._s())

    def k_mma_forward(self, lam, F, B, bounds):
        _native.call("dm_k_mma_forward", self._h, _ptr(lam), _ptr(F), _ptr(B), _ptr(bounds), self._s())

    def k_mma_backward(self, lam, F, B, bounds):
        _native.call("dm_k_mma_backward", self._h, _ptr(lam), _ptr(F), _ptr(B), _ptr(bounds), self._s())

    def set_mma_config(self, threads: int = 256, blocks_per_sm: int = 3, sleep_ns: int = 32, probe: bool = False,
                       lookahead: int = 1 << 16):
        """Launch shape of the exact passes (see dm_flat_set_mma_config)."""
        _native.call("dm_flat_set_mma_config", self._h, int(threads), int(blocks_per_sm), int(sleep_ns), int(probe),
                     int(lookahead))
        info = _native.FlatInfo()
        _native.check(_native.load().dm_flat_get_info(self._h, ctypes.byref(info)), "dm_flat_get_info")
        self.info = {k: getattr(info, k) for k, _ in _native.FlatInfo._fields_}

    def check_status(self):
        """Raise if an exact pass was aborted by its watchdog (synchronises)."""
        _native.call("dm_flat_status", self._h, self._s())

    def status_to(self, slot):
        """Watchdog word -> device double, stream-ordered (no synchronisation)."""
        _native.call("dm_flat_status_to", self._h, _ptr(slot), self._s())

    def k_min_marginals(self, lam, F, B, m0, m1):
        _native.call("dm_k_min_marginals", self._h, _ptr(lam), _ptr(F), _ptr(B), _ptr(m0), _ptr(m1), self._s())

    def k_argmin(self, lam, B, bits):
        _native.call("dm_k_argmin", self._h, _ptr(lam), _ptr(B), _ptr(bits), self._s())

    def k_argmin_from_pass(self, B, bits):
        """Argmin walk from the decisions of the last node-parallel backward pass."""
        _native.call("dm_k_argmin_from_pass", self._h, _ptr(B), _ptr(bits), self._s())

    @property
    def records_decisions(self) -> bool:
        """Whether the exact backward pass records argmin decisions (node-parallel kernels)."""
        return int(self.info.get("lanes_per_task", 32)) == 8

    # --- deferred (throughput) averaging schedule: dm_dfr_* ------------------
    def dfr_table_size(self) -> int:
        n = ctypes.c_int64()
        _native.check(_native.load().dm_dfr_table_size(self._h, ctypes.byref(n)), "dm_dfr_table_size")
        return int(n.value)

    def dfr_forward(self, omega, lam, avg, B_il, F_il, mbar, bounds):
        _native.call("dm_dfr_forward", self._h, float(omega), _ptr(lam), _ptr(avg), _ptr(B_il), _ptr(F_il),
                     _ptr(mbar), _ptr(bounds), self._s())

    def dfr_backward(self, omega, lam, avg, F_il, B_il, mbar, bounds, record_decisions=False):
        _native.call("dm_dfr_backward", self._h, float(omega), _ptr(lam), _ptr(avg), _ptr(F_il), _ptr(B_il),
                     _ptr(mbar), _ptr(bounds), int(bool(record_decisions)), self._s())

    def dfr_np_forward(self, omega, lam, avg, B, F, mbar, bounds):
        _native.call("dm_dfr_np_forward", self._h, float(omega), _ptr(lam), _ptr(avg), _ptr(B), _ptr(F), _ptr(mbar),
                     _ptr(bounds), self._s())

    def dfr_np_backward(self, omega, lam, avg, F, B, mbar, bounds, record_decisions=False):
        _native.call("dm_dfr_np_backward", self._h, float(omega), _ptr(lam), _ptr(avg), _ptr(F), _ptr(B), _ptr(mbar),
                     _ptr(bounds), int(bool(record_decisions)), self._s())

    @property
    def dfr_node_parallel(self) -> bool:
        return bool(self.info.get("dfr_node_parallel", 0))

    def dfr_average(self, mbar, avg):
        _native.call("dm_dfr_average", self._h, _ptr(mbar), _ptr(avg), self._s())

    def dfr_flush(self, mbar, lam):
        _native.call("dm_dfr_flush", self._h, _ptr(mbar), _ptr(lam), self._s())

    def dfr_to_nodes(self, x_il, x):
        _native.call("dm_dfr_to_nodes", self._h, _ptr(x_il), _ptr(x), self._s())

    @property
    def dfr_records_decisions(self) -> bool:
        return int(self.info.get("max_width", 99)) <= 8

    # --- per-variable vectors ------------------------------------------------
    def init_duals(self, costs_by_var, lam):
        _native.call("dm_init_duals", self._h, _ptr(costs_by_var), _ptr(lam), self._s())

    def project_direction(self, d_hat, d):
        _native.call("dm_project_direction", self._h, _ptr(d_hat), _ptr(d), self._s())

    def lambda_sums(self, lam, out):
        _native.call("dm_lambda_sums", self._h, _ptr(lam), _ptr(out), self._s())

    def perturb_round(self, m0, m1, lam, delta, boost, seed, round_, values, agrees, disagree):
        _native.call("dm_perturb_round", self._h, _ptr(m0), _ptr(m1), _ptr(lam), float(delta), float(boost), int(seed),
                     int(round_), _ptr(values), _ptr(agrees), _ptr(disagree), self._s())

    def agreement_scores(self, m0, m1, agrees, score, preferred):
        _native.call("dm_agreement_scores", self._h, _ptr(m0), _ptr(m1), _ptr(agrees), _ptr(score),
                     _ptr(preferred), self._s())


# --- reductions and elementwise vectors (no handle needed) ---------------------
def release_caches() -> None:
    """Free the library's cached reduction plans and dot scratch (keyed by
    device, length and stream; they otherwise live for the process).  Call
    with no solve in flight."""
    _native.check(_native.load().dm_release_caches(), "dm_release_caches")


def dev_sum(x: torch.Tensor, out: torch.Tensor) -> None:
    """out[0] = np.sum(x) in numpy's pairwise order."""
    _native.call("dm_sum", _ptr(x), x.numel(), _ptr(out), _stream(x.device))


def dev_dot(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> None:
    """out[0] = np.sum(a * b) (pairwise order)."""
    _native.call("dm_dot", _ptr(a), _ptr(b), a.numel(), _ptr(out), _stream(a.device),
                 launches=_chunk_launches(a.numel()))


def _chunk_launches(n: int) -> int:
    """Kernels one chunked-dot step launches: full chunks + the finishing block."""
    return 2 if n >= 4096 else 1


def dev_axpy_dev(x, y, alpha_host, dot_dev, alpha_out=None):
    _native.call("dm_axpy_dev", _ptr(x), _ptr(y), float(alpha_host), _ptr(dot_dev), _ptr(alpha_out), x.numel(),
                 _stream(x.device))


def dev_scale_dev(x, num_host, den_dev):
    _native.call("dm_scale_dev", _ptr(x), float(num_host), _ptr(den_dev), x.numel(), _stream(x.device))


def dev_lbfgs_up(x, s, alpha_dev, rho_host, dot_dev):
    _native.call("dm_lbfgs_up", _ptr(x), _ptr(s), _ptr(alpha_dev), float(rho_host), _ptr(dot_dev), x.numel(),
                 _stream(x.device))


def dev_lbfgs_direction(g, pairs, d):
    """d = two-loop(g) over ``pairs`` [(s, y, rho, sy)] newest first (qn.py:95-115), fused launches."""
    m = len(pairs)
    ptrs = (ctypes.c_void_p * m)
    s_p = ptrs(*[p[0].data_ptr() for p in pairs])
    y_p = ptrs(*[p[1].data_ptr() for p in pairs])
    rho = (ctypes.c_double * m)(*[float(p[2]) for p in pairs])
    sy = (ctypes.c_double * m)(*[float(p[3]) for p in pairs])
    _native.call("dm_lbfgs_direction", _ptr(g), s_p, y_p, rho, sy, m, g.numel(), _ptr(d), _stream(g.device),
                 launches=(2 * m + 2) * _chunk_launches(g.numel()))


def dev_curvature_pair(lam, lam_prev, g, g_prev, s, y, sy_out):
    """s = lam - lam_prev, y = g_prev - g, lam_prev = lam, sy_out[0] = s . y (one pass)."""
    _native.call("dm_curvature_pair", _ptr(lam), _ptr(lam_prev), _ptr(g), _ptr(g_prev), _ptr(s), _ptr(y),
                 lam.numel(), _ptr(sy_out), _stream(lam.device))


def dev_axpy_host(x, gamma, y):
    _native.call("dm_axpy_host", _ptr(x), float(gamma), _ptr(y), x.numel(), _stream(x.device))


def dev_sub(out, a, b):
    _native.call("dm_sub", _ptr(out), _ptr(a), _ptr(b), out.numel(), _stream(out.device))


class FlatBdds:
    """All diagrams of one instance, flattened (kernels.py:35-92)."""

    def __init__(self, instance):
        if isinstance(instance, IlpInstance):
            table = instance.flat
        elif hasattr(instance, "constraints") and hasattr(instance, "variable_order"):
            # duck-typed reference instance (prodmatch.ilp.IlpInstance)
            table = _lower_bdds(instance.costs, instance.constraints, instance.variable_order, 0)
        else:
            raise TypeError("FlatBdds needs an IlpInstance")
        self.table = table
        for name in ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd", "zero_t", "one_t", "proc_ptr",
                     "proc_layers"):
            setattr(self, name, getattr(table, name))
        self.max_degree = int(table.max_degree)
        self.max_width = int(table.max_width)
        self.num_bdds = table.num_bdds
        self.num_layers = table.num_layers
        self.num_nodes = table.num_nodes
        self.constraint_counts = table.constraint_counts
        self._dev: dict = {}

    def device(self, device=None, exact_plans: bool = True) -> DeviceFlat:
        """The device copy (cached per device); ``exact_plans=False`` skips the
        exact passes' schedules (a deferred-schedule state never uses them)."""
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        key = str(dev)
        have = self._dev.get(key)
        if have is None or (exact_plans and not have.exact_plans):
            self._dev[key] = DeviceFlat(self.table, dev, exact_plans)
        return self._dev[key]
