"""TEST INFRASTRUCTURE: a CPU engine for paper_2310_08230_b200.partition's
PartitionedSolver built on the C oracle (oracle/ckernels.c oracle_dfr_*), so
the partitioned solve loop, its plan and its exchange run over gloo on CPUs
(the product's DeviceEngine is the GPU counterpart)."""

import numpy as np
import torch

from oracle import model
from oracle.clib import lib, ptr

INF = np.inf


class OracleEngine:
    def __init__(self, part):
        t = part.table
        self.part = part
        self.oi, self.of = model.from_flat_table(t.costs, t.variable_order, t.constraint_counts,
                                                 {k: getattr(t, k) for k in ("bdd_layer_lo", "layer_node_lo",
                                                                             "layer_var", "layer_bdd", "zero_t",
                                                                             "one_t", "proc_ptr", "proc_layers")})
        f = self.of
        self.lam_t = torch.as_tensor(part.lam0.copy())
        self.lam = self.lam_t  # the solver hands these out
        self.F = np.zeros(f.num_nodes)
        self.B = np.zeros(f.num_nodes)
        self.mbar = np.zeros(f.num_layers)
        self.avg = np.zeros(f.num_layers)
        self.bounds = torch.zeros(f.num_bdds, dtype=torch.float64)
        self.geo = (f.num_bdds, ptr(f.bdd_layer_lo), ptr(f.layer_node_lo), ptr(f.zero_t), ptr(f.one_t))
        self.lp = np.ascontiguousarray(part.local_ptr, np.int64)
        self.ll = np.ascontiguousarray(part.local_layers, np.int64)

    def _lam(self):
        return self.lam_t.numpy()

    def new_buffer(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def sweep(self):
        lib.oracle_dfr_backward(*self.geo, 0.0, ptr(self._lam()), None, None, ptr(self.B), None,
                                ptr(self.bounds.numpy()))

    def forward_pass(self, omega):
        lib.oracle_dfr_forward(*self.geo, float(omega), ptr(self._lam()), None, ptr(self.B), ptr(self.F),
                               ptr(self.mbar), ptr(self.bounds.numpy()))

    def backward_pass(self, omega):
        lib.oracle_dfr_backward(*self.geo, float(omega), ptr(self._lam()), ptr(self.avg), ptr(self.F), ptr(self.B),
                                ptr(self.mbar), ptr(self.bounds.numpy()))

    def average_local(self, apply):
        tmp = np.zeros_like(self.avg)
        lib.oracle_dfr_average(len(self.lp) - 1, ptr(self.lp), ptr(self.ll), ptr(self.mbar), ptr(tmp))
        if apply:
            lam = self._lam()
            lam[self.ll] = lam[self.ll] + tmp[self.ll]
        else:
            self.avg[self.ll] = tmp[self.ll]

    def gather_boundary(self, buf):
        b = buf.numpy()
        b[:] = 0.0
        b[self.part.b_slot] = self.mbar[self.part.b_layer]

    def average_boundary(self, buf, apply):
        b = buf.numpy()
        out = self._lam() if apply else self.avg
        p = self.part
        for l, s, lo, hi in zip(p.b_layer, p.b_slot, p.b_lo, p.b_hi):
            total, cnt = 0.0, 0
            for x in b[lo:hi]:
                if x != INF:
                    total = total + x
                    cnt += 1
            mean = total / cnt if cnt else 0.0
            a = mean if b[s] != INF else 0.0
            out[l] = out[l] + a if apply else a

    def global_bound(self, all_bounds):
        return float(np.sum(all_bounds.numpy()))
