"""Generate tests/golden/primal.json by running the REAL reference's primal
side (`prodmatch.primal`, imported read-only from /root/reference/pkg/src) in
the build container; the outputs are committed, this script is provenance.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_primal_golden.py

Per case, from the duals of a bit-reproducible mma-only solve: the fixed
variables and conditioned residual instance (FlatBdds hashes, dropped
diagram count) of fix_and_reduce at several fractions (or the
InfeasibleAfterFixing it raises), and the status / assignment / objective /
ladder stage of recover_primal.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_NUM_THREADS", "8")

from prodmatch.config import SolveConfig  # noqa: E402
from prodmatch.errors import InfeasibleAfterFixing  # noqa: E402
from prodmatch.ilp import IlpInstance, make_row  # noqa: E402
from prodmatch.kernels import FlatBdds  # noqa: E402
from prodmatch.primal import fix_and_reduce, recover_primal  # noqa: E402
from prodmatch.qn import solve  # noqa: E402
from prodmatch.splitting import split_instance  # noqa: E402

from tests.cases import product_case, random_rows  # noqa: E402

FLAT_FIELDS = ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd", "zero_t", "one_t", "proc_ptr",
               "proc_layers")
FRACTIONS = (0.9, 0.5, 0.25)


def h(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + a.tobytes()).hexdigest()[:32]


def record(name, costs, rows, chunk, iters, extra=None, recover=True):
    t0 = time.time()
    inst = IlpInstance.from_rows(np.asarray(costs, np.float64), [make_row(*r) for r in rows])
    if chunk:
        inst = split_instance(inst, chunk)
    out = {"name": name, "chunk": chunk, "mma_iterations": iters}
    if extra:
        out.update(extra)
    res = solve(inst, SolveConfig(mode="mma-only", max_iterations=iters, dual_tolerance=0.0))
    st = res.state
    out["best_bound"] = st.best_bound
    out["fix"] = {}
    for frac in FRACTIONS:
        try:
            partial, residual = fix_and_reduce(inst, st, frac)
        except InfeasibleAfterFixing:
            out["fix"][str(frac)] = {"infeasible": True}
            continue
        fl = FlatBdds(residual)
        keys = sorted(partial.values)
        out["fix"][str(frac)] = {
            "fixed_vars": h(np.array(keys, np.int64)),
            "fixed_vals": h(np.array([partial.values[k] for k in keys], np.int64)),
            "num_fixed": len(keys),
            "num_constraints": int(residual.num_constraints),
            "dropped": int(inst.num_constraints - residual.num_constraints),
            "flat": {k: h(getattr(fl, k)) for k in FLAT_FIELDS},
        }
    if not recover:  # time-budgeted branch and bound: not reproducible, fixes only
        out["seconds"] = round(time.time() - t0, 2)
        return out
    sol = recover_primal(inst, st, SolveConfig(max_seconds=60.0))
    out["recover"] = {"status": sol.status, "ladder_stage": sol.ladder_stage}
    if sol.assignment is not None:
        out["recover"]["assignment"] = h(np.asarray(sol.assignment, np.int8))
        out["recover"]["objective"] = float(inst.costs @ sol.assignment)
    if sol.report is not None:
        out["recover"]["gap"] = sol.report.primal_dual_gap
        out["recover"]["certified"] = sol.report.certified
    out["seconds"] = round(time.time() - t0, 2)
    print(f"{name}: {out['recover']} {out['seconds']}s", file=sys.stderr)
    return out


def append_fix_only(configs):
    """``python tests/golden/make_primal_golden.py c3``: record fix_and_reduce
    residuals of larger product spaces (their recover_primal runs into the
    branch and bound's time budget, so it is not recorded) and merge them
    into primal.json."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "primal.json")
    with open(path) as fh:
        doc = json.load(fh)
    for cfg in configs:
        costs, rows, meta = product_case(cfg)
        case = record(f"ps_{cfg}", costs, rows, 128, 20, meta, recover=False)
        doc["cases"] = [c for c in doc["cases"] if c["name"] != case["name"]] + [case]
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(path)


def main():
    if len(sys.argv) > 1:
        append_fix_only(sys.argv[1:])
        return
    cases = []
    for seed in range(10):
        costs, rows = random_rows(seed)
        rows_j = [(list(map(int, v)), list(map(int, c)), int(b)) for v, c, b in rows]
        for chunk in (0, 3):
            cases.append(record(f"random{seed}_c{chunk}", costs, rows, chunk, 20,
                                {"costs": list(map(float, costs)), "rows": rows_j}))
    kinked = ([4.0, 1.0, 3.0], [([0, 1], [1, 1], 1), ([0, 2], [1, 1], 1)])
    toy = ([1.0, 1.0, 1.0], [([0, 1], [1, 1], 1), ([1, 2], [1, 1], 1)])
    for name, (costs, rows) in (("kinked", kinked), ("toy", toy)):
        cases.append(record(name, costs, rows, 0, 10, {"costs": costs, "rows": rows}))
    for cfg, chunk, iters in (("tetra", 128, 30),):
        costs, rows, meta = product_case(cfg)
        cases.append(record(f"ps_{cfg}", costs, rows, chunk, iters, meta))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "primal.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_primal_golden.py", "reference": "prodmatch 0.1.0",
                   "numpy": np.__version__, "cases": cases}, fh, indent=1)
    print(path)


if __name__ == "__main__":
    main()
