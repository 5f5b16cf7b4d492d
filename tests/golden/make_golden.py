"""Generate tests/golden/golden.json by running the REAL reference
(`prodmatch`, imported read-only from /root/reference/pkg/src) in the build
container.  /root/reference does not exist on the GPU box, so the outputs
are committed; the generating script is kept here for provenance.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Recorded per case: sha256 of every FlatBdds array after
IlpInstance.from_rows (+ split_instance), the init bound/duals, the bound
trajectory and final duals of mma-only and hybrid solves, and hashes of the
min-marginal table, subgradient and agreement scores after one averaging
iteration.  Product-space cases store only the builder config plus a hash
of the rows (the builder is deterministic and regenerates them).
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
from prodmatch.dual import BACKWARD, FORWARD, init_duals, mma_pass, subgradient  # noqa: E402
from prodmatch.ilp import IlpInstance, make_row  # noqa: E402
from prodmatch.kernels import FlatBdds  # noqa: E402
from prodmatch.primal import agreement_scores  # noqa: E402
from prodmatch.qn import solve  # noqa: E402
from prodmatch.splitting import split_instance  # noqa: E402

from tests.cases import product_case, random_rows  # noqa: E402

FLAT_FIELDS = ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd", "zero_t", "one_t", "proc_ptr",
               "proc_layers")


def h(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + a.tobytes()).hexdigest()[:32]


def record(name, costs, rows, chunk, iters_mma, iters_hyb, extra=None):
    t0 = time.time()
    inst = IlpInstance.from_rows(np.asarray(costs, np.float64), [make_row(*r) for r in rows])
    if chunk:
        inst = split_instance(inst, chunk)
    flat = FlatBdds(inst)
    out = {"name": name, "chunk": chunk}
    if extra:
        out.update(extra)
    out["sizes"] = {"variables": int(inst.num_variables), "bdds": int(flat.num_bdds),
                    "layers": int(flat.num_layers), "nodes": int(flat.num_nodes)}
    out["flat"] = {k: h(getattr(flat, k)) for k in FLAT_FIELDS}
    out["flat"]["variable_order"] = h(inst.variable_order)
    out["flat"]["costs"] = h(inst.costs)
    st = init_duals(inst)
    out["init"] = {"bound": st.bound, "lam": h(st.lam)}
    mma_pass(st, FORWARD)
    out["after_forward"] = {"bound": st.bound, "lam": h(st.lam), "F": h(st.F)}
    m0, m1 = st.min_marginal_table()
    out["after_forward"]["m0"] = h(m0)
    out["after_forward"]["m1"] = h(m1)
    out["after_forward"]["B"] = h(st.B)
    mma_pass(st, BACKWARD)
    out["after_backward"] = {"bound": st.bound, "lam": h(st.lam), "B": h(st.B),
                             "subgradient": h(subgradient(st))}
    sc = agreement_scores(st)
    out["agreement"] = {"agrees": h(sc.agrees), "score": h(sc.score), "preferred": h(sc.preferred)}
    for mode, iters in (("mma-only", iters_mma), ("hybrid", iters_hyb)):
        res = solve(inst, SolveConfig(mode=mode, max_iterations=iters))
        out[mode] = {"bounds": [r.dual_objective for r in res.records],
                     "kinds": [r.kind for r in res.records], "stop": res.stop_reason,
                     "lam": h(res.state.lam), "best_bound": res.best_bound}
    out["seconds"] = round(time.time() - t0, 2)
    print(f"{name}: {out['sizes']} {out['seconds']}s", file=sys.stderr)
    return out


def append_product_cases(configs, fname="golden.json"):
    """Record further product-space cases and merge them into golden.json
    (``python tests/golden/make_golden.py c3``) or, for the full-size bench
    configs, golden_large.json (``python tests/golden/make_golden.py --large``);
    existing cases are kept."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), fname)
    doc = {"generator": "tests/golden/make_golden.py", "reference": "prodmatch 0.1.0", "numpy": np.__version__,
           "cases": []}
    if os.path.exists(path):
        with open(path) as fh:
            doc = json.load(fh)
    for name, cfg, seed, chunk, im, ih in configs:
        costs, rows, meta = product_case(cfg, seed)
        case = record(name, costs, rows, chunk, im, ih, meta)
        doc["cases"] = [c for c in doc["cases"] if c["name"] != case["name"]] + [case]
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(path)


# C3 (k-NN pruned humanoid-like pair, 500 x 500): a few iterations of each mode
EXTRA = {"c3": ("ps_c3", "c3", 0, 128, 3, 4)}
# The benched configs at full size (bench.py's default C2 line, the north
# star's C4 target, two members of the C5 batch = C3-generator seeds):
# 3 mma-only and 8-10 hybrid iterations each -> golden_large.json
LARGE = [("ps_c2", "c2", 0, 128, 3, 8), ("ps_c4", "c4", 0, 128, 3, 10),
         ("ps_c5_s17", "c3", 17, 128, 3, 8), ("ps_c5_s42", "c3", 42, 128, 3, 8)]


def main():
    if sys.argv[1:2] == ["--large"]:
        pick = sys.argv[2:]  # optional case names: only these are re-recorded
        append_product_cases([c for c in LARGE if not pick or c[0] in pick], "golden_large.json")
        return
    if len(sys.argv) > 1:
        append_product_cases([EXTRA[c] for c in sys.argv[1:]])
        return
    cases = []
    for seed in range(10):
        costs, rows = random_rows(seed)
        rows_j = [(list(map(int, v)), list(map(int, c)), int(b)) for v, c, b in rows]
        for chunk in (0, 3):
            c = record(f"random{seed}_c{chunk}", costs, rows, chunk, 30, 30,
                       {"costs": list(map(float, costs)), "rows": rows_j})
            cases.append(c)
    kinked = ([4.0, 1.0, 3.0], [([0, 1], [1, 1], 1), ([0, 2], [1, 1], 1)])
    toy = ([1.0, 1.0, 1.0], [([0, 1], [1, 1], 1), ([1, 2], [1, 1], 1)])
    for name, (costs, rows) in (("kinked", kinked), ("toy", toy)):
        cases.append(record(name, costs, rows, 0, 10, 10, {"costs": costs, "rows": rows}))
    for cfg, chunk, im, ih in (("tetra", 128, 20, 20), ("icosa", 128, 8, 8), ("c1", 128, 4, 6)):
        costs, rows, meta = product_case(cfg)
        cases.append(record(f"ps_{cfg}", costs, rows, chunk, im, ih, meta))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "prodmatch 0.1.0",
                   "numpy": np.__version__, "cases": cases}, fh, indent=1)
    print(path)


if __name__ == "__main__":
    main()
