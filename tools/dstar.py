"""Best known dual bound d* of the benched instances (GPU tool) ->
profiles/dstar.json, the reference point of every time-to-gap number in
bench.py: long hybrid runs of both averaging schedules with no stopping rule
(dual_tolerance = -inf), d* = the best bound either reached.  Each entry
records the rows hash of the instance, the per-run best bounds and how much
the last 10 % of each run still gained.

usage: python tools/dstar.py c2 c3 c4 [--iters-exact N] [--iters-deferred N]"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import DSTAR_PATH, build_instance  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.qn import solve  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--iters-exact", type=int, default=1500)
ap.add_argument("--iters-deferred", type=int, default=4000)
ap.add_argument("--chunk", type=int, default=128, help="split length of the lowering (0: unsplit)")
a = ap.parse_args()
table = {}
if os.path.exists(DSTAR_PATH):
    with open(DSTAR_PATH) as fh:
        table = json.load(fh)
for cfg in a.configs:
    inst = build_instance(cfg, a.seed, a.chunk)
    runs = {}
    for sched, iters in (("exact", a.iters_exact), ("deferred", a.iters_deferred)):
        t = time.perf_counter()
        res = solve(inst, SolveConfig(mode="hybrid", max_iterations=iters, dual_tolerance=-float("inf"),
                                      mma_schedule=sched), device="cuda:0")
        torch.cuda.synchronize()
        b = res.bounds
        k = max(1, len(b) // 10)
        runs[sched] = {"iterations": res.iterations, "best_bound": res.best_bound, "seconds": time.perf_counter() - t,
                       "gain_last_10pct": res.best_bound - max(b[:-k])}
        print(cfg, sched, runs[sched], file=sys.stderr, flush=True)
    best = max(r["best_bound"] for r in runs.values())
    table[f"{cfg}:{a.seed}" + ("" if a.chunk == 128 else f":chunk{a.chunk}")] = {"d_star": best, "rows_hash": inst._rows_hash, "runs": runs,
                                "chunk": a.chunk,
                                "source": "best dual bound of long hybrid runs of both schedules on a B200 "
                                          f"(exact {a.iters_exact}, deferred {a.iters_deferred} iterations, no "
                                          "stopping rule; tools/dstar.py)"}
    with open(DSTAR_PATH, "w") as fh:
        json.dump(table, fh, indent=1)
print(json.dumps(table, indent=1))
