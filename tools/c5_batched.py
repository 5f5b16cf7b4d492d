"""C5 with each instance's own hybrid solve to the reference stopping rule:
separate solves one after another, solve_batch (concurrent streams) and
solve_batched (one merged instance, per-instance L-BFGS) — wall time from
host tables, and whether the batched bounds equal the separate ones (GPU tool).

usage: python tools/c5_batched.py [n_instances] [schedule]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.batch import solve_batched  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.qn import solve, solve_batch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
schedule = sys.argv[2] if len(sys.argv) > 2 else "exact"
insts = [build_instance("c3", s) for s in range(n)]
cfg = SolveConfig(mode="hybrid", mma_schedule=schedule)
dev = "cuda:0"


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t, r


solve(insts[0], cfg, device=dev)
solve_batched(insts[:2], cfg, device=dev)
t_seq, seq = timed(lambda: [solve(i, cfg, device=dev) for i in insts])
out = {"instances": n, "schedule": schedule, "sequential_s": t_seq,
       "iterations": [r.iterations for r in seq]}
print(json.dumps(out), flush=True)
t_bat, bat = timed(lambda: solve_batch(insts, cfg, device=dev, concurrency=8))
out["streams8_s"] = t_bat
print(json.dumps(out), flush=True)
for rep in range(2):
    t_b, got = timed(lambda: solve_batched(insts, cfg, device=dev))
    out[f"batched_s_{rep}"] = t_b
out["batched_identical"] = all(g.bounds == s.bounds for g, s in zip(got, seq))
out["batched_iterations"] = max(g.iterations for g in got)
print(json.dumps(out), flush=True)
long = max(range(n), key=lambda k: seq[k].iterations)
t_long, _ = timed(lambda: solve(insts[long], cfg, device=dev))
out["longest_alone_s"] = t_long
from paper_2310_08230_b200.batch import BatchedSolver  # noqa: E402

torch.cuda.synchronize()
t = time.perf_counter()
bs = BatchedSolver(insts, cfg, device=dev, compact=float(sys.argv[3]) if len(sys.argv) > 3 else 0.25)
t_init = time.perf_counter() - t
bs.solve()
torch.cuda.synchronize()
out["batched_init_s"] = t_init
out["batched_total_s"] = time.perf_counter() - t
out["pack_phases"] = bs.pack_phases
out["trace"] = [(i, p, l, round(s, 4)) for i, p, l, s in bs.trace if i < 40 or i % 20 == 0]
print(json.dumps(out), flush=True)
