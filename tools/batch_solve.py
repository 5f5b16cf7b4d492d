"""Throughput of independent solves: one after another vs solve_batch
(K concurrent streams) on one GPU (GPU tool)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.qn import solve, solve_batch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
config = sys.argv[2] if len(sys.argv) > 2 else "c2"
ks = [int(k) for k in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2, 3, 4]
insts = [build_instance(config, s) for s in range(n)]
cfg = SolveConfig(mode="hybrid", max_iterations=30, dual_tolerance=0.0)
solve(insts[0], cfg, device="cuda:0")  # warm-up (plans, pools)
torch.cuda.synchronize()
t = time.perf_counter()
seq = [solve(i, cfg, device="cuda:0") for i in insts]
torch.cuda.synchronize()
t_seq = time.perf_counter() - t
out = {"config": config, "instances": n, "sequential_s": t_seq}
for k in ks:
    torch.cuda.synchronize()
    t = time.perf_counter()
    bat = solve_batch(insts, cfg, device="cuda:0", concurrency=k)
    torch.cuda.synchronize()
    out[f"batch{k}_s"] = time.perf_counter() - t
    out[f"batch{k}_identical"] = all(a.bounds == b.bounds and a.state.lam.tobytes() == b.state.lam.tobytes()
                                    for a, b in zip(seq, bat))
    print(json.dumps(out), flush=True)
