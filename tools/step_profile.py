"""Where does a C2 solver step spend host time? (GPU tool)"""
import cProfile
import io
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.qn import DualSolver  # noqa: E402

inst = build_instance("c2", 0)
run = DualSolver(inst, SolveConfig(max_iterations=10**9, dual_tolerance=0.0), device="cuda:0").start()
for _ in range(3):
    run.step()
torch.cuda.synchronize()
t = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    run.step()
torch.cuda.synchronize()
pr.disable()
print(f"wall per step {(time.perf_counter() - t) / 5 * 1e3:.1f} ms")
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue())
