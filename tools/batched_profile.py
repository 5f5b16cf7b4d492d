"""Host profile of a BatchedSolver run (GPU tool): where a small pack's
iteration goes.  usage: python tools/batched_profile.py [n] [compact]"""
import cProfile
import io
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.batch import BatchedSolver  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
compact = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
insts = [build_instance("c3", s) for s in range(n)]
cfg = SolveConfig(mode="hybrid", max_iterations=40, dual_tolerance=-float("inf"))
BatchedSolver(insts, cfg, device="cuda:0", compact=compact).solve()
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
bs = BatchedSolver(insts, cfg, device="cuda:0", compact=compact)
t1 = time.perf_counter()
bs.solve()
torch.cuda.synchronize()
pr.disable()
t2 = time.perf_counter()
print(f"init {t1 - t:.3f}s, 40 iterations {t2 - t1:.3f}s ({(t2 - t1) / 40 * 1e3:.2f} ms/it)")
sio = io.StringIO()
pstats.Stats(pr, stream=sio).sort_stats("tottime").print_stats(18)
print(sio.getvalue())
