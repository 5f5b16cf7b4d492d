"""Where does an end-to-end solve from host arrays spend its time? (GPU tool)"""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
os.environ.setdefault("DM_VERBOSE", "1")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.dual import init_duals  # noqa: E402
from paper_2310_08230_b200.kernels import FlatBdds  # noqa: E402
from paper_2310_08230_b200.qn import solve  # noqa: E402

inst = build_instance("c2", 0)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inst._flat_dev = None
    flat = FlatBdds(inst)
    t1 = time.perf_counter()
    st = init_duals(inst, device="cuda:0", flat=flat)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = solve(inst, SolveConfig(mode="hybrid", max_iterations=50, dual_tolerance=0.0), device="cuda:0", state=st)
    lam = res.state.lam
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"rep {rep}: FlatBdds {t1 - t0:.3f}s init_duals {t2 - t1:.3f}s solve(50) {t3 - t2:.3f}s total {t3 - t0:.3f}s",
          flush=True)
    del flat, st, res
