"""Where a hybrid iteration's time goes, per phase (synchronised between
phases), for a config and schedule (GPU tool).

usage: python tools/c4_step.py [config] [schedule] [iterations]
"""
import cProfile
import io
import json
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200 import qn  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, mma_pass, subgradient_device  # noqa: E402
from paper_2310_08230_b200.kernels import dev_curvature_pair  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "c4"
schedule = sys.argv[2] if len(sys.argv) > 2 else "deferred"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
inst = build_instance(config, 0)
cfg = SolveConfig(mma_schedule=schedule, max_iterations=10**9, dual_tolerance=0.0)
run = qn.DualSolver(inst, cfg, device="cuda:0").start()
for _ in range(5):
    run.step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(n):
    run.step()
torch.cuda.synchronize()
out = {"config": config, "schedule": schedule, "ms_per_step": (time.perf_counter() - t) / n * 1e3}


def phase(log, name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    log[name] = log.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return r


log = {}
st = run.state
for _ in range(n):
    g = phase(log, "subgradient", lambda: subgradient_device(st))
    d = phase(log, "two_loop", lambda: qn.lbfgs_direction(g, run.history))
    d = phase(log, "project", lambda: qn.project_direction(d, st))
    sw0 = st.sweeps
    gamma, ok = phase(log, "step_search", lambda: qn.find_step_size(st, d, run.gamma, run.step_cfg))
    log["trials"] = log.get("trials", 0.0) + (st.sweeps - sw0)
    run.gamma = gamma
    if ok:
        phase(log, "shift", lambda: st.shift_lambda_scaled(gamma, d))
    if st.deferred:
        phase(log, "round", lambda: st.deferred_round(cfg.mma_damping))
    else:
        phase(log, "fw", lambda: mma_pass(st, FORWARD))
        phase(log, "bw", lambda: mma_pass(st, BACKWARD))
    g_now = phase(log, "subgradient_end", lambda: subgradient_device(st))
    s, y = run.history.reserve(st.lam_d)
    phase(log, "curvature", lambda: dev_curvature_pair(st.lam_d, run.lam_prev, g_now, run.g_prev, s, y,
                                                       st._slots[9:10]))
    vals = phase(log, "read_scalars", lambda: st.read_scalars())
    sy = float(vals[9])
    if sy >= run.step_cfg.curvature_eps:
        run.history.push(s, y, 1.0 / sy, sy)
    run.g_prev = g_now
out["phases_ms"] = {k: round(v / n, 4) for k, v in log.items()}
out["phases_sum_ms"] = round(sum(log.values()) / n, 4)
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    run.step()
torch.cuda.synchronize()
pr.disable()
sio = io.StringIO()
pstats.Stats(pr, stream=sio).sort_stats("tottime").print_stats(12)
print(json.dumps(out), flush=True)
print(sio.getvalue())
