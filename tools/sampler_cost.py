"""Cost of nvidia-smi sampling on the solver step (GPU tool)."""
import subprocess
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
FULL = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
        "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
variants = [("none", None), ("full_100", ["-lms", "100"], FULL), ("full_500", ["-lms", "500"], FULL),
            ("clocks_100", ["-lms", "100"], "clocks.sm"), ("reasons_100", ["-lms", "100"], "clocks_event_reasons.active"),
            ("power_100", ["-lms", "100"], "power.draw")]
for v in variants:
    name = v[0]
    proc = None
    if v[1] is not None:
        proc = subprocess.Popen(["nvidia-smi", "--id=0", f"--query-gpu={v[2]}", "--format=csv,noheader", *v[1]],
                                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        time.sleep(1.5)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        run.step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10 * 1e3
    if proc:
        proc.terminate()
        proc.wait()
    print(f"{name:12s} {dt:7.1f} ms/step", flush=True)
