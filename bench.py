#!/usr/bin/env python
"""Benchmark of the DiscoMatch dual solver hot path on B200.

Workload (BASELINE.json configs[1]): randomly non-rigidly deformed icosphere
pair, subdivision 2 (320 x 320 triangles), full product space (2.25 M
product triangles + 39,680 coupling variables after 128-chunk splitting,
636,800 diagrams, 9.4 M dual coordinates, 31 M diagram nodes), smooth
synthetic descriptors.  One step = one hybrid solver iteration (L-BFGS move
with bounded step search + exact forward/backward averaging passes +
history update), i.e. DualSolver.step() — the loop body of qn.solve.

metric: BDD arc updates/s (2 arcs per node per full-table sweep; an exact
averaging half-pass counts 2 sweeps: min-marginals + propagation), plus
time-to-1e-3 relative dual gap as ``time_to_gap``.

Arms: default = B200 path (sm_100a kernels via libdiscomatch_b200.so);
``--impl reference`` = the reference algorithm on the host's cores (the C
oracle port; the reference itself is Python/numba and not installable on
the GPU box).  N>1 (torchrun): one process per GPU, each rank solves its
own instance (seed = rank, instance sharding as in config C5; no
collective on the data path) -> "scaling": "weak".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-1e-3 duality gap (s) & BDD arc updates/s at 1/2/4/8 B200 vs CPU ref"
UNIT = "arc-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ttg", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--e2e-iters", type=int, default=50)
    ap.add_argument("--ttg-max-iters", type=int, default=150)
    ap.add_argument("--batch", type=int, default=0, help="also time K independent instances via qn.solve_batch")
    ap.add_argument("--batch-iters", type=int, default=30)
    ap.add_argument("--streams", type=int, default=8, help="concurrent solves per GPU for --config c5")
    return ap.parse_args()


WORKLOADS = {
    "c1": "icosphere pair subdiv-1 (80x80 tri), full product space, random descriptors",
    "c2": "deformed icosphere pair subdiv-2 (320x320 tri), full product space, smooth descriptors",
    "c3": "deformed humanoid-like genus-0 pair (500x500 tri), k-NN (k=10) pruned product space, "
          "heat-kernel-signature + smooth descriptors",
    "c4": "deformed humanoid-like genus-0 pair (980x980 tri), k-NN (k=16) pruned product space, "
          "heat-kernel-signature + smooth descriptors, one GPU",
    "c5": "batch of 64 independent c3-generator pairs (seeds 0..63), instance-sharded",
}


def workload(config: str) -> str:
    return f"{config}: {WORKLOADS.get(config, config)}"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def build_instance(config: str, seed: int):
    from paper_2310_08230_b200 import product_space as ps
    from paper_2310_08230_b200.ilp import IlpInstance

    t = time.perf_counter()
    p = ps.synthetic_product_space(config, seed)
    t1 = time.perf_counter()
    inst = IlpInstance.from_csr(p.costs, p.row_ptr, p.row_var, p.row_coef, p.row_rhs, 128)
    t2 = time.perf_counter()
    log(f"[bench] {config} seed {seed}: product space {t1 - t:.1f}s, lowering {t2 - t1:.1f}s, "
        f"{inst.num_variables} vars, {inst.flat.num_bdds} bdds, {inst.flat.num_layers} layers, "
        f"{inst.flat.num_nodes} nodes")
    return inst


def oracle_twin(inst):
    from oracle import model

    f = inst.flat
    arrays = {k: getattr(f, k) for k in ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd", "zero_t",
                                          "one_t", "proc_ptr", "proc_layers")}
    return model.from_flat_table(inst.costs, inst.variable_order, f.constraint_counts, arrays)


def cpu_reference_run(inst, warmup: int, steps: int):
    """The reference algorithm (C port of the numba kernels + numpy driver) on
    the host: untimed warm-up iterations, then ``steps`` timed iterations.
    Returns (arc_updates/s, seconds per iteration, threads)."""
    from oracle import solver
    from oracle.clib import lib

    threads = os.cpu_count() or 1
    lib.oracle_set_threads(threads)
    oi, of = oracle_twin(inst)
    gen = _oracle_iterations(oi, of)
    for _ in range(warmup):
        next(gen)
    st = next(gen)  # yields state after each iteration
    s0 = st.sweeps
    t0 = time.perf_counter()
    for _ in range(steps):
        st = next(gen)
    dt = time.perf_counter() - t0
    arcs = (st.sweeps - s0) * 2 * of.num_nodes
    return arcs / dt, dt / steps, threads


def _oracle_iterations(oi, of):
    """Generator form of oracle.solver.solve (qn.py:211-259), hybrid mode."""
    from collections import deque

    from oracle import solver

    st = solver.init_duals(oi, of)
    hist = deque(maxlen=10)
    first = st.objective()
    min_ascent = 0.0
    lam_prev = st.lam.copy()
    g_prev = st.subgradient()
    gamma = 1.0
    it = 0
    yield st
    while True:
        it += 1
        if hist:
            g = st.subgradient()
            d = solver.project(solver.lbfgs(g, list(hist), solver._dot_blas), st)
            gamma, better = solver.step_search(st, d, gamma, 0.8, 1.1, 5, min_ascent)
            if better:
                st.shift(gamma * d)
        st.mma(True)
        st.mma(False)
        bound = st.objective()
        if it == 1:
            min_ascent = 1e-6 * (bound - first)
        g_now = st.subgradient()
        s = st.lam - lam_prev
        y = g_prev - g_now
        sy = float(s @ y)
        if sy >= 1e-8:
            hist.appendleft((s, y, 1.0 / sy, sy))
        lam_prev = st.lam.copy()
        g_prev = g_now
        yield st


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.samples = []  # (host time, line)
        self.marks = []

    def __enter__(self):
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self

        def reader():
            for line in self.proc.stdout:
                if line.strip():
                    self.samples.append((time.time(), line))

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        return self

    def mark(self):
        self.marks.append(time.time())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=5)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lo, hi = (self.marks[0], self.marks[-1]) if len(self.marks) >= 2 else (0.0, float("inf"))
        window = [l for t, l in self.samples if lo <= t <= hi + 0.2] or [l for _, l in self.samples]
        for line in window:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def aggregate_work_time(work: float, ms: float, world: int, device=None):
    """Whole-job aggregation over ranks: total work (sum) and the slowest
    rank's time (max).  Works with the nccl (device tensor) and gloo (CPU)
    backends; instance sharding needs no other collective."""
    import torch

    t = torch.tensor([float(work), float(ms)], dtype=torch.float64, device=device)
    if world > 1:
        w, m = t[0:1].clone(), t[1:2].clone()
        torch.distributed.all_reduce(w, op=torch.distributed.ReduceOp.SUM)
        torch.distributed.all_reduce(m, op=torch.distributed.ReduceOp.MAX)
        t = torch.cat([w, m])
    return float(t[0]), float(t[1])


# one-way visibility of a relaxed gpu-scope store to a polling SM on B200,
# measured by tools/pingpong.cu (534 ns round trip / 2)
VISIBILITY_NS = 267.0


def _traffic(kernel, config="c2"):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture summary of this config (profiles/traffic.json for C2,
    profiles/traffic_<config>.json otherwise; tools/ncu_summary.py), or None."""
    name = "traffic.json" if config == "c2" else f"traffic_{config}.json"
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
    try:
        with open(path) as f:
            tr = json.load(f)
    except (OSError, ValueError):
        return None
    # the exact passes run their node-parallel instantiation when the instance allows it
    cands = [kernel.replace("mma_", "mma_np_"), kernel] if kernel.startswith("mma_") else [kernel]
    for cand in cands:
        for name, b in tr.items():
            if name.startswith(cand + "_kernel") or name.startswith(cand + "<") or name == cand:
                return b
    return None


def algorithmic_bytes(flat):
    """Per-launch algorithmic HBM bytes."""
    N, L, nb = flat.num_nodes, flat.num_layers, flat.num_bdds
    return {
        # arcs 8 + own distance read 8 + target distance read 8 + produced distance 8 + sentinel prime 8
        # per node; lam r/w 16 + task slot 8 + layer offset 4 per layer; bound 8 per diagram
        "mma": 40 * N + 28 * L + 8 * nb,
        # interleaved arcs 8 per node (next-layer distances stay in shared memory, trial writes no table);
        # lam 8 + d 8 per layer; bound 8 + offsets 8 per diagram
        "backward_trial": 8 * N + 16 * L + 16 * nb,
    }


def run_b200(args, rank, world, local_rank):
    import torch

    from paper_2310_08230_b200 import _native
    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.dual import KernelTimer
    from paper_2310_08230_b200.qn import DualSolver, solve

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    inst = build_instance(args.config, args.seed + rank)
    cfg = SolveConfig(mode="hybrid", max_iterations=10**9, dual_tolerance=0.0)
    run = DualSolver(inst, cfg, device=dev).start()
    st = run.state
    info = st.dev.info
    log(f"[bench] rank {rank}: exact-pass DAG depth fw {info['fw_depth']} bw {info['bw_depth']}, "
        f"tasks {info['fw_tasks']}, grid {info['mma_grid']}x{info['mma_block']}")
    # the clock sampler (nvidia-smi) starts before the warm-up: its start-up
    # touches the driver and must not fall inside the timed region
    with ClockSampler(local_rank) as clk:
        time.sleep(1.0)
        for _ in range(args.warmup):
            run.step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        timer = KernelTimer()
        st.pass_timer = timer
        s0 = st.sweeps
        l0 = _native.launch_count
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk.mark()
        torch.cuda.synchronize()
        start.record()
        step_wall = []
        for _ in range(args.steps):
            t_s = time.perf_counter()
            sw0 = st.sweeps
            run.step()
            step_wall.append((round((time.perf_counter() - t_s) * 1e3, 2), st.sweeps - sw0))
        end.record()
        torch.cuda.synchronize()
        clk.mark()
        log(f"[bench] per-step host wall ms / sweeps: {step_wall}")
    if world > 1:
        torch.distributed.barrier()
    st.pass_timer = None
    ms = start.elapsed_time(end)
    arcs = (st.sweeps - s0) * 2 * st.flat.num_nodes
    launches = _native.launch_count - l0
    kt = timer.summary()

    total_arcs, max_ms = aggregate_work_time(arcs, ms, world, dev)
    value = total_arcs / (max_ms / 1e3)

    result = None
    if rank == 0:
        abytes = algorithmic_bytes(st.flat)
        peaks = _peaks()
        hbm = peaks.get("hbm_gbs", 6650.0)
        kernels = {}
        for name, k in kt.items():
            if name == "step_search":
                # one event pair around the device trial sequence: per-trial
                # figures over the trials that ran (sweep + bound sum + decision)
                trials = max(timer.counts.get("step_search_trials", 0), 1)
                k = dict(k, searches=k["launches"], launches=trials, avg_ms=k["total_ms"] / trials)
                bpl = abytes["backward_trial"]
            else:
                bpl = abytes["mma" if name.startswith("mma") else name]
            kernels[name] = dict(k, bytes_per_launch=bpl, achieved_gbs=bpl / (k["avg_ms"] * 1e-3) / 1e9,
                                 share_of_step=k["total_ms"] / ms)
        dom = max(kernels, key=lambda n: kernels[n]["total_ms"]) if kernels else None
        roof = None
        if dom:
            a = kernels[dom]["achieved_gbs"]
            roof = {"bound": "hbm", "kernel": dom, "achieved": round(a, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(a / hbm, 4),
                    "traffic": _traffic(dom, args.config),
                    "algorithmic_bytes": kernels[dom]["bytes_per_launch"],
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"}
            if dom.startswith("mma"):
                # the exact passes are bound by their dependency chain, not by bytes
                depth = info["fw_depth"] if dom == "mma_forward" else info["bw_depth"]
                ns = kernels[dom]["avg_ms"] * 1e6 / depth
                roof["critical_path"] = {
                    "levels": depth, "ns_per_level": round(ns, 1),
                    "visibility_floor_ns": VISIBILITY_NS,
                    "frac": round(VISIBILITY_NS / ns, 4),
                    "note": "per level >= one-way store->poll visibility between SMs (tools/pingpong.cu)"}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args.config) + ", 128-chunk split, hybrid L-BFGS+exact MMA iteration; one instance per GPU",
                       "variables": inst.num_variables, "bdds": st.flat.num_bdds, "dual_coords": st.flat.num_layers,
                       "nodes": st.flat.num_nodes, "fw_depth": info["fw_depth"], "bw_depth": info["bw_depth"],
                       "l2": "working set 1.4 GB > 126 MB L2 (no flush needed)",
                       "parallelism": f"instance-sharded x{world}"},
            "gpu_launches": launches,
            "kernels": kernels,
            "roofline": roof,
            "clocks": clk.summary(),
        }
    # time to 1e-3 relative dual gap (gap vs the run's best bound; host clock incl. init)
    if rank == 0 and not args.no_ttg:
        res = solve(inst, SolveConfig(mode="hybrid", max_iterations=args.ttg_max_iters), device=dev, state=st)
        d_star = res.best_bound
        ttg = None
        for r in res.records:
            if (d_star - r.dual_objective) <= 1e-3 * abs(d_star):
                ttg = r
                break
        result["time_to_gap"] = {"value": ttg.time_s if ttg else None, "unit": "s", "gap": 1e-3,
                                 "iterations": ttg.iteration if ttg else None, "d_star": d_star,
                                 "d_star_iterations": res.iterations, "stop": res.stop_reason,
                                 "clock": "host perf_counter from solve() start, duals resident"}
    if rank == 0 and not args.no_ttg and args.config == "c2":
        result["c4_time_to_gap"] = c4_time_to_gap(args, dev)
    if rank == 0 and not args.no_e2e:
        result["e2e"] = e2e_run(args, inst, dev)
    if rank == 0 and args.batch > 1:
        result["batch"] = batch_run(args, inst, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, spi, thr = cpu_reference_run(inst, 1, args.cpu_iters)
        result["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": thr, "kind": "port",
                                  "sample": f"{args.cpu_iters} hybrid iterations of the same {args.config} instance "
                                            f"after 1 warm-up iteration ({spi:.2f} s/iteration); C port of the numba "
                                            "kernels, exact passes single-threaded as in the reference"}
        if result.get("time_to_gap", {}).get("iterations"):
            result["time_to_gap"]["cpu_projected_s"] = spi * result["time_to_gap"]["iterations"]
    return result


def c4_time_to_gap(args, dev):
    """The north star's single-instance target next to the C2 line: the
    ~1000 x 1000-triangle k-NN pruned pair (C4) on this GPU, time to a 1e-3
    relative gap to the run's best bound (same definition and clock as
    ``time_to_gap``: from solve() start, instance resident)."""
    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.dual import init_duals
    from paper_2310_08230_b200.qn import solve

    inst = build_instance("c4", args.seed)
    st = init_duals(inst, device=dev)  # upload + plans, outside the clock
    res = solve(inst, SolveConfig(mode="hybrid", max_iterations=args.ttg_max_iters), device=dev, state=st)
    d_star = res.best_bound
    hit = next((r for r in res.records if (d_star - r.dual_objective) <= 1e-3 * abs(d_star)), None)
    return {"value": hit.time_s if hit else None, "unit": "s", "gap": 1e-3, "iterations": hit.iteration if hit else None,
            "d_star": d_star, "d_star_iterations": res.iterations, "stop": res.stop_reason,
            "workload": workload("c4"), "nodes": st.flat.num_nodes}


def batch_run(args, inst, dev):
    """C5-style throughput on one GPU: --batch independent instances (seeds
    seed..seed+K-1, the first being the bench instance) solved one after
    another vs through qn.solve_batch (two concurrent streams); same
    iteration count, duals required identical."""
    import torch

    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.qn import solve, solve_batch

    insts = [inst] + [build_instance(args.config, args.seed + k) for k in range(1, args.batch)]
    cfg = SolveConfig(mode="hybrid", max_iterations=args.batch_iters, dual_tolerance=0.0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    seq = [solve(i, cfg, device=dev) for i in insts]
    torch.cuda.synchronize()
    t_seq = time.perf_counter() - t
    t = time.perf_counter()
    bat = solve_batch(insts, cfg, device=dev, concurrency=2)
    torch.cuda.synchronize()
    t_bat = time.perf_counter() - t
    same = all(a.state.lam.tobytes() == b.state.lam.tobytes() for a, b in zip(seq, bat))
    arcs = sum(r.state.arc_updates for r in bat)
    return {"instances": len(insts), "iterations": args.batch_iters, "concurrency": 2,
            "sequential_s": t_seq, "batch_s": t_bat, "value": arcs / t_bat, "unit": UNIT,
            "sequential_value": arcs / t_seq, "identical_to_sequential": same,
            "step": "qn.solve from the lowered host instances incl. device upload, per instance"}


def e2e_run(args, inst, dev):
    """Same metric through the public API from HOST buffers: every step
    uploads the lowered instance (FlatBdds.device: topology + schedules),
    runs qn.solve for --e2e-iters iterations and reads the duals back."""
    import numpy as np
    import torch

    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.kernels import FlatBdds
    from paper_2310_08230_b200.qn import solve

    f = inst.flat
    h2d = sum(getattr(f, k).nbytes for k in ("bdd_layer_lo", "layer_node_lo", "layer_var", "zero_t", "one_t",
                                             "proc_ptr", "proc_layers")) + inst.costs.nbytes
    reps = []
    arcs = 0
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        inst._flat_dev = None
        flat = FlatBdds(inst)
        from paper_2310_08230_b200.dual import init_duals

        state = init_duals(inst, device=dev, flat=flat)
        res = solve(inst, SolveConfig(mode="hybrid", max_iterations=args.e2e_iters, dual_tolerance=0.0),
                    device=dev, state=state)
        lam = res.state.lam  # D2H
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if rep:
            reps.append(dt)
            arcs = res.state.arc_updates
        d2h = lam.nbytes + 8 * len(res.records)
        del flat, state, res
    sec = float(np.median(reps))
    return {"value": arcs / sec, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "seconds_per_step": sec, "step": f"qn.solve({args.e2e_iters} hybrid iterations) from host arrays incl. "
                                             "device upload + schedule build"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def run_reference(args, rank):
    if rank != 0:
        return None
    # C5's instances are C3-generator pairs: the CPU arm times one of them
    inst = build_instance("c3" if args.config == "c5" else args.config, args.seed)
    steps = min(args.steps, 5)
    v, spi, thr = cpu_reference_run(inst, min(args.warmup, 1), steps)
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
            "warmup": min(args.warmup, 1), "ms_per_step": spi * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args.config) + ", 128-chunk split, hybrid iteration (same as the b200 arm)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": thr, "kind": "port",
                             "sample": f"{steps} hybrid iterations after {min(args.warmup, 1)} warm-up (bounded sample)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


C5_INSTANCES = 64


def c5_seeds(rank: int, world: int) -> list:
    """Rank r's share of the C5 batch: seeds r, r+N, ... (every seed exactly once)."""
    return list(range(rank, C5_INSTANCES, world))


def run_c5(args, rank, world, local_rank):
    """Config C5: a batch of 64 independent ~500-triangle pairs (the C3
    generator, seeds 0..63), instance-sharded over ranks (rank r solves
    seeds r, r+N, ...; no collective on the data path).  One step = the
    rank's share of the batch solved through qn.solve_batch (--streams
    concurrent solves) from the lowered HOST instances (device upload and every plan
    build included), --batch-iters hybrid iterations per instance; warm-up =
    W solves of the rank's first instance."""
    import torch

    from paper_2310_08230_b200 import _native
    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.qn import solve, solve_batch

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    seeds = c5_seeds(rank, world)
    insts = [build_instance("c3", args.seed + s) for s in seeds]
    cfg = SolveConfig(mode="hybrid", max_iterations=args.batch_iters, dual_tolerance=0.0)
    h2d = sum(sum(getattr(i.flat, k).nbytes for k in ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd",
                                                      "zero_t", "one_t", "proc_ptr", "proc_layers"))
              + i.costs.nbytes for i in insts)
    with ClockSampler(local_rank) as clk:
        time.sleep(1.0)
        for _ in range(args.warmup):
            solve(insts[0], cfg, device=dev)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        l0 = _native.launch_count
        clk.mark()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record()
        arcs = 0
        for _ in range(args.steps):
            res = solve_batch(insts, cfg, device=dev, concurrency=args.streams)
            arcs += sum(r.state.arc_updates for r in res)
        end.record()
        torch.cuda.synchronize()
        clk.mark()
    if world > 1:
        torch.distributed.barrier()
    ms = start.elapsed_time(end)
    total_arcs, max_ms = aggregate_work_time(arcs, ms, world, dev)
    n_inst, _ = aggregate_work_time(len(insts) * args.steps, ms, world, dev)
    if rank != 0:
        return None
    value = total_arcs / (max_ms / 1e3)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "instances_per_s": n_inst / (max_ms / 1e3),
        "config": {"workload": f"c5: batch of {C5_INSTANCES} independent pairs, each {WORKLOADS['c3']}; "
                               f"{args.batch_iters} hybrid iterations per instance from host arrays",
                   "parallelism": f"instance-sharded x{world} ({len(insts)} on rank 0), {args.streams} streams per GPU",
                   "l2": "each solve uploads its instance (inputs not L2-resident across steps)"},
        "gpu_launches": _native.launch_count - l0,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": sum(i.flat.num_layers * 8 for i in insts),
                "note": "the step is already end to end (host instances in, duals/bounds out)"},
        "clocks": clk.summary(),
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = (run_c5 if args.config == "c5" else run_b200)(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
