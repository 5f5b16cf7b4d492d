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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ttg", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--e2e-iters", type=int, default=50)
    ap.add_argument("--schedule", choices=["exact", "deferred"], default="exact",
                    help="averaging schedule of the headline line (the other one is reported as an extra key)")
    ap.add_argument("--no-extras", action="store_true", help="headline only: no other-schedule / C4 / C5 keys")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--split", action="store_true", help="one instance's diagrams partitioned over the ranks (C4)")
    ap.add_argument("--c5-solver", choices=["hybrid", "averaging"], default="hybrid",
                    help="--config c5: every instance's own hybrid solve (batch.BatchedSolver) or fixed-length "
                         "averaging-only merged batches")
    ap.add_argument("--cpu-budget", type=float, default=300.0, help="wall budget (s) of a CPU time-to-gap run")
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


def build_instance(config: str, seed: int, chunk: int = 128):
    """The config's product space lowered with ``chunk``-layer splitting (the
    reference's default 128; 0 = unsplit)."""
    from paper_2310_08230_b200 import product_space as ps
    from paper_2310_08230_b200.ilp import IlpInstance

    t = time.perf_counter()
    p = ps.synthetic_product_space(config, seed)
    t1 = time.perf_counter()
    inst = IlpInstance.from_csr(p.costs, p.row_ptr, p.row_var, p.row_coef, p.row_rhs, chunk)
    t2 = time.perf_counter()
    log(f"[bench] {config} seed {seed}: product space {t1 - t:.1f}s, lowering {t2 - t1:.1f}s, "
        f"{inst.num_variables} vars, {inst.flat.num_bdds} bdds, {inst.flat.num_layers} layers, "
        f"{inst.flat.num_nodes} nodes")
    inst._rows_hash = rows_hash(p)
    inst._chunk = chunk
    return inst


def rows_hash(p) -> str:
    import hashlib

    m = hashlib.sha256()
    for a in (p.row_ptr, p.row_var, p.row_coef, p.row_rhs, p.costs):
        import numpy as np

        a = np.ascontiguousarray(a)
        m.update(a.dtype.str.encode() + a.tobytes())
    return m.hexdigest()[:32]


def oracle_instance(config: str, seed: int, chunk: int = 128):
    """The CPU arm's instance, lowered by the ORACLE's restatement of the
    reference pipeline (rows -> equality diagrams -> 128-chunk split -> flat
    table, oracle/model.py), so the reference arm never maps the product
    library; the lowering is golden-pinned against the real reference
    (tests/test_oracle_golden.py, tests/test_large_parity.py)."""
    from oracle import clib, model
    from paper_2310_08230_b200 import product_space as ps

    t = time.perf_counter()
    p = ps.synthetic_product_space(config, seed, colouring=clib.row_colouring)
    oi = model.instance_from_rows(p.costs, p.rows())
    if chunk:
        oi = model.split_instance(oi, chunk)
    of = model.flatten(oi)
    log(f"[bench] oracle lowering of {config} seed {seed}: {time.perf_counter() - t:.1f}s, {of.num_nodes} nodes")
    return oi, of, rows_hash(p)


def oracle_twin(inst):
    from oracle import model

    f = inst.flat
    arrays = {k: getattr(f, k) for k in ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd", "zero_t",
                                          "one_t", "proc_ptr", "proc_layers")}
    return model.from_flat_table(inst.costs, inst.variable_order, f.constraint_counts, arrays)


def _oracle_iterations(oi, of, schedule="exact"):
    """Generator form of oracle.solver.solve (qn.py:211-259), hybrid mode;
    yields (state, bound) after init and after every iteration."""
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
    yield st, first
    while True:
        it += 1
        if hist:
            g = st.subgradient()
            d = solver.project(solver.lbfgs(g, list(hist), solver._dot_blas), st)
            gamma, better = solver.step_search(st, d, gamma, 0.8, 1.1, 5, min_ascent)
            if better:
                st.shift(gamma * d)
        if schedule == "deferred":
            st.deferred_round(0.5)
        else:
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
        yield st, bound


def cpu_reference_run(oi, of, warmup: int, steps: int, d_star=None, gap=1e-3, budget_s=240.0, threads=None):
    """The reference algorithm (C port of the numba kernels + numpy driver,
    exact passes single-threaded as in the reference) on the host, from a
    fresh init: ``warmup`` untimed iterations, ``steps`` timed ones, then
    (if ``d_star`` is given) on until the relative gap to d_star is <= gap or
    the wall budget runs out.  Returns a dict: arc-updates/s and ms per
    iteration of the timed window, and the measured time to the gap (clock
    from init, the same definition as the GPU arm)."""
    from oracle.clib import lib

    threads = threads or os.cpu_count() or 1
    lib.oracle_set_threads(threads)
    t0 = time.perf_counter()
    gen = _oracle_iterations(oi, of)
    st, b = next(gen)
    hit = (0, 0.0) if d_star is not None and d_star - b <= gap * abs(d_star) else None
    it = 0
    s0 = tw0 = None
    out = {"threads": threads}
    while True:
        if it == warmup:
            s0, tw0 = st.sweeps, time.perf_counter()
        if it == warmup + steps:
            dt = time.perf_counter() - tw0
            out["value"] = (st.sweeps - s0) * 2 * of.num_nodes / dt
            out["ms_per_iteration"] = dt / steps * 1e3
            out["timed_iterations"] = f"{warmup + 1}..{warmup + steps}"
        done_timing = it >= warmup + steps
        if done_timing and (d_star is None or hit is not None or time.perf_counter() - t0 > budget_s):
            break
        st, b = next(gen)
        it += 1
        if d_star is not None and hit is None and d_star - b <= gap * abs(d_star):
            hit = (it, time.perf_counter() - t0)
    if d_star is not None:
        out["time_to_gap"] = {"value": hit[1] if hit else None, "iterations": hit[0] if hit else None,
                              "unit": "s", "gap": gap, "d_star": d_star, "measured": True,
                              "budget_s": budget_s, "iterations_run": it, "last_bound": b,
                              "clock": "host perf_counter from init_duals start (instance lowered)"}
    return out


DSTAR_PATH = os.path.join(ROOT, "profiles", "dstar.json")


def d_star_for(config: str, seed: int, rhash: str, chunk: int = 128):
    """Best known dual bound of the instance (profiles/dstar.json: long runs of
    both schedules on a B200, plus a certified primal where one exists), or
    None when the file has no entry for this exact instance (rows hash,
    split length)."""
    try:
        with open(DSTAR_PATH) as fh:
            table = json.load(fh)
    except (OSError, ValueError):
        return None
    e = table.get(f"{config}:{seed}" + ("" if chunk == 128 else f":chunk{chunk}"))
    if not e or e.get("rows_hash") != rhash:
        return None
    return e


def gpu_time_to_gap(inst, dev, schedule, d_star, gap=1e-3, max_iterations=None):
    """Measured time to a relative gap to d_star: qn.solve from init_duals on
    the resident instance (upload and plans outside the clock), host clock."""
    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.dual import init_duals
    from paper_2310_08230_b200.qn import solve

    st = init_duals(inst, device=dev, schedule=schedule)
    cfg = SolveConfig(mode="hybrid", mma_schedule=schedule,
                      max_iterations=max_iterations or (300 if schedule == "exact" else 1500))
    res = solve(inst, cfg, device=dev, state=st)
    hit = next((r for r in res.records if d_star is not None and d_star - r.dual_objective <= gap * abs(d_star)),
               None)
    return {"value": hit.time_s if hit else None, "iterations": hit.iteration if hit else None, "unit": "s",
            "gap": gap, "best_bound": res.best_bound, "solve_iterations": res.iterations, "stop": res.stop_reason,
            "ms_per_iteration_solve": res.records[-1].time_s / max(res.iterations, 1) * 1e3}, res


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


def _traffic(kernel, config="c2", schedule="exact"):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture summary of this config (profiles/traffic_<config>[_deferred].json,
    tools/ncu_summary.py), or None."""
    name = f"traffic_{config}" + ("_deferred" if schedule == "deferred" else "") + ".json"
    if config == "c2" and schedule == "exact":
        name = "traffic.json"
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as f:
            tr = json.load(f)
    except (OSError, ValueError):
        return None
    # the exact passes run their node-parallel instantiation when the instance allows it
    cands = [kernel.replace("mma_", "mma_np_"), kernel] if kernel.startswith("mma_") else [kernel]
    for cand in cands:
        if cand in tr:
            return tr[cand]
        for name, b in tr.items():
            if name.startswith(cand + "_kernel") or name.startswith(cand + "<"):
                return b
    return None


def algorithmic_bytes(flat):
    """Per-launch algorithmic HBM bytes of each timed kernel (DESIGN.md
    'Kernels, their bound, algorithmic bytes')."""
    N, L, nb = flat.num_nodes, flat.num_layers, flat.num_bdds
    P = len(flat.proc_ptr) - 1
    return {
        # exact passes: arcs 8 + own distance read 8 + target distance read 8 + produced distance 8 +
        # sentinel prime 8 per node; lam r/w 16 + task slot 8 + layer offset 4 per layer; bound 8 per diagram
        "mma": 40 * N + 28 * L + 8 * nb,
        # trial sweep: interleaved arcs 8 per node (next-layer distances stay in shared memory, no table
        # written); lam 8 + d 8 per layer; bound 8 + offsets 8 per diagram
        "backward_trial": 8 * N + 16 * L + 16 * nb,
        # deferred passes (interleaved tables): arcs 8 + opposite table read 8 + own table write 8 per node;
        # lam r/w 16 + escrow write 8 (+ average read 8, backward) per layer; bound 8 per diagram
        "dfr_forward": 24 * N + 24 * L + 8 * nb,
        "dfr_backward": 24 * N + 32 * L + 8 * nb,
        # segmented average: escrow read 8 + copy index 4 + average write 8 per layer; CSR offset 4 per variable
        "dfr_average": 20 * L + 4 * P,
        # flush (average applied to the duals): escrow read 8 + copy index 4 + lam r/w 16 per layer; 4 per variable
        "dfr_flush": 28 * L + 4 * P,
        # plain sweep after the flush: arcs 8 + table write 8 per node; lam 8 + decision word 8 per layer
        "dfr_sweep": 16 * N + 16 * L + 8 * nb,
    }


def _bytes_for(name, abytes):
    if name.startswith("mma"):
        return abytes["mma"]
    if name == "step_search":
        return abytes["backward_trial"]
    return abytes.get(name)


def timed_steps(args, inst, dev, schedule, world, rank, local_rank, clocks=True):
    """W untimed + K timed hybrid iterations (DualSolver.step, the loop body
    of qn.solve) of one schedule on the resident instance; CUDA-event timing
    on the launching stream, per-kernel event pairs for the roofline."""
    import torch

    from paper_2310_08230_b200 import _native
    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.dual import KernelTimer
    from paper_2310_08230_b200.qn import DualSolver

    cfg = SolveConfig(mode="hybrid", max_iterations=10**9, dual_tolerance=0.0, mma_schedule=schedule)
    run = DualSolver(inst, cfg, device=dev).start()
    st = run.state
    clk = ClockSampler(local_rank) if clocks else None
    if clk:
        clk.__enter__()
        time.sleep(1.0)  # nvidia-smi start-up outside the timed region
    for _ in range(args.warmup):
        run.step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    timer = KernelTimer()
    st.pass_timer = timer
    s0, l0 = st.sweeps, _native.launch_count
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clk:
        clk.mark()
    torch.cuda.synchronize()
    start.record()
    for _ in range(args.steps):
        run.step()
    end.record()
    torch.cuda.synchronize()
    if clk:
        clk.mark()
        clk.__exit__(None, None, None)
    if world > 1:
        torch.distributed.barrier()
    st.pass_timer = None
    ms = start.elapsed_time(end)
    arcs = (st.sweeps - s0) * 2 * st.flat.num_nodes
    total_arcs, max_ms = aggregate_work_time(arcs, ms, world, dev)
    kt = timer.summary()
    abytes = algorithmic_bytes(st.flat)
    hbm = _peaks().get("hbm_gbs", 6650.0)
    kernels = {}
    for name, k in kt.items():
        if name == "step_search":
            # one event pair around the device trial sequence: per-trial figures
            # over the trials that ran (sweep + bound sum + decision)
            trials = max(timer.counts.get("step_search_trials", 0), 1)
            k = dict(k, searches=k["launches"], launches=trials, avg_ms=k["total_ms"] / trials)
        bpl = _bytes_for(name, abytes)
        kernels[name] = dict(k, bytes_per_launch=bpl, share_of_step=k["total_ms"] / ms)
        if bpl:
            a = bpl / (k["avg_ms"] * 1e-3) / 1e9
            kernels[name].update(achieved_gbs=round(a, 1), frac=round(a / hbm, 4))
    return {"value": total_arcs / (max_ms / 1e3), "ms_per_iteration": max_ms / args.steps, "kernels": kernels,
            "launches": _native.launch_count - l0, "clocks": clk.summary() if clk else None, "state": st,
            "info": st.dev.info, "hbm": hbm}


def roofline_of(t, config, schedule):
    """Roofline object for the dominant kernel of a timed_steps result."""
    kernels = t["kernels"]
    dom = max(kernels, key=lambda n: kernels[n]["total_ms"]) if kernels else None
    if not dom or not kernels[dom].get("bytes_per_launch"):
        return None
    k = kernels[dom]
    roof = {"bound": "hbm", "kernel": dom, "achieved": k["achieved_gbs"], "peak": t["hbm"], "unit": "GB/s",
            "frac": k["frac"], "traffic": _traffic(dom, config, schedule),
            "algorithmic_bytes": k["bytes_per_launch"],
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if _peaks() else "fallback 6650 GB/s"}
    if dom.startswith("mma"):
        # the exact passes are bound by their dependency chain, not by bytes
        depth = t["info"]["fw_depth"] if dom == "mma_forward" else t["info"]["bw_depth"]
        ns = k["avg_ms"] * 1e6 / depth
        roof["critical_path"] = {"levels": depth, "ns_per_level": round(ns, 1), "visibility_floor_ns": VISIBILITY_NS,
                                 "frac": round(VISIBILITY_NS / ns, 4),
                                 "note": "per level >= one-way store->poll visibility between SMs (tools/pingpong.cu)"}
    return roof


def run_b200(args, rank, world, local_rank):
    import torch

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    inst = build_instance(args.config, args.seed + rank)
    sched = args.schedule
    t = timed_steps(args, inst, dev, sched, world, rank, local_rank)
    st, info = t["state"], t["info"]
    log(f"[bench] rank {rank}: exact-pass DAG depth fw {info['fw_depth']} bw {info['bw_depth']}, "
        f"{sched} schedule {t['ms_per_iteration']:.3f} ms/iteration")
    result = None
    if rank == 0:
        result = {
            "metric": METRIC, "value": t["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t["ms_per_iteration"], "ms_per_iteration": t["ms_per_iteration"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args.config) + f", 128-chunk split, one hybrid L-BFGS + {sched}-schedule "
                                                           "averaging iteration per step; one instance per GPU",
                       "schedule": sched, "variables": inst.num_variables, "bdds": st.flat.num_bdds,
                       "dual_coords": st.flat.num_layers, "nodes": st.flat.num_nodes,
                       "fw_depth": info["fw_depth"], "bw_depth": info["bw_depth"],
                       "l2": "working set > 126 MB L2 (no flush needed)" if st.flat.num_nodes > 4_000_000
                       else "working set partly L2-resident", "parallelism": f"instance-sharded x{world}"},
            "gpu_launches": t["launches"], "kernels": t["kernels"], "roofline": roofline_of(t, args.config, sched),
            "clocks": t["clocks"],
        }
    del t, st
    if world > 1:
        # scaling runs report the headline and the end-to-end number only
        # (rank 0's other extras would keep it busy for minutes after the
        # other ranks finished); e2e: every rank solves its own instance from
        # host buffers at the same time, whole-job work over the slowest rank
        if not args.no_e2e:
            torch.distributed.barrier()
            e = e2e_run(args, inst, dev, sched)
            total, max_ms = aggregate_work_time(e["value"] * e["seconds_per_step"], e["seconds_per_step"] * 1e3,
                                                world, dev)
            if rank == 0:
                e["value"] = total / (max_ms / 1e3)
                e["seconds_per_step"] = max_ms / 1e3
                e["ms_per_iteration"] = max_ms / max(args.e2e_iters, 1)
                e["h2d_bytes_per_step"] *= world  # every rank's instance (the per-rank figure is rank 0's)
                e["d2h_bytes_per_step"] *= world
                e["ranks"] = world
                result["e2e"] = e
        return result
    if rank != 0:
        return None
    if not args.no_extras:
        other = "deferred" if sched == "exact" else "exact"
        o = timed_steps(args, inst, dev, other, 1, 0, local_rank, clocks=False)
        result[other] = {"value": o["value"], "unit": UNIT, "ms_per_iteration": o["ms_per_iteration"],
                         "kernels": o["kernels"], "roofline": roofline_of(o, args.config, other),
                         "gpu_launches": o["launches"], "steps": args.steps, "warmup": args.warmup}
        del o
    if not args.no_ttg:
        result["time_to_gap"] = time_to_gap_both(inst, dev, args.config, args.seed)
        if args.config == "c2" and not args.no_extras:
            c4 = build_instance("c4", args.seed)
            result["c4"] = {"workload": workload("c4"), "nodes": c4.flat.num_nodes,
                            "time_to_gap": time_to_gap_both(c4, dev, "c4", args.seed)}
            del c4
            # the same C2 ILP lowered WITHOUT splitting (chunk_size 0): splitting is the
            # reference's default, but its chained pieces slow both schedules down here
            un = build_instance(args.config, args.seed, chunk=0)
            result["time_to_gap_unsplit"] = dict(time_to_gap_both(un, dev, args.config, args.seed),
                                                 nodes=un.flat.num_nodes, max_layers=int(un.flat.max_layers))
            del un
    if args.config == "c2" and not args.no_extras and not args.no_c5:
        result["c5"] = c5_summary(args, dev)
    if not args.no_e2e:
        result["e2e"] = e2e_run(args, inst, dev, sched)
    if args.batch > 1:
        result["batch"] = batch_run(args, inst, dev)
    if world == 1 and not args.no_cpu_baseline:
        oi, of = oracle_twin(inst)
        c = cpu_reference_run(oi, of, 1, args.cpu_iters)
        result["cpu_baseline"] = {"value": c["value"], "unit": UNIT, "cores": c["threads"], "kind": "port",
                                  "ms_per_iteration": c["ms_per_iteration"],
                                  "sample": f"{args.cpu_iters} hybrid iterations (exact schedule) of the same "
                                            f"{args.config} instance after 1 warm-up iteration; C port of the numba "
                                            "kernels, exact passes single-threaded as in the reference; the full "
                                            "measured CPU run (same steps, time to gap) is bench.py --impl reference"}
    return result


def time_to_gap_both(inst, dev, config, seed):
    """Measured time to a 1e-3 relative gap for both schedules, against the
    best known dual bound d* (profiles/dstar.json) or, without an entry for
    this instance, the best bound either solve reached."""
    e = d_star_for(config, seed, getattr(inst, "_rows_hash", ""), getattr(inst, "_chunk", 128))
    d_star = e["d_star"] if e else None
    out = {}
    runs = {}
    for s in ("exact", "deferred"):
        out[s], runs[s] = gpu_time_to_gap(inst, dev, s, d_star)
    if d_star is None:  # re-read the records against the better of the two runs
        d_star = max(r.best_bound for r in runs.values())
        for s, res in runs.items():
            hit = next((r for r in res.records if d_star - r.dual_objective <= 1e-3 * abs(d_star)), None)
            out[s]["value"] = hit.time_s if hit else None
            out[s]["iterations"] = hit.iteration if hit else None
        out["d_star_source"] = "best bound of the two solves in this run (no profiles/dstar.json entry)"
    else:
        out["d_star_source"] = e["source"]
    out["d_star"] = d_star
    out["clock"] = "host perf_counter from qn.solve start; instance resident, upload and plans outside the clock"
    return out


def e2e_run(args, inst, dev, schedule="exact"):
    """Same metric through the public API from HOST buffers: every step
    uploads the lowered instance (FlatBdds.device: topology + schedules),
    runs qn.solve for --e2e-iters iterations and reads the duals back."""
    import numpy as np
    import torch

    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.dual import init_duals
    from paper_2310_08230_b200.kernels import FlatBdds
    from paper_2310_08230_b200.qn import solve

    f = inst.flat
    h2d = sum(getattr(f, k).nbytes for k in ("bdd_layer_lo", "layer_node_lo", "layer_var", "zero_t", "one_t",
                                             "proc_ptr", "proc_layers")) + inst.costs.nbytes
    reps = []
    arcs = iters = 0
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        flat = FlatBdds(inst)
        state = init_duals(inst, device=dev, flat=flat, schedule=schedule)
        res = solve(inst, SolveConfig(mode="hybrid", max_iterations=args.e2e_iters, dual_tolerance=0.0,
                                      mma_schedule=schedule), device=dev, state=state)
        lam = res.state.lam  # D2H
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if rep:
            reps.append(dt)
            arcs, iters = res.state.arc_updates, res.iterations
        d2h = lam.nbytes + 8 * len(res.records)
        del flat, state, res
    sec = float(np.median(reps))
    return {"value": arcs / sec, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "seconds_per_step": sec, "ms_per_iteration": sec / max(iters, 1) * 1e3, "schedule": schedule,
            "step": f"qn.solve({args.e2e_iters} hybrid iterations) from host arrays incl. device upload + "
                    "schedule build + duals read back"}


def batch_run(args, inst, dev):
    """--batch K independent instances (seeds seed..seed+K-1) solved one after
    another vs through qn.solve_batch; same iteration count, duals identical."""
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
            "sequential_value": arcs / t_seq, "identical_to_sequential": same}


C5_INSTANCES = 64


def c5_instances(seeds):
    return [build_instance("c3", s) for s in seeds]


def c5_solve(insts, dev, schedule):
    """One C5 step: the batch merged into one block-diagonal instance
    (batch.py) from the lowered HOST tables — merge, upload, plans, the hybrid
    solve to the reference's stopping rule and the per-instance bounds read
    back, all inside the clock.  Returns (seconds, BatchResult)."""
    import torch

    from paper_2310_08230_b200.batch import solve_merged

    torch.cuda.synchronize()
    t = time.perf_counter()
    res = solve_merged(insts, SolveConfigC5(schedule), device=dev, per_instance_stop=False, reuse_buffers=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t, res


def c5_batched(insts, dev, schedule="exact"):
    """One C5 step, hybrid: every instance's OWN qn.solve (default config, the
    reference's stopping rule) side by side on one merged instance
    (batch.BatchedSolver: per-instance L-BFGS, step search and stopping;
    stopped instances compacted away) — bounds and duals bit-identical to
    separate solves.  Merge, upload, plans, the solves and the per-instance
    duals read back all inside the clock.  Returns (seconds, results, solver)."""
    import torch

    from paper_2310_08230_b200.batch import BatchedSolver
    from paper_2310_08230_b200.config import SolveConfig

    torch.cuda.synchronize()
    t = time.perf_counter()
    solver = BatchedSolver(insts, SolveConfig(mode="hybrid", mma_schedule=schedule), device=dev, reuse_buffers=True)
    res = solver.solve()
    torch.cuda.synchronize()
    return time.perf_counter() - t, res, solver


C5_ITERATIONS = {"exact": 25, "deferred": 100}


def SolveConfigC5(schedule):  # noqa: N802 - a config factory
    """Averaging-only merged batches of a fixed length (bit-identical per
    instance to separate solves of that length; the reference's 1e-10
    stall rule keeps averaging-only solves running long after the 1e-3 gap,
    so the line reports the length and the quality it reaches instead)."""
    from paper_2310_08230_b200.config import SolveConfig

    return SolveConfig(mode="mma-only", mma_schedule=schedule, max_iterations=C5_ITERATIONS[schedule],
                       dual_tolerance=-float("inf"))


def c5_summary(args, dev, reps=5):
    """Config C5 on this GPU (the default line's extra key): 64 independent
    ~500-triangle pairs solved as one merged instance; median of ``reps``
    repetitions after one warm-up, their spread, and each instance's bound
    against its own d* (the best bound of its separate converged solve)."""
    import numpy as np

    from paper_2310_08230_b200.qn import solve

    insts = c5_instances(range(args.seed, args.seed + C5_INSTANCES))
    out = {"workload": f"c5: {C5_INSTANCES} independent pairs, each {WORKLOADS['c3']}, solved as ONE merged "
                       "block-diagonal instance (batch.py) from the lowered host tables: merge, upload, plans, "
                       "solve and per-instance bounds inside the clock. 'hybrid': every instance's own hybrid solve "
                       "to the reference's stopping rule (BatchedSolver); 'exact'/'deferred': averaging-only solves "
                       "of a fixed length (per-instance duals bit-identical to separate solves of that length), "
                       "quality = each instance's relative gap to its separate converged hybrid solve"}
    import gc

    import torch

    from paper_2310_08230_b200.config import SolveConfig

    torch.cuda.synchronize()
    t = time.perf_counter()
    sep_bounds = []
    for i in insts:
        r = solve(i, SolveConfig(mode="hybrid"), device=dev)
        sep_bounds.append(r.bounds)
        del r
    torch.cuda.synchronize()
    t_sep = time.perf_counter() - t
    sep = [max(b) for b in sep_bounds]
    c5_batched(insts, dev)  # warm-up
    times = []
    res = None
    for _ in range(reps):
        del res
        gc.collect()
        torch.cuda.synchronize()
        sec, res, solver = c5_batched(insts, dev)
        times.append(sec)
    med = float(np.median(times))
    out["hybrid"] = {"workload": "every instance's own hybrid qn.solve (default SolveConfig, the reference's stopping "
                                 "rule) on one merged instance with per-instance L-BFGS / step search / stopping, "
                                 "stopped instances compacted away (batch.BatchedSolver), from host tables",
                     "instances_per_s": C5_INSTANCES / med, "seconds": med, "runs_s": times,
                     "spread": (max(times) - min(times)) / med,
                     "iterations_max": max(r.iterations for r in res),
                     "iterations_sum": int(sum(r.iterations for r in res)),
                     "compactions": solver.repacks,
                     "bit_identical_to_separate_solves": all(r.bounds == b for r, b in zip(res, sep_bounds)),
                     "separate_solves_one_after_another_s": t_sep}
    for schedule in ("exact", "deferred"):
        c5_solve(insts, dev, schedule)  # warm-up
        times = []
        res = None
        for _ in range(reps):
            del res  # the previous batch's device state is released outside the clock
            gc.collect()
            torch.cuda.synchronize()
            sec, res = c5_solve(insts, dev, schedule)
            times.append(sec)
        med = float(np.median(times))
        rel = [abs(b - d) / abs(d) for b, d in zip(res.bounds, sep)]
        out[schedule] = {"instances_per_s": C5_INSTANCES / med, "seconds": med, "runs_s": times,
                         "spread": (max(times) - min(times)) / med, "iterations": res.iterations,
                         "stop": res.merged.stop_reason, "max_rel_gap_to_separate_solves": max(rel),
                         "instances_within_1e-3": int(sum(r <= 1e-3 for r in rel))}
    return out


def run_split(args, rank, world, local_rank):
    """Config C4 split: ONE instance's diagrams partitioned over the ranks
    (partition.py: breadth-first slabs), deferred-schedule averaging rounds
    (mode "mma-only") with one NCCL allreduce of the boundary variables'
    escrow per pass and an all-gather of the per-diagram optima per round.
    One step = one round on every rank; bit-identical to the one-GPU solve
    (tests/test_partition.py).  "scaling": "strong" (total work fixed)."""
    import torch

    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.partition import DeviceEngine, DistComm, LoopbackComm, PartitionedSolver, plan_partition

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    inst = build_instance(args.config, args.seed)
    t = time.perf_counter()
    plan = plan_partition(inst, world)
    t_plan = time.perf_counter() - t
    part = plan.parts[rank]
    eng = DeviceEngine(part, dev)
    comm = DistComm([p.table.num_bdds for p in plan.parts]) if world > 1 else LoopbackComm()
    cfg = SolveConfig(mode="mma-only", mma_schedule="deferred", max_iterations=10**9, dual_tolerance=-float("inf"))
    run = PartitionedSolver(plan, [eng], comm, cfg).start()
    with ClockSampler(local_rank) as clk:
        time.sleep(1.0)
        for _ in range(args.warmup):
            run.step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        clk.mark()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(args.steps):
            run.step()
        end.record()
        torch.cuda.synchronize()
        clk.mark()
    if world > 1:
        torch.distributed.barrier()
    ms = start.elapsed_time(end)
    arcs = args.steps * 5 * 2 * part.table.num_nodes  # fw + bw passes (2 sweeps each) + the sweep
    total_arcs, max_ms = aggregate_work_time(arcs, ms, world, dev)
    # time to the 1e-3 gap of the split solve from init (stopping rule on), same d* as the other lines
    e = d_star_for(args.config, args.seed, inst._rows_hash)
    ttg = None
    if not args.no_ttg and e:
        res = PartitionedSolver(plan, [eng_fresh(part, dev)], comm,
                                SolveConfig(mode="mma-only", mma_schedule="deferred", max_iterations=3000)).solve()
        hit = next((i for i, b in enumerate(res.bounds) if e["d_star"] - b <= 1e-3 * abs(e["d_star"])), None)
        ttg = {"value": res.times[hit] if hit is not None else None, "iterations": hit, "unit": "s", "gap": 1e-3,
               "d_star": e["d_star"], "best_bound": res.best_bound, "stop": res.stop_reason,
               "solve_iterations": res.iterations}
    if rank != 0:
        return None
    return {
        "metric": METRIC, "value": total_arcs / (max_ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "ms_per_iteration": max_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(args.config) + f", diagrams split over {world} GPU(s) (partition.py), "
                                                       "deferred-schedule averaging rounds (mode mma-only)",
                   "boundary_fraction": round(plan.boundary_fraction, 4),
                   "exchange_bytes_per_pass": 8 * plan.slots, "plan_s": round(t_plan, 2),
                   "parallelism": f"diagram-partitioned x{world}"},
        "time_to_gap": ttg, "clocks": clk.summary(),
    }


def eng_fresh(part, dev):
    from paper_2310_08230_b200.partition import DeviceEngine

    return DeviceEngine(part, dev)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def run_reference(args, rank):
    """--impl reference: the reference algorithm (exact schedule, hybrid) on
    the host's cores through the C oracle port, on an instance lowered by the
    oracle's own restatement of the reference pipeline — the product library
    is never loaded (``native_so_loaded`` says so).  Same --steps / --warmup
    as the GPU arm (iterations W+1..W+K timed), then on to the measured time
    to the 1e-3 gap against the same d* as the GPU arm."""
    if rank != 0:
        return None
    config = "c3" if args.config == "c5" else args.config
    oi, of, rh = oracle_instance(config, args.seed)
    e = d_star_for(config, args.seed, rh)
    c = cpu_reference_run(oi, of, args.warmup, args.steps, d_star=e["d_star"] if e else None,
                          budget_s=args.cpu_budget)
    line = {"impl": "reference", "metric": METRIC, "value": c["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": c["ms_per_iteration"],
            "ms_per_iteration": c["ms_per_iteration"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(config) + ", 128-chunk split, one hybrid L-BFGS + exact-schedule "
                                                      "averaging iteration per step (the reference algorithm)",
                       "schedule": "exact", "timed_iterations": c["timed_iterations"]},
            "cpu_baseline": {"value": c["value"], "unit": UNIT, "cores": c["threads"], "kind": "port",
                             "sample": f"iterations {c['timed_iterations']} of a hybrid solve from init of the "
                                       f"{config} instance; C port of the numba kernels (exact passes single-"
                                       "threaded as in the reference, sweeps on all host threads), numpy/OpenBLAS "
                                       "driver"},
            "e2e": {"value": c["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if "time_to_gap" in c:
        line["time_to_gap"] = dict(c["time_to_gap"], d_star_source=e["source"])
    if config == "c2" and not args.no_extras and not args.no_ttg:
        oi4, of4, rh4 = oracle_instance("c4", args.seed)
        e4 = d_star_for("c4", args.seed, rh4)
        if e4:
            c4 = cpu_reference_run(oi4, of4, 0, 1, d_star=e4["d_star"], budget_s=args.cpu_budget)
            line["c4"] = {"workload": workload("c4"), "ms_per_iteration": c4["ms_per_iteration"],
                          "time_to_gap": dict(c4["time_to_gap"], d_star_source=e4["source"])}
        oiu, ofu, rhu = oracle_instance(config, args.seed, chunk=0)
        eu = d_star_for(config, args.seed, rhu, chunk=0)
        if eu:
            cu = cpu_reference_run(oiu, ofu, 0, 1, d_star=eu["d_star"], budget_s=args.cpu_budget)
            line["time_to_gap_unsplit"] = dict(cu["time_to_gap"], d_star_source=eu["source"],
                                               ms_per_iteration=cu["ms_per_iteration"])
    from paper_2310_08230_b200 import _native

    line["native_so_loaded"] = _native._lib is not None
    return line


C5_INSTANCES = 64


def c5_seeds(rank: int, world: int) -> list:
    """Rank r's share of the C5 batch: seeds r, r+N, ... (every seed exactly once)."""
    return list(range(rank, C5_INSTANCES, world))


def run_c5(args, rank, world, local_rank):
    """Config C5: a batch of 64 independent ~500-triangle pairs (the C3
    generator, seeds 0..63), instance-sharded over ranks (rank r solves
    seeds r, r+N, ...; no collective on the data path).  One step = the
    rank's share of the batch merged into one block-diagonal instance
    (batch.py) and solved from the lowered HOST tables (merge, device upload
    and every plan build included): by default every instance's own hybrid
    solve to the reference's stopping rule (--c5-solver hybrid,
    BatchedSolver), else fixed-length averaging-only batches; --schedule
    picks the averaging schedule; warm-up = W such solves."""
    import torch

    from paper_2310_08230_b200 import _native

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    seeds = c5_seeds(rank, world)
    insts = c5_instances([args.seed + s for s in seeds])
    h2d = sum(sum(getattr(i.flat, k).nbytes for k in ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd",
                                                      "zero_t", "one_t", "proc_ptr", "proc_layers"))
              + i.costs.nbytes for i in insts)
    with ClockSampler(local_rank) as clk:
        time.sleep(1.0)
        hybrid = args.c5_solver == "hybrid"

        def step():
            if hybrid:
                _, _, solver = c5_batched(insts, dev, args.schedule)
                return solver.arc_updates
            _, res = c5_solve(insts, dev, args.schedule)
            return res.merged.state.arc_updates

        for _ in range(args.warmup):
            step()
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
            arcs += step()
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
                               "merged per GPU and solved from host arrays: "
                               + ("every instance's own hybrid solve to the reference's stopping rule "
                                  "(BatchedSolver, bit-identical to separate solves)" if hybrid else
                                  f"averaging-only, {C5_ITERATIONS[args.schedule]} iterations")
                               + f" ({args.schedule} schedule)",
                   "parallelism": f"instance-sharded x{world} ({len(insts)} on rank 0), merged into one instance per GPU",
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
    fn = run_split if args.split else (run_c5 if args.config == "c5" else run_b200)
    out = fn(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
