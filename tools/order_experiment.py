"""GPU A/B of the variable order of a pruned product space: exact-pass times
and time to the 1e-3 gap (same ILP, variables renumbered by a greedy row
colouring).  usage: python tools/order_experiment.py [config] [seed]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from order_depth import depth_of, greedy_colours, instance  # noqa: E402
from paper_2310_08230_b200 import product_space as ps  # noqa: E402
from paper_2310_08230_b200 import qn  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, init_duals, mma_pass  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "c4"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dstar = {"c4": 381.2446921751127, "c3": 357.618154320663, "c2": 253.29775545409842}.get(config)
M, N, fm, fn = ps.synthetic_pair(config, seed)
k = ps.PRUNING_K.get(config)
p = ps.build_product_space(M, N, fm, fn, order="colour", allowed=ps.knn_allowed(fm, fn, k) if k else None)
col = greedy_colours(p, np.arange(p.num_variables))
perm = np.lexsort((np.arange(p.num_variables), col))
for name, inst in (("colour", instance(p)), ("greedy", instance(p, perm))):
    st = init_duals(inst, device="cuda:0")
    for _ in range(3):
        mma_pass(st, FORWARD)
        mma_pass(st, BACKWARD)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(5):
        mma_pass(st, FORWARD)
    ev[1].record()
    for _ in range(5):
        mma_pass(st, BACKWARD)
    ev[2].record()
    torch.cuda.synchronize()
    out = {"order": name, "depth": depth_of(inst.flat), "fw_ms": ev[0].elapsed_time(ev[1]) / 5,
           "bw_ms": ev[1].elapsed_time(ev[2]) / 5}
    del st
    for sched in (("exact",) if config == "c2" else ("exact", "deferred")):
        qn.solve(inst, SolveConfig(mma_schedule=sched, max_iterations=3), device="cuda:0")
        t = time.perf_counter()
        res = qn.solve(inst, SolveConfig(mma_schedule=sched), device="cuda:0")
        el = time.perf_counter() - t
        hit = next((r for r in res.records if dstar and (dstar - r.dual_objective) <= 1e-3 * abs(dstar)), None)
        out[sched] = {"ttg_s": hit.time_s if hit else None, "ttg_it": hit.iteration if hit else None,
                      "iters": res.iterations, "best": res.best_bound, "s": el}
    print(json.dumps(out), flush=True)
