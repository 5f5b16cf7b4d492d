"""Exact-pass DAG depth of a product space under different variable orders
(host tool, CPU only): the forward pass's level of a variable is one more
than the deepest previous-layer variable over its diagrams (kernels.py:194-269
in visitation order), so the depth is the longest chain of the union of the
diagrams' variable chains.

usage: python tools/order_depth.py [config] [seed]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2310_08230_b200 import product_space as ps  # noqa: E402
from paper_2310_08230_b200.ilp import IlpInstance  # noqa: E402


def depth_of(flat) -> int:
    """Longest chain: levels by a DP over variables in visitation order."""
    lv = flat.layer_var
    bl = flat.bdd_layer_lo
    first = np.zeros(flat.num_layers, bool)
    first[bl[:-1]] = True
    # previous layer's variable in the same diagram (-1 for first layers)
    prev_var = np.where(first, -1, np.roll(lv, 1))
    order = flat.variable_order
    pos_of = np.empty(len(order), np.int64)
    pos_of[order] = np.arange(len(order))
    level = np.zeros(len(order), np.int64)
    ptr, lay = flat.proc_ptr, flat.proc_layers
    # visitation position k = variable order[k]; its copies proc_layers[ptr[k]:ptr[k+1]]
    pv = prev_var[lay]
    seg = np.repeat(np.arange(len(order)), np.diff(ptr))
    # process in position order: level[k] = 1 + max(level[pos(prev)]) — sequential DP by chunks
    best = np.zeros(len(order), np.int64)
    for k in range(len(order)):
        a, b = ptr[k], ptr[k + 1]
        m = 0
        for p in pv[a:b]:
            if p >= 0:
                q = level[pos_of[p]]
                if q + 1 > m:
                    m = q + 1
        level[k] = m
    del seg, best
    return int(level.max()) + 1


def instance(p, perm=None):
    if perm is None:
        return IlpInstance.from_csr(p.costs, p.row_ptr, p.row_var, p.row_coef, p.row_rhs, 128)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    return IlpInstance.from_csr(p.costs[perm], p.row_ptr, inv[p.row_var], p.row_coef, p.row_rhs, 128)


def greedy_colours(p, visit):
    """Smallest colour not used by an already coloured variable of any of the
    variable's rows, variables taken in `visit` order."""
    nv = p.num_variables
    var_rows = [[] for _ in range(nv)]
    for r in range(p.num_rows):
        for v in p.row_var[p.row_ptr[r]:p.row_ptr[r + 1]]:
            var_rows[v].append(r)
    used = [set() for _ in range(p.num_rows)]
    colour = np.empty(nv, np.int64)
    for v in visit:
        taken = set()
        for r in var_rows[v]:
            taken |= used[r]
        c = 0
        while c in taken:
            c += 1
        colour[v] = c
        for r in var_rows[v]:
            used[r].add(c)
    return colour



if __name__ == "__main__":
    config = sys.argv[1] if len(sys.argv) > 1 else "c4"
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    p = ps.synthetic_product_space(config, seed)
    lens = np.diff(p.row_ptr)
    print(f"{config}: {p.num_variables} vars, {p.num_rows} rows, longest row {lens.max()}, "
          f"rows > 128: {(lens > 128).sum()}", flush=True)
    t = time.perf_counter()
    inst = instance(p)
    print(f"colour order: depth {depth_of(inst.flat)}, max layers {inst.flat.max_layers} ({time.perf_counter() - t:.1f}s)",
          flush=True)
    for name, visit in (("greedy/colour order", np.arange(p.num_variables)),
                        ("greedy/reverse", np.arange(p.num_variables)[::-1]),
                        ("greedy/random", np.random.default_rng(0).permutation(p.num_variables))):
        t = time.perf_counter()
        col = greedy_colours(p, visit)
        perm = np.lexsort((np.arange(p.num_variables), col))
        inst2 = instance(p, perm)
        print(f"{name}: {col.max() + 1} colours, depth {depth_of(inst2.flat)} ({time.perf_counter() - t:.1f}s)", flush=True)
