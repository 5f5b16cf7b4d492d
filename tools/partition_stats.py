"""Boundary-variable fraction of the diagram partition (partition.py) for
k = 2/4/8 on the benched instances (host tool): python tools/partition_stats.py c4 c2"""
import json
import sys

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.partition import plan_partition  # noqa: E402

out = {}
for cfg in sys.argv[1:] or ["c4"]:
    inst = build_instance(cfg, 0)
    for k in (2, 4, 8):
        p = plan_partition(inst, k)
        nodes = [int(x.table.num_nodes) for x in p.parts]
        out[f"{cfg}/k{k}"] = {"boundary_variables": p.boundary_variables,
                              "variables": p.variables_with_copies,
                              "boundary_fraction": round(p.boundary_fraction, 4),
                              "exchange_bytes_per_pass": 8 * p.slots,
                              "node_balance": round(max(nodes) / (sum(nodes) / k), 4)}
        print(cfg, k, out[f"{cfg}/k{k}"], file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
