"""Exact passes, refresh and one trial sweep on the C5 batch merged into one
instance (GPU tool): the throughput regime of the exact passes (wide, shallow DAG)."""
import sys, json, time
sys.path.insert(0, "."); sys.path.insert(0, "tools")
import torch
from bench import build_instance
from paper_2310_08230_b200.batch import merge_instances
from paper_2310_08230_b200.dual import init_duals, mma_pass, FORWARD, BACKWARD
insts = [build_instance("c3", s) for s in range(64)]
merged, idx = merge_instances(insts)
st = init_duals(merged, device="cuda:0")
for _ in range(2):
    mma_pass(st, FORWARD); mma_pass(st, BACKWARD)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
ev[0].record(); mma_pass(st, FORWARD); ev[1].record(); mma_pass(st, BACKWARD); ev[2].record()
st.refresh_backward(); ev[3].record()
d = torch.randn(merged.flat.num_layers, dtype=torch.float64, device="cuda:0") * 1e-3
st.dev.k_backward_trial(st.lam_d, d, 0.5, None, st._scratch_bounds); ev[4].record()
torch.cuda.synchronize()
info = st.dev.info
print(json.dumps({"nodes": merged.flat.num_nodes, "depth": [info["fw_depth"], info["bw_depth"]], "fw_ms": ev[0].elapsed_time(ev[1]), "bw_ms": ev[1].elapsed_time(ev[2]), "refresh_ms": ev[2].elapsed_time(ev[3]), "trial_ms": ev[3].elapsed_time(ev[4])}))
