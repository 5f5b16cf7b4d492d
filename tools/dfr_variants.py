"""CUDA-event times of the deferred-schedule kernels and their variants on a
benched config (GPU tool): python tools/dfr_variants.py c2"""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.dual import init_duals  # noqa: E402

import os

os.environ["DM_DFR_NP"] = "0"  # this state keeps interleaved tables; the node-parallel passes use st.F / st.B
inst = build_instance(sys.argv[1] if len(sys.argv) > 1 else "c2", 0, int(sys.argv[2]) if len(sys.argv) > 2 else 128)
st = init_duals(inst, device="cuda:0", schedule="deferred")
st.deferred_round(0.5)
dev = st.dev
lam0 = st.lam_d.clone()


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    st.lam_d.copy_(lam0)
    return round(a.elapsed_time(b) / reps * 1e3, 1)


bounds = st._bounds
out = {
    "fw_mm": t(lambda: dev.dfr_forward(0.5, st.lam_d, None, st.B_il, st.F_il, st.mbar, bounds)),
    "fw_sweep": t(lambda: dev.dfr_forward(0.0, st.lam_d, None, None, st.F_il, None, bounds)),
    "bw_mm_avg": t(lambda: dev.dfr_backward(0.5, st.lam_d, st.avg, st.F_il, st.B_il, st.mbar, bounds)),
    "bw_mm": t(lambda: dev.dfr_backward(0.5, st.lam_d, None, st.F_il, st.B_il, st.mbar, bounds)),
    "flush_dec": t(lambda: dev.dfr_backward(0.0, st.lam_d, st.avg, None, st.B_il, None, bounds, True)),
    "flush_nodec": t(lambda: dev.dfr_backward(0.0, st.lam_d, st.avg, None, st.B_il, None, bounds, False)),
    "sweep_dec": t(lambda: dev.dfr_backward(0.0, st.lam_d, None, None, st.B_il, None, bounds, True)),
    "sweep_nodec": t(lambda: dev.dfr_backward(0.0, st.lam_d, None, None, st.B_il, None, bounds, False)),
    "k_backward_nodes": t(lambda: dev.k_backward(st.lam_d, st.B, bounds)),
    "average": t(lambda: dev.dfr_average(st.mbar, st.avg)),
    "np_fw_mm": t(lambda: dev.dfr_np_forward(0.5, st.lam_d, None, st.B, st.F, st.mbar, bounds)),
    "np_bw_mm_avg": t(lambda: dev.dfr_np_backward(0.5, st.lam_d, st.avg, st.F, st.B, st.mbar, bounds)),
    "np_sweep_dec": t(lambda: dev.dfr_np_backward(0.0, st.lam_d, None, None, st.B, None, bounds, True)),
    "np_fw_sweep": t(lambda: dev.dfr_np_forward(0.0, st.lam_d, None, None, st.F, None, bounds)),
    "flush_apply": t(lambda: dev.dfr_flush(st.mbar, st.lam_d)),
}
print(json.dumps(out))
