"""Can independent instances share the GPU? Exact passes of K copies of the
C2 instance launched on K streams at once vs one after another (GPU tool)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, init_duals, mma_pass  # noqa: E402
from paper_2310_08230_b200.kernels import FlatBdds  # noqa: E402

inst = build_instance("c2", 0)
res = {}
for K, bps in ((1, 3), (2, 1), (3, 1), (2, 2)):
    states = []
    for k in range(K):
        inst._flat_dev = None
        st = init_duals(inst, device="cuda:0", flat=FlatBdds(inst))
        st.dev.set_mma_config(256, bps, 0, False, 1 << 16)
        states.append(st)
    streams = [torch.cuda.Stream() for _ in range(K)]
    for st, s in zip(states, streams):
        with torch.cuda.stream(s):
            mma_pass(st, FORWARD)
            mma_pass(st, BACKWARD)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    evs = []
    for st, s in zip(states, streams):
        s.wait_event(e0)
        with torch.cuda.stream(s):
            st.dev.k_mma_forward(st.lam_d, st.F, st.B, st._bounds)
            st.dev.k_mma_backward(st.lam_d, st.F, st.B, st._bounds)
            ev = torch.cuda.Event()
            ev.record(s)
            evs.append(ev)
    for ev in evs:
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    res[f"K{K}_bps{bps}"] = {"ms": ms, "ms_per_instance": ms / K}
    print(json.dumps(res), flush=True)
    del states
