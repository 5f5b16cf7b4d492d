"""A/B of the exact passes' streaming-load hints (DM_MMA_HINTS bits: 1 copy
records, 2 arcs, 4 the static table) on a benched config: CUDA-event time of
a forward + backward pass from the same state, duals required identical."""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, init_duals, mma_pass  # noqa: E402

inst = build_instance(sys.argv[1] if len(sys.argv) > 1 else "c2", 0)
st = init_duals(inst, device="cuda:0")
for _ in range(2):
    mma_pass(st, FORWARD)
    mma_pass(st, BACKWARD)
lam0, B0 = st.lam_d.clone(), st.B.clone()
out = {}
for rep in range(2):
    for hints in (0, 1, 2, 4, 3, 7):
        os.environ["DM_MMA_HINTS"] = str(hints)
        fw, bw = [], []
        for _ in range(3):
            st.lam_d.copy_(lam0)
            st.B.copy_(B0)
            st.f_valid, st.b_valid = False, True
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record()
            mma_pass(st, FORWARD)
            b.record()
            mma_pass(st, BACKWARD)
            c.record()
            torch.cuda.synchronize()
            fw.append(a.elapsed_time(b))
            bw.append(b.elapsed_time(c))
        hsh = hashlib.sha256(st.lam_d.cpu().numpy().tobytes() + st.B.cpu().numpy().tobytes()).hexdigest()[:12]
        out.setdefault(hints, []).append({"fw_ms": round(min(fw), 3), "bw_ms": round(min(bw), 3), "hash": hsh})
print(json.dumps(out))
