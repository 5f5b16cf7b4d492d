"""One deferred averaging round on a benched config, for ncu: the state is
initialised (one refresh sweep: dfr_backward_kernel), then exactly one round
runs (dfr_forward, dfr_average, dfr_backward, dfr_average, dfr_backward flush)
-> ncu -k regex:dfr_ -s 1 -c 5 python tools/dfr_round.py c2"""
import sys

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.dual import init_duals  # noqa: E402

inst = build_instance(sys.argv[1] if len(sys.argv) > 1 else "c2", 0)
st = init_duals(inst, device="cuda:0", schedule="deferred")
st.deferred_round(0.5)
torch.cuda.synchronize()
print("bound", st.bound)
