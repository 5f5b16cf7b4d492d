"""Post-wait work latency of one exact-pass task without contention (GPU tool):
one 32-thread block runs every task of a small instance in level order, so
each task's inputs are already published when it starts.  Prints the
distribution of (outputs stored - group go) and (go - start)."""
import os
import sys

os.environ["DM_MMA_MAX_BLOCKS"] = "1"
os.environ["DM_MMA_THREADS"] = "32"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2310_08230_b200 import _native  # noqa: E402
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, init_duals, mma_pass  # noqa: E402
from paper_2310_08230_b200.ilp import IlpInstance  # noqa: E402
from tests.cases import product_space  # noqa: E402

p = product_space(sys.argv[1] if len(sys.argv) > 1 else "icosa", 0)
inst = IlpInstance.from_csr(p.costs, p.row_ptr, p.row_var, p.row_coef, p.row_rhs, 128)
st = init_duals(inst, device="cuda:0")
for forward, name in ((True, "forward"), (False, "backward")):
    mma_pass(st, FORWARD if forward else BACKWARD)
    ntask = st.dev.info["fw_tasks" if forward else "bw_tasks"]
    lpt = int(st.dev.info["lanes_per_task"])
    tr = torch.zeros(ntask * lpt * 6, dtype=torch.int64, device=st.device)
    _native.check(_native.load().dm_flat_set_trace(st.dev.handle, tr.data_ptr()))
    mma_pass(st, FORWARD if forward else BACKWARD)
    torch.cuda.synchronize()
    _native.check(_native.load().dm_flat_set_trace(st.dev.handle, None))
    t = tr.cpu().numpy().reshape(-1, 6)
    ok = t[:, 4] > 0
    work = (t[ok, 4] - t[ok, 2]).astype(np.float64)
    wait = (t[ok, 2] - t[ok, 0]).astype(np.float64)
    avg = (t[ok, 3] - t[ok, 2]).astype(np.float64)
    q = lambda x: [float(np.percentile(x, k)) for k in (10, 50, 90)]
    print(name, "tasks", ntask, "work p10/50/90", q(work), "go->lam", q(avg), "start->go", q(wait),
          "total ms", (t[ok, 4].max() - t[ok, 0].min()) / 1e6, flush=True)
