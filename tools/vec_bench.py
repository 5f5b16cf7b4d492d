"""Timing of the L-BFGS vector kernels at the C2 dual length (GPU tool)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_08230_b200 import qn  # noqa: E402
from paper_2310_08230_b200.kernels import dev_axpy_dev, dev_dot, dev_sub  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 9402880
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10
torch.manual_seed(0)
dev = torch.device("cuda:0")
g = torch.randn(n, dtype=torch.float64, device=dev)
h = qn.LbfgsHistory(m)
for _ in range(m):
    s = torch.randn(n, dtype=torch.float64, device=dev)
    y = s * 1.5
    qn.update_history(s, y, h, qn.StepConfig())
out = torch.empty(1, dtype=torch.float64, device=dev)
a, b = torch.randn(n, dtype=torch.float64, device=dev), torch.randn(n, dtype=torch.float64, device=dev)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


res = {
    "n": n,
    "dot_us": timed(lambda: dev_dot(a, b, out)),
    "sub_us": timed(lambda: dev_sub(g, a, b)),
    "axpy_us": timed(lambda: dev_axpy_dev(g, a, 1.0, out)),
    "copy_us": timed(lambda: g.copy_(a)),
    "two_loop_fused_us": timed(lambda: qn.lbfgs_direction(g, h), 5),
    "two_loop_plain_us": timed(lambda: qn.lbfgs_direction(g, h, fused=False), 5),
}
res["dot_gbs"] = 16 * n / res["dot_us"] / 1e3
res["sub_gbs"] = 24 * n / res["sub_us"] / 1e3
print(json.dumps(res))
