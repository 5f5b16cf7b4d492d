"""Per-phase timing of dm_flat_create (GPU tool): DM_VERBOSE=2 prints the
phases; run twice in one process to separate first-call costs."""
import os
import sys
import time

os.environ.setdefault("DM_VERBOSE", "2")
import torch  # noqa: E402

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.kernels import FlatBdds  # noqa: E402
from paper_2310_08230_b200.dual import init_duals  # noqa: E402

inst = build_instance(sys.argv[1] if len(sys.argv) > 1 else "c2", 0)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inst._flat_dev = None
    st = init_duals(inst, device="cuda:0", flat=FlatBdds(inst))
    torch.cuda.synchronize()
    print(f"rep {rep}: init_duals {time.perf_counter() - t0:.3f}s", file=sys.stderr, flush=True)
    del st
