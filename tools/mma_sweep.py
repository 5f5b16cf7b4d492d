"""Sweep the launch shape of the exact averaging passes on one instance and
check every configuration is bit-identical (GPU tool, not a test)."""

import hashlib
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, init_duals, mma_pass  # noqa: E402


def h(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    inst = build_instance(cfg, 0)
    st = init_duals(inst, device="cuda:0")
    for _ in range(2):
        mma_pass(st, FORWARD)
        mma_pass(st, BACKWARD)
    lam0, F0, B0 = st.lam_d.clone(), st.F.clone(), st.B.clone()
    results = []
    ref = None
    configs = []
    for threads, bps, sleep in ((256, 3, 32), (256, 3, 0), (256, 3, 16), (256, 3, 64), (256, 2, 32), (256, 4, 32),
                                (128, 4, 32), (128, 6, 32), (256, 2, 0), (256, 4, 0), (512, 1, 32), (512, 2, 32),
                                (256, 3, 32)):
        configs.append((threads, bps, sleep, 0, 1 << 16))
    for threads, bps, sleep, probe, look in configs:
        try:
            st.dev.set_mma_config(threads, bps, sleep, probe, look)
        except Exception as exc:  # occupancy limits
            results.append({"threads": threads, "bps": bps, "sleep": sleep, "probe": probe, "look": look, "error": str(exc)})
            continue
        times = []
        for rep in range(2):
            st.lam_d.copy_(lam0); st.F.copy_(F0); st.B.copy_(B0)
            st.f_valid, st.b_valid = False, True
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            st.dev.k_mma_forward(st.lam_d, st.F, st.B, st._bounds)
            e[1].record()
            st.dev.k_mma_backward(st.lam_d, st.F, st.B, st._bounds)
            e[2].record()
            torch.cuda.synchronize()
            st.dev.check_status()
            times.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
        key = h(st.lam_d)
        ref = ref or key
        fw, bw = min(t[0] for t in times), min(t[1] for t in times)
        r = {"threads": threads, "bps": bps, "sleep": sleep, "probe": probe, "look": look, "grid": st.dev.info["mma_grid"], "fw_ms": fw,
             "bw_ms": bw, "exact": key == ref}
        print(json.dumps(r), flush=True)
        results.append(r)
    info = st.dev.info
    print(json.dumps({"depth": [info["fw_depth"], info["bw_depth"]], "tasks": info["fw_tasks"]}))


if __name__ == "__main__":
    main()
