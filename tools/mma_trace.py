"""Per-level latency breakdown of the exact averaging passes (GPU tool).

Stamps (%globaltimer) per lane: task start, inputs seen, outputs published.
For every lane we find its producer (the copy at the previous layer of the
same diagram) and split the critical chain into
  comm  = inputs seen  - producer published
  work  = published    - inputs seen
"""

import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200 import _native  # noqa: E402
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, init_duals, mma_pass  # noqa: E402


def analyse(st, forward, trace, name):
    ntask = st.dev.info["fw_tasks" if forward else "bw_tasks"]
    lpt = int(st.dev.info.get("lanes_per_task", 32) or 32)
    levels = np.zeros(ntask, np.int32)
    layers = np.zeros(ntask * lpt, np.int32)
    _native.check(_native.load().dm_flat_task_levels(st.dev.handle, int(forward), levels.ctypes.data,
                                                    layers.ctypes.data))
    tr = trace.cpu().numpy().reshape(ntask * lpt, 6).astype(np.int64)
    act = layers >= 0
    t0 = tr[act, 0].min()
    start, own, seen, upd, done, issue = (tr[:, k] - t0 for k in range(6))
    issue = np.where(tr[:, 5] == 0, start, issue)
    own = np.where(tr[:, 1] == 0, start, own)  # lanes without dependencies are ready at start
    lane_level = np.repeat(levels, lpt)
    # producer lane of each lane: layer l-1 (forward) / l+1 (backward) in the same diagram
    f = st.flat
    L = f.num_layers
    slot_of_layer = np.full(L, -1, np.int64)
    slot_of_layer[layers[act]] = np.flatnonzero(act)
    layer_bdd = f.layer_bdd
    lo, hi = f.bdd_layer_lo[layer_bdd], f.bdd_layer_lo[layer_bdd + 1]
    l = layers.astype(np.int64)
    has_pred = act.copy()
    pred_layer = np.where(act, l - 1 if forward else l + 1, 0)
    if forward:
        has_pred &= l > lo[np.maximum(l, 0)]
    else:
        has_pred &= l + 1 < hi[np.maximum(l, 0)]
    pslot = np.where(has_pred, slot_of_layer[np.clip(pred_layer, 0, L - 1)], -1)
    waiting = has_pred.copy()
    waiting[has_pred] = start[has_pred] < done[pslot[has_pred]]
    comm = seen[waiting] - done[pslot[waiting]]
    comm_own = own[waiting] - done[pslot[waiting]]
    gate = seen[act] - own[act]
    work = done[act] - seen[act]
    wait_after_start = seen[act] - start[act]
    lv_done = np.zeros(levels.max() + 1, np.int64)
    np.maximum.at(lv_done, lane_level[act], done[act])
    per_level = np.diff(lv_done)
    q = lambda x: {k: float(np.percentile(x, p)) for k, p in (("p10", 10), ("p50", 50), ("p90", 90), ("max", 100))}
    out = {"pass": name, "levels": int(levels.max() + 1), "total_ns": int(done[act].max()),
           "ns_per_level_mean": float(done[act].max() / (levels.max() + 1)),
           "level_advance_ns": q(per_level), "comm_waiting_ns": q(comm), "own_visible_ns": q(comm_own), "group_gate_ns": q(gate), "work_ns": q(work),
           "average_ns": q(upd[act] - seen[act]), "publish_ns": q(done[act] - upd[act]),
           "seen_minus_start_ns": q(wait_after_start),
           "late_start_frac": float(np.mean(start[has_pred] > done[pslot[has_pred]]))}
    # critical chain: walk back from the last published lane
    var_of = np.where(act, f.layer_var[np.clip(l, 0, L - 1)], -1)
    nwarps = int(st.dev.info["mma_grid"] * st.dev.info["mma_block"] // 32)
    task_done = np.where(act, done, 0).reshape(-1, lpt).max(axis=1)
    seg = {"work": 0, "gate": 0, "comm": 0, "comm_to_issue": 0, "comm_poll_rtt": 0, "late_poll": 0, "warp_busy": 0}
    nseg = {k: 0 for k in seg}
    cur = int(np.flatnonzero(act)[np.argmax(done[act])])
    steps = 0
    while steps < 100000:
        steps += 1
        t = cur // lpt
        lanes = np.arange(t * lpt, t * lpt + lpt)
        grp = lanes[(var_of[lanes] == var_of[cur]) & act[lanes]]
        crit = int(grp[np.argmax(own[grp])])
        seg["work"] += done[cur] - seen[cur]; nseg["work"] += 1
        seg["gate"] += seen[cur] - own[crit]; nseg["gate"] += 1
        if has_pred[crit] and start[crit] < done[pslot[crit]]:
            seg["comm"] += own[crit] - done[pslot[crit]]; nseg["comm"] += 1
            seg["comm_to_issue"] += issue[crit] - done[pslot[crit]]; nseg["comm_to_issue"] += 1
            seg["comm_poll_rtt"] += own[crit] - issue[crit]; nseg["comm_poll_rtt"] += 1
            cur = int(pslot[crit])
        else:
            seg["late_poll"] += own[crit] - start[crit]; nseg["late_poll"] += 1
            prev = (cur // lpt) - nwarps
            if prev < 0:
                break
            seg["warp_busy"] += start[crit] - task_done[prev]; nseg["warp_busy"] += 1
            cur = int(prev * lpt + np.argmax(np.where(act[prev * lpt:prev * lpt + lpt], done[prev * lpt:prev * lpt + lpt], -1)))
    out["critical_chain"] = {k: {"total_ns": int(v), "n": nseg[k], "mean_ns": float(v / max(nseg[k], 1))}
                             for k, v in seg.items()}
    out["critical_chain_start_ns"] = int(start[cur])
    late = has_pred.copy()
    late[has_pred] = start[has_pred] > done[pslot[has_pred]]
    if late.any():
        out["late_by_ns"] = q(start[late] - done[pslot[late]])
        out["late_seen_after_start_ns"] = q(own[late] - start[late])
    print(json.dumps(out), flush=True)


def main():
    inst = build_instance(sys.argv[1] if len(sys.argv) > 1 else "c2", 0)
    st = init_duals(inst, device="cuda:0")
    for _ in range(2):
        mma_pass(st, FORWARD)
        mma_pass(st, BACKWARD)
    for forward, name in ((True, "forward"), (False, "backward")):
        ntask = st.dev.info["fw_tasks" if forward else "bw_tasks"]
        lpt = int(st.dev.info.get("lanes_per_task", 32) or 32)
        trace = torch.zeros(ntask * lpt * 6, dtype=torch.int64, device=st.device)
        _native.check(_native.load().dm_flat_set_trace(st.dev.handle, trace.data_ptr()))
        mma_pass(st, FORWARD if forward else BACKWARD)
        torch.cuda.synchronize()
        _native.check(_native.load().dm_flat_set_trace(st.dev.handle, None))
        analyse(st, forward, trace, name)


if __name__ == "__main__":
    main()
