"""A/B timing of the exact passes across library builds (GPU tool).

usage: python tools/ab_mma.py <lib.so | KEY=VAL[,KEY=VAL]> ...   (each in a fresh process;
       KEY=VAL arguments run the in-tree library with those environment settings)
"""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, json, torch
sys.path.insert(0, ".")
from bench import build_instance
from paper_2310_08230_b200 import _native
from paper_2310_08230_b200.dual import init_duals, mma_pass, FORWARD, BACKWARD
inst = build_instance("c2", 0)
st = init_duals(inst, device="cuda:0")
for _ in range(2):
    mma_pass(st, FORWARD); mma_pass(st, BACKWARD)
res = []
for rep in range(3):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize(); e[0].record()
    st.dev.k_mma_forward(st.lam_d, st.F, st.B, st._bounds); e[1].record()
    st.dev.k_mma_backward(st.lam_d, st.F, st.B, st._bounds); e[2].record()
    torch.cuda.synchronize()
    res.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
d = torch.randn_like(st.lam_d)
bnd = torch.empty_like(st._bounds)
for _ in range(3):
    st.dev.k_backward_trial(st.lam_d, d, 0.37, None, bnd)
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize(); e[0].record()
for _ in range(20):
    st.dev.k_backward_trial(st.lam_d, d, 0.37, None, bnd)
e[1].record(); torch.cuda.synchronize()
trial_ms = e[0].elapsed_time(e[1]) / 20
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize(); e[0].record()
for _ in range(20):
    st.dev.k_backward(st.lam_d, st.B, bnd)
e[1].record(); torch.cuda.synchronize()
refresh_ms = e[0].elapsed_time(e[1]) / 20
print(json.dumps({"lib": os.environ.get("DM_LIB_PATH", os.environ.get("AB_SPEC")), "trial_ms": trial_ms, "refresh_ms": refresh_ms, "fw_ms": min(r[0] for r in res), "bw_ms": min(r[1] for r in res),
                  "lam_hash": __import__("hashlib").sha256(st.lam.tobytes()).hexdigest()[:16]}))
'''

for lib in sys.argv[1:]:
    if "=" in lib:
        env = dict(os.environ, AB_SPEC=lib, **dict(kv.split("=", 1) for kv in lib.split(",")))
    else:
        env = dict(os.environ, DM_LIB_PATH=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-2000:], flush=True)
