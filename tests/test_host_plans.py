"""CPU checks of the two plans the device kernels execute:

* the numpy pairwise-summation tree (dm_host_pairwise_sum == np.sum), and
* the level schedule of the exact averaging passes: running the scheduled
  warp tasks in task order with the kernel's lane semantics reproduces the
  sequential reference pass bit-for-bit (dm_debug_emulate_mma vs oracle).
"""

import ctypes

import numpy as np
import pytest

from oracle import model, solver
from paper_2310_08230_b200 import _native
from tests.golden_util import case_inputs, load_cases

CASES = [c for c in load_cases() if c["name"] != "ps_c1"] + [c for c in load_cases() if c["name"] == "ps_c1"]


def host_sum(x):
    x = np.ascontiguousarray(x, np.float64)
    out = ctypes.c_double()
    _native.check(_native.load().dm_host_pairwise_sum(x.ctypes.data, len(x), ctypes.byref(out)))
    return out.value


@pytest.mark.parametrize("n", list(range(0, 270, 7)) + [1000, 4097, 8192, 65537, 636_800])
def test_pairwise_plan_matches_numpy(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 6, n)
    assert np.float64(host_sum(x)).tobytes() == np.sum(x).tobytes()


def test_pairwise_plan_signed_zero():
    for n in (1, 7, 8, 200):
        assert np.float64(host_sum(np.full(n, -0.0))).tobytes() == np.sum(np.full(n, -0.0)).tobytes()


def desc_of(flat):
    d = _native.FlatDesc()
    d.num_bdds, d.num_layers, d.num_nodes = flat.num_bdds, flat.num_layers, flat.num_nodes
    d.num_positions = len(flat.proc_ptr) - 1
    for k in ("bdd_layer_lo", "layer_node_lo", "layer_var", "zero_t", "one_t", "proc_ptr", "proc_layers"):
        setattr(d, k, getattr(flat, k).ctypes.data)
    return d


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_schedule_reproduces_sequential_passes(case):
    costs, rows, chunk = case_inputs(case)
    if not isinstance(rows, list):
        rows = rows.rows()
    inst = model.instance_from_rows(costs, rows)
    if chunk:
        inst = model.split_instance(inst, chunk)
    flat = model.flatten(inst)
    st = solver.init_duals(inst, flat)
    d = desc_of(flat)
    lib = _native.load()
    depth = ctypes.c_int64()
    for forward in (True, False, True, False):
        lam, F, B = st.lam.copy(), st.F.copy(), st.B.copy()
        bounds = np.zeros(flat.num_bdds)
        _native.check(lib.dm_debug_emulate_mma(ctypes.byref(d), int(forward), lam.ctypes.data, F.ctypes.data,
                                               B.ctypes.data, bounds.ctypes.data, ctypes.byref(depth)))
        st.mma(forward)
        assert lam.tobytes() == st.lam.tobytes()
        assert bounds.tobytes() == st.bounds.tobytes()
        if forward:
            assert F.tobytes() == st.F.tobytes()
        else:
            assert B.tobytes() == st.B.tobytes()
        assert 0 < depth.value <= len(flat.proc_ptr) - 1
